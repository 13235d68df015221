timeout 600 python -m pytest tests -m gpu -x -q -k "single_input_map or bundled" 2>&1 | tail -3 > gpurun_out/dtc_pytest.txt
for d in 0 1; do VXG_DIRECT_TC=$d timeout 300 python tools/kbench.py --which direct > gpurun_out/dtc_k$d.txt 2>&1; done
