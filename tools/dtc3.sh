VXG_DIRECT_TC_MIN=16 timeout 600 python -m pytest tests -m gpu -x -q -k "single_input_map or bundled or toy or conv_matches or random_vs" 2>&1 | tail -3 > gpurun_out/dtc3_pytest16.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "single_input_map" 2>&1 | tail -3 > gpurun_out/dtc3_pytest.txt
for d in 0 1; do VXG_DIRECT_TC=$d timeout 300 python tools/kbench.py --which direct > gpurun_out/dtc3_k$d.txt 2>&1; done
VXG_DIRECT_TC_MIN=16 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dtc3_bench16.json 2> gpurun_out/dtc3_bench16.err
