timeout 900 python -m pytest tests -m gpu -x -q -k "direct or bundled or toy or bench_patch or conv_matches or random_vs" 2>&1 | tail -15 > gpurun_out/dtc_pytest.txt
for d in 0 1; do VXG_DIRECT_TC=$d timeout 300 python tools/kbench.py --which direct --n 85 > gpurun_out/dtc_k$d.txt 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dtc_bench.json 2> gpurun_out/dtc_bench.err
