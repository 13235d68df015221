timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest.log
VXG_TRACE=1 timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/sw_cur.json 2> gpurun_out/sw_cur.err
