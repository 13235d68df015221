mkdir -p gpurun_out
TAG=${TAG:-n726e}
VXG_TRACE=1 timeout 900 python bench.py --net n726 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench537.json 2> gpurun_out/${TAG}_bench537.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.txt 2>&1
