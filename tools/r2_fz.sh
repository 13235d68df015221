mkdir -p gpurun_out
TAG=${TAG:-rc1}
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_net.py -q -x -k "recombine or fused or bundled or golden or tiled" > gpurun_out/${TAG}_pytest.txt 2>&1
timeout 900 python bench.py --net n726 --no-cpu-baseline > gpurun_out/${TAG}_bench_n726.json 2> gpurun_out/${TAG}_bench_n726.err
