mkdir -p gpurun_out
TAG=${TAG:-cap1}
timeout 900 python -m pytest tests/test_gpu_primitives.py -q -x -k "budget or tensor_core or match_ffma or conv_matches or large" > gpurun_out/${TAG}_pytest.txt 2>&1
for n in n926 n726 n537; do
  timeout 900 python bench.py --net $n --no-cpu-baseline > gpurun_out/${TAG}_bench_$n.json 2> gpurun_out/${TAG}_bench_$n.err
done
