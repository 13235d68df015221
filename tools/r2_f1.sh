mkdir -p gpurun_out
TAG=${TAG:-f1a}
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_net.py -q -x -k "single_input or every_tile or bundled or measured_planner or conv_matches" > gpurun_out/${TAG}_pytest.txt 2>&1
for n in n926 n726; do
  timeout 900 python bench.py --net $n --no-cpu-baseline > gpurun_out/${TAG}_bench_$n.json 2> gpurun_out/${TAG}_bench_$n.err
done
