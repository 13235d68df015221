# full check: smoke, GPU tests, bench lines for the bundled nets
mkdir -p gpurun_out
TAG=${TAG:-r2i}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/${TAG}_pytest.txt 2>&1
VXG_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
for n in ${NETS:-n726 n926}; do
  timeout 900 python bench.py --net $n --no-cpu-baseline > gpurun_out/${TAG}_bench_$n.json 2> gpurun_out/${TAG}_bench_$n.err
done
