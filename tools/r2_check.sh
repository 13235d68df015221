# round-2 check on one box: smoke, GPU tests, bench line, reference arm
mkdir -p gpurun_out
TAG=${TAG:-r2b}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.txt 2>&1
[ -n "$NOBENCH" ] || timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
[ -n "$NOREF" ] || timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
