# end-of-round evidence on one box: smoke, GPU tests, bench + ncu (gpu_prof.sh), reference arm
mkdir -p gpurun_out
TAG=${TAG:-r1d}
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/${TAG}_pytest.txt
TAG=$TAG bash tools/gpu_prof.sh > gpurun_out/${TAG}_prof.log 2>&1
[ -n "$NOREF" ] || timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
