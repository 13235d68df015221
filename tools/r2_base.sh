# round-2 baseline on one box: smoke, GPU tests, one bench line
mkdir -p gpurun_out
TAG=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
nproc >> gpurun_out/${TAG}_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/${TAG}_pytest.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
