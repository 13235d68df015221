mkdir -p gpurun_out
TAG=${TAG:-val1}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/${TAG}_pytest.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
