mkdir -p gpurun_out
TAG=${TAG:-nx1}
timeout 600 python tools/pcie_bw.py > gpurun_out/${TAG}_pcie.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_net.py -q > gpurun_out/${TAG}_pytest_net.txt 2>&1
timeout 300 python tools/kbench.py --which conv --n 256 --S 1 > gpurun_out/${TAG}_c2_auto.json 2>&1
for n in n726 n537; do
  timeout 900 python bench.py --net $n --no-cpu-baseline > gpurun_out/${TAG}_bench_$n.json 2> gpurun_out/${TAG}_bench_$n.err
done
