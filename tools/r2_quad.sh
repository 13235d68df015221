mkdir -p gpurun_out
TAG=${TAG:-q7}
timeout 900 python -m pytest tests/test_gpu_primitives.py -q -x -k "tensor_core or every_tile or pair_tile or conv_matches or random_vs" > gpurun_out/${TAG}_pytest.txt 2>&1
for d in 0 2; do
  VXG_TC_DBG=$d VXG_TC_PROF=1 VXG_FFT_TILE=32 timeout 300 python tools/kbench.py --which conv --n 256 --S 1 > gpurun_out/${TAG}_dbg$d.txt 2>&1
done
VXG_FFT_TILE=24 timeout 300 python tools/kbench.py --which conv --n 256 --S 1 > gpurun_out/${TAG}_T24.json 2>&1
