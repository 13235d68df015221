mkdir -p gpurun_out
TAG=${TAG:-q8}
for d in 0 32 0 32; do
  VXG_TC_DBG=$d VXG_FFT_TILE=32 timeout 300 python tools/kbench.py --which conv --n 256 --S 1 >> gpurun_out/${TAG}_dbg$d.txt 2>&1
done
VXG_TC_DBG=32 timeout 600 python -m pytest tests/test_gpu_primitives.py -q -k "match_ffma" > gpurun_out/${TAG}_pytest32.txt 2>&1
