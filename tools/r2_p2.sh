mkdir -p gpurun_out
TAG=${TAG:-p2a}
VXG_PAIR2=1 timeout 900 python -m pytest tests/test_gpu_primitives.py -q -x -k "every_tile or fused or conv_matches or pair_kernel or match_ffma or tensor_core" > gpurun_out/${TAG}_pytest.txt 2>&1
for T in 32 24; do
  VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 84 > gpurun_out/${TAG}_base_T$T.json 2>&1
  VXG_PAIR2=1 VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 84 > gpurun_out/${TAG}_p2_T$T.json 2>&1
done
