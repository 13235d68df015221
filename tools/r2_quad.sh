mkdir -p gpurun_out
TAG=${TAG:-bf3}
timeout 900 python -m pytest tests/test_gpu_primitives.py -q -x -k "tensor_core or every_tile or pair_tile or match_ffma or conv_matches or fused" > gpurun_out/${TAG}_pytest.txt 2>&1
for T in 32 24; do
  VXG_TC_PROF=1 VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_T$T.txt 2>&1
  VXG_Q_3TF32=1 VXG_TC_PROF=1 VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_3tf_T$T.txt 2>&1
done
