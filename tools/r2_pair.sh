mkdir -p gpurun_out
TAG=${TAG:-pr1}
for T in 24 32; do
  VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 84 > gpurun_out/${TAG}_pair_T$T.json 2>&1
  VXG_TILE_PAIR=0 VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 84 > gpurun_out/${TAG}_single_T$T.json 2>&1
  VXG_INV_PAIR=0 VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 84 > gpurun_out/${TAG}_invsingle_T$T.json 2>&1
done
