for y in 0 1; do for T in ${TS:-24 32}; do
 echo "T=$T ypair=$y"; VXG_YPAIR=$y VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 85 2>&1 | grep -A5 '"s"' | grep -E "tile_inv|tile_fwd|cgemm"
done; done > gpurun_out/variants.txt 2>&1
