for v in "" 1; do for T in ${TS:-24}; do
 echo "T=$T fwdpair24=$v"; env ${v:+VXG_FWD_PAIR24=1} VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 85 2>&1 | grep -A5 '"s"' | grep -E "tile_inv|tile_fwd|cgemm"
done; done > gpurun_out/variants.txt 2>&1
