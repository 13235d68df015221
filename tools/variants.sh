for v in ${PAIRS:-0 1}; do for T in ${TS:-30 32}; do
 echo "T=$T invpair=$v"; VXG_INV_PAIR=$v VXG_FFT_TILE=$T timeout 300 python tools/kbench.py --which conv --S 64 --n 85 2>&1 | grep -A5 '"s"' | grep -E "tile_inv|tile_fwd"
done; done > gpurun_out/variants.txt 2>&1
