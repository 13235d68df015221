# ncu --set full of the three FFT-conv kernels on one 80->80 k5 layer
# (kbench conv: S entries of n^3), skipping the warm-up call.
set -x
mkdir -p gpurun_out
TAG=${TAG:-layer}
S=${S:-64}; N=${N:-85}
timeout 300 python tools/kbench.py --which conv --S $S --n $N > gpurun_out/${TAG}_kbench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-cgemm_tc_kernel|tile_fwd_kernel|tile_inv_kernel}" --launch-skip 3 --launch-count 3 \
  -o gpurun_out/${TAG} -f python tools/kbench.py --which conv --S $S --n $N > gpurun_out/${TAG}_ncu.log 2>&1
