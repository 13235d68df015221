# Round evidence: bench line, ncu launch list of the same bench command, and
# --set full captures of the hot kernels on one deep 80->80 layer (kbench).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
# the normal run records its measured layer costs; the profiled runs replay
# them (under ncu launches are serialised, so measuring there would change the plan)
VXG_TUNE_SAVE=gpurun_out/${TAG}_tune.txt timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
export VXG_TUNE_FILE=gpurun_out/${TAG}_tune.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"cgemm_tc_kernel|tile_fwd_pair_kernel|tile_inv_pair_kernel" --launch-skip 3 --launch-count 3 \
  -o gpurun_out/${TAG}_layer -f python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_ncu_layer.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"mpf222_kernel|conv_direct_kernel|direct_tc_kernel" --launch-skip 1 --launch-count 3 \
  -o gpurun_out/${TAG}_small -f python tools/kbench.py --which direct,mpf --n 85 > gpurun_out/${TAG}_ncu_small.log 2>&1
ls -la gpurun_out
