# ncu evidence for the bench workload: launch list (per-launch durations) and
# one --set full capture of each hot kernel.  Run through gpurun.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"cgemm_tc_kernel|tile_fwd_kernel|tile_inv_kernel|mpf222_kernel|conv_direct_kernel" \
  --launch-skip 40 --launch-count 8 -o gpurun_out/${TAG}_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out
