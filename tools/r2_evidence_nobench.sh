# Round-2 evidence on one box: smoke, GPU tests, headline bench (+ its ncu launch
# list), --set full captures of the hot kernels, the other BASELINE configs,
# and the reference arm.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2z}


VXG_TUNE_SAVE=gpurun_out/${TAG}_tune.txt timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
export VXG_TUNE_FILE=gpurun_out/${TAG}_tune.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_bench.log 2>&1
unset VXG_TUNE_FILE
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"cgemm_q_kernel|tile_fwd_pair_kernel|tile_inv_pair_kernel" --launch-skip 3 --launch-count 3 \
  -o gpurun_out/${TAG}_layer -f python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_ncu_layer.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"mpf222_kernel|direct_tc_kernel|recombine_kernel" --launch-skip 1 --launch-count 3 \
  -o gpurun_out/${TAG}_small -f python tools/kbench.py --which direct,mpf --n 85 > gpurun_out/${TAG}_ncu_small.log 2>&1
VXG_FFT_TILE=32 timeout 300 python tools/kbench.py --which conv --n 256 --S 1 > gpurun_out/${TAG}_c2_T32.json 2>&1
for n in n726 n926 n337; do
  timeout 900 python bench.py --net $n --no-cpu-baseline > gpurun_out/${TAG}_bench_$n.json 2> gpurun_out/${TAG}_bench_$n.err
done
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
ls -la gpurun_out
