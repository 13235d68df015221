timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -5 > gpurun_out/pytest.log
for v in ${VARIANTS:-1}; do
  VXG_FWD_PIPE=$v timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/layer_kbench_$v.json 2>&1
done
[ -n "$NOBENCH" ] || timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw_cur.json 2>&1
