set -x
mkdir -p gpurun_out
rm -f gpurun_out/sw_*
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest.log
VXG_TRACE=1 timeout 300 python tools/kbench.py --which net --extent ${TRACE_E:-714} > gpurun_out/trace.json 2> gpurun_out/trace.err
for R in ${ROWS:-256 1024}; do for E in ${EXTENTS:-714 650}; do
 VXG_FFT_ROWS=$R timeout 300 python bench.py --extent $E --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw_${R}_${E}.json 2>&1
done; done
