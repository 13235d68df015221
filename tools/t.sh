for envs in "" "VXG_NO_TC=1" "VXG_TILE_PAIR=0" "CUDA_LAUNCH_BLOCKING=1"; do
  echo "== $envs"; env $envs timeout 300 python -m pytest tests/test_gpu_primitives.py -x -q -k "fft_vs_direct_large" 2>&1 | grep -E "passed|failed|assert 0" | head -3
done > gpurun_out/t.txt 2>&1
