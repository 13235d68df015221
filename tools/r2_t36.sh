mkdir -p gpurun_out
TAG=${TAG:-t36}
timeout 900 python -m pytest tests/test_gpu_primitives.py -q -k "every_tile or match_ffma or pair_kernel_matches" > gpurun_out/${TAG}_pytest.txt 2>&1
