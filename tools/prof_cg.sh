timeout 600 ncu --set full --import-source on -k regex:cgemm_tc_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/cg -f python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/cg.log 2>&1
