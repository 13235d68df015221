VXG_TC_PROF=1 timeout 120 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/tcprof.txt 2>&1
