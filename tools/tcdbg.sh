for d in 0 8 16 24; do echo "dbg $d"; VXG_TC_DBG=$d timeout 120 python tools/kbench.py --which conv --S 64 --n 85 2>&1 | grep -A4 kernels | grep cgemm; done > gpurun_out/tcdbg.txt
