mkdir -p gpurun_out
TAG=${TAG:-mc3}
VXG_TC_PROF=1 VXG_FFT_TILE=24 timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_T24.txt 2>&1
VXG_Q_NOMC=1 VXG_TC_PROF=1 VXG_FFT_TILE=24 timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_nomc_T24.txt 2>&1
VXG_TC_PAIR=1 VXG_FFT_TILE=24 timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_pair_T24.txt 2>&1
VXG_TC_PROF=1 VXG_FFT_TILE=32 timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_T32.txt 2>&1
VXG_Q_NOMC=1 VXG_TC_PROF=1 VXG_FFT_TILE=32 timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_nomc_T32.txt 2>&1
VXG_TRACE=1 VXG_FFT_TILE=24 timeout 300 python tools/kbench.py --which conv --S 64 --n 85 > gpurun_out/${TAG}_trace.txt 2>&1
