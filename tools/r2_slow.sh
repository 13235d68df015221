mkdir -p gpurun_out
TAG=${TAG:-slow3}
cat > /tmp/loop.py <<'PY'
import sys, os, time
sys.path.insert(0, '.')
import torch, paper_1606_05688_b200 as v
ctx = v.Context(0)
g = torch.Generator(device="cuda").manual_seed(1)
n, S = 85, 64
x = torch.rand((S, 80, n, n, n), device="cuda", generator=g) * 2 - 1
w = (torch.rand((80, 80, 5, 5, 5), device="cuda", generator=g) * 2 - 1) * 0.02
b = torch.rand((80,), device="cuda", generator=g) * 0.2 - 0.1
p = v.ConvLayerParams(w, b, "relu")
T = int(os.environ.get("T", "24"))
for i in range(6):
    ctx.profile(True)
    y = v.conv_fft_tiled(x, p, T, tensor_cores=True, ctx=ctx)
    ctx.sync()
    ks = ctx.kernel_stats()
    ctx.profile(False)
    print(i, {k: (s["launches"], round(s["seconds"] * 1e3, 2)) for k, s in ks.items()}, flush=True)
    del y
PY
T=24 timeout 300 python /tmp/loop.py > gpurun_out/${TAG}_full.txt 2>&1
VXG_MAX_ROWS=2000 T=24 timeout 300 python /tmp/loop.py > gpurun_out/${TAG}_cap2000.txt 2>&1
VXG_MAX_ROWS=1024 T=24 timeout 300 python /tmp/loop.py > gpurun_out/${TAG}_cap1024.txt 2>&1
VXG_TC_PAIR=1 T=24 timeout 300 python /tmp/loop.py > gpurun_out/${TAG}_pair.txt 2>&1
