mkdir -p gpurun_out
TAG=${TAG:-slow2}
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
    print(i, {k: round(s["seconds"] * 1e3, 2) for k, s in ks.items()}, flush=True)
    del y
PY
VXG_TC_PROF=1 T=24 timeout 300 python /tmp/loop.py > gpurun_out/${TAG}_quad24.txt 2>&1
VXG_TC_PROF=1 T=32 timeout 300 python /tmp/loop.py > gpurun_out/${TAG}_quad32.txt 2>&1
