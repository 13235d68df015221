"""PCIe copy bandwidth of pinned host <-> device copies (one stream vs split across streams)."""
import time
import torch
n = 4 << 30  # 4 GiB
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
def run(dir_, parts):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    chunk = (n // 4) // parts
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            if dir_ == "d2h":
                h[i * chunk:(i + 1) * chunk].copy_(d[i * chunk:(i + 1) * chunk], non_blocking=True)
            else:
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize()
    return n / (time.perf_counter() - t0) / 1e9
for dir_ in ("d2h", "h2d"):
    for parts in (1, 2, 4):
        run(dir_, parts)
        print(dir_, parts, "streams: %.1f GB/s" % max(run(dir_, parts) for _ in range(3)), flush=True)
