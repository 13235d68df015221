import glob, json
for f in sorted(glob.glob("gpurun_out/sw_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"] / 1e6, 2), round(d["ms_per_step"]), "e2e", round(d["e2e"]["value"] / 1e6, 2),
              {k: round(v["seconds"] / d["steps"], 3) for k, v in d["kernels"].items()})
    except Exception:
        print(f, open(f).read().strip().splitlines()[-1][:200])
