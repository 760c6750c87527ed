"""Per-kernel CUPTI breakdown (warm) of one conv pass.
    python scripts/kbreak.py N H W C K R S PAD STRIDE PASS [ALGO] [PREC]"""
import json
import os
import sys
import tempfile

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from launch_summary import kclass  # noqa: E402
from paper_1709_06622_b200 import device  # noqa: E402

a = sys.argv[1:]
n, h, w, c, k, r, s, pad, stride = (int(v) for v in a[:9])
pss = a[9]
algo = a[10] if len(a) > 10 else "gemm"
prec = a[11] if len(a) > 11 else "bf16"
g = device.geom(n, h, w, c, k, r, s, pad=pad, stride=stride)
plan = device.ConvPlan(g, algo, prec)
dt = plan.dtype
x = torch.randn(n, h, w, c, device="cuda").to(dt)
wt = (torch.randn(k, r, s, c, device="cuda") * 0.05).to(dt)
dy = torch.randn(n, g.ho, g.wo, k, device="cuda").to(dt)
fn = {"fwd": lambda: plan.fwd(x, wt), "dgrad": lambda: plan.dgrad(dy, wt), "wgrad": lambda: plan.wgrad(dy, x)}[pss]
for _ in range(3):
    fn()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
path = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
os.unlink(path)
cls = {}
for e in ev:
    kc = kclass(e["name"])
    cls[kc] = round(cls.get(kc, 0.0) + e["dur"] / 5, 1)
print(json.dumps({"pass": pss, "geom": g.as_dict(), "us_per_call": cls}))
