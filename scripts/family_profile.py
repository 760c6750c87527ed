"""One fwd / dgrad / wgrad of the Winograd and FFT families (and the GEMM
for reference) on BASELINE layer shapes, plus the fused momentum-SGD over a
ResNet-50-sized shard, for `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum` launch lists (HBM GB/s of every
transform). Without ncu it prints CUDA-event times.
    python scripts/family_profile.py [reps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_06622_b200 import device  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
CASES = [("alexnet_conv3", (256, 13, 13, 256, 384, 3, 3, 1)),
         ("resnet50_s3_3x3", (256, 14, 14, 256, 256, 3, 3, 1)),
         ("alexnet_conv2_5x5", (256, 27, 27, 96, 256, 5, 5, 2))]
out = []
for name, (n, h, w, c, k, r, s, pad) in CASES:
    g = device.geom(n, h, w, c, k, r, s, pad=pad)
    x = torch.randn(n, h, w, c, device="cuda").bfloat16()
    wt = (torch.randn(k, r, s, c, device="cuda") * 0.05).bfloat16()
    dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
    for algo in ("gemm", "winograd", "fft"):
        try:
            plan = device.ConvPlan(g, algo, "bf16")
        except device.Unsupported:
            continue
        row = {"layer": name, "algo": algo}
        for pname, fn in (("fwd", lambda: plan.fwd(x, wt)), ("dgrad", lambda: plan.dgrad(dy, wt)),
                          ("wgrad", lambda: plan.wgrad(dy, x))):
            fn()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(reps):
                fn()
            s1.record()
            s1.synchronize()
            row[pname + "_ms"] = round(s0.elapsed_time(s1) / reps, 4)
        out.append(row)
        del plan
# momentum SGD over a ResNet-50-sized flat buffer (25.5M fp32 params + bf16 refresh)
npar = 25_503_936
wv, gv, vv = (torch.randn(npar, device="cuda") for _ in range(3))
wc = torch.empty(npar, dtype=torch.bfloat16, device="cuda")
device.sgd_momentum(wv, gv, vv, 0.01, 0.9, 0.0, 1.0, w_compute=wc)
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(reps):
    device.sgd_momentum(wv, gv, vv, 0.01, 0.9, 0.0, 1.0, w_compute=wc)
s1.record()
s1.synchronize()
out.append({"layer": "sgd_resnet50_flat", "params": npar, "ms": round(s0.elapsed_time(s1) / reps, 4),
            "algorithmic_bytes": npar * 22})
if "--cupti" in sys.argv:
    # warm per-kernel breakdown of one fwd / dgrad / wgrad per (layer, algo) from CUPTI
    import os
    import tempfile
    from torch.profiler import ProfilerActivity, profile
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from launch_summary import kclass  # noqa: E402
    brk = {}
    for name, (n, h, w, c, k, r, s, pad) in CASES:
        g = device.geom(n, h, w, c, k, r, s, pad=pad)
        x = torch.randn(n, h, w, c, device="cuda").bfloat16()
        wt = (torch.randn(k, r, s, c, device="cuda") * 0.05).bfloat16()
        dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
        for algo in ("winograd", "fft"):
            try:
                plan = device.ConvPlan(g, algo, "bf16")
            except device.Unsupported:
                continue
            for pname, fn in (("fwd", lambda: plan.fwd(x, wt)), ("dgrad", lambda: plan.dgrad(dy, wt)),
                              ("wgrad", lambda: plan.wgrad(dy, x))):
                fn()
                torch.cuda.synchronize()
                with profile(activities=[ProfilerActivity.CUDA]) as prof:
                    fn()
                    torch.cuda.synchronize()
                path = tempfile.mktemp(suffix=".json")
                prof.export_chrome_trace(path)
                ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
                os.unlink(path)
                cls = {}
                for e in ev:
                    kc = kclass(e["name"])
                    cls[kc] = round(cls.get(kc, 0.0) + e["dur"], 1)
                brk[f"{name}/{algo}/{pname}"] = cls
    out.append({"cupti_breakdown_us": brk})
print(json.dumps(out, indent=1))
