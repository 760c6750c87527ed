"""Time (or profile under ncu) one conv pass of one layer geometry.

    python scripts/conv_bench.py N H W C K R S PAD STRIDE PASS [REPS] [ALGO] [PREC]

PASS in fwd|dgrad|wgrad. Prints one JSON line with ms and TFLOP/s
(algorithmic 2*N*Ho*Wo*K*C*R*S per pass).
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_06622_b200 import device  # noqa: E402


def main():
    a = sys.argv[1:]
    n, h, w, c, k, r, s, pad, stride = (int(v) for v in a[:9])
    pss = a[9]
    reps = int(a[10]) if len(a) > 10 else 20
    algo = a[11] if len(a) > 11 else "gemm"
    prec = a[12] if len(a) > 12 else "bf16"
    g = device.geom(n, h, w, c, k, r, s, pad=pad, stride=stride)
    plan = device.ConvPlan(g, algo, prec)
    dt = plan.dtype
    x = torch.randn(n, h, w, c, device="cuda").to(dt)
    wt = (torch.randn(k, r, s, c, device="cuda") * 0.05).to(dt)
    dy = torch.randn(n, g.ho, g.wo, k, device="cuda").to(dt)
    fn = {"fwd": lambda: plan.fwd(x, wt), "dgrad": lambda: plan.dgrad(dy, wt),
          "wgrad": lambda: plan.wgrad(dy, x)}[pss]
    for _ in range(3):
        fn()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record()
    for _ in range(reps):
        fn()
    s1.record()
    s1.synchronize()
    ms = s0.elapsed_time(s1) / reps
    flop = 2.0 * n * g.ho * g.wo * k * c * r * s
    print(json.dumps({"geom": g.as_dict(), "pass": pss, "algo": algo, "prec": prec, "ms": ms,
                      "tflops": flop / ms / 1e9, "workspace_bytes": plan.workspace_bytes}))


if __name__ == "__main__":
    main()
