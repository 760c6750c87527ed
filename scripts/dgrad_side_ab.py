"""Time one conv dgrad with / without the fused ReLU mask and residual-gradient
side inputs (the executor's in-step form), for epilogue A/B runs:

    TCB_EPI_STAGE=0|1 python scripts/dgrad_side_ab.py N H W C K R PAD STRIDE
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_06622_b200 import device  # noqa: E402


def main():
    n, h, w, c, k, r, pad, stride = (int(v) for v in sys.argv[1:9])
    g = device.geom(n, h, w, c, k, r, pad=pad, stride=stride)
    plan = device.ConvPlan(g, "gemm", "bf16")
    wt = (torch.randn(k, r, r, c, device="cuda") * 0.05).bfloat16()
    dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
    mask = torch.randn(n, h, w, c, device="cuda").bfloat16()
    res = torch.randn(n, h, w, c, device="cuda").bfloat16()
    dx = torch.empty(n, h, w, c, device="cuda").bfloat16()
    out = {}
    for name, kw in (("plain", {}), ("mask", {"mask": mask}), ("mask_res", {"mask": mask, "residual": res})):
        fn = lambda: plan.dgrad(dy, wt, out=dx, **kw)  # noqa: E731
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        out[name] = round(e0.elapsed_time(e1) / 20 * 1000, 1)
    print(json.dumps({"geom": sys.argv[1:9], "us": out}))


if __name__ == "__main__":
    main()
