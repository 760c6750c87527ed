"""Tiny launches of every tensor-core conv path for compute-sanitizer
(racecheck / synccheck / memcheck): bf16 im2col-TMA, plain-TMA, gather,
CTA pairs, TMA-store epilogue, window fwd / dgrad / wgrad, TF32; one call
each, small shapes (the tools replay every access).
    compute-sanitizer --tool racecheck python scripts/sanitize_small.py"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_06622_b200 import device  # noqa: E402

L = device.lib()
L.tcb_set_conv_operand_path.argtypes = [ctypes.c_int]
CASES = [  # n h w c k r pad stride
    (2, 10, 10, 64, 128, 3, 1, 1),   # im2col TMA (+ window when forced)
    (2, 6, 6, 64, 64, 1, 0, 1),      # plain TMA, TMA-store epilogue
    (2, 16, 16, 128, 256, 3, 1, 1),  # CTA pairs
    (2, 9, 9, 40, 72, 3, 1, 2),      # gather, strided dgrad phases
    (2, 20, 20, 64, 64, 3, 1, 1),    # window fwd / dgrad / wgrad (N = 64)
]
for mode in (0, 4):  # auto, window wherever it applies
    L.tcb_set_conv_operand_path(mode)
    for n, h, w, c, k, r, pad, stride in CASES:
        for prec in ("bf16", "tf32"):
            g = device.geom(n, h, w, c, k, r, pad=pad, stride=stride)
            try:
                plan = device.ConvPlan(g, "gemm", prec)
            except device.Unsupported:
                continue
            dt = plan.dtype
            x = torch.randn(n, h, w, c, device="cuda").to(dt)
            wt = (torch.randn(k, r, r, c, device="cuda") * 0.05).to(dt)
            dy = torch.randn(n, g.ho, g.wo, k, device="cuda").to(dt)
            plan.fwd(x, wt, residual=torch.randn(n, g.ho, g.wo, k, device="cuda").to(dt), relu=True)
            plan.dgrad(dy, wt, mask=x)
            plan.wgrad(dy, x)
            torch.cuda.synchronize()
            print("ok", mode, prec, (n, h, w, c, k, r, pad, stride), flush=True)
L.tcb_set_conv_operand_path(0)
print("done")
