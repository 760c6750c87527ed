"""Isolated bf16 wgrad timings for one 3x3 conv at a fixed pixel count and
different image sizes (N x H x W): shows whether wgrad time depends on the
image width beyond the pixel count.  python scripts/wgrad_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_06622_b200 import device  # noqa: E402


def t_wgrad(n, h, w, c, k, r=3, pad=1, reps=5):
    g = device.geom(n, h, w, c, k, r, pad=pad, stride=1)
    plan = device.ConvPlan(g, "gemm", "bf16")
    x = torch.randn(n, h, w, c, device="cuda").bfloat16()
    dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
    plan.wgrad(dy, x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        plan.wgrad(dy, x)
    e.record()
    e.synchronize()
    return round(s.elapsed_time(e) / reps, 3)


for c, k in ((64, 64), (128, 128)):
    for n, hw in ((64, 224), (256, 112), (1024, 56), (4096, 28)):
        print(c, k, n, hw, t_wgrad(n, hw, hw, c, k), "ms", flush=True)
