"""Time wide-image stride-1 3x3 passes (rectangular window tiles vs im2col TMA):
Inception-v3 Conv2d_2a / 2b at bs128 (32 -> 64-channel allocation), VGG-16
conv1_2 at bs64.  TCB_WIN_RECT=0 python scripts/wide_ab.py for the im2col path."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1709_06622_b200 import device  # noqa: E402
from epi_ab import timeit  # noqa: E402

CASES = [("incep_2a", 128, 149, 149, 64, 64, 0), ("incep_2b", 128, 147, 147, 64, 64, 1),
         ("vgg_conv1_2", 64, 224, 224, 64, 64, 1)]
out = {}
for name, n, h, w, c, k, pad in CASES:
    g = device.geom(n, h, w, c, k, 3, pad=pad)
    plan = device.ConvPlan(g, "gemm", "bf16")
    x = torch.randn(n, h, w, c, device="cuda").bfloat16()
    wt = (torch.randn(k, 3, 3, c, device="cuda") * 0.05).bfloat16()
    dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
    y = torch.empty(n, g.ho, g.wo, k, device="cuda").bfloat16()
    dx = torch.empty_like(x)
    out[name] = {"fwd_relu_us": timeit(lambda: plan.fwd(x, wt, relu=True, out=y), 20),
                 "fwd_load": device.last_launch()["load"],
                 "dgrad_mask_us": timeit(lambda: plan.dgrad(dy, wt, mask=x, out=dx), 20),
                 "dgrad_load": device.last_launch()["load"]}
print(json.dumps(out))
