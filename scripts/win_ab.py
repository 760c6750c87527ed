"""Time the window-path stage-1 3x3 passes (ResNet-50 bs256, 56x56x64) through
the conv plan API: fwd (+ReLU), dgrad (+ReLU mask), wgrad.
    python scripts/win_ab.py [--iters 30]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_06622_b200 import device  # noqa: E402
from epi_ab import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    g = device.geom(256, 56, 56, 64, 64, 3, pad=1)
    plan = device.ConvPlan(g, "gemm", "bf16")
    x = torch.randn(256, 56, 56, 64, device="cuda").bfloat16()
    wt = (torch.randn(64, 3, 3, 64, device="cuda") * 0.05).bfloat16()
    dy = torch.randn(256, 56, 56, 64, device="cuda").bfloat16()
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    dw = torch.empty(64, 3, 3, 64, device="cuda")
    print(json.dumps({"fwd_relu_us": timeit(lambda: plan.fwd(x, wt, relu=True, out=y), a.iters),
                      "dgrad_mask_us": timeit(lambda: plan.dgrad(dy, wt, mask=x, out=dx), a.iters),
                      "wgrad_us": timeit(lambda: plan.wgrad(dy, x, out=dw), a.iters)}))


if __name__ == "__main__":
    main()
