"""Time the ResNet-50 bs256 stem (7x7/2, 3 of 8 channels -> 64) through the
conv plan API: row-window stem kernels vs the explicit-im2col GEMM path.
    python scripts/stem_profile.py [--iters 20] [--only-stem]"""
import argparse
import ctypes
import json

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1709_06622_b200 import device


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only-stem", action="store_true")
    ap.add_argument("--n", type=int, default=256)
    a = ap.parse_args()
    L = device.lib()
    L.tcb_set_conv_stem.argtypes = [ctypes.c_int]
    g = device.geom(a.n, 224, 224, 8, 64, 7, pad=3, stride=2)
    x = torch.randn(a.n, 224, 224, 8, device="cuda")
    x[..., 3:] = 0
    x = x.bfloat16()
    w = (torch.randn(64, 7, 7, 8, device="cuda") * 0.05).bfloat16()
    dy = torch.randn(a.n, 112, 112, 64, device="cuda").bfloat16()
    out = {}
    for on in ((1,) if a.only_stem else (1, 0)):
        L.tcb_set_conv_stem(on)
        plan = device.ConvPlan(g, "gemm", "bf16").set_valid_channels(3)
        for name, fn in (("fwd", lambda: plan.fwd(x, w, relu=True)), ("wgrad", lambda: plan.wgrad(dy, x))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            out[f"{'stem' if on else 'im2col'}_{name}_ms"] = round(e0.elapsed_time(e1) / a.iters, 4)
    L.tcb_set_conv_stem(-1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
