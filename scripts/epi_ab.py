"""Time HBM-bound K-light conv passes (TMA epilogue with residual / mask side
inputs) of the ResNet-50 bs256 step through the conv plan API.
    python scripts/epi_ab.py [--iters 30]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_06622_b200 import device  # noqa: E402

CASES = [  # name, n, h, w, c, k, r, pad, stride
    ("s1_c3_1x1_64_256", 256, 56, 56, 64, 256, 1, 0, 1),
    ("s1_c1_1x1_256_64", 256, 56, 56, 256, 64, 1, 0, 1),
    ("s2_c3_1x1_128_512", 256, 28, 28, 128, 512, 1, 0, 1),
    ("s2_c1_1x1_512_128", 256, 28, 28, 512, 128, 1, 0, 1),
    ("s3_c3_1x1_256_1024", 256, 14, 14, 256, 1024, 1, 0, 1),
]
S3X3_CASES = [  # stride-1 3x3 passes of stages 2-4 (tensor-bound)
    ("s2_c2_3x3_128", 256, 28, 28, 128, 128, 3, 1, 1),
    ("s3_c2_3x3_256", 256, 14, 14, 256, 256, 3, 1, 1),
    ("s4_c2_3x3_512", 256, 7, 7, 512, 512, 3, 1, 1),
]
REG_CASES = [  # K-heavy passes (register epilogue)
    ("s3_c2_3x3_256", 256, 14, 14, 256, 256, 3, 1, 1),
    ("s4_c2_3x3_512", 256, 7, 7, 512, 512, 3, 1, 1),
    ("s4_c1_1x1_2048_512", 256, 7, 7, 2048, 512, 1, 0, 1),
    ("s3_c1_1x1_1024_256", 256, 14, 14, 1024, 256, 1, 0, 1),
]


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / iters * 1000, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--set", default="epi", choices=["epi", "reg", "3x3"])
    a = ap.parse_args()
    out = {}
    sets = {"epi": CASES, "reg": REG_CASES, "3x3": S3X3_CASES}
    for name, n, h, w, c, k, r, pad, st in sets[a.set]:
        g = device.geom(n, h, w, c, k, r, pad=pad, stride=st)
        plan = device.ConvPlan(g, "gemm", "bf16")
        x = torch.randn(n, h, w, c, device="cuda").bfloat16()
        wt = (torch.randn(k, r, r, c, device="cuda") * 0.05).bfloat16()
        res = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
        dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
        y = torch.empty(n, g.ho, g.wo, k, device="cuda").bfloat16()
        dx = torch.empty(n, h, w, c, device="cuda").bfloat16()
        dw = torch.empty(k, r, r, c, device="cuda")
        out[name] = {"fwd_res_relu_us": timeit(lambda: plan.fwd(x, wt, residual=res, relu=True, out=y), a.iters),
                     "fwd_us": timeit(lambda: plan.fwd(x, wt, out=y), a.iters),
                     "fwd_launch": device.last_launch(),
                     "dgrad_mask_us": timeit(lambda: plan.dgrad(dy, wt, mask=x, out=dx), a.iters),
                     "dgrad_launch": device.last_launch()}
        if a.set == "3x3":
            out[name]["wgrad_us"] = timeit(lambda: plan.wgrad(dy, x, out=dw), a.iters)
            out[name]["wgrad_launch"] = device.last_launch()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
