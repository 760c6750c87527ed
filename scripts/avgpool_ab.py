"""Time the windowed average pool (Inception branch pools, 3x3/1/1) fwd / bwd at bs128."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1709_06622_b200 import device  # noqa: E402
from epi_ab import timeit  # noqa: E402

out = {}
for (h, c) in ((35, 256), (17, 768), (8, 2048)):
    x = torch.randn(128, h, h, c, device="cuda").bfloat16()
    y = device.avgpool2d_fwd(x, 3, 1, 1)
    out[f"{h}x{c}_fwd_us"] = timeit(lambda: device.avgpool2d_fwd(x, 3, 1, 1), 20)
    out[f"{h}x{c}_bwd_us"] = timeit(lambda: device.avgpool2d_bwd(y, (128, h, h, c), 3, 1, 1), 20)
print(json.dumps(out))
