"""Time the ResNet stem max pool (3x3/2/1 over 256x112x112x64 bf16) fwd / bwd."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1709_06622_b200 import device  # noqa: E402
from epi_ab import timeit  # noqa: E402

x = torch.randn(256, 112, 112, 64, device="cuda").relu().bfloat16()
y, arg = device.maxpool_fwd(x, 3, 2, 1)
dy = torch.randn_like(y)
print(json.dumps({"fwd_us": timeit(lambda: device.maxpool_fwd(x, 3, 2, 1), 20),
                  "bwd_us": timeit(lambda: device.maxpool_bwd(dy, arg, tuple(x.shape), 3, 2, 1, relu_y=y), 20)}))
