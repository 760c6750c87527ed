"""Where the e2e gap comes from: ResNet-50 bs256 steps timed with CUDA events
(a) resident batch, (b) + per-step async loss D2H, (c) staged uint8 host
batches, (d) staged + loss D2H (= bench.py's e2e loop).
    python scripts/diag_e2e.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_06622_b200 import models  # noqa: E402
from paper_1709_06622_b200.trainer import Trainer  # noqa: E402

steps = 30
tr = Trainer(models.build("resnet50", batch=256))
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
inp = tr.describe()["layers"][0]
host = [(torch.randint(0, 256, (256, inp["shape"][1], inp["shape"][2], inp["c_logical"]), dtype=torch.uint8).pin_memory(),
         torch.randint(0, 1000, (256,), dtype=torch.int32).pin_memory()) for _ in range(2)]
lossbuf = torch.empty(1, dtype=torch.float32).pin_memory()
st = torch.cuda.current_stream()


def run(stage, d2h):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    if stage:
        tr.stage_batch(*host[0])
    for i in range(steps):
        tr.step()
        if stage and i + 1 < steps:
            tr.stage_batch(*host[(i + 1) % 2])
        if d2h:
            lossbuf.copy_(tr.tensor("loss")[:1], non_blocking=True)
    e.record(st)
    e.synchronize()
    return round(s.elapsed_time(e) / steps, 3)


for _ in range(2):
    print({"resident": run(False, False), "resident+d2h": run(False, True), "staged": run(True, False),
           "staged+d2h": run(True, True)}, flush=True)
