"""Run warm-up steps, then ONE training step inside cudaProfilerStart/Stop, so
`ncu --profile-from-start off` captures exactly the launches of one step.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python scripts/step_profile.py [model] [batch] [precision]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_06622_b200 import models  # noqa: E402
from paper_1709_06622_b200.trainer import Trainer  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
t = Trainer(models.build(model, batch=batch, precision=prec))
for _ in range(3):
    t.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
t.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches", t.launch_count(), "loss", t.loss())
