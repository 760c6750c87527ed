"""Does CUDA-graph replay of the whole training step beat stream launches?
Captures one ResNet-50 bs256 step (1 GPU) with torch.cuda.graph and times
replays against plain tr.step() calls."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_06622_b200 import models  # noqa: E402
from paper_1709_06622_b200.trainer import Trainer  # noqa: E402

t = Trainer(models.build("resnet50", batch=256, precision="bf16"))
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for _ in range(5):
    t.step()
torch.cuda.synchronize()


def timed(fn, n=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


plain = timed(t.step)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    t.step()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
graph = timed(g.replay)
plain2 = timed(t.step)
print({"plain_ms": round(plain, 3), "graph_ms": round(graph, 3), "plain2_ms": round(plain2, 3)})
