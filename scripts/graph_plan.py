"""C3 / C4 through the planner: profile every feature conv of
ResNet-50 and Inception-v3 for gemm / winograd / fft at several mini-batches
on this B200 (reference catalog format), plan with the executor's exact
layout as the memory model (profiler.plan_graph, 180 GB), then run every
candidate batch's training step with its Selection and report the measured
images/s beside the planner's predicted b / sum T.

    python scripts/graph_plan.py > gpurun_out/graph_plan.json
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_06622_b200 import models, profiler  # noqa: E402
from paper_1709_06622_b200.trainer import Trainer  # noqa: E402

GB180 = 180 * 10**9 * 8


def measure(cfg, steps=8, warmup=3):
    t = Trainer(cfg)
    for _ in range(warmup):
        t.step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        t.step()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / steps
    del t
    torch.cuda.empty_cache()
    return round(cfg["batch"] * 1e3 / ms, 1)


def run(name, build, batches):
    t0 = time.time()
    specs = profiler.feature_conv_specs(build(1))
    prof = profiler.profile(specs, list(batches), reps=3)
    with open(os.path.join(ROOT, "gpurun_out", f"b200_catalog_{name}.csv"), "w") as f:
        f.write(prof["csv"])
    plan = profiler.plan_graph(build, prof["csv"], batches, GB180, 1_281_167)
    out = {"layers": len(specs), "profile_seconds": round(time.time() - t0, 1),
           "recommended": plan["recommended"], "candidates": []}
    for c in plan["candidates"]:
        sel = (c["solve"] or {}).get("assignment") or {}
        counts = {}
        for a in sel.values():
            counts[a] = counts.get(a, 0) + 1
        row = {"batch": c["batch_size"], "feasible": c["solve"]["feasible"],
               "resident_bits": c["breakdown"]["feature_maps"], "bound_bits": c["breakdown"]["bound"],
               "predicted_images_per_sec": c["throughput"], "selection_counts": counts,
               "memory_limited_layers": c["memory_limited_layers"]}
        if sel:
            row["measured_images_per_sec"] = measure(models.apply_selection(build(c["batch_size"]), sel))
        out["candidates"].append(row)
    return out


def main():
    res = {"device": torch.cuda.get_device_name(0), "gpu_bits": GB180}
    res["resnet50"] = run("resnet50", lambda b: models.resnet50(batch=b), (32, 64, 128, 256))
    res["inception_v3"] = run("inception_v3", lambda b: models.inception_v3(batch=b), (32, 64, 128, 256))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
