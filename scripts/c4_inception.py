"""C4 — Inception-v3 (299x299, batch 128, bf16) training steps on one B200:
all-GEMM vs the paper's per-layer algorithm selection (Eq 6 via the traincap
solver over the committed B200 catalog, tests/golden/b200/
b200_catalog_inception_v3.csv), the executor obeying the Selection.
The memory bound for the workspace choice is the HBM left after the
executor's own arena (the branched graph has no chain memory model, Eq 2-5).

    python scripts/c4_inception.py > gpurun_out/c4_inception.json
"""
import collections
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_06622_b200 import models, planner  # noqa: E402
from paper_1709_06622_b200.trainer import Trainer  # noqa: E402


def measure(cfg, steps=10, warmup=3):
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
    t.enable_timing(True)
    t.step()
    out = {"ms_per_step": round(ms, 3), "images_per_sec": round(cfg["batch"] * 1e3 / ms, 1),
           "phases_ms": {k: round(v, 3) for k, v in t.phase_times().items()}, "loss": t.loss(),
           "arena_bytes": t.describe()["arena_bytes"], "launches": t.launch_count()}
    del t
    torch.cuda.empty_cache()
    return out


def main():
    batch = 128
    cfg = models.inception_v3(batch=batch, precision="bf16")
    res = {"device": torch.cuda.get_device_name(0), "workload": "inception_v3_synthetic_299",
           "batch": batch, "gflop_per_image_fwd": models.flops_per_image(cfg) / 1e9}
    res["gemm_only"] = measure(cfg)
    cat = open(os.path.join(ROOT, "tests", "golden", "b200", "b200_catalog_inception_v3.csv")).read()
    bound = 180 * 10**9 * 8 - res["gemm_only"]["arena_bytes"] * 8
    sol = planner.default().call("solve_catalog", catalog=cat, batch=batch, bound=bound)
    assign = sol.get("assignment") or {}
    res["selection"] = {"bound_bits": bound, "feasible": sol.get("feasible"),
                        "counts": dict(collections.Counter(assign.values())),
                        "predicted_conv_seconds_per_batch": sol.get("total_time")}
    res["planner_selection"] = measure(models.apply_selection(cfg, assign))
    # the alternative families forced where they apply (stride-1 3x3 -> Winograd,
    # stride-1 5x5 -> FFT), to show what the Selection avoided
    forced = {}
    for i, (name, g) in enumerate(models.conv_layers(cfg)[:-1], 1):
        if g["stride_h"] == 1 and g["r"] == g["s"] == 3:
            forced[str(i)] = "winograd"
        elif g["stride_h"] == 1 and g["r"] == g["s"] == 5:
            forced[str(i)] = "fft"
    res["forced_winograd_fft"] = {"counts": dict(collections.Counter(forced.values())),
                                  **measure(models.apply_selection(cfg, forced))}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
