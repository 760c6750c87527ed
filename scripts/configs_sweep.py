"""Single-GPU measurements of the other BASELINE configs (C1 LeNet, C2
AlexNet-227 mini-batch sweep, C5 VGG-16), and — for C2 — the planner's
predicted throughput (`plan_batch_size` on the committed B200-measured catalog,
b / sum T over the conv layers) beside the measured full-step throughput.

    python scripts/configs_sweep.py > gpurun_out/configs.json
"""
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
    st = torch.cuda.current_stream()
    s.record(st)
    for _ in range(steps):
        t.step()
    e.record(st)
    e.synchronize()
    ms = s.elapsed_time(e) / steps
    t.enable_timing(True)
    t.step()
    ph = t.phase_times()
    return {"ms_per_step": round(ms, 3), "images_per_sec": round(cfg["batch"] * 1e3 / ms, 1),
            "phases_ms": {k: round(v, 3) for k, v in ph.items()}, "loss": t.loss()}


def main():
    out = {"device": torch.cuda.get_device_name(0)}
    out["C1_lenet_b64"] = {p: measure(models.build("lenet", batch=64, precision=p))
                           for p in ("ffma", "bf16")}
    gold = os.path.join(ROOT, "tests", "golden", "b200")
    net = open(os.path.join(gold, "b200_alexnet.net")).read()
    cat = open(os.path.join(gold, "b200_catalog_alexnet.csv")).read()
    plan = planner.default().call("plan_batch_size", network=net, catalog=cat,
                                  gpu_bits=180 * 10**9 * 8, dataset=1_281_167)
    pred = {c["batch_size"]: c for c in plan["candidates"]}
    c2 = {}
    for b in (32, 64, 128, 256, 512):
        m = measure(models.build("alexnet", batch=b, precision="bf16"))
        c = pred.get(b, {})
        m["planner_predicted_images_per_sec"] = c.get("throughput")
        m["planner_conv_time_per_batch_s"] = (c.get("solve") or {}).get("total_time")
        m["planner_assignment"] = sorted(set(((c.get("solve") or {}).get("assignment") or {}).values()))
        c2[str(b)] = m
    out["C2_alexnet227_sweep"] = {"recommended_batch": plan["recommended"], "per_batch": c2}
    out["C5_vgg16_b64"] = measure(models.build("vgg16", batch=64, precision="bf16"))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
