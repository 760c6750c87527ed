"""Re-drive the paper's selection procedure with B200 measurements (GPU box).

  C2  AlexNet-227 conv stack: profile gemm / winograd / fft for mini-batches
      32..512 -> reference-format catalog -> plan_batch_size at 180 GB and at
      the fixtures' 12 GiB (algorithm choice under a binding memory bound).
  C4  Inception-v3 (299x299, batch 128): per-layer time and workspace of the
      three algorithm families.
  C5  VGG-16: catalog at batches 32/64 and the plan at 180 GB.

Writes gpurun_out/b200_*.{csv,json}; tests/golden keeps the committed copies
so the decision-parity tests (this planner vs the reference's on the same
B200 catalog) run anywhere.
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
from paper_1709_06622_b200 import models, profiler  # noqa: E402

OUT = "gpurun_out"
os.makedirs(OUT, exist_ok=True)
GB180 = 180 * 10**9 * 8
GIB12 = 12 * 2**30 * 8
DATASET = 1_281_167


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, indent=1)


def run_chain(tag, cfg, batches, reps):
    t0 = time.time()
    prof = profiler.profile(profiler.feature_conv_specs(cfg), batches, reps=reps)
    with open(os.path.join(OUT, f"b200_catalog_{tag}.csv"), "w") as f:
        f.write(prof["csv"])
    net = profiler.net_text(cfg)
    with open(os.path.join(OUT, f"b200_{tag}.net"), "w") as f:
        f.write(net)
    dump(f"b200_profile_{tag}.json", {"rows": prof["rows"], "skipped": prof["skipped"],
                                      "seconds": time.time() - t0})
    for label, bits in (("180GB", GB180), ("12GiB", GIB12)):
        plan = profiler.plan(net, prof["csv"], bits, DATASET)
        dump(f"b200_plan_{tag}_{label}.json", plan)
        rec = plan["recommended"]
        sel = next((c["solve"] for c in plan["candidates"] if c["batch_size"] == rec), None)
        print(tag, label, "recommended", rec, "assignment", sel and sel.get("assignment"),
              "throughput", [round(c["throughput"] or 0, 1) for c in plan["candidates"]], flush=True)


def main():
    run_chain("alexnet", models.alexnet(batch=1), [32, 64, 128, 256, 512], reps=5)
    run_chain("vgg16", models.vgg16(batch=1), [16, 32, 64], reps=3)
    t0 = time.time()
    inc = models.inception_v3_convs(batch=128)
    specs = [{k: L[k] for k in ("h", "w", "c", "k", "r", "s", "pad_h", "pad_w")} | {
        "stride_h": L["stride"], "stride_w": L["stride"]} for L in inc]
    prof = profiler.profile(specs, [128], reps=3)
    dump("b200_profile_inception_v3.json", {"layers": [L["name"] for L in inc], "rows": prof["rows"],
                                            "skipped": prof["skipped"], "seconds": time.time() - t0})
    with open(os.path.join(OUT, "b200_catalog_inception_v3.csv"), "w") as f:
        f.write(prof["csv"])
    best = {}
    for r in prof["rows"]:
        cur = best.get(r["layer_id"])
        if cur is None or r["total_ms"] < cur["total_ms"]:
            best[r["layer_id"]] = r
    counts = {}
    for r in best.values():
        counts[r["algorithm"]] = counts.get(r["algorithm"], 0) + 1
    print("inception fastest-algorithm counts", counts, flush=True)


if __name__ == "__main__":
    main()
