"""Decision-path timing: this build's traincap planner vs the
reference planner compiled from /root/reference (oracle/_ref, prebuilt; it
travels with the repo snapshot), on the B200-measured catalogs, same requests,
identical replies required. Host CPU only.

    python scripts/planner_timing.py [reps]
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libtraincap_ref.so")
B200 = os.path.join(ROOT, "tests", "golden", "b200")


def _read(name):
    with open(os.path.join(B200, name)) as f:
        return f.read()


def requests():
    alex_net, alex_cat = _read("b200_alexnet.net"), _read("b200_catalog_alexnet.csv")
    vgg_net, vgg_cat = _read("b200_vgg16.net"), _read("b200_catalog_vgg16.csv")
    inc_cat = _read("b200_catalog_inception_v3.csv")
    return {
        "plan_batch_size alexnet-227 @180GB": dict(op="plan_batch_size", network=alex_net,
                                                   catalog=alex_cat, gpu_bits=180 * 10**9 * 8,
                                                   dataset=1_281_167),
        "plan_batch_size vgg16 @12GiB": dict(op="plan_batch_size", network=vgg_net, catalog=vgg_cat,
                                             gpu_bits=12 * 2**30 * 8, dataset=1_281_167),
        "solve_catalog inception-v3 (94 layers) b=128": dict(op="solve_catalog", catalog=inc_cat,
                                                            batch=128, bound=10**12),
    }


def time_planners(reps=100):
    import ctypes
    from paper_1709_06622_b200 import planner
    ours = planner.Planner()
    ref = planner.Planner(ctypes.CDLL(REF_LIB), prefix="tcref_") if os.path.exists(REF_LIB) else None
    out = {}
    for name, req in requests().items():
        req = dict(req)
        op = req.pop("op")
        row = {}
        for tag, lib in (("ours", ours), ("reference", ref)):
            if lib is None:
                row[tag] = None
                continue
            reply = lib.raw(op, **req)
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                lib.raw(op, **req)
                ts.append(time.perf_counter() - t0)
            row[tag + "_us_median"] = round(statistics.median(ts) * 1e6, 1)
            row[tag + "_reply"] = reply
        if ref is not None:
            row["identical"] = row.pop("ours_reply") == row.pop("reference_reply")
        else:
            row.pop("ours_reply", None)
        out[name] = row
    return {"reps": reps, "cores": os.cpu_count(), "requests": out,
            "reference_lib": os.path.relpath(REF_LIB, ROOT) if ref else None}


if __name__ == "__main__":
    print(json.dumps(time_planners(int(sys.argv[1]) if len(sys.argv) > 1 else 100), indent=1))
