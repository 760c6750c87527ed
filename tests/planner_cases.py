"""Deterministic planner request corpus shared by the golden generator and the
parity tests.

Every case is a JSON request for the planner C-ABI (`<prefix>planner_call`).
The generators restate the *behaviour* of the reference's own test helpers
(/root/reference/proj/tests/helpers.hpp:19-170): random valid networks, random
multiple-choice instances on a 0.125 s time grid (so ties really occur) with
bounds drawn from {-1, min-1, min, max, uniform}, the sweep network/catalog
with the cubic FFT workspace, plus malformed inputs for every error path.
"""
from __future__ import annotations

import json
import os
import random

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = os.path.join(HERE, "golden", "fixtures")


def fixture(name: str) -> str:
    with open(os.path.join(FIXTURES, name)) as f:
        return f.read()


ALEXNET_NET = "fixtures/alexnet.net"


def structured(inp, feats, fcs):
    return {"input": list(inp), "features": [list(f) for f in feats], "classifier": list(fcs)}


TOY_NET = structured((4, 4, 1), [("conv", 3, 1, 1, 2)], (8, 4))
SWEEP_NET = structured((8, 8, 1), [("conv", 3, 1, 1, 4), ("conv", 3, 1, 1, 8)], (16, 4))
CONV_STACK = structured((224, 224, 3), [("conv", 11, 4, 2, 96), ("conv", 5, 2, 1, 256),
                                        ("conv", 3, 2, 0, 384), ("conv", 3, 1, 1, 384),
                                        ("conv", 3, 1, 1, 256)], (4096, 4096, 1000))


def sweep_catalog_csv() -> str:
    batches = [32, 64, 128, 256, 512]
    gemm = [0.040, 0.070, 0.130, 0.240, 0.520]
    fft = [0.016, 0.029, 0.050, 0.080, 0.150]
    rows = ["layer_id,algorithm,batch_size,time_seconds,memory_bits"]
    for layer in (1, 2):
        for i, b in enumerate(batches):
            rows.append(f"{layer},gemm,{b},{gemm[i]!r},{100 * b}")
            rows.append(f"{layer},fft,{b},{fft[i]!r},{3 * b * b * b}")
    return "\n".join(rows) + "\n"


def random_network(rng: random.Random):
    inp = (rng.randint(4, 64), rng.randint(4, 64), rng.randint(1, 8))
    w, h = inp[0], inp[1]
    feats = []
    for _ in range(rng.randint(1, 6)):
        f = rng.randint(1, min(min(w, h), 5))
        s, p = rng.randint(1, 3), rng.randint(0, 2)
        conv = rng.randint(0, 2) != 0
        k = rng.randint(1, 8) if conv else 0

        def nxt(v):
            return (v - f + 2 * p) // s + 1
        if nxt(w) < 1 or nxt(h) < 1:
            s, p = 1, f // 2 + 1
        w, h = nxt(w), nxt(h)
        feats.append(("conv" if conv else "pool", f, s, p, k))
    fcs = [rng.randint(1, 100) for _ in range(rng.randint(1, 3))]
    return structured(inp, feats, fcs)


def random_mckp(rng: random.Random, max_layers: int, max_algos: int):
    names = "abcde"
    q = rng.randint(1, max_layers)
    options, lo_sum, hi_sum = [], 0, 0
    for k in range(1, q + 1):
        p = rng.randint(1, max_algos)
        layer = [{"layer_id": k, "algorithm": names[j], "batch_size": 1,
                  "time_seconds": rng.randint(1, 64) * 0.125,
                  "memory_bits": rng.randint(0, 1000)} for j in range(p)]
        mems = [e["memory_bits"] for e in layer]
        lo_sum += min(mems)
        hi_sum += max(mems)
        options.append(layer)
    mode = rng.randint(0, 4)
    bound = [-1, lo_sum - 1, lo_sum, hi_sum, None][mode]
    if bound is None:
        bound = lo_sum + rng.randint(0, max(1, hi_sum - lo_sum))
    return options, bound


def random_catalog_csv(rng: random.Random, layers: int, batches, algos, fmt="csv"):
    rows = []
    for l in range(1, layers + 1):
        for b in batches:
            chosen = [a for a in algos if rng.random() < 0.8] or [algos[0]]
            for a in chosen:
                t = rng.choice([rng.randint(1, 40) * 0.0625, rng.uniform(1e-4, 2.0)])
                m = rng.randint(0, 5_000_000) * b
                rows.append((l, a, b, t, m))
    rng.shuffle(rows)
    if fmt == "json":
        return json.dumps([{"layer_id": l, "algorithm": a, "batch_size": b,
                            "time_seconds": t, "memory_bits": m} for l, a, b, t, m in rows])
    out = ["layer_id,algorithm,batch_size,time_seconds,memory_bits"]
    out += [f"{l},{a},{b},{t!r},{m}" for l, a, b, t, m in rows]
    return "\n".join(out) + "\n"


BAD_NETS = [
    "", "# only a comment\n", "conv 3 1 1 4\n", "input 8 8\n", "input 8 8 1\ninput 8 8 1\n",
    "input 8 8 1\nconv 3 1 1\n", "input 8 8 1\nconv 3 1 1 x\n", "input 8 8 1\nconv y 1 1 4\n",
    "input 8 8 1\nfc 10\nconv 3 1 1 4\n", "input 8 8 1\nrelu\n", "input a 8 1\n",
    "input 8 8 1\npool 3 1\n", "input 8 8 1\nfc 1 2\n", "input 8 8 1 # c\nconv 3 1 1 4 # x\nfc 2\n",
    "input 4 4 1\nconv 9 1 0 4\nfc 2\n", "input 4 4 1\nconv 3 0 1 4\nfc 2\n",
    "input 0 4 1\nconv 3 1 1 0\npool 2 2 0\nfc 0\n", "input 4 4 1\npool 2 2 -1\n",
    "input 4 4 1\r\nconv 3 1 1 4\r\nfc 2\r\n",
]

BAD_CATALOGS = [
    ("", "csv"), ("layer,algorithm\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,0.1\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,0.1,5,\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\nx,gemm,32,0.1,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,3.5,0.1,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,fast,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,0.1,-5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,0,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n0,gemm,32,0.1,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1, ,32,0.1,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,0.1,5\n\n1,gemm,32,0.2,6\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,0.1,5\n3,gemm,32,0.1,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,0.1,5\n2,fft,64,0.1,5\n", "csv"),
    ("  layer_id,algorithm,batch_size,time_seconds,memory_bits \r\n 1 , gemm , 32 , 0.1 , 5 \r\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,nan,5\n", "csv"),
    ("layer_id,algorithm,batch_size,time_seconds,memory_bits\n1,gemm,32,1e-3,0\n1,fft,32,5e-4,70\n", "csv"),
    ("[", "json"), ("{}", "json"), ("[1]", "json"), ('[{"layer_id":1}]', "json"),
    ('[{"layer_id":"a","algorithm":"g","batch_size":1,"time_seconds":1,"memory_bits":1}]', "json"),
    ('[{"layer_id":1.7,"algorithm":"g","batch_size":1,"time_seconds":1,"memory_bits":1}]', "json"),
    ('[{"layer_id":1,"algorithm":"g","batch_size":1,"time_seconds":1,"memory_bits":1},'
     '{"layer_id":1,"algorithm":"g","batch_size":1,"time_seconds":2,"memory_bits":1}]', "json"),
    ("[]", "json"),
]

BAD_TRACES = [
    "gpu_processing 1.0\nparameter_update x\n", "gpu_processing\n", "warp_drive 1\n",
    "gpu_processing 1 hidden extra\n", "gpu_processing 1 visible\n",
    "gpu_processing 1\ngpu_processing 2\n", "parameter_update 0.1\n",
    "gpu_processing 0\n", "gpu_processing 1\nparameter_update -0.5\n",
]

UNIT_STRINGS = ["12GiB", "180MB", "1.5 TB", "10", "MB", "12 XB", "  4KiB ", "-3GB", "1e3B",
                "10Gbps", "1.25GB/s", "800Mbps", "5 MiB/s", "3bps", "7Xbps", "9/s", "1 Tbps"]


def build_cases() -> list[dict]:
    rng = random.Random(20260810)
    alex = fixture("alexnet.net")
    profile = fixture("alexnet_profile.csv")
    b128 = fixture("alexnet_profile_batch128.csv")
    b128j = fixture("alexnet_profile_batch128.json")
    steps = fixture("steps_example.txt")
    cases: list[dict] = []
    add = cases.append

    # --- Eq 1 shapes and validation -----------------------------------------
    for net in (alex, TOY_NET, SWEEP_NET, CONV_STACK):
        add({"op": "propagate_shapes", "network": net})
        add({"op": "validate_network", "network": net})
        add({"op": "parameter_bits", "network": net})
        add({"op": "model_param_memory", "network": net})
    for text in BAD_NETS:
        # A zero stride divides by zero inside the reference's propagate_shapes
        # (undefined behaviour, SIGFPE); only validate_network may see it.
        if "conv 3 0" not in text:
            add({"op": "propagate_shapes", "network": text})
        add({"op": "validate_network", "network": text})
    for _ in range(60):
        net = random_network(rng)
        add({"op": "propagate_shapes", "network": net})
        add({"op": "validate_network", "network": net})
        add({"op": "memory_bound", "network": net, "gpu_bits": rng.randint(-10, 1 << 40),
             "batch": rng.randint(1, 1 << 20)})
        add({"op": "parameter_bits", "network": net})
    # invalid structured networks (validation collects everything)
    add({"op": "validate_network", "network": structured((0, 3, -1), [("pool", 0, 0, -1, 3),
                                                                        ("conv", 3, 1, 0, 0)], (0,))})
    add({"op": "validate_network", "network": structured((5, 5, 1), [("conv", 7, 1, 0, 3)], (2,))})
    add({"op": "validate_network", "network": structured((5, 5, 1), [], ())})

    # --- Eq 2-5 memory ------------------------------------------------------
    for b in (1, 2, 32, 64, 128, 256, 512):
        for net in (alex, TOY_NET, CONV_STACK):
            add({"op": "memory_bound", "network": net, "gpu_bits": 12 * 2**30 * 8, "batch": b})
            add({"op": "feature_map_memory", "network": net, "batch": b})
    add({"op": "memory_bound", "network": alex, "gpu_bits": 1_440_000_000_000, "batch": 512})
    add({"op": "feature_map_memory", "network": alex, "batch": 0})
    add({"op": "memory_bound", "network": alex, "gpu_bits": -(2**63) + 5, "batch": 2})
    add({"op": "memory_bound", "network": alex, "gpu_bits": 1, "batch": 2**61})
    add({"op": "classifier_memory", "layers": [8, 4]})
    add({"op": "classifier_memory", "layers": [9216, 4096, 1000]})
    add({"op": "classifier_memory", "layers": []})
    add({"op": "classifier_memory", "layers": [2**40, 2**40]})

    # --- catalog ------------------------------------------------------------
    for text, fmt in ((profile, "csv"), (b128, "csv"), (b128j, "json"), (sweep_catalog_csv(), "csv")):
        add({"op": "load_catalog", "catalog": text, "format": fmt, "batch": 128})
        add({"op": "default_batch_candidates", "catalog": text, "format": fmt})
    for text, fmt in BAD_CATALOGS:
        add({"op": "load_catalog", "catalog": text, "format": fmt})
    for i in range(25):
        fmt = "json" if i % 3 == 0 else "csv"
        text = random_catalog_csv(rng, rng.randint(1, 6), [32, 64, 128], ["gemm", "fft", "winograd"], fmt)
        add({"op": "load_catalog", "catalog": text, "format": fmt, "batch": 64})

    # --- Eq 6 selection ------------------------------------------------------
    for _ in range(300):
        opts, bound = random_mckp(rng, 12, 3)
        add({"op": "solve", "options": opts, "bound": bound})
        add({"op": "solve", "options": opts, "bound": bound, "brute": True})
    for _ in range(40):
        opts, bound = random_mckp(rng, 40, 5)
        add({"op": "solve", "options": opts, "bound": bound})
    add({"op": "solve", "options": [[], []], "bound": 10})
    add({"op": "solve", "options": [[{"layer_id": 1, "algorithm": "a", "batch_size": 1,
                                       "time_seconds": 1.0, "memory_bits": 1}]] * 24,
         "bound": 100, "brute": True})
    big = [[{"layer_id": k, "algorithm": n, "batch_size": 1, "time_seconds": 1.0 + j,
             "memory_bits": 5 - j} for j, n in enumerate("abc")] for k in range(1, 16)]
    add({"op": "solve", "options": big, "bound": 40, "brute": True})  # 3^15 > 1e7
    add({"op": "solve", "options": big, "bound": 40})
    for b in (32, 64, 128, 256, 512):
        for bound in (-1, 0, 10**10, 5 * 10**10, 10**11, 10**12):
            add({"op": "solve_catalog", "catalog": profile, "batch": b, "bound": bound})
            add({"op": "solve_catalog", "catalog": profile, "batch": b, "bound": bound, "brute": True})
    add({"op": "catalog_options", "catalog": profile, "batch": 100})

    # --- §3.1.3 sweep --------------------------------------------------------
    for gib in (1, 4, 8, 12, 16, 24, 48, 180):
        add({"op": "plan_batch_size", "network": alex, "catalog": profile,
             "gpu_bits": gib * 2**30 * 8, "dataset": 1_281_167})
    add({"op": "plan_batch_size", "network": alex, "catalog": profile,
         "gpu_bits": 1_440_000_000_000, "dataset": 1_281_167})
    add({"op": "plan_batch_size", "network": SWEEP_NET, "catalog": sweep_catalog_csv(),
         "gpu_bits": 20_000_000, "dataset": 46_080, "candidates": [32, 64, 128, 256, 512]})
    add({"op": "plan_batch_size", "network": SWEEP_NET, "catalog": sweep_catalog_csv(),
         "gpu_bits": 20_000_000, "dataset": 46_080, "candidates": [512, 64, 64, 256]})
    add({"op": "plan_batch_size", "network": SWEEP_NET, "catalog": sweep_catalog_csv(),
         "gpu_bits": 10, "dataset": 46_080})
    add({"op": "plan_batch_size", "network": alex, "catalog": profile, "gpu_bits": 10**11,
         "dataset": 1000, "candidates": []})
    add({"op": "plan_batch_size", "network": alex, "catalog": profile, "gpu_bits": 10**11,
         "dataset": 0})
    add({"op": "plan_batch_size", "network": alex, "catalog": profile, "gpu_bits": 10**11,
         "dataset": 10, "candidates": [100]})
    add({"op": "plan_batch_size", "network": TOY_NET, "catalog": profile, "gpu_bits": 10**11,
         "dataset": 10})
    for _ in range(30):
        layers = rng.randint(1, 5)
        feats = [("conv", 3, 1, 1, rng.randint(1, 16)) for _ in range(layers)]
        net = structured((16, 16, 3), feats, (10,))
        cat = random_catalog_csv(rng, layers, [32, 64, 128, 256], ["fft", "gemm", "winograd"])
        add({"op": "plan_batch_size", "network": net, "catalog": cat,
             "gpu_bits": rng.randint(10**7, 10**10), "dataset": rng.randint(1, 10**6)})
    add({"op": "model_caveats"})

    # --- Lemma 1 / 2 ---------------------------------------------------------
    for g in range(0, 10):
        for r in (-0.1, 0.0, 0.01, 0.0259, 0.0625, 0.1, 0.2143, 1.0, 3.5):
            add({"op": "efficiency", "gpus": g, "r": r})
    for g in (0, 1, 2, 4, 8):
        for a in (0.1, 0.25, 0.5, 0.8, 0.85, 0.99, 1.0):
            add({"op": "max_overhead_ratio", "gpus": g, "alpha": a})
    for t in (0.5, 1, 2, 3, 3.2, 7, 11, 100):
        for r in (0.0, 0.01, 0.1, 0.5):
            add({"op": "recommend_gpus", "target": t, "r": r, "max_gpus": 8})
    add({"op": "scaling_table", "max_gpus": 8, "r": 0.1})
    add({"op": "scaling_table", "max_gpus": 0, "r": 0.1})
    for _ in range(200):
        add({"op": "min_parameter_servers", "workers": rng.randint(1, 128),
             "param_bytes": rng.uniform(1.0, 2e9), "bandwidth": rng.uniform(1e6, 2e10),
             "compute_time": rng.uniform(1e-3, 20.0)})
    add({"op": "min_parameter_servers", "workers": 4, "param_bytes": 180e6,
         "bandwidth": 1.25e9, "compute_time": 1.0})
    add({"op": "min_parameter_servers", "workers": 0, "param_bytes": 1.0, "bandwidth": 1.0,
         "compute_time": 1.0})
    add({"op": "min_parameter_servers", "workers": 1, "param_bytes": 0.0, "bandwidth": 1.0,
         "compute_time": 1.0})
    add({"op": "estimate_overhead_ratio", "trace": steps})
    for t in BAD_TRACES:
        add({"op": "estimate_overhead_ratio", "trace": t})

    # --- units, number text --------------------------------------------------
    for s in UNIT_STRINGS:
        add({"op": "parse_bytes", "text": s})
        add({"op": "parse_bandwidth", "text": s})
    for v in (0.0, 1.0, 1023.0, 1024.0, 1536.5, 2.0**30 * 12, 1e15, -2048.0):
        add({"op": "human_bytes", "value": v})
    for v in (0.1, 1 / 3, 0.0864, 1e-300, 123456789.123, 0.068160000000000004, 2.5e-7):
        add({"op": "to_shortest_string", "value": v})
    for s in ("12", " 12 ", "1.5", "1e3", "+4", "-4", "0x10", "", "12a", "inf", "\t7\r"):
        add({"op": "parse_number", "text": s})
    return cases


B200_DIR = os.path.join(HERE, "golden", "b200")


def b200(name: str) -> str:
    with open(os.path.join(B200_DIR, name)) as f:
        return f.read()


def build_b200_cases() -> list[dict]:
    """Decisions re-driven by catalogs MEASURED on B200 (scripts/b200_plan.py):
    the mini-batch sweep at several GPU memory sizes (from 180 GB down to sizes
    where feature maps no longer fit) and Eq 6 selection on the 94-layer
    Inception-v3 catalog under loose and binding workspace bounds."""
    cases = []
    for tag in ("alexnet", "vgg16"):
        net, cat = b200(f"b200_{tag}.net"), b200(f"b200_catalog_{tag}.csv")
        for gbits in (180 * 10**9 * 8, 12 * 2**30 * 8, 4 * 2**30 * 8, 2 * 2**30 * 8, 2**30 * 8,
                      3 * 10**8 * 8):
            cases.append({"op": "plan_batch_size", "network": net, "catalog": cat,
                          "gpu_bits": gbits, "dataset": 1_281_167})
    inc = b200("b200_catalog_inception_v3.csv")
    lo = None
    import csv as _csv
    import io as _io
    rows = list(_csv.DictReader(_io.StringIO(inc)))
    per = {}
    for r in rows:
        per.setdefault(int(r["layer_id"]), []).append(int(r["memory_bits"]))
    lo = sum(min(v) for v in per.values())
    hi = sum(max(v) for v in per.values())
    for bound in (lo - 1, lo, lo + (hi - lo) // 100, lo + (hi - lo) // 10, lo + (hi - lo) // 2, hi):
        cases.append({"op": "solve_catalog", "catalog": inc, "batch": 128, "bound": bound})
    return cases


def build_plan_cases(fixture_dir: str) -> list[dict]:
    """Full run_plan / renderer cases (file-path based)."""
    net = os.path.join(fixture_dir, "alexnet.net")
    cat = os.path.join(fixture_dir, "alexnet_profile.csv")
    cat_json = os.path.join(fixture_dir, "alexnet_profile_batch128.json")
    base = {"op": "run_plan", "network_path": net, "catalog_path": cat,
            "dataset": 1_281_167, "timestamp": "2026-01-01T00:00:00Z"}
    cases = []
    for gib in (12, 180):
        cases.append(dict(base, gpu_bits=gib * 2**30 * 8, workers=4, ro=0.1, verify=True))
    cases.append(dict(base, gpu_bits=1, workers=4, ro=0.1))
    cases.append(dict(base, gpu_bits=12 * 2**30 * 8, candidates=[64, 128], max_gpus=4,
                      param_size=180e6, bandwidth=1.25e9, workers=2, ro=0.05))
    cases.append(dict(base, catalog_path=cat_json, gpu_bits=12 * 2**30 * 8))
    cases.append(dict(base, catalog_path=cat_json, gpu_bits=12 * 2**30 * 8, candidates=[128]))
    cases.append(dict(base, network_path=net + ".missing", gpu_bits=12 * 2**30 * 8))
    cases.append({"op": "render_scale", "r": 0.1, "max_gpus": 8, "target": 3.0,
                  "timestamp": "T"})
    cases.append({"op": "render_scale", "r": 0.0, "max_gpus": 4, "target": 9.0,
                  "timestamp": "T"})
    cases.append({"op": "render_scale", "r": 0.5, "max_gpus": 8, "target": 2.5,
                  "timestamp": "T"})
    cases.append({"op": "render_scale", "r": 0.1, "max_gpus": 2, "target": 5.0,
                  "steps_path": "x.txt", "timestamp": "T"})
    cases.append({"op": "render_ps", "workers": 4, "param_bytes": 180e6, "bandwidth": 1.25e9,
                  "compute_time": 1.0, "timestamp": "T"})
    return cases
