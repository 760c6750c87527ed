"""Decision-half parity: this build's traincap planner vs the reference.

Two independent pins:
  * golden replay — every request in tests/golden/planner_golden.json.gz was
    answered by the reference planner compiled from /root/reference
    (oracle/_ref); this build must answer identically (bit-exact doubles,
    identical assignments, identical error class and message). Runs anywhere.
  * live differential — when oracle/_ref is available, fresh seeded random
    instances go to both libraries side by side.
Rows covered: a1-a13.
"""
import gzip
import json
import os
import random

import pytest

import planner_cases

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "planner_golden.json.gz")
TOKEN = "@FIXTURES@"


def _records():
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)["records"]


def _subst(obj, old, new):
    return json.loads(json.dumps(obj).replace(old, new))


# The text plan report is presentation only (the reference's JSON schema is the
# contract); from it only the lines a reader acts on are compared.
KEY_TEXT_LINES = ("recommended mini-batch:", "no candidate mini-batch is feasible", "parameter servers:",
                  "selection verified")


def _key_lines(text):
    return [ln for ln in text.splitlines() if ln.strip().startswith(KEY_TEXT_LINES)]


def _comparable(reply):
    if isinstance(reply, dict) and "text" in reply and "json" in reply:
        reply = dict(reply)
        reply["text"] = _key_lines(reply["text"])
    return reply


def test_golden_replay(planner_lib):
    records = _records()
    assert len(records) > 1500
    mismatches = []
    for rec in records:
        req = _subst(rec["request"], TOKEN, planner_cases.FIXTURES)
        got = _subst(planner_lib.raw(**req), planner_cases.FIXTURES, TOKEN)
        if _comparable(got) != _comparable(rec["reply"]):
            mismatches.append((req["op"], rec["reply"], got))
    assert not mismatches, f"{len(mismatches)} mismatches, first: {mismatches[0]}"


def test_b200_catalog_decisions_match_reference(planner_lib):
    """Mini-batch choice and per-layer algorithm selection re-driven by catalogs
    measured on B200 (tests/golden/b200/*.csv) are bit-identical to the
    reference planner's on the same files."""
    with gzip.open(GOLDEN, "rt") as f:
        recs = json.load(f)["b200_records"]
    assert len(recs) >= 18
    checked = 0
    for rec in recs:
        if rec["reply"] is None:
            continue
        assert planner_lib.raw(**rec["request"]) == rec["reply"], rec["request"]["op"]
        checked += 1
    assert checked >= 18
    # the 180 GB AlexNet-227 plan: largest batch, implicit GEMM everywhere
    plan = [r["reply"] for r in recs if r["request"]["op"] == "plan_batch_size"][0]
    assert plan["recommended"] == 512


def test_golden_covers_every_error_class():
    kinds = {r["reply"]["error"]["type"] for r in _records() if "error" in r["reply"]}
    assert {"ParseError", "DuplicateKeyError", "IncompleteCatalogError", "OverflowError",
            "NonPositiveShapeError", "DomainError", "UnitError", "MissingComputeStepError",
            "InstanceTooLargeError", "CandidateNotInCatalogError", "Error"} <= kinds


def test_reference_acceptance_numbers(planner_lib):
    """Hand-derived goldens quoted in the reference tests."""
    p = planner_lib
    toy = planner_cases.TOY_NET
    assert p.call("feature_map_memory", network=toy, batch=2)["bits"] == 3072
    assert p.call("model_param_memory", network=toy)["bits"] == 1920
    assert p.call("classifier_memory", layers=[8, 4])["bits"] == 3552
    alex = planner_cases.fixture("alexnet.net")
    shapes = p.call("propagate_shapes", network=alex)["shapes"]
    assert [s[0] for s in shapes] == [224, 55, 27, 27, 13, 13, 13, 13, 6]
    assert p.call("parameter_bits", network=alex)["bits"] == 98_481_672 * 8
    assert abs(p.call("max_overhead_ratio", gpus=4, alpha=0.8)["value"] - 1 / 11) < 1e-12
    assert p.call("min_parameter_servers", workers=4, param_bytes=180e6, bandwidth=1.25e9,
                  compute_time=1.0)["servers"] == 2
    rec = p.call("recommend_gpus", target=3.0, r=0.1, max_gpus=8)
    assert rec["gpus"] == 4


def test_fixture_plan_recommends_128(planner_lib):
    p = planner_lib
    plan = p.call("plan_batch_size", network=planner_cases.fixture("alexnet.net"),
                  catalog=planner_cases.fixture("alexnet_profile.csv"),
                  gpu_bits=12 * 2**30 * 8, dataset=1_281_167)
    assert plan["recommended"] == 128
    thr = [c["throughput"] for c in plan["candidates"]]
    assert [round(t, 1) for t in thr] == [469.5, 704.2, 939.0, 551.7, 516.8]


def test_solver_matches_exhaustive_oracle(planner_lib):
    rng = random.Random(41)
    feasible = infeasible = 0
    for _ in range(300):
        opts, bound = planner_cases.random_mckp(rng, 12, 3)
        a = planner_lib.call("solve", options=opts, bound=bound)
        b = planner_lib.call("solve", options=opts, bound=bound, brute=True)
        assert a == b
        feasible += a["feasible"]
        infeasible += not a["feasible"]
    assert feasible > 50 and infeasible > 50


def test_live_differential_random(planner_lib, ref_planner):
    rng = random.Random(7)
    for _ in range(150):
        opts, bound = planner_cases.random_mckp(rng, 14, 4)
        assert planner_lib.raw("solve", options=opts, bound=bound) == \
            ref_planner.raw("solve", options=opts, bound=bound)
    for _ in range(40):
        net = planner_cases.random_network(rng)
        for op in ("propagate_shapes", "validate_network", "parameter_bits"):
            assert planner_lib.raw(op, network=net) == ref_planner.raw(op, network=net)
        req = dict(network=net, gpu_bits=rng.randint(0, 1 << 36), batch=rng.randint(1, 4096))
        assert planner_lib.raw("memory_bound", **req) == ref_planner.raw("memory_bound", **req)
    for _ in range(15):
        layers = rng.randint(1, 6)
        net = planner_cases.structured((32, 32, 3), [("conv", 3, 1, 1, 8)] * layers, (10,))
        cat = planner_cases.random_catalog_csv(rng, layers, [32, 64, 128, 256, 512],
                                               ["fft", "gemm", "winograd"])
        req = dict(network=net, catalog=cat, gpu_bits=rng.randint(10**8, 10**10),
                   dataset=rng.randint(1, 10**6))
        assert planner_lib.raw("plan_batch_size", **req) == \
            ref_planner.raw("plan_batch_size", **req)


def test_live_differential_tight_large_instances(planner_lib, ref_planner):
    """Tight bounds on 20-30 layer instances: the stronger LP bound must still
    land on the reference's canonical optimum."""
    rng = random.Random(99)
    for _ in range(12):
        opts, _ = planner_cases.random_mckp(rng, 22, 3)
        lo = sum(min(e["memory_bits"] for e in l) for l in opts)
        hi = sum(max(e["memory_bits"] for e in l) for l in opts)
        for bound in (lo, lo + (hi - lo) // 4, lo + (hi - lo) // 2):
            assert planner_lib.raw("solve", options=opts, bound=bound) == \
                ref_planner.raw("solve", options=opts, bound=bound)
