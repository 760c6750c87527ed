"""Planner for branched networks: the executor's exact HBM
layout (tcb_trainer_layout, no GPU) as the memory model of ResNet / Inception,
fed to plan_batch_size_resident.

Pins: (1) on a chain network, handing plan_batch_size_resident the chain
model's own Eq 2-5 bits reproduces plan_batch_size exactly (same selections,
bit-identical epoch times, same recommendation) on the reference's AlexNet
fixture — the new entry point only swaps the memory model; (2) the layout's
resident bytes are the arena minus the conv workspaces and grow with the
batch; (3) on a synthetic Inception-v3 catalog the plan follows the
reference's rules (fastest algorithm per layer when the bound is loose, the
low-memory one when it binds, infeasible candidates skipped, min epoch time).
Runs on CPU."""
import pytest

import planner_cases


def _models():
    from paper_1709_06622_b200 import models
    return models


def test_resident_entry_point_equals_chain_plan(planner_lib):
    p = planner_lib
    net = planner_cases.fixture("alexnet.net")
    cat = planner_cases.fixture("alexnet_profile.csv")
    gpu = 12 * 2**30 * 8
    ref = p.call("plan_batch_size", network=net, catalog=cat, gpu_bits=gpu, dataset=1_281_167)
    resident = {}
    for c in ref["candidates"]:
        bd = c["breakdown"]
        resident[str(c["batch_size"])] = bd["feature_maps"] + bd["model_params"] + bd["classifier"]
    got = p.call("plan_batch_size_graph", catalog=cat, resident_bits=resident, gpu_bits=gpu,
                 dataset=1_281_167)
    assert got["recommended"] == ref["recommended"] == 128
    for a, b in zip(got["candidates"], ref["candidates"]):
        assert a["batch_size"] == b["batch_size"]
        assert a["breakdown"]["bound"] == b["breakdown"]["bound"]
        assert a["epoch_time_seconds"] == b["epoch_time_seconds"]
        assert a["solve"] == b["solve"]
        assert a["memory_limited_layers"] == b["memory_limited_layers"]


@pytest.mark.parametrize("model,batches", [("resnet50", (32, 64, 128, 256)),
                                           ("inception_v3", (32, 64, 128))])
def test_layout_is_the_exact_memory_model(model, batches):
    from paper_1709_06622_b200 import profiler
    m = _models()
    prev = 0
    for b in batches:
        lay = profiler.layout(m.build(model, batch=b))
        assert lay["arena_bytes"] == lay["resident_bytes"] + lay["algorithm_workspace_bytes"]
        assert lay["resident_bytes"] > prev
        prev = lay["resident_bytes"]
    assert lay["conv_layers"] == {"resnet50": 54, "inception_v3": 95}[model]


def _synthetic_catalog(n_layers, batches):
    """gemm: time 1e-4*b*(1+l%5), 1 Mbit workspace; winograd on every 3rd
    layer (31 of 94): 40% faster but 0.5 Gbit * b/32 of workspace."""
    rows = ["layer_id,algorithm,batch_size,time_seconds,memory_bits"]
    for l in range(1, n_layers + 1):
        for b in batches:
            t = 1e-4 * b * (1 + l % 5)
            rows.append(f"{l},gemm,{b},{t!r},{10**6}")
            if l % 3 == 0:
                rows.append(f"{l},winograd,{b},{t * 0.6!r},{5 * 10**8 * b // 32}")
    return "\n".join(rows) + "\n"


def test_inception_plan_follows_reference_rules(planner_lib):
    from paper_1709_06622_b200 import profiler
    m = _models()
    convs = [n for n, _ in m.conv_layers(m.inception_v3(batch=2)) if not n.startswith("fc")]
    assert len(convs) == 94
    batches = (32, 64, 128, 256)
    cat = _synthetic_catalog(94, batches)
    res = {b: profiler.layout(m.inception_v3(batch=b))["resident_bytes"] * 8 for b in batches}
    # HBM such that 256 does not fit at all and 128 affords only 30 of the 31
    # Winograd workspaces (2 Gbit each at 128)
    gpu = res[128] + 30 * 2 * 10**9 + 94 * 10**6
    assert res[256] > gpu
    plan = profiler.plan_graph(lambda b: m.inception_v3(batch=b), cat, batches, gpu, 1_281_167,
                               planner_handle=planner_lib)
    by_b = {c["batch_size"]: c for c in plan["candidates"]}
    assert by_b[256]["solve"]["feasible"] is False and by_b[256]["epoch_time_seconds"] is None
    # loose at 32 / 64: every 3rd layer takes the faster Winograd
    for b in (32, 64):
        sel = by_b[b]["solve"]["assignment"]
        assert all(sel[str(l)] == ("winograd" if l % 3 == 0 else "gemm") for l in range(1, 95))
        assert by_b[b]["memory_limited_layers"] == []
    # binding at 128: one Winograd layer must fall back to GEMM (the cheapest
    # one to give up), within the bound, reported as memory-limited
    c128 = by_b[128]
    assert c128["solve"]["feasible"]
    assert c128["solve"]["total_memory"] <= c128["breakdown"]["bound"]
    assert len(c128["memory_limited_layers"]) == 1
    assert sum(a == "winograd" for a in c128["solve"]["assignment"].values()) == 30
    epochs = {b: c["epoch_time_seconds"] for b, c in by_b.items() if c["epoch_time_seconds"]}
    best = min(epochs.values())
    assert plan["recommended"] == max(b for b, e in epochs.items() if e == best)
