"""B200 profiler -> reference cost catalog -> traincap planner.

`profile()` drives `tcb_profile_catalog` (C++, csrc/runtime/profiler.cpp):
every (conv layer, algorithm, mini-batch) is timed on the GPU and emitted as
the reference's CostEntry CSV. `plan()` feeds that catalog and the network
(the reference's `.net` format) to this build's traincap planner
(`plan_batch_size`, Eq 2-6 + §3.1.3), exactly as the reference's `run_plan`
consumes a profiled catalog (/root/reference/proj/src/report.cpp:57-108).
"""
from __future__ import annotations

import ctypes
import json

from . import device, models, planner


def profile(layers: list[dict], batches: list[int], algorithms=("gemm", "winograd", "fft"),
            precision: str = "bf16", reps: int = 5) -> dict:
    L = device.lib()
    L.tcb_profile_catalog.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
    L.tcb_free.argtypes = [ctypes.c_void_p]
    req = {"layers": layers, "batches": list(batches), "algorithms": list(algorithms),
           "precision": precision, "reps": reps}
    out = ctypes.c_char_p()
    device.check(L.tcb_profile_catalog(json.dumps(req).encode(), ctypes.byref(out)))
    d = json.loads(out.value.decode())
    L.tcb_free(ctypes.cast(out, ctypes.c_void_p))
    return d


def conv_layer_specs(cfg: dict) -> list[dict]:
    """Per-image conv geometries (layer order) of a model config, with the
    executor's channel allocation (c_alloc / k_alloc / c_valid from
    tcb_trainer_describe — no GPU needed) so a profiled catalog times exactly
    the convs the training step runs."""
    specs = [{k: g[k] for k in ("h", "w", "c", "k", "r", "s", "pad_h", "pad_w", "stride_h", "stride_w")}
             for _, g in models.conv_layers(cfg)]
    try:
        import ctypes as _ct

        from . import trainer as _tr
        L = _tr._lib()
        h = _ct.c_void_p()
        device.check(L.tcb_trainer_create(json.dumps(cfg).encode(), _ct.byref(h)))
        out = _ct.c_char_p()
        device.check(L.tcb_trainer_describe(h, _ct.byref(out)))
        d = json.loads(out.value.decode())
        L.tcb_free(_ct.cast(out, _ct.c_void_p))
        L.tcb_trainer_destroy(h)
    except device.TcbError:
        return specs
    convs = [x for x in d["layers"] if x["op"] == "conv"]
    for sp, x in zip(specs, convs):
        n, h, w, c, k = x["geom"][:5]
        sp["c_alloc"], sp["k_alloc"] = c, k
        cl = d["layers"][x["in"]]["c_logical"]
        if cl < c:
            sp["c_valid"] = cl
    return specs


def net_text(cfg: dict) -> str:
    """The reference `.net` description of a chain model: feature layers
    (conv/pool), then the classifier as `fc` lines starting with the flattened
    feature vector (the junction convention of SURVEY §0.6: `fc 9216` first for
    AlexNet-227, so parameter_bits counts the flatten->fc1 weights). Layers
    named `fc*` are whole-map convs (this build's fc layers)."""
    lines, fcs = [], []
    shape = None
    for L in cfg["layers"]:
        if L["op"] == "input":
            lines.append(f"input {L['w']} {L['h']} {L['c']}")
            shape = (L["h"], L["w"], L["c"])
        elif L["op"] == "conv" and L["name"].startswith("fc"):
            if not fcs:
                fcs.append(shape[0] * shape[1] * shape[2])
            fcs.append(L["k"])
        elif L["op"] == "conv":
            if L["r"] != L["s"] or L["pad_h"] != L["pad_w"] or L["stride_h"] != L["stride_w"]:
                raise ValueError("the reference network model needs square filters")
            lines.append(f"conv {L['r']} {L['stride_h']} {L['pad_h']} {L['k']}")
            shape = ((shape[0] + 2 * L["pad_h"] - L["r"]) // L["stride_h"] + 1,
                     (shape[1] + 2 * L["pad_w"] - L["s"]) // L["stride_w"] + 1, L["k"])
        elif L["op"] == "maxpool":
            lines.append(f"pool {L['f']} {L['stride']} {L['pad']}")
            shape = ((shape[0] + 2 * L["pad"] - L["f"]) // L["stride"] + 1,
                     (shape[1] + 2 * L["pad"] - L["f"]) // L["stride"] + 1, shape[2])
    lines += [f"fc {n}" for n in fcs]
    return "\n".join(lines) + "\n"


def feature_conv_specs(cfg: dict) -> list[dict]:
    """Conv layers the catalog indexes (the feature chain; fc layers excluded,
    matching NetworkSpec::convolution_layer_count)."""
    names = [n for n, _ in models.conv_layers(cfg)]
    return [s for n, s in zip(names, conv_layer_specs(cfg)) if not n.startswith("fc")]


def plan(net: str, catalog_csv: str, gpu_bits: int, dataset: int, candidates=None,
         planner_handle=None) -> dict:
    p = planner_handle or planner.default()
    req = dict(network=net, catalog=catalog_csv, gpu_bits=gpu_bits, dataset=dataset)
    if candidates:
        req["candidates"] = list(candidates)
    return p.call("plan_batch_size", **req)


def layout(cfg: dict) -> dict:
    """The executor's exact HBM layout of `cfg` (no GPU, no allocation):
    arena / algorithm-workspace / resident bytes (tcb_trainer_layout)."""
    import ctypes
    import json

    from . import device
    L = device.lib()
    L.tcb_trainer_layout.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
    L.tcb_free.argtypes = [ctypes.c_void_p]
    out = ctypes.c_char_p()
    device.check(L.tcb_trainer_layout(json.dumps(cfg).encode(), ctypes.byref(out)))
    d = json.loads(out.value.decode())
    L.tcb_free(ctypes.cast(out, ctypes.c_void_p))
    return d


def plan_graph(build, catalog_csv: str, batches, gpu_bits: int, dataset: int, planner_handle=None) -> dict:
    """Mini-batch + per-layer algorithm plan for a branched network (ResNet,
    Inception): `build(batch) -> cfg`; each candidate's
    workspace bound is gpu_bits minus the executor's resident bits at that
    batch (its exact layout without conv workspaces), then the reference's
    selection / epoch-time / recommendation rules (plan_batch_size_resident)."""
    p = planner_handle or planner.default()
    resident = {str(b): layout(build(b))["resident_bytes"] * 8 for b in batches}
    return p.call("plan_batch_size_graph", catalog=catalog_csv, resident_bits=resident, gpu_bits=gpu_bits,
                  dataset=dataset)
