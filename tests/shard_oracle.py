"""CPU restatement of the parameter-server shard layout — TEST INFRASTRUCTURE.

The reference has no layer-to-PS-shard code: Lemma 2 returns only a count
(/root/reference/proj/src/scale_plan.cpp:93-112) and the paper assumes an even
split. SURVEY §8 a15 fixes the definition this
build implements (csrc/runtime/trainer.cpp plan_params) and this file restates
independently: conv layers 1..q (fc = whole-map conv) flattened in layer
order, [K][R][S][C] weights then bias, each segment padded to 64 elements, the
total padded to G*64; rank r owns [r*P/G, (r+1)*P/G). Channel counts are the
allocated ones (bf16 pads K and the input C to multiples of 8).
"""
from __future__ import annotations

ALIGN = 64


def _up(v, a):
    return (v + a - 1) // a * a


def _pad(cfg):
    # tensor-core layouts pad channels to 16-byte rows: 8 bf16 / 4 fp32 (tf32)
    return {"bf16": 8, "tf32": 4}.get(cfg.get("precision", "bf16"), 1)


def _k_alloc(L, cfg, concat_inputs):
    # bf16 rounds a conv's K up to 64 when K < 64, or when a spatial (R*S > 1) conv
    # reads it and K % 64 != 0 — unless the tensor feeds a concat
    spatial = {x["in"] for x in cfg["layers"] if x["op"] == "conv" and x["r"] * x["s"] > 1}
    if cfg.get("precision", "bf16") == "bf16" and cfg.get("pad_narrow_channels", True) \
            and L["name"] not in concat_inputs \
            and (L["k"] < 64 or (L["k"] % 64 and L["name"] in spatial)):
        return _up(L["k"], 64)
    return _up(L["k"], _pad(cfg))


def _concat_inputs(cfg):
    return {x for L in cfg["layers"] if L["op"] == "concat" for x in L["in"]}


def layout(cfg: dict, world: int) -> dict:
    pad = _pad(cfg)
    cat_in = _concat_inputs(cfg)
    ch = {}
    layers = []
    off = 0
    logical = 0
    for L in cfg["layers"]:
        if L["op"] == "input":
            ch[L["name"]] = (_up(L["c"], pad), L["c"])
        elif L["op"] == "conv":
            c_alloc, c_log = ch[L["in"]]
            k_alloc = _k_alloc(L, cfg, cat_in)
            ch[L["name"]] = (k_alloc, L["k"])
            wcount = k_alloc * L["r"] * L["s"] * c_alloc
            entry = {"name": L["name"], "woff": off, "wcount": wcount, "boff": None}
            off = _up(off + wcount, ALIGN)
            logical += L["k"] * L["r"] * L["s"] * c_log
            if L.get("bias"):
                entry["boff"] = off
                off = _up(off + k_alloc, ALIGN)
                logical += L["k"]
            layers.append(entry)
        elif L["op"] in ("maxpool", "avgpool"):
            ch[L["name"]] = ch[L["in"]]
        elif L["op"] == "concat":
            ch[L["name"]] = (sum(ch[x][0] for x in L["in"]), sum(ch[x][1] for x in L["in"]))
    padded = _up(max(off, 1), world * ALIGN)
    shard = padded // world
    for e in layers:
        end = e["boff"] + _k_of(e, cfg) if e["boff"] is not None else e["woff"] + e["wcount"]
        e["shards"] = [e["woff"] // shard, (end - 1) // shard]
    return {"param_count": logical, "param_padded": padded, "shard": shard, "layers": layers}


def _k_of(entry, cfg):
    for L in cfg["layers"]:
        if L.get("name") == entry["name"]:
            return _k_alloc(L, cfg, _concat_inputs(cfg))
    raise KeyError(entry["name"])


def owner_of(flat_index: int, lay: dict) -> int:
    return flat_index // lay["shard"]
