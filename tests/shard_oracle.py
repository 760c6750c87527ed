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


def layout(cfg: dict, world: int) -> dict:
    pad = _pad(cfg)
    ch = {}
    layers = []
    off = 0
    logical = 0
    for L in cfg["layers"]:
        if L["op"] == "input":
            ch[L["name"]] = (_up(L["c"], pad), L["c"])
        elif L["op"] == "conv":
            c_alloc, c_log = ch[L["in"]]
            k_alloc = _up(L["k"], pad)
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
            return _up(L["k"], _pad(cfg))
    raise KeyError(entry["name"])


def owner_of(flat_index: int, lay: dict) -> int:
    return flat_index // lay["shard"]
