"""CPU restatement of the executor's model description — TEST INFRASTRUCTURE.

What `tcb_trainer_describe` reports (node shapes, allocated channels, conv
geometry, init scale, flat PS offsets), recomputed from the model config in
Python so the CPU oracle step (tests/oracle_step.py, bench.py's reference arm)
needs nothing from the product library. Follows the executor's rules
(csrc/runtime/trainer.cpp build_graph / plan_params) and the shard layout of
tests/shard_oracle.py; tests/test_shard_layout.py pins the two against
each other.
"""
from __future__ import annotations

import numpy as np

import shard_oracle


def describe(cfg: dict, world: int = 1) -> dict:
    pad = shard_oracle._pad(cfg)
    cat_in = shard_oracle._concat_inputs(cfg)
    flat = {e["name"]: e for e in shard_oracle.layout(cfg, world)["layers"]}
    sl = shard_oracle.layout(cfg, world)
    nodes, idx = [], {}
    n = cfg["batch"]
    conv_index = 0
    for L in cfg["layers"]:
        d = {"index": len(nodes), "name": L["name"], "op": L["op"], "in": -1, "residual": -1}
        op = L["op"]
        if op == "input":
            c = shard_oracle._up(L["c"], pad)
            d.update(shape=[n, L["h"], L["w"], c], c_logical=L["c"])
        elif op == "conv":
            x = nodes[idx[L["in"]]]
            d["in"] = idx[L["in"]]
            d["residual"] = idx[L["residual"]] if L.get("residual") else -1
            r, s = L["r"], L.get("s", L["r"])
            ph, pw = L.get("pad_h", L.get("pad", 0)), L.get("pad_w", L.get("pad", 0))
            sh, sw = L.get("stride_h", L.get("stride", 1)), L.get("stride_w", L.get("stride", 1))
            _, h, w, c = x["shape"]
            k_alloc = shard_oracle._k_alloc(L, cfg, cat_in)
            ho, wo = (h + 2 * ph - r) // sh + 1, (w + 2 * pw - s) // sw + 1
            conv_index += 1
            fan_in = x["c_logical"] * r * s
            scale = np.float32(L.get("init_gain", 1.0)) * np.sqrt(np.float32(6.0) / np.float32(fan_in))
            e = flat[L["name"]]
            d.update(shape=[n, ho, wo, k_alloc], c_logical=L["k"], conv_index=conv_index,
                     geom=[n, h, w, c, k_alloc, r, s, ph, pw, sh, sw], relu=bool(L.get("relu", False)),
                     bias=bool(L.get("bias", False)), woff=e["woff"], wcount=e["wcount"], boff=e["boff"],
                     init_scale=float(scale), algo=L.get("algo", "gemm"), shards=e["shards"])
        elif op in ("maxpool", "avgpool"):
            x = nodes[idx[L["in"]]]
            d["in"] = idx[L["in"]]
            _, h, w, c = x["shape"]
            if op == "maxpool" or "f" in L:
                f = L["f"]
                st = L.get("stride", f)
                p = L.get("pad", 0)
                d.update(shape=[n, (h + 2 * p - f) // st + 1, (w + 2 * p - f) // st + 1, c],
                         c_logical=x["c_logical"], pool=[f, st, p])
            else:
                d.update(shape=[n, 1, 1, c], c_logical=x["c_logical"])
        elif op == "concat":
            ins = [idx[nm] for nm in L["in"]]
            coff, tot = [], 0
            for j in ins:
                coff.append(tot)
                tot += nodes[j]["shape"][3]
            x = nodes[ins[0]]
            d.update(**{"in": ins[0]}, ins=ins, coff=coff, shape=[n, x["shape"][1], x["shape"][2], tot],
                     c_logical=tot)
        elif op == "loss":
            d.update(**{"in": idx[L["in"]]}, shape=[0, 0, 0, 0], c_logical=0)  # no tensor of its own
        idx[L["name"]] = d["index"]
        nodes.append(d)
    return {"precision": cfg.get("precision", "bf16"), "batch": n, "classes": cfg["classes"],
            "world": world, "param_count": sl["param_count"], "param_padded": sl["param_padded"],
            "shard": sl["shard"], "layers": nodes}
