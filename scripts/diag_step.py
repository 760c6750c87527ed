"""Per-tensor diagnosis of one executor step vs the oracle step (GPU box).

    python scripts/diag_step.py [model] [precision] [batch]

For every conv it also recomputes wgrad through the oracle from the DEVICE's
own operands, separating kernel error from propagated bf16 rounding.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import oracle_binding  # noqa: E402
import oracle_step  # noqa: E402
from oracle_binding import rel_err  # noqa: E402
from paper_1709_06622_b200 import models  # noqa: E402
from paper_1709_06622_b200.trainer import Trainer  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "tiny_resnet"
precs = [sys.argv[2]] if len(sys.argv) > 2 else ["ffma", "bf16"]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 4
o = oracle_binding.Oracle("oracle/liboracle.so")
for prec in precs:
    cfg = models.build(model, batch=batch, precision=prec)
    t = Trainer(cfg)
    t.step()
    torch.cuda.synchronize()
    lay = t.describe()
    ref = oracle_step.OracleStep(o, cfg, lay)
    ref.run()
    print(prec, model, "loss", t.loss(), ref.loss)
    gd = t.tensor("grad").cpu().numpy()
    gr = ref.flat_grad()
    for L in lay["layers"][1:-1]:
        i = L["index"]
        shp, cl = L["shape"], L["c_logical"]
        a = t.tensor(f"act:{i}").float().cpu().numpy().reshape(shp)[..., :cl]
        g = t.tensor(f"dact:{i}").float().cpu().numpy().reshape(shp)[..., :cl]
        rg = ref.G.get(i)
        line = f"  {L['name']:12s} act {rel_err(a, ref.act[i]):.2e} grad {rel_err(g, rg):.2e}"
        if L["op"] == "conv":
            sl = slice(L["woff"], L["woff"] + L["wcount"])
            xin_l = lay["layers"][L["in"]]
            x = t.tensor(f"act:{L['in']}").float().cpu().numpy().reshape(xin_l["shape"])[..., :xin_l["c_logical"]]
            geo = ref._geom(L, x.shape[-1])
            dw_local = o.conv_wgrad(geo, g, x)
            ka, r, s, cp = L["geom"][4], L["geom"][5], L["geom"][6], L["geom"][3]
            w4 = np.zeros((ka, r, s, cp))
            w4[:cl, ..., :x.shape[-1]] = dw_local.reshape(cl, r, s, x.shape[-1])
            line += f" | W vs oracle-step {rel_err(gd[sl], gr[sl]):.2e}  W vs oracle(dev operands) {rel_err(gd[sl], w4.ravel()):.2e}"
        print(line)
