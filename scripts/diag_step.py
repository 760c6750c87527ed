import sys, numpy as np, torch
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import oracle_binding, oracle_step
from oracle_binding import rel_err
from paper_1709_06622_b200 import models
from paper_1709_06622_b200.trainer import Trainer
o = oracle_binding.Oracle('oracle/liboracle.so')
for prec in ("ffma","bf16"):
    cfg = models.tiny_resnet(batch=4, precision=prec)
    t = Trainer(cfg); t.step(); torch.cuda.synchronize()
    lay = t.describe(); ref = oracle_step.OracleStep(o, cfg, lay); ref.run()
    print(prec, "loss", t.loss(), ref.loss)
    # activations
    for L in lay["layers"][1:-1]:
        i = L["index"]
        shp = L["shape"]; cl = L["c_logical"]
        a = t.tensor(f"act:{i}").float().cpu().numpy().reshape(shp)[..., :cl]
        ra = ref.act[i]
        g = t.tensor(f"dact:{i}").float().cpu().numpy().reshape(shp)[..., :cl]
        rg = ref.G.get(i)
        print(f"  {L['name']:12s} act {rel_err(a, ra):.2e}  grad {rel_err(g, rg) if rg is not None else -1:.2e}  |g| {np.abs(g).max():.3e} |rg| {np.abs(rg).max() if rg is not None else 0:.3e}")
    gd = t.tensor("grad").cpu().numpy(); gr = ref.flat_grad()
    for L in lay["layers"]:
        if L["op"]!="conv": continue
        sl = slice(L["woff"], L["woff"]+L["wcount"])
        print(f"  W {L['name']:12s} {rel_err(gd[sl], gr[sl]):.2e}")
