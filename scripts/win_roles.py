"""Per-role timing of the window conv kernel (clock64 inside the kernel via
tcb_conv_win_debug): producer / MMA issuer / epilogue busy vs waiting.
    python scripts/win_roles.py N H W C K R S PAD PASS"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1709_06622_b200 import device  # noqa: E402

a = sys.argv[1:]
n, h, w, c, k, r, s, pad = (int(v) for v in a[:8])
pss = a[8]
g = device.geom(n, h, w, c, k, r, s, pad=pad)
plan = device.ConvPlan(g, "gemm", "bf16")
x = torch.randn(n, h, w, c, device="cuda").bfloat16()
wt = (torch.randn(k, r, s, c, device="cuda") * 0.05).bfloat16()
dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
fn = {"fwd": lambda: plan.fwd(x, wt), "dgrad": lambda: plan.dgrad(dy, wt)}[pss]
for _ in range(3):
    fn()
buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
L = device.lib()
L.tcb_conv_win_debug.argtypes = [ctypes.c_void_p]
L.tcb_conv_win_debug(ctypes.c_void_p(buf.data_ptr()))
fn()
torch.cuda.synchronize()
L.tcb_conv_win_debug(None)
info = device.last_launch()
d = buf.view(148, 8).cpu().numpy().astype("uint64")
grid = info["grid"]
d = d[:grid]
lead = d[::2] if info["cta2"] else d
out = {"info": info,
       "producer_total": float(d[:, 0].mean()), "producer_wait_win_slot": float(d[:, 1].mean()),
       "producer_wait_b_slot": float(d[:, 2].mean()),
       "mma_total": float(lead[:, 3].mean()), "mma_wait_acc": float(lead[:, 4].mean()),
       "mma_wait_window": float(lead[:, 5].mean()), "mma_wait_b": float(lead[:, 6].mean()),
       "epi_total": float((d[:, 7] >> 32).mean()), "epi_wait_tfull": float((d[:, 7] & 0xffffffff).mean())}
print(json.dumps(out))
