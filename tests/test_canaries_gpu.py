"""Out-of-bounds and race checks without compute-sanitizer (closed on this
pool: runs under it left GPUs needing a reset — profiles/r02_compute_sanitizer_refused.log).
Every tensor-core conv path writes into an output, and uses a workspace,
that sit between 1 MiB guard regions filled with a NaN pattern: after fwd /
dgrad / wgrad the guards must be bit-identical (no stray TMA store, epilogue
or split-K partial write), and a second identical launch must reproduce the
first bit for bit (no race between the producer / MMA / epilogue roles or
between CTAs of the split-K reduction). Operand paths: auto (window / im2col /
plain TMA, CTA pairs, TMA-store epilogue), cp.async gather, and the window
path wherever it applies."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GUARD = 1 << 20  # bytes
CASES = [  # n h w c k r pad stride
    (3, 56, 56, 64, 64, 3, 1, 1),     # window fwd / dgrad / wgrad
    (2, 28, 28, 128, 128, 3, 1, 1),   # im2col TMA, CTA pairs, 384-column wgrad tiles
    (4, 14, 14, 256, 1024, 1, 0, 1),  # plain TMA, TMA-store epilogue, split-K wgrad
    (2, 28, 28, 256, 512, 1, 0, 2),   # strided 1x1: dgrad phases incl. empty ones
    (3, 9, 11, 40, 72, 3, 1, 2),      # gather path, ragged tails
    (2, 35, 35, 64, 64, 5, 2, 1),     # 5x5 window
    (8, 7, 7, 512, 4096, 7, 0, 1),    # fully connected: split-K forward + reduce
    (4, 14, 14, 512, 512, 3, 1, 1),   # 512-column CTA-pair wgrad tiles
    (2, 28, 28, 128, 128, 3, 1, 2),   # strided 3x3 dgrad phases, staged register epilogue
]


def _guarded(nbytes, device="cuda"):
    """(whole buffer, middle view as uint8) with NaN-pattern guards both sides."""
    buf = torch.empty(GUARD * 2 + nbytes, dtype=torch.uint8, device=device)
    buf.fill_(0xFF)
    return buf, buf[GUARD:GUARD + nbytes]


def _guards_ok(buf):
    return bool((buf[:GUARD] == 0xFF).all()) and bool((buf[-GUARD:] == 0xFF).all())


@pytest.fixture(params=[0, 1, 4], ids=["auto", "gather", "allwin"])
def path(request):
    from paper_1709_06622_b200 import device
    L = device.lib()
    L.tcb_set_conv_operand_path.argtypes = [ctypes.c_int]
    L.tcb_set_conv_operand_path(request.param)
    yield request.param
    L.tcb_set_conv_operand_path(0)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_conv_outputs_and_workspace_stay_in_bounds(case, path):
    from paper_1709_06622_b200 import device
    n, h, w, c, k, r, pad, stride = case
    g = device.geom(n, h, w, c, k, r, pad=pad, stride=stride)
    plan = device.ConvPlan(g, "gemm", "bf16")
    wsbuf, ws = _guarded(plan.workspace_bytes)
    ws.zero_()
    plan.workspace = ws
    bf = torch.bfloat16
    x = torch.randn(n, h, w, c, device="cuda").to(bf)
    wt = (torch.randn(k, r, r, c, device="cuda") * 0.05).to(bf)
    dy = torch.randn(n, g.ho, g.wo, k, device="cuda").to(bf)
    res = torch.randn(n, g.ho, g.wo, k, device="cuda").to(bf)
    outs = {}
    for name, shape, dt in (("y", (n, g.ho, g.wo, k), bf), ("dx", (n, h, w, c), bf), ("dw", (k, r, r, c), torch.float32)):
        numel = 1
        for d in shape:
            numel *= d
        esz = torch.tensor([], dtype=dt).element_size()
        buf, mid = _guarded(numel * esz)
        outs[name] = (buf, mid.view(dt).view(*shape))
    runs = []
    for _ in range(2):
        plan.fwd(x, wt, residual=res, relu=True, out=outs["y"][1])
        plan.dgrad(dy, wt, mask=x, out=outs["dx"][1])
        plan.wgrad(dy, x, out=outs["dw"][1])
        torch.cuda.synchronize()
        runs.append([outs[k_][1].clone() for k_ in ("y", "dx", "dw")])
    for name, (buf, _) in outs.items():
        assert _guards_ok(buf), f"{name}: write outside the tensor"
    assert _guards_ok(wsbuf), "workspace overrun"
    for a, b_ in zip(*runs):
        assert torch.equal(a, b_), "not bitwise reproducible"


@pytest.mark.parametrize("case", [(4, 28, 28, 64, 64), (4, 28, 28, 256, 128), (8, 14, 14, 128, 256)],
                         ids=lambda c: "x".join(map(str, c)))
def test_tma_epilogue_many_tiles_per_cta(case):
    """1x1 K-light passes with more tiles than SMs (every CTA loops over several
    tiles): side inputs double-buffered across tiles (residual / mask) must
    stay in order; compared against the register-epilogue path."""
    from paper_1709_06622_b200 import device
    n, h, w, c, k = case
    n *= 16  # > 148 tiles of 128 rows
    g = device.geom(n, h, w, c, k, 1)
    plan = device.ConvPlan(g, "gemm", "bf16")
    bf = torch.bfloat16
    x = torch.randn(n, h, w, c, device="cuda").to(bf)
    wt = (torch.randn(k, 1, 1, c, device="cuda") * 0.1).to(bf)
    res = torch.randn(n, h, w, k, device="cuda").to(bf)
    dy = torch.randn(n, h, w, k, device="cuda").to(bf)
    L = device.lib()
    L.tcb_set_conv_operand_path.argtypes = [ctypes.c_int]
    outs = []
    try:
        for mode in (0, 2):  # auto (TMA epilogue) / register epilogue
            L.tcb_set_conv_operand_path(mode)
            y = plan.fwd(x, wt, residual=res, relu=True)
            dx = plan.dgrad(dy, wt, residual=x, mask=x)
            dx2 = plan.dgrad(dy, wt, mask=x)
            torch.cuda.synchronize()
            outs.append((y, dx, dx2))
    finally:
        L.tcb_set_conv_operand_path(0)
    for a, b_ in zip(*outs):
        assert torch.equal(a, b_)
