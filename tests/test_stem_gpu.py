"""Row-window stem kernels (conv_stem.cu) against an fp64 PyTorch reference of
the same convolution and against the explicit-im2col GEMM path they replace.

Geometries: the ResNet-50 stem at full 224 width (Wo = 112, one tile per
output row), Inception-v3's 3x3/2 stem at 299 (Wo = 149: two tiles per row,
the second with out-of-range rows), an 11x11 stem (two 32-element chunks
per filter row, 11x11/2), and ragged small cases with 4 valid channels and K = 64 /
128. Inputs are 8-channel bf16 with channels >= c_valid zero, as the executor
stores the RGB input."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

# name, n, h, w, k, r, pad, stride, c_valid
STEMS = [
    ("rn50_224", 2, 224, 224, 64, 7, 3, 2, 3),
    ("rn50_small", 3, 32, 30, 64, 7, 3, 2, 3),
    ("incep_299", 2, 299, 299, 32, 3, 0, 2, 3),
    ("k11_s2", 2, 45, 43, 64, 11, 5, 2, 3),
    ("c4_5x5_ragged", 2, 21, 19, 64, 5, 2, 2, 4),
    ("c4_k128_3x3", 3, 17, 23, 128, 3, 1, 2, 4),
    ("k32_7x7_ragged", 2, 40, 37, 32, 7, 3, 2, 3),
]


def _lib():
    import ctypes
    from paper_1709_06622_b200 import device
    L = device.lib()
    L.tcb_set_conv_stem.argtypes = [ctypes.c_int]
    return device, L


def _inputs(case, seed):
    _, n, h, w, k, r, pad, stride, cv = case
    gen = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.rand(n, h, w, 8, device="cuda", generator=gen) * 2 - 1
    x[..., cv:] = 0
    wt = (torch.rand(k, r, r, 8, device="cuda", generator=gen) * 2 - 1) * (1.0 / (r * r * cv) ** 0.5)
    bias = torch.rand(k, device="cuda", generator=gen) * 0.2 - 0.1
    return x.bfloat16(), wt.bfloat16(), bias


def _ref_fwd(x, wt, bias, pad, stride, relu):
    y = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(0, 3, 1, 2),
                                   bias.double(), stride=stride, padding=pad)
    y = y.permute(0, 2, 3, 1)
    return torch.relu(y) if relu else y


def _ref_wgrad(dy, x, k, r, pad, stride):
    xd = x.double().permute(0, 3, 1, 2)
    dyd = dy.double().permute(0, 3, 1, 2)
    dw = torch.nn.grad.conv2d_weight(xd, (k, 8, r, r), dyd, stride=stride, padding=pad)
    return dw.permute(0, 2, 3, 1)


@pytest.fixture
def stem_on():
    _, L = _lib()
    L.tcb_set_conv_stem(1)
    yield L
    L.tcb_set_conv_stem(-1)


@pytest.mark.parametrize("case", STEMS, ids=[c[0] for c in STEMS])
def test_stem_fwd_and_wgrad_match_reference(case, stem_on):
    device, L = _lib()
    _, n, h, w, k, r, pad, stride, cv = case
    g = device.geom(n, h, w, 8, k, r, pad=pad, stride=stride)
    plan = device.ConvPlan(g, "gemm", "bf16").set_valid_channels(cv)
    x, wt, bias = _inputs(case, 11)
    y = plan.fwd(x, wt, bias=bias, relu=True)
    torch.cuda.synchronize()
    info = device.last_launch()
    assert info["load"] == 5, f"stem path not taken: {info}"
    ref = _ref_fwd(x, wt, bias, pad, stride, True)
    err = (y.double() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
    assert err < 8e-3, f"fwd rel err {err}"

    gen = torch.Generator(device="cuda").manual_seed(5)
    dy = (torch.rand(n, g.ho, g.wo, k, device="cuda", generator=gen) * 2 - 1).bfloat16()
    dw = plan.wgrad(dy, x)
    torch.cuda.synchronize()
    assert device.last_launch()["load"] == 5
    refw = _ref_wgrad(dy, x, k, r, pad, stride)
    errw = (dw.double() - refw).abs().max().item() / max(refw.abs().max().item(), 1e-6)
    assert errw < 2e-5, f"wgrad rel err {errw}"
    assert torch.count_nonzero(dw[..., cv:]) == 0  # padded channels get an exact zero gradient


@pytest.mark.parametrize("case", STEMS[:3], ids=[c[0] for c in STEMS[:3]])
def test_stem_matches_explicit_im2col_path(case):
    device, L = _lib()
    _, n, h, w, k, r, pad, stride, cv = case
    g = device.geom(n, h, w, 8, k, r, pad=pad, stride=stride)
    x, wt, bias = _inputs(case, 23)
    gen = torch.Generator(device="cuda").manual_seed(7)
    dy = (torch.rand(n, g.ho, g.wo, k, device="cuda", generator=gen) * 2 - 1).bfloat16()
    outs = []
    try:
        for on in (1, 0):
            L.tcb_set_conv_stem(on)
            plan = device.ConvPlan(g, "gemm", "bf16").set_valid_channels(cv)
            y = plan.fwd(x, wt, bias=bias, relu=False)
            dw = plan.wgrad(dy, x)
            torch.cuda.synchronize()
            outs.append((y, dw, device.last_launch()["load"]))
    finally:
        L.tcb_set_conv_stem(-1)
    (y1, dw1, l1), (y0, dw0, l0) = outs
    assert l1 == 5 and l0 != 5
    # both accumulate the same bf16 products in fp32 (different order): bf16 outputs
    # agree to an ulp, weight gradients to fp32 summation noise
    assert (y1.float() - y0.float()).abs().max().item() <= 2 ** -7 * max(y0.float().abs().max().item(), 1.0)
    assert torch.allclose(dw1, dw0, rtol=1e-4, atol=1e-4 * dw0.abs().max().item())


@pytest.mark.parametrize("case", [STEMS[0], STEMS[2], STEMS[6]], ids=[STEMS[0][0], STEMS[2][0], STEMS[6][0]])
def test_stem_cta_pairs_match_single_cta(case, monkeypatch):
    """$TCB_STEM_CTA2=1 (M = 256 MMAs over CTA pairs, odd tile counts included)
    gives the same bits as the single-CTA forward: same products, same fp32
    accumulation order per output element."""
    import subprocess
    import sys
    code = (
        "import sys, torch; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
        "import test_stem_gpu as t;"
        f"case = {case!r};"
        "device, L = t._lib();"
        "_, n, h, w, k, r, pad, stride, cv = case;"
        "g = device.geom(n, h, w, 8, k, r, pad=pad, stride=stride);"
        "plan = device.ConvPlan(g, 'gemm', 'bf16').set_valid_channels(cv);"
        "x, wt, bias = t._inputs(case, 11);"
        "y = plan.fwd(x, wt, bias=bias, relu=True); torch.cuda.synchronize();"
        "print(device.last_launch()['cta2']);"
        "torch.save(y.cpu(), sys.argv[1])")
    outs = []
    for on in ("0", "1"):
        path = f"/tmp/stem_cta2_{on}.pt"
        env = dict(__import__("os").environ, TCB_STEM_CTA2=on)
        res = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True,
                             timeout=300)
        assert res.returncode == 0, res.stderr[-2000:]
        assert res.stdout.strip().splitlines()[-1] == on
        outs.append(torch.load(path))
    assert torch.equal(outs[0], outs[1])


def test_stem_repeat_is_bitwise_and_in_bounds():
    """Guard regions around y / dw and the workspace; two launches bit-identical."""
    device, L = _lib()
    case = STEMS[1]
    _, n, h, w, k, r, pad, stride, cv = case
    g = device.geom(n, h, w, 8, k, r, pad=pad, stride=stride)
    plan = device.ConvPlan(g, "gemm", "bf16").set_valid_channels(cv)
    G = 1 << 20
    wsbuf = torch.full((plan.workspace_bytes + 2 * G,), 0xFF, dtype=torch.uint8, device="cuda")
    plan.workspace = wsbuf[G:G + plan.workspace_bytes]
    x, wt, bias = _inputs(case, 3)
    dy = torch.randn(n, g.ho, g.wo, k, device="cuda").bfloat16()
    ybuf = torch.full((n * g.ho * g.wo * k * 2 + 2 * G,), 0xFF, dtype=torch.uint8, device="cuda")
    dwbuf = torch.full((k * r * r * 8 * 4 + 2 * G,), 0xFF, dtype=torch.uint8, device="cuda")
    y = ybuf[G:-G].view(torch.bfloat16).view(n, g.ho, g.wo, k)
    dw = dwbuf[G:-G].view(torch.float32).view(k, r, r, 8)
    runs = []
    for _ in range(2):
        plan.fwd(x, wt, bias=bias, relu=True, out=y)
        plan.wgrad(dy, x, out=dw)
        torch.cuda.synchronize()
        runs.append((y.clone(), dw.clone()))
    for buf in (ybuf, dwbuf, wsbuf):
        assert bool((buf[:G] == 0xFF).all()) and bool((buf[-G:] == 0xFF).all())
    assert torch.equal(runs[0][0], runs[1][0]) and torch.equal(runs[0][1], runs[1][1])
