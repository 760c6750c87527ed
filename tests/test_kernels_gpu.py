"""Numeric-half parity: every sm_100a kernel vs the CPU oracle (oracle/numerics.c)
on identical seeded inputs, through the C-ABI (libtcb.so).

Tolerances (north_star): normwise relative error <= 1e-5 in fp32-FFMA mode,
<= 2e-2 in the TF32 and bf16 tensor-core modes (bf16: the oracle is fed the
same bf16-rounded inputs; outputs are bf16. TF32: fp32 inputs and outputs,
tf32 multiplies). Integer/byte work (RNG, labels,
argmax) and the SGD update are bit-exact.
SURVEY §8 rows: a14 (conv fwd/dgrad/wgrad), a16 (SGD), a17 (pools, loss), d1 (RNG).
"""
import numpy as np
import pytest

from oracle_binding import elem_err, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"ffma": 1e-5, "tf32": 2e-2, "bf16": 2e-2}
SEED = 20260810

# (name, n, h, w, c, k, r, pad, stride) — drawn from the BASELINE configs' layer shapes,
# shrunk in N so the fp64 oracle finishes in seconds; ragged M/N/K tails on purpose.
GEOMS = [
    ("lenet_conv2", 4, 12, 12, 24, 56, 5, 0, 1),
    ("alex_conv2", 2, 27, 27, 96, 256, 5, 2, 1),
    ("alex_conv3", 2, 13, 13, 256, 384, 3, 1, 1),
    ("rn50_3x3_s1", 2, 14, 14, 64, 64, 3, 1, 1),
    ("rn50_3x3_s2", 2, 28, 28, 128, 128, 3, 1, 2),
    ("rn50_1x1", 4, 14, 14, 256, 64, 1, 0, 1),
    ("rn50_1x1_s2", 2, 28, 28, 256, 512, 1, 0, 2),
    ("rn50_stem_7x7_s2", 2, 32, 32, 8, 64, 7, 3, 2),
    ("vgg_fc_as_conv", 3, 7, 7, 64, 136, 7, 0, 1),
    ("ragged", 3, 9, 11, 40, 72, 3, 1, 1),
    ("plain_1x1_ragged", 3, 5, 7, 24, 40, 1, 0, 1),
    ("plain_1x1_wide", 2, 9, 9, 520, 264, 1, 0, 1),
    ("plain_1x1_k48", 2, 7, 9, 200, 48, 1, 0, 1),
    ("bn192_fwd_k192", 2, 9, 9, 64, 192, 3, 1, 1),
    ("bn192_dgrad_c192", 2, 9, 9, 192, 64, 1, 0, 1),
    ("cta2_fwd_dgrad_3x3", 2, 16, 16, 128, 256, 3, 1, 1),
    ("cta2_ragged_3x3", 3, 9, 11, 128, 128, 3, 1, 1),
    ("cta2_wgrad_1x1", 8, 14, 14, 256, 512, 1, 0, 1),
    ("dgrad_phase_3x3_s2_odd", 2, 15, 13, 32, 48, 3, 1, 2),
    ("dgrad_phase_5x5_s3", 2, 17, 16, 16, 24, 5, 2, 3),
    ("im2col_ragged", 3, 9, 11, 64, 72, 3, 1, 1),
    ("im2col_k128_c64", 2, 10, 9, 64, 128, 3, 1, 1),
    ("im2col_s2_odd", 2, 11, 13, 64, 64, 3, 1, 2),
    ("im2col_5x5_pad2", 2, 8, 8, 128, 64, 5, 2, 1),
    ("c8_3x3", 2, 12, 10, 8, 24, 3, 1, 1),
    ("c8_11x11_s4", 2, 35, 35, 8, 96, 11, 2, 4),
    # Inception-v3 (C4) non-square filters at their real channel counts
    ("incep_1x7_768_192", 2, 17, 17, 768, 192, (1, 7), (0, 3), 1),
    ("incep_7x1_768_192", 2, 17, 17, 768, 192, (7, 1), (3, 0), 1),
    ("incep_1x3_384", 2, 8, 8, 384, 384, (1, 3), (0, 1), 1),
    ("incep_3x1_384", 2, 8, 8, 384, 384, (3, 1), (1, 0), 1),
    ("incep_1x1_2048_448", 2, 8, 8, 2048, 448, 1, 0, 1),
]
C4_ONLY = [  # channel counts % 4 but not % 8: fp32 modes only
    ("c4_3x3_k20", 2, 9, 9, 12, 20, 3, 1, 1),
    ("c4_5x5_s2", 2, 13, 11, 4, 36, 5, 2, 2),
    ("c4_stem_7x7_s2", 2, 32, 30, 4, 64, 7, 3, 2),  # tf32 4-channel im2col-TMA stem
]
FFMA_ONLY = [
    ("lenet_conv1_c1", 4, 28, 28, 1, 20, 5, 0, 1),
    ("odd_channels", 2, 10, 10, 3, 7, 3, 1, 2),
]


def _dev():
    from paper_1709_06622_b200 import device
    return device


def _rand(oracle, shape, tag, scale=1.0, bf16=False):
    n = int(np.prod(shape))
    a = oracle.uniform(n, SEED, tag, -scale, scale)
    if bf16:
        a = oracle.round_bf16(a)
    return a.reshape(shape)


def _to_dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to("cuda").to(dtype)


def _host(t):
    return t.float().cpu().numpy()


@pytest.fixture(params=["auto", "gather", "regepi", "nowin", "allwin"])
def operand_path(request):
    """auto = the window path (stride-1 R x S, activation channels % 64 == 0:
    one TMA window of padded rows per tile, taps as shifted descriptors), else
    2-D TMA (1x1/s1) or im2col-mode TMA (channels % 64 == 0 for bf16, % 32 for
    tf32), TMA epilogue on K-light layers; gather = force the cp.async gather
    path (bf16 and tf32); regepi = auto loads with the register epilogue
    everywhere (bf16); nowin = auto without the window path (bf16); allwin =
    the window path on every geometry it applies to (128/256-column tiles and
    CTA pairs included; bf16). All must agree with the oracle."""
    import ctypes
    lib = _dev().lib()
    lib.tcb_set_conv_operand_path.argtypes = [ctypes.c_int]
    lib.tcb_set_conv_operand_path({"auto": 0, "gather": 1, "regepi": 2, "nowin": 3, "allwin": 4}[request.param])
    yield request.param
    lib.tcb_set_conv_operand_path(0)


@pytest.mark.parametrize("prec", ["ffma", "tf32", "bf16"])
@pytest.mark.parametrize("spec", GEOMS + C4_ONLY + FFMA_ONLY, ids=lambda s: s[0])
def test_conv_gemm_parity(oracle, prec, spec, operand_path):
    if (prec != "ffma" and spec in FFMA_ONLY) or (prec == "bf16" and spec in C4_ONLY):
        pytest.skip("tensor-core paths need C, K multiples of 8 (bf16) / 4 (tf32)")
    if (prec == "ffma" and operand_path != "auto") or (prec == "tf32" and operand_path in ("regepi", "nowin", "allwin")):
        pytest.skip("operand path does not apply to this kernel")
    dev = _dev()
    name, n, h, w, c, k, r, pad, stride = spec
    rr, ss = (r, r) if isinstance(r, int) else r
    ph, pw = (pad, pad) if isinstance(pad, int) else pad
    g = dev.geom(n, h, w, c, k, rr, ss, pad=ph, pad_w=pw, stride=stride)
    gd = g.as_dict()
    plan = dev.ConvPlan(g, "gemm", prec)
    bf = prec == "bf16"
    dt = plan.dtype
    fan_in = c * rr * ss
    x = _rand(oracle, (n, h, w, c), 1, 1.0, bf)
    wt = _rand(oracle, (k, rr, ss, c), 2, (6.0 / fan_in) ** 0.5, bf)
    bias = _rand(oracle, (k,), 3, 0.1)
    res = _rand(oracle, (n, g.ho, g.wo, k), 4, 0.5, bf)
    dy = _rand(oracle, (n, g.ho, g.wo, k), 5, 1.0, bf)
    mask = _rand(oracle, (n, h, w, c), 6, 1.0, bf)
    rgrad = _rand(oracle, (n, h, w, c), 7, 0.5, bf)
    tol = TOL[prec]

    # forward with every epilogue feature
    y = plan.fwd(_to_dev(x, dt), _to_dev(wt, dt), bias=_to_dev(bias, torch.float32),
                 residual=_to_dev(res, dt), relu=True)
    ref = oracle.conv_fwd(gd, x, wt, bias=bias, residual=res, relu=True)
    assert rel_err(_host(y), ref) <= tol, (name, "fwd", rel_err(_host(y), ref))
    y0 = plan.fwd(_to_dev(x, dt), _to_dev(wt, dt))
    ref0 = oracle.conv_fwd(gd, x, wt)
    assert rel_err(_host(y0), ref0) <= tol

    # data gradient (+ residual gradient, ReLU mask of the layer input)
    dx = plan.dgrad(_to_dev(dy, dt), _to_dev(wt, dt), residual=_to_dev(rgrad, dt),
                    mask=_to_dev(mask, dt))
    refd = oracle.conv_dgrad(gd, dy, wt, residual=rgrad, mask=mask)
    assert rel_err(_host(dx), refd) <= tol, (name, "dgrad", rel_err(_host(dx), refd))
    dx0 = plan.dgrad(_to_dev(dy, dt), _to_dev(wt, dt))
    assert rel_err(_host(dx0), oracle.conv_dgrad(gd, dy, wt)) <= tol

    # weight + bias gradient (fp32, deterministic)
    dw, db = plan.wgrad(_to_dev(dy, dt), _to_dev(x, dt), want_db=True)
    refw, refb = oracle.conv_wgrad(gd, dy, x, want_db=True)
    assert rel_err(_host(dw), refw) <= tol, (name, "wgrad", rel_err(_host(dw), refw))
    assert rel_err(_host(db), refb) <= tol
    dw2 = plan.wgrad(_to_dev(dy, dt), _to_dev(x, dt))
    assert torch.equal(dw, dw2), "wgrad must be bitwise deterministic"
    if prec == "ffma":
        # fp32 accumulation error grows ~ sqrt(reduction depth)
        assert elem_err(_host(y), ref, 1e-2) <= 1e-4 * max(1.0, (fan_in / 2048) ** 0.5)
    if prec == "tf32":  # 10-bit mantissa products, fp32 accumulate: far inside 2e-2
        assert rel_err(_host(y0), ref0) <= 2e-3 and rel_err(_host(dw), refw) <= 2e-3


WINDOW_CASES = [  # (name, n, h, w, c, k, (r, s), (ph, pw), expected fwd / dgrad configuration)
    ("rn50_s1_3x3", 3, 56, 56, 64, 64, (3, 3), (1, 1), dict(fwd=(64, 0, 1), dgrad=(64, 0, 1), wgrad=64)),
    ("rn50_s1_3x3_n9", 9, 56, 56, 64, 64, (3, 3), (1, 1), dict(fwd=(64, 0, 1), dgrad=(64, 0, 1), wgrad=64)),
    ("incep_3x3_64_128", 2, 35, 35, 64, 128, (3, 3), (1, 1), dict(fwd=(128, 1, 1), dgrad=(64, 0, 0))),
    ("rn50_s2_3x3", 2, 28, 28, 128, 128, (3, 3), (1, 1), dict(fwd=(128, 1, 0), dgrad=(128, 1, 0))),
    ("rn50_s3_3x3_k256", 2, 14, 14, 256, 256, (3, 3), (1, 1), dict(fwd=(256, 1, 0), dgrad=(256, 1, 0))),
    ("incep_5x5_48_64", 3, 35, 35, 64, 64, (5, 5), (2, 2), dict(fwd=(64, 0, 0), dgrad=(64, 0, 0))),
    ("incep_7x1_192", 2, 17, 17, 192, 192, (7, 1), (3, 0), dict(fwd=(256, 1, 0), dgrad=(256, 1, 0))),
    # window weight gradient as tap groups: 14 tap-slices x K = 192 -> 7 M tiles, 2 per group
    ("incep_7x1_128_192", 2, 17, 17, 128, 192, (7, 1), (3, 0), dict(fwd=(256, 1, 0), dgrad=(128, 1, 0))),
    # wide rows: rectangular window tiles (Inception Conv2d_2a / 2b, VGG conv1_2), ragged corners
    ("incep_2a_wide_valid", 2, 37, 149, 64, 64, (3, 3), (0, 0), dict(fwd=(64, 0, 1), dgrad=(64, 0, 1))),
    ("incep_2b_wide", 2, 21, 147, 64, 64, (3, 3), (1, 1), dict(fwd=(64, 0, 1), dgrad=(64, 0, 1))),
    ("vgg_wide_224", 1, 9, 224, 64, 64, (3, 3), (1, 1), dict(fwd=(64, 0, 1), dgrad=(64, 0, 1))),
]


@pytest.fixture
def all_window():
    import ctypes
    lib = _dev().lib()
    lib.tcb_set_conv_operand_path.argtypes = [ctypes.c_int]
    lib.tcb_set_conv_operand_path(4)
    yield
    lib.tcb_set_conv_operand_path(0)


@pytest.mark.parametrize("spec", WINDOW_CASES, ids=lambda s: s[0])
def test_window_conv_path(oracle, spec, all_window):
    """The window implicit GEMM at real layer sizes: fwd with the fused
    bias + residual + ReLU epilogue, dgrad with residual-grad + ReLU mask,
    against the oracle (bf16, 2e-2) and bitwise against itself; the launch
    configuration (tile N, CTA pair, resident weights) is the planned one."""
    dev = _dev()
    name, n, h, w, c, k, (rr, ss), (ph, pw), want = spec
    g = dev.geom(n, h, w, c, k, rr, ss, pad=ph, pad_w=pw)
    gd = g.as_dict()
    plan = dev.ConvPlan(g, "gemm", "bf16")
    bf = torch.bfloat16
    x = _rand(oracle, (n, h, w, c), 1, 1.0, True)
    wt = _rand(oracle, (k, rr, ss, c), 2, (6.0 / (c * rr * ss)) ** 0.5, True)
    bias = _rand(oracle, (k,), 3, 0.1)
    res = _rand(oracle, (n, g.ho, g.wo, k), 4, 0.5, True)
    dy = _rand(oracle, (n, g.ho, g.wo, k), 5, 1.0, True)
    mask = _rand(oracle, (n, h, w, c), 6, 1.0, True)
    rgrad = _rand(oracle, (n, h, w, c), 7, 0.5, True)
    y = plan.fwd(_to_dev(x, bf), _to_dev(wt, bf), bias=_to_dev(bias, torch.float32), residual=_to_dev(res, bf),
                 relu=True)
    info = dev.last_launch()
    assert info["load"] == 4 and (info["bn"], info["cta2"], info["b_resident"]) == want["fwd"], info
    ref = oracle.conv_fwd(gd, x, wt, bias=bias, residual=res, relu=True)
    assert rel_err(_host(y), ref) <= 2e-2, rel_err(_host(y), ref)
    dx = plan.dgrad(_to_dev(dy, bf), _to_dev(wt, bf), residual=_to_dev(rgrad, bf), mask=_to_dev(mask, bf))
    info = dev.last_launch()
    assert info["load"] == 4 and (info["bn"], info["cta2"], info["b_resident"]) == want["dgrad"], info
    refd = oracle.conv_dgrad(gd, dy, wt, residual=rgrad, mask=mask)
    assert rel_err(_host(dx), refd) <= 2e-2, rel_err(_host(dx), refd)
    y2 = plan.fwd(_to_dev(x, bf), _to_dev(wt, bf), bias=_to_dev(bias, torch.float32), residual=_to_dev(res, bf),
                  relu=True)
    assert torch.equal(y, y2)
    if "wgrad" in want:
        dw = plan.wgrad(_to_dev(dy, bf), _to_dev(x, bf))
        info = dev.last_launch()
        assert info["mode"] == 2 and info["load"] == 4 and info["bn"] == want["wgrad"], info
        refw = oracle.conv_wgrad(gd, dy, x)
        assert rel_err(_host(dw), refw) <= 1e-3, rel_err(_host(dw), refw)
        assert torch.equal(dw, plan.wgrad(_to_dev(dy, bf), _to_dev(x, bf)))


def test_wgrad_many_splits_and_cta_pairs(oracle):
    """A ResNet-50 stage-2-shaped 1x1 wgrad whose one-wave split-K plan has 37
    splits over 2 CTA-pair units (M = 512 -> 2 pairs of 128-row tiles): the
    tree split reduction and the pair path at a real reduction depth
    (25,088 pixels), bf16 vs the fp64 oracle, and bitwise deterministic."""
    dev = _dev()
    g = dev.geom(32, 28, 28, 128, 512, 1)
    gd = g.as_dict()
    plan = dev.ConvPlan(g, "gemm", "bf16")
    x = _rand(oracle, (32, 28, 28, 128), 1, 1.0, True)
    dy = _rand(oracle, (32, 28, 28, 512), 5, 1.0, True)
    dw = plan.wgrad(_to_dev(dy, torch.bfloat16), _to_dev(x, torch.bfloat16))
    info = dev.last_launch()
    assert info["mode"] == 2 and info["cta2"] == 1 and info["splits"] >= 16, info
    assert info["units"] == 2 * info["splits"], info
    refw = oracle.conv_wgrad(gd, dy, x)
    assert rel_err(_host(dw), refw) <= 1e-3
    assert torch.equal(dw, plan.wgrad(_to_dev(dy, torch.bfloat16), _to_dev(x, torch.bfloat16)))


@pytest.mark.parametrize("spec", [(8, 7, 512, 4096, 7, 16), (2, 14, 1024, 256, 1, 4), (3, 5, 2048, 1000, 1, 4)],
                         ids=["vgg_fc6_n8", "rn50_1x1_n2", "fc_like_1x1_ragged"])
def test_fc_forward_split_k(oracle, spec):
    """Split-K forward of plain GEMMs with few output tiles and a deep reduction:
    VGG fc6 at a reduced batch (7x7x512 -> 4096, depth 25,088) runs as a 1x1
    GEMM over H*W*C channels; small-batch 1x1 layers (M = N*H*W rows) likewise.
    k-ranges go to fp32 partials, reduced with bias + residual + ReLU in fixed
    split order; vs the fp64 oracle, and bitwise repeatable."""
    dev = _dev()
    n, hw, c, k, r, tiles = spec
    g = dev.geom(n, hw, hw, c, k, r)
    gd = g.as_dict()
    plan = dev.ConvPlan(g, "gemm", "bf16")
    assert plan.workspace_bytes > 0
    x = _rand(oracle, (n, hw, hw, c), 1, 1.0, True)
    wt = _rand(oracle, (k, r, r, c), 2, (6.0 / (r * r * c)) ** 0.5, True)
    bias = _rand(oracle, (k,), 3, 0.1)
    res = _rand(oracle, (n, g.ho, g.wo, k), 4, 0.5, True)
    xd, wd = _to_dev(x, torch.bfloat16), _to_dev(wt, torch.bfloat16)
    bd, rd = _to_dev(bias, torch.float32), _to_dev(res, torch.bfloat16)
    y = plan.fwd(xd, wd, bias=bd, residual=rd, relu=True)
    info = dev.last_launch()
    assert info["mode"] == 0 and info["splits"] >= 2 and info["units"] == tiles * info["splits"], info
    ref = oracle.conv_fwd(gd, x, wt, bias=bias, residual=res, relu=True)
    assert rel_err(_host(y), ref) <= 1e-2
    assert torch.equal(y, plan.fwd(xd, wd, bias=bd, residual=rd, relu=True))
    y0 = plan.fwd(xd, wd)
    assert rel_err(_host(y0), oracle.conv_fwd(gd, x, wt)) <= 1e-2


@pytest.mark.parametrize("spec", [(12, 7, 512, 256, 3, 1, 512), (4, 14, 512, 512, 3, 1, 512),
                                  (8, 9, 512, 384, 3, 1, 512), (4, 12, 128, 128, 3, 1, 384),
                                  (3, 11, 128, 96, 3, 1, 384)],
                         ids=["3x3_c512_k256", "3x3_c512_k512", "3x3_k384_odd_pairs", "3x3_c128_384", "3x3_k96_384"])
def test_wgrad_double_n_tiles(oracle, spec):
    """Spatial weight gradients on double-N tiles: N = R*S*C a multiple of 512 as
    512-column CTA-pair tiles (two N = 256 MMAs per k-step into all of TMEM, B
    boxes interleaved per MMA half), a multiple of 384 with one 128-row M tile
    as 384-column single-CTA tiles (two N = 192 MMAs): vs the fp64 oracle,
    bitwise repeatable."""
    dev = _dev()
    n, hw, c, k, r, pad, bn = spec
    g = dev.geom(n, hw, hw, c, k, r, pad=pad)
    gd = g.as_dict()
    plan = dev.ConvPlan(g, "gemm", "bf16")
    x = _rand(oracle, (n, hw, hw, c), 1, 1.0, True)
    dy = _rand(oracle, (n, g.ho, g.wo, k), 5, 1.0, True)
    xd, dyd = _to_dev(x, torch.bfloat16), _to_dev(dy, torch.bfloat16)
    dw = plan.wgrad(dyd, xd)
    info = dev.last_launch()
    assert info["mode"] == 2 and info["bn"] == bn and info["cta2"] == (1 if bn == 512 else 0), info
    refw = oracle.conv_wgrad(gd, dy, x)
    assert rel_err(_host(dw), refw) <= 1e-3
    assert torch.equal(dw, plan.wgrad(dyd, xd))


def test_fill_and_labels_bit_exact(oracle):
    dev = _dev()
    for tag, lo, hi in ((1, -1.0, 1.0), (99, -0.05, 0.05), (7, 0.0, 3.0)):
        t = torch.empty(100_003, dtype=torch.float32, device="cuda")
        dev.fill_uniform(t, SEED, tag, lo, hi)
        assert np.array_equal(t.cpu().numpy(), oracle.uniform(t.numel(), SEED, tag, lo, hi))
        tb = torch.empty(100_003, dtype=torch.bfloat16, device="cuda")
        dev.fill_uniform(tb, SEED, tag, lo, hi)
        assert np.array_equal(tb.float().cpu().numpy(),
                              oracle.round_bf16(oracle.uniform(tb.numel(), SEED, tag, lo, hi)))
    lab = torch.empty(4097, dtype=torch.int32, device="cuda")
    dev.fill_labels(lab, 1000, SEED)
    assert np.array_equal(lab.cpu().numpy(), oracle.labels(4097, 1000, SEED))


@pytest.mark.parametrize("n", [1, 7, 4096, 1_000_003])
def test_sgd_bit_exact(oracle, n):
    dev = _dev()
    w = oracle.uniform(n, SEED, 11, -0.1, 0.1)
    g = oracle.uniform(n, SEED, 12, -1.0, 1.0)
    v = oracle.uniform(n, SEED, 13, -0.01, 0.01)
    wd, vd, gd = (torch.from_numpy(a.copy()).cuda() for a in (w, v, g))
    wc = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    dev.sgd_momentum(wd, gd, vd, 0.01, 0.9, 5e-4, 0.25, w_compute=wc)
    w_ref, v_ref = oracle.sgd(w, g, v, 0.01, 0.9, 5e-4, 0.25)
    assert np.array_equal(wd.cpu().numpy(), w_ref)
    assert np.array_equal(vd.cpu().numpy(), v_ref)
    assert np.array_equal(wc.float().cpu().numpy(), oracle.round_bf16(w_ref))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("pool", [(3, 2, 0), (2, 2, 0), (3, 2, 1), (3, 1, 1)])
def test_maxpool_parity(oracle, dtype, pool):
    dev = _dev()
    f, s, p = pool
    n, h, w, c = 2, 13, 15, 24
    bf = dtype == "bf16"
    dt = torch.bfloat16 if bf else torch.float32
    x = _rand(oracle, (n, h, w, c), 21, 1.0, bf)
    y, arg = dev.maxpool_fwd(_to_dev(x, dt), f, s, p)
    ry, rarg = oracle.maxpool_fwd(x, n, h, w, c, f, s, p)
    assert np.array_equal(arg.cpu().numpy().ravel(), rarg)
    assert np.array_equal(_host(y).ravel(), ry.astype(np.float32))
    dy = _rand(oracle, tuple(y.shape), 22, 1.0, bf)
    dx = dev.maxpool_bwd(_to_dev(dy, dt), arg, (n, h, w, c), f, s, p)
    rdx = oracle.maxpool_bwd(dy, rarg, n, h, w, c, f, s, p)
    assert rel_err(_host(dx), rdx) <= TOL["bf16" if bf else "ffma"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("pool", [(3, 2, 1), (3, 2, 0), (2, 2, 0)])
def test_maxpool_relu_ties_parity(oracle, dtype, pool):
    """ReLU'd input quantised to a few levels (many ties, many zeros): argmax
    keeps the first maximum in window order, and the fused ReLU backward
    (mask from the pool output) equals maxpool_bwd followed by the ReLU mask."""
    dev = _dev()
    f, s, p = pool
    n, h, w, c = 2, 14, 12, 16
    bf = dtype == "bf16"
    dt = torch.bfloat16 if bf else torch.float32
    x = np.maximum(np.round(_rand(oracle, (n, h, w, c), 31, 1.0, bf) * 2.0) / 2.0, 0.0).astype(np.float32)
    y, arg = dev.maxpool_fwd(_to_dev(x, dt), f, s, p)
    ry, rarg = oracle.maxpool_fwd(x, n, h, w, c, f, s, p)
    assert np.array_equal(arg.cpu().numpy().ravel(), rarg)
    assert np.array_equal(_host(y).ravel(), ry.astype(np.float32))
    dy = _rand(oracle, tuple(y.shape), 32, 1.0, bf)
    dx = dev.maxpool_bwd(_to_dev(dy, dt), arg, (n, h, w, c), f, s, p, relu_y=y)
    rdx = oracle.maxpool_bwd(dy, rarg, n, h, w, c, f, s, p) * (x.ravel() > 0)
    assert rel_err(_host(dx), rdx) <= TOL["bf16" if bf else "ffma"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("pool", [(3, 1, 1), (3, 2, 0), (2, 2, 1), (5, 3, 2)])
def test_avgpool2d_parity(oracle, dtype, pool):
    """Windowed average pool (Inception's branch pool, padding counted) and its
    owner-computes backward, with and without the fused ReLU mask."""
    dev = _dev()
    bf = dtype == "bf16"
    f, s, p = pool
    n, h, w, c = 2, 11, 9, 24
    x = _rand(oracle, (n, h, w, c), 21, 1.0, bf)
    dt = torch.bfloat16 if bf else torch.float32
    tol = TOL["bf16" if bf else "ffma"]
    y = dev.avgpool2d_fwd(_to_dev(x, dt), f, s, p)
    assert rel_err(_host(y), oracle.avgpool2d_fwd(x, n, h, w, c, f, s, p)) <= tol
    ho, wo = y.shape[1], y.shape[2]
    dy = _rand(oracle, (n, ho, wo, c), 22, 1.0, bf)
    ref = oracle.avgpool2d_bwd(dy, n, h, w, c, f, s, p)
    dx = dev.avgpool2d_bwd(_to_dev(dy, dt), (n, h, w, c), f, s, p)
    assert rel_err(_host(dx), ref) <= tol
    mask = _rand(oracle, (n, h, w, c), 23, 1.0, bf)
    dxm = dev.avgpool2d_bwd(_to_dev(dy, dt), (n, h, w, c), f, s, p, mask=_to_dev(mask, dt))
    assert rel_err(_host(dxm), np.where(mask.ravel() > 0, ref, 0.0)) <= tol


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_concat_slice_copy_bit_exact(dtype):
    dev = _dev()
    xs = [torch.randn(2, 5, 7, c, device="cuda").to(dtype) for c in (8, 24, 16, 3)]
    got = dev.concat(xs)  # the last width (3) takes the scalar path
    assert torch.equal(got, torch.cat(xs, dim=3))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_avgpool_and_softmax_parity(oracle, dtype):
    dev = _dev()
    bf = dtype == "bf16"
    dt = torch.bfloat16 if bf else torch.float32
    tol = TOL["bf16" if bf else "ffma"]
    x = _rand(oracle, (3, 7, 7, 64), 31, 1.0, bf)
    y = dev.avgpool_fwd(_to_dev(x, dt))
    assert rel_err(_host(y), oracle.avgpool_fwd(x, 3, 49, 64)) <= tol
    dy = _rand(oracle, (3, 64), 32, 1.0, bf)
    dx = dev.avgpool_bwd(_to_dev(dy, dt), 7, 7)
    assert rel_err(_host(dx), oracle.avgpool_bwd(dy, 3, 49, 64)) <= tol
    z = _rand(oracle, (17, 1000), 33, 4.0, bf)
    lab = oracle.labels(17, 1000, SEED)
    loss, dl = dev.softmax_xent(_to_dev(z, dt), torch.from_numpy(lab).cuda())
    rl, rdl = oracle.softmax_xent(z, lab, 17, 1000)
    assert abs(float(loss) - rl) <= 1e-5 * abs(rl)
    assert rel_err(_host(dl), rdl) <= tol


# 3x3 stride-1 layers of the BASELINE configs for the Winograd / FFT families
FAMILY_GEOMS = [
    ("alex_conv3", 2, 13, 13, 256, 384, 3, 1, 1),
    ("rn50_3x3", 2, 14, 14, 64, 64, 3, 1, 1),
    ("vgg_3x3_odd", 2, 15, 9, 32, 48, 3, 1, 1),
    ("pad0_3x3", 2, 10, 11, 16, 24, 3, 0, 1),
]


@pytest.mark.parametrize("prec", ["ffma", "bf16"])
@pytest.mark.parametrize("spec", FAMILY_GEOMS, ids=lambda s: s[0])
def test_conv_winograd_parity(oracle, prec, spec):
    """Winograd F(2x2,3x3): fwd / dgrad / wgrad vs the direct-conv oracle."""
    dev = _dev()
    name, n, h, w, c, k, r, pad, stride = spec
    g = dev.geom(n, h, w, c, k, r, pad=pad, stride=stride)
    gd = g.as_dict()
    plan = dev.ConvPlan(g, "winograd", prec)
    bf = prec == "bf16"
    dt = plan.dtype
    x = _rand(oracle, (n, h, w, c), 1, 1.0, bf)
    wt = _rand(oracle, (k, r, r, c), 2, (6.0 / (c * 9)) ** 0.5, bf)
    bias = _rand(oracle, (k,), 3, 0.1)
    res = _rand(oracle, (n, g.ho, g.wo, k), 4, 0.5, bf)
    dy = _rand(oracle, (n, g.ho, g.wo, k), 5, 1.0, bf)
    mask = _rand(oracle, (n, h, w, c), 6, 1.0, bf)
    tol = TOL[prec]
    y = plan.fwd(_to_dev(x, dt), _to_dev(wt, dt), bias=_to_dev(bias, torch.float32),
                 residual=_to_dev(res, dt), relu=True)
    assert rel_err(_host(y), oracle.conv_fwd(gd, x, wt, bias=bias, residual=res, relu=True)) <= tol
    dx = plan.dgrad(_to_dev(dy, dt), _to_dev(wt, dt), mask=_to_dev(mask, dt))
    assert rel_err(_host(dx), oracle.conv_dgrad(gd, dy, wt, mask=mask)) <= tol
    dw, db = plan.wgrad(_to_dev(dy, dt), _to_dev(x, dt), want_db=True)
    refw, refb = oracle.conv_wgrad(gd, dy, x, want_db=True)
    assert rel_err(_host(dw), refw) <= tol, (name, rel_err(_host(dw), refw))
    assert rel_err(_host(db), refb) <= tol


FFT_GEOMS = FAMILY_GEOMS + [
    ("alex_conv2_5x5", 2, 27, 27, 96, 256, 5, 2, 1),
    ("incep_1x7", 2, 17, 17, 32, 48, (1, 7), (0, 3), 1),
    ("incep_7x1", 2, 17, 17, 32, 48, (7, 1), (3, 0), 1),
]


@pytest.mark.parametrize("prec", ["ffma", "bf16"])
@pytest.mark.parametrize("spec", FFT_GEOMS, ids=lambda s: s[0])
def test_conv_fft_parity(oracle, prec, spec):
    """Tiled FFT convolution (overlap-save 8x8): fwd / dgrad / wgrad vs the oracle."""
    dev = _dev()
    name, n, h, w, c, k, r, pad, stride = spec
    rr, ss = (r, r) if isinstance(r, int) else r
    ph, pw = (pad, pad) if isinstance(pad, int) else pad
    g = dev.geom(n, h, w, c, k, rr, ss, pad=ph, pad_w=pw, stride=stride)
    gd = g.as_dict()
    plan = dev.ConvPlan(g, "fft", prec)
    bf = prec == "bf16"
    dt = plan.dtype
    x = _rand(oracle, (n, h, w, c), 1, 1.0, bf)
    wt = _rand(oracle, (k, rr, ss, c), 2, (6.0 / (c * rr * ss)) ** 0.5, bf)
    bias = _rand(oracle, (k,), 3, 0.1)
    res = _rand(oracle, (n, g.ho, g.wo, k), 4, 0.5, bf)
    dy = _rand(oracle, (n, g.ho, g.wo, k), 5, 1.0, bf)
    mask = _rand(oracle, (n, h, w, c), 6, 1.0, bf)
    tol = TOL[prec]
    y = plan.fwd(_to_dev(x, dt), _to_dev(wt, dt), bias=_to_dev(bias, torch.float32),
                 residual=_to_dev(res, dt), relu=True)
    e = rel_err(_host(y), oracle.conv_fwd(gd, x, wt, bias=bias, residual=res, relu=True))
    assert e <= tol, (name, "fwd", e)
    dx = plan.dgrad(_to_dev(dy, dt), _to_dev(wt, dt), mask=_to_dev(mask, dt))
    e = rel_err(_host(dx), oracle.conv_dgrad(gd, dy, wt, mask=mask))
    assert e <= tol, (name, "dgrad", e)
    dw, db = plan.wgrad(_to_dev(dy, dt), _to_dev(x, dt), want_db=True)
    refw, refb = oracle.conv_wgrad(gd, dy, x, want_db=True)
    e = rel_err(_host(dw), refw)
    assert e <= tol, (name, "wgrad", e)
    assert rel_err(_host(db), refb) <= tol


def test_fft_rejects_strided_geometry():
    dev = _dev()
    with pytest.raises(dev.Unsupported):
        dev.ConvPlan(dev.geom(2, 27, 27, 96, 256, 11, pad=2, stride=4), "fft", "bf16")


def test_winograd_rejects_inapplicable_geometry():
    dev = _dev()
    with pytest.raises(dev.Unsupported):
        dev.ConvPlan(dev.geom(2, 14, 14, 64, 64, 3, pad=1, stride=2), "winograd", "bf16")
    with pytest.raises(dev.Unsupported):
        dev.ConvPlan(dev.geom(2, 14, 14, 64, 64, 5, pad=2), "winograd", "bf16")
