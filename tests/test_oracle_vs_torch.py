"""The numeric oracle (oracle/numerics.c) cross-checked against an independent
implementation — PyTorch's CPU operators in float64 — on seeded small cases.

The reference has no numeric code to pin the oracle to (parity of
the numeric half is unpinned by the reference); this establishes that the
restatement computes the textbook operators: conv fwd/dgrad/wgrad with
bias/residual/ReLU epilogues (NHWC, KRSC), max pool with argmax routing, global
average pool, softmax cross-entropy and its gradient. Runs on CPU.
"""
import numpy as np
import pytest

from oracle_binding import out_hw

torch = pytest.importorskip("torch")
F = torch.nn.functional

GEOMS = [  # n, h, w, c, k, r, pad, stride
    (2, 9, 11, 5, 7, 3, 1, 1),
    (1, 12, 10, 4, 6, 5, 2, 2),
    (2, 7, 7, 3, 4, 1, 0, 1),
    (1, 13, 13, 2, 3, 7, 3, 2),
    (2, 8, 9, 6, 5, 3, 0, 3),
]


def _t(a, shape):  # NHWC numpy -> NCHW float64 tensor
    return torch.from_numpy(np.asarray(a, np.float64).reshape(shape)).permute(0, 3, 1, 2)


def _nhwc(t):
    return t.permute(0, 2, 3, 1).contiguous().numpy().ravel()


@pytest.mark.parametrize("spec", GEOMS, ids=lambda s: "x".join(map(str, s)))
def test_conv_passes_match_torch_fp64(oracle, spec):
    n, h, w, c, k, r, pad, stride = spec
    g = dict(n=n, h=h, w=w, c=c, k=k, r=r, s=r, pad_h=pad, pad_w=pad, stride_h=stride, stride_w=stride)
    ho, wo = out_hw(g)
    x = oracle.uniform(n * h * w * c, 7, 1)
    wt = oracle.uniform(k * r * r * c, 7, 2)
    bias = oracle.uniform(k, 7, 3)
    res = oracle.uniform(n * ho * wo * k, 7, 4)
    dy = oracle.uniform(n * ho * wo * k, 7, 5)
    mask = oracle.uniform(n * h * w * c, 7, 6)

    X = _t(x, (n, h, w, c)).requires_grad_(True)
    W = torch.from_numpy(wt.astype(np.float64).reshape(k, r, r, c)).permute(0, 3, 1, 2).requires_grad_(True)
    Y = F.conv2d(X, W, torch.from_numpy(bias.astype(np.float64)), stride=stride, padding=pad)
    ref_fwd = torch.relu(Y + _t(res, (n, ho, wo, k)))
    got = oracle.conv_fwd(g, x, wt, bias=bias, residual=res, relu=True)
    np.testing.assert_allclose(got, _nhwc(ref_fwd.detach()), rtol=1e-12, atol=1e-12)

    Y.backward(_t(dy, (n, ho, wo, k)))
    # the fused epilogue adds the residual gradient, then applies the ReLU mask
    dx_ref = (X.grad + _t(x, (n, h, w, c))) * (_t(mask, (n, h, w, c)) > 0)
    got_dx = oracle.conv_dgrad(g, dy, wt, residual=x, mask=mask)
    np.testing.assert_allclose(got_dx, _nhwc(dx_ref), rtol=1e-12, atol=1e-12)
    got_dw, got_db = oracle.conv_wgrad(g, dy, x, want_db=True)
    np.testing.assert_allclose(got_dw, W.grad.permute(0, 2, 3, 1).contiguous().numpy().ravel(),
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(got_db, _t(dy, (n, ho, wo, k)).sum(dim=(0, 2, 3)).numpy(),
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("pool", [(3, 2, 1), (2, 2, 0), (3, 1, 1)])
def test_maxpool_matches_torch_fp64(oracle, pool):
    f, s, p = pool
    n, h, w, c = 2, 9, 10, 3
    x = oracle.uniform(n * h * w * c, 9, 1)
    ho, wo = (h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1
    dy = oracle.uniform(n * ho * wo * c, 9, 2)
    X = _t(x, (n, h, w, c)).requires_grad_(True)
    Y = F.max_pool2d(X, f, s, p)
    y, arg = oracle.maxpool_fwd(x, n, h, w, c, f, s, p)
    np.testing.assert_array_equal(y, _nhwc(Y.detach()))
    Y.backward(_t(dy, (n, ho, wo, c)))
    np.testing.assert_allclose(oracle.maxpool_bwd(dy, arg, n, h, w, c, f, s, p), _nhwc(X.grad),
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("pool", [(3, 1, 1), (3, 2, 0), (2, 2, 1)])
def test_avgpool2d_matches_torch_fp64(oracle, pool):
    f, s, p = pool
    n, h, w, c = 2, 9, 8, 3
    x = oracle.uniform(n * h * w * c, 13, 1)
    ho, wo = (h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1
    dy = oracle.uniform(n * ho * wo * c, 13, 2)
    X = _t(x, (n, h, w, c)).requires_grad_(True)
    Y = F.avg_pool2d(X, f, s, p, count_include_pad=True)
    np.testing.assert_allclose(oracle.avgpool2d_fwd(x, n, h, w, c, f, s, p), _nhwc(Y.detach()), rtol=1e-12)
    Y.backward(_t(dy, (n, ho, wo, c)))
    np.testing.assert_allclose(oracle.avgpool2d_bwd(dy, n, h, w, c, f, s, p), _nhwc(X.grad),
                               rtol=1e-12, atol=1e-15)


def test_avgpool_and_softmax_xent_match_torch_fp64(oracle):
    n, hw, c, classes = 3, 5, 8, 10
    x = oracle.uniform(n * hw * c, 11, 1)
    X = torch.from_numpy(x.astype(np.float64).reshape(n, hw, c)).requires_grad_(True)
    Y = X.mean(dim=1)
    np.testing.assert_allclose(oracle.avgpool_fwd(x, n, hw, c), Y.detach().numpy().ravel(), rtol=1e-12)
    dy = oracle.uniform(n * c, 11, 2)
    Y.backward(torch.from_numpy(dy.astype(np.float64).reshape(n, c)))
    np.testing.assert_allclose(oracle.avgpool_bwd(dy, n, hw, c), X.grad.numpy().ravel(), rtol=1e-12)

    z = oracle.uniform(n * classes, 11, 3, -4.0, 4.0)
    lab = oracle.labels(n, classes, 11)
    Z = torch.from_numpy(z.astype(np.float64).reshape(n, classes)).requires_grad_(True)
    L = F.cross_entropy(Z, torch.from_numpy(lab.astype(np.int64)))
    L.backward()
    loss, dl = oracle.softmax_xent(z, lab, n, classes)
    assert abs(loss - L.item()) <= 1e-12 * max(1.0, abs(L.item()))
    np.testing.assert_allclose(dl, Z.grad.numpy().ravel(), rtol=1e-10, atol=1e-14)
