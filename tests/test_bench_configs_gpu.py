"""Parity at the configurations the benchmark lines are quoted on
(BASELINE.json configs C3 / C4 / C5), not shrunk copies:

* C3 ResNet-50, 224x224, 256 images (the exact bf16 `bench.py` step, three
  steps so the last one is the replayed CUDA graph): layer-local parity of
  every forward activation and activation gradient on two images of the
  batch (first and last tile rows) and, at the full 256-image reduction,
  the weight gradients of sampled layers (stem, one 3x3 and one 1x1 per
  stage, the strided projections, fc) on a subset of output channels.
* C5 VGG-16, 224x224: the fp32-FFMA step end to end at N = 2 (1e-5), and the
  bf16 step at 64 images with the same sampled scheme (fc6 / fc7 / conv5).
* C4 Inception-v3 at full width and 299x299 (batch 2, bf16, layer-local).

Tolerances (north_star): 1e-5 fp32-FFMA, 2e-2 bf16; the sampled weight
gradients see the device's own bf16 operands, so they are also held to 1e-3.
The oracle is the fp64 CPU restatement (oracle/numerics.c) — test
infrastructure only. The learning rate is 0 so every step sees W_0 and the
replayed graph step must reproduce the eager one.
"""
import numpy as np
import pytest

from oracle_binding import rel_err
from oracle_step import OracleStep, SubsetTeacher

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _models():
    from paper_1709_06622_b200 import models
    return models


def _trainer(cfg, steps):
    from paper_1709_06622_b200.trainer import Trainer
    t = Trainer(cfg)
    for _ in range(steps):
        t.step()
    torch.cuda.synchronize()
    return t


def _sampled_check(oracle, cfg, images, wgrad_layers, k_sub=4, steps=3):
    """Layer-local fwd + dgrad parity of the large-batch step on `images`,
    and full-batch weight gradients of `wgrad_layers` on k_sub channels."""
    t = _trainer(cfg, steps)
    lay = t.describe()
    teach = SubsetTeacher(t, lay, images)
    sub_lay = teach.layout()
    ref = OracleStep(oracle, cfg, sub_lay)
    x = teach.act(0)
    labels = t.tensor("labels").cpu().numpy()[images]
    ref.run(x, labels, teacher=teach, wgrad=False, loss_batch=cfg["batch"])
    nconv = sum(L["op"] == "conv" for L in lay["layers"])
    assert len(ref.local_err) >= 2 * nconv - 1
    bad = {k: e for k, e in ref.local_err.items() if not e <= 2e-2}
    assert not bad, bad
    worst = max(ref.local_err.values())

    g_dev = t.tensor("grad").cpu().numpy()
    by_name = {L["name"]: L for L in lay["layers"]}
    werr = {}
    for name in wgrad_layers:
        L = by_name[name]
        ka, r, s, cp = L["geom"][4], L["geom"][5], L["geom"][6], L["geom"][3]
        k, cl = L["c_logical"], lay["layers"][L["in"]]["c_logical"]
        ks = sorted({0, k - 1} | {int(v) for v in np.linspace(0, k - 1, k_sub)})
        dy = teach.full("dact", L["index"], ks)
        xin = teach.full("act", L["in"])
        g = dict(n=cfg["batch"], h=L["geom"][1], w=L["geom"][2], c=cl, k=len(ks), r=r, s=s,
                 pad_h=L["geom"][7], pad_w=L["geom"][8], stride_h=L["geom"][9], stride_w=L["geom"][10])
        dw, db = oracle.conv_wgrad(g, dy, xin, want_db=True)
        w4 = g_dev[L["woff"]:L["woff"] + ka * r * s * cp].reshape(ka, r, s, cp)
        got = w4[ks][..., :cl]
        werr[name] = rel_err(got, dw)
        if L["boff"] is not None:
            werr[name + ".bias"] = rel_err(g_dev[L["boff"]:L["boff"] + ka][ks], db)
        del dy, xin
    bad = {k: e for k, e in werr.items() if not e <= 1e-3}
    assert not bad, (bad, werr)
    return t, worst, werr


def test_resnet50_bs256_bench_step_sampled(oracle):
    """C3: the bench step (ResNet-50, 256 images, bf16, graph-replayed)."""
    m = _models()
    cfg = m.resnet50(batch=256, precision="bf16", lr=0.0)
    wl = ["stem", "s1b1_c1", "s1b2_c2", "s1b1_proj", "s2b1_c2", "s2b3_c3", "s3b1_proj",
          "s3b4_c2", "s4b1_c2", "s4b3_c1", "fc"]
    t, worst, werr = _sampled_check(oracle, cfg, [0, 255], wl)
    assert t.describe()["layers"][1]["stem_rows"]


def test_vgg16_ffma_step_end_to_end_n2(oracle):
    """C5 VGG-16 (224x224, 138M parameters) fp32-FFMA step end to end at N = 2:
    every conv / fc weight gradient, the loss and the SGD update within 1e-5.
    The five 2x2 max pools route gradients by the device's argmax (at most
    1e-4 of the windows may disagree with the fp64 oracle, on near-ties):
    one flipped argmax moves a whole gradient value, which is a decision on
    the last rounding bit, not arithmetic error."""
    from test_trainer_gpu import _check
    cfg = _models().vgg16(batch=2, precision="ffma")
    t, worst = _check(oracle, cfg, device_argmax=True)
    assert worst <= 1e-5
    assert t.describe()["param_count"] == 138_357_544


def test_vgg16_bs64_bf16_step_sampled(oracle):
    """C5 bf16 step at the bench's 64 images per GPU: fc6 (7x7x512 -> 4096,
    whole-map conv; dgrad as the 1x1 GEMM), fc7, fc8, conv5 and conv1
    weight gradients at the full reduction, layer-local elsewhere."""
    cfg = _models().vgg16(batch=64, precision="bf16", lr=0.0)
    names = [L["name"] for L in cfg["layers"] if L["op"] == "conv"]
    wl = [names[0], names[7], names[12], names[13], names[14], names[15]]
    _sampled_check(oracle, cfg, [0, 63], wl)


def test_inception_v3_full_width_299_step_bf16(oracle):
    """C4 Inception-v3 at full width and 299x299 (batch 2, bf16), layer-local:
    the 94 convs at their real channel counts incl. the 1x7 / 7x1 / 1x3 / 3x1
    branches, windowed average pools, concat and 4-way gradient fan-in."""
    from test_trainer_gpu import _check
    cfg = _models().inception_v3(batch=2, image=299, width=1.0, precision="bf16")
    t, _ = _check(oracle, cfg)
    convs = [L for L in t.describe()["layers"] if L["op"] == "conv"]
    shapes = {(L["geom"][5], L["geom"][6]) for L in convs}
    assert {(1, 7), (7, 1), (1, 3), (3, 1)} <= shapes
