"""Step-level parity: the C++ executor's full training step (fwd -> loss ->
bwd -> fused SGD) vs the CPU oracle step on identical seeded inputs/weights.
Tolerances: normwise 1e-5 (fp32-FFMA mode), 2e-2 (TF32 / bf16 tensor-core modes).
SURVEY §8 rows a14-a17 end to end, d1 (synthetic inputs)."""
import numpy as np
import pytest

from oracle_binding import rel_err
from oracle_step import DeviceTeacher, OracleStep

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"ffma": 1e-5, "tf32": 2e-2, "bf16": 2e-2}


def _models():
    from paper_1709_06622_b200 import models
    return models


def _run_step(cfg):
    from paper_1709_06622_b200.trainer import Trainer
    t = Trainer(cfg)
    t.step()
    torch.cuda.synchronize()
    return t


def _check(oracle, cfg, per_layer=True, teacher=None, device_argmax=False):
    """fp32-FFMA: end-to-end step vs the oracle step (1e-5).
    bf16: layer-local (teacher-forced) — every activation, activation gradient
    and weight gradient of the step is recomputed by the oracle from the
    device's own inputs (2e-2). End-to-end bf16 agreement degrades with depth
    because independent bf16 roundings flip max-pool argmaxes on near-ties;
    that drift is measured in test_bf16_end_to_end_drift_is_small_on_shallow_net."""
    prec = cfg["precision"]
    tol = TOL[prec]
    t = _run_step(cfg)
    lay = t.describe()
    ref = OracleStep(oracle, cfg, lay)
    teacher = (prec != "ffma") if teacher is None else teacher
    ref.run(teacher=DeviceTeacher(t, lay) if teacher else None,
            argmax_src=DeviceTeacher(t, lay) if device_argmax and not teacher else None)
    if ref.argmax_mismatch:  # near-ties only: a tiny fraction of the decisions
        assert max(ref.argmax_mismatch.values()) <= 1e-4, ref.argmax_mismatch
        assert max(ref.relu_mismatch.values()) <= 1e-4, ref.relu_mismatch
        print("decision mismatch: argmax", ref.argmax_mismatch, "relu", ref.relu_mismatch)
    if teacher:
        assert len(ref.local_err) >= 2 * sum(L["op"] == "conv" for L in lay["layers"]) - 1
        bad = {k: e for k, e in ref.local_err.items() if not e <= tol}
        assert not bad, bad
    loss = t.loss()
    assert abs(loss - ref.loss) <= max(tol, 1e-6) * abs(ref.loss), (loss, ref.loss)
    g_dev = t.tensor("grad").cpu().numpy().astype(np.float64)
    g_ref = ref.flat_grad()
    worst = 0.0
    for L in lay["layers"]:
        if L["op"] != "conv":
            continue
        sl = slice(L["woff"], L["woff"] + L["wcount"])
        e = rel_err(g_dev[sl], g_ref[sl])
        worst = max(worst, e)
        if per_layer:
            assert e <= tol, (L["name"], e)
        if L["boff"] is not None:
            sb = slice(L["boff"], L["boff"] + L["geom"][4])
            assert rel_err(g_dev[sb], g_ref[sb]) <= tol, (L["name"], "bias")
    # update: device SGD applied to device grads must equal the oracle SGD bit-exactly
    w_ref, _ = ref.sgd(g_dev.astype(np.float32))
    w_dev = t.tensor("param").cpu().numpy()
    assert np.array_equal(w_dev, w_ref)
    # and the delta against the oracle's own gradients within tolerance
    w_ref2, _ = ref.sgd(g_ref.astype(np.float32))
    w0 = ref.flat_params()
    assert rel_err(w_dev - w0, w_ref2 - w0) <= tol
    if prec == "bf16":
        wc = t.tensor("wcompute").float().cpu().numpy()
        assert np.array_equal(wc, oracle.round_bf16(w_dev))
    return t, worst


@pytest.mark.parametrize("prec", ["ffma", "tf32", "bf16"])
def test_tiny_resnet_step(oracle, prec):
    _check(oracle, _models().tiny_resnet(batch=4, precision=prec))


def test_bf16_end_to_end_drift_is_small_on_shallow_net(oracle):
    _check(oracle, _models().tiny_resnet(batch=4, precision="bf16"), teacher=False)


def test_resnet50_geometry_step_bf16(oracle):
    """C3 geometry (full ResNet-50-shaped graph, 224x224) at batch 1, layer-local.
    The 3-channel stem runs on the row-window stem kernels (fwd and wgrad)."""
    t, _ = _check(oracle, _models().resnet50(batch=1, precision="bf16"))
    convs = [L for L in t.describe()["layers"] if L["op"] == "conv"]
    assert convs[0]["stem_rows"] and not any(L["explicit_im2col"] or L["stem_rows"] for L in convs[1:])


def test_resnet50_geometry_step_tf32(oracle):
    """C3 geometry in the TF32 tensor-core mode (fp32 storage, the 3-channel
    input padded to 4 so the stem runs on tcgen05 kind::tf32 too), layer-local."""
    t, _ = _check(oracle, _models().resnet50(batch=1, precision="tf32"))
    lay = t.describe()
    assert lay["precision"] == "tf32"
    assert lay["layers"][0]["shape"][3] == 4


@pytest.mark.parametrize("prec", ["ffma", "bf16"])
def test_inception_v3_step(oracle, prec):
    """C4 graph (every Inception-v3 module: 1x1 / 5x5 / 3x3-double / 1x7-7x1 /
    1x3-3x1 split branches, 3x3 average-pool and max-pool branches, channel
    concat with fan-out gradients) at width 1/4, 75x75, batch 2."""
    cfg = _models().inception_v3(batch=2, image=75, width=0.25, classes=10, precision=prec)
    t, _ = _check(oracle, cfg)
    ops = [L["op"] for L in t.describe()["layers"]]
    assert ops.count("concat") == 11 and ops.count("conv") == 95


def test_inception_v3_mixed_algorithms_step(oracle):
    """The executor obeys a per-layer Selection on the C4 graph: FFT / Winograd
    on stride-1 3x3 and 5x5 branch convs, GEMM elsewhere (bf16, layer-local)."""
    m = _models()
    cfg = m.inception_v3(batch=2, image=75, width=0.25, classes=10, precision="bf16")
    names = [n for n, _ in m.conv_layers(cfg)]
    sel = {}
    for i, n in enumerate(names, 1):
        if n.endswith("_b3x3dbl_2") or n == "Mixed_6a_dbl_2" or n.endswith("_dbl_2") and n.startswith("Mixed_7"):
            sel[str(i)] = "winograd"
        elif n.endswith("_b5x5_2"):
            sel[str(i)] = "fft"
    cfg = m.apply_selection(cfg, sel)
    assert sum(L.get("algo") == "winograd" for L in cfg["layers"]) >= 5
    _check(oracle, cfg)


def test_row_window_stem_batch8(oracle):
    """Stem-only net at batch 8: row-window stem fwd (input rows packed with the
    uint8 / fp32 input preparation) and wgrad against the oracle, layer-local."""
    cfg = _models().from_net("input 64 64 3\nconv 7 2 3 64\npool 3 2 1\nconv 3 1 1 64\nfc 10\n",
                             batch=8, precision="bf16")
    t, _ = _check(oracle, cfg)
    assert t.describe()["layers"][1]["stem_rows"]


@pytest.mark.parametrize("net", ["stem_pool", "resnet50_b2"])
def test_stem_fused_max_pool_matches_separate_pool(net):
    """The row-window stem forward writing the following 3x3/2/1 max pool itself
    (config fuse_stem_pool) gives the same bits as the separate pool kernel:
    pooled activation, argmax, the stem activation, loss, gradients and
    parameters after two steps."""
    from paper_1709_06622_b200.trainer import Trainer
    if net == "stem_pool":
        cfg = _models().from_net("input 48 46 3\nconv 7 2 3 64\npool 3 2 1\nconv 3 1 1 64\nfc 10\n",
                                 batch=4, precision="bf16")
    else:
        cfg = _models().resnet50(batch=2, precision="bf16")
    a, b = Trainer(dict(cfg, fuse_stem_pool=True)), Trainer(cfg)
    for _ in range(2):
        a.step()
        b.step()
    torch.cuda.synchronize()
    la = a.describe()["layers"]
    stem = next(L for L in la if L["op"] == "conv")
    pool = next(L for L in la if L["op"] == "maxpool")
    assert stem["stem_pool_fused"] and not next(L for L in b.describe()["layers"] if L["op"] == "conv")["stem_pool_fused"]
    for name in (f"act:{stem['index']}", f"act:{pool['index']}", f"argmax:{pool['index']}", "grad", "param", "loss"):
        ta, tb = a.tensor(name), b.tensor(name)
        assert torch.equal(ta, tb), name


def test_explicit_im2col_first_layer_batch8(oracle):
    """An 11x11/4 first layer (AlexNet-style; stride 4 is outside the stem
    kernels): explicit-im2col fwd (TMA epilogue) and wgrad (col kept from the
    forward pass) against the oracle, layer-local."""
    cfg = _models().from_net("input 67 67 3\nconv 11 4 2 64\npool 3 2 0\nconv 3 1 1 64\nfc 10\n",
                             batch=8, precision="bf16")
    t, _ = _check(oracle, cfg)
    assert t.describe()["layers"][1]["explicit_im2col"]


def test_lenet_step_c1(oracle):
    """C1: LeNet 28x28x1 batch 64, 1 worker + 1 PS shard, fp32-FFMA mode."""
    _check(oracle, _models().lenet(batch=64))


@pytest.mark.parametrize("prec", ["ffma", "tf32", "bf16"])
def test_alexnet_step_small_batch(oracle, prec):
    """C2 geometry (227x227x3, ungrouped AlexNet + 4096/4096/1000) at N=2."""
    _check(oracle, _models().alexnet(batch=2, precision=prec))


@pytest.mark.parametrize("prec", ["ffma", "bf16"])
def test_step_obeys_per_layer_algorithms(oracle, prec):
    """The executor runs the planner's Selection: conv2 FFT, conv3 Winograd,
    conv4 FFT, conv5 Winograd inside the AlexNet-227 step."""
    m = _models()
    cfg = m.apply_selection(m.alexnet(batch=2, precision=prec),
                            {"2": "fft", "3": "winograd", "4": "fft", "5": "winograd"})
    algos = [L.get("algo", "gemm") for L in cfg["layers"] if L["op"] == "conv"]
    assert algos[:5] == ["gemm", "fft", "winograd", "fft", "winograd"]
    _check(oracle, cfg)


def test_profile_plan_train_loop(oracle):
    """Profile -> reference-format catalog -> plan_batch_size -> train with the
    chosen mini-batch and per-layer algorithms (tiny chain, all three families)."""
    from paper_1709_06622_b200 import planner, profiler
    m = _models()
    base = m.from_net("input 20 20 8\nconv 3 1 1 16\npool 2 2 0\nconv 3 1 1 24\nconv 5 1 2 32\n"
                      "pool 2 2 0\nfc 10\n", batch=1, precision="bf16")
    prof = profiler.profile(profiler.feature_conv_specs(base), [32, 64], reps=2)
    assert prof["csv"].startswith("layer_id,algorithm,batch_size,time_seconds,memory_bits")
    algos = {r["algorithm"] for r in prof["rows"]}
    assert algos == {"gemm", "winograd", "fft"}
    plan = profiler.plan(profiler.net_text(base), prof["csv"], 180 * 10**9 * 8, 50_000)
    rec = plan["recommended"]
    assert rec in (32, 64)
    sel = next(c["solve"] for c in plan["candidates"] if c["batch_size"] == rec)
    cfg = m.apply_selection(m.from_net(profiler.net_text(base), batch=rec, precision="bf16"),
                            sel["assignment"])
    _check(oracle, cfg)
    assert planner.default().call("catalog_options", catalog=prof["csv"], batch=rec)["options"]


def test_from_net_fixture_chain(oracle):
    """The reference's own alexnet.net fixture, executed as a chain."""
    import planner_cases
    cfg = _models().from_net(planner_cases.fixture("alexnet.net"), batch=2, precision="bf16")
    _check(oracle, cfg)


def test_step_is_deterministic():
    cfg = _models().tiny_resnet(batch=4, precision="bf16")
    a, b = _run_step(cfg), _run_step(cfg)
    assert torch.equal(a.tensor("grad"), b.tensor("grad"))
    assert torch.equal(a.tensor("param"), b.tensor("param"))
    a.step()
    b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.tensor("param"), b.tensor("param"))


def test_host_batch_path_matches_resident_batch(oracle):
    from paper_1709_06622_b200.trainer import Trainer
    cfg = _models().tiny_resnet(batch=4, precision="bf16")
    a = _run_step(cfg)
    b = Trainer(cfg)
    ref = OracleStep(oracle, cfg, b.describe())
    x, lab = ref.inputs()
    b.set_batch(torch.from_numpy(x.copy()).pin_memory(), torch.from_numpy(lab.copy()).pin_memory())
    b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.tensor("grad"), b.tensor("grad"))


def _stem_net(batch=4):
    return _models().from_net("input 40 38 3\nconv 7 2 3 64\npool 3 2 1\nconv 3 1 1 64\nfc 10\n",
                              batch=batch, precision="bf16")


@pytest.mark.parametrize("net", ["tiny_resnet", "stem_rows"])
def test_staged_u8_batches_pipeline(oracle, net):
    """Staged uint8 batches (copy stream, two slots) feed consecutive steps in
    order and equal the synchronous fp32 host path on the converted values
    (the uint8 preparation writes the stem's 4-channel rows directly, the fp32
    path repacks them from the 8-channel input)."""
    from paper_1709_06622_b200.trainer import Trainer
    cfg = _models().tiny_resnet(batch=4, precision="bf16") if net == "tiny_resnet" else _stem_net()
    a, b = Trainer(cfg), Trainer(cfg)
    lay = a.describe()
    n, h, w = lay["layers"][0]["shape"][:3]
    cl = lay["layers"][0]["c_logical"]
    rng = np.random.default_rng(5)
    batches = [rng.integers(0, 256, (n, h, w, cl), dtype=np.uint8) for _ in range(3)]
    labels = [rng.integers(0, cfg["classes"], (n,), dtype=np.int32) for _ in range(3)]
    pinned = [(torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory())
              for x, y in zip(batches, labels)]
    a.stage_batch(*pinned[0])
    a.stage_batch(*pinned[1])
    for i in range(3):
        a.step()
        if i + 2 < 3:
            a.stage_batch(*pinned[i + 2])
        xf = ((batches[i].astype(np.float32) + 0.5) * np.float32(0.0078125) - 1).astype(np.float32)
        b.set_batch(torch.from_numpy(xf).pin_memory(), torch.from_numpy(labels[i]).pin_memory())
        b.step()
        torch.cuda.synchronize()
        assert torch.equal(a.tensor("grad"), b.tensor("grad")), i
        assert torch.equal(a.tensor("param"), b.tensor("param")), i
    first_conv = next(L for L in a.describe()["layers"] if L["op"] == "conv")  # (planned at the first step)
    assert first_conv["stem_rows"]  # both stems (K padded to 64) take the row-window kernels


def test_cuda_graph_replay_matches_eager_steps():
    """After two eager warm-up steps the trainer replays a captured CUDA graph
    of the step; parameters and momentum must match eager execution bitwise."""
    from paper_1709_06622_b200.trainer import Trainer
    cfg = _models().tiny_resnet(batch=4, precision="bf16")
    eager = dict(cfg, cuda_graph=False)
    a, b = Trainer(cfg), Trainer(eager)
    for _ in range(6):
        a.step()
        b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.tensor("param"), b.tensor("param"))
    assert torch.equal(a.tensor("grad"), b.tensor("grad"))
    assert a.launch_count() == b.launch_count()


def test_async_ps_single_gpu_staleness_one(oracle):
    """ps_async on one GPU: the update of step 0 overlaps step 1, which still
    computes with W_0, so both updates apply g(W_0): W_2 = sgd(sgd(W_0, g), g)."""
    from paper_1709_06622_b200.trainer import Trainer
    cfg = _models().tiny_resnet(batch=4, precision="bf16")
    c0 = dict(cfg, lr=0.0)
    t0 = Trainer(c0)
    t0.step()
    torch.cuda.synchronize()
    w0 = t0.tensor("param").cpu().numpy()
    g = t0.tensor("grad").cpu().numpy()
    w1, v1 = oracle.sgd(w0, g, np.zeros_like(w0), cfg["lr"], cfg["momentum"], cfg["weight_decay"], 1.0)
    w2, _ = oracle.sgd(w1, g, v1, cfg["lr"], cfg["momentum"], cfg["weight_decay"], 1.0)
    t = Trainer(dict(cfg, ps_async=True))
    t.step()
    t.step()
    t.finish()
    torch.cuda.synchronize()
    assert np.array_equal(t.tensor("param").cpu().numpy(), w2)
    assert np.array_equal(t.tensor("wcompute").float().cpu().numpy(), oracle.round_bf16(w2))


@pytest.mark.parametrize("model", ["tiny_resnet", "tiny_packnet"])
def test_async_ps_four_steps_staleness_one(oracle, model):
    """ps_async over four steps, so the step reads weight buffer 1 (steps 2)
    as well as buffer 0: every step's gradient must be taken at the
    one-update-old weights, including the dgrad of layers whose bf16 w^T is
    packed per step (tiny_packnet's K = 96 3x3 conv)."""
    from async_ref import expected_async_weights
    from paper_1709_06622_b200.trainer import Trainer
    cfg = getattr(_models(), model)(batch=4, precision="bf16")
    t = Trainer(dict(cfg, ps_async=True))
    t0 = Trainer(dict(cfg, lr=0.0))
    t0.step()
    torch.cuda.synchronize()
    w0 = t0.tensor("param").cpu().numpy()
    if model == "tiny_packnet":
        assert any(L.get("packed_dgrad_weights") for L in t0.describe()["layers"])
    for _ in range(4):
        t.step()
    t.finish()
    torch.cuda.synchronize()
    w4 = expected_async_weights(oracle, cfg, w0, 4)
    assert np.array_equal(t.tensor("param").cpu().numpy(), w4)
    assert np.array_equal(t.tensor("wcompute").float().cpu().numpy(), oracle.round_bf16(w4))


def test_loss_decreases_over_steps():
    from paper_1709_06622_b200.trainer import Trainer
    cfg = _models().tiny_resnet(batch=8, precision="bf16", lr=0.05)
    t = Trainer(cfg)
    losses = []
    for _ in range(15):
        t.step()
        losses.append(t.loss())
    assert losses[-1] < losses[0], losses


def test_phase_times_and_launch_count():
    from paper_1709_06622_b200.trainer import Trainer
    t = Trainer(_models().tiny_resnet(batch=4, precision="bf16"))
    t.enable_timing(True)
    t.step()
    ph = t.phase_times()
    assert set(ph) == set(Trainer.PHASES) and all(v >= 0 for v in ph.values())
    assert ph["fwd"] > 0 and ph["bwd"] > 0
    assert t.launch_count() > 20
