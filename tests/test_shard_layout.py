"""PS shard assignment (e): the executor's flat-buffer layout and
layer->shard table vs the independent CPU restatement (tests/shard_oracle.py),
bit-exact, for every model and G in 1..8; plus a world_size-2 gloo run showing
every rank derives the identical table (host logic of the multi-GPU path).
No GPU needed: layout planning happens at trainer creation."""
import ctypes
import json
import os

import pytest

import shard_oracle

MODELS = [("lenet", dict(batch=64)), ("alexnet", dict(batch=8)), ("vgg16", dict(batch=2)),
          ("resnet50", dict(batch=2)), ("tiny_resnet", dict(batch=2)), ("inception_v3", dict(batch=2))]


def _describe(cfg):
    from paper_1709_06622_b200 import device, trainer
    L = trainer._lib()
    h = ctypes.c_void_p()
    device.check(L.tcb_trainer_create(json.dumps(cfg).encode(), ctypes.byref(h)))
    out = ctypes.c_char_p()
    device.check(L.tcb_trainer_describe(h, ctypes.byref(out)))
    d = json.loads(out.value.decode())
    L.tcb_trainer_destroy(h)
    return d


@pytest.mark.parametrize("precision", ["bf16", "tf32", "ffma"])
@pytest.mark.parametrize("model,kw", MODELS, ids=[m for m, _ in MODELS])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_layout_matches_restatement(model, kw, precision, world):
    from paper_1709_06622_b200 import models
    cfg = models.build(model, precision=precision, **kw)
    cfg["world"] = world
    dev = _describe(cfg)
    ref = shard_oracle.layout(cfg, world)
    assert dev["param_count"] == ref["param_count"]
    assert dev["param_padded"] == ref["param_padded"]
    assert dev["shard"] == ref["shard"]
    convs = [L for L in dev["layers"] if L["op"] == "conv"]
    assert len(convs) == len(ref["layers"])
    for a, b in zip(convs, ref["layers"]):
        assert (a["name"], a["woff"], a["wcount"], a["boff"], a["shards"]) == \
            (b["name"], b["woff"], b["wcount"], b["boff"], b["shards"])
    # shards tile the padded buffer exactly
    assert dev["shard"] * world == dev["param_padded"]
    assert dev["param_padded"] % (64 * world) == 0


def test_true_parameter_counts():
    """Logical parameter counts of the BASELINE configs."""
    from paper_1709_06622_b200 import models
    counts = {m: _describe(models.build(m, precision="ffma", **kw))["param_count"]
              for m, kw in MODELS[:4]}
    assert counts["vgg16"] == 138_357_544          # torchvision VGG-16
    assert counts["alexnet"] == 62_378_344         # ungrouped AlexNet, fc 9216 first
    assert counts["resnet50"] == 25_503_912        # torchvision ResNet-50 minus 53,120 BN params
    assert counts["lenet"] == 431_080
    # torchvision Inception-v3 without the aux head (23,834,568) minus its BN
    # affine parameters: 2 per conv output channel, sum of k over the 94 convs = 17,216
    assert _describe(models.build("inception_v3", batch=2, precision="ffma"))["param_count"] == 23_834_568 - 34_432


def _gloo_rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1709_06622_b200 import models
    cfg = models.build("resnet50", batch=2, precision="bf16")
    cfg["world"] = world
    d = _describe(cfg)
    table = [(L["name"], L["woff"], L["shards"]) for L in d["layers"] if L["op"] == "conv"]
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, d["shard"], d["param_padded"], table))
    dist.destroy_process_group()
    q.put(gathered)


def test_gloo_two_ranks_agree_on_shard_table():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for gathered in results:
        (r0, s0, p0, t0), (r1, s1, p1, t1) = gathered
        assert (r0, r1) == (0, 1)
        assert (s0, p0, t0) == (s1, p1, t1)
        assert s0 * 2 == p0


KEYS = ("index", "name", "op", "in", "residual", "shape", "c_logical", "conv_index", "geom", "relu",
        "bias", "woff", "wcount", "boff", "algo", "shards", "pool", "ins", "coff")


@pytest.mark.parametrize("precision", ["bf16", "ffma"])
@pytest.mark.parametrize("model,kw", MODELS, ids=[m for m, _ in MODELS])
def test_full_description_matches_restatement(model, kw, precision):
    """tests/layout_oracle.py (what the CPU oracle step and bench's reference
    arm use instead of the product library) reproduces tcb_trainer_describe
    node for node, init scales bit-exact in fp32."""
    import numpy as np

    import layout_oracle
    from paper_1709_06622_b200 import models
    cfg = models.build(model, precision=precision, **kw)
    dev = _describe(cfg)
    ref = layout_oracle.describe(cfg)
    for k in ("param_count", "param_padded", "shard", "batch", "classes"):
        assert dev[k] == ref[k], k
    assert len(dev["layers"]) == len(ref["layers"])
    for a, b in zip(dev["layers"], ref["layers"]):
        for k in KEYS:
            if k in a or k in b:
                assert a.get(k) == b.get(k), (a["name"], k, a.get(k), b.get(k))
        if a["op"] == "conv":
            assert np.float32(a["init_scale"]) == np.float32(b["init_scale"]), a["name"]
