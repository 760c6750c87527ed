"""Model graphs for the training-step executor (libtcb.so tcb_trainer_*).

A model is a JSON-able dict: {"batch", "classes", "precision", "seed", "lr",
"momentum", "weight_decay", "layers": [...]}; layers are in topological order
and name their inputs. Ops: input, conv (fc layers are convs spanning the
whole input map), maxpool, avgpool (global, or windowed with f/stride/pad),
concat (channel concatenation of same-size tensors), loss (softmax
cross-entropy).

Configs follow BASELINE.json:
  C1 lenet        28x28x1, the CPU-oracle scale case
  C2 alexnet      227x227x3 conv stack + 4096/4096/1000 classifier (ungrouped)
  C3 resnet50     224x224x3, torchvision v1.5 geometry (stride on the 3x3),
                  ResNet-50-shaped: conv/ReLU/residual topology exact, no BN
                  (the reference's network model has no normalisation layers)
  C4 inception_v3 299x299x3, torchvision geometry without the aux head: the
                  full branched graph (5b-7c modules, concat, avg/max pool
                  branches), no BN; `inception_v3_convs` lists its convs for
                  the per-layer algorithm profiling
  C5 vgg16        224x224x3, 13 convs + 25088/4096/4096/1000 classifier
`from_net` builds a chain from the reference's `.net` format (conv/pool/fc),
so the planner's network model and the executor share one description.
"""
from __future__ import annotations

import copy

DEFAULTS = {"precision": "bf16", "seed": 20260810, "lr": 0.01, "momentum": 0.9,
            "weight_decay": 0.0, "classes": 1000}


class _Builder:
    def __init__(self, batch, h, w, c, **opts):
        self.cfg = dict(DEFAULTS)
        self.cfg.update(opts)
        self.cfg["batch"] = batch
        self.layers = [{"name": "data", "op": "input", "h": h, "w": w, "c": c}]
        self.shape = {"data": (h, w, c)}
        self.last = "data"
        self._n = 0

    def _name(self, prefix):
        self._n += 1
        return f"{prefix}{self._n}"

    def conv(self, k, r, s=None, pad=0, stride=1, relu=True, bias=False, src=None, residual=None,
             name=None, pad_w=None, stride_w=None, init_gain=None):
        src = src or self.last
        s = r if s is None else s
        name = name or self._name("conv")
        h, w, c = self.shape[src]
        pw = pad if pad_w is None else pad_w
        sw = stride if stride_w is None else stride_w
        ho = (h + 2 * pad - r) // stride + 1
        wo = (w + 2 * pw - s) // sw + 1
        L = {"name": name, "op": "conv", "in": src, "k": k, "r": r, "s": s, "pad_h": pad,
             "pad_w": pw, "stride_h": stride, "stride_w": sw, "relu": relu, "bias": bias}
        if residual:
            L["residual"] = residual
        if init_gain is not None:
            L["init_gain"] = init_gain
        self.layers.append(L)
        self.shape[name] = (ho, wo, k)
        self.last = name
        return name

    def fc(self, k, relu=True, bias=True, name=None):
        h, w, _ = self.shape[self.last]
        return self.conv(k, h, w, relu=relu, bias=bias, name=name or self._name("fc"))

    def maxpool(self, f, stride=None, pad=0, src=None):
        src = src or self.last
        stride = f if stride is None else stride
        name = self._name("pool")
        h, w, c = self.shape[src]
        self.layers.append({"name": name, "op": "maxpool", "in": src, "f": f, "stride": stride, "pad": pad})
        self.shape[name] = ((h + 2 * pad - f) // stride + 1, (w + 2 * pad - f) // stride + 1, c)
        self.last = name
        return name

    def avgpool(self, f=None, stride=None, pad=0, src=None):
        """Global average pool, or a windowed one (count_include_pad) with f."""
        src = src or self.last
        h, w, c = self.shape[src]
        if f is None:
            name = self._name("gap")
            self.layers.append({"name": name, "op": "avgpool", "in": src})
            self.shape[name] = (1, 1, c)
        else:
            stride = f if stride is None else stride
            name = self._name("apool")
            self.layers.append({"name": name, "op": "avgpool", "in": src, "f": f, "stride": stride, "pad": pad})
            self.shape[name] = ((h + 2 * pad - f) // stride + 1, (w + 2 * pad - f) // stride + 1, c)
        self.last = name
        return name

    def concat(self, srcs, name=None):
        name = name or self._name("cat")
        h, w, _ = self.shape[srcs[0]]
        self.layers.append({"name": name, "op": "concat", "in": list(srcs)})
        self.shape[name] = (h, w, sum(self.shape[x][2] for x in srcs))
        self.last = name
        return name

    def done(self):
        self.layers.append({"name": "loss", "op": "loss", "in": self.last})
        cfg = dict(self.cfg)
        cfg["layers"] = self.layers
        return cfg


def lenet(batch=64, **opts):
    opts.setdefault("classes", 10)
    opts.setdefault("precision", "ffma")
    b = _Builder(batch, 28, 28, 1, **opts)
    b.conv(20, 5, bias=True)
    b.maxpool(2)
    b.conv(50, 5, bias=True)
    b.maxpool(2)
    b.fc(500)
    b.fc(opts["classes"], relu=False)
    return b.done()


def alexnet(batch=128, **opts):
    b = _Builder(batch, 227, 227, 3, **opts)
    b.conv(96, 11, stride=4, bias=True)
    b.maxpool(3, 2)
    b.conv(256, 5, pad=2, bias=True)
    b.maxpool(3, 2)
    b.conv(384, 3, pad=1, bias=True)
    b.conv(384, 3, pad=1, bias=True)
    b.conv(256, 3, pad=1, bias=True)
    b.maxpool(3, 2)
    b.fc(4096)
    b.fc(4096)
    b.fc(b.cfg["classes"], relu=False)
    return b.done()


def vgg16(batch=64, **opts):
    b = _Builder(batch, 224, 224, 3, **opts)
    for width, reps in ((64, 2), (128, 2), (256, 3), (512, 3), (512, 3)):
        for _ in range(reps):
            b.conv(width, 3, pad=1, bias=True)
        b.maxpool(2)
    b.fc(4096)
    b.fc(4096)
    b.fc(b.cfg["classes"], relu=False)
    return b.done()


def resnet50(batch=256, stages=(3, 4, 6, 3), width=64, image=224, **opts):
    b = _Builder(batch, image, image, 3, **opts)
    b.conv(width, 7, pad=3, stride=2, name="stem")
    x = b.maxpool(3, 2, pad=1)
    inplanes = width
    for si, blocks in enumerate(stages):
        planes = width * (2 ** si)
        for bi in range(blocks):
            stride = 2 if (bi == 0 and si > 0) else 1
            pre = f"s{si + 1}b{bi + 1}"
            y = b.conv(planes, 1, src=x, name=pre + "_c1")
            y = b.conv(planes, 3, pad=1, stride=stride, name=pre + "_c2")
            # the projection comes after c1 in graph order so that c1 (dense, stride 1)
            # is the final writer of the block input's gradient: the strided projection
            # dgrad then writes plain zeros at the pixels its stride skips, instead of
            # copying c1's gradient x ReLU mask there
            if bi == 0:
                short = b.conv(planes * 4, 1, stride=stride, relu=False, src=x, name=pre + "_proj")
            else:
                short = x
            # no BN: a small init gain on the branch's last conv keeps the residual
            # stream's variance bounded over the 16 blocks (Fixup-style)
            x = b.conv(planes * 4, 1, src=y, residual=short, name=pre + "_c3", init_gain=0.2)
            inplanes = planes * 4
    b.avgpool()
    b.fc(b.cfg["classes"], relu=False, name="fc")
    del inplanes
    return b.done()


def tiny_resnet(batch=4, **opts):
    """Small residual net covering every executor feature (stem stride, maxpool,
    projection + identity shortcuts, global pool, fc) for parity tests."""
    opts.setdefault("classes", 10)
    return resnet50(batch, stages=(2, 1), width=8, image=20, **opts)


def tiny_packnet(batch=4, **opts):
    """Small chain whose middle 3x3 conv has K % 64 != 0 (96 filters) and feeds
    a 1x1 conv, so its bf16 dgrad takes the cp.async-gather path with the
    per-step packed w^T (the executor's pack_wT layers: AlexNet conv1-style and
    many Inception-v3 convs)."""
    opts.setdefault("classes", 10)
    b = _Builder(batch, 12, 12, 8, **opts)
    b.conv(64, 3, pad=1, bias=True)
    b.conv(96, 3, pad=1, bias=True)
    b.conv(64, 1)
    b.avgpool()
    b.fc(b.cfg["classes"], relu=False)
    return b.done()


def from_net(text: str, batch: int, classes: int | None = None, **opts):
    """Chain network from the reference `.net` format (input/conv/pool/fc):
    ReLU after every conv and every fc but the last; pools are max pools."""
    b = None
    fcs = []
    for raw in text.splitlines():
        tok = raw.split("#", 1)[0].split()
        if not tok:
            continue
        if tok[0] == "input":
            w, h, d = (int(v) for v in tok[1:4])
            b = _Builder(batch, h, w, d, **opts)
        elif tok[0] == "conv":
            f, s, p, k = (int(v) for v in tok[1:5])
            b.conv(k, f, pad=p, stride=s, bias=True)
        elif tok[0] == "pool":
            f, s, p = (int(v) for v in tok[1:4])
            b.maxpool(f, s, p)
        elif tok[0] == "fc":
            fcs.append(int(tok[1]))
    # A first fc line equal to the flattened feature size is the classifier's
    # input vector (the junction convention), not a layer.
    h, w, c = b.shape[b.last]
    if len(fcs) > 1 and fcs[0] == h * w * c:
        fcs = fcs[1:]
    if classes is not None:
        fcs[-1] = classes
    b.cfg["classes"] = fcs[-1]
    for i, n in enumerate(fcs):
        b.fc(n, relu=i + 1 < len(fcs))
    return b.done()


def inception_v3_convs(batch=128):
    """Conv geometries of Inception-v3 (299x299x3, no aux head) in execution
    order: (name, h, w, c, k, r, s, pad_h, pad_w, stride). Used for the C4
    per-layer algorithm comparison; branches/concat are not executed."""
    L = []

    def add(name, h, w, c, k, r, s, ph, pw, st=1):
        L.append((name, h, w, c, k, r, s, ph, pw, st))
        return (h + 2 * ph - r) // st + 1, (w + 2 * pw - s) // st + 1

    h, w = add("Conv2d_1a_3x3", 299, 299, 3, 32, 3, 3, 0, 0, 2)
    h, w = add("Conv2d_2a_3x3", h, w, 32, 32, 3, 3, 0, 0)
    h, w = add("Conv2d_2b_3x3", h, w, 32, 64, 3, 3, 1, 1)
    h, w = (h - 3) // 2 + 1, (w - 3) // 2 + 1
    h, w = add("Conv2d_3b_1x1", h, w, 64, 80, 1, 1, 0, 0)
    h, w = add("Conv2d_4a_3x3", h, w, 80, 192, 3, 3, 0, 0)
    h, w = (h - 3) // 2 + 1, (w - 3) // 2 + 1  # 35x35x192
    c = 192
    for i, pool_feat in enumerate((32, 64, 64)):  # Mixed_5b/5c/5d
        p = f"Mixed_5{'bcd'[i]}"
        add(p + "_b1x1", h, w, c, 64, 1, 1, 0, 0)
        add(p + "_b5x5_1", h, w, c, 48, 1, 1, 0, 0)
        add(p + "_b5x5_2", h, w, 48, 64, 5, 5, 2, 2)
        add(p + "_b3x3dbl_1", h, w, c, 64, 1, 1, 0, 0)
        add(p + "_b3x3dbl_2", h, w, 64, 96, 3, 3, 1, 1)
        add(p + "_b3x3dbl_3", h, w, 96, 96, 3, 3, 1, 1)
        add(p + "_bpool", h, w, c, pool_feat, 1, 1, 0, 0)
        c = 64 + 64 + 96 + pool_feat
    add("Mixed_6a_b3x3", h, w, c, 384, 3, 3, 0, 0, 2)
    add("Mixed_6a_dbl_1", h, w, c, 64, 1, 1, 0, 0)
    add("Mixed_6a_dbl_2", h, w, 64, 96, 3, 3, 1, 1)
    add("Mixed_6a_dbl_3", h, w, 96, 96, 3, 3, 0, 0, 2)
    h, w = (h - 3) // 2 + 1, (w - 3) // 2 + 1  # 17x17
    c = 384 + 96 + c
    for i, c7 in enumerate((128, 160, 160, 192)):
        p = f"Mixed_6{'bcde'[i]}"
        add(p + "_b1x1", h, w, c, 192, 1, 1, 0, 0)
        add(p + "_b7x7_1", h, w, c, c7, 1, 1, 0, 0)
        add(p + "_b7x7_2", h, w, c7, c7, 1, 7, 0, 3)
        add(p + "_b7x7_3", h, w, c7, 192, 7, 1, 3, 0)
        add(p + "_dbl_1", h, w, c, c7, 1, 1, 0, 0)
        add(p + "_dbl_2", h, w, c7, c7, 7, 1, 3, 0)
        add(p + "_dbl_3", h, w, c7, c7, 1, 7, 0, 3)
        add(p + "_dbl_4", h, w, c7, c7, 7, 1, 3, 0)
        add(p + "_dbl_5", h, w, c7, 192, 1, 7, 0, 3)
        add(p + "_bpool", h, w, c, 192, 1, 1, 0, 0)
        c = 768
    add("Mixed_7a_b3x3_1", h, w, c, 192, 1, 1, 0, 0)
    add("Mixed_7a_b3x3_2", h, w, 192, 320, 3, 3, 0, 0, 2)
    add("Mixed_7a_b7x7x3_1", h, w, c, 192, 1, 1, 0, 0)
    add("Mixed_7a_b7x7x3_2", h, w, 192, 192, 1, 7, 0, 3)
    add("Mixed_7a_b7x7x3_3", h, w, 192, 192, 7, 1, 3, 0)
    add("Mixed_7a_b7x7x3_4", h, w, 192, 192, 3, 3, 0, 0, 2)
    h, w = (h - 3) // 2 + 1, (w - 3) // 2 + 1  # 8x8
    c = 320 + 192 + 768
    for i in range(2):
        p = f"Mixed_7{'bc'[i]}"
        add(p + "_b1x1", h, w, c, 320, 1, 1, 0, 0)
        add(p + "_b3x3_1", h, w, c, 384, 1, 1, 0, 0)
        add(p + "_b3x3_2a", h, w, 384, 384, 1, 3, 0, 1)
        add(p + "_b3x3_2b", h, w, 384, 384, 3, 1, 1, 0)
        add(p + "_dbl_1", h, w, c, 448, 1, 1, 0, 0)
        add(p + "_dbl_2", h, w, 448, 384, 3, 3, 1, 1)
        add(p + "_dbl_3a", h, w, 384, 384, 1, 3, 0, 1)
        add(p + "_dbl_3b", h, w, 384, 384, 3, 1, 1, 0)
        add(p + "_bpool", h, w, c, 192, 1, 1, 0, 0)
        c = 2048
    return [dict(zip(("name", "h", "w", "c", "k", "r", "s", "pad_h", "pad_w", "stride"), t),
                 n=batch) for t in L]


def inception_v3(batch=128, image=299, width=1.0, **opts):
    """C4: Inception-v3 (torchvision geometry, no aux head, no BN) as a
    branched graph — every module's branches, their channel concat, the 3x3
    average-pool (stride 1, pad 1) and max-pool branches. `width` scales every
    channel count (multiples of 8 kept) for small parity cases. Its convs in
    graph order are `inception_v3_convs` (the planner's layer ids)."""
    def ch(k):
        return max(8, int(round(k * width / 8)) * 8)

    b = _Builder(batch, image, image, 3, **opts)
    b.conv(ch(32), 3, stride=2, name="Conv2d_1a_3x3")
    b.conv(ch(32), 3, name="Conv2d_2a_3x3")
    b.conv(ch(64), 3, pad=1, name="Conv2d_2b_3x3")
    b.maxpool(3, 2)
    b.conv(ch(80), 1, name="Conv2d_3b_1x1")
    b.conv(ch(192), 3, name="Conv2d_4a_3x3")
    x = b.maxpool(3, 2)
    for i, pool_feat in enumerate((32, 64, 64)):  # Mixed_5b/5c/5d (35x35)
        p = f"Mixed_5{'bcd'[i]}"
        b1 = b.conv(ch(64), 1, src=x, name=p + "_b1x1")
        b5 = b.conv(ch(48), 1, src=x, name=p + "_b5x5_1")
        b5 = b.conv(ch(64), 5, pad=2, src=b5, name=p + "_b5x5_2")
        b3 = b.conv(ch(64), 1, src=x, name=p + "_b3x3dbl_1")
        b3 = b.conv(ch(96), 3, pad=1, src=b3, name=p + "_b3x3dbl_2")
        b3 = b.conv(ch(96), 3, pad=1, src=b3, name=p + "_b3x3dbl_3")
        bp = b.avgpool(3, 1, 1, src=x)
        bp = b.conv(ch(pool_feat), 1, src=bp, name=p + "_bpool")
        x = b.concat([b1, b5, b3, bp], name=p)
    # Mixed_6a (35 -> 17)
    b3 = b.conv(ch(384), 3, stride=2, src=x, name="Mixed_6a_b3x3")
    bd = b.conv(ch(64), 1, src=x, name="Mixed_6a_dbl_1")
    bd = b.conv(ch(96), 3, pad=1, src=bd, name="Mixed_6a_dbl_2")
    bd = b.conv(ch(96), 3, stride=2, src=bd, name="Mixed_6a_dbl_3")
    bp = b.maxpool(3, 2, src=x)
    x = b.concat([b3, bd, bp], name="Mixed_6a")
    for i, c7 in enumerate((128, 160, 160, 192)):  # Mixed_6b-6e (17x17)
        p = f"Mixed_6{'bcde'[i]}"
        b1 = b.conv(ch(192), 1, src=x, name=p + "_b1x1")
        b7 = b.conv(ch(c7), 1, src=x, name=p + "_b7x7_1")
        b7 = b.conv(ch(c7), 1, 7, pad=0, pad_w=3, src=b7, name=p + "_b7x7_2")
        b7 = b.conv(ch(192), 7, 1, pad=3, pad_w=0, src=b7, name=p + "_b7x7_3")
        bd = b.conv(ch(c7), 1, src=x, name=p + "_dbl_1")
        bd = b.conv(ch(c7), 7, 1, pad=3, pad_w=0, src=bd, name=p + "_dbl_2")
        bd = b.conv(ch(c7), 1, 7, pad=0, pad_w=3, src=bd, name=p + "_dbl_3")
        bd = b.conv(ch(c7), 7, 1, pad=3, pad_w=0, src=bd, name=p + "_dbl_4")
        bd = b.conv(ch(192), 1, 7, pad=0, pad_w=3, src=bd, name=p + "_dbl_5")
        bp = b.avgpool(3, 1, 1, src=x)
        bp = b.conv(ch(192), 1, src=bp, name=p + "_bpool")
        x = b.concat([b1, b7, bd, bp], name=p)
    # Mixed_7a (17 -> 8)
    b3 = b.conv(ch(192), 1, src=x, name="Mixed_7a_b3x3_1")
    b3 = b.conv(ch(320), 3, stride=2, src=b3, name="Mixed_7a_b3x3_2")
    b7 = b.conv(ch(192), 1, src=x, name="Mixed_7a_b7x7x3_1")
    b7 = b.conv(ch(192), 1, 7, pad=0, pad_w=3, src=b7, name="Mixed_7a_b7x7x3_2")
    b7 = b.conv(ch(192), 7, 1, pad=3, pad_w=0, src=b7, name="Mixed_7a_b7x7x3_3")
    b7 = b.conv(ch(192), 3, stride=2, src=b7, name="Mixed_7a_b7x7x3_4")
    bp = b.maxpool(3, 2, src=x)
    x = b.concat([b3, b7, bp], name="Mixed_7a")
    for i in range(2):  # Mixed_7b / 7c (8x8)
        p = f"Mixed_7{'bc'[i]}"
        b1 = b.conv(ch(320), 1, src=x, name=p + "_b1x1")
        t3 = b.conv(ch(384), 1, src=x, name=p + "_b3x3_1")
        t3a = b.conv(ch(384), 1, 3, pad=0, pad_w=1, src=t3, name=p + "_b3x3_2a")
        t3b = b.conv(ch(384), 3, 1, pad=1, pad_w=0, src=t3, name=p + "_b3x3_2b")
        td = b.conv(ch(448), 1, src=x, name=p + "_dbl_1")
        td = b.conv(ch(384), 3, pad=1, src=td, name=p + "_dbl_2")
        tda = b.conv(ch(384), 1, 3, pad=0, pad_w=1, src=td, name=p + "_dbl_3a")
        tdb = b.conv(ch(384), 3, 1, pad=1, pad_w=0, src=td, name=p + "_dbl_3b")
        bp = b.avgpool(3, 1, 1, src=x)
        bp = b.conv(ch(192), 1, src=bp, name=p + "_bpool")
        x = b.concat([b1, t3a, t3b, tda, tdb, bp], name=p)
    b.avgpool()
    b.fc(b.cfg["classes"], relu=False, name="fc")
    return b.done()


def apply_selection(cfg: dict, assignment: dict) -> dict:
    """Set each feature conv's algorithm from a planner Selection.assignment
    ({layer_id (1-based over the feature convs, as the catalog indexes them):
    "gemm"|"winograd"|"fft"}); fc layers always run as GEMMs."""
    out = copy.deepcopy(cfg)
    i = 0
    for L in out["layers"]:
        if L["op"] == "conv" and not L["name"].startswith("fc"):
            i += 1
            algo = assignment.get(str(i), assignment.get(i))
            if algo is not None:
                L["algo"] = algo
    return out


CONFIGS = {"lenet": lenet, "alexnet": alexnet, "vgg16": vgg16, "resnet50": resnet50,
           "tiny_resnet": tiny_resnet, "inception_v3": inception_v3}


def build(name: str, **kw):
    return copy.deepcopy(CONFIGS[name](**kw))


def conv_layers(cfg):
    """(name, geometry dict) of every conv layer in execution order."""
    shapes = {}
    out = []
    for L in cfg["layers"]:
        if L["op"] == "input":
            shapes[L["name"]] = (L["h"], L["w"], L["c"])
        elif L["op"] == "conv":
            h, w, c = shapes[L["in"]]
            g = dict(n=cfg["batch"], h=h, w=w, c=c, k=L["k"], r=L["r"], s=L["s"],
                     pad_h=L["pad_h"], pad_w=L["pad_w"], stride_h=L["stride_h"], stride_w=L["stride_w"])
            ho = (h + 2 * g["pad_h"] - g["r"]) // g["stride_h"] + 1
            wo = (w + 2 * g["pad_w"] - g["s"]) // g["stride_w"] + 1
            shapes[L["name"]] = (ho, wo, L["k"])
            out.append((L["name"], g))
        elif L["op"] == "maxpool":
            h, w, c = shapes[L["in"]]
            f, s, p = L["f"], L["stride"], L["pad"]
            shapes[L["name"]] = ((h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1, c)
        elif L["op"] == "avgpool":
            h, w, c = shapes[L["in"]]
            if "f" in L:
                f, s, p = L["f"], L["stride"], L["pad"]
                shapes[L["name"]] = ((h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1, c)
            else:
                shapes[L["name"]] = (1, 1, c)
        elif L["op"] == "concat":
            h, w, _ = shapes[L["in"][0]]
            shapes[L["name"]] = (h, w, sum(shapes[x][2] for x in L["in"]))
    return out


def flops_per_image(cfg):
    """Direct-conv multiply-add FLOPs (2*MACs) of one forward pass per image."""
    tot = 0
    for _, g in conv_layers(cfg):
        ho = (g["h"] + 2 * g["pad_h"] - g["r"]) // g["stride_h"] + 1
        wo = (g["w"] + 2 * g["pad_w"] - g["s"]) // g["stride_w"] + 1
        tot += 2 * ho * wo * g["k"] * g["c"] * g["r"] * g["s"]
    return tot
