"""CPU restatement of one data-parallel training step — TEST INFRASTRUCTURE.

Walks the same model graph as the C++ executor (paper_1709_06622_b200/models.py
config) with the C oracle ops (oracle/numerics.c, fp64 accumulation):
forward (conv + bias + residual + ReLU, max/avg pools, channel concat), softmax
cross-entropy, backward (dgrad with residual-gradient fan-in and ReLU masks,
wgrad + bias grads in the flat PS layout), then the momentum-SGD update of
paper step 6. In bf16 mode every stored
tensor is rounded to bf16 exactly where the device stores bf16, so the two
paths see the same operands.

Parity of this restatement is unpinned by the reference (no conv/SGD values
exist in /root/reference — SURVEY.md §8c); it follows the paper's definitions.
"""
from __future__ import annotations

import numpy as np


def _rel(got, ref):
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0))


class DeviceTeacher:
    """Reads the executor's tensors (logical channels) for teacher-forced parity."""

    def __init__(self, trainer, layout):
        self.t, self.layers = trainer, layout["layers"]

    def _get(self, name, i):
        L = self.layers[i]
        a = self.t.tensor(f"{name}:{i}").float().cpu().numpy().reshape(L["shape"])
        return a[..., :L["c_logical"]].astype(np.float32)

    def act(self, i):
        return self._get("act", i)

    def grad(self, i):
        return self._get("dact", i)

    def argmax(self, i):
        import torch
        L = self.layers[i]
        a = self.t.tensor(f"argmax:{i}", dtype=torch.uint8).cpu().numpy().reshape(L["shape"])
        return np.ascontiguousarray(a[..., :L["c_logical"]]).ravel()


class SubsetTeacher(DeviceTeacher):
    """The device's tensors restricted to a few images of its batch (sliced on
    the device before the copy), for layer-local parity of a large-batch step:
    every op but the weight gradient is independent per image."""

    def __init__(self, trainer, layout, images):
        super().__init__(trainer, layout)
        self.images = list(images)

    def _sub(self, name, i, dtype=None):
        import torch
        L = self.layers[i]
        t = self.t.tensor(f"{name}:{i}", dtype=dtype).view(*L["shape"])
        return t[torch.tensor(self.images, device=t.device)][..., :L["c_logical"]]

    def act(self, i):
        return self._sub("act", i).float().cpu().numpy()

    def grad(self, i):
        return self._sub("dact", i).float().cpu().numpy()

    def argmax(self, i):
        import torch
        return np.ascontiguousarray(self._sub("argmax", i, torch.uint8).cpu().numpy()).ravel()

    def full(self, name, i, channels=None):
        """A whole-batch tensor (logical channels, or the given channel subset)."""
        import torch
        L = self.layers[i]
        t = self.t.tensor(f"{name}:{i}").view(*L["shape"])[..., :L["c_logical"]]
        if channels is not None:
            t = t[..., torch.tensor(channels, device=t.device)]
        return t.float().cpu().numpy()

    def layout(self):
        """Copy of the layout with the batch dimension set to the subset size."""
        import copy
        lay = copy.deepcopy({"layers": self.layers})
        for L in lay["layers"]:
            L["shape"][0] = len(self.images)
            if "geom" in L:
                L["geom"][0] = len(self.images)
        return lay


class OracleStep:
    def __init__(self, oracle, cfg: dict, layout: dict, rank: int = 0, world: int = 1):
        self.o = oracle
        self.cfg = cfg
        self.layout = layout
        self.rank, self.world = rank, world
        self.bf16 = cfg.get("precision", "bf16") == "bf16"
        self.seed = cfg.get("seed", 20260810)
        self.layers = layout["layers"]
        self.params = {}  # conv index -> (w logical [K,R,S,Cl] float32, bias float32 or None)
        for L in self.layers:
            if L["op"] != "conv":
                continue
            k, r, s = L["c_logical"], L["geom"][5], L["geom"][6]
            cl = self.layers[L["in"]]["c_logical"]
            n = k * r * s * cl
            a = np.float32(L["init_scale"])
            w = oracle.uniform(n, self.seed, 1000 + L["conv_index"], -a, a).reshape(k, r, s, cl)
            b = np.zeros(k, np.float32) if L["bias"] else None
            self.params[L["index"]] = [w, b]

    # storage rounding of activations / gradients
    def _st(self, a):
        a = np.asarray(a, np.float32)
        return self.o.round_bf16(a) if self.bf16 else a

    def _geom(self, L, logical_in_c):
        g = L["geom"]
        return dict(n=g[0], h=g[1], w=g[2], c=logical_in_c, k=L["c_logical"], r=g[5], s=g[6],
                    pad_h=g[7], pad_w=g[8], stride_h=g[9], stride_w=g[10])

    def inputs(self):
        inp = self.layers[0]
        n, h, w, _ = inp["shape"]
        cl = inp["c_logical"]
        x = self.o.uniform(n * h * w * cl, self.seed + self.rank, 1, -1.0, 1.0).reshape(n, h, w, cl)
        lab = self.o.labels(n, self.cfg["classes"], self.seed + self.rank)
        return x, lab

    def run(self, x=None, labels=None, teacher=None, wgrad=True, loss_batch=None, argmax_src=None):
        """One step. With `teacher` (an object exposing the DEVICE's tensors:
        act(i), grad(i), argmax(i), in logical channels), every op is
        recomputed from the device's own inputs — layer-local parity — and the
        relative error of each device output is recorded in self.local_err.
        Image-subset replays of a large batch (SubsetTeacher): `loss_batch` is
        the device's batch N (the loss gradient is (p - y) / N), and
        wgrad=False skips the weight gradients (they sum over all N images;
        checked separately per sampled layer). `argmax_src`: end to end, but
        the step's discrete decisions taken from the device — max-pool argmax
        routing and the ReLU masks (a near-tie of two window values, or a
        pre-activation within rounding of 0, is decided by the last bit, fp32
        vs fp64, and moves a whole gradient value). The fraction of
        disagreeing decisions is recorded in self.argmax_mismatch /
        self.relu_mismatch."""
        o = self.o
        if x is None:
            x, labels = self.inputs()
        act = {0: self._st(x)}
        wq = {i: (self._st(w) if self.bf16 else w) for i, (w, _) in self.params.items()}
        self.local_err = {}
        self.argmax_mismatch = {}
        self.relu_mismatch = {}
        relu_on = {}

        def adopt(kind, i, ref, dev_value):
            if teacher is None:
                return ref
            self.local_err[(kind, self.layers[i]["name"])] = _rel(dev_value, ref)
            return dev_value.reshape(ref.shape)

        # ---------------------------------------------------------- forward
        loss = None
        dlogits = None
        for L in self.layers[1:]:
            i = L["index"]
            if L["op"] == "conv":
                xin = act[L["in"]]
                g = self._geom(L, xin.shape[-1])
                res = act[L["residual"]] if L["residual"] >= 0 else None
                if argmax_src is not None and L["relu"] and teacher is None:
                    pre = o.conv_fwd(g, xin, wq[i], bias=self.params[i][1], residual=res, relu=False)
                    pre = pre.reshape(g["n"], L["shape"][1], L["shape"][2], g["k"])
                    dev_on = argmax_src.act(i) > 0
                    self.relu_mismatch[L["name"]] = float(np.mean(dev_on != (pre > 0)))
                    y = np.where(dev_on, pre, 0.0)
                    relu_on[i] = dev_on
                else:
                    y = o.conv_fwd(g, xin, wq[i], bias=self.params[i][1], residual=res, relu=L["relu"])
                y = self._st(y).reshape(g["n"], L["shape"][1], L["shape"][2], g["k"])
                act[i] = adopt("fwd", i, y, teacher.act(i) if teacher else None)
            elif L["op"] == "maxpool":
                xin = act[L["in"]]
                n, h, w, c = xin.shape
                f, s, p = L["pool"]
                y, arg = o.maxpool_fwd(xin, n, h, w, c, f, s, p)
                y = self._st(y).reshape(L["shape"][0], L["shape"][1], L["shape"][2], c)
                act[i] = adopt("fwd", i, y, teacher.act(i) if teacher else None)
                if teacher:
                    L["_arg"] = teacher.argmax(i)
                elif argmax_src is not None:
                    dev_arg = argmax_src.argmax(i)
                    self.argmax_mismatch[L["name"]] = float(np.mean(dev_arg != arg))
                    L["_arg"] = dev_arg
                else:
                    L["_arg"] = arg
            elif L["op"] == "avgpool":
                xin = act[L["in"]]
                n, h, w, c = xin.shape
                if "pool" in L:
                    f, s, p = L["pool"]
                    y = self._st(o.avgpool2d_fwd(xin, n, h, w, c, f, s, p)).reshape(
                        n, L["shape"][1], L["shape"][2], c)
                else:
                    y = self._st(o.avgpool_fwd(xin, n, h * w, c)).reshape(n, 1, 1, c)
                act[i] = adopt("fwd", i, y, teacher.act(i) if teacher else None)
            elif L["op"] == "concat":
                y = np.concatenate([act[j] for j in L["ins"]], axis=-1)
                act[i] = adopt("fwd", i, y, teacher.act(i) if teacher else None)
            elif L["op"] == "loss":
                z = act[L["in"]]
                n = z.shape[0]
                loss, dl = o.softmax_xent(z.reshape(n, -1), labels, n, z.shape[-1])
                if loss_batch:
                    dl = dl * (n / loss_batch)
                logits_idx = L["in"]
                dlogits = self._st(dl).reshape(z.shape)
                dlogits = adopt("grad", logits_idx, dlogits,
                                teacher.grad(logits_idx) if teacher else None)
        # --------------------------------------------------------- backward
        contrib = {}  # tensor index -> list of float arrays
        G = {logits_idx: dlogits}
        grads = {}
        for L in reversed(self.layers[1:]):
            i = L["index"]
            if L["op"] == "loss":
                continue
            if i not in G:  # finalise this tensor's gradient
                parts = contrib.get(i, [])
                tot = np.sum(parts, axis=0) if parts else np.zeros_like(act[i], np.float64)
                if L["op"] == "conv" and L["relu"]:
                    tot = np.where(relu_on[i] if i in relu_on else act[i] > 0, tot, 0.0)
                ref = self._st(tot).reshape(act[i].shape)
                G[i] = adopt("grad", i, ref, teacher.grad(i) if teacher else None)
            gi = G[i]
            if L["op"] == "conv":
                xin = act[L["in"]]
                g = self._geom(L, xin.shape[-1])
                if wgrad:
                    dw, db = o.conv_wgrad(g, gi, xin, want_db=True)
                    grads[i] = (dw, db if L["bias"] else None)
                if L["residual"] >= 0 and self.layers[L["residual"]]["op"] != "input":
                    contrib.setdefault(L["residual"], []).append(gi.astype(np.float64))
                if self.layers[L["in"]]["op"] != "input":
                    dx = o.conv_dgrad(g, gi, wq[i]).reshape(xin.shape)
                    contrib.setdefault(L["in"], []).append(dx)
            elif L["op"] == "maxpool":
                xin = act[L["in"]]
                n, h, w, c = xin.shape
                f, s, p = L["pool"]
                dx = o.maxpool_bwd(gi, L["_arg"], n, h, w, c, f, s, p).reshape(xin.shape)
                if self.layers[L["in"]]["op"] != "input":
                    contrib.setdefault(L["in"], []).append(dx)
            elif L["op"] == "avgpool":
                xin = act[L["in"]]
                n, h, w, c = xin.shape
                if "pool" in L:
                    f, s, p = L["pool"]
                    dx = o.avgpool2d_bwd(gi, n, h, w, c, f, s, p).reshape(xin.shape)
                else:
                    dx = o.avgpool_bwd(gi.reshape(n, c), n, h * w, c).reshape(xin.shape)
                if self.layers[L["in"]]["op"] != "input":
                    contrib.setdefault(L["in"], []).append(dx)
            elif L["op"] == "concat":
                for j, off in zip(L["ins"], L["coff"]):
                    if self.layers[j]["op"] != "input":
                        cj = act[j].shape[-1]
                        contrib.setdefault(j, []).append(gi[..., off:off + cj].astype(np.float64))
        self.loss, self.act, self.G, self.grads = loss, act, G, grads
        return loss

    def flat_grad(self):
        """Gradients in the executor's flat PS layout (padded channels = 0)."""
        flat = np.zeros(self.layout["param_padded"], np.float64)
        for L in self.layers:
            if L["op"] != "conv":
                continue
            dw, db = self.grads[L["index"]]
            ka, r, s, cp = L["geom"][4], L["geom"][5], L["geom"][6], L["geom"][3]
            k, cl = L["c_logical"], self.layers[L["in"]]["c_logical"]
            w4 = np.zeros((ka, r, s, cp), np.float64)
            w4[:k, ..., :cl] = dw.reshape(k, r, s, cl)
            flat[L["woff"]:L["woff"] + w4.size] = w4.ravel()
            if db is not None:
                flat[L["boff"]:L["boff"] + k] = db
        return flat

    def flat_params(self):
        flat = np.zeros(self.layout["param_padded"], np.float32)
        for L in self.layers:
            if L["op"] != "conv":
                continue
            w, b = self.params[L["index"]]
            ka, r, s, cp = L["geom"][4], L["geom"][5], L["geom"][6], L["geom"][3]
            k, cl = w.shape[0], w.shape[-1]
            w4 = np.zeros((ka, r, s, cp), np.float32)
            w4[:k, ..., :cl] = w
            flat[L["woff"]:L["woff"] + w4.size] = w4.ravel()
            if b is not None:
                flat[L["boff"]:L["boff"] + k] = b
        return flat

    def sgd(self, flat_grad_f32):
        c = self.cfg
        w = self.flat_params()
        v = np.zeros_like(w)
        return self.o.sgd(w, flat_grad_f32, v, c.get("lr", 0.01), c.get("momentum", 0.9),
                          c.get("weight_decay", 0.0), 1.0 / self.world)
