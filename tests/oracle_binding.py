"""ctypes/numpy binding of oracle/liboracle.so — test infrastructure only."""
from __future__ import annotations

import ctypes

import numpy as np

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class Geom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("n", "h", "w", "c", "k", "r", "s", "pad_h", "pad_w", "stride_h", "stride_w")]


def out_hw(g):
    return ((g["h"] + 2 * g["pad_h"] - g["r"]) // g["stride_h"] + 1,
            (g["w"] + 2 * g["pad_w"] - g["s"]) // g["stride_w"] + 1)


def _opt(a, dtype=np.float32):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype).ctypes.data_as(ctypes.c_void_p)


class Oracle:
    def __init__(self, path: str):
        L = self.lib = ctypes.CDLL(path)
        L.oracle_fill_uniform.argtypes = [_f32p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_float, ctypes.c_float]
        L.oracle_fill_labels.argtypes = [_i32p, ctypes.c_int, ctypes.c_int, ctypes.c_uint64]
        L.oracle_round_bf16.argtypes = [_f32p, ctypes.c_size_t]
        vp = ctypes.c_void_p
        L.oracle_conv_fwd.argtypes = [ctypes.POINTER(Geom), _f32p, _f32p, vp, vp, ctypes.c_int, _f64p]
        L.oracle_conv_dgrad.argtypes = [ctypes.POINTER(Geom), _f32p, _f32p, vp, vp, _f64p]
        L.oracle_conv_wgrad.argtypes = [ctypes.POINTER(Geom), _f32p, _f32p, _f64p, vp]
        L.oracle_maxpool_fwd.argtypes = [_f32p, _f64p, _u8p] + [ctypes.c_int] * 7
        L.oracle_maxpool_bwd.argtypes = [_f32p, _u8p, _f64p] + [ctypes.c_int] * 7
        L.oracle_avgpool_fwd.argtypes = [_f32p, _f64p] + [ctypes.c_int] * 3
        L.oracle_avgpool_bwd.argtypes = [_f32p, _f64p] + [ctypes.c_int] * 3
        L.oracle_avgpool2d_fwd.argtypes = [_f32p, _f64p] + [ctypes.c_int] * 7
        L.oracle_avgpool2d_bwd.argtypes = [_f32p, _f64p] + [ctypes.c_int] * 7
        L.oracle_softmax_xent.argtypes = [_f32p, _i32p, _f64p, ctypes.c_int, ctypes.c_int]
        L.oracle_softmax_xent.restype = ctypes.c_double
        L.oracle_sgd.argtypes = [_f32p, _f32p, _f32p, ctypes.c_size_t] + [ctypes.c_float] * 4
        L.oracle_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]

    def threads(self):
        return self.lib.oracle_threads()

    def uniform(self, n, seed, tag, lo=-1.0, hi=1.0):
        out = np.empty(n, np.float32)
        self.lib.oracle_fill_uniform(out, n, seed, tag, lo, hi)
        return out

    def labels(self, n, classes, seed):
        out = np.empty(n, np.int32)
        self.lib.oracle_fill_labels(out, n, classes, seed)
        return out

    def round_bf16(self, a):
        a = np.ascontiguousarray(a, np.float32).copy()
        self.lib.oracle_round_bf16(a.reshape(-1), a.size)
        return a

    def conv_fwd(self, g, x, w, bias=None, residual=None, relu=False):
        ho, wo = out_hw(g)
        y = np.empty(g["n"] * ho * wo * g["k"], np.float64)
        keep = [np.ascontiguousarray(v, np.float32) for v in (bias, residual) if v is not None]
        self.lib.oracle_conv_fwd(ctypes.byref(Geom(**g)), np.ascontiguousarray(x, np.float32).ravel(),
                                 np.ascontiguousarray(w, np.float32).ravel(),
                                 _opt(bias), _opt(residual), int(relu), y)
        del keep
        return y

    def conv_dgrad(self, g, dy, w, residual=None, mask=None):
        dx = np.empty(g["n"] * g["h"] * g["w"] * g["c"], np.float64)
        res = None if residual is None else np.ascontiguousarray(residual, np.float32)
        msk = None if mask is None else np.ascontiguousarray(mask, np.float32)
        self.lib.oracle_conv_dgrad(ctypes.byref(Geom(**g)), np.ascontiguousarray(dy, np.float32).ravel(),
                                   np.ascontiguousarray(w, np.float32).ravel(),
                                   None if res is None else res.ctypes.data_as(ctypes.c_void_p),
                                   None if msk is None else msk.ctypes.data_as(ctypes.c_void_p), dx)
        return dx

    def conv_wgrad(self, g, dy, x, want_db=False):
        dw = np.empty(g["k"] * g["r"] * g["s"] * g["c"], np.float64)
        db = np.empty(g["k"], np.float64) if want_db else None
        self.lib.oracle_conv_wgrad(ctypes.byref(Geom(**g)), np.ascontiguousarray(dy, np.float32).ravel(),
                                   np.ascontiguousarray(x, np.float32).ravel(), dw,
                                   None if db is None else db.ctypes.data_as(ctypes.c_void_p))
        return (dw, db) if want_db else dw

    def maxpool_fwd(self, x, n, h, w, c, f, s, p):
        ho, wo = (h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1
        y = np.empty(n * ho * wo * c, np.float64)
        arg = np.empty(n * ho * wo * c, np.uint8)
        self.lib.oracle_maxpool_fwd(np.ascontiguousarray(x, np.float32).ravel(), y, arg, n, h, w, c, f, s, p)
        return y, arg

    def maxpool_bwd(self, dy, arg, n, h, w, c, f, s, p):
        dx = np.empty(n * h * w * c, np.float64)
        self.lib.oracle_maxpool_bwd(np.ascontiguousarray(dy, np.float32).ravel(),
                                    np.ascontiguousarray(arg, np.uint8).ravel(), dx, n, h, w, c, f, s, p)
        return dx

    def avgpool_fwd(self, x, n, hw, c):
        y = np.empty(n * c, np.float64)
        self.lib.oracle_avgpool_fwd(np.ascontiguousarray(x, np.float32).ravel(), y, n, hw, c)
        return y

    def avgpool_bwd(self, dy, n, hw, c):
        dx = np.empty(n * hw * c, np.float64)
        self.lib.oracle_avgpool_bwd(np.ascontiguousarray(dy, np.float32).ravel(), dx, n, hw, c)
        return dx

    def avgpool2d_fwd(self, x, n, h, w, c, f, s, p):
        ho, wo = (h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1
        y = np.empty(n * ho * wo * c, np.float64)
        self.lib.oracle_avgpool2d_fwd(np.ascontiguousarray(x, np.float32).ravel(), y, n, h, w, c, f, s, p)
        return y

    def avgpool2d_bwd(self, dy, n, h, w, c, f, s, p):
        dx = np.empty(n * h * w * c, np.float64)
        self.lib.oracle_avgpool2d_bwd(np.ascontiguousarray(dy, np.float32).ravel(), dx, n, h, w, c, f, s, p)
        return dx

    def softmax_xent(self, z, labels, n, classes):
        dl = np.empty(n * classes, np.float64)
        loss = self.lib.oracle_softmax_xent(np.ascontiguousarray(z, np.float32).ravel(),
                                            np.ascontiguousarray(labels, np.int32), dl, n, classes)
        return loss, dl

    def sgd(self, w, g, v, lr, mom, wd, gscale):
        w = np.ascontiguousarray(w, np.float32).copy()
        v = np.ascontiguousarray(v, np.float32).copy()
        self.lib.oracle_sgd(w, np.ascontiguousarray(g, np.float32), v, w.size, lr, mom, wd, gscale)
        return w, v


def rel_err(got, ref):
    """Normwise relative error ||got-ref|| / ||ref|| (float64)."""
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0))


def elem_err(got, ref, floor_frac=1e-3):
    """Max elementwise relative error with the denominator floored at
    floor_frac * max|ref| (near-zero elements would otherwise dominate)."""
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    floor = floor_frac * max(np.abs(ref).max(initial=0.0), 1e-30)
    return float((np.abs(got - ref) / np.maximum(np.abs(ref), floor)).max(initial=0.0))
