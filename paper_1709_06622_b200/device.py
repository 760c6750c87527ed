"""ctypes binding of libtcb.so (include/tcb.h) for single-op use.

Device memory and streams come from torch (plumbing only): tensors are passed
by data_ptr() and the current torch stream is handed to the C-ABI, so CUDA
events recorded on torch's current stream time exactly the kernels launched.
There is no fallback: if libtcb.so is missing, import fails loudly.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native

ALGO = {"gemm": 0, "winograd": 1, "fft": 2}
PREC = {"ffma": 0, "tf32": 1, "bf16": 2}
DT = {torch.float32: 0, torch.bfloat16: 1}

TCB_OK, TCB_ERR_UNSUPPORTED = 0, -2


class TcbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"tcb error {code}: {msg}")
        self.code = code


class Unsupported(TcbError):
    pass


class ConvGeom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("n", "h", "w", "c", "k", "r", "s", "pad_h", "pad_w", "stride_h", "stride_w")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}

    @property
    def ho(self):
        return (self.h + 2 * self.pad_h - self.r) // self.stride_h + 1

    @property
    def wo(self):
        return (self.w + 2 * self.pad_w - self.s) // self.stride_w + 1


def geom(n, h, w, c, k, r, s=None, pad=0, stride=1, pad_w=None, stride_w=None) -> ConvGeom:
    s = r if s is None else s
    return ConvGeom(n, h, w, c, k, r, s, pad, pad if pad_w is None else pad_w, stride,
                    stride if stride_w is None else stride_w)


_vp = ctypes.c_void_p
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    L = _native.load("libtcb.so")
    L.tcb_last_error.restype = ctypes.c_char_p
    L.tcb_conv_plan_create.argtypes = [ctypes.POINTER(ConvGeom), ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_size_t)]
    L.tcb_conv_plan_destroy.argtypes = [_vp]
    L.tcb_conv_plan_set_valid_channels.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
    L.tcb_set_conv_stem.argtypes = [ctypes.c_int]
    L.tcb_conv_fwd.argtypes = [_vp, _vp, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _vp]
    L.tcb_conv_dgrad.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.tcb_conv_wgrad.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.tcb_maxpool_fwd.argtypes = [ctypes.c_int, _vp, _vp, _vp] + [ctypes.c_int] * 7 + [_vp]
    L.tcb_avgpool2d_fwd.argtypes = [ctypes.c_int, _vp, _vp] + [ctypes.c_int] * 7 + [_vp]
    L.tcb_avgpool2d_bwd.argtypes = [ctypes.c_int, _vp, _vp, _vp] + [ctypes.c_int] * 7 + [_vp]
    L.tcb_slice_copy.argtypes = [ctypes.c_int, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t, ctypes.c_int,
                                 ctypes.c_size_t, _vp]
    L.tcb_maxpool_bwd.argtypes = [ctypes.c_int, _vp, _vp, _vp] + [ctypes.c_int] * 7 + [_vp]
    L.tcb_avgpool_global_fwd.argtypes = [ctypes.c_int, _vp, _vp] + [ctypes.c_int] * 3 + [_vp]
    L.tcb_avgpool_global_bwd.argtypes = [ctypes.c_int, _vp, _vp] + [ctypes.c_int] * 3 + [_vp]
    L.tcb_softmax_xent.argtypes = [ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp]
    L.tcb_fill_uniform.argtypes = [ctypes.c_int, _vp, ctypes.c_size_t, ctypes.c_uint64,
                                   ctypes.c_uint64, ctypes.c_float, ctypes.c_float, _vp]
    L.tcb_fill_labels.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _vp]
    L.tcb_cast.argtypes = [ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
    L.tcb_sgd_momentum.argtypes = [_vp, _vp, _vp, ctypes.c_int, _vp, ctypes.c_size_t,
                                   ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                   ctypes.c_float, _vp]
    L.tcb_conv_out_hw.argtypes = [ctypes.POINTER(ConvGeom), ctypes.POINTER(ctypes.c_int),
                                  ctypes.POINTER(ctypes.c_int)]
    _lib = L
    return L


def check(code: int):
    if code != TCB_OK:
        msg = lib().tcb_last_error().decode()
        raise (Unsupported if code == TCB_ERR_UNSUPPORTED else TcbError)(code, msg)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class ConvPlan:
    """One (geometry, algorithm, precision) plan with its workspace."""

    g: ConvGeom
    algo: str
    prec: str

    def __post_init__(self):
        h = _vp()
        ws = ctypes.c_size_t()
        check(lib().tcb_conv_plan_create(ctypes.byref(self.g), ALGO[self.algo], PREC[self.prec],
                                         ctypes.byref(h), ctypes.byref(ws)))
        self.handle = h
        self.workspace_bytes = ws.value
        # zero-filled once: split-K counters inside must start at 0 (they self-reset)
        self.workspace = torch.zeros(max(ws.value, 1), dtype=torch.uint8, device="cuda")

    def set_valid_channels(self, c_valid):
        """Only the first c_valid input channels can be non-zero (narrow first
        layers): enables the explicit-im2col / row-window stem paths."""
        ws = ctypes.c_size_t()
        check(lib().tcb_conv_plan_set_valid_channels(self.handle, int(c_valid), ctypes.byref(ws)))
        self.workspace_bytes = ws.value
        self.workspace = torch.zeros(max(ws.value, 1), dtype=torch.uint8, device="cuda")
        return self

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().tcb_conv_plan_destroy(self.handle)
                self.handle = None
        except Exception:  # interpreter teardown
            pass

    @property
    def dtype(self):
        return torch.bfloat16 if self.prec == "bf16" else torch.float32

    def fwd(self, x, w, bias=None, residual=None, relu=False, out=None):
        g = self.g
        y = out if out is not None else torch.empty(g.n, g.ho, g.wo, g.k, dtype=self.dtype, device="cuda")
        check(lib().tcb_conv_fwd(self.handle, _p(x), _p(w), _p(bias), _p(residual), int(relu),
                                 _p(y), _p(self.workspace), _stream()))
        return y

    def dgrad(self, dy, w, residual=None, mask=None, out=None):
        g = self.g
        dx = out if out is not None else torch.empty(g.n, g.h, g.w, g.c, dtype=self.dtype, device="cuda")
        check(lib().tcb_conv_dgrad(self.handle, _p(dy), _p(w), _p(residual), _p(mask), _p(dx),
                                   _p(self.workspace), _stream()))
        return dx

    def wgrad(self, dy, x, want_db=False, out=None):
        g = self.g
        dw = out if out is not None else torch.empty(g.k, g.r, g.s, g.c, dtype=torch.float32, device="cuda")
        db = torch.empty(g.k, dtype=torch.float32, device="cuda") if want_db else None
        check(lib().tcb_conv_wgrad(self.handle, _p(dy), _p(x), _p(dw), _p(db),
                                   _p(self.workspace), _stream()))
        return (dw, db) if want_db else dw


def fill_uniform(t: torch.Tensor, seed: int, tag: int, lo=-1.0, hi=1.0):
    check(lib().tcb_fill_uniform(DT[t.dtype], _p(t), t.numel(), seed, tag, lo, hi, _stream()))
    return t


def fill_labels(t: torch.Tensor, classes: int, seed: int):
    check(lib().tcb_fill_labels(_p(t), t.numel(), classes, seed, _stream()))
    return t


def maxpool_fwd(x, f, s, p):
    n, h, w, c = x.shape
    ho, wo = (h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1
    y = torch.empty(n, ho, wo, c, dtype=x.dtype, device="cuda")
    arg = torch.empty(n, ho, wo, c, dtype=torch.uint8, device="cuda")
    check(lib().tcb_maxpool_fwd(DT[x.dtype], _p(x), _p(y), _p(arg), n, h, w, c, f, s, p, _stream()))
    return y, arg


def maxpool_bwd(dy, arg, shape, f, s, p, relu_y=None):
    """relu_y: the pool output of a ReLU'd input — fuses the ReLU backward."""
    n, h, w, c = shape
    dx = torch.empty(n, h, w, c, dtype=dy.dtype, device="cuda")
    if relu_y is not None:
        check(lib().tcb_maxpool_relu_bwd(DT[dy.dtype], _p(dy), _p(arg), _p(relu_y), _p(dx), n, h, w,
                                         c, f, s, p, _stream()))
    else:
        check(lib().tcb_maxpool_bwd(DT[dy.dtype], _p(dy), _p(arg), _p(dx), n, h, w, c, f, s, p,
                                    _stream()))
    return dx


def avgpool2d_fwd(x, f, s, p):
    n, h, w, c = x.shape
    ho, wo = (h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1
    y = torch.empty(n, ho, wo, c, dtype=x.dtype, device="cuda")
    check(lib().tcb_avgpool2d_fwd(DT[x.dtype], _p(x), _p(y), n, h, w, c, f, s, p, _stream()))
    return y


def avgpool2d_bwd(dy, shape, f, s, p, mask=None):
    n, h, w, c = shape
    dx = torch.empty(n, h, w, c, dtype=dy.dtype, device="cuda")
    check(lib().tcb_avgpool2d_bwd(DT[dy.dtype], _p(dy), _p(mask), _p(dx), n, h, w, c, f, s, p, _stream()))
    return dx


def concat(xs):
    """Channel concat of NHWC tensors via tcb_slice_copy (what the executor runs)."""
    n, h, w = xs[0].shape[:3]
    C = sum(x.shape[3] for x in xs)
    y = torch.empty(n, h, w, C, dtype=xs[0].dtype, device="cuda")
    off = 0
    for x in xs:
        c = x.shape[3]
        check(lib().tcb_slice_copy(DT[x.dtype], _p(x), c, ctypes.c_void_p(y.data_ptr() + off * y.element_size()),
                                   C, c, n * h * w, _stream()))
        off += c
    return y


def avgpool_fwd(x):
    n, h, w, c = x.shape
    y = torch.empty(n, c, dtype=x.dtype, device="cuda")
    check(lib().tcb_avgpool_global_fwd(DT[x.dtype], _p(x), _p(y), n, h * w, c, _stream()))
    return y


def avgpool_bwd(dy, h, w):
    n, c = dy.shape
    dx = torch.empty(n, h, w, c, dtype=dy.dtype, device="cuda")
    check(lib().tcb_avgpool_global_bwd(DT[dy.dtype], _p(dy), _p(dx), n, h * w, c, _stream()))
    return dx


def softmax_xent(logits, labels):
    n, k = logits.shape
    dl = torch.empty_like(logits)
    loss = torch.empty(n + 1, dtype=torch.float32, device="cuda")
    check(lib().tcb_softmax_xent(DT[logits.dtype], _p(logits), _p(labels), _p(dl), _p(loss), n, k,
                                 _stream()))
    return loss[0], dl


def sgd_momentum(w, g, v, lr, mom, wd=0.0, gscale=1.0, w_compute=None):
    cdt = DT[w_compute.dtype] if w_compute is not None else 0
    check(lib().tcb_sgd_momentum(_p(w), _p(g), _p(v), cdt, _p(w_compute), w.numel(), lr, mom, wd,
                                 gscale, _stream()))


LAUNCH_FIELDS = ("mode", "load", "bn", "epi", "cta2", "splits", "units", "grid", "fused_reduce", "b_resident")


def last_launch() -> dict:
    """Configuration of the last bf16 tensor-core conv kernel launch (test hook,
    tcb_conv_last_launch_info)."""
    out = (ctypes.c_int * 10)()
    check(lib().tcb_conv_last_launch_info(out))
    return dict(zip(LAUNCH_FIELDS, list(out)))
