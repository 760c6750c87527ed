"""Python handle over the C++ training-step executor (libtcb.so tcb_trainer_*).

One Trainer per GPU process. For world > 1 the NCCL unique id is created on
rank 0 and broadcast with torch.distributed (plumbing only); the gradient
aggregation / parameter refresh itself runs inside the C++ step — over NCCL
(reduce-scatter, SGD, all-gather), or with cfg["ps_transport"] = "nvls" as
one fused kernel over NVSwitch multicast on buffers allocated here with torch
symmetric memory (allocation / handle exchange only).
"""
from __future__ import annotations

import ctypes
import json

import torch

from . import device, models

_vp = ctypes.c_void_p
_bound = False


def _lib():
    global _bound
    L = device.lib()
    if not _bound:
        L.tcb_trainer_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(_vp)]
        L.tcb_trainer_destroy.argtypes = [_vp]
        L.tcb_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.tcb_trainer_join.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
        L.tcb_trainer_set_batch.argtypes = [_vp, _vp, _vp, _vp]
        L.tcb_trainer_stage_batch.argtypes = [_vp, _vp, ctypes.c_int, _vp]
        L.tcb_trainer_step.argtypes = [_vp, _vp]
        L.tcb_trainer_loss.argtypes = [_vp, ctypes.POINTER(ctypes.c_float), _vp]
        L.tcb_trainer_phase_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_float)]
        L.tcb_trainer_enable_timing.argtypes = [_vp, ctypes.c_int]
        L.tcb_trainer_describe.argtypes = [_vp, ctypes.POINTER(ctypes.c_char_p)]
        L.tcb_trainer_tensor.argtypes = [_vp, ctypes.c_char_p, ctypes.POINTER(_vp),
                                         ctypes.POINTER(ctypes.c_size_t)]
        L.tcb_trainer_launch_count.argtypes = [_vp, ctypes.POINTER(ctypes.c_int)]
        L.tcb_trainer_enable_layer_timing.argtypes = [_vp, ctypes.c_int]
        L.tcb_trainer_layer_times.argtypes = [_vp, ctypes.POINTER(ctypes.c_char_p)]
        L.tcb_trainer_attach_nvls.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t]
        L.tcb_trainer_health.argtypes = [_vp, _vp]
        L.tcb_trainer_attach_nvls_async.argtypes = [_vp, _vp, _vp]
        L.tcb_trainer_finish.argtypes = [_vp, _vp]
        L.tcb_free.argtypes = [_vp]
        _bound = True
    return L


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    device.check(_lib().tcb_nccl_unique_id(buf))
    return buf.raw


class _DevBuf:
    """Exposes a device pointer to torch via __cuda_array_interface__."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


def small_config(precision="bf16"):
    return models.tiny_resnet(precision=precision)


class Trainer:
    PHASES = ("fwd", "bwd", "reduce_scatter", "sgd", "all_gather")

    def __init__(self, cfg: dict, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self.cfg = cfg
        self.handle = _vp()
        device.check(_lib().tcb_trainer_create(json.dumps(cfg).encode(), ctypes.byref(self.handle)))
        self.rank, self.world = rank, world
        if world > 1 or nccl_id is not None:
            device.check(_lib().tcb_trainer_join(self.handle, rank, world, nccl_id))
        self._symm = None
        if world > 1 and cfg.get("ps_transport", "nccl") == "nvls":
            self.attach_nvls()

    def attach_nvls(self, group=None):
        """Place the flat gradient / bf16 weight buffers in symmetric memory
        bound to NVSwitch multicast objects and switch the PS step to the fused
        multimem kernel (tcb_trainer_attach_nvls). Needs torch.distributed."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        group = group or dist.group.WORLD
        n = self.describe()["param_padded"]
        bufs, handles, mcs = [], [], []
        dts = (torch.float32, torch.bfloat16) + ((torch.bfloat16,) if self.cfg.get("ps_async") else ())
        for dt in dts:
            t = symm.empty(n, dtype=dt, device="cuda")
            h = symm.rendezvous(t, group.group_name)
            if not h.multicast_ptr:
                raise RuntimeError("NVLS multicast is not available on this system")
            delta = t.data_ptr() - h.buffer_ptrs[h.rank]
            if delta < 0:
                raise RuntimeError("unexpected symmetric-memory layout")
            bufs.append(t)
            handles.append(h)
            mcs.append(h.multicast_ptr + delta)
        device.check(_lib().tcb_trainer_attach_nvls(self.handle, _vp(bufs[0].data_ptr()), _vp(mcs[0]),
                                                    _vp(bufs[1].data_ptr()), _vp(mcs[1]),
                                                    _vp(handles[0].signal_pad_ptrs_dev),
                                                    int(handles[0].signal_pad_size)))
        if len(bufs) > 2:  # asynchronous PS: the second weight buffer
            device.check(_lib().tcb_trainer_attach_nvls_async(self.handle, _vp(bufs[2].data_ptr()), _vp(mcs[2])))
        self._symm = (bufs, handles)  # keep the allocations alive

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib().tcb_trainer_destroy(self.handle)
                self.handle = None
        except Exception:  # interpreter teardown
            pass

    @staticmethod
    def _stream():
        return _vp(torch.cuda.current_stream().cuda_stream)

    def set_batch(self, images=None, labels=None):
        """Host (CPU, ideally pinned) fp32 NHWC images / int32 labels -> device."""
        device.check(_lib().tcb_trainer_set_batch(
            self.handle, None if images is None else _vp(images.data_ptr()),
            None if labels is None else _vp(labels.data_ptr()), self._stream()))

    def stage_batch(self, images, labels):
        """Pipelined input: queue a pinned host batch (NHWC uint8 pixels or fp32)
        for the next step; the H2D copy runs on the trainer's copy stream,
        overlapping the current step."""
        fmt = {torch.uint8: 1, torch.float32: 0}[images.dtype]
        device.check(_lib().tcb_trainer_stage_batch(self.handle, _vp(images.data_ptr()), fmt,
                                                    _vp(labels.data_ptr())))

    def step(self):
        device.check(_lib().tcb_trainer_step(self.handle, self._stream()))

    def finish(self):
        """Join the in-flight parameter updates (asynchronous PS) into the stream."""
        device.check(_lib().tcb_trainer_finish(self.handle, self._stream()))

    def loss(self) -> float:
        out = ctypes.c_float()
        device.check(_lib().tcb_trainer_loss(self.handle, ctypes.byref(out), self._stream()))
        return out.value

    def data_times(self) -> dict:
        """Paper steps 3-4 of the last staged batch consumed with timing on."""
        ms = (ctypes.c_float * 2)()
        device.check(_lib().tcb_trainer_data_times(self.handle, ms))
        return {"host_to_gpu_transfer": ms[0], "data_preparation": ms[1]}

    def health(self):
        """Failure detection: raises on an NCCL asynchronous error or an NVLS
        barrier timeout (a peer rank stalled or died); synchronises the stream."""
        device.check(_lib().tcb_trainer_health(self.handle, self._stream()))

    def enable_timing(self, on=True):
        device.check(_lib().tcb_trainer_enable_timing(self.handle, int(on)))

    def phase_times(self) -> dict:
        buf = (ctypes.c_float * 5)()
        device.check(_lib().tcb_trainer_phase_times(self.handle, buf))
        return dict(zip(self.PHASES, list(buf)))

    def enable_layer_timing(self, on=True):
        device.check(_lib().tcb_trainer_enable_layer_timing(self.handle, int(on)))

    def layer_times(self) -> list:
        """Per-conv [fwd, dgrad, wgrad] ms measured inside the last step."""
        out = ctypes.c_char_p()
        device.check(_lib().tcb_trainer_layer_times(self.handle, ctypes.byref(out)))
        d = json.loads(out.value.decode())
        _lib().tcb_free(ctypes.cast(out, _vp))
        return d

    def launch_count(self) -> int:
        n = ctypes.c_int()
        device.check(_lib().tcb_trainer_launch_count(self.handle, ctypes.byref(n)))
        return n.value

    def describe(self) -> dict:
        out = ctypes.c_char_p()
        device.check(_lib().tcb_trainer_describe(self.handle, ctypes.byref(out)))
        d = json.loads(out.value.decode())
        _lib().tcb_free(ctypes.cast(out, _vp))
        return d

    def tensor(self, name: str, dtype=None) -> torch.Tensor:
        ptr, nbytes = _vp(), ctypes.c_size_t()
        device.check(_lib().tcb_trainer_tensor(self.handle, name.encode(), ctypes.byref(ptr),
                                               ctypes.byref(nbytes)))
        if dtype is None:
            if name in ("param", "grad", "momentum", "loss", "input_f32"):
                dtype = torch.float32
            elif name == "labels":
                dtype = torch.int32
            else:
                dtype = torch.bfloat16 if self.cfg.get("precision", "bf16") == "bf16" else torch.float32
        esz = torch.tensor([], dtype=dtype).element_size()
        typestr = {torch.float32: "<f4", torch.int32: "<i4", torch.bfloat16: "<f2",
                   torch.uint8: "|u1"}[dtype]
        count = nbytes.value // esz
        if dtype == torch.bfloat16:  # no bf16 typestr in the interface: view int16 bits
            t = torch.as_tensor(_DevBuf(ptr.value, count, "<i2"), device="cuda")
            return t.view(torch.bfloat16)
        return torch.as_tensor(_DevBuf(ptr.value, count, typestr), device="cuda")
