"""Python binding of the traincap C++ planner (libtraincap.so, C-ABI
`tcb_planner_call`, declared in include/tcb_planner.h).

`Planner.call(op, **args)` sends one JSON request through the C-ABI and maps
error replies back onto exception classes named after the reference's
(`/root/reference/proj/include/traincap/errors.hpp:10-89`).
"""
from __future__ import annotations

import ctypes
import json
from typing import Any

from . import _native


class Error(RuntimeError):
    """Base of all planner errors (traincap::Error)."""

    type_name = "Error"

    def __init__(self, message: str, line: int | None = None, layer_id: int | None = None):
        super().__init__(message)
        self.line = line
        self.layer_id = layer_id


_ERROR_TYPES: dict[str, type] = {"Error": Error}
for _n in ("ParseError", "DuplicateKeyError", "IncompleteCatalogError", "OverflowError",
           "NonPositiveShapeError", "DomainError", "UnitError", "MissingComputeStepError",
           "InstanceTooLargeError", "CandidateNotInCatalogError", "ValidationError",
           "BadRequest"):
    _ERROR_TYPES[_n] = type(_n, (Error,), {"type_name": _n})
globals().update({k: v for k, v in _ERROR_TYPES.items()})


def raise_for(reply: dict[str, Any]) -> dict[str, Any]:
    err = reply.get("error")
    if err is None:
        return reply
    cls = _ERROR_TYPES.get(err["type"], Error)
    raise cls(err["message"], line=err.get("line"), layer_id=err.get("layer_id"))


class Planner:
    """Thin handle over one planner C-ABI (`<prefix>planner_call`)."""

    def __init__(self, lib: ctypes.CDLL | None = None, prefix: str = "tcb_"):
        self.lib = lib if lib is not None else _native.load("libtraincap.so")
        self._call = getattr(self.lib, prefix + "planner_call")
        self._call.restype = ctypes.c_void_p
        self._call.argtypes = [ctypes.c_char_p]
        self._free = getattr(self.lib, prefix + "planner_free")
        self._free.argtypes = [ctypes.c_void_p]
        self._free.restype = None

    def raw(self, op: str, **args: Any) -> dict[str, Any]:
        """Reply dict including an "error" member instead of raising."""
        req = dict(args)
        req["op"] = op
        ptr = self._call(json.dumps(req).encode())
        try:
            text = ctypes.string_at(ptr).decode()
        finally:
            self._free(ptr)
        return json.loads(text)

    def call(self, op: str, **args: Any) -> dict[str, Any]:
        return raise_for(self.raw(op, **args))


_default: Planner | None = None


def default() -> Planner:
    global _default
    if _default is None:
        _default = Planner()
    return _default
