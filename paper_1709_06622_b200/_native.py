"""Locate and load the in-tree native libraries.

The product path has no fallback: if a library is missing the loader raises,
it never substitutes Python or oracle code.
"""
from __future__ import annotations

import ctypes
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# $TCB_LIB_DIR: an alternative in-tree build directory (A/B measurements)
LIB_DIR = os.environ.get("TCB_LIB_DIR") or os.path.join(PKG_DIR, "lib")

_cache: dict[str, ctypes.CDLL] = {}


class NativeLibraryMissing(RuntimeError):
    """The compiled library is absent: run __graft_entry__.build() (make -C csrc)."""


def load(name: str) -> ctypes.CDLL:
    if name in _cache:
        return _cache[name]
    path = os.path.join(LIB_DIR, name)
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
    _cache[name] = lib
    return lib
