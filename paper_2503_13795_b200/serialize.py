"""Bit-exact save / load of value and gradient ranges (reference module
`serialize`), over the C-ABI (tg_save_range & co).

Ranges are numpy arrays or torch tensors (host or device: parameters and
grad_sum stay on the GPU).  Raw ranges are headerless little-endian IEEE-754
(7 fp64 values = 56 bytes); snapshots carry the 18-byte "BTSG" header.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib


def _info(a):
    """(pointer, count, tg_dtype) of a contiguous fp32 / fp64 array or tensor."""
    if a is None:
        return None, 0, None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("ranges must be contiguous")
        dt = {np.dtype(np.float64): _lib.TG_F64, np.dtype(np.float32): _lib.TG_F32}[a.dtype]
        return C.c_void_p(a.ctypes.data), a.size, dt
    import torch
    if not a.is_contiguous():
        raise ValueError("ranges must be contiguous")
    dt = {torch.float64: _lib.TG_F64, torch.float32: _lib.TG_F32}[a.dtype]
    return C.c_void_p(a.data_ptr()), a.numel(), dt


def _pair(values, grads):
    vp, n, dt = _info(values)
    gp, gn, gdt = _info(grads)
    if grads is not None and (gn != n or gdt != dt):
        raise ValueError("values and grads must have the same length and dtype")
    return vp, gp, n, dt


def save_range(values, grads=None) -> bytes:
    """Raw range bytes: values, then grads when given."""
    vp, gp, n, dt = _pair(values, grads)
    nbytes = lib.tg_range_bytes(dt, n, 1 if grads is not None else 0)
    buf = (C.c_char * max(nbytes, 1))()
    written = C.c_size_t()
    check(lib.tg_save_range(dt, vp, gp, n, buf, nbytes, C.byref(written)))
    return bytes(buf)[: written.value]


def load_range(data: bytes, values, grads=None) -> None:
    """Overwrites values (and grads) from raw range bytes; TG_FORMAT on a size mismatch."""
    vp, gp, n, dt = _pair(values, grads)
    check(lib.tg_load_range(dt, vp, gp, n, data, len(data)))


def save_snapshot(values, grads=None) -> bytes:
    vp, gp, n, dt = _pair(values, grads)
    nbytes = lib.tg_snapshot_bytes(dt, n, 1 if grads is not None else 0)
    buf = (C.c_char * nbytes)()
    written = C.c_size_t()
    check(lib.tg_save_snapshot(dt, vp, gp, n, buf, nbytes, C.byref(written)))
    return bytes(buf)[: written.value]


def load_snapshot(data: bytes, values, grads=None) -> dict:
    """Loads a BTSG snapshot into values (and grads); returns its header fields."""
    vp, gp, n, dt = _pair(values, grads)
    on, og = C.c_size_t(), C.c_int()
    check(lib.tg_load_snapshot(data, len(data), dt, vp, gp, n, C.byref(on), C.byref(og)))
    return {"dtype": "f64" if dt == _lib.TG_F64 else "f32", "count": on.value, "grads": bool(og.value)}
