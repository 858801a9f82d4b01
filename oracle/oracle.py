"""ctypes binding of liboracle.so (TEST INFRASTRUCTURE; see gdraa_oracle.h).

Argument marshalling only: all arithmetic is in gdraa_oracle.c.  Arrays are numpy:
fp32 buffers as float32, bf16 buffers as their raw uint16 bit patterns.
"""
import ctypes
import os

import numpy as np

from . import build as _build

F32 = 0
BF16 = 1

_lib = None


def lib_path() -> str:
    return _build.LIB


def _load():
    global _lib
    if _lib is None:
        # GDRAA_ORACLE_LIB: a separately built copy (tools/oracle_mutations.py loads
        # deliberately broken builds through it to check that the pins catch them)
        path = os.environ.get("GDRAA_ORACLE_LIB") or _build.build()
        lib = ctypes.CDLL(path)
        u64, i32, f32 = ctypes.c_uint64, ctypes.c_int, ctypes.c_float
        pu64 = ctypes.POINTER(u64)
        vp, pvp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)
        lib.oracle_partition.argtypes = [u64, i32, u64, i32, pu64, pu64]
        lib.oracle_partition.restype = i32
        lib.oracle_bf16_to_f32.argtypes = [ctypes.c_uint16]
        lib.oracle_bf16_to_f32.restype = f32
        lib.oracle_f32_to_bf16_rne.argtypes = [f32]
        lib.oracle_f32_to_bf16_rne.restype = ctypes.c_uint16
        lib.oracle_allreduce_mean.argtypes = [i32, u64, i32, pvp, vp]
        lib.oracle_allreduce_mean.restype = i32
        lib.oracle_sgd_step.argtypes = [i32, u64, i32, pvp, vp, vp, f32, f32]
        lib.oracle_sgd_step.restype = i32
        lib.oracle_counters.argtypes = [u64, i32, u64, i32, i32, i32, vp]
        lib.oracle_counters.restype = i32
        lib.oracle_sgd_step_wd.argtypes = [i32, u64, i32, pvp, vp, vp, f32, f32, f32, vp, i32]
        lib.oracle_sgd_step_wd.restype = i32
        lib.oracle_poly_lr.argtypes = [f32, u64, u64, f32]
        lib.oracle_poly_lr.restype = f32
        _lib = lib
    return _lib


class _Counters(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in
                ("rs_sent", "rs_recv", "ag_sent", "ag_recv", "adds", "divides", "sync_waits")]


def partition(L: int, N: int, r: int, Q: int = 64):
    """(off_r, len_r) of Algorithm 1's block split, Q-aligned ceil rule (AMB-8)."""
    off, ln = ctypes.c_uint64(), ctypes.c_uint64()
    rc = _load().oracle_partition(L, N, Q, r, ctypes.byref(off), ctypes.byref(ln))
    if rc != 0:
        raise ValueError(f"oracle_partition(L={L}, N={N}, Q={Q}, r={r}) invalid")
    return off.value, ln.value


def bf16_to_f32(b: int) -> float:
    return float(_load().oracle_bf16_to_f32(int(b)))


def f32_to_bf16_rne(f: float) -> int:
    return int(_load().oracle_f32_to_bf16_rne(float(np.float32(f))))


def _dtype_of(arrs):
    dt = arrs[0].dtype
    for a in arrs:
        if a.dtype != dt or a.ndim != 1 or a.shape != arrs[0].shape:
            raise ValueError("all rank buffers must be 1-D with the same dtype and length")
    if dt == np.float32:
        return F32
    if dt == np.uint16:
        return BF16
    raise ValueError(f"unsupported dtype {dt} (float32, or uint16 bf16 bit patterns)")


def _ptrs(arrs):
    arrs = [np.ascontiguousarray(a) for a in arrs]
    return arrs, (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def allreduce_mean(bufs):
    """Rank-ordered mean of the N rank buffers, the value every rank holds after
    the broadcast.  bufs: list of N 1-D float32 (or uint16 bf16 bit) arrays."""
    dtype = _dtype_of(bufs)
    bufs, ptrs = _ptrs(bufs)
    out = np.empty_like(bufs[0])
    rc = _load().oracle_allreduce_mean(len(bufs), bufs[0].shape[0], dtype, ptrs, out.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_allreduce_mean: invalid arguments")
    return out


def sgd_step(grads, w, v, lr: float, mom: float):
    """One synchronous momentum-SGD step with the averaged gradient.
    Returns new (w, v) arrays; inputs are not modified."""
    dtype = _dtype_of(grads)
    grads, ptrs = _ptrs(grads)
    w = np.array(w, dtype=np.float32, copy=True)
    v = np.array(v, dtype=np.float32, copy=True)
    if w.shape != grads[0].shape or v.shape != grads[0].shape:
        raise ValueError("w, v must match the gradient length")
    rc = _load().oracle_sgd_step(len(grads), grads[0].shape[0], dtype, ptrs, w.ctypes.data,
                                 v.ctypes.data, float(lr), float(mom))
    if rc != 0:
        raise ValueError("oracle_sgd_step: invalid arguments")
    return w, v


def sgd_step_wd(grads, w, v, lr: float, mom: float, wd: float, model_dtype=None):
    """Momentum SGD with weight decay.  Returns (w, v) or, with
    model_dtype in {F32, BF16}, (w, v, model) where model is the broadcast copy."""
    dtype = _dtype_of(grads)
    grads, ptrs = _ptrs(grads)
    w = np.array(w, dtype=np.float32, copy=True)
    v = np.array(v, dtype=np.float32, copy=True)
    if w.shape != grads[0].shape or v.shape != grads[0].shape:
        raise ValueError("w, v must match the gradient length")
    model = None
    if model_dtype is not None:
        model = np.empty(w.shape, np.float32 if model_dtype == F32 else np.uint16)
    rc = _load().oracle_sgd_step_wd(len(grads), grads[0].shape[0], dtype, ptrs, w.ctypes.data,
                                    v.ctypes.data, float(lr), float(mom), float(wd),
                                    None if model is None else model.ctypes.data,
                                    F32 if model_dtype is None else model_dtype)
    if rc != 0:
        raise ValueError("oracle_sgd_step_wd: invalid arguments")
    return (w, v) if model is None else (w, v, model)


def poly_lr(lr0: float, it: int, max_iter: int, power: float) -> float:
    """lr0 * (1 - it/max_iter)^power ("poly")."""
    return float(_load().oracle_poly_lr(lr0, it, max_iter, power))


def counters(L: int, N: int, r: int, s_g: int, s_w: int, Q: int = 64) -> dict:
    """Lemma 1 / Lemma 2 accounting for rank r (Eq. 1-4)."""
    c = _Counters()
    rc = _load().oracle_counters(L, N, Q, r, s_g, s_w, ctypes.byref(c))
    if rc != 0:
        raise ValueError("oracle_counters: invalid arguments")
    return {name: getattr(c, name) for name, _ in c._fields_}

