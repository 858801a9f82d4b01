"""Thin ctypes binding of lib/libgdraa.so (include/gdraa.h).

Argument marshalling only: every step of the hot path runs in the library's sm_100a
kernels.  Functions keep the C names.  Tensors are torch CUDA tensors (or raw device
pointers as ints); streams are torch.cuda.Stream objects (default: the current stream).
There is no fallback: if the native library is missing this module raises on import.
"""
import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# GDRAA_LIB_PATH: load another build of the same library (A/B timing of two builds on one
# box only); the default is the in-tree build.
LIB_PATH = os.environ.get("GDRAA_LIB_PATH") or os.path.join(PKG, "lib", "libgdraa.so")

GDRAA_F32 = 0
GDRAA_BF16 = 1
GDRAA_SHARD_QUANTUM = 64
GDRAA_MAX_WORLD = 8

ERRORS = {0: "GDRAA_OK", -1: "GDRAA_EINVAL", -2: "GDRAA_ENOTREG", -3: "GDRAA_ESHAPE",
          -4: "GDRAA_ECUDA", -5: "GDRAA_ETIMEOUT", -6: "GDRAA_ESTATE", -7: "GDRAA_EJOBSERVER"}

EXPORTED = ["gdraa_sgd_step_ex", "gdraa_sgd_step_mp", "gdraa_poly_lr",
            "gdraa_small_message_bytes", "gdraa_small_step_bytes", "gdraa_allreduce_mean_range",
            "gdraa_sgd_step_range", "gdraa_sgd_step_mp_range",
            "gdraa_vr_sgd_step_ex", "gdraa_vr_sgd_step_mp",
            "gdraa_init", "gdraa_register", "gdraa_deregister","gdraa_allreduce_mean", "gdraa_sgd_step",
            "gdraa_shard", "gdraa_get_stats", "gdraa_finalize", "gdraa_last_error",
            "gdraa_version", "gdraa_vr_allreduce_mean", "gdraa_vr_sgd_step",
            "gdraa_vr_allreduce_mean_range", "gdraa_vr_sgd_step_range",
            "gdraa_vr_sgd_step_mp_range", "gdraa_bucket_set_begin", "gdraa_bucket_set_end",
            "gdraa_vr_bucket_set_begin", "gdraa_vr_bucket_set_end",
            "gdraa_bucket_set_begin_streamed", "gdraa_vr_bucket_set_begin_streamed"]


class GdraaError(RuntimeError):
    def __init__(self, code, fn, msg):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        super().__init__(f"{fn}: {self.name}: {msg}")


class gdraa_stats_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in
                ("calls", "sync_waits", "rs_bytes_in", "rs_bytes_out", "ag_bytes_out",
                 "ag_bytes_in", "adds", "divides", "launches", "ll_calls", "iter_done",
                 "iter_start")]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with "
                      "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)
_vp, _i, _sz, _f = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_float
_psz = ctypes.POINTER(ctypes.c_size_t)
_sig = {
    "gdraa_init": ([_i, _i], _i),
    "gdraa_register": ([_vp, _sz, _i], _i),
    "gdraa_deregister": ([_vp], _i),
    "gdraa_allreduce_mean": ([_vp, _vp], _i),
    "gdraa_sgd_step": ([_vp, _vp, _vp, _f, _f, _vp], _i),
    "gdraa_shard": ([_i, _i, _sz, _psz, _psz], _i),
    "gdraa_get_stats": ([ctypes.POINTER(gdraa_stats_t)], _i),
    "gdraa_finalize": ([], _i),
    "gdraa_last_error": ([], ctypes.c_char_p),
    "gdraa_version": ([], ctypes.c_char_p),
    "gdraa_vr_allreduce_mean": ([_i, ctypes.POINTER(_vp), _sz, _i, _vp], _i),
    "gdraa_vr_sgd_step": ([_i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                           _sz, _i, _f, _f, _vp], _i),
    "gdraa_sgd_step_ex": ([_vp, _vp, _vp, _f, _f, _f, _vp], _i),
    "gdraa_sgd_step_mp": ([_vp, _vp, _vp, _vp, _f, _f, _f, _vp], _i),
    "gdraa_poly_lr": ([_f, ctypes.c_uint64, ctypes.c_uint64, _f], _f),
    "gdraa_small_message_bytes": ([_i], _sz),
    "gdraa_small_step_bytes": ([_i, _i, _i], _sz),
    "gdraa_allreduce_mean_range": ([_vp, _sz, _sz, _vp], _i),
    "gdraa_sgd_step_range": ([_vp, _vp, _vp, _sz, _sz, _f, _f, _f, _vp], _i),
    "gdraa_sgd_step_mp_range": ([_vp, _vp, _vp, _vp, _sz, _sz, _f, _f, _f, _vp], _i),
    "gdraa_vr_sgd_step_ex": ([_i, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), _sz, _i, _f, _f, _f, _vp], _i),
    "gdraa_vr_sgd_step_mp": ([_i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), _sz, _i, _f, _f, _f, _vp], _i),
    "gdraa_vr_allreduce_mean_range": ([_i, ctypes.POINTER(_vp), _sz, _i, _sz, _sz, _vp], _i),
    "gdraa_vr_sgd_step_range": ([_i, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                 ctypes.POINTER(_vp), _sz, _i, _sz, _sz, _f, _f, _f, _vp], _i),
    "gdraa_vr_sgd_step_mp_range": ([_i, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                    ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _i, _sz, _sz,
                                    _f, _f, _f, _vp], _i),
    "gdraa_bucket_set_begin": ([], _i),
    "gdraa_bucket_set_end": ([_vp], _i),
    "gdraa_vr_bucket_set_begin": ([_i], _i),
    "gdraa_vr_bucket_set_end": ([_i, _vp], _i),
    "gdraa_bucket_set_begin_streamed": ([_i], _i),
    "gdraa_vr_bucket_set_begin_streamed": ([_i, _i], _i),
}
for _name, (_args, _res) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


def _check(rc, fn):
    if rc != 0:
        raise GdraaError(rc, fn, _lib.gdraa_last_error().decode(errors="replace"))


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    # the library sees only the pointer: a host or strided tensor would be read as if it
    # were a dense device buffer, so refuse it here
    if not x.is_cuda:
        raise ValueError("gdraa: tensor arguments must live on a CUDA device")
    if not x.is_contiguous():
        raise ValueError("gdraa: tensor arguments must be contiguous")
    return x.data_ptr()


def _stream(s):
    if s is None:
        import torch
        s = torch.cuda.current_stream()
    if isinstance(s, int):
        return s
    return s.cuda_stream


def dtype_code(t):
    import torch
    if t.dtype == torch.float32:
        return GDRAA_F32
    if t.dtype == torch.bfloat16:
        return GDRAA_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


def gdraa_version():
    return _lib.gdraa_version().decode()


def gdraa_last_error():
    return _lib.gdraa_last_error().decode(errors="replace")


def gdraa_init(world: int, rank: int):
    _check(_lib.gdraa_init(world, rank), "gdraa_init")


def gdraa_register(buf, n: int = None, dtype: int = None):
    """Register a device buffer (tensor, or raw pointer with n and dtype)."""
    if n is None:
        n = buf.numel()
    if dtype is None:
        dtype = dtype_code(buf)
    _check(_lib.gdraa_register(_ptr(buf), n, dtype), "gdraa_register")


def gdraa_deregister(buf):
    _check(_lib.gdraa_deregister(_ptr(buf)), "gdraa_deregister")


def gdraa_allreduce_mean(buf, stream=None):
    _check(_lib.gdraa_allreduce_mean(_ptr(buf), _stream(stream)), "gdraa_allreduce_mean")


def gdraa_sgd_step(w, g, v, lr: float, mom: float, stream=None):
    _check(_lib.gdraa_sgd_step(_ptr(w), _ptr(g), _ptr(v), lr, mom, _stream(stream)),
           "gdraa_sgd_step")


def gdraa_sgd_step_ex(w, g, v, lr: float, mom: float, wd: float, stream=None):
    _check(_lib.gdraa_sgd_step_ex(_ptr(w), _ptr(g), _ptr(v), lr, mom, wd, _stream(stream)),
           "gdraa_sgd_step_ex")


def gdraa_sgd_step_mp(w_master, w_model, g, v, lr: float, mom: float, wd: float = 0.0,
                      stream=None):
    _check(_lib.gdraa_sgd_step_mp(_ptr(w_master), _ptr(w_model), _ptr(g), _ptr(v), lr, mom, wd,
                                  _stream(stream)), "gdraa_sgd_step_mp")


def gdraa_poly_lr(lr0: float, it: int, max_iter: int, power: float = 1.0) -> float:
    return float(_lib.gdraa_poly_lr(lr0, it, max_iter, power))


def gdraa_allreduce_mean_range(buf, first: int, count: int, stream=None):
    _check(_lib.gdraa_allreduce_mean_range(_ptr(buf), first, count, _stream(stream)),
           "gdraa_allreduce_mean_range")


def gdraa_sgd_step_range(w, g, v, first: int, count: int, lr: float, mom: float,
                         wd: float = 0.0, stream=None):
    _check(_lib.gdraa_sgd_step_range(_ptr(w), _ptr(g), _ptr(v), first, count, lr, mom, wd,
                                     _stream(stream)), "gdraa_sgd_step_range")


def gdraa_sgd_step_mp_range(w_master, w_model, g, v, first: int, count: int, lr: float,
                            mom: float, wd: float = 0.0, stream=None):
    _check(_lib.gdraa_sgd_step_mp_range(_ptr(w_master), _ptr(w_model), _ptr(g), _ptr(v), first,
                                        count, lr, mom, wd, _stream(stream)),
           "gdraa_sgd_step_mp_range")


def gdraa_bucket_set_begin():
    _check(_lib.gdraa_bucket_set_begin(), "gdraa_bucket_set_begin")


def gdraa_bucket_set_begin_streamed(ctas: int):
    _check(_lib.gdraa_bucket_set_begin_streamed(ctas), "gdraa_bucket_set_begin_streamed")


def gdraa_bucket_set_end(stream=None):
    _check(_lib.gdraa_bucket_set_end(_stream(stream)), "gdraa_bucket_set_end")


def gdraa_small_message_bytes(world: int) -> int:
    return int(_lib.gdraa_small_message_bytes(world))


def gdraa_small_step_bytes(world: int, dtype: int = GDRAA_F32, mixed: bool = False) -> int:
    return int(_lib.gdraa_small_step_bytes(world, dtype, 1 if mixed else 0))


def gdraa_shard(world: int, rank: int, n: int):
    off, ln = ctypes.c_size_t(), ctypes.c_size_t()
    _check(_lib.gdraa_shard(world, rank, n, ctypes.byref(off), ctypes.byref(ln)), "gdraa_shard")
    return off.value, ln.value


def gdraa_get_stats() -> dict:
    st = gdraa_stats_t()
    _check(_lib.gdraa_get_stats(ctypes.byref(st)), "gdraa_get_stats")
    return {n: getattr(st, n) for n, _ in st._fields_}


def gdraa_finalize():
    _check(_lib.gdraa_finalize(), "gdraa_finalize")


def _ptr_array(xs):
    return (_vp * len(xs))(*[_ptr(x) for x in xs])


def _same_numel(n, *lists):
    """Every virtual rank's buffers hold n elements (the library trusts n)."""
    for xs in lists:
        for x in xs:
            if not isinstance(x, int) and x.numel() != n:
                raise ValueError(f"gdraa: virtual-rank buffers differ in length ({x.numel()} != {n})")


def gdraa_vr_allreduce_mean(bufs, stream=None):
    """`len(bufs)` virtual ranks on one GPU, one cooperative launch."""
    n = bufs[0].numel()
    _same_numel(n, bufs)
    _check(_lib.gdraa_vr_allreduce_mean(len(bufs), _ptr_array(bufs), n, dtype_code(bufs[0]),
                                        _stream(stream)), "gdraa_vr_allreduce_mean")


def gdraa_vr_sgd_step(w, g, v, lr: float, mom: float, stream=None):
    n = g[0].numel()
    _same_numel(n, w, g, v)
    _check(_lib.gdraa_vr_sgd_step(len(g), _ptr_array(w), _ptr_array(g), _ptr_array(v), n,
                                  dtype_code(g[0]), lr, mom, _stream(stream)),
           "gdraa_vr_sgd_step")


def gdraa_vr_sgd_step_ex(w, g, v, lr: float, mom: float, wd: float, stream=None):
    n = g[0].numel()
    _same_numel(n, w, g, v)
    _check(_lib.gdraa_vr_sgd_step_ex(len(g), _ptr_array(w), _ptr_array(g), _ptr_array(v), n,
                                     dtype_code(g[0]), lr, mom, wd, _stream(stream)),
           "gdraa_vr_sgd_step_ex")


def gdraa_vr_sgd_step_mp(w_master, w_model, g, v, lr: float, mom: float, wd: float = 0.0,
                         stream=None):
    n = g[0].numel()
    _same_numel(n, w_master, w_model, g, v)
    _check(_lib.gdraa_vr_sgd_step_mp(len(g), _ptr_array(w_master), _ptr_array(w_model),
                                     _ptr_array(g), _ptr_array(v), n, dtype_code(g[0]), lr, mom,
                                     wd, _stream(stream)), "gdraa_vr_sgd_step_mp")


def gdraa_vr_allreduce_mean_range(bufs, first: int, count: int, stream=None):
    """Bucketed form: [first, first + count) of every virtual rank's buffer."""
    n = bufs[0].numel()
    _same_numel(n, bufs)
    _check(_lib.gdraa_vr_allreduce_mean_range(len(bufs), _ptr_array(bufs), n,
                                              dtype_code(bufs[0]), first, count,
                                              _stream(stream)),
           "gdraa_vr_allreduce_mean_range")


def gdraa_vr_sgd_step_range(w, g, v, first: int, count: int, lr: float, mom: float,
                            wd: float = 0.0, stream=None):
    n = g[0].numel()
    _same_numel(n, w, g, v)
    _check(_lib.gdraa_vr_sgd_step_range(len(g), _ptr_array(w), _ptr_array(g), _ptr_array(v), n,
                                        dtype_code(g[0]), first, count, lr, mom, wd,
                                        _stream(stream)), "gdraa_vr_sgd_step_range")


def gdraa_vr_sgd_step_mp_range(w_master, w_model, g, v, first: int, count: int, lr: float,
                               mom: float, wd: float = 0.0, stream=None):
    n = g[0].numel()
    _same_numel(n, w_master, w_model, g, v)
    _check(_lib.gdraa_vr_sgd_step_mp_range(len(g), _ptr_array(w_master), _ptr_array(w_model),
                                           _ptr_array(g), _ptr_array(v), n, dtype_code(g[0]),
                                           first, count, lr, mom, wd, _stream(stream)),
           "gdraa_vr_sgd_step_mp_range")


def gdraa_vr_bucket_set_begin(world: int):
    _check(_lib.gdraa_vr_bucket_set_begin(world), "gdraa_vr_bucket_set_begin")


def gdraa_vr_bucket_set_end(world: int, stream=None):
    _check(_lib.gdraa_vr_bucket_set_end(world, _stream(stream)), "gdraa_vr_bucket_set_end")


def gdraa_vr_bucket_set_begin_streamed(world: int, ctas: int):
    _check(_lib.gdraa_vr_bucket_set_begin_streamed(world, ctas),
           "gdraa_vr_bucket_set_begin_streamed")
