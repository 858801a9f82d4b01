"""Seeded synthetic inputs for the GDRAA hot path, shared by the oracle side and the
CUDA side of every parity test and by bench.py.

This module holds NONE of the method's arithmetic (no partition, no sum, no mean, no
update, no rounding to the output dtype): only a counter-based random generator and
the workload recipe of DESIGN.md "Input recipe".  Random numbers are a pure function
of (seed, rank, stream, index), so any slice can be regenerated independently.

Workload sizes: the flat gradient buffer of ResNet-50 /
ResNet-101 (exact torchvision requires_grad counts), the paper's two models;
"a whole and continuous GPU memory" -> one flat buffer.
"""
import numpy as np

L_R50 = 25_557_032
L_R101 = 44_549_160
L_C1 = 1 << 20

# "learning rate is 0.1, momentum is 0.9"
PAPER_LR = 0.1
PAPER_MOM = 0.9

# Streams: independent sub-sequences per tensor role.
S_GRAD, S_W, S_V, S_SCALE, S_ZERO, S_SEG = range(1, 7)


def _splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _key(seed: int, rank: int, stream: int) -> np.uint64:
    k = _splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    k = _splitmix64(k ^ np.uint64(rank & 0xFFFFFFFF))
    return _splitmix64(k ^ np.uint64(stream))


def u64(seed: int, rank: int, stream: int, n: int, start: int = 0) -> np.ndarray:
    """n counter-based 64-bit draws for indices [start, start+n)."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _splitmix64(_key(seed, rank, stream) + idx * np.uint64(0xD1B54A32D192ED03))


def uniform01(seed, rank, stream, n, start=0) -> np.ndarray:
    """float64 uniform in (0, 1]."""
    return ((u64(seed, rank, stream, n, start) >> np.uint64(11)).astype(np.float64) + 1.0) \
        * (1.0 / 9007199254740992.0)


def normal(seed, rank, stream, n, start=0) -> np.ndarray:
    """float64 standard normal (Box-Muller on two independent streams)."""
    u1 = uniform01(seed, rank, stream, n, start)
    u2 = uniform01(seed, rank, stream + 100, n, start)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def integers(seed, rank, stream, n, lo, hi, start=0) -> np.ndarray:
    """float32 integers uniform in [lo, hi)."""
    span = np.uint64(hi - lo)
    return ((u64(seed, rank, stream, n, start) % span).astype(np.int64) + lo).astype(np.float32)


# ---------------------------------------------------------------------------------------
# Families.
# ---------------------------------------------------------------------------------------

def grad_integer(seed, rank, n, bf16=False):
    """Integer-valued gradient: [-2^13, 2^13) for fp32, [-128, 128) for bf16 (exactly
    representable in bf16's 8-bit significand).  Returned as float32 values."""
    lim = 128 if bf16 else 1 << 13
    return integers(seed, rank, S_GRAD, n, -lim, lim)


def w_integer(seed, n):
    return integers(seed, 0, S_W, n, -(1 << 12), 1 << 12)


def v_integer(seed, n):
    return integers(seed, 0, S_V, n, -(1 << 10), 1 << 10)


INT_LR = 0.125   # 2^-3
INT_MOM = 0.5    # 2^-1

SEGMENT = 4096


def neg_zero_segment(seed, n):
    """Index of the 4096-element segment that holds -0.0 on every rank (AMB-3)."""
    nseg = max(1, (n + SEGMENT - 1) // SEGMENT)
    return int(u64(seed, 0, S_SEG, 1)[0] % np.uint64(nseg))


_CHUNK = 1 << 20


def _chunked(fn, n, start, dtype):
    """Evaluate fn(count, start) over [start, start+n) in 1M-element chunks on a thread
    pool (numpy releases the GIL).  Values are counter-based, so chunking is invisible."""
    if n <= _CHUNK:
        return fn(n, start)
    from concurrent.futures import ThreadPoolExecutor
    import os
    out = np.empty(n, dtype=dtype)
    spans = [(a, min(_CHUNK, n - a)) for a in range(0, n, _CHUNK)]

    def run(span):
        a, c = span
        out[a:a + c] = fn(c, start + a)

    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(run, spans))
    return out


def grad_like(seed, rank, n, start=0):
    """Gradient-like float32 for indices [start, start+n): N(0,1) x 10^U(-6,-1) per
    4096-element segment (per-layer scales), 1% exact +0.0 and 0.1% -0.0."""
    return _chunked(lambda c, s: _grad_like(seed, rank, c, s), n, start, np.float32)


def _grad_like(seed, rank, n, start):
    seg = np.arange(start, start + n, dtype=np.uint64) // np.uint64(SEGMENT)
    with np.errstate(over="ignore"):
        e = _splitmix64(_key(seed, rank, S_SCALE) + seg * np.uint64(0xD1B54A32D192ED03))
    e = ((e >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)
    scale = 10.0 ** (-6.0 + 5.0 * e)
    g = (normal(seed, rank, S_GRAD, n, start) * scale).astype(np.float32)
    z = u64(seed, rank, S_ZERO, n, start) % np.uint64(1000)
    g[z < 10] = np.float32(0.0)
    g[z == 10] = np.float32(-0.0)
    return g


def grad_like_full(seed, rank, n):
    """grad_like over [0, n) with the shared all-ranks -0.0 segment applied."""
    g = grad_like(seed, rank, n)
    k = neg_zero_segment(seed, n)
    g[k * SEGMENT:(k + 1) * SEGMENT] = np.float32(-0.0)
    return g


def w_like(seed, n):
    """Weights ~ N(0, 0.05^2), identical on every rank."""
    return _chunked(lambda c, s: (normal(seed, 0, S_W, c, s) * 0.05).astype(np.float32),
                    n, 0, np.float32)


def to_bf16_bits_trunc(x: np.ndarray) -> np.ndarray:
    """Input-side bf16: keep the top 16 bits of each float32 (truncation).  This shapes
    an input distribution; it is not the method's output rounding."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> np.uint32(16)) \
        .astype(np.uint16)
