"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a worked example printed in the paper /
SPEC (tests/golden/spec_examples.json, cited per entry), exact rational arithmetic, a
closed form, an invariant, or an independent library routine (torch's bf16 cast).
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth
from tests._exact import exact, f32_bits, fraction_to_f32

F32 = np.float32


# ---------------------------------------------------------------------------------------
# Partition, Algorithm 1 "Divide D(i) by N", AMB-8
# ---------------------------------------------------------------------------------------

def test_partition_spec_examples(golden):
    for ex in golden["partition_q1"]:
        got = [oracle.partition(ex["L"], ex["N"], r, Q=1) for r in range(ex["N"])]
        assert [list(b) for b in got] == ex["blocks"], ex["cite"]


@pytest.mark.parametrize("Q", [1, 64])
def test_partition_invariants(Q):
    # blocks cover [0, L) exactly, sorted, disjoint; pure function.
    rng = np.random.default_rng(0)
    cases = [(L, N) for L in (1, 2, 3, 7, 63, 64, 65, 1000, 4096, 1 << 20, synth.L_R50,
                              synth.L_R101) for N in range(1, 33)]
    cases += [(int(rng.integers(1, 10**7)), int(rng.integers(1, 33))) for _ in range(200)]
    for L, N in cases:
        blocks = [oracle.partition(L, N, r, Q=Q) for r in range(N)]
        assert blocks == [oracle.partition(L, N, r, Q=Q) for r in range(N)]
        pos = 0
        for off, ln in blocks:
            assert off == pos
            pos += ln
        assert pos == L
        blk = math.ceil(math.ceil(L / N) / Q) * Q
        lens = [ln for _, ln in blocks]
        # every block but the trailing (short / empty) ones is exactly one block length
        full = [ln == blk for ln in lens]
        k = full.index(False) if False in full else N
        assert all(full[:k]) and all(ln < blk for ln in lens[k:])
        assert all(lens[i] >= lens[i + 1] for i in range(N - 1))
        assert all(off % Q == 0 or ln == 0 for off, ln in blocks)


def test_partition_resnet_sizes():
    # R50 N=8 -> 7 x 3,194,688 + 3,194,216; R101 N=8 -> 7 x 5,568,704
    # + 5,568,232 (closed form: ceil(L/8) rounded up to 64, remainder in the last block).
    r50 = [oracle.partition(synth.L_R50, 8, r)[1] for r in range(8)]
    assert r50 == [3_194_688] * 7 + [3_194_216]
    r101 = [oracle.partition(synth.L_R101, 8, r)[1] for r in range(8)]
    assert r101 == [5_568_704] * 7 + [5_568_232]


def test_partition_rejects():
    for args in [(0, 2, 0), (10, 0, 0), (10, 33, 0), (10, 2, 2), (10, 2, -1)]:
        with pytest.raises(ValueError):
            oracle.partition(*args)


# ---------------------------------------------------------------------------------------
# bf16 conversions (AMB-13): pinned to torch's own bf16 cast (library routine).
# ---------------------------------------------------------------------------------------

def test_bf16_rne_ties_to_even():
    assert oracle.f32_to_bf16_rne(1.0 + 2.0**-8) == 0x3F80          # tie -> even (1.0)
    assert oracle.f32_to_bf16_rne(1.0 + 3 * 2.0**-8) == 0x3F82      # tie -> even (1.015625)
    assert oracle.f32_to_bf16_rne(-0.0) == 0x8000


def test_bf16_matches_torch():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.standard_normal(20000).astype(F32) * F32(10) ** rng.integers(
        -30, 30, 20000).astype(F32),
        rng.integers(-(1 << 24), 1 << 24, 20000).astype(F32),
        np.array([0.0, -0.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, 65504.0], dtype=F32)])
    x = x[np.isfinite(x)]
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([oracle.f32_to_bf16_rne(float(v)) for v in x[:5000]], dtype=np.uint16)
    assert np.array_equal(got, ref[:5000])
    # widening is exact: compare with torch bf16 -> f32
    bits = rng.integers(0, 1 << 16, 4000).astype(np.uint16)
    bits = bits[((bits >> 7) & 0xFF) != 0xFF]                    # finite only (AMB-16)
    wide = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float().numpy()
    got_w = np.array([oracle.bf16_to_f32(int(b)) for b in bits], dtype=F32)
    assert np.array_equal(got_w.view(np.uint32), wide.view(np.uint32))


# ---------------------------------------------------------------------------------------
# Aggregation "Average D(k,i)" (Eq. 3)
# ---------------------------------------------------------------------------------------

def test_mean_spec_examples(golden):
    for ex in golden["mean"]:
        got = oracle.allreduce_mean([np.array(x, dtype=F32) for x in ex["inputs"]])
        assert np.array_equal(got, np.array(ex["out"], dtype=F32)), ex["cite"]


def test_mean_n1_identity_bits():
    # S:179 N=1 -> output = input, including the sign of zero and subnormals.
    x = np.array([-0.0, 0.0, 1e-45, -3.5, 7e30], dtype=F32)
    assert np.array_equal(oracle.allreduce_mean([x]).view(np.uint32), x.view(np.uint32))


VALUES = [-2.0, -1.0, -0.5, -0.0, 0.0, 0.5, 1.0, 3.0]


def _exact_expected(cols, N):
    """Exact rational mean, rounded once; sign of an exact zero per IEEE RN rules for a
    left fold: -0.0 iff every addend is -0.0."""
    s = sum(exact(c) for c in cols)
    m = fraction_to_f32(s / N)
    if s == 0:
        allneg = all(np.signbit(F32(c)) for c in cols)
        return F32(-0.0) if allneg else F32(0.0)
    return m


def test_mean_bf16_output_rne_ties():
    # AMB-13 / P:169: allreduce_mean on a bf16 buffer stores bf16_rne(fp32 mean).  N = 2,
    # bf16 inputs whose exact mean lands on a bf16 rounding tie: 1+2^-8 rounds to even
    # 1.0 (0x3F80), 1+3*2^-8 rounds to even 1.015625 (0x3F82; truncation gives 0x3F81).
    a = np.array([0x3F80, 0x3F81, 0xBF81], dtype=np.uint16)      # 1, 1+2^-7, -(1+2^-7)
    b = np.array([0x3F81, 0x3F82, 0xBF82], dtype=np.uint16)      # 1+2^-7, 1+2^-6, -(1+2^-6)
    got = oracle.allreduce_mean([a, b])
    assert got.tolist() == [0x3F80, 0x3F82, 0xBF82]


@pytest.mark.parametrize("N", [2, 3, 5])
def test_mean_bf16_output_matches_torch_cast_of_exact_mean(N):
    # bf16 inputs with a small exponent spread, so the fp32 left fold is exact; the fp32
    # mean is then the correctly rounded exact mean (fraction_to_f32), and the stored
    # bf16 is torch's fp32 -> bf16 cast of it (a library routine).  Near-ties and exact
    # ties both occur; a truncating or ties-away cast fails.
    rng = np.random.default_rng(40 + N)
    L = 3000
    sig = rng.integers(0x80, 0x100, size=(N, L))                  # 8-bit significands
    ex = rng.integers(125, 129, size=(N, L))                      # exponents 2^-2 .. 2^1
    sg = rng.integers(0, 2, size=(N, L))
    sg[:, : L // 2] = 0                                            # half same-sign
    bits = ((sg << 15) | (ex << 7) | (sig & 0x7F)).astype(np.uint16)
    got = oracle.allreduce_mean([bits[p] for p in range(N)])
    vals = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float().numpy()
    means = np.array([fraction_to_f32(sum(exact(vals[p, i]) for p in range(N)) / N)
                      for i in range(L)], dtype=F32)
    ref = torch.from_numpy(means).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)
    # the case set really contains values that truncation would get wrong
    assert np.count_nonzero((means.view(np.uint32) >> 16).astype(np.uint16) != ref) > L // 10


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_mean_bruteforce_exact(N):
    # Brute force over a tiny value set: every partial sum of these dyadics is exact in
    # fp32, so the only rounding is the single division (exact result rounded once).
    cols = list(itertools.product(VALUES, repeat=N))
    L = len(cols)
    bufs = [np.array([c[p] for c in cols], dtype=F32) for p in range(N)]
    got = oracle.allreduce_mean(bufs)
    exp = np.array([_exact_expected(c, N) for c in cols], dtype=F32)
    assert got.shape == (L,)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))


def test_mean_rank_order_pinned():
    # AMB-2: a left fold in ascending rank starting at rank 0.  With x = [1, 2^-24,
    # 2^-24, 2^-24]: 1 + 2^-24 ties to even -> 1 at every step, mean = 1/4 exactly.
    # Any other order (e.g. right-to-left: 3*2^-24 + 1 -> 1 + 2^-22) gives 1/4 + 2^-24.
    x = [np.array([v], dtype=F32) for v in (1.0, 2.0**-24, 2.0**-24, 2.0**-24)]
    assert f32_bits(oracle.allreduce_mean(x)[0]) == f32_bits(0.25)
    rev = x[::-1]
    assert f32_bits(oracle.allreduce_mean(rev)[0]) == f32_bits(0.25 + 2.0**-24)


def test_mean_division_not_reciprocal():
    # AMB-2: one IEEE division by N (not multiplication by fl(1/N)).  For N = 3 and
    # s = 3 * 5 = 15 ... pick s where fl(s/3) != fl(s * fl(1/3)): exact rounding decides.
    N = 3
    found = 0
    for k in range(1, 2000):
        s = F32(k) * F32(1.0 + 2.0**-20)
        exp = fraction_to_f32(exact(s) / N)
        recip = fraction_to_f32(exact(s) * exact(fraction_to_f32(Fraction(1, 3))))
        if exp != recip:
            found += 1
            got = oracle.allreduce_mean([np.array([s], F32), np.array([0.0], F32),
                                         np.array([0.0], F32)])[0]
            assert f32_bits(got) == f32_bits(exp)
    assert found > 10


@pytest.mark.parametrize("N", [2, 3, 5, 7, 8, 16, 32])
def test_mean_within_error_bound(N):
    # Exact mean by rational arithmetic; the fp32 left fold + division must lie within
    # the standard bound |m^ - m| <= (gamma_{N-1} sum|x| + u(|s| + gamma sum|x|)) / N.
    L = 257
    bufs = [synth.grad_like(7, p, L) for p in range(N)]
    got = oracle.allreduce_mean(bufs)
    u = Fraction(1, 2**24)
    gamma = (N - 1) * u / (1 - (N - 1) * u)
    for i in range(L):
        xs = [exact(b[i]) for b in bufs]
        s = sum(xs)
        a = sum(abs(x) for x in xs)
        bound = (gamma * a + u * (abs(s) + gamma * a)) / N
        assert abs(exact(got[i]) - s / N) <= bound, i
    # and against torch's float64 mean (library routine), same bound in float
    ref = torch.from_numpy(np.stack(bufs)).double().mean(0).numpy()
    assert np.allclose(got, ref, rtol=0, atol=float(N * 2.0**-22) * np.abs(np.stack(bufs)).max())


@pytest.mark.parametrize("N", list(range(1, 33)))
def test_mean_of_constant(N):
    # "the mean of a constant is that constant" / "sum of N identical inputs = N x"
    # (north star), with the precondition that x has <= 24 - ceil(log2 N) significant bits
    # so that every partial sum k*x is exact (SURVEY.md §8(c) O3/O4 pin).
    bits = 24 - math.ceil(math.log2(N)) if N > 1 else 24
    rng = np.random.default_rng(N)
    mant = rng.integers(1 << (bits - 1), 1 << bits, 500)
    x = (mant * 2.0 ** rng.integers(-60, 20, 500).astype(np.float64)
         * rng.choice([-1, 1], 500)).astype(F32)
    got = oracle.allreduce_mean([x] * N)
    assert np.array_equal(got.view(np.uint32), x.view(np.uint32))


# ---------------------------------------------------------------------------------------
# Update "Update model with gradient of differential D", AMB-4
# ---------------------------------------------------------------------------------------

def _one(v):
    return np.array([v], dtype=F32)


def test_sgd_spec_single_step(golden):
    ex = golden["sgd"][0]
    w, v = oracle.sgd_step([_one(ex["g"])], _one(ex["w"]), _one(0.0), ex["lr"], ex["mom"])
    assert abs(float(w[0]) - ex["w_out"]) <= 2.0**-24 * 2, ex["cite"]
    # exact: w' = RNE(1 - RNE(lr*1)) -- one rounding per operation (AMB-4)
    lr = F32(ex["lr"])
    assert f32_bits(w[0]) == f32_bits(fraction_to_f32(1 - exact(lr)))


def test_sgd_spec_two_steps(golden):
    ex = golden["sgd"][1]
    w, v = _one(ex["w"]), _one(0.0)
    ws = [float(w[0])]
    for _ in range(ex["steps"]):
        w, v = oracle.sgd_step([_one(ex["g"])] * 4, w, v, ex["lr"], ex["mom"])
        ws.append(float(w[0]))
    dec = [ws[k] - ws[k + 1] for k in range(ex["steps"])]
    assert np.allclose(dec, ex["decreases"], rtol=0, atol=1e-6), ex["cite"]


def test_sgd_dyadic_closed_form():
    # mu = 1/2, lr = 1/4, g = 1 on every rank, w0 = 1, v0 = 0: every value is dyadic, so
    # the closed form v_k = (1 - mu^k)/(1 - mu), w_k = w0 - lr * sum_j v_j holds exactly.
    mu, lr = Fraction(1, 2), Fraction(1, 4)
    for N in (1, 2, 3, 4, 8):
        w, v = _one(1.0), _one(0.0)
        wk = Fraction(1)
        for k in range(1, 12):
            w, v = oracle.sgd_step([_one(1.0)] * N, w, v, float(lr), float(mu))
            vk = (1 - mu**k) / (1 - mu)
            wk = wk - lr * vk
            assert exact(v[0]) == vk and exact(w[0]) == wk, (N, k)


@pytest.mark.parametrize("N", [1, 2, 4, 8])
@pytest.mark.parametrize("bf16", [False, True])
def test_sgd_integer_family_exact(N, bf16):
    # Integer family (north star: "integer-valued test gradients must match bit-exactly"):
    # with N a power of two every intermediate is exactly representable, so the result is
    # the exact rational update.  Computed here with Fractions, checked representable.
    L = 3000
    gs = [synth.grad_integer(3, p, L, bf16=bf16) for p in range(N)]
    w0, v0 = synth.w_integer(3, L), synth.v_integer(3, L)
    lr, mom = synth.INT_LR, synth.INT_MOM
    gin = [synth.to_bf16_bits_trunc(g) for g in gs] if bf16 else gs
    w, v = oracle.sgd_step(gin, w0, v0, lr, mom)
    for i in range(0, L, 7):
        m = sum(exact(g[i]) for g in gs) / N
        vn = Fraction(mom) * exact(v0[i]) + m
        wn = exact(w0[i]) - Fraction(lr) * vn
        assert exact(fraction_to_f32(vn)) == vn and exact(fraction_to_f32(wn)) == wn
        assert exact(v[i]) == vn and exact(w[i]) == wn, i


def test_sgd_signed_zero():
    # AMB-3 + IEEE: all ranks -0.0 -> mean -0.0; v' = fl(fl(mu * (+0)) + (-0)) = +0.0,
    # and with v = -0.0: fl(mu * -0) = -0, -0 + -0 = -0.
    g = [_one(-0.0)] * 3
    w, v = oracle.sgd_step(g, _one(1.0), _one(0.0), 0.1, 0.9)
    assert f32_bits(v[0]) == f32_bits(0.0) and w[0] == F32(1.0)
    w, v = oracle.sgd_step(g, _one(1.0), _one(-0.0), 0.1, 0.9)
    assert f32_bits(v[0]) == f32_bits(-0.0)
    assert f32_bits(oracle.allreduce_mean(g)[0]) == f32_bits(-0.0)


def test_sgd_unfused_rounding():
    # AMB-4: four separately rounded operations; find elements where fma(mu, v, m) would
    # differ and check the oracle matches the exact per-operation rounding instead.
    rng = np.random.default_rng(5)
    L = 2000
    g = [rng.standard_normal(L).astype(F32) for _ in range(2)]
    w0 = rng.standard_normal(L).astype(F32)
    v0 = rng.standard_normal(L).astype(F32)
    lr, mom = F32(0.1), F32(0.9)
    w, v = oracle.sgd_step(g, w0, v0, lr, mom)
    diff_fma = 0
    for i in range(L):
        s = fraction_to_f32(exact(g[0][i]) + exact(g[1][i]))
        m = fraction_to_f32(exact(s) / 2)
        t = fraction_to_f32(exact(mom) * exact(v0[i]))
        vn = fraction_to_f32(exact(t) + exact(m))
        u = fraction_to_f32(exact(lr) * exact(vn))
        wn = fraction_to_f32(exact(w0[i]) - exact(u))
        assert f32_bits(v[i]) == f32_bits(vn) and f32_bits(w[i]) == f32_bits(wn), i
        if fraction_to_f32(exact(mom) * exact(v0[i]) + exact(m)) != vn:
            diff_fma += 1
    assert diff_fma > 0          # the test distinguishes fused from unfused


# ---------------------------------------------------------------------------------------
# Lemma 1 / Lemma 2 counters
# ---------------------------------------------------------------------------------------

def test_counters_lemmas(golden):
    ex = golden["lemma1_bytes"][0]
    for r in range(ex["N"]):
        c = oracle.counters(ex["L"], ex["N"], r, ex["width"], ex["width"], Q=1)
        assert c["rs_sent"] == c["rs_recv"] == c["ag_sent"] == c["ag_recv"] \
            == ex["bytes_per_phase"], ex["cite"]
        assert c["sync_waits"] == 2
    ex = golden["lemma2_ops"][0]
    c = oracle.counters(ex["L"], ex["N"], 0, 4, 4, Q=1)
    assert (c["adds"], c["divides"], c["adds"] + c["divides"]) == \
        (ex["adds"], ex["muls"], ex["total"]), ex["cite"]


@pytest.mark.parametrize("L,N", [(1000, 8), (7, 3), (3, 4), (synth.L_R50, 8), (1, 1),
                                 (synth.L_R101, 5)])
def test_counters_conservation(L, N):
    cs = [oracle.counters(L, N, r, 2, 4) for r in range(N)]
    # every byte sent is received (reduce and broadcast), and Eq. 4's Op = L per worker
    # sums to N * L over the ring of owners.
    assert sum(c["rs_sent"] for c in cs) == sum(c["rs_recv"] for c in cs)
    assert sum(c["ag_sent"] for c in cs) == sum(c["ag_recv"] for c in cs)
    assert sum(c["adds"] + c["divides"] for c in cs) == N * L
    assert all(c["sync_waits"] == (2 if N > 1 else 0) for c in cs)


# ---------------------------------------------------------------------------------------
# NEXT-1: weight decay ("weight decay is 0.001"), the bf16 model copy of the
# mixed-precision all-gather, and the "poly" learning-rate policy.
# ---------------------------------------------------------------------------------------

def test_sgd_wd_zero_is_core_update():
    # wd = 0 forms no decay term: bitwise the pinned core update (incl. -0.0 handling)
    N, L = 4, 5000
    gs = [synth.grad_like(41, p, L) for p in range(N)]
    w0, v0 = synth.w_like(41, L), synth.w_like(42, L)
    w1, v1 = oracle.sgd_step(gs, w0, v0, 0.1, 0.9)
    w2, v2 = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.0)
    assert np.array_equal(w1.view(np.uint32), w2.view(np.uint32))
    assert np.array_equal(v1.view(np.uint32), v2.view(np.uint32))


def test_sgd_wd_dyadic_closed_form():
    # S:412 v <- mu v + (g + lambda w); w <- w - lr v with dyadic mu = lr = lambda = 1/2,
    # 1/4, 1/2: every value is exact, so the float trajectory equals the rational one.
    mu, lr, lam = Fraction(1, 2), Fraction(1, 4), Fraction(1, 2)
    for N in (1, 2, 4):
        w, v = _one(1.0), _one(0.0)
        wk, vk = Fraction(1), Fraction(0)
        for k in range(5):      # the rational trajectory outgrows 24 bits after ~6 steps
            w, v = oracle.sgd_step_wd([_one(1.0)] * N, w, v, float(lr), float(mu), float(lam))
            vk = mu * vk + (1 + lam * wk)
            wk = wk - lr * vk
            assert exact(fraction_to_f32(vk)) == vk and exact(fraction_to_f32(wk)) == wk
            assert exact(v[0]) == vk and exact(w[0]) == wk, (N, k)
    # first two steps by hand: v1 = 1.5, w1 = 0.625; v2 = 2.0625, w2 = 0.109375
    w, v = oracle.sgd_step_wd([_one(1.0)], _one(1.0), _one(0.0), 0.25, 0.5, 0.5)
    assert (float(v[0]), float(w[0])) == (1.5, 0.625)
    w, v = oracle.sgd_step_wd([_one(1.0)], w, v, 0.25, 0.5, 0.5)
    assert (float(v[0]), float(w[0])) == (2.0625, 0.109375)


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_sgd_wd_integer_family_exact(N):
    # integer family with lambda = 2^-4: every intermediate stays exactly representable
    L = 3000
    gs = [synth.grad_integer(13, p, L) for p in range(N)]
    w0, v0 = synth.w_integer(13, L), synth.v_integer(13, L)
    lr, mom, lam = synth.INT_LR, synth.INT_MOM, 2.0**-4
    w, v = oracle.sgd_step_wd(gs, w0, v0, lr, mom, lam)
    for i in range(0, L, 11):
        m = sum(exact(g[i]) for g in gs) / N
        ge = m + Fraction(lam) * exact(w0[i])
        vn = Fraction(mom) * exact(v0[i]) + ge
        wn = exact(w0[i]) - Fraction(lr) * vn
        assert exact(fraction_to_f32(vn)) == vn and exact(fraction_to_f32(wn)) == wn
        assert exact(v[i]) == vn and exact(w[i]) == wn, i


def test_sgd_mp_model_copy_is_bf16_of_master():
    # the broadcast model copy is bf16 RNE of the updated fp32 master (torch's cast)
    N, L = 3, 4000
    gs = [synth.to_bf16_bits_trunc(synth.grad_like(51, p, L)) for p in range(N)]
    w0, v0 = synth.w_like(51, L), synth.w_like(52, L)
    w, v, model = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001, model_dtype=oracle.BF16)
    ref = torch.from_numpy(w).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(model, ref)
    w2, v2 = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
    assert np.array_equal(w.view(np.uint32), w2.view(np.uint32))
    w3, v3, m3 = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001, model_dtype=oracle.F32)
    assert np.array_equal(m3.view(np.uint32), w.view(np.uint32))


def test_poly_lr(golden):
    for ex in golden["poly_lr"]:
        assert oracle.poly_lr(ex["lr0"], ex["iter"], ex["max_iter"], ex["power"]) == \
            np.float32(ex["lr"]), ex["cite"]
    assert oracle.poly_lr(0.1, 0, 1000, 1.0) == np.float32(0.1)
    assert oracle.poly_lr(0.1, 1000, 1000, 1.0) == 0.0
    assert oracle.poly_lr(0.1, 500, 1000, 2.0) == np.float32(0.025)
    # monotone non-increasing in iter for power > 0
    lrs = [oracle.poly_lr(0.1, i, 997, 1.0) for i in range(0, 998, 7)]
    assert all(a >= b for a, b in zip(lrs, lrs[1:]))


# ---------------------------------------------------------------------------------------
# NEXT-4: synchronous data-parallel SGD equals serial large-batch SGD
# ---------------------------------------------------------------------------------------

def _ls_grad(X, y, w):
    return X.T @ (X @ w - y) / X.shape[0]


def test_oracle_ssgd_equals_serial_large_batch():
    """N=4 ranks with b=8 samples each, the oracle averaging their fp32 gradients and
    applying momentum SGD, tracks the float64 serial run on batches of 32 within 1e-5
    over 100 iterations."""
    from synth.least_squares import Problem
    P = Problem(seed=3)
    N, b, lr, mom = 4, 8, 0.05, 0.9
    w64, v64 = np.zeros(P.d), np.zeros(P.d)
    w32, v32 = np.zeros(P.d, np.float32), np.zeros(P.d, np.float32)
    gap = 0.0
    for it in range(100):
        X, y = P.batch(it, N, b)
        v64 = mom * v64 + _ls_grad(X, y, w64)
        w64 = w64 - lr * v64
        gs = [_ls_grad(*P.batch(it, N, b, r), w32.astype(np.float64)).astype(np.float32)
              for r in range(N)]
        w32, v32 = oracle.sgd_step(gs, w32, v32, lr, mom)
        gap = max(gap, float(np.max(np.abs(w32 - w64))))
    assert gap < 1e-5, gap
    r = P.X @ w64 - P.y
    assert 0.5 * np.mean(r * r) < 1e-3           # it actually trained
