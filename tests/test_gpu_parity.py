"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Single-GPU coverage of every world size uses the virtual-rank entry points
(gdraa_vr_*): the same kernel runs N ranks in one cooperative launch on one B200, with
rank r's CTAs reading and writing rank p's buffers and the two synchronisations going
through per-rank signal pads.  The multi-process NVLink path is in test_multigpu.py.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests._parity import compare
from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA GPU")]

if has_cuda():
    from paper_1802_02326_b200 import gdraa

DEV = "cuda:0"


def to_dev(x, bf16=False, dev=DEV):
    if bf16:
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).to(dev).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def from_dev(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def make_grads(family, seed, N, L, bf16):
    if family == "int":
        gs = [synth.grad_integer(seed, p, L, bf16=bf16) for p in range(N)]
    else:
        gs = [synth.grad_like(seed, p, L) for p in range(N)]
        k = synth.neg_zero_segment(seed, L)
        for g in gs:
            g[k * synth.SEGMENT:(k + 1) * synth.SEGMENT] = np.float32(-0.0)
    if bf16:
        gs = [synth.to_bf16_bits_trunc(g) for g in gs]
    return gs


def make_wv(family, seed, L):
    if family == "int":
        return synth.w_integer(seed, L), synth.v_integer(seed, L), synth.INT_LR, synth.INT_MOM
    return synth.w_like(seed, L), np.zeros(L, np.float32), synth.PAPER_LR, synth.PAPER_MOM


SIZES = [1, 5, 64, 257, 1000, 70_001, 1 << 20]


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("family", ["int", "like"])
def test_vr_allreduce_mean(N, dt, family):
    bf16 = dt == "bf16"
    for L in SIZES:
        gs = make_grads(family, 100 + N, N, L, bf16)
        exp = oracle.allreduce_mean(gs)
        bufs = [to_dev(g, bf16) for g in gs]
        gdraa.gdraa_vr_allreduce_mean(bufs)
        torch.cuda.synchronize()
        for r in range(N):
            compare(from_dev(bufs[r]), exp, dt, what=f"mean N={N} L={L} rank {r}")


@pytest.mark.parametrize("N", [2, 3, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_vr_allreduce_mean_latency_path(N, dt):
    """Sizes on both sides of the small-message (LL) threshold, odd bf16 lengths (ragged
    8-byte pairs), repeated calls (epoch parity of the receive slots)."""
    bf16 = dt == "bf16"
    es = 2 if bf16 else 4
    lim = gdraa.gdraa_small_message_bytes(N) // es      # largest LL element count
    for L in (1, 2, 3, 4097, 65535, 65536, lim - 1, lim, lim + 1):
        for it in range(3):
            gs = make_grads("like", 700 + it, N, L, bf16)
            exp = oracle.allreduce_mean(gs)
            bufs = [to_dev(g, bf16) for g in gs]
            gdraa.gdraa_vr_allreduce_mean(bufs)
            torch.cuda.synchronize()
            for r in range(N):
                compare(from_dev(bufs[r]), exp, dt, what=f"LL mean N={N} L={L} it{it} r{r}")


@pytest.mark.parametrize("N", [1, 2, 3, 4, 6, 7, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("family", ["int", "like"])
def test_vr_sgd_step(N, dt, family):
    bf16 = dt == "bf16"
    for L in SIZES:
        gs = make_grads(family, 200 + N, N, L, bf16)
        w0, v0, lr, mom = make_wv(family, 200 + N, L)
        if family == "like":
            v0 = synth.w_like(300 + N, L)          # non-zero momentum state
        w_exp, v_exp = oracle.sgd_step(gs, w0, v0, lr, mom)
        g_d = [to_dev(g, bf16) for g in gs]
        w_d = [to_dev(w0) for _ in range(N)]
        v_d = [to_dev(v0) for _ in range(N)]
        gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, lr, mom)
        torch.cuda.synchronize()
        for r in range(N):
            compare(from_dev(w_d[r]), w_exp, "f32", what=f"w N={N} L={L} rank {r}")
            off, ln = gdraa.gdraa_shard(N, r, L)
            vr = from_dev(v_d[r])
            compare(vr[off:off + ln], v_exp[off:off + ln], "f32", what=f"v N={N} L={L} r{r}")
            # AMB-19: non-owned momentum entries are untouched
            keep = np.ones(L, bool)
            keep[off:off + ln] = False
            assert np.array_equal(vr[keep].view(np.uint32), v0[keep].view(np.uint32))
            # AMB-18: g is read only
            assert np.array_equal(from_dev(g_d[r]), gs[r])


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("mixed", [False, True])
def test_vr_sgd_latency_path(N, dt, mixed):
    """The small-message SGD kernel (gradient and updated blocks pushed as flagged LL
    entries, no device barrier): sizes on both sides of its threshold, ragged shards
    (odd lengths, empty shards), 3 chained steps (epoch parity of the receive slots),
    weight decay, and the mixed-precision broadcast."""
    bf16 = dt == "bf16"
    es = 2 if bf16 else 4
    code = gdraa.GDRAA_BF16 if bf16 else gdraa.GDRAA_F32
    lim = gdraa.gdraa_small_step_bytes(N, code, mixed) // es   # largest LL element count
    assert lim > 0
    for L in (1, 3, 63, 65, 127, 4097, 65_537, lim - 1, lim, lim + 1):
        gs0 = make_grads("like", 900 + L % 13, N, L, bf16)
        w, v = synth.w_like(901, L), synth.w_like(902, L)
        w_d = [to_dev(w) for _ in range(N)]
        v_d = [to_dev(v) for _ in range(N)]
        mo_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
        for it in range(3):
            gs = gs0 if it == 0 else make_grads("like", 910 + it, N, L, bf16)
            g_d = [to_dev(g, bf16) for g in gs]
            if mixed:
                w, v, model = oracle.sgd_step_wd(gs, w, v, synth.PAPER_LR, synth.PAPER_MOM,
                                                 0.001, model_dtype=oracle.BF16)
                gdraa.gdraa_vr_sgd_step_mp(w_d, mo_d, g_d, v_d, synth.PAPER_LR,
                                           synth.PAPER_MOM, 0.001)
            else:
                w, v = oracle.sgd_step_wd(gs, w, v, synth.PAPER_LR, synth.PAPER_MOM, 0.001)
                gdraa.gdraa_vr_sgd_step_ex(w_d, g_d, v_d, synth.PAPER_LR, synth.PAPER_MOM,
                                           0.001)
            torch.cuda.synchronize()
            for r in range(N):
                off, ln = gdraa.gdraa_shard(N, r, L)
                what = f"LL sgd N={N} {dt} mp={mixed} L={L} it{it} r{r}"
                if mixed:
                    compare(from_dev(mo_d[r]), model, "bf16", what=what + " model")
                    compare(from_dev(w_d[r])[off:off + ln], w[off:off + ln], "f32",
                            what=what + " master")
                else:
                    compare(from_dev(w_d[r]), w, "f32", what=what + " w")
                compare(from_dev(v_d[r])[off:off + ln], v[off:off + ln], "f32",
                        what=what + " v")
                assert np.array_equal(from_dev(g_d[r]), gs[r]), what + " g changed"


@pytest.mark.parametrize("N", [2, 4])
def test_vr_mixed_call_sequence(N):
    """Receive-slot parity alternates over every call of a rank, whichever kernel serves
    it: interleave small means, small steps and two-shot steps on the same ranks."""
    L_small, L_big = 10_001, 1_500_001
    rng_calls = ["mean_s", "sgd_s", "sgd_b", "sgd_s", "mean_s", "mean_s", "sgd_s", "sgd_b",
                 "sgd_s"]
    w = {L: synth.w_like(31, L) for L in (L_small, L_big)}
    v = {L: np.zeros(L, np.float32) for L in (L_small, L_big)}
    w_d = {L: [to_dev(w[L]) for _ in range(N)] for L in w}
    v_d = {L: [to_dev(v[L]) for _ in range(N)] for L in v}
    for k, call in enumerate(rng_calls):
        L = L_big if call.endswith("_b") else L_small
        gs = make_grads("like", 40 + k, N, L, False)
        g_d = [to_dev(g) for g in gs]
        if call.startswith("mean"):
            gdraa.gdraa_vr_allreduce_mean(g_d)
            torch.cuda.synchronize()
            exp = oracle.allreduce_mean(gs)
            for r in range(N):
                compare(from_dev(g_d[r]), exp, "f32", what=f"call {k} mean r{r}")
            continue
        w[L], v[L] = oracle.sgd_step(gs, w[L], v[L], 0.1, 0.9)
        gdraa.gdraa_vr_sgd_step(w_d[L], g_d, v_d[L], 0.1, 0.9)
        torch.cuda.synchronize()
        for r in range(N):
            off, ln = gdraa.gdraa_shard(N, r, L)
            compare(from_dev(w_d[L][r]), w[L], "f32", what=f"call {k} {call} w r{r}")
            compare(from_dev(v_d[L][r])[off:off + ln], v[L][off:off + ln], "f32",
                    what=f"call {k} {call} v r{r}")


@pytest.mark.parametrize("N,dt", [(2, "f32"), (4, "f32"), (8, "bf16")])
def test_vr_chained_iterations(N, dt):
    """10 chained steps with fresh gradients each iteration (random family, P:246
    hyper-parameters), compared after every iteration."""
    bf16 = dt == "bf16"
    L = 300_007
    w, v = synth.w_like(9, L), np.zeros(L, np.float32)
    w_d = [to_dev(w) for _ in range(N)]
    v_full = [to_dev(v) for _ in range(N)]
    for it in range(10):
        gs = make_grads("like", 1000 + it, N, L, bf16)
        g_d = [to_dev(g, bf16) for g in gs]
        w, v = oracle.sgd_step(gs, w, v, synth.PAPER_LR, synth.PAPER_MOM)
        gdraa.gdraa_vr_sgd_step(w_d, g_d, v_full, synth.PAPER_LR, synth.PAPER_MOM)
        torch.cuda.synchronize()
        for r in range(N):
            compare(from_dev(w_d[r]), w, "f32", what=f"it {it} w rank {r}")
            off, ln = gdraa.gdraa_shard(N, r, L)
            compare(from_dev(v_full[r])[off:off + ln], v[off:off + ln], "f32",
                    what=f"it {it} v rank {r}")


def test_vr_determinism_and_partition_independence():
    """bitwise identical across runs; w' and the mean do not depend on N's
    partition (same inputs averaged by 4 ranks in two different launches)."""
    L, N = 1 << 20, 4
    gs = make_grads("like", 77, N, L, False)
    outs = []
    for _ in range(3):
        bufs = [to_dev(g) for g in gs]
        gdraa.gdraa_vr_allreduce_mean(bufs)
        torch.cuda.synchronize()
        outs.append([from_dev(b) for b in bufs])
    for run in outs[1:]:
        for a, b in zip(run, outs[0]):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_vr_full_size_resnet50_bf16_n8():
    """Config 4 at its stated N=8: ResNet-50 gradients in bf16, fp32 accumulation, fp32
    master w/v -- full size, every element, both iteration 1 and a chained iteration 2."""
    N, L = 8, synth.L_R50
    gs = make_grads("like", 4, N, L, True)
    w0, v0 = synth.w_like(4, L), np.zeros(L, np.float32)
    w1, v1 = oracle.sgd_step(gs, w0, v0, synth.PAPER_LR, synth.PAPER_MOM)
    g_d = [to_dev(g, True) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, synth.PAPER_LR, synth.PAPER_MOM)
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(w_d[r]), w1, "f32", what=f"R50 bf16 w rank {r}")
        off, ln = gdraa.gdraa_shard(N, r, L)
        compare(from_dev(v_d[r])[off:off + ln], v1[off:off + ln], "f32", what=f"v rank {r}")


@pytest.mark.parametrize("L", [synth.L_R50, synth.L_R101])
def test_vr_full_size_fp32_n4(L):
    """Configs 2/3 at full size (fp32, N=4 virtual ranks): every element."""
    N = 4
    gs = make_grads("like", 5, N, L, False)
    w0, v0 = synth.w_like(5, L), synth.w_like(6, L)
    w1, v1 = oracle.sgd_step(gs, w0, v0, synth.PAPER_LR, synth.PAPER_MOM)
    g_d = [to_dev(g) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, synth.PAPER_LR, synth.PAPER_MOM)
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(w_d[r]), w1, "f32", what=f"w rank {r}")
        off, ln = gdraa.gdraa_shard(N, r, L)
        compare(from_dev(v_d[r])[off:off + ln], v1[off:off + ln], "f32", what=f"v rank {r}")


# ---------------------------------------------------------------------------------------
# The multi-process ABI at world = 1 (init / register / sgd_step / allreduce / stats).
# ---------------------------------------------------------------------------------------

@pytest.fixture
def world1():
    gdraa.gdraa_init(1, 0)
    yield
    gdraa.gdraa_finalize()


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_world1_sgd_and_mean(world1, dt):
    bf16 = dt == "bf16"
    L = synth.L_R50
    gs = make_grads("like", 8, 1, L, bf16)
    w0, v0 = synth.w_like(8, L), synth.w_like(9, L)
    g = to_dev(gs[0], bf16)
    w, v = to_dev(w0), to_dev(v0)
    gdraa.gdraa_register(w)
    gdraa.gdraa_register(g)
    for it in range(3):
        w0, v0 = oracle.sgd_step(gs, w0, v0, synth.PAPER_LR, synth.PAPER_MOM)
        gdraa.gdraa_sgd_step(w, g, v, synth.PAPER_LR, synth.PAPER_MOM)
    torch.cuda.synchronize()
    compare(from_dev(w), w0, "f32", what="w")
    compare(from_dev(v), v0, "f32", what="v")
    gdraa.gdraa_allreduce_mean(g)         # N = 1: identity, bit for bit
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(g), gs[0])
    st = gdraa.gdraa_get_stats()
    assert st["calls"] == 4 and st["launches"] == 4 and st["sync_waits"] == 0, st


def test_world1_bucketed_ranges(world1):
    """NEXT-3 range calls at world 1: buckets stepped out of order equal one full step."""
    L = 300_008
    gs = make_grads("like", 12, 1, L, False)
    w0, v0 = synth.w_like(12, L), synth.w_like(13, L)
    w_exp, v_exp = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
    g, w, v = to_dev(gs[0]), to_dev(w0), to_dev(v0)
    gdraa.gdraa_register(w)
    gdraa.gdraa_register(g)
    for first, count in [(200_000, 100_008), (8, 199_992), (0, 8)]:
        gdraa.gdraa_sgd_step_range(w, g, v, first, count, 0.1, 0.9, 0.001)
    torch.cuda.synchronize()
    compare(from_dev(w), w_exp, "f32", what="w")
    compare(from_dev(v), v_exp, "f32", what="v")
    for bad in [(1, 10), (4, 10), (0, 0), (300_000, 9), (400_000, 8)]:
        with pytest.raises(gdraa.GdraaError) as e:
            gdraa.gdraa_sgd_step_range(w, g, v, bad[0], bad[1], 0.1, 0.9)
        assert e.value.name == "GDRAA_EINVAL", bad


def test_world1_iter_done_flag(world1):
    """a0 at world 1: the kernel's last CTA writes IterDone into the go/done page
    after every call, through both the two-shot/local and the mean kernels."""
    L = 70_001
    g = to_dev(synth.grad_like(14, 0, L))
    w, v = to_dev(synth.w_like(14, L)), torch.zeros(L, device=DEV)
    gdraa.gdraa_register(w)
    gdraa.gdraa_register(g)
    for k in range(1, 6):
        gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9)
        if k % 2 == 0:
            gdraa.gdraa_allreduce_mean(g)
        st = gdraa.gdraa_get_stats()
        assert st["iter_done"] == st["calls"] == k + k // 2, st


def test_world1_calls_on_alternating_streams(world1):
    """Calls share the rank's pad (epoch, arrival and work counters): a call issued on
    another stream than the previous one must not overlap it on the device.  Two buffer
    sets stepped alternately on two streams with no user synchronisation equal the
    oracle (without the library's ordering the two grids would share one work counter)."""
    L = 3_000_017
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    sets = []
    for k in range(2):
        gs = make_grads("like", 90 + k, 1, L, False)
        w0, v0 = synth.w_like(90 + k, L), np.zeros(L, np.float32)
        g, w, v = to_dev(gs[0]), to_dev(w0), to_dev(v0)
        gdraa.gdraa_register(w)
        gdraa.gdraa_register(g)
        sets.append([gs, w0, v0, g, w, v])
    torch.cuda.synchronize()
    for it in range(6):
        for k, st in enumerate(sets):
            gs, w0, v0, g, w, v = st
            gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9, stream=(s1, s2)[(it + k) % 2])
            st[1], st[2] = oracle.sgd_step(gs, w0, v0, 0.1, 0.9)
    torch.cuda.synchronize()
    for k, (gs, w0, v0, g, w, v) in enumerate(sets):
        compare(from_dev(w), w0, "f32", what=f"set {k} w")
        compare(from_dev(v), v0, "f32", what=f"set {k} v")
    assert gdraa.gdraa_get_stats()["iter_done"] == 12


def test_world1_errors(world1):
    a = torch.zeros(1000, device=DEV)
    b = torch.zeros(1000, device=DEV)
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_sgd_step(a, b, a, 0.1, 0.9)
    assert e.value.name == "GDRAA_ENOTREG"
    gdraa.gdraa_register(a)
    gdraa.gdraa_register(b)
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_sgd_step(a, b, a, float("nan"), 0.9)
    assert e.value.name == "GDRAA_EINVAL"
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_register(a)
    assert e.value.name == "GDRAA_EINVAL"
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_register(a[1:], 999, gdraa.GDRAA_F32)       # misaligned
    assert e.value.name == "GDRAA_EINVAL"
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_init(1, 0)
    assert e.value.name == "GDRAA_ESTATE"
    c = torch.zeros(999, device=DEV)
    gdraa.gdraa_register(c)
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_sgd_step(a, c, b, 0.1, 0.9)                  # length mismatch
    assert e.value.name == "GDRAA_EINVAL"


def test_graph_capture_replays():
    """The epoch lives in device memory, so a captured step replays correctly."""
    N, L = 2, 100_003
    gs = make_grads("like", 21, N, L, False)
    w0, v0 = synth.w_like(21, L), np.zeros(L, np.float32)
    g_d = [to_dev(g) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    s = torch.cuda.Stream()
    gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, 0.1, 0.9, stream=s)   # warm up (pads allocated)
    s.synchronize()
    w_ref, v_ref = oracle.sgd_step(gs, w0, v0, 0.1, 0.9)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, 0.1, 0.9, stream=s)
    for _ in range(3):
        graph.replay()
        w_ref, v_ref = oracle.sgd_step(gs, w_ref, v_ref, 0.1, 0.9)
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(w_d[r]), w_ref, "f32", what=f"graph w rank {r}")


@pytest.mark.parametrize("N", [2, 4])
def test_graph_capture_bucket_set(N):
    """A bucket set (per-call kernels with the deferred exit, and the exit kernel)
    captured once into a CUDA graph and replayed as three chained iterations; a streamed
    set refuses capture (EINVAL)."""
    L = 1_500_007
    buckets = _buckets(L)
    gs = make_grads("like", 31 + N, N, L, False)
    w0, v0 = synth.w_like(31 + N, L), synth.w_like(32 + N, L)
    g_d = [to_dev(g) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    s = torch.cuda.Stream()

    def one_iteration():
        gdraa.gdraa_vr_bucket_set_begin(N)
        for first, count in buckets:
            gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, first, count, 0.1, 0.9, 0.001, stream=s)
        gdraa.gdraa_vr_bucket_set_end(N, stream=s)

    w_ref, v_ref = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
    one_iteration()                                   # warm up (pads, LL slots allocated)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        one_iteration()
    for _ in range(3):
        graph.replay()
        w_ref, v_ref = oracle.sgd_step_wd(gs, w_ref, v_ref, 0.1, 0.9, 0.001)
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(w_d[r]), w_ref, "f32", what=f"graph bucket set w N={N} r{r}")
    gdraa.gdraa_vr_bucket_set_begin_streamed(N, 8)   # (its device state exists before
    gdraa.gdraa_vr_bucket_set_end(N, stream=s)         #  the capture below)
    s.synchronize()
    with pytest.raises(gdraa.GdraaError) as e:
        with torch.cuda.graph(torch.cuda.CUDAGraph(), stream=s):
            gdraa.gdraa_vr_bucket_set_begin_streamed(N, 8)
            try:
                gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, 0, 1024, 0.1, 0.9, 0.0, stream=s)
            finally:
                gdraa.gdraa_vr_bucket_set_end(N, stream=s)
    assert e.value.name == "GDRAA_EINVAL" and "captured" in str(e.value)


# ---------------------------------------------------------------------------------------
# NEXT-1: weight decay and the mixed-precision (bf16 model copy) all-gather.
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("family", ["int", "like"])
def test_vr_sgd_step_ex_weight_decay(N, dt, family):
    bf16 = dt == "bf16"
    wd = 2.0**-4 if family == "int" else 0.001          # weight decay 0.001
    for L in (1, 257, 70_001, 1 << 20):
        gs = make_grads(family, 400 + N, N, L, bf16)
        w0, v0, lr, mom = make_wv(family, 400 + N, L)
        w_exp, v_exp = oracle.sgd_step_wd(gs, w0, v0, lr, mom, wd)
        g_d = [to_dev(g, bf16) for g in gs]
        w_d = [to_dev(w0) for _ in range(N)]
        v_d = [to_dev(v0) for _ in range(N)]
        gdraa.gdraa_vr_sgd_step_ex(w_d, g_d, v_d, lr, mom, wd)
        torch.cuda.synchronize()
        for r in range(N):
            compare(from_dev(w_d[r]), w_exp, "f32", what=f"w N={N} L={L} rank {r}")
            off, ln = gdraa.gdraa_shard(N, r, L)
            compare(from_dev(v_d[r])[off:off + ln], v_exp[off:off + ln], "f32", what=f"v r{r}")


@pytest.mark.parametrize("N", [1, 2, 4, 5, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_vr_sgd_step_mp(N, dt):
    """fp32 master sharded like v; every rank receives bf16 RNE(w') of every shard."""
    bf16 = dt == "bf16"
    for L in (1, 5, 1000, 70_001, 1 << 20):
        gs = make_grads("like", 500 + N, N, L, bf16)
        w0, v0 = synth.w_like(500 + N, L), synth.w_like(600 + N, L)
        w_exp, v_exp, model_exp = oracle.sgd_step_wd(gs, w0, v0, synth.PAPER_LR,
                                                     synth.PAPER_MOM, 0.001,
                                                     model_dtype=oracle.BF16)
        g_d = [to_dev(g, bf16) for g in gs]
        wm_d = [to_dev(w0) for _ in range(N)]
        v_d = [to_dev(v0) for _ in range(N)]
        model_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
        gdraa.gdraa_vr_sgd_step_mp(wm_d, model_d, g_d, v_d, synth.PAPER_LR, synth.PAPER_MOM,
                                   0.001)
        torch.cuda.synchronize()
        for r in range(N):
            compare(from_dev(model_d[r]), model_exp, "bf16", what=f"model N={N} L={L} r{r}")
            off, ln = gdraa.gdraa_shard(N, r, L)
            wm = from_dev(wm_d[r])
            compare(wm[off:off + ln], w_exp[off:off + ln], "f32", what=f"master r{r}")
            compare(from_dev(v_d[r])[off:off + ln], v_exp[off:off + ln], "f32", what=f"v r{r}")
            keep = np.ones(L, bool)
            keep[off:off + ln] = False
            assert np.array_equal(wm[keep].view(np.uint32), w0[keep].view(np.uint32))


# ---------------------------------------------------------------------------------------
# NEXT-3 across virtual ranks: buckets in backward (out-of-order) order, each with its own
# owner partition, equal the whole-buffer oracle step.
# ---------------------------------------------------------------------------------------

def _buckets(L):
    """Out-of-order buckets covering [0, L): starts multiples of 8, ragged sizes, one
    bucket smaller than the world (empty shards), one above the small-message limit."""
    cuts = sorted({0, 8, 64, 4104, L // 3 // 8 * 8, (L // 2 + 5) // 8 * 8, L})
    spans = [(a, b - a) for a, b in zip(cuts, cuts[1:]) if b > a]
    return spans[::-1]


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_vr_bucketed_ranges(N, dt):
    bf16 = dt == "bf16"
    L = 5_000_017
    buckets = _buckets(L)
    lim = gdraa.gdraa_small_step_bytes(N, gdraa.GDRAA_BF16 if bf16 else gdraa.GDRAA_F32)
    sizes = [c * (2 if bf16 else 4) for _, c in buckets]
    assert min(sizes) <= lim < max(sizes)           # both the LL and the two-shot kernel
    gs = make_grads("like", 700 + N, N, L, bf16)
    w0, v0 = synth.w_like(700 + N, L), synth.w_like(800 + N, L)
    wd = 0.001
    w_exp, v_exp = oracle.sgd_step_wd(gs, w0, v0, synth.PAPER_LR, synth.PAPER_MOM, wd)
    g_d = [to_dev(g, bf16) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    for first, count in buckets:
        gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, first, count, synth.PAPER_LR,
                                      synth.PAPER_MOM, wd)
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(w_d[r]), w_exp, "f32", what=f"bucketed w N={N} r{r}")
        vh, vmask = from_dev(v_d[r]), np.zeros(L, bool)
        for first, count in buckets:            # the owner rule applies per range
            off, ln = gdraa.gdraa_shard(N, r, count)
            vmask[first + off:first + off + ln] = True
        compare(vh[vmask], v_exp[vmask], "f32", what=f"bucketed v N={N} r{r}")
        assert np.array_equal(vh[~vmask].view(np.uint32), v0[~vmask].view(np.uint32))
    # the mixed-precision form on the same buckets
    w_exp2, v_exp2, m_exp = oracle.sgd_step_wd(gs, w0, v0, synth.PAPER_LR, synth.PAPER_MOM,
                                               wd, model_dtype=oracle.BF16)
    wm_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    model_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
    for first, count in buckets:
        gdraa.gdraa_vr_sgd_step_mp_range(wm_d, model_d, g_d, v_d, first, count, synth.PAPER_LR,
                                         synth.PAPER_MOM, wd)
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(model_d[r]), m_exp, "bf16", what=f"bucketed mp model N={N} r{r}")
        wm, vmask = from_dev(wm_d[r]), np.zeros(L, bool)
        for first, count in buckets:
            off, ln = gdraa.gdraa_shard(N, r, count)
            vmask[first + off:first + off + ln] = True
        compare(wm[vmask], w_exp2[vmask], "f32", what=f"bucketed mp master N={N} r{r}")
        compare(from_dev(v_d[r])[vmask], v_exp2[vmask], "f32", what=f"bucketed mp v r{r}")
    # allreduce_mean on the same buckets
    bufs = [to_dev(g, bf16) for g in gs]
    for first, count in buckets:
        gdraa.gdraa_vr_allreduce_mean_range(bufs, first, count)
    torch.cuda.synchronize()
    m_exp = oracle.allreduce_mean(gs)
    for r in range(N):
        compare(from_dev(bufs[r]), m_exp, dt, what=f"bucketed mean N={N} r{r}")


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_vr_bucket_set(N, dt):
    """NEXT-3 "two syncs per bucket-set": the same out-of-order buckets inside one bucket
    set -- every two-shot call skips its exit barrier, gdraa_vr_bucket_set_end runs one
    for all of them -- give the whole-buffer oracle step, for sgd, the mixed-precision
    step and the mean (three destination buffers in the same set, LL and two-shot calls
    mixed), and a second set right after the first sees the first set's results."""
    bf16 = dt == "bf16"
    L = 5_000_017
    buckets = _buckets(L)
    gs = make_grads("like", 900 + N, N, L, bf16)
    w0, v0 = synth.w_like(900 + N, L), synth.w_like(950 + N, L)
    wd, lr, mom = 0.001, synth.PAPER_LR, synth.PAPER_MOM
    w1, v1 = oracle.sgd_step_wd(gs, w0, v0, lr, mom, wd)
    w2, v2 = oracle.sgd_step_wd(gs, w1, v1, lr, mom, wd)
    wm_exp, vm_exp, m_exp = oracle.sgd_step_wd(gs, w0, v0, lr, mom, wd, model_dtype=oracle.BF16)
    mean_exp = oracle.allreduce_mean(gs)
    g_d = [to_dev(g, bf16) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    wm_d = [to_dev(w0) for _ in range(N)]
    vm_d = [to_dev(v0) for _ in range(N)]
    model_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
    bufs = [to_dev(g, bf16) for g in gs]
    for it in range(2):                  # two iterations = two sets, chained through w, v
        gdraa.gdraa_vr_bucket_set_begin(N)
        for first, count in buckets:
            gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, first, count, lr, mom, wd)
            if it == 0:
                gdraa.gdraa_vr_sgd_step_mp_range(wm_d, model_d, g_d, vm_d, first, count, lr,
                                                 mom, wd)
                gdraa.gdraa_vr_allreduce_mean_range(bufs, first, count)
        gdraa.gdraa_vr_bucket_set_end(N)
        if it == 0:
            torch.cuda.synchronize()
            for r in range(N):
                compare(from_dev(w_d[r]), w1, "f32", what=f"set w it0 N={N} r{r}")
                compare(from_dev(model_d[r]), m_exp, "bf16", what=f"set mp model N={N} r{r}")
                compare(from_dev(bufs[r]), mean_exp, dt, what=f"set mean N={N} r{r}")
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(w_d[r]), w2, "f32", what=f"set w it1 N={N} r{r}")
        vh, wmh, vmh, vmask = from_dev(v_d[r]), from_dev(wm_d[r]), from_dev(vm_d[r]), np.zeros(L, bool)
        for first, count in buckets:
            off, ln = gdraa.gdraa_shard(N, r, count)
            vmask[first + off:first + off + ln] = True
        compare(vh[vmask], v2[vmask], "f32", what=f"set v N={N} r{r}")
        compare(wmh[vmask], wm_exp[vmask], "f32", what=f"set mp master N={N} r{r}")
        compare(vmh[vmask], vm_exp[vmask], "f32", what=f"set mp v N={N} r{r}")


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("ctas", [4, 32])
def test_vr_bucket_set_streamed(N, dt, ctas):
    """Streamed bucket sets: one persistent kernel serves every bucket of the set (bucket
    descriptions arrive by stream memory operations); out-of-order ragged buckets, one
    of them smaller than the world; two chained sgd sets, then an mp set and a mean set --
    the whole-buffer oracle's bits."""
    bf16 = dt == "bf16"
    L = 3_000_017
    buckets = _buckets(L)
    gs = make_grads("like", 960 + N, N, L, bf16)
    w0, v0 = synth.w_like(960 + N, L), synth.w_like(970 + N, L)
    wd, lr, mom = 0.001, synth.PAPER_LR, synth.PAPER_MOM
    w1, v1 = oracle.sgd_step_wd(gs, w0, v0, lr, mom, wd)
    w2, v2 = oracle.sgd_step_wd(gs, w1, v1, lr, mom, wd)
    wm_exp, vm_exp, m_exp = oracle.sgd_step_wd(gs, w0, v0, lr, mom, wd, model_dtype=oracle.BF16)
    g_d = [to_dev(g, bf16) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    for it in range(2):
        gdraa.gdraa_vr_bucket_set_begin_streamed(N, ctas)
        for first, count in buckets:
            gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, first, count, lr, mom, wd)
        gdraa.gdraa_vr_bucket_set_end(N)
        if it == 0:
            torch.cuda.synchronize()
            for r in range(N):
                compare(from_dev(w_d[r]), w1, "f32", what=f"streamed w it0 N={N} r{r}")
    wm_d = [to_dev(w0) for _ in range(N)]
    vm_d = [to_dev(v0) for _ in range(N)]
    model_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
    gdraa.gdraa_vr_bucket_set_begin_streamed(N, ctas)
    for first, count in buckets:
        gdraa.gdraa_vr_sgd_step_mp_range(wm_d, model_d, g_d, vm_d, first, count, lr, mom, wd)
    gdraa.gdraa_vr_bucket_set_end(N)
    bufs = [to_dev(g, bf16) for g in gs]
    gdraa.gdraa_vr_bucket_set_begin_streamed(N, ctas)
    for first, count in buckets:
        gdraa.gdraa_vr_allreduce_mean_range(bufs, first, count)
    gdraa.gdraa_vr_bucket_set_end(N)
    torch.cuda.synchronize()
    mean_exp = oracle.allreduce_mean(gs)
    for r in range(N):
        compare(from_dev(w_d[r]), w2, "f32", what=f"streamed w it1 N={N} r{r}")
        compare(from_dev(model_d[r]), m_exp, "bf16", what=f"streamed mp model N={N} r{r}")
        compare(from_dev(bufs[r]), mean_exp, dt, what=f"streamed mean N={N} r{r}")
        vh, wmh, vmh, vmask = from_dev(v_d[r]), from_dev(wm_d[r]), from_dev(vm_d[r]), np.zeros(L, bool)
        for first, count in buckets:
            off, ln = gdraa.gdraa_shard(N, r, count)
            vmask[first + off:first + off + ln] = True
        compare(vh[vmask], v2[vmask], "f32", what=f"streamed v N={N} r{r}")
        compare(wmh[vmask], wm_exp[vmask], "f32", what=f"streamed mp master N={N} r{r}")
        compare(vmh[vmask], vm_exp[vmask], "f32", what=f"streamed mp v N={N} r{r}")
        assert np.array_equal(vh[~vmask].view(np.uint32), v0[~vmask].view(np.uint32))


@pytest.mark.parametrize("N", [1, 2, 4])
@pytest.mark.parametrize("kind", ["set", "streamed"])
def test_vr_bucket_sets_two_streams(N, kind):
    """Bucket calls alternating between two streams inside one set (each bucket's stream
    waits for an event that marks its gradient final), the set closed on a third: the
    cross-stream ordering of the library makes it the whole-buffer oracle step.  N = 1:
    both kinds degenerate to plain calls."""
    L = 2_000_003
    buckets = _buckets(L)
    gs = make_grads("like", 990 + N, N, L, False)
    w0, v0 = synth.w_like(990 + N, L), synth.w_like(995 + N, L)
    w_exp, v_exp = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
    g_d = [to_dev(g) for g in gs]
    w_d = [to_dev(w0) for _ in range(N)]
    v_d = [to_dev(v0) for _ in range(N)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    closer = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    if kind == "set":
        gdraa.gdraa_vr_bucket_set_begin(N)
    else:
        gdraa.gdraa_vr_bucket_set_begin_streamed(N, 32)
    for k, (first, count) in enumerate(buckets):
        ev = torch.cuda.Event()
        ev.record(main)
        st = streams[k % 2]
        st.wait_event(ev)
        gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, first, count, 0.1, 0.9, 0.001, stream=st)
    for st in streams:
        closer.wait_stream(st)
    gdraa.gdraa_vr_bucket_set_end(N, stream=closer)
    main.wait_stream(closer)
    torch.cuda.synchronize()
    for r in range(N):
        compare(from_dev(w_d[r]), w_exp, "f32", what=f"{kind} two streams w N={N} r{r}")
        vh, vmask = from_dev(v_d[r]), np.zeros(L, bool)
        for first, count in buckets:
            off, ln = gdraa.gdraa_shard(N, r, count)
            vmask[first + off:first + off + ln] = True
        compare(vh[vmask], v_exp[vmask], "f32", what=f"{kind} two streams v N={N} r{r}")


def test_vr_bucket_set_streamed_rules():
    """A streamed set serves one buffer set, mode and hyper-parameter set."""
    N, L = 2, 1 << 16
    w = [torch.zeros(L, device=DEV) for _ in range(N)]
    w2 = [torch.zeros(L, device=DEV) for _ in range(N)]
    g = [torch.ones(L, device=DEV) for _ in range(N)]
    v = [torch.zeros(L, device=DEV) for _ in range(N)]
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_vr_bucket_set_begin_streamed(N, 0)
    assert e.value.name == "GDRAA_EINVAL"
    gdraa.gdraa_vr_bucket_set_begin_streamed(N, 8)
    gdraa.gdraa_vr_sgd_step_range(w, g, v, 0, 1024, 0.5, 0.0)
    for call in (lambda: gdraa.gdraa_vr_sgd_step_range(w, g, v, 1024, 1024, 0.25, 0.0),  # lr
                 lambda: gdraa.gdraa_vr_sgd_step_range(w2, g, v, 1024, 1024, 0.5, 0.0),  # w
                 lambda: gdraa.gdraa_vr_allreduce_mean_range(w, 1024, 1024)):             # mode
        with pytest.raises(gdraa.GdraaError) as e:
            call()
        assert e.value.name == "GDRAA_EINVAL"
    gdraa.gdraa_vr_sgd_step_range(w, g, v, 1024, L - 1024, 0.5, 0.0)
    gdraa.gdraa_vr_bucket_set_end(N)
    torch.cuda.synchronize()
    for r in range(N):
        assert torch.equal(w[r], torch.full((L,), -0.5, device=DEV))
    # an empty streamed set launches nothing and closes cleanly
    gdraa.gdraa_vr_bucket_set_begin_streamed(N, 8)
    gdraa.gdraa_vr_bucket_set_end(N)
    torch.cuda.synchronize()


def test_vr_bucket_set_rules():
    """Set state errors and the disjoint-destination rule inside a set."""
    N, L = 2, 1 << 16
    w = [torch.zeros(L, device=DEV) for _ in range(N)]
    g = [torch.ones(L, device=DEV) for _ in range(N)]
    v = [torch.zeros(L, device=DEV) for _ in range(N)]
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_vr_bucket_set_end(N)
    assert e.value.name == "GDRAA_ESTATE"
    for bad in (0, 9):
        with pytest.raises(gdraa.GdraaError) as e:
            gdraa.gdraa_vr_bucket_set_begin(bad)
        assert e.value.name == "GDRAA_EINVAL"
    gdraa.gdraa_vr_bucket_set_begin(N)
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_vr_bucket_set_begin(N)
    assert e.value.name == "GDRAA_ESTATE"
    gdraa.gdraa_vr_sgd_step_range(w, g, v, 0, 1024, 0.5, 0.0)
    with pytest.raises(gdraa.GdraaError) as e:       # overlaps [0, 1024) of the same w
        gdraa.gdraa_vr_sgd_step_range(w, g, v, 1016, 64, 0.5, 0.0)
    assert e.value.name == "GDRAA_EINVAL" and "overlaps" in str(e.value)
    gdraa.gdraa_vr_sgd_step_range(w, g, v, 1024, L - 1024, 0.5, 0.0)   # disjoint: fine
    gdraa.gdraa_vr_bucket_set_end(N)
    torch.cuda.synchronize()
    for r in range(N):                    # w = 0 - 0.5 * mean(1) everywhere, once
        assert torch.equal(w[r], torch.full((L,), -0.5, device=DEV))
    gdraa.gdraa_vr_sgd_step_range(w, g, v, 0, 1024, 0.5, 0.0)          # outside a set
    torch.cuda.synchronize()
    assert torch.equal(w[0][:1024], torch.full((1024,), -1.0, device=DEV))


def test_vr_range_rejects_bad_ranges():
    N, L = 2, 1000
    w = [torch.zeros(L, device=DEV) for _ in range(N)]
    g = [torch.zeros(L, device=DEV) for _ in range(N)]
    v = [torch.zeros(L, device=DEV) for _ in range(N)]
    for bad in [(1, 10), (4, 10), (0, 0), (992, 9), (1000, 8)]:
        with pytest.raises(gdraa.GdraaError) as e:
            gdraa.gdraa_vr_sgd_step_range(w, g, v, bad[0], bad[1], 0.1, 0.9)
        assert e.value.name == "GDRAA_EINVAL", bad


# ---------------------------------------------------------------------------------------
# Randomised call sequences: every entry point, sizes on both sides of every threshold,
# chained state, one persistent set of pads / LL slots per world size.
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("N", [3, 8])
def test_vr_random_call_sequence(N):
    rng = np.random.default_rng(1000 + N)
    lim = gdraa.gdraa_small_step_bytes(N) // 4
    sizes = [1, 7, 64, 1000, lim - 1, lim + 1, 3 * lim + 5, 1_000_003]
    for step in range(14):
        L = int(rng.choice(sizes))
        kind = rng.choice(["mean", "sgd", "ex", "mp", "range"])
        bf16 = bool(rng.integers(0, 2))
        gs = make_grads("like", 2000 + 17 * step + N, N, L, bf16)
        g_d = [to_dev(g, bf16) for g in gs]
        what = f"step {step} {kind} N={N} L={L} bf16={bf16}"
        if kind == "mean":
            gdraa.gdraa_vr_allreduce_mean(g_d)
            torch.cuda.synchronize()
            exp = oracle.allreduce_mean(gs)
            for r in range(N):
                compare(from_dev(g_d[r]), exp, "bf16" if bf16 else "f32", what=f"{what} r{r}")
            continue
        w0, v0 = synth.w_like(3000 + step, L), synth.w_like(4000 + step, L)
        v_d = [to_dev(v0) for _ in range(N)]
        if kind == "mp":
            wm_d = [to_dev(w0) for _ in range(N)]
            mo_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
            gdraa.gdraa_vr_sgd_step_mp(wm_d, mo_d, g_d, v_d, 0.1, 0.9, 0.001)
            we, ve, me = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001, model_dtype=oracle.BF16)
            torch.cuda.synchronize()
            for r in range(N):
                compare(from_dev(mo_d[r]), me, "bf16", what=f"{what} model r{r}")
            continue
        w_d = [to_dev(w0) for _ in range(N)]
        wd = 0.0 if kind == "sgd" else 0.001
        if kind == "range" and L >= 16:
            cut = (L // 2) // 8 * 8
            for first, count in ((cut, L - cut), (0, cut)):
                gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, first, count, 0.1, 0.9, wd)
        elif kind == "sgd":
            gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, 0.1, 0.9)
        else:
            gdraa.gdraa_vr_sgd_step_ex(w_d, g_d, v_d, 0.1, 0.9, wd)
        we, ve = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, wd)
        torch.cuda.synchronize()
        for r in range(N):
            compare(from_dev(w_d[r]), we, "f32", what=f"{what} w r{r}")


# ---------------------------------------------------------------------------------------
# Maximum sizes: a buffer past 2^32 bytes (64-bit indexing of elements, chunks and byte
# offsets), inputs built on the device from an integer formula the host can recompute on
# any window, compared with the oracle on windows at the start, at every 2^31- and
# 2^32-byte boundary, at the shard boundary and at the ragged end.
# ---------------------------------------------------------------------------------------

def _int_formula(i, p, lo, span, salt):
    """Integer values in [lo, lo + span) from index i (int64 array / tensor) and rank p,
    exactly representable in fp32 (|value| < 2^24); identical on host and device."""
    return ((i * 2654435761 + (p + 1) * 40503 + salt) >> 7) % span + lo


def _fill_device(L, p, lo, span, salt, dev=DEV, chunk=1 << 26):
    out = torch.empty(L, dtype=torch.float32, device=dev)
    for a in range(0, L, chunk):
        i = torch.arange(a, min(L, a + chunk), dtype=torch.int64, device=dev)
        out[a:a + i.numel()] = _int_formula(i, p, lo, span, salt).to(torch.float32)
    return out


def test_vr_max_size_64bit_indexing():
    N = 2
    L = (1 << 30) + 9                       # 4 GiB + 36 B of fp32 per buffer
    free, _ = torch.cuda.mem_get_info()
    if free < 3 * N * L * 4 + (4 << 30):
        pytest.skip("not enough device memory")
    # integer family (exact for N a power of two): g in [-2^13, 2^13), w in [-2^12, 2^12),
    # v in [-2^10, 2^10), lr = 2^-3, mom = 2^-1
    g_d = [_fill_device(L, p, -(1 << 13), 1 << 14, 11) for p in range(N)]
    w_d = [_fill_device(L, 0, -(1 << 12), 1 << 13, 22) for _ in range(N)]
    v_d = [_fill_device(L, 0, -(1 << 10), 1 << 11, 33) for _ in range(N)]
    gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, synth.INT_LR, synth.INT_MOM)
    torch.cuda.synchronize()
    off1, _ = gdraa.gdraa_shard(N, 1, L)
    W = 4096
    starts = sorted({0, (1 << 29) - W // 2, (1 << 30) - W, off1 - W // 2, L - W,
                     (1 << 28) - W // 2, 3 * (1 << 28) - W // 2})
    for a in starts:
        i = np.arange(a, a + W, dtype=np.int64)
        gs = [_int_formula(i, p, -(1 << 13), 1 << 14, 11).astype(np.float32) for p in range(N)]
        w0 = _int_formula(i, 0, -(1 << 12), 1 << 13, 22).astype(np.float32)
        v0 = _int_formula(i, 0, -(1 << 10), 1 << 11, 33).astype(np.float32)
        we, ve = oracle.sgd_step(gs, w0, v0, synth.INT_LR, synth.INT_MOM)
        for r in range(N):
            compare(from_dev(w_d[r][a:a + W]), we, "f32", what=f"max-size w @{a} r{r}")
            off, ln = gdraa.gdraa_shard(N, r, L)
            lo, hi = max(a, off), min(a + W, off + ln)
            if lo < hi:
                compare(from_dev(v_d[r][lo:hi]), ve[lo - a:hi - a], "f32", what=f"v @{a} r{r}")


def test_vr_calls_on_alternating_streams():
    """Virtual-rank calls share one set of pads per world size: calls alternating between
    two streams without user synchronisation must still run one after the other."""
    N, L = 4, 2_000_003
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    sets = []
    for k in range(2):
        gs = make_grads("like", 95 + k, N, L, False)
        w0, v0 = synth.w_like(95 + k, L), np.zeros(L, np.float32)
        sets.append([gs, w0, v0, [to_dev(g) for g in gs], [to_dev(w0) for _ in range(N)],
                     [to_dev(v0) for _ in range(N)]])
    torch.cuda.synchronize()
    for it in range(4):
        for k, st in enumerate(sets):
            gs, w0, v0, g_d, w_d, v_d = st
            gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, 0.1, 0.9, stream=(s1, s2)[(it + k) % 2])
            st[1], st[2] = oracle.sgd_step(gs, w0, v0, 0.1, 0.9)
    torch.cuda.synchronize()
    for k, (gs, w0, v0, g_d, w_d, v_d) in enumerate(sets):
        for r in range(N):
            compare(from_dev(w_d[r]), w0, "f32", what=f"set {k} w r{r}")
