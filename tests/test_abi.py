"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/gdraa.h declares, carries sm_100a SASS, and its host logic (the partition, the
argument checks that precede any CUDA call) behaves as documented."""
import os
import re
import subprocess

import pytest

import oracle
import synth
from paper_1802_02326_b200 import gdraa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gdraa.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gdraa_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert "gdraa_sgd_step" in syms and "gdraa_allreduce_mean" in syms
    out = subprocess.run(["nm", "-D", "--defined-only", gdraa.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gdraa_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(gdraa.EXPORTED) == syms


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gdraa.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out, out
    assert "sm_100a" in gdraa.gdraa_version()


def test_no_oracle_in_product():
    """The product never links or imports the oracle (and vice versa)."""
    out = subprocess.run(["nm", "-D", gdraa.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle_" not in out
    pkg = os.path.join(ROOT, "paper_1802_02326_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gdraa_oracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_1802_02326_b200", txt, re.M), f
            assert not re.search(r'#include\s+"gdraa(_internal)?\.h"', txt), f


@pytest.mark.parametrize("N", range(1, 9))
def test_shard_matches_oracle_partition(N):
    for L in (1, 2, 63, 64, 65, 1000, 4096 * N + 7, 1 << 20, synth.L_R50, synth.L_R101):
        for r in range(N):
            assert gdraa.gdraa_shard(N, r, L) == oracle.partition(L, N, r, Q=64)


def test_shard_alignment():
    for N in range(1, 9):
        for r in range(N):
            off, ln = gdraa.gdraa_shard(N, r, synth.L_R50)
            assert off % gdraa.GDRAA_SHARD_QUANTUM == 0


@pytest.mark.parametrize("args", [(0, 0, 10), (9, 0, 10), (2, 2, 10), (2, -1, 10), (2, 0, 0)])
def test_shard_rejects(args):
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_shard(*args)
    assert e.value.name == "GDRAA_EINVAL"


def test_calls_before_init_fail_cleanly():
    for fn, args in [(gdraa.gdraa_register, (1 << 20, 10, 0)), (gdraa.gdraa_get_stats, ()),
                     (gdraa.gdraa_finalize, ()), (gdraa.gdraa_deregister, (1 << 20,)),
                     (gdraa.gdraa_bucket_set_begin, ()), (gdraa.gdraa_bucket_set_end, (0,))]:
        with pytest.raises(gdraa.GdraaError) as e:
            fn(*args)
        assert e.value.name == "GDRAA_ESTATE", fn
    assert "gdraa_init" in gdraa.gdraa_last_error()


@pytest.mark.parametrize("world", [0, 9, -1])
def test_vr_bucket_set_rejects_world(world):
    """World is checked before any device work (no GPU needed)."""
    for fn, args in [(gdraa.gdraa_vr_bucket_set_begin, (world,)),
                     (gdraa.gdraa_vr_bucket_set_end, (world, 0))]:
        with pytest.raises(gdraa.GdraaError) as e:
            fn(*args)
        assert e.value.name == "GDRAA_EINVAL", fn


def test_failed_init_leaves_clean_state():
    """Without a usable GPU gdraa_init fails with ECUDA; it must not leave a half-built
    state behind: a retry fails the same way (not ESTATE) and no call sees a communicator."""
    from tests.conftest import has_cuda
    if has_cuda():
        pytest.skip("needs a machine without a GPU")
    for _ in range(2):
        with pytest.raises(gdraa.GdraaError) as e:
            gdraa.gdraa_init(1, 0)
        assert e.value.name == "GDRAA_ECUDA"
    with pytest.raises(gdraa.GdraaError) as e:
        gdraa.gdraa_get_stats()
    assert e.value.name == "GDRAA_ESTATE"


def test_binding_refuses_host_and_strided_tensors():
    import torch
    with pytest.raises(ValueError, match="CUDA"):
        gdraa.gdraa_sgd_step(torch.zeros(8), torch.zeros(8), torch.zeros(8), 0.1, 0.9, 0)
    with pytest.raises(ValueError):
        gdraa.gdraa_allreduce_mean(torch.zeros(16)[::2], 0)
    with pytest.raises(ValueError, match="differ in length"):
        gdraa.gdraa_vr_sgd_step([torch.zeros(8)] * 2, [torch.zeros(8), torch.zeros(4)],
                                [torch.zeros(8)] * 2, 0.1, 0.9, 0)


def test_poly_lr_matches_oracle(golden):
    ex = golden["poly_lr"][0]
    assert gdraa.gdraa_poly_lr(ex["lr0"], ex["iter"], ex["max_iter"], ex["power"]) == \
        oracle.poly_lr(ex["lr0"], ex["iter"], ex["max_iter"], ex["power"])
    for it in range(0, 5000, 37):
        for power in (0.5, 1.0, 2.0):
            assert gdraa.gdraa_poly_lr(0.1, it, 4999, power) == oracle.poly_lr(0.1, it, 4999, power)
    assert gdraa.gdraa_poly_lr(0.1, 1, 0, 1.0) == -1.0


def test_small_message_threshold():
    """NEXT-2 latency-path threshold: 4 MiB / (N-1), 8-byte multiple, none at N=1."""
    assert gdraa.gdraa_small_message_bytes(1) == 0
    for n in range(2, 9):
        lim = gdraa.gdraa_small_message_bytes(n)
        assert lim % 8 == 0 and (4 << 20) // (n - 1) - 8 < lim <= (4 << 20) // (n - 1)
    assert gdraa.gdraa_small_message_bytes(9) == 0


@pytest.mark.parametrize("mixed", [False, True])
def test_small_step_threshold(mixed):
    """Small-message SGD threshold: at most 4 MiB / (N-1) of gradient bytes, and the
    largest n whose padded shard (gradient + broadcast part) fits one sender's slot."""
    assert gdraa.gdraa_small_step_bytes(1) == 0 and gdraa.gdraa_small_step_bytes(9) == 0
    for N in range(2, 9):
        pairs = gdraa.gdraa_small_message_bytes(N) // 8
        for code, sg in ((gdraa.GDRAA_F32, 4), (gdraa.GDRAA_BF16, 2)):
            sw = 2 if mixed else 4
            lim = gdraa.gdraa_small_step_bytes(N, code, mixed)
            assert 0 < lim <= (4 << 20) // (N - 1) and lim % sg == 0

            def fits(n):
                blk = oracle.partition(n, N, 0, Q=64)[1]
                return (blk * sg + 7) // 8 + (blk * sw + 7) // 8 <= pairs

            n = lim // sg
            assert fits(n)
            assert n == (4 << 20) // (N - 1) // sg or not fits(n + 1)
