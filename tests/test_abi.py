"""CPU: the C-ABI library loads without a GPU and exports exactly what include/ckv.h declares;
host-side layout and shard planning."""

import ctypes
import re

import numpy as np
import pytest

from paper_2503_23294_b200 import _build, _lib
from paper_2503_23294_b200.batched import CHUNK, plan_layout
from paper_2503_23294_b200.distributed import batch_shard, sequence_shard_plan


def test_library_is_built_for_sm100a():
    _build.build()  # no-op when up to date
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = _lib.header_functions()
    assert len(names) >= 19
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib._SIGNATURES), "ctypes signatures out of sync with ckv.h"


def test_status_strings_and_version():
    lib = _lib.load()
    assert lib.ckv_abi_version() == 1
    assert b"bitwidth" in lib.ckv_status_string(_lib.CKV_ERR_BITS)
    with pytest.raises(ValueError):
        _lib.check(_lib.CKV_ERR_SHAPE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.CKV_ERR_CUDA)


def test_load_refuses_a_library_of_another_abi(monkeypatch):
    """_lib.load() checks ckv_abi_version() against the package's ABI_VERSION: a stale build
    fails loudly instead of being called with mismatched signatures."""
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "ABI_VERSION", _lib.ABI_VERSION + 1)
    with pytest.raises(RuntimeError, match="ABI"):
        _lib.load()


def test_argument_validation_without_gpu():
    lib = _lib.load()
    # validation happens before any launch, so these run on a CPU-only host
    assert lib.ckv_pack_codes(None, 4, 3, None, None) == _lib.CKV_ERR_BITS
    assert lib.ckv_unpack_codes(None, 1, 2, 17, None, None) == _lib.CKV_ERR_CAPACITY
    assert lib.ckv_quantize_groups_f64(None, 2, 2, 4, 0, None, None, None, None, None) == _lib.CKV_ERR_GROUP
    assert lib.ckv_matmul_packed_f64(None, 2, 5, 5, None, 6, None, None, 4, 6, 4, 3, 0, None, 6, 0,
                                     None) == _lib.CKV_ERR_SHAPE
    assert lib.ckv_search(None, None, None, None, None, 1, 4, 8, 1.5, 0.0, None, None, None, None,
                          None, None, None) == _lib.CKV_ERR_ARG
    ar = _lib.Arena()
    assert lib.ckv_decode_attention(ctypes.c_void_p(16), 0, 0, ar, ar, ctypes.c_void_p(16), 1, 1, 1, 9,
                                    0.1, 1, None, ctypes.c_void_p(16), 0, 0, None, 0, None) == _lib.CKV_ERR_UNSUPPORTED
    # zero-size work is a no-op success
    assert lib.ckv_pack_codes(None, 0, 2, None, None) == _lib.CKV_OK


def test_header_declares_reference_citations():
    text = open(_lib.HEADER_PATH).read()
    for cite in ("_core.pyx", "_numpy.py", "retrieval.py", "kv_store.py", "attention.py", "quantizer.py"):
        assert cite in text


def test_plan_layout_offsets_and_capacity():
    seq, cap = plan_layout([3, 1, 0], [1, 0, 0], [0, 2, 1], [4 * CHUNK + 5, 3 * CHUNK, CHUNK], 10)
    off2, len2, off4, len4, offf, lenf, tsrc, ctx = seq.T
    assert len2.tolist() == [96, 32, 0] and off2.tolist() == [0, 96, 128]
    assert len4.tolist() == [32, 0, 0] and off4.tolist() == [0, 32, 32]
    assert lenf.tolist() == [5, 64, 32]
    assert (cap % 16 == 0).all() and (cap >= lenf + 10).all()
    assert offf.tolist() == [0, cap[0], cap[0] + cap[1]]
    assert tsrc.tolist() == [128, 96, 32]
    with pytest.raises(ValueError):
        plan_layout([1], [0], [0], [CHUNK + CHUNK], 0)  # tail >= chunk


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sequence_shard_plan_partitions_every_tier(world):
    counts = np.array([[100, 13, 2], [7, 0, 1], [0, 0, 0], [1, 1, 1]])
    seen = [set() for _ in counts]
    for r in range(world):
        plan, owns_tail = sequence_shard_plan(counts, world, r)
        assert owns_tail == (r == world - 1)
        for b, (a2, b2, a4, b4, af, bf) in enumerate(plan):
            n2, n4, nf = counts[b]
            assert 0 <= a2 <= b2 <= n2 and n2 <= a4 <= b4 <= n2 + n4 and n2 + n4 <= af <= bf <= n2 + n4 + nf
            for lo, hi in ((a2, b2), (a4, b4), (af, bf)):
                rng = set(range(lo, hi))
                assert not (rng & seen[b])
                seen[b] |= rng
    for b, c in enumerate(counts):
        assert seen[b] == set(range(int(c.sum())))


def test_batch_shard_covers_batch():
    for world in (1, 2, 4, 8):
        spans = [batch_shard(64, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 64
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_sequence_shard_cache_layout_partitions_the_context(world):
    """Host planning of a sequence split-KV shard (no kernels): the ranks' caches hold every
    chunk of every tier exactly once (perm slots), the last rank also the tail and the decode
    capacity, and every rank's arena rows add up to the full cache's."""
    import torch
    from paper_2503_23294_b200.distributed import sequence_shard_cache
    from paper_2503_23294_b200.retrieval import SearchResult

    rng = np.random.default_rng(7)
    B, N, tail = 3, 45, 11
    tiers = rng.choice([0, 0, 0, 1, 2], size=(B, N)).astype(np.uint8)
    perm = np.zeros((B, N), np.int32)
    counts = np.zeros((B, 3), np.int32)
    for b in range(B):
        order = np.concatenate([np.nonzero(tiers[b] == t)[0] for t in range(3)])
        perm[b] = order
        counts[b] = np.bincount(tiers[b], minlength=3)
    z = torch.zeros
    s = SearchResult(z((B, N), dtype=torch.float64), z((B, 4), dtype=torch.float64),
                     torch.from_numpy(tiers), torch.from_numpy(perm), torch.from_numpy(counts),
                     z(B, dtype=torch.int32))
    ctx = np.full(B, N * 32 + tail)
    seen = [[] for _ in range(B)]
    rows = np.zeros(3, np.int64)
    for r in range(world):
        cache, perm_r = sequence_shard_cache(s, 2, 2, ctx, world, r, decode_capacity=8,
                                             device=torch.device("cpu"))
        sh = cache.seq_host
        rows += [cache.rows2, cache.rows4, int(sh[:, 5].sum())]
        for b in range(B):
            n_r = (sh[b, 1] + sh[b, 3]) // 32 + (sh[b, 5] - (tail if r == world - 1 else 0)) // 32
            seen[b] += perm_r[b, :n_r].tolist()
            assert (sh[b, 5] % 32 == tail % 32) if r == world - 1 else (sh[b, 5] % 32 == 0)
            assert (cache.cap_fp[b] >= sh[b, 5] + (8 if r == world - 1 else 0))
    for b in range(B):
        assert sorted(seen[b]) == list(range(N))
    assert rows.tolist() == [int(counts[:, 0].sum()) * 32, int(counts[:, 1].sum()) * 32,
                             int(counts[:, 2].sum()) * 32 + B * tail]


def test_product_path_fails_loudly_without_gpu_or_library():
    """No CPU fallback: without a visible CUDA device the public API raises instead of
    computing, and a missing libckv.so is an error at load time (not a silent substitute)."""
    import subprocess
    import sys

    import numpy as np
    import torch

    import paper_2503_23294_b200 as P

    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError, match="CUDA"):
            P.quantize(np.ones((2, 4)), 4, group_size=4)
        with pytest.raises(RuntimeError, match="CUDA"):
            P.HashedBowEncoder().encode("a b c")
    code = ("import os; os.environ['CKV_LIB_PATH'] = '/nonexistent/libckv.so'\n"
            "from paper_2503_23294_b200 import _lib\n"
            "try:\n    _lib.load()\nexcept RuntimeError as e:\n    print('raised', 'missing' in str(e))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=_build.ROOT)
    assert "raised True" in out.stdout, out.stdout + out.stderr
