"""GPU: the per-head drop-in API (kernels / quantizer / kv_store / attention) replayed the way
the reference's own tests exercise chunkkv, plus bit-identity against the reference's golden
vectors and the oracle.  Every call runs the sm_100a kernels in libckv.so."""

import struct

import numpy as np
import pytest

from oracle import ckv_oracle as O
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2503_23294_b200")
from paper_2503_23294_b200 import kernels as K  # noqa: E402
from paper_2503_23294_b200.attention import AttentionInstance, mixed_decode_attention, reference_attention, stable_softmax  # noqa: E402
from paper_2503_23294_b200.kv_store import (ChunkedKVCache, build_cache, cache_layout,  # noqa: E402
                                            deserialize_cache, memory_footprint, reconstruct,
                                            serialize_cache, token_order)
from paper_2503_23294_b200.quantizer import (QuantizedBlock, dequantize, deserialize_block, fqm,  # noqa: E402
                                             quantize, serialize_block)
from paper_2503_23294_b200.retrieval import segment_context  # noqa: E402
from paper_2503_23294_b200.tiers import Tier  # noqa: E402


def test_backend_is_the_cuda_library():
    assert K.BACKEND == "cuda-sm100a"


# -- kernels facade (test_kernels.py) ------------------------------------------------------

def test_pack_layout_frozen():
    assert K.pack_codes(np.array([1, 2, 3], np.uint8), 4).tolist() == [0x321]
    assert K.pack_codes(np.array([3, 0, 1, 2], np.uint8), 2).tolist() == [147]
    c = np.zeros(17, np.uint8)
    c[16] = 3
    assert K.pack_codes(c, 2).tolist() == [0, 3]


@pytest.mark.parametrize("bits", [2, 4])
def test_pack_unpack_bijection(bits):
    rng = np.random.default_rng(1)
    for n in list(range(1, 70)) + [100, 257, 1000]:
        codes = rng.integers(0, 2**bits, size=n).astype(np.uint8)
        packed = K.pack_codes(codes, bits)
        assert np.array_equal(packed, O.pack_codes(codes, bits))
        assert np.array_equal(K.unpack_codes(packed, bits, n), codes)


def test_kernel_errors():
    with pytest.raises(ValueError):
        K.pack_codes(np.zeros(4, np.uint8), 3)
    with pytest.raises(ValueError):
        K.unpack_codes(np.zeros(1, np.uint32), 8, 1)
    with pytest.raises(ValueError):
        K.unpack_codes(K.pack_codes(np.ones(16, np.uint8), 2), 2, 17)
    codes, scales, zps = K.quantize_groups(np.ones((4, 6)) * np.arange(6), 4, 3)
    packed = K.pack_codes(codes.reshape(-1), 4)
    with pytest.raises(ValueError):
        K.matmul_packed(np.ones((2, 5)), packed, scales, zps, 4, 6, 4, 3, False)


def test_quantize_bit_identical_to_reference_golden():
    g = load_golden("quantize.npz")
    for i in range(int(g["n"])):
        rows, cols, gs, bits = (int(x) for x in g[f"meta{i}"])
        codes, scales, zps = K.quantize_groups(g[f"x{i}"], bits, gs)
        assert np.array_equal(codes, g[f"codes{i}"]), i
        assert np.array_equal(scales.view(np.uint64), g[f"scales{i}"].view(np.uint64)), i
        assert np.array_equal(zps.view(np.uint64), g[f"zps{i}"].view(np.uint64)), i
        assert np.array_equal(K.pack_codes(codes.reshape(-1), bits), g[f"packed{i}"]), i
        deq = K.dequantize_codes(g[f"packed{i}"], scales, zps, rows, cols, bits, gs)
        want = O.dequantize_codes(g[f"packed{i}"], scales, zps, rows, cols, bits, gs)
        assert np.array_equal(deq.view(np.uint64), want.view(np.uint64)), i


def test_quantize_f16_input_matches_reference_golden():
    import torch
    g = load_golden("fp16_rows.npz")
    x = torch.from_numpy(g["x16"]).cuda()
    for bits in (2, 4):
        blk = quantize(x, bits, 32)  # fp16 device tensor -> f16 kernel
        assert np.array_equal(blk.packed, g[f"packed{bits}"])
        assert np.array_equal(blk.scales.view(np.uint64), g[f"scales{bits}"].view(np.uint64))
        assert np.array_equal(blk.zero_points.view(np.uint64), g[f"zps{bits}"].view(np.uint64))


@pytest.mark.parametrize("bits", [2, 4])
@pytest.mark.parametrize("transpose", [False, True])
def test_matmul_packed_close_to_oracle(bits, transpose):
    rng = np.random.default_rng(4)
    for rows, cols, gs, m in [(16, 16, 8, 1), (64, 32, 32, 3), (33, 17, 5, 2), (512, 128, 32, 4)]:
        x = rng.normal(size=(rows, cols))
        codes, scales, zps = O.quantize_groups(x, bits, gs)
        packed = O.pack_codes(codes.reshape(-1), bits)
        a = rng.normal(size=(m, cols if transpose else rows))
        want = O.matmul_packed(a, packed, scales, zps, rows, cols, bits, gs, transpose)
        got = K.matmul_packed(a, packed, scales, zps, rows, cols, bits, gs, transpose)
        assert np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-12) < 1e-12


# -- quantizer (test_quantizer.py) ------------------------------------------------------------

def test_unit_interval_midpoint_4bit():
    block = quantize(np.array([[0.0, 0.5, 1.0]]), 4, group_size=3)
    assert block.scales[0] == 1.0 / 15.0 and block.zero_points[0] == 0.0
    assert K.unpack_codes(block.packed, 4, 3).tolist() == [0, 8, 15]
    assert dequantize(block)[0, 1] == 8 * (1.0 / 15.0)


def test_constant_group_exact():
    block = quantize(np.full((1, 3), 3.7), 2, group_size=3)
    assert block.scales[0] == 0.0 and block.zero_points[0] == 3.7
    assert np.array_equal(dequantize(block), np.full((1, 3), 3.7))


def test_grid_aligned_round_trip_bit_exact():
    rng = np.random.default_rng(5)
    for bits in (2, 4):
        qmax = 2**bits - 1
        codes = rng.integers(0, qmax + 1, size=(6, 16))
        codes[:, 0] = 0
        codes[:, 1] = qmax
        x = -2.0 + 0.125 * codes
        block = quantize(x, bits, group_size=16)
        assert np.array_equal(K.unpack_codes(block.packed, bits, 96).reshape(6, 16), codes)
        assert np.array_equal(dequantize(block), x)


@pytest.mark.parametrize("bits", [2, 4])
def test_round_trip_bound(bits):
    rng = np.random.default_rng(7)
    x = rng.normal(size=(2000, 16)) * 10.0 ** rng.uniform(-3, 3, size=(2000, 1))
    block = quantize(x, bits, group_size=16)
    span = x.max(axis=1) - x.min(axis=1)
    err = np.abs(dequantize(block) - x).max(axis=1)
    assert (err <= span / (2 * (2**bits - 1))).all()


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_quantize_rejects_nonfinite(bad):
    x = np.ones((2, 4))
    x[1, 2] = bad
    with pytest.raises(ValueError):
        quantize(x, 4)


def test_quantize_rejects_bad_bitwidth_and_group():
    with pytest.raises(ValueError):
        quantize(np.ones((2, 2)), 3)
    with pytest.raises(ValueError):
        quantize(np.ones((2, 2)), 4, group_size=0)


def test_fqm_matches_mm_oracle():
    rng = np.random.default_rng(11)
    for transpose in (False, True):
        for m, rows, cols, gs, bits in [(1, 4, 4, 4, 4), (16, 64, 64, 32, 2), (64, 512, 64, 32, 4), (5, 33, 17, 8, 2)]:
            block = quantize(rng.normal(size=(rows, cols)), bits, group_size=gs)
            a = rng.normal(size=(m, cols if transpose else rows))
            ref = a @ (dequantize(block).T if transpose else dequantize(block))
            out = fqm(a, block, transpose_block=transpose)
            assert np.max(np.abs(out - ref)) / max(np.max(np.abs(ref)), 1e-12) <= 1e-6


def test_fqm_dimension_mismatch():
    block = quantize(np.ones((4, 6)), 4, group_size=6)
    with pytest.raises(ValueError):
        fqm(np.ones((2, 5)), block)
    with pytest.raises(ValueError):
        fqm(np.ones((2, 4)), block, transpose_block=True)


def test_wire_format_frozen():
    block = quantize(np.array([[0.0, 1.0]]), 4, group_size=2)
    raw = serialize_block(block)
    assert struct.unpack_from("<4I", raw, 0) == (1, 2, 4, 2)
    assert struct.unpack_from("<d", raw, 16)[0] == 1.0 / 15.0
    assert struct.unpack_from("<I", raw, 32)[0] == 0xF0 and len(raw) == 36
    back, end = deserialize_block(raw)
    assert end == len(raw) and serialize_block(back) == raw


def test_block_validation():
    with pytest.raises(ValueError):
        QuantizedBlock(rows=1, cols=2, bitwidth=4, group_size=2, packed=np.zeros(5, np.uint32),
                       scales=np.zeros(1), zero_points=np.zeros(1))


# -- kv_store (test_kv_store.py) --------------------------------------------------------------

def _build(tokens, dim, tiers, cs, gs, seed=0, tail=0):
    rng = np.random.default_rng(seed)
    k, v = rng.normal(size=(tokens + tail, dim)), rng.normal(size=(tokens + tail, dim))
    return build_cache(k, v, tiers, segment_context(list(range(tokens + tail)), cs), group_size=gs), k, v


def test_perm_and_token_order_worked_example():
    tiers = [Tier.INT2, Tier.FP16, Tier.INT2, Tier.INT4]
    cache, k, v = _build(16, 8, tiers, 4, 8, tail=2)
    assert cache.perm.tolist() == [0, 2, 3, 1]
    assert cache.len_2 == 8 and cache.len_4 == 4 and cache.tiers == tiers
    assert np.array_equal(cache.k_fp[:4], k[4:8])
    assert token_order(cache).tolist() == [0, 1, 2, 3, 8, 9, 10, 11, 12, 13, 14, 15, 4, 5, 6, 7, 16, 17]


def test_build_cache_matches_oracle_bitwise():
    rng = np.random.default_rng(1)
    for _ in range(10):
        n = int(rng.integers(1, 12))
        tiers_c = rng.choice([0, 1, 2], size=n).astype(np.uint8)
        tiers = [Tier.from_code(t) for t in tiers_c]
        cache, k, v = _build(4 * n, 8, tiers, 4, 8, seed=int(rng.integers(1e6)), tail=int(rng.integers(0, 4)))
        oc = O.build_cache(k, v, tiers_c, 4, 8)
        assert np.array_equal(cache.perm, oc.perm)
        for name in ("k_q2", "v_q2", "k_q4", "v_q4"):
            a, b = getattr(cache, name), getattr(oc, name)
            assert np.array_equal(a.packed, b.packed)
            assert np.array_equal(a.scales.view(np.uint64), b.scales.view(np.uint64))
        assert np.array_equal(cache.k_fp, oc.k_fp)


def test_reconstruction_and_serialization():
    tiers = [Tier.INT2, Tier.INT4, Tier.FP16, Tier.INT2, Tier.INT4]
    cache, k, v = _build(5 * 8, 16, tiers, 8, 8, seed=3, tail=5)
    kh, vh = reconstruct(cache)
    ok, ov = O.reconstruct(O.build_cache(k, v, np.array([t.code for t in tiers], np.uint8), 8, 8))
    assert np.array_equal(kh, ok) and np.array_equal(vh, ov)
    rng = np.random.default_rng(7)
    for _ in range(5):
        cache.append(rng.normal(size=16), rng.normal(size=16))
    raw = serialize_cache(cache)
    back = deserialize_cache(raw)
    assert serialize_cache(back) == raw and back.decode_len == 5
    pos = 0
    for _, off, size in cache_layout(cache):
        assert off == pos
        pos += size
    assert pos == len(raw)
    rep = memory_footprint(cache)
    assert rep.total_bytes > 0 and 0 < rep.compression_ratio < 2


def test_empty_cache_rolls():
    cache = ChunkedKVCache.empty(head_dim=3, chunk_size=4, group_size=4)
    rows = [np.array([1.0, 2.0, 3.0]) * i for i in range(5)]
    for r in rows:
        cache.append(r, -r)
    assert np.array_equal(reconstruct(cache)[0], np.stack(rows))


# -- attention (test_attention.py, test_acceptance.py:52-91) ------------------------------------

def test_mixed_attention_matches_reference_golden():
    g = load_golden("attention.npz")
    for i in range(int(g["n"])):
        n, cs, d, gs, m, tail, dec = (int(x) for x in g[f"spec{i}"])
        tiers = [Tier.from_code(t) for t in g[f"tiers{i}"]]
        cache = build_cache(g[f"k{i}"], g[f"v{i}"], tiers, segment_context(list(range(n * cs + tail)), cs), gs)
        for r in range(dec):
            cache.append(g[f"kd{i}"][r], g[f"vd{i}"][r])
        out = mixed_decode_attention(AttentionInstance(q=g[f"q{i}"], cache=cache))
        assert np.max(np.abs(out - g[f"mixed{i}"])) < 1e-12
        ref = reference_attention(g[f"q{i}"], *reconstruct(cache))
        assert np.max(np.abs(ref - g[f"ref{i}"])) < 1e-12


def test_blocking_equivalence_random():  # acceptance 1, fewer instances
    rng = np.random.default_rng(2024)
    for _ in range(20):
        cs = int(rng.choice([8, 16, 32]))
        n = int(rng.integers(1, 8))
        d = int(rng.choice([16, 64]))
        tiers = [Tier(t) for t in rng.choice(["int2", "int4", "fp16"], size=n)]
        T = n * cs + int(rng.integers(0, cs))
        k, v = rng.normal(size=(T, d)), rng.normal(size=(T, d))
        cache = build_cache(k, v, tiers, segment_context(list(range(T)), cs), 16)
        q = rng.normal(size=(int(rng.integers(1, 5)), d))
        got = mixed_decode_attention(AttentionInstance(q=q, cache=cache))
        want = reference_attention(q, *reconstruct(cache))
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= 1e-9


def test_attention_mask_and_errors():
    rng = np.random.default_rng(11)
    tiers = [Tier.INT2, Tier.FP16]
    cache, _, _ = _build(8, 8, tiers, 4, 8)
    q = rng.normal(size=(2, 8))
    mask = np.zeros((2, 8))
    mask[:, 3] = -np.inf
    got = mixed_decode_attention(AttentionInstance(q=q, cache=cache, mask=mask, scale=0.25))
    kr, vr = O.reconstruct(O.build_cache(*_build(8, 8, tiers, 4, 8)[1:], np.array([0, 2], np.uint8), 4, 8))
    order = O.token_order(O.build_cache(*_build(8, 8, tiers, 4, 8)[1:], np.array([0, 2], np.uint8), 4, 8))
    full_mask = np.zeros((2, 8))
    full_mask[:, order[3]] = -np.inf
    want = O.reference_attention(q, kr, vr, mask=full_mask, scale=0.25)
    assert np.max(np.abs(got - want)) < 1e-12
    with pytest.raises(ValueError):
        mixed_decode_attention(AttentionInstance(q=q, cache=ChunkedKVCache.empty(head_dim=8)))
    with pytest.raises(ValueError):
        reference_attention(np.ones((1, 3)), np.ones((2, 4)), np.ones((2, 4)))
    w = stable_softmax(np.array([[1e6, 1e6 + 1.0, -np.inf], [0.0, -np.inf, -np.inf]]))
    assert np.all(np.isfinite(w)) and w[0, 2] == 0.0 and w[1, 0] == 1.0
