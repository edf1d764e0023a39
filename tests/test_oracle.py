"""CPU: pin the oracle (oracle/ckv_oracle.py) against golden vectors produced by the
reference itself (tests/golden/make_golden.py) and the reference's frozen known-answer tests."""

import numpy as np
import pytest

from oracle import ckv_oracle as O
from tests.conftest import load_golden


def test_oracle_quantize_matches_reference_golden():
    g = load_golden("quantize.npz")
    for i in range(int(g["n"])):
        rows, cols, gs, bits = (int(x) for x in g[f"meta{i}"])
        codes, scales, zps = O.quantize_groups(g[f"x{i}"], bits, gs)
        assert np.array_equal(codes, g[f"codes{i}"])
        assert np.array_equal(scales.view(np.uint64), g[f"scales{i}"].view(np.uint64))
        assert np.array_equal(zps.view(np.uint64), g[f"zps{i}"].view(np.uint64))
        assert np.array_equal(O.pack_codes(codes.reshape(-1), bits), g[f"packed{i}"])


def test_oracle_fp16_rows_and_lohi_metadata():
    g = load_golden("fp16_rows.npz")
    x = g["x16"].astype(np.float64)
    lohi = O.arena_meta_lohi(g["x16"]).astype(np.float64)
    for bits in (2, 4):
        codes, scales, zps = O.quantize_groups(x, bits, 32)
        assert np.array_equal(O.pack_codes(codes.reshape(-1), bits), g[f"packed{bits}"])
        # GPU metadata (lo, hi) fp16 expands to the reference's f64 scale/zp bit for bit
        qmax = float(2**bits - 1)
        sc = (lohi[..., 1] - lohi[..., 0]).reshape(-1) / qmax
        assert np.array_equal(sc.view(np.uint64), g[f"scales{bits}"].view(np.uint64))
        assert np.array_equal(lohi[..., 0].reshape(-1).view(np.uint64), g[f"zps{bits}"].view(np.uint64))


def test_oracle_search_matches_reference_golden():
    g = load_golden("search.npz")
    for s in g["seeds"]:
        scores = O.score_chunks(g[f"q{s}"], float(g[f"qnorm{s}"]), g[f"emb{s}"], g[f"norm{s}"])
        assert np.allclose(scores, g[f"scores{s}"], rtol=0, atol=1e-15)
        t_low, t_high = O.compute_thresholds(scores, 0.6, 0.1)
        assert np.allclose([t_low, t_high], g[f"stats{s}"][2:], rtol=0, atol=1e-15)
        tiers = O.assign_tiers(scores, t_low, t_high)
        assert np.array_equal(tiers, g[f"tiers{s}"])
        perm, counts = O.stable_perm(tiers)
        assert np.array_equal(perm, g[f"perm{s}"])
        assert counts.sum() == tiers.size


def test_oracle_attention_matches_reference_golden():
    g = load_golden("attention.npz")
    for i in range(int(g["n"])):
        n, cs, d, gs, m, tail, dec = (int(x) for x in g[f"spec{i}"])
        cache = O.build_cache(g[f"k{i}"], g[f"v{i}"], g[f"tiers{i}"], cs, gs)
        assert np.array_equal(cache.perm, g[f"perm{i}"])
        assert np.array_equal(cache.k_q2.packed, g[f"k_q2_packed{i}"])
        assert np.array_equal(cache.v_q4.scales.view(np.uint64), g[f"v_q4_scales{i}"].view(np.uint64))
        for r in range(dec):
            cache.append(g[f"kd{i}"][r], g[f"vd{i}"][r])
        out = O.mixed_decode_attention(g[f"q{i}"], cache)
        assert np.max(np.abs(out - g[f"mixed{i}"])) < 1e-12
        kr, vr = O.reconstruct(cache)
        ref = O.reference_attention(g[f"q{i}"], kr, vr)
        assert np.max(np.abs(ref - g[f"ref{i}"])) < 1e-12


def test_oracle_batched_case_matches_reference_golden():
    g = load_golden("batched.npz")
    L, B, H, m, T = (int(x) for x in g["dims"])
    for l in range(L):
        for b in range(B):
            for h in range(H):
                key = f"{l}_{b}_{h}"
                cache = O.build_cache(g["k"][l, b, :, h].astype(np.float64),
                                      g["v"][l, b, :, h].astype(np.float64), g["tiers"][b], 32, 32)
                assert np.array_equal(cache.k_q2.packed, g[f"k_q2_packed_{key}"])
                assert np.array_equal(cache.v_q4.packed, g[f"v_q4_packed_{key}"])
                q = g["q"][l, b, h * m:(h + 1) * m].astype(np.float64)
                assert np.max(np.abs(O.mixed_decode_attention(q, cache) - g[f"out_{key}"])) < 1e-12


# -- the reference's own frozen known-answer tests, restated on the oracle ---------------

def test_kat_pack_layout():  # test_kernels.py:27-37
    assert O.pack_codes(np.array([1, 2, 3], np.uint8), 4).tolist() == [0x321]
    assert O.pack_codes(np.array([3, 0, 1, 2], np.uint8), 2).tolist() == [147]
    c = np.zeros(17, np.uint8)
    c[16] = 3
    assert O.pack_codes(c, 2).tolist() == [0, 3]


def test_kat_unit_interval_midpoint():  # test_quantizer.py:30-37
    blk = O.quantize(np.array([[0.0, 0.5, 1.0]]), 4, group_size=3)
    assert blk.scales[0] == 1.0 / 15.0 and blk.zero_points[0] == 0.0
    assert O.unpack_codes(blk.packed, 4, 3).tolist() == [0, 8, 15]


def test_kat_constant_group():  # test_quantizer.py:40-45
    blk = O.quantize(np.full((1, 3), 3.7), 2, group_size=3)
    assert blk.scales[0] == 0.0 and blk.zero_points[0] == 3.7
    assert O.unpack_codes(blk.packed, 2, 3).tolist() == [0, 0, 0]


def test_kat_thresholds_and_perm():  # test_retrieval.py:213-217, test_kv_store.py:38-49
    t_low, t_high = O.compute_thresholds([0.1, 0.5, 0.9], 0.5, 0.25)
    assert t_low == 0.5 and abs(t_high - 0.7) < 1e-12
    assert O.assign_tiers([0.1, 0.5, 0.9], t_low, t_high).tolist() == [0, 1, 2]
    perm, counts = O.stable_perm([0, 2, 0, 1])
    assert perm.tolist() == [0, 2, 3, 1] and counts.tolist() == [2, 1, 1]


def test_kat_precomputed_scores_tiers():  # test_harness.py:298-327
    q = np.array([1.0, 0.0])
    emb = np.array([[1.0, 0.0], [0.8, 0.6], [0.0, 1.0], [-1.0, 0.0]])
    s = O.score_chunks(q, 1.0, emb, np.linalg.norm(emb, axis=1))
    assert np.allclose(s, [1.0, 0.8, 0.0, -1.0])
    t = O.assign_tiers(s, *O.compute_thresholds(s, 0.6, 0.1))
    assert t.tolist() == [2, 1, 0, 0]


def test_kat_zero_norm_substitution():  # test_retrieval.py:190-203
    q = np.array([1.0, 0.0])
    emb = np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 0.0]])
    assert O.score_chunks(q, 1.0, emb, [1.0, 1.0, 0.0]) == [1.0, -1.0, -1.0]
    assert O.score_chunks(q, 1.0, emb[2:] .repeat(3, 0), [0.0] * 3) == [0.0] * 3
    with pytest.raises(ValueError):
        O.score_chunks(q, 0.0, emb, [1.0, 1.0, 0.0])


def test_oracle_lse_merge_equals_single_softmax():
    rng = np.random.default_rng(0)
    s = rng.normal(size=(3, 40)) * 4
    v = rng.normal(size=(40, 5))
    full = O.stable_softmax(s * np.log(2), axis=1) @ v  # log2-domain scores
    ms, ls, accs = [], [], []
    for a, b in ((0, 10), (10, 25), (25, 40)):
        m = s[:, a:b].max(axis=1)
        p = np.exp2(s[:, a:b] - m[:, None])
        ms.append(m)
        ls.append(p.sum(axis=1))
        accs.append(p @ v[a:b])
    assert np.allclose(O.lse_merge(ms, ls, accs), full, atol=1e-12)
