"""GPU: Module I (ckv_search) — scores, thresholds, tier maps and permutations against the
reference's golden vectors (bit-exact maps), its frozen KATs, and the oracle at full size."""

import numpy as np
import pytest

from oracle import ckv_oracle as O
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

from paper_2503_23294_b200.retrieval import (Embedding, assign_tiers, build_similarity_report,  # noqa: E402
                                             compute_thresholds, score_chunks, search_batched)
from paper_2503_23294_b200.tiers import Tier  # noqa: E402


def test_search_batched_matches_reference_golden():
    g = load_golden("search.npz")
    seeds = list(g["seeds"])
    emb = np.stack([g[f"emb{s}"] for s in seeds])
    norm = np.stack([g[f"norm{s}"] for s in seeds])
    q = np.stack([g[f"q{s}"] for s in seeds])
    qn = np.array([float(g[f"qnorm{s}"]) for s in seeds])
    r = search_batched(emb, norm, q, qn, 0.6, 0.1)
    for i, s in enumerate(seeds):
        assert np.allclose(r.scores[i].cpu().numpy(), g[f"scores{s}"], rtol=0, atol=1e-15)
        assert np.allclose(r.stats[i].cpu().numpy(), g[f"stats{s}"], rtol=0, atol=1e-15)
        assert np.array_equal(r.tiers[i].cpu().numpy(), g[f"tiers{s}"])
        assert np.array_equal(r.perm[i].cpu().numpy().view(np.uint32), g[f"perm{s}"])
        c = r.seg_counts[i].cpu().numpy()
        assert c.tolist() == [int((g[f"tiers{s}"] == t).sum()) for t in (0, 1, 2)]


def test_workload_tier_maps_match_reference_at_32k_and_128k():
    import bench
    for ctx, seeds in ((32768, range(8)), (131072, range(1))):
        wls = [bench.load_workload(ctx, s) for s in seeds]
        r = search_batched(np.stack([w["emb"] for w in wls]), np.stack([w["norm"] for w in wls]),
                           np.stack([w["q"] for w in wls]), np.array([w["qnorm"] for w in wls]))
        for i, w in enumerate(wls):
            assert np.array_equal(r.tiers[i].cpu().numpy(), w["tiers"])
            perm, _ = O.stable_perm(w["tiers"])
            assert np.array_equal(r.perm[i].cpu().numpy().view(np.uint32), perm)


def test_search_random_large_matches_oracle():
    rng = np.random.default_rng(0)
    B, N, d = 4, 4096, 256
    emb = rng.normal(size=(B, N, d))
    emb[:, 7] = 0.0  # zero-norm chunks
    norm = np.linalg.norm(emb, axis=2)
    q = rng.normal(size=(B, d))
    r = search_batched(emb, norm, q, np.linalg.norm(q, axis=1), 0.6, 0.1)
    for b in range(B):
        s = O.score_chunks(q[b], np.linalg.norm(q[b]), emb[b], norm[b])
        t = O.assign_tiers(s, *O.compute_thresholds(s, 0.6, 0.1))
        assert np.allclose(r.scores[b].cpu().numpy(), s, atol=1e-14)
        assert np.array_equal(r.tiers[b].cpu().numpy(), t)


def test_ragged_batch():
    rng = np.random.default_rng(1)
    emb = rng.normal(size=(3, 50, 16))
    norm = np.linalg.norm(emb, axis=2)
    q = rng.normal(size=(3, 16))
    r = search_batched(emb, norm, q, np.linalg.norm(q, axis=1), 0.5, 0.2, seq_chunks=np.array([50, 10, 1]))
    for b, n in enumerate([50, 10, 1]):
        s = O.score_chunks(q[b], np.linalg.norm(q[b]), emb[b, :n], norm[b, :n])
        t = O.assign_tiers(s, *O.compute_thresholds(s, 0.5, 0.2))
        assert np.array_equal(r.tiers[b, :n].cpu().numpy(), t)
        assert r.seg_counts[b].sum().item() == n


def test_reference_kats():
    t_low, t_high = compute_thresholds([0.1, 0.5, 0.9], 0.5, 0.25)
    assert t_low == 0.5 and t_high == pytest.approx(0.7, abs=1e-12)
    assert assign_tiers([0.1, 0.5, 0.9], t_low, t_high) == [Tier.INT2, Tier.INT4, Tier.FP16]
    assert compute_thresholds([0.2, 0.8, 0.5], 0.0, 0.0) == (0.2, 0.8)
    assert compute_thresholds([0.4, 0.4], 0.6, 0.1) == (0.4, 0.4)
    assert assign_tiers([0.5], 0.5, 0.7) == [Tier.INT4] and assign_tiers([0.7], 0.5, 0.7) == [Tier.INT4]
    with pytest.raises(ValueError):
        compute_thresholds([0.1, 0.9], 0.7, 0.7)
    assert compute_thresholds([0.5, 0.5], 0.7, 0.7) == (0.5, 0.5)
    with pytest.raises(ValueError):
        compute_thresholds([], 0.5, 0.1)
    with pytest.raises(ValueError):
        compute_thresholds([0.1], -0.1, 0.0)
    q = Embedding.from_vector([1.0, 0.0])
    assert score_chunks(q, [Embedding.from_vector(v) for v in ([1.0, 0.0], [-1.0, 0.0], [0.0, 0.0])]) == [1.0, -1.0, -1.0]
    assert score_chunks(q, [Embedding.from_vector([0.0, 0.0])] * 3) == [0.0, 0.0, 0.0]
    with pytest.raises(ValueError):
        score_chunks(Embedding.from_vector([0.0]), [Embedding.from_vector([1.0])])
    s = score_chunks(q, [Embedding.from_vector(v) for v in ([1.0, 0.0], [0.8, 0.6], [0.0, 1.0], [-1.0, 0.0])])
    rep = build_similarity_report(s, 0.6, 0.1)
    assert [t.value for t in rep.tiers] == ["fp16", "int4", "int2", "int2"]
