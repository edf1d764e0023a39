"""Text encoders upstream of the search (retrieval.py:70-196): the oracle's
restatement against the reference's own outputs (CPU), the GPU encoders against the same
fixtures (hashed bag of words bit-exact, TF-IDF within a few ulp), and texts -> tiers through
``search_texts`` against the reference's tier maps (tests/golden/encoders.npz, search.npz)."""

import json

import numpy as np
import pytest

from oracle import ckv_oracle as O
from tests.conftest import load_golden

# str.isspace() code points the CUDA splitter decodes (csrc/ckv_encode.cu ws_len)
KERNEL_SPACES = ([*range(0x09, 0x0E), *range(0x1C, 0x21), 0x85, 0xA0, 0x1680, *range(0x2000, 0x200B),
                  0x2028, 0x2029, 0x202F, 0x205F, 0x3000])


def _texts(g, key="text", okey="offsets"):
    blob, off = g[key].tobytes(), g[okey]
    return [blob[off[i]:off[i + 1]].decode("utf-8") for i in range(len(off) - 1)]


def test_kernel_whitespace_set_is_python_isspace():
    assert load_golden("encoders.npz")["spaces"].tolist() == KERNEL_SPACES


def test_oracle_bow_matches_reference():
    g = load_golden("encoders.npz")
    texts = _texts(g)
    for seed in (0, 7, 123456789):
        for dim in (256, 100, 1, 4096):
            for i, t in enumerate(texts):
                v, n = O.bow_encode(t, dim, seed)
                assert np.array_equal(v.view(np.uint64), g[f"bow_{seed}_{dim}"][i].view(np.uint64)), (seed, dim, i)
                assert n == g[f"bow_norm_{seed}_{dim}"][i]


def test_oracle_tfidf_matches_reference():
    g = load_golden("encoders.npz")
    texts = _texts(g)
    index, idf = O.tfidf_fit(texts)
    for i, t in enumerate(texts):
        v, n = O.tfidf_encode(t, index, idf)
        assert np.array_equal(v, g["tfidf"][i]) and n == g["tfidf_norm"][i]


def test_fixture_covers_edge_cases():
    g = load_golden("encoders.npz")
    texts = _texts(g)
    norms = g["bow_norm_0_256"]
    assert norms[0] == 0.0 and norms[1] == 0.0                      # empty, blank
    assert any(len(w.encode()) > 128 for t in texts for w in t.split())  # multi-block words
    cancel = [i for i, t in enumerate(texts) if len(t.split()) == 2 and t.startswith("w") and norms[i] == 0.0]
    assert cancel, "a cancelling word pair (norm 0 from non-empty text)"


def test_make_encoder_and_precomputed(tmp_path):
    from paper_2503_23294_b200 import retrieval as R

    assert isinstance(R.make_encoder("bow", seed=3), R.HashedBowEncoder)
    assert isinstance(R.make_encoder("tfidf"), R.TfidfEncoder)
    with pytest.raises(ValueError):
        R.make_encoder("nope")
    with pytest.raises(ValueError):
        R.HashedBowEncoder(dim=0)
    p = tmp_path / "emb.jsonl"
    p.write_text(json.dumps({"id": "a", "vector": [3.0, 4.0]}) + "\n\n" + json.dumps({"id": "b", "vector": [0, 0]}) + "\n")
    enc = R.make_encoder(f"file:{p}")
    e = R.encode("a", enc)
    assert e.norm == 5.0 and np.array_equal(e.vector, [3.0, 4.0]) and enc.encode("b").norm == 0.0
    with pytest.raises(KeyError):
        enc.encode("c")
    bad = tmp_path / "bad.jsonl"
    bad.write_text(json.dumps({"id": "a", "vector": [1.0]}) + "\n" + json.dumps({"id": "a", "vector": [2.0]}) + "\n")
    with pytest.raises(ValueError):
        R.PrecomputedEncoder(str(bad))
    with pytest.raises(RuntimeError):
        R.TfidfEncoder().encode_batch_dev(["x"])


# ---- GPU -------------------------------------------------------------------------------

@pytest.mark.gpu
def test_gpu_bow_bit_exact():
    from paper_2503_23294_b200.retrieval import HashedBowEncoder

    g = load_golden("encoders.npz")
    texts = _texts(g)
    for seed in (0, 7, 123456789):
        for dim in (256, 100, 1, 4096):
            v, n = HashedBowEncoder(dim=dim, seed=seed).encode_batch_dev(texts)
            v, n = v.cpu().numpy(), n.cpu().numpy()
            want = g[f"bow_{seed}_{dim}"]
            bad = np.nonzero(~np.all(v.view(np.uint64) == want.view(np.uint64), axis=1))[0]
            assert bad.size == 0, (seed, dim, [texts[i][:40] for i in bad[:5]])
            assert np.array_equal(n, g[f"bow_norm_{seed}_{dim}"])
    e = HashedBowEncoder(seed=7).encode(texts[5])
    assert np.array_equal(e.vector, g["bow_7_256"][5]) and e.norm == g["bow_norm_7_256"][5]


@pytest.mark.gpu
def test_gpu_tfidf_within_ulps():
    from paper_2503_23294_b200.retrieval import TfidfEncoder

    g = load_golden("encoders.npz")
    texts = _texts(g)
    enc = TfidfEncoder()
    enc.fit(texts)
    v, n = enc.encode_batch_dev(texts)
    v = v.cpu().numpy()[:, :enc.dim]
    assert np.array_equal(n.cpu().numpy(), g["tfidf_norm"])
    assert np.max(np.abs(v - g["tfidf"])) <= 4 * np.finfo(np.float64).eps
    assert np.array_equal(v == 0, g["tfidf"] == 0)


@pytest.mark.gpu
def test_gpu_search_texts_matches_reference_tiers():
    from paper_2503_23294_b200.retrieval import HashedBowEncoder, search_texts

    g, s = load_golden("encoders.npz"), load_golden("search.npz")
    chunk_texts, queries = [], []
    for seed in (0, 1, 2, 3):
        t = _texts(g, f"wl_text{seed}", f"wl_offsets{seed}")
        chunk_texts.append(t[:-1])
        queries.append(t[-1])
    # every sequence encoded with its own seed's key, as the harness does: one call per seed
    for seed in (0, 1, 2, 3):
        r = search_texts([chunk_texts[seed]], [queries[seed]], 0.6, 0.1, HashedBowEncoder(seed=seed))
        assert np.array_equal(r.tiers[0].cpu().numpy(), s[f"tiers{seed}"])
        assert np.array_equal(r.perm[0].cpu().numpy().astype(np.uint32), s[f"perm{seed}"])
        assert np.allclose(r.scores[0].cpu().numpy(), s[f"scores{seed}"], rtol=0, atol=1e-15)
    # ragged batch (sequences truncated to different chunk counts) in one launch
    cut = [128, 100, 77, 128]
    r = search_texts([c[:k] for c, k in zip(chunk_texts, cut)], queries, 0.6, 0.1, HashedBowEncoder(seed=0))
    for b in range(4):
        enc = [O.bow_encode(t, 256, 0) for t in chunk_texts[b][:cut[b]]]
        qv, qn = O.bow_encode(queries[b], 256, 0)
        sc = O.score_chunks(qv, qn, np.stack([e[0] for e in enc]), [e[1] for e in enc])
        t_lo, t_hi = O.compute_thresholds(sc, 0.6, 0.1)
        assert np.array_equal(r.tiers[b, :cut[b]].cpu().numpy(), O.assign_tiers(sc, t_lo, t_hi))


@pytest.mark.gpu
def test_gpu_encoder_errors():
    from paper_2503_23294_b200.retrieval import HashedBowEncoder, search_texts

    with pytest.raises(ValueError):
        search_texts([["a b", "c"]], ["   "])  # zero-norm query
    with pytest.raises(Exception):
        HashedBowEncoder(dim=9000).encode_batch_dev(["a"])
    v, n = HashedBowEncoder().encode_batch_dev([])
    assert v.shape == (0, 256) and n.shape == (0,)
