"""Chunk-level quantization search (Module I) — drop-in for ``chunkkv.retrieval``
(retrieval.py:17-279): scoring, thresholds, tiers and the stable permutation in the
ckv_search kernel, and the text encoders upstream of it.

Encoders (retrieval.py:70-191): ``HashedBowEncoder`` runs on the GPU (ckv_bow_encode:
UTF-8 whitespace split, keyed BLAKE2b-64 per word, signed buckets, L2 normalisation; the
embeddings equal the reference's bit for bit).  ``TfidfEncoder`` fits its sorted vocabulary
and smoothed idf on the host like the reference, maps words to ids on the host, and counts,
weights and normalises on the GPU (ckv_tfidf_encode; the norm's summation order differs
from BLAS, so vectors agree to a few ulp).  ``PrecomputedEncoder`` reads JSON lines.
``search_texts`` goes from chunk/query texts to tiers and permutations with the embeddings
never leaving the device.

``search_batched`` is the batched device form: B sequences x N chunks in one launch,
returning scores, thresholds, tiers, the stable INT2||INT4||FP16 permutation and
per-tier chunk counts, all resident on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels
from .tiers import Tier


@dataclass(frozen=True)
class ChunkSet:
    """retrieval.py:17-37: full chunks plus a tail shorter than one chunk."""

    chunks: tuple
    tail: tuple
    chunk_size: int

    @property
    def n(self) -> int:
        return len(self.chunks)

    @property
    def context_len(self) -> int:
        return self.n * self.chunk_size + len(self.tail)


def segment_context(tokens, chunk_size) -> ChunkSet:
    """retrieval.py:40-50."""
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    tokens = tuple(tokens)
    if not tokens:
        raise ValueError("tokens must be non-empty")
    n = len(tokens) // chunk_size
    chunks = tuple(tokens[i * chunk_size:(i + 1) * chunk_size] for i in range(n))
    return ChunkSet(chunks=chunks, tail=tokens[n * chunk_size:], chunk_size=chunk_size)


@dataclass(frozen=True)
class Embedding:
    """retrieval.py:53-67: vector with its cached L2 norm (norm == 0 flags an empty span)."""

    vector: np.ndarray
    norm: float

    @classmethod
    def from_vector(cls, vector) -> "Embedding":
        v = np.asarray(vector, dtype=np.float64).reshape(-1)
        return cls(vector=v, norm=float(np.linalg.norm(v)))


# -- encoders (retrieval.py:70-196) ---------------------------------------------------

def _pack_texts(texts):
    """UTF-8 bytes of all texts back to back + int64 offsets [n + 1], on the device."""
    bufs = [t.encode("utf-8") for t in texts]
    offsets = np.zeros(len(bufs) + 1, dtype=np.int64)
    np.cumsum([len(b) for b in bufs], out=offsets[1:])
    data = b"".join(bufs) or b"\0"
    dev = _lib.device()
    text = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev)
    return text, torch.from_numpy(offsets).to(dev)


class HashedBowEncoder:
    """retrieval.py:70-100: order-free hashed bag of words with a hash-derived sign, L2
    normalised, keyed BLAKE2b (key = the seed's decimal digits), on the GPU."""

    def __init__(self, dim=256, seed=0):
        if dim < 1:
            raise ValueError("dim must be >= 1")
        self.dim = dim
        self._key = str(int(seed)).encode("ascii")

    def fit(self, texts):
        pass  # stateless

    def encode_batch_dev(self, texts, out=None, norms=None):
        """All texts in one launch -> (vectors f64 [n, dim], norms f64 [n]) on the GPU."""
        texts = list(texts)
        dev = _lib.device()
        n = len(texts)
        if out is None:
            out = torch.empty((n, self.dim), dtype=torch.float64, device=dev)
        if norms is None:
            norms = torch.empty(n, dtype=torch.float64, device=dev)
        if n:
            text, offsets = _pack_texts(texts)
            _lib.call("ckv_bow_encode", _lib.ptr(text), _lib.ptr(offsets), n, self.dim, self._key,
                      len(self._key), _lib.ptr(out), _lib.ptr(norms), _lib.stream())
        return out, norms

    def encode(self, text) -> Embedding:
        v, n = self.encode_batch_dev([text])
        return Embedding(vector=v[0].cpu().numpy(), norm=float(n[0].item()))


class TfidfEncoder:
    """retrieval.py:103-138: TF-IDF over the texts of one run; sorted vocabulary, smoothed
    idf ln((1 + n_docs) / (1 + df)) + 1.  fit() on the host (the reference's algorithm);
    counting, weighting and normalisation on the GPU."""

    def __init__(self):
        self._index = None
        self._idf = None
        self._idf_dev = None

    def fit(self, texts):
        texts = list(texts)
        vocab = sorted({w for t in texts for w in t.split()})
        self._index = {w: i for i, w in enumerate(vocab)}
        df = np.zeros(len(vocab), dtype=np.float64)
        for t in texts:
            for w in set(t.split()):
                df[self._index[w]] += 1.0
        self._idf = np.log((1.0 + len(texts)) / (1.0 + df)) + 1.0
        self._idf_dev = None

    @property
    def dim(self):
        return len(self._index) if self._index is not None else 0

    def encode_batch_dev(self, texts, out=None, norms=None):
        if self._index is None:
            raise RuntimeError("TfidfEncoder.encode called before fit")
        texts = list(texts)
        dev = _lib.device()
        if self._idf_dev is None:
            self._idf_dev = kernels.to_dev(self._idf, torch.float64)
        get = self._index.get
        ids = [[i for i in map(get, t.split()) if i is not None] for t in texts]
        offsets = np.zeros(len(ids) + 1, dtype=np.int64)
        np.cumsum([len(x) for x in ids], out=offsets[1:])
        flat = np.fromiter((i for x in ids for i in x), dtype=np.int32, count=int(offsets[-1]))
        n, dim = len(texts), max(self.dim, 1)
        if out is None:
            out = torch.empty((n, dim), dtype=torch.float64, device=dev)
        if norms is None:
            norms = torch.empty(n, dtype=torch.float64, device=dev)
        if n:
            ids_d = kernels.to_dev(flat if flat.size else np.zeros(1, np.int32), torch.int32)
            _lib.call("ckv_tfidf_encode", _lib.ptr(ids_d), _lib.ptr(kernels.to_dev(offsets, torch.int64)), n,
                      _lib.ptr(self._idf_dev), self.dim, out.stride(0), _lib.ptr(out), _lib.ptr(norms),
                      _lib.stream())
        return out, norms

    def encode(self, text) -> Embedding:
        v, n = self.encode_batch_dev([text])
        return Embedding(vector=v[0, :self.dim].cpu().numpy(), norm=float(n[0].item()))


class PrecomputedEncoder:
    """retrieval.py:141-181: vectors injected from a JSON-lines file of {"id", "vector"}."""

    def __init__(self, path):
        import json

        self.path = path
        self._vectors = {}
        dim = None
        with open(path, "r", encoding="utf-8") as fh:
            for lineno, line in enumerate(fh, start=1):
                if not line.strip():
                    continue
                try:
                    record = json.loads(line)
                    key = record["id"]
                    vec = np.asarray(record["vector"], dtype=np.float64).reshape(-1)
                except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
                    raise ValueError(f"{path}:{lineno}: bad embedding record: {exc}") from exc
                if dim is None:
                    dim = vec.shape[0]
                elif vec.shape[0] != dim:
                    raise ValueError(f"{path}:{lineno}: vector dimension {vec.shape[0]} != {dim}")
                if key in self._vectors:
                    raise ValueError(f"{path}:{lineno}: duplicate id {key!r}")
                self._vectors[key] = vec
        if not self._vectors:
            raise ValueError(f"{path}: no embedding records")
        self.dim = dim

    def fit(self, texts):
        pass  # vectors are fixed

    def encode(self, key) -> Embedding:
        try:
            vec = self._vectors[key]
        except KeyError:
            raise KeyError(f"no precomputed embedding for id {key!r} in {self.path}") from None
        return Embedding.from_vector(vec)

    def encode_batch_dev(self, keys, out=None, norms=None):
        embs = [self.encode(k) for k in keys]
        dev = _lib.device()
        v = kernels.to_dev(np.stack([e.vector for e in embs]) if embs else np.zeros((0, self.dim)), torch.float64)
        nm = kernels.to_dev(np.array([e.norm for e in embs], np.float64), torch.float64)
        if out is not None:
            out.copy_(v)
            v = out
        if norms is not None:
            norms.copy_(nm)
            nm = norms
        return v.to(dev), nm.to(dev)


def make_encoder(spec, seed=0):
    """retrieval.py:184-192: bow, tfidf, or file:PATH."""
    if spec == "bow":
        return HashedBowEncoder(seed=seed)
    if spec == "tfidf":
        return TfidfEncoder()
    if spec.startswith("file:"):
        return PrecomputedEncoder(spec[len("file:"):])
    raise ValueError(f"unknown encoder {spec!r} (expected bow, tfidf, or file:PATH)")


def encode(text, encoder) -> Embedding:
    """retrieval.py:195-196."""
    return encoder.encode(text)


@dataclass
class SearchResult:
    """Device-resident output of one batched search launch."""

    scores: torch.Tensor      # f64 [B, N]
    stats: torch.Tensor       # f64 [B, 4] = s_min, s_max, t_low, t_high
    tiers: torch.Tensor       # u8  [B, N]  (0 INT2, 1 INT4, 2 FP16)
    perm: torch.Tensor        # i32 [B, N]  (u32 chunk ids, INT2 || INT4 || FP16, stable)
    seg_counts: torch.Tensor  # i32 [B, 3]
    flags: torch.Tensor       # i32 [B]

    def raise_on_error(self):
        """Map device flags to the reference's ValueErrors (one host sync)."""
        fl = self.flags.cpu().numpy()
        f = int(np.bitwise_or.reduce(fl)) if fl.size else 0
        if f & _lib.FLAG_ZERO_QUERY:
            raise ValueError("query embedding has zero norm")
        if f & _lib.FLAG_EMPTY_SCORES:
            raise ValueError("scores must be non-empty")
        if f & _lib.FLAG_CROSSING:
            raise ValueError("alpha + beta > 1 makes the thresholds cross")


def _check_alpha_beta(alpha, beta):
    if not (0.0 <= alpha <= 1.0 and 0.0 <= beta <= 1.0):  # retrieval.py:227-228
        raise ValueError("alpha and beta must lie in [0, 1]")


def search_batched(emb, emb_norm, q, q_norm, alpha=0.6, beta=0.1, seq_chunks=None,
                   check=True) -> SearchResult:
    """Batched Module I on the GPU.

    emb f64 [B, N, d], emb_norm f64 [B, N], q f64 [B, d], q_norm f64 [B]; seq_chunks
    optional i32 [B] for ragged batches.  One launch, one CTA per sequence.
    """
    _check_alpha_beta(alpha, beta)
    emb = kernels.to_dev(emb, torch.float64)
    B, N, d = emb.shape
    emb_norm = kernels.to_dev(emb_norm, torch.float64)
    q = kernels.to_dev(q, torch.float64)
    q_norm = kernels.to_dev(q_norm, torch.float64)
    sc = kernels.to_dev(seq_chunks, torch.int32) if seq_chunks is not None else None
    dev = emb.device
    res = SearchResult(
        scores=torch.empty((B, N), dtype=torch.float64, device=dev),
        stats=torch.empty((B, 4), dtype=torch.float64, device=dev),
        tiers=torch.zeros((B, N), dtype=torch.uint8, device=dev),
        perm=torch.zeros((B, N), dtype=torch.int32, device=dev),
        seg_counts=torch.zeros((B, 3), dtype=torch.int32, device=dev),
        flags=torch.zeros(B, dtype=torch.int32, device=dev),
    )
    _lib.call("ckv_search", _lib.ptr(emb), _lib.ptr(emb_norm), _lib.ptr(q), _lib.ptr(q_norm),
              _lib.ptr(sc), B, N, d, float(alpha), float(beta), _lib.ptr(res.scores),
              _lib.ptr(res.stats), _lib.ptr(res.tiers), _lib.ptr(res.perm),
              _lib.ptr(res.seg_counts), _lib.ptr(res.flags), _lib.stream())
    if check:
        res.raise_on_error()
    return res


def search_texts(chunk_texts, query_texts, alpha=0.6, beta=0.1, encoder=None, fit=True,
                 check=True) -> SearchResult:
    """Texts to tiers for B sequences: ``chunk_texts`` a list (per sequence) of chunk strings,
    ``query_texts`` one string per sequence.  All chunks and queries are encoded in one launch
    (default ``HashedBowEncoder()``) into a [B, N_max, dim] embedding block that ckv_search
    reads in place (ragged sequences: padded rows are empty texts, excluded via seq_chunks).
    ``fit`` calls ``encoder.fit`` on every chunk and query text first, as the harness does
    (harness.py:181-190; a no-op for bow)."""
    encoder = HashedBowEncoder() if encoder is None else encoder
    chunk_texts = [list(c) for c in chunk_texts]
    query_texts = list(query_texts)
    B = len(chunk_texts)
    if B != len(query_texts):
        raise ValueError("one query text per sequence")
    n = [len(c) for c in chunk_texts]
    N = max(n) if n else 0
    if fit:
        encoder.fit([t for c in chunk_texts for t in c] + query_texts)
    flat = [t for c in chunk_texts for t in c + [""] * (N - len(c))] + query_texts
    vec, norms = encoder.encode_batch_dev(flat)
    d = vec.shape[1]
    emb, emb_norm = vec[:B * N].view(B, N, d), norms[:B * N].view(B, N)
    return search_batched(emb, emb_norm, vec[B * N:], norms[B * N:], alpha, beta,
                          np.array(n, np.int32), check)


def tiers_from_scores_batched(scores, alpha, beta, check=True) -> SearchResult:
    """compute_thresholds + assign_tiers + stable grouping for given scores f64 [B, N]."""
    _check_alpha_beta(alpha, beta)
    s = kernels.to_dev(scores, torch.float64).clone()
    if s.ndim == 1:
        s = s.reshape(1, -1)
    B, N = s.shape
    dev = s.device
    res = SearchResult(
        scores=s,
        stats=torch.empty((B, 4), dtype=torch.float64, device=dev),
        tiers=torch.zeros((B, N), dtype=torch.uint8, device=dev),
        perm=torch.zeros((B, N), dtype=torch.int32, device=dev),
        seg_counts=torch.zeros((B, 3), dtype=torch.int32, device=dev),
        flags=torch.zeros(B, dtype=torch.int32, device=dev),
    )
    _lib.call("ckv_search", None, None, None, None, None, B, N, 0, float(alpha), float(beta),
              _lib.ptr(res.scores), _lib.ptr(res.stats), _lib.ptr(res.tiers), _lib.ptr(res.perm),
              _lib.ptr(res.seg_counts), _lib.ptr(res.flags), _lib.stream())
    if check:
        res.raise_on_error()
    return res


# -- per-head, reference-shaped API ---------------------------------------------------

def cosine_similarity(q: Embedding, c: Embedding) -> float:
    """retrieval.py:199-202."""
    if q.norm == 0.0 or c.norm == 0.0:
        raise ValueError("cosine similarity of a zero-norm embedding is undefined")
    return score_chunks(q, [c])[0]


def score_chunks(query: Embedding, chunk_embeddings) -> list:
    """retrieval.py:205-219: cosine per chunk; zero-norm chunks score min(valid) (0.0 if none)."""
    if query.norm == 0.0:
        raise ValueError("query embedding has zero norm")
    chunk_embeddings = list(chunk_embeddings)
    if not chunk_embeddings:
        return []
    emb = np.stack([np.asarray(c.vector, np.float64).reshape(-1) for c in chunk_embeddings])[None]
    norms = np.array([[float(c.norm) for c in chunk_embeddings]])
    qv = np.asarray(query.vector, np.float64).reshape(1, -1)
    res = search_batched(emb, norms, qv, np.array([float(query.norm)]), 0.0, 0.0, check=False)
    return [float(s) for s in res.scores[0].cpu().numpy()]


def compute_thresholds(scores, alpha, beta):
    """retrieval.py:222-237: t_low = s_min + (s_max-s_min)*alpha; t_high = s_max - (s_max-s_min)*beta."""
    scores = list(scores)
    if not scores:
        raise ValueError("scores must be non-empty")
    _check_alpha_beta(alpha, beta)
    res = tiers_from_scores_batched(np.asarray(scores, np.float64), alpha, beta)
    st = res.stats[0].cpu().numpy()
    return float(st[2]), float(st[3])


def assign_tiers(scores, t_low, t_high) -> list:
    """retrieval.py:240-250: strict rule; scores equal to a threshold fall to INT4."""
    scores = np.asarray(list(scores), np.float64)
    if scores.size == 0:
        return []
    res = assign_tiers_batched(scores.reshape(1, -1), np.array([[float(t_low), float(t_high)]]))
    return [Tier.from_code(c) for c in res.tiers[0].cpu().numpy()]


def assign_tiers_batched(scores, thresholds, seq_chunks=None) -> SearchResult:
    """Strict three-way rule + stable grouping for given scores [B, N] and thresholds [B, 2]."""
    s = kernels.to_dev(scores, torch.float64)
    t = kernels.to_dev(thresholds, torch.float64)
    B, N = s.shape
    dev = s.device
    sc = kernels.to_dev(seq_chunks, torch.int32) if seq_chunks is not None else None
    res = SearchResult(
        scores=s,
        stats=torch.empty((B, 4), dtype=torch.float64, device=dev),
        tiers=torch.zeros((B, N), dtype=torch.uint8, device=dev),
        perm=torch.zeros((B, N), dtype=torch.int32, device=dev),
        seg_counts=torch.zeros((B, 3), dtype=torch.int32, device=dev),
        flags=torch.zeros(B, dtype=torch.int32, device=dev),
    )
    _lib.call("ckv_assign_tiers", _lib.ptr(s), _lib.ptr(t), _lib.ptr(sc), B, N, _lib.ptr(res.tiers),
              _lib.ptr(res.perm), _lib.ptr(res.seg_counts), _lib.ptr(res.stats), _lib.ptr(res.flags),
              _lib.stream())
    return res


@dataclass(frozen=True)
class SimilarityReport:
    """retrieval.py:253-264."""

    scores: tuple
    s_min: float
    s_max: float
    alpha: float
    beta: float
    t_low: float
    t_high: float
    tiers: tuple


def build_similarity_report(scores, alpha, beta) -> SimilarityReport:
    """retrieval.py:267-279, one device pass (thresholds + tiers)."""
    scores = list(scores)
    if not scores:
        raise ValueError("scores must be non-empty")
    _check_alpha_beta(alpha, beta)
    res = tiers_from_scores_batched(np.asarray(scores, np.float64), alpha, beta)
    st = res.stats[0].cpu().numpy()
    tiers = tuple(Tier.from_code(c) for c in res.tiers[0].cpu().numpy())
    return SimilarityReport(
        scores=tuple(float(s) for s in scores),
        s_min=float(st[0]), s_max=float(st[1]), alpha=float(alpha), beta=float(beta),
        t_low=float(st[2]), t_high=float(st[3]), tiers=tiers,
    )
