"""Chunk-level quantization search (Module I) — drop-in for the scoring half of
``chunkkv.retrieval`` (retrieval.py:17-67, 199-279), computed by the ckv_search kernel.

Text encoders (HashedBow/TF-IDF/precomputed, retrieval.py:70-191) produce the kernel's
*input* embeddings on the host; they are outside this hot path and not
rebuilt.  ``Embedding`` and ``segment_context`` are kept as plain host types because
build_cache's signature uses them.

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
