"""CPU ORACLE — test infrastructure only.

A numpy restatement of the chunkkv reference algorithm for the Cocktail
hot path (chunk search, tier-contiguous reorder + INT2/INT4 pack, blocked
mixed-precision decode attention).  It is the CHECKER for the CUDA path:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import it.  Nothing in ``paper_2503_23294_b200`` imports or calls it.

Pinning: every function here is checked against golden vectors produced by
the reference itself (``tests/golden/make_golden.py`` imports chunkkv from
/root/reference in the build container) and against the reference's own
frozen known-answer tests (``tests/test_oracle.py``).

All arithmetic is float64 with the reference's expression trees; numpy
never contracts a*b+c into an FMA, matching the reference's
``-ffp-contract=off`` Cython build (``pkg/setup.py:22-24``).
"""

from __future__ import annotations

import math

import numpy as np

ALLOWED_BITS = (2, 4)  # kernels/__init__.py:41
TIER_INT2, TIER_INT4, TIER_FP16 = 0, 1, 2  # tiers.py:6-15 (u8 codes on the GPU)


def _check_bits(bits):
    # kernels/_numpy.py:14-16
    if bits not in ALLOWED_BITS:
        raise ValueError(f"bitwidth must be one of {ALLOWED_BITS}, got {bits}")


def _group_lengths(cols, group_size):
    # kernels/_numpy.py:19-24
    n_groups = -(-cols // group_size)
    lengths = np.full(n_groups, group_size, dtype=np.int64)
    lengths[-1] = cols - (n_groups - 1) * group_size
    return lengths


def quantize_groups(x, bits, group_size):
    """kernels/_numpy.py:27-67 (== _core.pyx:27-79 bit for bit)."""
    _check_bits(bits)
    if group_size < 1:
        raise ValueError("group_size must be >= 1")
    x = np.ascontiguousarray(x, dtype=np.float64)
    rows, cols = x.shape
    qmax = float(2**bits - 1)
    if rows == 0 or cols == 0:
        gpr = -(-cols // group_size) if cols else 0
        return (np.zeros((rows, cols), np.uint8), np.zeros(rows * gpr), np.zeros(rows * gpr))
    lengths = _group_lengths(cols, group_size)
    starts = np.arange(lengths.shape[0], dtype=np.int64) * group_size
    mins = np.minimum.reduceat(x, starts, axis=1)
    maxs = np.maximum.reduceat(x, starts, axis=1)
    span = maxs - mins
    m = np.repeat(mins, lengths, axis=1)
    r = np.repeat(span, lengths, axis=1)
    live = r > 0.0
    safe = np.where(live, r, 1.0)
    codes = np.floor((x - m) * qmax / safe + 0.5)  # _numpy.py:61 / _core.pyx:72
    np.clip(codes, 0.0, qmax, out=codes)
    codes = np.where(live, codes, 0.0).astype(np.uint8)
    return codes, (span / qmax).reshape(-1), mins.reshape(-1)


def pack_codes(codes, bits):
    """kernels/_numpy.py:70-86: element i at bits [i*b, (i+1)*b) of LE u32 word i*b//32."""
    _check_bits(bits)
    codes = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    n = codes.shape[0]
    per_word = 32 // bits
    n_words = -(-n * bits // 32)
    padded = np.zeros(n_words * per_word, dtype=np.uint32)
    padded[:n] = codes
    shifts = np.arange(per_word, dtype=np.uint32) * np.uint32(bits)
    return np.bitwise_or.reduce(padded.reshape(n_words, per_word) << shifts, axis=1).astype(np.uint32)


def unpack_codes(packed, bits, count):
    """kernels/_numpy.py:89-99."""
    _check_bits(bits)
    packed = np.ascontiguousarray(packed, dtype=np.uint32)
    per_word = 32 // bits
    if count > packed.shape[0] * per_word:
        raise ValueError("count exceeds packed capacity")
    shifts = np.arange(per_word, dtype=np.uint32) * np.uint32(bits)
    mask = np.uint32((1 << bits) - 1)
    return ((packed[:, None] >> shifts) & mask).astype(np.uint8).reshape(-1)[:count]


def dequantize_codes(packed, scales, zero_points, rows, cols, bits, group_size):
    """kernels/_numpy.py:102-112: zero_point[g] + scale[g] * code (no FMA)."""
    codes = unpack_codes(packed, bits, rows * cols).reshape(rows, cols).astype(np.float64)
    if rows == 0 or cols == 0:
        return codes
    lengths = _group_lengths(cols, group_size)
    ng = lengths.shape[0]
    s = np.repeat(np.asarray(scales, np.float64).reshape(rows, ng), lengths, axis=1)
    z = np.repeat(np.asarray(zero_points, np.float64).reshape(rows, ng), lengths, axis=1)
    return z + s * codes


# Optional compiled backend: the reference's own chunkkv.kernels._core (oracle/ref_core.py),
# the "compiled" side of the reference's import-time backend choice (kernels/__init__.py:18-39).
_KERNELS = None


def use_reference_kernels(mod):
    """Route matmul_packed (the decode's hot op, attention.py:75-90) through the reference's
    compiled module `mod` (None: the numpy restatement)."""
    global _KERNELS
    _KERNELS = mod


def matmul_packed(a, packed, scales, zero_points, rows, cols, bits, group_size, transpose):
    """kernels/_numpy.py:115-125 (or the reference's compiled _core.pyx:148-192 when selected)."""
    if _KERNELS is not None:
        return _KERNELS.matmul_packed(np.ascontiguousarray(a, dtype=np.float64), packed, scales, zero_points,
                                      rows, cols, bits, group_size, bool(transpose))
    a = np.ascontiguousarray(a, dtype=np.float64)
    inner = cols if transpose else rows
    if a.ndim != 2 or a.shape[1] != inner:
        raise ValueError("inner dimension mismatch")
    deq = dequantize_codes(packed, scales, zero_points, rows, cols, bits, group_size)
    return a @ (deq.T if transpose else deq)


class Block:
    """quantizer.QuantizedBlock (quantizer.py:20-57), minus validation."""

    def __init__(self, rows, cols, bitwidth, group_size, packed, scales, zero_points):
        self.rows, self.cols, self.bitwidth, self.group_size = rows, cols, bitwidth, group_size
        self.packed, self.scales, self.zero_points = packed, scales, zero_points


def quantize(matrix, bitwidth, group_size=32):
    """quantizer.py:60-83."""
    arr = np.ascontiguousarray(matrix, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("expected a 2D matrix")
    if arr.size and not np.isfinite(arr).all():
        raise ValueError("matrix contains non-finite values")
    codes, scales, zps = quantize_groups(arr, bitwidth, group_size)
    packed = pack_codes(codes.reshape(-1), bitwidth)
    return Block(arr.shape[0], arr.shape[1], bitwidth, group_size, packed, scales, zps)


def dequantize(block):
    """quantizer.py:86-96."""
    return dequantize_codes(block.packed, block.scales, block.zero_points, block.rows,
                            block.cols, block.bitwidth, block.group_size)


def fqm(a, block, transpose_block=False):
    """quantizer.py:99-123."""
    return matmul_packed(a, block.packed, block.scales, block.zero_points, block.rows,
                         block.cols, block.bitwidth, block.group_size, bool(transpose_block))


# -- search (retrieval.py) ----------------------------------------------------

def score_chunks(q_vec, q_norm, c_vecs, c_norms):
    """retrieval.py:199-219: cosine per chunk; zero-norm chunks take min(valid) (0.0 if none)."""
    if q_norm == 0.0:
        raise ValueError("query embedding has zero norm")
    c_vecs = np.asarray(c_vecs, np.float64)
    raw = []
    for vec, nrm in zip(c_vecs, c_norms):
        raw.append(float(q_vec @ vec / (q_norm * nrm)) if nrm > 0.0 else None)
    valid = [s for s in raw if s is not None]
    floor = min(valid) if valid else 0.0
    return [s if s is not None else floor for s in raw]


def compute_thresholds(scores, alpha, beta):
    """retrieval.py:222-237 (two roundings each, no FMA)."""
    scores = list(scores)
    if not scores:
        raise ValueError("scores must be non-empty")
    if not (0.0 <= alpha <= 1.0 and 0.0 <= beta <= 1.0):
        raise ValueError("alpha and beta must lie in [0, 1]")
    s_min, s_max = min(scores), max(scores)
    if alpha + beta > 1.0 and s_max > s_min:
        raise ValueError("alpha + beta > 1 makes the thresholds cross")
    return s_min + (s_max - s_min) * alpha, s_max - (s_max - s_min) * beta


def assign_tiers(scores, t_low, t_high):
    """retrieval.py:240-250: strict rule, ties to INT4.  Returns u8 tier codes."""
    out = []
    for s in scores:
        out.append(TIER_INT2 if s < t_low else (TIER_FP16 if s > t_high else TIER_INT4))
    return np.array(out, dtype=np.uint8)


def stable_perm(tiers):
    """kv_store.py:190-192,204-206: perm = INT2 ids || INT4 ids || FP16 ids (stable)."""
    tiers = np.asarray(tiers, np.uint8)
    idx = np.arange(tiers.shape[0], dtype=np.uint32)
    perm = np.concatenate([idx[tiers == t] for t in (TIER_INT2, TIER_INT4, TIER_FP16)])
    counts = np.array([(tiers == t).sum() for t in (TIER_INT2, TIER_INT4, TIER_FP16)], np.int32)
    return perm.astype(np.uint32), counts


# -- cache build (kv_store.py) -------------------------------------------------

class Cache:
    """kv_store.ChunkedKVCache (kv_store.py:24-166): arenas in tier order."""

    def __init__(self, chunk_size, head_dim, group_size, context_len, perm, k_q2, v_q2, k_q4, v_q4, k_fp, v_fp):
        self.chunk_size, self.head_dim, self.group_size = chunk_size, head_dim, group_size
        self.context_len, self.perm = context_len, np.asarray(perm, np.uint32)
        self.k_q2, self.v_q2, self.k_q4, self.v_q4 = k_q2, v_q2, k_q4, v_q4
        self.k_fp = np.asarray(k_fp, np.float64).reshape(-1, head_dim)
        self.v_fp = np.asarray(v_fp, np.float64).reshape(-1, head_dim)

    @property
    def len_2(self):
        return self.k_q2.rows

    @property
    def len_4(self):
        return self.k_q4.rows

    @property
    def len_fp(self):
        return self.k_fp.shape[0]

    @property
    def n_chunks(self):
        return self.perm.shape[0]

    @property
    def total_tokens(self):
        return self.len_2 + self.len_4 + self.len_fp

    def append(self, k_vec, v_vec):
        # kv_store.py:135-148
        self.k_fp = np.vstack([self.k_fp, np.asarray(k_vec, np.float64).reshape(1, -1)])
        self.v_fp = np.vstack([self.v_fp, np.asarray(v_vec, np.float64).reshape(1, -1)])


def build_cache(k, v, tiers, chunk_size, group_size=32):
    """kv_store.py:169-219.  tiers: u8 codes per full chunk; rows past n*chunk_size are the tail."""
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    tiers = np.asarray(tiers, np.uint8)
    n = tiers.shape[0]
    cs = chunk_size
    head_dim = k.shape[1]
    perm, counts = stable_perm(tiers)

    def gather_from(mat, idxs):  # kv_store.py:194-197
        if len(idxs) == 0:
            return np.zeros((0, head_dim))
        return np.concatenate([mat[i * cs:(i + 1) * cs] for i in idxs])

    by = [perm[:counts[0]], perm[counts[0]:counts[0] + counts[1]], perm[counts[0] + counts[1]:]]
    k_fp = np.concatenate([gather_from(k, by[2]), k[n * cs:]])
    v_fp = np.concatenate([gather_from(v, by[2]), v[n * cs:]])
    return Cache(cs, head_dim, group_size, k.shape[0], perm,
                 quantize(gather_from(k, by[0]), 2, group_size), quantize(gather_from(v, by[0]), 2, group_size),
                 quantize(gather_from(k, by[1]), 4, group_size), quantize(gather_from(v, by[1]), 4, group_size),
                 k_fp, v_fp)


def token_order(cache):
    """kv_store.py:227-233."""
    cs = cache.chunk_size
    parts = [np.arange(o * cs, (o + 1) * cs) for o in cache.perm.tolist()]
    parts.append(np.arange(cache.n_chunks * cs, cache.context_len))
    decode_len = cache.len_fp - (cache.n_chunks * cs - cache.len_2 - cache.len_4) - (cache.context_len - cache.n_chunks * cs)
    parts.append(np.arange(cache.context_len, cache.context_len + decode_len))
    return np.concatenate(parts).astype(np.int64)


def reconstruct(cache):
    """kv_store.py:236-253."""
    rk = np.concatenate([dequantize(cache.k_q2), dequantize(cache.k_q4), cache.k_fp])
    rv = np.concatenate([dequantize(cache.v_q2), dequantize(cache.v_q4), cache.v_fp])
    order = token_order(cache)
    k = np.zeros_like(rk)
    v = np.zeros_like(rv)
    k[order] = rk
    v[order] = rv
    return k, v


# -- attention (attention.py) --------------------------------------------------

def stable_softmax(x, axis=-1):
    """attention.py:24-31."""
    m = np.max(x, axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / np.sum(e, axis=axis, keepdims=True)


def mixed_decode_attention(q, cache, mask=None, scale=None):
    """attention.py:63-90: per-tier QK^T, concat, scale, mask, one softmax, PV summed INT2->INT4->FP16."""
    if cache.total_tokens == 0:
        raise ValueError("cache holds no tokens")
    q = np.ascontiguousarray(q, np.float64)
    if scale is None:
        scale = 1.0 / math.sqrt(cache.head_dim)
    att = np.concatenate([fqm(q, cache.k_q2, True), fqm(q, cache.k_q4, True), q @ cache.k_fp.T], axis=1)
    att *= scale
    if mask is not None:
        att = att + mask
    w = stable_softmax(att, axis=1)
    n2, n4 = cache.len_2, cache.len_4
    return fqm(w[:, :n2], cache.v_q2) + fqm(w[:, n2:n2 + n4], cache.v_q4) + w[:, n2 + n4:] @ cache.v_fp


def reference_attention(q, k, v, mask=None, scale=None):
    """attention.py:93-112."""
    q = np.ascontiguousarray(q, np.float64)
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    att = q @ np.asarray(k, np.float64).T
    att *= scale
    if mask is not None:
        att = att + mask
    return stable_softmax(att, axis=1) @ np.asarray(v, np.float64)


# -- batched GPU-format restatement (test helpers) -------------------------------

def arena_meta_lohi(x_fp16_rows, group_size=32):
    """(lo, hi) per (row, group) as float16, the GPU metadata format.

    Since fp16 differences are exact in f64, scale = (f64(hi)-f64(lo))/qmax and
    zp = f64(lo) reproduce quantize_groups' f64 metadata bit for bit.
    """
    x = np.asarray(x_fp16_rows, np.float16).astype(np.float64)
    r, c = x.shape
    g = x.reshape(r, c // group_size, group_size)
    return np.stack([g.min(axis=2), g.max(axis=2)], axis=-1).astype(np.float16)


def lse_merge(ms, ls, accs):
    """Split-KV merge of partial (m, l, acc) (log2 domain): o = sum acc_p 2^(m_p-m*) / sum l_p 2^(m_p-m*)."""
    ms = np.asarray(ms, np.float64)
    mstar = ms.max(axis=0)
    w = np.exp2(ms - mstar)
    den = (np.asarray(ls, np.float64) * w).sum(axis=0)
    num = (np.asarray(accs, np.float64) * w[..., None]).sum(axis=0)
    return num / den[..., None]


# -- text encoders upstream of the search (retrieval.py:70-138) --------------------------

def bow_encode(text, dim=256, seed=0):
    """HashedBowEncoder.encode (retrieval.py:87-100): keyed BLAKE2b-64 per whitespace word
    (hashlib, the reference's own hash), sign from bit 63, bucket h % dim, L2-normalised."""
    import hashlib

    key = str(int(seed)).encode("ascii")
    vec = np.zeros(dim, dtype=np.float64)
    for word in text.split():
        h = int.from_bytes(hashlib.blake2b(word.encode("utf-8"), key=key, digest_size=8).digest(), "little")
        vec[h % dim] += -1.0 if h >> 63 else 1.0
    norm = float(np.linalg.norm(vec))
    if norm > 0.0:
        return vec / norm, 1.0
    return vec, norm


def tfidf_fit(texts):
    """TfidfEncoder.fit (retrieval.py:111-120) -> (word -> index, idf)."""
    texts = list(texts)
    vocab = sorted({w for t in texts for w in t.split()})
    index = {w: i for i, w in enumerate(vocab)}
    df = np.zeros(len(vocab), dtype=np.float64)
    for t in texts:
        for w in set(t.split()):
            df[index[w]] += 1.0
    return index, np.log((1.0 + len(texts)) / (1.0 + df)) + 1.0


def tfidf_encode(text, index, idf):
    """TfidfEncoder.encode (retrieval.py:122-138)."""
    vec = np.zeros(len(index), dtype=np.float64)
    for w in text.split():
        i = index.get(w)
        if i is not None:
            vec[i] += 1.0
    vec *= idf
    norm = float(np.linalg.norm(vec))
    if norm > 0.0:
        return vec / norm, 1.0
    return vec, norm
