"""Blocked mixed-precision decode attention — drop-in for ``chunkkv.attention``
(attention.py:1-112), per head, float64, on the GPU.

``mixed_decode_attention`` keeps the reference's blocked structure (per-tier q.K^T via
the packed matmul kernel, one scaled+masked softmax, per-tier P.V accumulated
INT2 -> INT4 -> FP16) so results match the reference to f64 accumulation order.  The
fp16 batched hot path (online softmax, split-KV, tensor cores) is
``paper_2503_23294_b200.batched.decode``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, kernels, quantizer
from .kv_store import ChunkedKVCache


def _softmax_dev(x, scale=1.0, mask=None):
    _lib.call("ckv_scale_mask_softmax_f64", _lib.ptr(x), x.shape[0], x.shape[1], float(scale),
              _lib.ptr(mask), _lib.stream())
    return x


def stable_softmax(x, axis=-1):
    """attention.py:24-31 (row softmax; -inf entries get weight 0), on the GPU."""
    arr = np.asarray(x, dtype=np.float64)
    if arr.ndim == 1:
        return stable_softmax(arr[None, :], axis=-1)[0]
    if arr.ndim != 2:
        raise ValueError("stable_softmax expects a 1D or 2D array")
    transposed = axis in (0, -2)
    xd = kernels.to_dev(arr.T if transposed else arr, torch.float64)
    out = _softmax_dev(xd).cpu().numpy()
    return out.T if transposed else out


@dataclass
class AttentionInstance:
    """attention.py:34-60."""

    q: np.ndarray
    cache: ChunkedKVCache
    mask: np.ndarray = None
    scale: float = field(default=None)

    def __post_init__(self):
        self.q = np.ascontiguousarray(self.q, dtype=np.float64)
        if self.q.ndim != 2:
            raise ValueError("q must be 2D (m x head_dim)")
        if self.q.shape[1] != self.cache.head_dim:
            raise ValueError("q width != cache head_dim")
        if self.scale is None:
            self.scale = 1.0 / math.sqrt(self.cache.head_dim)
        if self.mask is not None:
            self.mask = np.asarray(self.mask, dtype=np.float64)
            if self.mask.shape != (self.q.shape[0], self.cache.total_tokens):
                raise ValueError("mask shape must be (m, total_tokens)")


def mixed_decode_attention(inst: AttentionInstance) -> np.ndarray:
    """attention.py:63-90 on the GPU (f64)."""
    if inst.cache.total_tokens == 0:
        raise ValueError("cache holds no tokens")
    mask = kernels.to_dev(inst.mask, torch.float64) if inst.mask is not None else None
    return mixed_decode_dev(kernels.to_dev(inst.q, torch.float64), inst.cache, inst.scale, mask).cpu().numpy()


def mixed_decode_dev(q, cache: ChunkedKVCache, scale, mask=None, out=None):
    """The blocked attention of ``mixed_decode_attention`` on device tensors (q f64 [m, d] on
    the GPU, optional f64 mask on the GPU) -> f64 [m, d] on the GPU (into ``out`` if given)."""
    m = q.shape[0]
    n2, n4, nf = cache.len_2, cache.len_4, cache.len_fp
    total = n2 + n4 + nf
    kfp, vfp = cache.fp_device()
    att = torch.empty((m, total), dtype=torch.float64, device=q.device)
    quantizer.fqm_dev(q, cache.k_q2, True, out=att[:, :n2])            # attention.py:75
    quantizer.fqm_dev(q, cache.k_q4, True, out=att[:, n2:n2 + n4])     # attention.py:76
    kernels.matmul_dev(q, kfp, True, out=att[:, n2 + n4:])             # attention.py:77
    _softmax_dev(att, scale, mask)                                     # attention.py:79-82
    if out is None:
        out = torch.empty((m, cache.head_dim), dtype=torch.float64, device=q.device)
    quantizer.fqm_dev(att[:, :n2], cache.v_q2, False, out=out)          # attention.py:90
    quantizer.fqm_dev(att[:, n2:n2 + n4], cache.v_q4, False, out=out, accumulate=True)
    kernels.matmul_dev(att[:, n2 + n4:], vfp, False, out=out, accumulate=True)
    return out


def reference_attention(q, k, v, mask=None, scale=None) -> np.ndarray:
    """attention.py:93-112: naive softmax(scale * q @ k.T + mask) @ v in float64 (GPU)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ValueError("q, k, v must be 2D")
    if q.shape[1] != k.shape[1] or k.shape[0] != v.shape[0]:
        raise ValueError("attention shape mismatch")
    if mask is not None:
        mask = np.asarray(mask, dtype=np.float64)
        if mask.shape != (q.shape[0], k.shape[0]):
            raise ValueError("mask shape must be (m, tokens)")
    qd, kd, vd = (kernels.to_dev(x, torch.float64) for x in (q, k, v))
    md = kernels.to_dev(mask, torch.float64) if mask is not None else None
    return reference_attention_dev(qd, kd, vd, md, scale).cpu().numpy()


def reference_attention_dev(q, k, v, mask=None, scale=None, out=None):
    """``reference_attention`` on device f64 tensors (column slices allowed: rows are strided)."""
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    att = kernels.matmul_dev(q, k, True)
    _softmax_dev(att, scale, mask)
    return kernels.matmul_dev(att, v, False, out=out)


def causal_mask(n) -> np.ndarray:
    """attention.py:115-117."""
    return np.triu(np.full((n, n), -np.inf), k=1)


def prefill_attention(embeddings, model, return_hidden=False):
    """attention.py:120-145: single-layer causal self-attention over the prompt of the toy
    model, on the GPU in f64.  Returns the full-precision K and V projections (tokens x
    embed_dim, heads side by side), the last position's logits and optionally the hidden
    states (embeddings + concatenated head outputs)."""
    emb = np.ascontiguousarray(embeddings, dtype=np.float64)
    if emb.ndim != 2 or emb.shape[1] != model.embed_dim:
        raise ValueError("embeddings must be (tokens, embed_dim)")
    n, d = emb.shape[0], model.head_dim
    if n == 0:  # the reference fails on logits[-1] of an empty prompt
        raise IndexError("index -1 is out of bounds for axis 0 with size 0")
    w = model.device_weights()
    e = kernels.to_dev(emb, torch.float64)
    q, k, v = (kernels.matmul_dev(e, w[name], False) for name in ("w_q", "w_k", "w_v"))
    mask = kernels.to_dev(causal_mask(n), torch.float64)
    hidden = e.clone()
    for h in range(model.n_heads):
        cols = slice(h * d, (h + 1) * d)
        hidden[:, cols] += reference_attention_dev(q[:, cols], k[:, cols], v[:, cols], mask)
    logits = kernels.matmul_dev(hidden, w["w_o"], False)
    k_h, v_h = k.cpu().numpy(), v.cpu().numpy()
    last = logits[-1].cpu().numpy()
    if return_hidden:
        return k_h, v_h, last, hidden.cpu().numpy()
    return k_h, v_h, last
