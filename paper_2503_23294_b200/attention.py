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
    cache = inst.cache
    if cache.total_tokens == 0:
        raise ValueError("cache holds no tokens")
    q = kernels.to_dev(inst.q, torch.float64)
    m = q.shape[0]
    n2, n4, nf = cache.len_2, cache.len_4, cache.len_fp
    total = n2 + n4 + nf
    kfp, vfp = cache.fp_device()
    att = torch.empty((m, total), dtype=torch.float64, device=q.device)
    quantizer.fqm_dev(q, cache.k_q2, True, out=att[:, :n2])            # attention.py:75
    quantizer.fqm_dev(q, cache.k_q4, True, out=att[:, n2:n2 + n4])     # attention.py:76
    kernels.matmul_dev(q, kfp, True, out=att[:, n2 + n4:])             # attention.py:77
    mask = kernels.to_dev(inst.mask, torch.float64) if inst.mask is not None else None
    _softmax_dev(att, inst.scale, mask)                                # attention.py:79-82
    out = torch.empty((m, cache.head_dim), dtype=torch.float64, device=q.device)
    quantizer.fqm_dev(att[:, :n2], cache.v_q2, False, out=out)          # attention.py:90
    quantizer.fqm_dev(att[:, n2:n2 + n4], cache.v_q4, False, out=out, accumulate=True)
    kernels.matmul_dev(att[:, n2 + n4:], vfp, False, out=out, accumulate=True)
    return out.cpu().numpy()


def reference_attention(q, k, v, mask=None, scale=None) -> np.ndarray:
    """attention.py:93-112: naive softmax(scale * q @ k.T + mask) @ v in float64 (GPU)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ValueError("q, k, v must be 2D")
    if q.shape[1] != k.shape[1] or k.shape[0] != v.shape[0]:
        raise ValueError("attention shape mismatch")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[1])
    if mask is not None:
        mask = np.asarray(mask, dtype=np.float64)
        if mask.shape != (q.shape[0], k.shape[0]):
            raise ValueError("mask shape must be (m, tokens)")
    qd, kd, vd = (kernels.to_dev(x, torch.float64) for x in (q, k, v))
    att = kernels.matmul_dev(qd, kd, True)
    _softmax_dev(att, scale, kernels.to_dev(mask, torch.float64) if mask is not None else None)
    return kernels.matmul_dev(att, vd, False).cpu().numpy()


def causal_mask(n) -> np.ndarray:
    """attention.py:115-117."""
    return np.triu(np.full((n, n), -np.inf), k=1)
