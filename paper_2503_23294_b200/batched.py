"""Batched fp16 hot path: the B200-resident chunked KV cache for all
(layer, sequence, kv-head) units of a model, head_dim 128, group 32, chunk 32.

Pipeline (one launch each, everything stays in HBM):

  search_batched(...)           -> tiers, perm, per-tier counts     (retrieval.py:199-250)
  BatchedKVCache.build(k, v, s) -> INT2/INT4 arenas + FP16 region    (kv_store.py:169-219)
  cache.decode(q)               -> attention output per q head       (attention.py:63-90)
  cache.append(k_new, v_new)    -> decode-token append               (kv_store.py:135-148)

HBM layout (see include/ckv.h ckv_arena):
  tiles2 u8 [L][H][rows2/16][1536]  = per 16-row INT2 tile [K codes | V codes | K meta | V meta]
  tiles4 u8 [L][H][rows4/16][2560]  = the same for INT4
  fp     fp16 [L][H][rows_fp][128]  per K and V
Rows of one sequence are contiguous inside each arena (varlen concatenation over the
batch); the per-sequence table seq i32 [B][8] holds the offsets and lengths.  Quantized
tiles hold exactly the bits of the reference's pack_codes rows and (lo, hi) metadata,
permuted into the decode kernel's fragment order (tile-native layout, csrc/ckv_common.cuh);
export_unit restores reference rows on the device (ckv_arena_export).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import ctypes

import numpy as np
import torch

from . import _lib, kernels, quantizer
from .kv_store import ChunkedKVCache
from .quantizer import QuantizedBlock

HEAD_DIM = 128
GROUP = 32
CHUNK = 32
TILE = 16
BLOCK2 = 1536  # interleaved INT2 tile: K codes 512 | V codes 512 | K meta 256 | V meta 256
BLOCK4 = 2560  # interleaved INT4 tile: K codes 1024 | V codes 1024 | K meta 256 | V meta 256
# algorithmic bytes per token per kv-head, K+V (codes + fp16 (lo,hi) metadata)
BYTES_INT2 = 2 * (32 + 16)
BYTES_INT4 = 2 * (64 + 16)
BYTES_FP16 = 2 * 256


MAX_Q_PER_KV = 8  # q rows per kv head in one decode launch (the MMA's N columns)


def _round_up(x, m):
    return -(-x // m) * m


def _num_sms():
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def plan_layout(n2, n4, nfp, context_lens, decode_capacity=128, tail_src=None):
    """Host-side arena layout: the per-sequence table i32 [B, 8] (include/ckv.h) and the FP16
    region capacity per sequence (rounded to whole 16-token tiles)."""
    n2 = np.asarray(n2, np.int64).reshape(-1)
    n4 = np.asarray(n4, np.int64).reshape(-1)
    nfp = np.asarray(nfp, np.int64).reshape(-1)
    ctx = np.asarray(context_lens, np.int64).reshape(-1)
    if not (n2.size == n4.size == nfp.size == ctx.size):
        raise ValueError("per-sequence arrays must have equal length")
    if (n2 < 0).any() or (n4 < 0).any() or (nfp < 0).any():
        raise ValueError("negative chunk counts")
    tail = ctx - CHUNK * (n2 + n4 + nfp)
    if (tail < 0).any() or (tail >= CHUNK).any():
        raise ValueError("context_lens inconsistent with chunk counts")
    len2, len4 = n2 * CHUNK, n4 * CHUNK
    len_fp = nfp * CHUNK + tail
    cap_fp = np.array([_round_up(int(x) + int(decode_capacity), TILE) for x in len_fp], np.int64)
    excl = lambda a: np.concatenate([[0], np.cumsum(a)[:-1]]).astype(np.int64) if a.size else a  # noqa: E731
    tsrc = CHUNK * (n2 + n4 + nfp) if tail_src is None else np.asarray(tail_src, np.int64).reshape(-1)
    seq = np.stack([excl(len2), len2, excl(len4), len4, excl(cap_fp), len_fp, tsrc, ctx], axis=1)
    if seq.size and (seq[:, [0, 2, 4]].max() + np.maximum(cap_fp, np.maximum(len2, len4)).max() >= 2**31):
        raise ValueError("arena rows exceed int32 offsets")
    return seq.astype(np.int32).reshape(-1, 8), cap_fp


class BatchedKVCache:
    """Device-resident chunked KV cache for [layers, batch, kv_heads] units."""

    def __init__(self, layers, batch, kv_heads, n2, n4, nfp, context_lens, decode_capacity=128,
                 tail_src=None, device=None):
        self.L, self.B, self.H = int(layers), int(batch), int(kv_heads)
        dev = device or _lib.device()
        self.device = dev
        self.seq_host, self.cap_fp = plan_layout(n2, n4, nfp, context_lens, decode_capacity, tail_src)
        if self.seq_host.shape[0] != self.B:
            raise ValueError("per-sequence arrays must have length batch")
        self.rows2 = int(self.seq_host[:, 1].sum())
        self.rows4 = int(self.seq_host[:, 3].sum())
        self.rows_fp = int(self.cap_fp.sum())
        self.seq = torch.from_numpy(self.seq_host.copy()).to(dev)
        L, H = self.L, self.H
        z32 = lambda *s: torch.zeros(s, dtype=torch.int32, device=dev)  # noqa: E731
        u8 = lambda *s: torch.zeros(s, dtype=torch.uint8, device=dev)  # noqa: E731
        self.tiles2 = u8(L, H, self.rows2 // TILE, BLOCK2)
        self.tiles4 = u8(L, H, self.rows4 // TILE, BLOCK4)
        self.k = dict(fp=torch.zeros((L, H, self.rows_fp, HEAD_DIM), dtype=torch.float16, device=dev),
                      span_flags=z32(L, H, self.B), span_max=z32(L, H, self.B))
        self.v = {k: torch.zeros_like(t) for k, t in self.k.items()}
        self._ws, self._ws_ptr = {}, {}
        self._arenas = {}
        self._perm = None
        self._wp = {}  # warp plans per sequence range (b0, b1)
        # decode schedule of whole-batch launches: "wp" (warp plan: one 16-warp CTA per SM,
        # units split at warp granularity), "split" (4-warp CTAs, `splits` per unit) or "auto"
        # (the warp plan unless the cache is small, fewer than 8 tiles per warp, or more than half
        # of its bytes are FP16)
        self.schedule = "auto"
        self._any_empty = bool((self.total_tokens() == 0).any())
        # micro-batch chains: per-layer launches of a chain as programmatic dependents (PDL).  An
        # early-launched CTA holds an SM slot while it waits for its chain's previous layer (22 %
        # of CTA residency, tools/chain_timeline.py), yet PDL still wins: cfg2 8 chains 4706 vs
        # 4515 GB/s without (launch gaps then leave slots empty: 2.76 vs 3.55 resident of 4)
        self.chain_pdl = os.environ.get("CKV_CHAIN_PDL", "1") == "1"

    # -- construction ------------------------------------------------------------------
    @classmethod
    def from_search(cls, k, v, search, context_lens=None, decode_capacity=128, check=True):
        """Build from fp16 K/V [L, B, T, H, 128] (any strides, head_dim contiguous) and a
        SearchResult (perm + seg_counts on the device).  One host sync for the layout."""
        L, B, T, H, D = k.shape
        if D != HEAD_DIM:
            raise ValueError(f"batched path requires head_dim {HEAD_DIM}")
        counts = search.seg_counts.cpu().numpy().astype(np.int64)
        ctx = np.full(B, T, np.int64) if context_lens is None else np.asarray(context_lens, np.int64)
        cache = cls(L, B, H, counts[:, 0], counts[:, 1], counts[:, 2], ctx, decode_capacity,
                    device=k.device)
        cache.build(k, v, search.perm, check=check)
        return cache

    def arena(self, which, layer=0):
        """ckv_arena view starting at `layer` (per-layer launches index layers from there):
        codes/meta pointers into the interleaved tile buffers (K at block offsets 0 / 2x codes,
        V one code tile / one meta tile further).  Cached: the buffers never move."""
        key = (which, layer)
        cached = self._arenas.get(key)
        if cached is None:
            cached = self._arenas[key] = self._make_arena(which, layer)
        return cached

    def _make_arena(self, which, layer):
        t = self.k if which == "k" else self.v
        ptr = lambda x: x.data_ptr() + layer * x.stride(0) * x.element_size()  # noqa: E731
        v = which == "v"
        b2, b4 = ptr(self.tiles2), ptr(self.tiles4)
        return _lib.Arena(b2 + (512 if v else 0), b2 + 1024 + (256 if v else 0),
                          b4 + (1024 if v else 0), b4 + 2048 + (256 if v else 0), ptr(t["fp"]),
                          ptr(t["span_flags"]), ptr(t["span_max"]), self.rows2, self.rows4, self.rows_fp)

    def build(self, k, v, perm, check=True, layer=0):
        """ckv_reorder_quantize_pack over every unit of layers [layer, layer + L'); k, v fp16
        [L', B, T, H, 128] (L' = L for the whole cache at once, or a slice so that a cache
        larger than its fp16 source can be built layer by layer); perm i32/u32 [B, max_chunks]."""
        if k.dtype != torch.float16 or v.dtype != torch.float16:
            raise ValueError("batched build expects fp16 K/V")
        if k.shape != v.shape or k.stride() != v.stride():
            raise ValueError("k and v must have equal shape and strides")
        L, B, T, H, D = k.shape
        if layer < 0 or layer + L > self.L or (B, H) != (self.B, self.H) or D != HEAD_DIM or k.stride(4) != 1:
            raise ValueError("K/V shape does not match the cache")
        perm = kernels.to_dev(perm, torch.int32)
        self._perm = perm  # the build permutation (source chunk per slot), for export_unit
        for t in (self.k, self.v):
            t["span_flags"][layer:layer + L].zero_()
            t["span_max"][layer:layer + L].zero_()
        flag = torch.zeros(1, dtype=torch.int32, device=k.device)
        _lib.call("ckv_reorder_quantize_pack", _lib.ptr(k), _lib.ptr(v), L, B, H, k.stride(0),
                  k.stride(1), k.stride(2), k.stride(3), _lib.ptr(perm), perm.shape[1],
                  _lib.ptr(self.seq), int(self.seq_host[:, 7].max()) if B else 0,
                  self.arena("k", layer), self.arena("v", layer), _lib.ptr(flag), _lib.stream())
        if check and int(flag.item()) & _lib.FLAG_NONFINITE:
            raise ValueError("matrix contains non-finite values")
        return self

    # -- decode ------------------------------------------------------------------------
    def total_tokens(self):
        s = self.seq_host
        return (s[:, 1] + s[:, 3] + s[:, 5]).astype(np.int64)

    def default_splits(self, m, layers=None):
        """Split-KV factor: the whole grid should fill whole waves of resident CTAs (a
        byte-balanced split makes every CTA equally long, so the tail is the partial wave),
        while keeping >= ~16 tiles per CTA so partial traffic stays negligible."""
        units = (self.L if layers is None else layers) * self.B * self.H
        per_sm = _lib.load().ckv_decode_ctas_per_sm()
        slots = _num_sms() * max(per_sm, 1)
        tiles = int(max(1, (self.total_tokens().max() + TILE - 1) // TILE))
        if units * tiles < 64 * _num_sms():
            # latency regime (a few tiles per warp, e.g. cfg1's 15 MB): about two CTAs per SM —
            # more splits add co-resident CTAs and merge work without adding bandwidth
            # (cfg1: 8 / 12 / 16 splits 16.5 / 16.8 / 22.0 us)
            return int(max(1, min(64, (2 * _num_sms()) // max(units, 1), tiles // 4)))
        best, best_cost = 1, None
        for s in range(1, 65):
            if s > 1 and tiles // s < 16:
                break
            waves = -(-units * s // slots)
            cost = waves / (units * s / slots) + 0.002 * s  # tail waste + merge overhead
            if best_cost is None or cost < best_cost - 1e-9:
                best, best_cost = s, cost
        return best

    def chain_splits(self, m):
        """Split-KV factor for micro-batch chains (concurrent per-range launches): the chains'
        launches together should slightly oversubscribe the resident CTA slots (~1.05x: CTAs of
        a later wave fill the gaps other chains' tails leave), with >= 16 tiles per CTA."""
        units = self.B * self.H
        slots = _num_sms() * max(_lib.load().ckv_decode_ctas_per_sm(), 1)
        tiles = int(max(1, (self.total_tokens().max() + TILE - 1) // TILE))
        s = max(1, min(64, -(-int(1.05 * slots) // max(units, 1))))
        while s > 1 and tiles // s < 16:
            s -= 1
        return s

    def warp_plan(self, seqs=None):
        """Warp-plan schedule (ckv_decode_attention_wp): unit u = b*H + h gets n_u warps in
        proportion to its tile cost (INT2 1, INT4 1.2, FP16-region 3 per 16-token tile, measured), at
        least 2, summing to 16 x the SM count; returns (plan table i32 on the device, ctas,
        max_slots, max_ctas) or None when the units do not fit (more than 8 per CTA).  Computed
        once per sequence range (``seqs`` = (b0, b1), default the whole batch; a range is one
        micro-batch chain's launches): any plan is exact, later appends only shift the balance
        slightly.  The table (ckv_decode_wp_plan, include/ckv.h) holds every warp's tile ranges
        and every CTA's unit slots, so a CTA's prologue needs no dependent loads."""
        key = (0, self.B) if seqs is None else (int(seqs[0]), int(seqs[1]))
        if key not in self._wp:
            plan, n = self._build_wp_plan(*key)
            self._wp[key] = plan
            if key == (0, self.B) and plan is not None:
                self.wp_unit_warps = n  # warps per unit (host copy, for reports)
        return self._wp[key]

    def _build_wp_plan(self, b0, b1):
        """(plan, warps per unit) for sequences [b0, b1), or (None, None)."""
        cw = _lib.load().ckv_decode_wp_cta_warps()  # warps per CTA (16 / cw CTAs per SM)
        T = 16 * _num_sms()
        n_cta = T // cw
        U = (b1 - b0) * self.H
        s = self.seq_host[b0:b1].astype(np.int64)
        # per-tile costs (INT2 1): INT4 1.2, FP16 region 3 — cfg2 lockstep 4485 GB/s with the
        # instruction-count ratios (1.06, 2), 4500-4504 anywhere in INT4 1.2-1.4 x FP16 2-4
        cost_b = s[:, 1] // TILE + 1.2 * (s[:, 3] // TILE) + 3.0 * (-(-s[:, 5] // TILE))
        cost = np.repeat(cost_b, self.H).astype(np.float64)
        if not (U and 2 * U <= T and cost.sum() > 0):
            return None, None
        raw = T * cost / cost.sum()
        n = np.maximum(np.floor(raw).astype(np.int64), 2)
        order = np.argsort(-(raw - np.floor(raw)), kind="stable")
        i = 0
        while n.sum() < T:
            n[order[i % U]] += 1
            i += 1
        while n.sum() > T:
            j = int(np.argmax(np.where(n > 2, n - raw, -np.inf)))
            n[j] -= 1
        lib = _lib.load()
        plan = np.zeros(int(lib.ckv_decode_wp_plan_ints(n_cta)), dtype=np.int32)
        seq = np.ascontiguousarray(self.seq_host[b0:b1], dtype=np.int32)
        nw = np.ascontiguousarray(n, dtype=np.int32)
        ms, mc = ctypes.c_int32(0), ctypes.c_int32(0)
        st = lib.ckv_decode_wp_plan(seq.ctypes.data, b1 - b0, self.H, nw.ctypes.data, n_cta,
                                    plan.ctypes.data, ctypes.byref(ms), ctypes.byref(mc))
        if st != 0:
            return None, None
        return (torch.from_numpy(plan).to(self.device), n_cta, ms.value, mc.value), n

    def _wp_workspace(self, m, layers, layer, max_ctas, seqs=None):
        sid = torch.cuda.current_stream(self.device).cuda_stream
        b0, b1 = (0, self.B) if seqs is None else seqs
        wkey = ("wp", m, layers, layer, b0, b1, sid)
        hit = self._ws_ptr.get(wkey)
        if hit is not None:
            return hit
        lib = _lib.load()
        per = lib.ckv_decode_wp_workspace_bytes(layers, b1 - b0, self.H, m, max_ctas)
        per = -(-per // 256) * 256
        key = ("wp", m, layers, b0, b1, sid)
        nbytes = per * (self.L if layers == 1 else 1)
        if key not in self._ws:
            self._ws[key] = torch.zeros(max(nbytes // 4, 1), dtype=torch.float32, device=self.device)
        self._ws_ptr[wkey] = ptr = self._ws[key].data_ptr() + (per * layer if layers == 1 else 0)
        return ptr

    def _use_wp(self, m, seqs, splits, schedule):
        sched = self.schedule if schedule is None else schedule
        if sched == "split" or splits is not None or m > MAX_Q_PER_KV:
            return None
        if sched == "auto" and seqs is not None and tuple(seqs) != (0, self.B):
            # a micro-batch chain's range: its launches run beside the other chains' launches,
            # which the one-CTA-per-SM warp plan cannot share SMs with (cfg2, 8 chains: split
            # 4641 vs warp plan 2907-3732 GB/s); the split schedule's 4-warp CTAs interleave
            return None
        if sched == "auto" and (self._tiles_per_warp() < 8 or self._fp16_byte_share() > 0.5):
            # small caches (a few tiles per warp): the split schedule's latency wins; mostly-FP16
            # caches are HBM bound, where SMs stream at unequal rates and the split schedule's
            # waves of CTAs rebalance dynamically (cfg4 all-FP16: split 6375 vs warp plan 5823 GB/s)
            return None
        return self.warp_plan(seqs)

    def _fp16_byte_share(self):
        s = self.seq_host.astype(np.float64)
        fp = 512.0 * s[:, 5].sum()
        tot = 96.0 * s[:, 1].sum() + 160.0 * s[:, 3].sum() + fp
        return fp / tot if tot > 0 else 0.0

    def _tiles_per_warp(self):
        s = self.seq_host.astype(np.int64)
        tiles = self.H * int((s[:, 1] // TILE + s[:, 3] // TILE + -(-s[:, 5] // TILE)).sum())
        return tiles / (16 * _num_sms())

    def _workspace(self, m, splits, layers, layer):
        """Zero-initialised decode workspace (split partials + self-resetting arrival counters).
        Launches covering a single layer get a private per-layer slice, so consecutive
        per-layer launches never share counters (required for programmatic dependent launch).
        Keyed by the current stream as well: decodes of one cache on concurrent streams never
        share counters (the C-ABI's re-entrancy is per stream, include/ckv.h)."""
        sid = torch.cuda.current_stream(self.device).cuda_stream
        wkey = (m, splits, layers, layer, sid)
        hit = self._ws_ptr.get(wkey)
        if hit is not None:
            return hit
        lib = _lib.load()
        if layers == self.L:
            key = (m, splits, "all", sid)
            nbytes = lib.ckv_decode_workspace_bytes(self.L, self.B, self.H, m, splits)
            off = 0
        else:
            key = (m, splits, "per-layer", layers, sid)
            per = lib.ckv_decode_workspace_bytes(layers, self.B, self.H, m, splits)
            per = -(-per // 256) * 256
            nbytes = per * self.L
            off = per * layer
        if key not in self._ws:
            self._ws[key] = torch.zeros(max(nbytes // 4, 1), dtype=torch.float32, device=self.device)
        self._ws_ptr[wkey] = ptr = self._ws[key].data_ptr() + off
        return ptr

    def decode(self, q, splits=None, out=None, scale=None, layer=0, pdl=False, seqs=None, schedule=None,
               heads=None):
        """Mixed-precision decode attention for q fp16 [L', B, H*m, 128] -> fp16 same shape,
        over layers [layer, layer + L') of the cache (L' = L for the whole model in one launch,
        1 for the per-layer launches of a real decode step).  pdl=True launches as a
        programmatic dependent of the previous kernel on the stream; use it only when that
        kernel was itself a decode of this cache (it overlaps this launch's K/V prefetch with
        the previous launch's tail).  seqs=(b0, b1) computes sequences [b0, b1) only (q / out
        keep the full batch; the other rows of out are left untouched), so disjoint sequence
        ranges can run as concurrent micro-batch chains; heads=(h0, h1) likewise restricts the
        launch to kv heads [h0, h1) (split kernel), so a batch-1 context can run as chains over
        its heads."""
        L, B, Hq, D = q.shape
        if B != self.B or layer < 0 or layer + L > self.L or D != HEAD_DIM or Hq % self.H:
            raise ValueError("q shape does not match the cache")
        if q.dtype != torch.float16 or q.stride(3) != 1 or q.stride(2) != HEAD_DIM:
            raise ValueError("q must be fp16 with contiguous heads")
        if self._any_empty:
            raise ValueError("cache holds no tokens")  # attention.py:71-72
        b0, b1 = (0, B) if seqs is None else (int(seqs[0]), int(seqs[1]))
        if not 0 <= b0 <= b1 <= B:
            raise ValueError("seqs must be a range inside the batch")
        h0, h1 = (0, self.H) if heads is None else (int(heads[0]), int(heads[1]))
        if not 0 <= h0 <= h1 <= self.H:
            raise ValueError("heads must be a range of the kv heads")
        m = Hq // self.H
        if out is None:
            out = torch.empty((L, B, Hq, D), dtype=torch.float16, device=q.device)
        elif (out.shape != q.shape or out.dtype != torch.float16 or out.device != q.device
              or out.stride(3) != 1 or out.stride(2) != HEAD_DIM):
            raise ValueError("out must be fp16 [L', B, H*m, 128] with contiguous heads on q's device")
        if m > MAX_Q_PER_KV:
            # more q heads per kv head than one CTA's MMA columns hold: groups of <= 8 rows,
            # each a separate launch over the same cache (K/V read once per group)
            qv = q.view(L, B, self.H, m, D)
            for r0 in range(0, m, MAX_Q_PER_KV):
                r1 = min(m, r0 + MAX_Q_PER_KV)
                og = self.decode(qv[:, :, :, r0:r1].reshape(L, B, self.H * (r1 - r0), D),
                                 splits=splits, scale=scale, layer=layer, pdl=False, seqs=(b0, b1),
                                 heads=(h0, h1))
                out.view(L, B, self.H, m, D)[:, b0:b1, :, r0:r1] = og.view(L, B, self.H, r1 - r0, D)[:, b0:b1]
            return out
        scale = 1.0 / math.sqrt(HEAD_DIM) if scale is None else float(scale)
        rng = None if (b0, b1) == (0, B) else (b0, b1)
        plan = self._use_wp(m, rng, splits, schedule) if b1 > b0 and (h0, h1) == (0, self.H) else None
        if plan is not None:
            prefix, ctas, slots, max_ctas = plan
            ws = self._wp_workspace(m, L, layer, max_ctas, rng)
            _lib.call("ckv_decode_attention_wp_seqs", _lib.ptr(q), q.stride(0), q.stride(1), self.arena("k", layer),
                      self.arena("v", layer), _lib.ptr(self.seq), L, B, b0, b1 - b0, self.H, m, scale,
                      _lib.ptr(prefix), ctas, slots, max_ctas, ws, _lib.ptr(out), out.stride(0), out.stride(1),
                      None, _lib.DECODE_PDL if pdl else 0, _lib.stream())
            return out
        splits = self.default_splits(m, L) if splits is None else int(splits)
        ws = self._workspace(m, splits, L, layer)
        _lib.call("ckv_decode_attention_range", _lib.ptr(q), q.stride(0), q.stride(1),
                  self.arena("k", layer), self.arena("v", layer), _lib.ptr(self.seq), L, B, b0, b1 - b0,
                  self.H, h0, h1 - h0, m, scale, splits, ws, _lib.ptr(out), out.stride(0), out.stride(1), None,
                  _lib.DECODE_PDL if pdl else 0, _lib.stream())
        return out

    def decode_step_host(self, q_host, out_host, splits=None, scale=None, d2h_every=None, order_current=True,
                         chains=1):
        """One decode step for all layers from HOST buffers: pinned fp16 q [L, B, H*m, 128] ->
        pinned fp16 output of the same shape.  The q upload runs on its own copy stream (it
        overlaps the previous step's layers); the layers run as CUDA-graph segments of
        `d2h_every` (default: all) PDL-chained per-layer launches (captured once per staging
        buffer, so the host enqueues one replay per segment instead of one launch per layer);
        each segment's outputs go back on a second copy stream while the next segment (or, for
        the last one, the next step) computes.  Device
        staging is double-buffered across steps, so consecutive steps never wait on each
        other's copies.  With ``order_current`` the current stream is ordered after the last
        download on return; without it the downloads stay on the copy stream (they overlap the
        next step's layers) and ``self.host_step_ready`` is the event that completes them."""
        L, B, Hq, D = q_host.shape
        if (L, B) != (self.L, self.B) or D != HEAD_DIM or Hq % self.H or q_host.dtype != torch.float16:
            raise ValueError("q shape does not match the cache")
        if out_host.shape != q_host.shape or out_host.dtype != torch.float16:
            raise ValueError("out_host must match q_host")
        seg = L if d2h_every is None else max(1, min(int(d2h_every), L))
        key = (tuple(q_host.shape), splits, scale, seg, chains)
        st = getattr(self, "_host_step", None)
        if st is None or st["key"] != key:
            dev = self.device
            shape = tuple(q_host.shape)
            st = dict(key=key, q=[torch.empty(shape, dtype=torch.float16, device=dev) for _ in range(2)],
                      o=[torch.empty(shape, dtype=torch.float16, device=dev) for _ in range(2)],
                      cin=torch.cuda.Stream(device=dev), cout=torch.cuda.Stream(device=dev),
                      q_free=[None, None], o_free=[None, None], i=0, graphs=[None, None])
            for b in range(2):
                st["graphs"][b] = self._segment_graphs(st["q"][b], st["o"][b], seg, splits, scale, chains)
            self._host_step = st
        ms = torch.cuda.current_stream()
        cin, cout = st["cin"], st["cout"]
        buf = st["i"] & 1
        st["i"] += 1
        qd, od = st["q"][buf], st["o"][buf]
        ev_q = torch.cuda.Event()
        with torch.cuda.stream(cin):
            if st["q_free"][buf] is not None:  # the step two back has read this staging buffer
                cin.wait_event(st["q_free"][buf])
            qd.copy_(q_host, non_blocking=True)
            ev_q.record(cin)
        if st["o_free"][buf] is not None:  # ... and its outputs have left this staging buffer
            ms.wait_event(st["o_free"][buf])
        ms.wait_event(ev_q)
        for i, g in enumerate(st["graphs"][buf]):
            g.replay()
            lo, hi = i * seg, min(L, (i + 1) * seg)
            ev = torch.cuda.Event()
            ev.record(ms)
            cout.wait_event(ev)
            with torch.cuda.stream(cout):
                out_host[lo:hi].copy_(od[lo:hi], non_blocking=True)
        q_free, o_free = torch.cuda.Event(), torch.cuda.Event()
        q_free.record(ms)
        o_free.record(cout)
        st["q_free"][buf], st["o_free"][buf] = q_free, o_free
        self.host_step_ready = o_free
        if order_current:
            ms.wait_stream(cout)
        return out_host

    def _chain_ranges(self, chains):
        chains = max(1, min(int(chains), self.B))
        return [(c * self.B // chains, (c + 1) * self.B // chains) for c in range(chains)]

    def _chain_units(self, chains):
        """Micro-batch chains as (b0, b1, h0, h1) ranges: sequence ranges while chains <= B, else
        every sequence split further into chains // B kv-head ranges (a batch-1 context runs as
        chains over its heads)."""
        chains = max(1, int(chains))
        if chains <= self.B:
            return [(b0, b1, 0, self.H) for (b0, b1) in self._chain_ranges(chains)]
        k = max(1, min(chains // self.B, self.H))
        return [(b, b + 1, j * self.H // k, (j + 1) * self.H // k) for b in range(self.B) for j in range(k)]

    def _launch_layers(self, q, out, lo, hi, splits, scale, chains, streams):
        """Per-layer launches of layers [lo, hi): one PDL chain per micro-batch (sequence range),
        each on its own stream forked from (and joined back into) the current stream."""
        units = self._chain_units(chains)
        if len(units) == 1:
            for l in range(lo, hi):
                self.decode(q[l:l + 1], splits=splits, out=out[l:l + 1], scale=scale, layer=l, pdl=l > lo)
            return
        cur = torch.cuda.current_stream()
        for st in streams:
            st.wait_stream(cur)
        for (b0, b1, h0, h1), st in zip(units, streams):
            with torch.cuda.stream(st):
                for l in range(lo, hi):
                    self.decode(q[l:l + 1], splits=splits, out=out[l:l + 1], scale=scale, layer=l,
                                pdl=l > lo and self.chain_pdl, seqs=(b0, b1), heads=(h0, h1))
        for st in streams:
            cur.wait_stream(st)

    def _segment_graphs(self, q, out, seg, splits, scale, chains=1):
        """CUDA graphs of layers [i seg, (i+1) seg): per-layer launches, PDL-chained inside a
        segment (one chain per micro-batch), over the fixed staging buffers q / out."""
        graphs = []
        side = torch.cuda.Stream(device=self.device)
        streams = [torch.cuda.Stream(device=self.device) for _ in self._chain_units(chains)]
        side.wait_stream(torch.cuda.current_stream())
        for lo in range(0, self.L, seg):
            hi = min(self.L, lo + seg)
            with torch.cuda.stream(side):  # warm-up: workspace, launch attributes
                self._launch_layers(q, out, lo, hi, splits, scale, chains, streams)
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):  # the warm-up's stream: same workspaces
                self._launch_layers(q, out, lo, hi, splits, scale, chains, streams)
            graphs.append(g)
        return graphs

    def decode_graph(self, q, out, splits=None, scale=None, chains=1):
        """Capture one decode step — every layer as its own PDL-chained launch, as in
        ``decode(q[l:l+1], layer=l, pdl=l > 0)`` — into a CUDA graph over the fixed device
        buffers q / out (fp16 [L, B, H*m, 128]).  ``graph.replay()`` runs a step; refill q in
        place between replays.  chains > 1 splits the batch into that many micro-batches, each
        its own chain of per-layer launches on its own stream inside the graph: a sequence's
        layer l+1 still waits for its layer l, but one micro-batch's layer boundary (the tail
        of layer l and the ramp of layer l+1) overlaps the other micro-batches' work.  The
        workspace is allocated by an eager warm-up step first."""
        if q.shape != out.shape or q.shape[0] != self.L:
            raise ValueError("q and out must be [L, B, H*m, 128] for all layers")
        return self._segment_graphs(q, out, self.L, splits, scale, chains)[0]

    def decode_partial(self, q, splits=None, scale=None, layer=0, pdl=False, out=None, schedule=None,
                       heads=None):
        """Unnormalised split-KV partials f32 [L'*B*H*m, 130] = (acc[128], m (log2), l) for q
        fp16 [L', B, H*m, 128] over layers [layer, layer + L') (per-layer launches: L' = 1,
        pdl as in decode); `out` may be a preallocated [L'*B*H*m, 130] view; heads=(h0, h1)
        computes those kv heads' rows only (split kernel; chains over heads)."""
        L, B, Hq, D = q.shape
        if B != self.B or layer < 0 or layer + L > self.L or D != HEAD_DIM or Hq % self.H:
            raise ValueError("q shape does not match the cache")
        m = Hq // self.H
        splits_arg = splits
        splits = self.default_splits(m, L) if splits is None else int(splits)
        part = out if out is not None else torch.empty((L * B * Hq, HEAD_DIM + 2), dtype=torch.float32,
                                                       device=q.device)
        if part.shape != (L * B * Hq, HEAD_DIM + 2) or not part.is_contiguous():
            raise ValueError("partials buffer must be contiguous [L*B*Hq, 130]")
        scale = 1.0 / math.sqrt(HEAD_DIM) if scale is None else float(scale)
        if heads is not None and tuple(heads) != (0, self.H):
            h0, h1 = int(heads[0]), int(heads[1])
            if not 0 <= h0 <= h1 <= self.H:
                raise ValueError("heads must be a range of the kv heads")
            ws = self._workspace(m, splits, L, layer)
            _lib.call("ckv_decode_attention_range", _lib.ptr(q), q.stride(0), q.stride(1), self.arena("k", layer),
                      self.arena("v", layer), _lib.ptr(self.seq), L, B, 0, B, self.H, h0, h1 - h0, m, scale, splits,
                      ws, None, 0, 0, _lib.ptr(part), _lib.DECODE_PDL if pdl else 0, _lib.stream())
            return part
        plan = self._use_wp(m, None, None if schedule == "wp" else splits_arg, schedule)
        if plan is not None:
            prefix, ctas, slots, max_ctas = plan
            ws = self._wp_workspace(m, L, layer, max_ctas)
            _lib.call("ckv_decode_attention_wp", _lib.ptr(q), q.stride(0), q.stride(1), self.arena("k", layer),
                      self.arena("v", layer), _lib.ptr(self.seq), L, B, self.H, m, scale, _lib.ptr(prefix), ctas,
                      slots, max_ctas, ws, None, 0, 0, _lib.ptr(part), _lib.DECODE_PDL if pdl else 0,
                      _lib.stream())
            return part
        ws = self._workspace(m, splits, L, layer)
        _lib.call("ckv_decode_attention", _lib.ptr(q), q.stride(0), q.stride(1),
                  self.arena("k", layer), self.arena("v", layer), _lib.ptr(self.seq), L, B, self.H,
                  m, scale, splits, ws, None, 0, 0, _lib.ptr(part), _lib.DECODE_PDL if pdl else 0,
                  _lib.stream())
        return part

    def append(self, k_new, v_new):
        """Append one decode token per (layer, sequence, kv-head): fp16 [L, B, H, 128]."""
        if k_new.shape != (self.L, self.B, self.H, HEAD_DIM) or k_new.shape != v_new.shape:
            raise ValueError(f"decode vectors must have shape {(self.L, self.B, self.H, HEAD_DIM)}")
        self._reserve_decode_token()
        self._append_device(k_new.to(torch.float16).contiguous(), v_new.to(torch.float16).contiguous())

    def _reserve_decode_token(self):
        """Host mirror of one append (kv_store.py:135-148: capacity is a host decision)."""
        if (self.seq_host[:, 5] + 1 > self.cap_fp).any():
            raise ValueError("decode capacity exhausted; rebuild with a larger decode_capacity")
        self.seq_host[:, 5] += 1
        self._any_empty = bool((self.total_tokens() == 0).any())

    def _append_device(self, k_new, v_new):
        """ckv_append_tokens on the current stream (device side only; graph-capturable)."""
        _lib.call("ckv_append_tokens", _lib.ptr(k_new), _lib.ptr(v_new), self.L, self.B, self.H,
                  _lib.ptr(self.seq), self.arena("k"), self.arena("v"), _lib.stream())

    # -- accounting --------------------------------------------------------------------
    def algorithmic_bytes(self, m):
        """K/V bytes one decode step must read + q and o."""
        s = self.seq_host.astype(np.int64)
        per_unit = s[:, 1] * BYTES_INT2 + s[:, 3] * BYTES_INT4 + s[:, 5] * BYTES_FP16
        return int(self.L * self.H * per_unit.sum() + 2 * self.L * self.B * self.H * m * HEAD_DIM * 2)

    def memory_bytes(self):
        return (self.tiles2.numel() + self.tiles4.numel() +
                sum(t.numel() * t.element_size() for d in (self.k, self.v) for t in d.values()))

    def memory_footprint(self):
        """Byte accounting of the whole cache (kv_store.memory_footprint, kv_store.py:256-307,
        summed over the (layer, sequence, kv-head) units), for the tile-native device format:
        INT2 / INT4 tiles carry packed codes plus fp16 (lo, hi) metadata (96 / 160 B per
        token-head, K+V); the FP16 region 512 B per token-head (FP16-tier chunks, tail and
        decode tokens); metadata = the per-sequence table and the per-unit span words.
        ``reference`` is the same cache under the reference's accounting (float64 scale and
        zero point per group, the serialized header and chunk permutation per unit)."""
        s = self.seq_host.astype(np.int64)
        len2, len4, lenf, ctx = s[:, 1], s[:, 3], s[:, 5], s[:, 7]
        units = self.L * self.H
        total = len2 + len4 + lenf
        n_chunks = ctx // CHUNK
        from .kv_store import MemoryReport, _HEADER
        ref = MemoryReport(
            int2_bytes=int(units * (2 * (32 + 64) * len2).sum()),   # u32 words + f64 scale/zp, K and V
            int4_bytes=int(units * (2 * (64 + 64) * len4).sum()),
            fp16_bytes=int(units * (BYTES_FP16 * lenf).sum()),
            metadata_bytes=int(units * (_HEADER.size + 4 * n_chunks).sum()),
            fp16_baseline_bytes=int(units * (BYTES_FP16 * total).sum()))
        return BatchedMemoryReport(
            int2_bytes=int(units * (BYTES_INT2 * len2).sum()),
            int4_bytes=int(units * (BYTES_INT4 * len4).sum()),
            fp16_bytes=int(units * (BYTES_FP16 * lenf).sum()),
            metadata_bytes=int(self.seq.numel() * 4 + 4 * sum(self.k[x].numel() + self.v[x].numel()
                                                               for x in ("span_flags", "span_max"))),
            fp16_baseline_bytes=int(units * (BYTES_FP16 * total).sum()),
            fp16_capacity_bytes=int(units * (BYTES_FP16 * self.cap_fp).sum()),
            reference=ref)

    def wide_scale_units(self):
        """Number of (layer, kv-head, sequence) units with a group scale above 4000 (diagnostic
        span flag of the quantize kernel; the decode has one path for every unit)."""
        return int(((self.k["span_flags"] | self.v["span_flags"]) != 0).sum().item())

    # -- export to the reference per-head format ------------------------------------------
    def token_order(self, seq):
        """kv_store.token_order (kv_store.py:227-233) of one sequence: the original position of
        every row in arena order (INT2 ‖ INT4 ‖ FP16 region)."""
        s = self.seq_host[seq].astype(np.int64)
        n_chunks = int(s[7]) // CHUNK
        perm = self._build_perm()[seq].cpu().numpy().astype(np.int64)[:n_chunks]
        chunks = (perm[:, None] * CHUNK + np.arange(CHUNK)[None, :]).reshape(-1)
        n_after = int(s[1] + s[3] + s[5]) - n_chunks * CHUNK  # the tail, then the decode tokens
        return np.concatenate([chunks, n_chunks * CHUNK + np.arange(n_after)]).astype(np.int64)

    def _build_perm(self):
        if getattr(self, "_perm", None) is None:
            raise ValueError("cache was not built here: no build permutation")
        return self._perm

    def reconstruct(self, layer=0, layers=None, t_out=None):
        """kv_store.reconstruct (kv_store.py:236-253) for the whole cache on the device: K and V
        f64 [L', B, T_out, H, 128] of layers [layer, layer + L') in ORIGINAL token order (every
        row dequantized as the reference's dequantize_codes does, FP16-region rows widened; the
        tail and the decode tokens after the chunks), one launch (ckv_reconstruct).  T_out
        defaults to the longest sequence's context + decode tokens; shorter sequences leave
        their later rows zero."""
        L = self.L - layer if layers is None else int(layers)
        if layer < 0 or L < 0 or layer + L > self.L:
            raise ValueError("layer range outside the cache")
        total = self.total_tokens()  # rows = original positions (context + decode tokens)
        T = (int(total.max()) if self.B else 0) if t_out is None else int(t_out)
        shape = (L, self.B, T, self.H, HEAD_DIM)
        ok = torch.zeros(shape, dtype=torch.float64, device=self.device)
        ov = torch.zeros_like(ok)
        perm = self._build_perm()
        _lib.call("ckv_reconstruct", self.arena("k", layer), self.arena("v", layer), _lib.ptr(self.seq),
                  _lib.ptr(perm), perm.shape[1], L, self.B, self.H, int(total.max()) if self.B else 0,
                  _lib.ptr(ok), _lib.ptr(ov), ok.stride(0), ok.stride(1), ok.stride(2), ok.stride(3), T,
                  _lib.stream())
        return ok, ov

    def export_unit(self, layer, seq, head, perm=None):
        """The reference-format ChunkedKVCache of one unit (kv_store.py:24-166): packed words and
        (lo, hi) metadata gathered back from the tile-native arenas to reference rows, f64
        scale/zero_point expanded from (lo, hi), all on the device."""
        s = self.seq_host[seq]
        off2, len2, off4, len4, offf, lenf, _, ctx = (int(x) for x in s)

        def block(t, which, bits):
            off, rows = (off2, len2) if bits == 2 else (off4, len4)
            buf = (self.tiles2 if bits == 2 else self.tiles4)[layer, head, off // TILE:]
            stride = BLOCK2 if bits == 2 else BLOCK4
            code_bytes = 512 if bits == 2 else 1024
            v = which == "v"
            packed = torch.empty((rows, 8 if bits == 2 else 16), dtype=torch.int32, device=self.device)
            mt = torch.empty((rows, 4), dtype=torch.int32, device=self.device)
            base = buf.data_ptr()
            _lib.call("ckv_arena_export", _lib._vp(base + (code_bytes if v else 0)),
                      _lib._vp(base + 2 * code_bytes + (256 if v else 0)), rows, bits, int(v), stride,
                      _lib.ptr(packed), _lib.ptr(mt), _lib.stream())
            packed = packed.reshape(-1)
            mt = mt.reshape(-1)
            sc = torch.empty(mt.numel(), dtype=torch.float64, device=self.device)
            zp = torch.empty(mt.numel(), dtype=torch.float64, device=self.device)
            _lib.call("ckv_expand_meta", _lib.ptr(mt), mt.numel(), bits, _lib.ptr(sc), _lib.ptr(zp),
                      _lib.stream())
            return QuantizedBlock._from_device(rows, HEAD_DIM, bits, GROUP, packed, sc, zp)

        n_chunks = ctx // CHUNK
        if perm is None:  # the permutation this cache was built with
            if getattr(self, "_perm", None) is None:
                raise ValueError("cache was not built here: pass the build perm to export_unit")
            perm = self._build_perm()[seq].cpu().numpy()
        perm = np.asarray(perm)
        if perm.shape[0] < n_chunks:
            raise ValueError("perm shorter than the sequence's chunk count")
        kf = self.k["fp"][layer, head, offf:offf + lenf].double().cpu().numpy()
        vf = self.v["fp"][layer, head, offf:offf + lenf].double().cpu().numpy()
        return ChunkedKVCache(CHUNK, HEAD_DIM, GROUP, ctx, np.asarray(perm, np.uint32)[:n_chunks],
                              block(self.k, "k", 2), block(self.v, "v", 2), block(self.k, "k", 4),
                              block(self.v, "v", 4), kf, vf)


@dataclass(frozen=True)
class BatchedMemoryReport:
    """Bytes of a BatchedKVCache at its device precision (see BatchedKVCache.memory_footprint);
    same fields and derived values as the reference's MemoryReport (kv_store.py:256-292)."""

    int2_bytes: int
    int4_bytes: int
    fp16_bytes: int
    metadata_bytes: int
    fp16_baseline_bytes: int
    fp16_capacity_bytes: int = 0   # the FP16 region as allocated (decode capacity included)
    reference: object = None       # kv_store.MemoryReport of the same cache, reference accounting

    @property
    def total_bytes(self) -> int:
        return self.int2_bytes + self.int4_bytes + self.fp16_bytes + self.metadata_bytes

    @property
    def compression_ratio(self) -> float:
        return self.total_bytes / self.fp16_baseline_bytes if self.fp16_baseline_bytes else 0.0

    def as_dict(self) -> dict:
        d = {"int2_bytes": self.int2_bytes, "int4_bytes": self.int4_bytes, "fp16_bytes": self.fp16_bytes,
             "metadata_bytes": self.metadata_bytes, "fp16_baseline_bytes": self.fp16_baseline_bytes,
             "total_bytes": self.total_bytes, "compression_ratio": self.compression_ratio,
             "fp16_capacity_bytes": self.fp16_capacity_bytes}
        if self.reference is not None:
            d["reference"] = self.reference.as_dict()
        return d


class DecodeLoop:
    """Serving-style decode loop on the device (the reference's generate loop, toy_model.py:
    89-108, with its per-head attention replaced by the batched cache): every step appends the
    step's new K/V (one token per (layer, sequence, kv head), ckv_append_tokens) and runs each
    layer as its own PDL-chained decode launch; the whole step (append + L launches) is one CUDA
    graph over fixed staging buffers.  ``step(q, k_new, v_new)`` copies the inputs into the
    staging buffers (any device), replays the graph and returns the output buffer
    (fp16 [L, B, H*m, 128], valid until the next step)."""

    def __init__(self, cache, m, splits=None, chains=1):
        self.cache = cache
        L, B, H, dev = cache.L, cache.B, cache.H, cache.device
        self.q = torch.zeros((L, B, H * m, HEAD_DIM), dtype=torch.float16, device=dev)
        self.out = torch.empty_like(self.q)
        self.k_new = torch.zeros((L, B, H, HEAD_DIM), dtype=torch.float16, device=dev)
        self.v_new = torch.zeros_like(self.k_new)
        streams = [torch.cuda.Stream(device=dev) for _ in cache._chain_units(chains)]
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up (workspaces, attributes) without appending
            cache._launch_layers(self.q, self.out, 0, L, splits, None, chains, streams)
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=side):  # the warm-up's stream: same workspaces
            cache._append_device(self.k_new, self.v_new)
            cache._launch_layers(self.q, self.out, 0, L, splits, None, chains, streams)
        self.steps = 0

    def step(self, q=None, k_new=None, v_new=None):
        self.cache._reserve_decode_token()
        for dst, src in ((self.q, q), (self.k_new, k_new), (self.v_new, v_new)):
            if src is not None:
                dst.copy_(src, non_blocking=True)
        self.graph.replay()
        self.steps += 1
        return self.out


def build_cache_batched(k, v, search, context_lens=None, decode_capacity=128, check=True):
    """Batched kv_store.build_cache: fp16 K/V [L, B, T, H, 128] + SearchResult -> BatchedKVCache."""
    return BatchedKVCache.from_search(k, v, search, context_lens, decode_capacity, check)


def mixed_decode_attention_batched(cache: BatchedKVCache, q, splits=None, out=None):
    """Batched attention.mixed_decode_attention: q fp16 [L, B, H*m, 128] -> fp16 output."""
    return cache.decode(q, splits=splits, out=out)


def lse_merge(partials, out=None):
    """Merge split-KV partials f32 [P, rows, 130] (from several shards/ranks) -> fp16 [rows, 128]."""
    P, rows, w = partials.shape
    if w != HEAD_DIM + 2:
        raise ValueError("partials must be [P, rows, 130]")
    partials = partials.contiguous()
    if out is None:
        out = torch.empty((rows, HEAD_DIM), dtype=torch.float16, device=partials.device)
    _lib.call("ckv_lse_merge", _lib.ptr(partials), P, rows, _lib.ptr(out), _lib.stream())
    return out
