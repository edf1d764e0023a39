"""Multi-GPU partitioning of the hot path.  One process per GPU.

* Batch sharding (cfg2/cfg4): independent units, no exchange -> ``batch_shard``.
* KV-head sharding (cfg3 alternative to split-KV): every rank owns whole kv heads (all
  layers, all tokens) -> ``head_shard`` / ``build_head_shard``; no exchange either (the
  q heads of a kv head stay on its rank, as in tensor-parallel attention).
* Sequence split-KV (cfg3, long contexts): every rank owns a chunk-aligned 1/P slice of
  each tier segment (INT2, INT4 and FP16 chunks separately, so bytes are balanced); the
  last rank also owns the context tail and the decode tokens.  Each rank computes
  unnormalised partials (acc[128], m, l) for all (layer, q-head) rows of its slice; one
  ``all_gather_into_tensor`` (NCCL over NVLink/NVSwitch) exchanges them, batched over all
  layers of the step, and ``ckv_lse_merge`` combines them:
      m* = max_p m_p,  o = sum_p acc_p 2^(m_p - m*) / sum_p l_p 2^(m_p - m*).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, kernels
from .batched import CHUNK, HEAD_DIM, BatchedKVCache, lse_merge


def batch_shard(batch, world, rank):
    """Contiguous slice of sequences owned by `rank` (cfg4 weak scaling)."""
    lo = rank * batch // world
    hi = (rank + 1) * batch // world
    return lo, hi


def head_shard(kv_heads, world, rank):
    """Contiguous slice of kv heads owned by `rank` (head-parallel decode: no collective)."""
    return _split(kv_heads, world, rank)


def build_head_shard(k, v, search, world, rank, decode_capacity=128, check=True):
    """This rank's BatchedKVCache over its kv heads [lo, hi): k, v fp16 [L, B, T, H, 128] (the
    full model's K/V or any view holding at least those heads).  Decode it with the matching q
    heads, q[:, :, lo*m:hi*m]."""
    L, B, T, H, D = k.shape
    lo, hi = head_shard(H, world, rank)
    return BatchedKVCache.from_search(k[:, :, :, lo:hi], v[:, :, :, lo:hi], search,
                                      decode_capacity=decode_capacity, check=check)


def layer_shard(layers, world, rank):
    """Contiguous slice of layers built by `rank` (cfg5 prefill sharded by layer, SURVEY §8e:
    every rank runs the search for the sequence — N bytes of tier map — and quantizes its own
    layers; no exchange)."""
    return _split(layers, world, rank)


def _split(n, world, rank):
    return rank * n // world, (rank + 1) * n // world


def sequence_shard_plan(seg_counts, world, rank):
    """Per-sequence chunk ranges of this rank inside each tier segment (perm order).

    seg_counts int [B, 3] (n2, n4, nfp).  Returns int64 [B, 6] = (a2, b2, a4, b4, af, bf)
    in perm positions, plus owns_tail (bool): the last rank owns the tail/decode tokens.
    """
    seg_counts = np.asarray(seg_counts, np.int64).reshape(-1, 3)
    out = np.zeros((seg_counts.shape[0], 6), np.int64)
    for b, (n2, n4, nf) in enumerate(seg_counts):
        a2, b2 = _split(n2, world, rank)
        a4, b4 = _split(n4, world, rank)
        af, bf = _split(nf, world, rank)
        out[b] = (a2, b2, n2 + a4, n2 + b4, n2 + n4 + af, n2 + n4 + bf)
    return out, rank == world - 1


def sequence_shard_cache(search, layers, kv_heads, context, world, rank, decode_capacity=128,
                         device=None):
    """This rank's empty BatchedKVCache for a sequence-split (split-KV) layout and the perm of
    its chunks (source chunk per destination slot), to be filled with ``cache.build(k, v,
    perm_r[, layer=...])`` from the full-context K/V (all layers at once or layer by layer)."""
    counts = search.seg_counts.cpu().numpy().astype(np.int64)
    B = counts.shape[0]
    plan, owns_tail = sequence_shard_plan(counts, world, rank)
    perm = search.perm
    n_max = perm.shape[1]
    n2r = plan[:, 1] - plan[:, 0]
    n4r = plan[:, 3] - plan[:, 2]
    nfr = plan[:, 5] - plan[:, 4]
    width = int((n2r + n4r + nfr).max()) if B else 0
    idx = np.zeros((B, max(width, 1)), np.int64)
    for b in range(B):
        sel = np.concatenate([np.arange(plan[b, 0], plan[b, 1]), np.arange(plan[b, 2], plan[b, 3]),
                              np.arange(plan[b, 4], plan[b, 5])])
        idx[b, :sel.size] = sel
    idx_d = torch.from_numpy(idx).to(perm.device)
    perm_r = torch.gather(perm, 1, idx_d.clamp(max=n_max - 1)) if n_max else perm
    n_glob = counts.sum(axis=1)
    tail = np.asarray(context, np.int64).reshape(-1) - CHUNK * n_glob
    ctx_r = CHUNK * (n2r + n4r + nfr) + (tail if owns_tail else 0)
    cache = BatchedKVCache(layers, B, kv_heads, n2r, n4r, nfr, ctx_r,
                           decode_capacity if owns_tail else 0, tail_src=CHUNK * n_glob,
                           device=device or perm.device)
    return cache, perm_r


def build_sequence_shard(k, v, search, world, rank, decode_capacity=128, check=True):
    """This rank's BatchedKVCache for a sequence-split (split-KV) layout.

    k, v fp16 [L, B, T, H, 128] (the full context, e.g. prefilled redundantly or loaded
    per rank); search = SearchResult of the full context (tiers are global).
    """
    L, B, T, H, D = k.shape
    cache, perm_r = sequence_shard_cache(search, L, H, np.full(B, T), world, rank, decode_capacity,
                                         device=k.device)
    cache.build(k, v, perm_r, check=check)
    return cache


def exchange_partials(part, group=None):
    """all_gather of f32 partials [rows, 130] -> [P, rows, 130] on part's device: NCCL for CUDA
    tensors (NVLink / NVSwitch), gloo for host tensors; CUDA partials over a gloo group are
    staged through pinned host memory (e.g. several ranks sharing one GPU in a test)."""
    world = dist.get_world_size(group)
    part = part.contiguous()
    dev = part.device
    if dev.type == "cuda" and dist.get_backend(group) == "gloo":
        part = part.to("cpu")
    out = torch.empty((world * part.shape[0],) + tuple(part.shape[1:]), dtype=part.dtype,
                      device=part.device)
    if dist.get_backend(group) == "gloo":
        dist.all_gather(list(out.chunk(world)), part, group=group)
    else:
        dist.all_gather_into_tensor(out, part, group=group)
    return out.view((world,) + tuple(part.shape)).to(dev)


class P2PExchange:
    """Split-KV partial exchange over peer memory instead of a collective ("use
    symmetric memory if NCCL latency dominates").  Every rank's partials [rows, 130] live in a
    symmetric-memory buffer (torch.distributed._symmetric_memory: one allocation per rank, mapped
    into every peer over NVLink); a step is: decode_partial writes the local buffer, a device-side
    barrier (the allocation's signal pads) orders all ranks' writes, and ckv_lse_merge_ptrs reads
    every peer's rows straight from its buffer (ordinary loads through the peer mappings) and
    writes the merged output — no gathered copy, no NCCL kernel.  Two buffers alternate, so one
    barrier per step also keeps a rank from overwriting partials a slower peer is still reading
    (rank r writes buffer i again only after passing the next step's barrier, which every rank
    reaches after its merge of buffer i)."""

    def __init__(self, rows, group=None, device=None, slots=2):
        self.group = group or dist.group.WORLD
        self.P = dist.get_world_size(self.group)
        self.rows = int(rows)
        self.device = device
        # every rank allocates first and the ranks agree before the (collective) rendezvous, so a
        # rank that cannot use symmetric memory makes all of them raise instead of leaving the
        # others waiting in the rendezvous
        bufs, err = [], None
        try:
            import torch.distributed._symmetric_memory as symm_mem

            dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
            peers_ok = all(torch.cuda.can_device_access_peer(dev.index, j)
                           for j in range(torch.cuda.device_count()) if j != dev.index)
            if not peers_ok:
                raise RuntimeError("no peer access between the visible GPUs")
            bufs = [symm_mem.empty((self.rows, HEAD_DIM + 2), dtype=torch.float32, device=device)
                    for _ in range(slots)]
        except Exception as e:  # noqa: BLE001
            err = e
        if self.P > 1:
            flag = torch.tensor([0 if err else 1], dtype=torch.int32,
                                device=device if dist.get_backend(self.group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
            if int(flag.item()) == 0 and err is None:
                err = RuntimeError("symmetric memory unavailable on another rank")
        if err is not None:
            raise err
        self.bufs, self.hdls, self.ptrs = [], [], []
        for t in bufs:
            h = symm_mem.rendezvous(t, self.group)
            base = list(h.buffer_ptrs)
            off = t.data_ptr() - base[h.rank]
            self.bufs.append(t)
            self.hdls.append(h)
            self.ptrs.append(torch.tensor([b + off for b in base], dtype=torch.int64, device=device))
        self.i = 0

    def buffer(self, i=None):
        """The local partial buffer of step slot i (default: the current step's)."""
        return self.bufs[self.i if i is None else i]

    def merge(self, out=None, i=None):
        """Barrier + peer-read merge of slot i's partials -> fp16 [rows, 128]; advances the slot
        when i is None."""
        j = self.i if i is None else i
        self.hdls[j].barrier(channel=0)
        if out is None:
            out = torch.empty((self.rows, HEAD_DIM), dtype=torch.float16, device=self.bufs[j].device)
        _lib.call("ckv_lse_merge_ptrs", _lib.ptr(self.ptrs[j]), self.P, self.rows, _lib.ptr(out), _lib.stream())
        if i is None:
            self.i = (self.i + 1) % len(self.bufs)
        return out


def split_kv_decode(cache: BatchedKVCache, q, group=None, splits=None):
    """Sequence-split decode step across ranks: local partials -> all_gather -> LSE merge.

    q fp16 [L, B, H*m, 128] (replicated on every rank) -> fp16 [L, B, H*m, 128]."""
    part = cache.decode_partial(q, splits=splits)
    gathered = exchange_partials(part, group)
    out = lse_merge(gathered)
    return out.view(q.shape)


__all__ = ["batch_shard", "head_shard", "build_head_shard", "layer_shard", "sequence_shard_plan",
           "sequence_shard_cache", "build_sequence_shard", "exchange_partials", "P2PExchange", "split_kv_decode"]
