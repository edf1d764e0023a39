"""The serving decode loop (append + per-layer decode graph per step) and the tile-native
memory accounting, against the reference algorithm (oracle) and the reference's own
memory_footprint of the exported units."""

import numpy as np
import pytest
import torch

from oracle import ckv_oracle as O
from paper_2503_23294_b200 import batched, kv_store, retrieval

pytestmark = pytest.mark.gpu

TOL_ABS = 1e-2
TOL_REL = 1e-2


def _search(tiers):
    return retrieval.assign_tiers_batched(tiers.astype(np.float64), np.tile([[0.5, 1.5]], (tiers.shape[0], 1)))


@pytest.mark.parametrize("chains", [1, 2])
def test_decode_loop_matches_oracle_each_step(chains):
    """DecodeLoop: N steps of (append one token per unit, per-layer decode graph) track the
    reference ChunkedKVCache.append + mixed_decode_attention unit by unit (toy_model.py:89-108,
    kv_store.py:135-148, attention.py:63-90)."""
    rng = np.random.default_rng(90 + chains)
    L, B, H, m, D, N, steps = 2, 3, 2, 4, 128, 11, 6
    T = N * 32 + 7
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    tiers = rng.choice([0, 0, 1, 2], size=(B, N)).astype(np.uint8)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search(tiers),
                                        decode_capacity=steps)
    loop = batched.DecodeLoop(cache, m, splits=3, chains=chains)
    refs = {(l, b, h): O.build_cache(k[l, b, :, h].astype(np.float64), v[l, b, :, h].astype(np.float64),
                                     tiers[b], 32, 32)
            for l in range(L) for b in range(B) for h in range(H)}
    for _ in range(steps):
        q = rng.normal(size=(L, B, H * m, D)).astype(np.float16)
        kn = rng.normal(size=(L, B, H, D)).astype(np.float16)
        vn = rng.normal(size=(L, B, H, D)).astype(np.float16)
        out = loop.step(torch.from_numpy(q).cuda(), torch.from_numpy(kn).cuda(),
                        torch.from_numpy(vn).cuda()).float().cpu().numpy()
        for (l, b, h), oc in refs.items():
            oc.append(kn[l, b, h].astype(np.float64), vn[l, b, h].astype(np.float64))
            ref = O.mixed_decode_attention(q[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
            err = np.max(np.abs(out[l, b, h * m:(h + 1) * m] - ref))
            assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL, (l, b, h, err)
    for _ in range(int((cache.cap_fp - cache.seq_host[:, 5]).min())):  # the rounded-up capacity
        loop.step()
    with pytest.raises(ValueError):  # capacity is a host decision, as in the reference
        loop.step()


def test_memory_footprint_matches_reference_accounting():
    """BatchedKVCache.memory_footprint().reference equals the sum of the reference's
    memory_footprint over the exported units; the tile-native figures are the device format's
    96 / 160 / 512 B per token-head."""
    rng = np.random.default_rng(95)
    L, B, H, D, N = 2, 2, 3, 128, 9
    T = N * 32 + 5
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    tiers = rng.choice([0, 1, 2], size=(B, N)).astype(np.uint8)
    s = _search(tiers)
    cache = batched.build_cache_batched(k, v, s, decode_capacity=4)
    cache.append(torch.zeros((L, B, H, D), dtype=torch.float16, device="cuda"),
                 torch.zeros((L, B, H, D), dtype=torch.float16, device="cuda"))
    rep = cache.memory_footprint()
    perm = s.perm.cpu().numpy()
    tot = dict(int2_bytes=0, int4_bytes=0, fp16_bytes=0, metadata_bytes=0, fp16_baseline_bytes=0)
    for l in range(L):
        for b in range(B):
            for h in range(H):
                r = kv_store.memory_footprint(cache.export_unit(l, b, h, perm=perm[b])).as_dict()
                for key in tot:
                    tot[key] += r[key]
    ref = rep.reference.as_dict()
    for key, val in tot.items():
        assert ref[key] == val, key
    cnt = s.seg_counts.cpu().numpy()
    units = L * H
    assert rep.int2_bytes == units * 96 * 32 * int(cnt[:, 0].sum())
    assert rep.int4_bytes == units * 160 * 32 * int(cnt[:, 1].sum())
    assert rep.fp16_bytes == units * 512 * int((32 * cnt[:, 2] + 5 + 1).sum())
    assert rep.fp16_baseline_bytes == units * 512 * B * (T + 1)
    assert 0 < rep.compression_ratio < rep.reference.compression_ratio


def test_bench_default_step_one_chain_per_sequence():
    """The bench's default decode step: one micro-batch chain per sequence (per-layer PDL launches
    on their own streams, one CUDA graph), auto schedule (chained ranges run the split kernel)
    with chain_splits.  Every unit meets the oracle; each chain equals its eager per-range
    launches bit for bit; decode_step_host (pinned host buffers) and DecodeLoop with the same
    chains give the same rows."""
    rng = np.random.default_rng(97)
    L, B, H, m, D, N = 2, 4, 2, 4, 128, 30
    T = N * 32 + 5
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    q = rng.normal(size=(L, B, H * m, D)).astype(np.float16)
    tiers = rng.choice([0, 0, 0, 1, 2], size=(B, N)).astype(np.uint8)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search(tiers),
                                        decode_capacity=4)
    assert cache.schedule == "auto"
    splits = cache.chain_splits(m)
    assert splits >= 1
    for r in cache._chain_ranges(B):
        assert cache._use_wp(m, r, None, None) is None  # chained ranges: the split kernel
    qd = torch.from_numpy(q).cuda()
    out = torch.empty_like(qd)
    g = cache.decode_graph(qd, out, splits=splits, chains=B)
    g.replay()
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for l in range(L):
        for b in range(B):
            for h in range(H):
                oc = O.build_cache(k[l, b, :, h].astype(np.float64), v[l, b, :, h].astype(np.float64), tiers[b], 32, 32)
                ref = O.mixed_decode_attention(q[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
                err = np.max(np.abs(got[l, b, h * m:(h + 1) * m] - ref))
                assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL, (l, b, h, err)
    want = torch.empty_like(qd)
    for b in range(B):
        for l in range(L):
            cache.decode(qd[l:l + 1], splits=splits, out=want[l:l + 1], layer=l, pdl=l > 0, seqs=(b, b + 1))
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    qh = qd.cpu().pin_memory()
    oh = torch.empty(qh.shape, dtype=torch.float16, pin_memory=True)
    cache.decode_step_host(qh, oh, splits=splits, chains=B)
    torch.cuda.synchronize()
    assert torch.equal(oh, want.cpu())
    loop = batched.DecodeLoop(cache, m, splits=splits, chains=B)
    kn = torch.zeros((L, B, H, D), dtype=torch.float16, device="cuda")
    step = loop.step(qd, kn, kn).float().cpu().numpy()  # one appended zero key/value per unit
    for (l, b, h) in ((0, 0, 0), (L - 1, B - 1, H - 1)):
        oc = O.build_cache(k[l, b, :, h].astype(np.float64), v[l, b, :, h].astype(np.float64), tiers[b], 32, 32)
        oc.append(np.zeros(D), np.zeros(D))
        ref = O.mixed_decode_attention(q[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
        err = np.max(np.abs(step[l, b, h * m:(h + 1) * m] - ref))
        assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL, (l, b, h, err)


def test_head_range_chains_batch_one():
    """A batch-1 cache decoded as micro-batch chains over its kv heads (ckv_decode_attention_range:
    each chain's launches cover a kv-head range; decode_partial with heads=) equals the
    oracle, and each range's launch leaves the other heads' rows untouched."""
    rng = np.random.default_rng(99)
    L, B, H, m, D, N = 2, 1, 5, 2, 128, 40
    T = N * 32 + 3
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    q = rng.normal(size=(L, B, H * m, D)).astype(np.float16)
    tiers = rng.choice([0, 0, 0, 1, 2], size=(B, N)).astype(np.uint8)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search(tiers))
    units = cache._chain_units(4)
    assert [u[2:] for u in units] == [(0, 1), (1, 2), (2, 3), (3, 5)]
    qd = torch.from_numpy(q).cuda()
    sentinel = torch.full_like(qd, 3.0)
    cache.decode(qd, out=sentinel, splits=3, heads=(1, 3))
    sn = sentinel.float().cpu().numpy()
    assert (sn[:, :, :m] == 3.0).all() and (sn[:, :, 3 * m:] == 3.0).all()
    out = torch.empty_like(qd)
    g = cache.decode_graph(qd, out, splits=cache.chain_splits(m), chains=4)
    g.replay()
    part = torch.full((L * B * H * m, D + 2), float("nan"), dtype=torch.float32, device="cuda")
    for (_, _, h0, h1) in units:
        cache.decode_partial(qd, splits=2, out=part, heads=(h0, h1))
    merged = batched.lse_merge(part[None]).view(qd.shape).float().cpu().numpy()
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for l in range(L):
        for h in range(H):
            oc = O.build_cache(k[l, 0, :, h].astype(np.float64), v[l, 0, :, h].astype(np.float64), tiers[0], 32, 32)
            ref = O.mixed_decode_attention(q[l, 0, h * m:(h + 1) * m].astype(np.float64), oc)
            for arr in (got, merged, sn if 1 <= h < 3 else None):
                if arr is None:
                    continue
                err = np.max(np.abs(arr[l, 0, h * m:(h + 1) * m] - ref))
                assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL, (l, h, err)


@pytest.mark.parametrize("m", [3, 12])
def test_chained_step_mixed_sequences(m):
    """Chained per-layer graph over sequences of different tier mixes — one all-FP16, one
    all-INT2, one mixed, each with a 17-token context tail — with m = 3 (odd GQA ratio) and
    m = 12 (groups of <= 8 q rows per launch): every unit meets the oracle."""
    rng = np.random.default_rng(200 + m)
    L, B, H, D = 2, 3, 2, 128
    N = 12
    T = N * 32 + 17
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    q = rng.normal(size=(L, B, H * m, D)).astype(np.float16)
    tiers = np.stack([np.full(N, 2), np.zeros(N, np.int64), rng.choice([0, 1, 2], size=N)]).astype(np.uint8)
    s = _search(tiers)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), s)
    qd = torch.from_numpy(q).cuda()
    out = torch.empty_like(qd)
    g = cache.decode_graph(qd, out, splits=cache.chain_splits(min(m, 8)), chains=B)
    g.replay()
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for l in range(L):
        for b in range(B):
            for h in range(H):
                oc = O.build_cache(k[l, b, :, h].astype(np.float64), v[l, b, :, h].astype(np.float64), tiers[b], 32, 32)
                ref = O.mixed_decode_attention(q[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
                err = np.max(np.abs(got[l, b, h * m:(h + 1) * m] - ref))
                assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL, (l, b, h, err)
