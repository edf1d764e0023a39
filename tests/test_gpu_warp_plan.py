"""The warp-plan decode schedule (ckv_decode_attention_wp: one 16-warp CTA per SM, units split
at warp granularity, multi-CTA units merged in the launch) against the reference
algorithm (oracle) and against the split schedule, on unit counts from a few (many CTAs per
unit) to many (several units per CTA), with m = 1 / 4 / 8, decode tokens, partials, per-layer
PDL launches and CUDA-graph replay."""

import numpy as np
import pytest
import torch

from oracle import ckv_oracle as O
from paper_2503_23294_b200 import batched, retrieval
from tests.conftest import SCHED_TOL  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _search(tiers):
    return retrieval.assign_tiers_batched(tiers.astype(np.float64), np.tile([[0.5, 1.5]], (tiers.shape[0], 1)))


def _case(seed, L, B, H, m, N, tail, p=(0.8, 0.15, 0.05)):
    rng = np.random.default_rng(seed)
    T = N * 32 + tail
    k = rng.normal(size=(L, B, T, H, 128)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, 128)).astype(np.float16)
    q = rng.normal(size=(L, B, H * m, 128)).astype(np.float16)
    tiers = rng.choice([0, 1, 2], size=(B, N), p=p).astype(np.uint8)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search(tiers),
                                        decode_capacity=16)
    cache.schedule = "wp"  # force the warp plan (these caches are below the "auto" size threshold)
    return cache, k, v, q, tiers


def _check(out, k, v, q, tiers, m, units):
    for (l, b, h) in units:
        oc = O.build_cache(k[l, b, :, h].astype(np.float64), v[l, b, :, h].astype(np.float64), tiers[b], 32, 32)
        ref = O.mixed_decode_attention(q[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
        got = out[l, b, h * m:(h + 1) * m]
        err = np.max(np.abs(got - ref))
        assert err <= TOL and err / np.max(np.abs(ref)) <= TOL, (l, b, h, err)


@pytest.mark.parametrize("B,H,m,N", [(1, 2, 4, 300), (2, 8, 4, 60), (8, 8, 1, 9), (3, 5, 8, 40), (64, 8, 4, 6)])
def test_warp_plan_matches_oracle_and_split(B, H, m, N):
    L = 2
    cache, k, v, q, tiers = _case(100 + B + H + m, L, B, H, m, N, 7)
    plan = cache.warp_plan()
    assert plan is not None
    table, ctas, slots, max_ctas = plan
    from paper_2503_23294_b200 import _lib
    cw = _lib.load().ckv_decode_wp_cta_warps()
    rec = table.cpu().numpy()[:8 * cw * ctas].reshape(cw * ctas, 8)   # per-warp records
    counts = np.bincount(rec[:, 0], minlength=B * H)
    assert counts.sum() == cw * ctas and (counts >= 2).all() and (np.diff(rec[:, 0]) >= 0).all()
    assert (rec[:, 7] == counts[rec[:, 0]]).all()                      # nw = the unit's warps
    n2 = np.zeros(B * H, np.int64)
    np.add.at(n2, rec[:, 0], np.where((rec[:, 1] & 0xffff) == 0, rec[:, 2], 0))  # INT2 tiles, once per part
    assert (n2 == np.repeat(cache.seq_host[:, 1] // 16, H)).all()      # the parts cover every tile
    qd = torch.from_numpy(q).cuda()
    out = cache.decode(qd).float().cpu().numpy()            # warp plan (whole batch, no splits)
    ref_split = cache.decode(qd, splits=3).float().cpu().numpy()
    assert np.max(np.abs(out - ref_split)) < SCHED_TOL
    rng = np.random.default_rng(7)
    units = {(l, int(rng.integers(B)), int(rng.integers(H))) for l in range(L) for _ in range(3)}
    _check(out, k, v, q, tiers, m, units)
    # partials + LSE merge give the same rows
    part = cache.decode_partial(qd)
    merged = batched.lse_merge(part[None]).view(q.shape).float().cpu().numpy()
    assert np.max(np.abs(merged - out)) < SCHED_TOL


def test_warp_plan_per_layer_graph_and_appends():
    L, B, H, m = 3, 2, 4, 4
    cache, k, v, q, tiers = _case(200, L, B, H, m, 50, 3)
    qd = torch.from_numpy(q).cuda()
    out = torch.empty_like(qd)
    g = cache.decode_graph(qd, out)      # per-layer PDL-chained launches of the warp-plan kernel
    rng = np.random.default_rng(8)
    for _ in range(3):
        kn = torch.from_numpy(rng.normal(size=(L, B, H, 128)).astype(np.float16)).cuda()
        vn = torch.from_numpy(rng.normal(size=(L, B, H, 128)).astype(np.float16)).cuda()
        cache.append(kn, vn)
        g.replay()
        want = torch.empty_like(qd)
        for l in range(L):
            cache.decode(qd[l:l + 1], out=want[l:l + 1], layer=l, pdl=l > 0)
        torch.cuda.synchronize()
        assert torch.equal(out, want)   # deterministic: graph replay == eager, bit for bit
        assert torch.equal(cache.decode(qd), want)


@pytest.mark.parametrize("chains", [2, 3])
def test_warp_plan_micro_batch_chains(chains):
    """Sequence-range launches of the warp plan (ckv_decode_attention_wp_seqs): each range has
    its own plan and workspace; a decode step as `chains` micro-batch chains of per-layer PDL
    launches on their own streams (one CUDA graph) equals the whole-batch per-layer step bit for
    bit per sequence range's own plan, meets the oracle, and leaves other rows untouched."""
    L, B, H, m = 2, 5, 4, 4
    cache, k, v, q, tiers = _case(400 + chains, L, B, H, m, 40, 9)
    qd = torch.from_numpy(q).cuda()
    ranges = cache._chain_ranges(chains)
    for r in ranges:
        assert cache.warp_plan(r) is not None and cache._use_wp(m, r, None, None) is not None
    # one range alone: rows outside it untouched
    sentinel = torch.full_like(qd, 7.0)
    b0, b1 = ranges[1]
    cache.decode(qd, out=sentinel, seqs=(b0, b1))
    sn = sentinel.float().cpu().numpy()
    assert (sn[:, :b0] == 7.0).all() and (sn[:, b1:] == 7.0).all()
    _check(sn, k, v, q, tiers, m, [(l, b, h) for l in range(L) for b in range(b0, b1) for h in range(H)])
    # the chained per-layer graph
    out = torch.empty_like(qd)
    g = cache.decode_graph(qd, out, chains=chains)
    g.replay()
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for (r0, r1) in ranges:
        want = torch.empty_like(qd)
        for l in range(L):
            cache.decode(qd[l:l + 1], out=want[l:l + 1], layer=l, pdl=l > 0, seqs=(r0, r1))
        torch.cuda.synchronize()
        assert torch.equal(out[:, r0:r1], want[:, r0:r1])
    _check(got, k, v, q, tiers, m, [(l, b, h) for l in range(L) for b in range(B) for h in range(H)])
    whole = cache.decode(qd).float().cpu().numpy()
    assert np.max(np.abs(whole - got)) < SCHED_TOL


def test_warp_plan_outlier_precise_and_exact_units():
    L, B, H, m = 1, 2, 3, 8
    rng = np.random.default_rng(300)
    N = 40
    T = N * 32 + 5
    k = rng.normal(size=(L, B, T, H, 128)).astype(np.float16)
    k[..., [3, 40, 77, 100]] *= 8          # wide K groups (round 1: the precise path)
    k[0, 1, 10, 2, 5] = 20000.0            # one unit with a huge scale (round 1: the exact mode)
    v = rng.normal(size=(L, B, T, H, 128)).astype(np.float16)
    q = (rng.normal(size=(L, B, H * m, 128)) * 3).astype(np.float16)
    tiers = rng.choice([0, 1, 2], size=(B, N), p=(0.7, 0.25, 0.05)).astype(np.uint8)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search(tiers))
    cache.schedule = "wp"
    out = cache.decode(torch.from_numpy(q).cuda()).float().cpu().numpy()
    _check(out, k, v, q, tiers, m, [(0, b, h) for b in range(B) for h in range(H)])


@pytest.mark.parametrize("schedule", ["wp", "split"])
def test_concurrent_streams_use_private_workspaces(schedule):
    """Decodes of one cache on two concurrent streams: each stream gets its own workspace
    (self-resetting arrival counters + partials), so interleaved launches on both streams give
    the serial result (include/ckv.h: re-entrant per stream)."""
    L, B, H, m = 2, 2, 8, 4
    cache, k, v, q, tiers = _case(11, L, B, H, m, 60, 5)
    cache.schedule = schedule
    splits = 3 if schedule == "split" else None
    qd = torch.from_numpy(q).cuda()
    ref = cache.decode(qd, splits=splits).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = {s: [torch.empty_like(qd) for _ in range(20)] for s in (s1, s2)}
    for st in (s1, s2):
        st.wait_stream(torch.cuda.current_stream())
    for i in range(20):  # interleaved: both streams' launches are in flight together
        for st in (s1, s2):
            with torch.cuda.stream(st):
                for l in range(L):
                    cache.decode(qd[l:l + 1], splits=splits, out=outs[st][i][l:l + 1], layer=l, pdl=l > 0)
    torch.cuda.synchronize()
    ws = cache._ws_ptr
    ptrs = {v for key, v in ws.items() if key[-1] in (s1.cuda_stream, s2.cuda_stream)}
    assert len(ptrs) == 2 * L  # one per-layer slice per stream
    for st in (s1, s2):
        for o in outs[st]:
            assert torch.equal(o, ref) or (o.float() - ref.float()).abs().max().item() < SCHED_TOL
