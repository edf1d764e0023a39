"""GPU: the batched fp16 hot path — fused reorder/quantize/pack (bit-exact codes, metadata,
permutation) and mixed-precision decode attention (1e-2 abs / 1e-2 rel of the reference's
f64 result on the same fp16 inputs), edge cases, split-KV shards, and full-size properties."""

import hashlib
import zlib

import numpy as np
import pytest
import torch

from oracle import ckv_oracle as O
from tests.conftest import SCHED_TOL, load_golden

pytestmark = pytest.mark.gpu

from paper_2503_23294_b200 import batched, distributed, retrieval  # noqa: E402
from paper_2503_23294_b200.kv_store import serialize_cache  # noqa: E402

TOL_ABS = 1e-2
TOL_REL = 1e-2


def _search_from_tiers(tiers):
    tiers = np.asarray(tiers, np.float64)
    return retrieval.assign_tiers_batched(tiers, np.tile([[0.5, 1.5]], (tiers.shape[0], 1)))


def _check_unit(cache, l, b, h, k, v, tiers_b, q_rows, out_rows, ctx=None):
    T = k.shape[2] if ctx is None else ctx
    oc = O.build_cache(k[l, b, :T, h].astype(np.float64), v[l, b, :T, h].astype(np.float64), tiers_b, 32, 32)
    ex = cache.export_unit(l, b, h)
    for name in ("k_q2", "v_q2", "k_q4", "v_q4"):
        a, w = getattr(ex, name), getattr(oc, name)
        assert np.array_equal(a.packed, w.packed), name
        assert np.array_equal(a.scales.view(np.uint64), w.scales.view(np.uint64)), name
        assert np.array_equal(a.zero_points.view(np.uint64), w.zero_points.view(np.uint64)), name
    assert np.array_equal(ex.k_fp[:oc.len_fp], oc.k_fp)
    ref = O.mixed_decode_attention(q_rows.astype(np.float64), oc)
    err = np.max(np.abs(out_rows.astype(np.float64) - ref))
    scale = max(np.max(np.abs(ref)), 1e-30)
    assert err <= TOL_ABS * max(1.0, scale) and err / scale <= TOL_REL, (err, scale)
    return err / scale


def test_batched_golden_case():
    g = load_golden("batched.npz")
    L, B, H, m, T = (int(x) for x in g["dims"])
    k = torch.from_numpy(g["k"]).cuda()
    v = torch.from_numpy(g["v"]).cuda()
    q = torch.from_numpy(g["q"]).cuda()
    cache = batched.build_cache_batched(k, v, _search_from_tiers(g["tiers"]))
    out = cache.decode(q).float().cpu().numpy()
    for l in range(L):
        for b in range(B):
            for h in range(H):
                key = f"{l}_{b}_{h}"
                ex = cache.export_unit(l, b, h, perm=g[f"perm_{key}"])
                # the reference's wire format straight from the GPU arenas
                wire = serialize_cache(ex)
                assert len(wire) == int(g[f"wire_len_{key}"])
                assert hashlib.sha256(wire).digest() == g[f"wire_sha256_{key}"].tobytes(), key
                for name in ("k_q2", "v_q2", "k_q4", "v_q4"):
                    blk = getattr(ex, name)
                    assert np.array_equal(blk.packed, g[f"{name}_packed_{key}"])
                    assert np.array_equal(blk.scales.view(np.uint64), g[f"{name}_scales_{key}"].view(np.uint64))
                    assert np.array_equal(blk.zero_points.view(np.uint64), g[f"{name}_zps_{key}"].view(np.uint64))
                ref = g[f"out_{key}"]
                got = out[l, b, h * m:(h + 1) * m]
                err = np.max(np.abs(got - ref))
                assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL


@pytest.mark.parametrize("m", [1, 4, 8])
@pytest.mark.parametrize("kind", ["mix", "int2", "int4", "fp16"])
def test_decode_tiers_and_gqa(m, kind):
    rng = np.random.default_rng(zlib.crc32(f"{m}-{kind}".encode()))
    L, B, H, D, N, tail = 2, 3, 2, 128, 20, 9
    T = N * 32 + tail
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    q = (rng.normal(size=(L, B, H * m, D)) * 2).astype(np.float16)
    if kind == "mix":
        tiers = rng.choice([0, 0, 1, 2], size=(B, N)).astype(np.uint8)
    else:
        tiers = np.full((B, N), {"int2": 0, "int4": 1, "fp16": 2}[kind], np.uint8)
    kd, vd, qd = (torch.from_numpy(x).cuda() for x in (k, v, q))
    cache = batched.build_cache_batched(kd, vd, _search_from_tiers(tiers))
    outs = [cache.decode(qd, splits=s).float().cpu().numpy() for s in (1, 2, 5)]
    for o in outs[1:]:
        assert np.max(np.abs(o - outs[0])) < SCHED_TOL  # schedules agree to ~1e-3 (conftest.SCHED_TOL)
    for l in range(L):
        for b in range(B):
            for h in range(H):
                _check_unit(cache, l, b, h, k, v, tiers[b], q[l, b, h * m:(h + 1) * m], outs[0][l, b, h * m:(h + 1) * m])


def test_large_values_take_the_exact_slow_path():
    rng = np.random.default_rng(9)
    L, B, H, D, N = 1, 2, 1, 128, 8
    T = N * 32
    k = (rng.normal(size=(L, B, T, H, D)) * 2000).astype(np.float16)   # spans >> 192 -> slow path
    v = (rng.uniform(-60000, 60000, size=(L, B, T, H, D))).astype(np.float16)
    q = (rng.normal(size=(L, B, 4 * H, D)) * 1e-3).astype(np.float16)
    tiers = np.array([[0, 1, 0, 2, 0, 1, 0, 0], [1, 1, 0, 0, 0, 0, 2, 2]], np.uint8)
    cache = batched.build_cache_batched(*(torch.from_numpy(x).cuda() for x in (k, v)), _search_from_tiers(tiers))
    out = cache.decode(torch.from_numpy(q).cuda()).float().cpu().numpy()
    for b in range(B):
        _check_unit(cache, 0, b, 0, k, v, tiers[b], q[0, b, :4], out[0, b, :4])


def test_nonfinite_input_rejected():
    k = torch.zeros((1, 1, 64, 1, 128), dtype=torch.float16, device="cuda")
    v = torch.zeros_like(k)
    k[0, 0, 3, 0, 7] = float("inf")
    with pytest.raises(ValueError):
        batched.build_cache_batched(k, v, _search_from_tiers([[0, 1]]))


def test_ragged_contexts_and_decode_appends():
    rng = np.random.default_rng(12)
    L, B, H, m, D = 2, 3, 2, 4, 128
    ctx = np.array([5 * 32 + 3, 12 * 32, 2 * 32 + 31])
    Tmax = int(ctx.max())
    k = rng.normal(size=(L, B, Tmax, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, Tmax, H, D)).astype(np.float16)
    N = ctx // 32
    tiers = np.zeros((B, int(N.max())), np.uint8)
    for b in range(B):
        tiers[b, :N[b]] = rng.choice([0, 1, 2], size=N[b])
    s = retrieval.assign_tiers_batched(tiers.astype(np.float64), np.tile([[0.5, 1.5]], (B, 1)), seq_chunks=N)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), s,
                                        context_lens=ctx, decode_capacity=20)
    kh, vh = k.copy(), v.copy()
    appended_k, appended_v = [], []
    for step in range(17):
        kn = rng.normal(size=(L, B, H, D)).astype(np.float16)
        vn = rng.normal(size=(L, B, H, D)).astype(np.float16)
        cache.append(torch.from_numpy(kn).cuda(), torch.from_numpy(vn).cuda())
        appended_k.append(kn)
        appended_v.append(vn)
    q = (rng.normal(size=(L, B, H * m, D))).astype(np.float16)
    out = cache.decode(torch.from_numpy(q).cuda()).float().cpu().numpy()
    AK, AV = np.stack(appended_k, 2), np.stack(appended_v, 2)  # [L, B, steps, H, D]
    for l in range(L):
        for b in range(B):
            for h in range(H):
                oc = O.build_cache(kh[l, b, :ctx[b], h].astype(np.float64), vh[l, b, :ctx[b], h].astype(np.float64),
                                   tiers[b, :N[b]], 32, 32)
                for t in range(AK.shape[2]):
                    oc.append(AK[l, b, t, h], AV[l, b, t, h])
                ref = O.mixed_decode_attention(q[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
                err = np.max(np.abs(out[l, b, h * m:(h + 1) * m] - ref))
                assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL
    with pytest.raises(ValueError):  # capacity = round_up(len_fp + 20, 16) rows per sequence
        for _ in range(64):
            cache.append(torch.from_numpy(kn).cuda(), torch.from_numpy(vn).cuda())


def test_sequence_split_kv_shards_merge_to_full_decode():
    rng = np.random.default_rng(21)
    L, B, H, m, D, N, tail = 2, 2, 2, 4, 128, 37, 11
    T = N * 32 + tail
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    q = torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16)).cuda()
    s = _search_from_tiers(rng.choice([0, 0, 0, 1, 2], size=(B, N)).astype(np.uint8))
    full = batched.build_cache_batched(k, v, s).decode(q).float()
    for world in (2, 3, 8):
        parts = [distributed.build_sequence_shard(k, v, s, world, r).decode_partial(q) for r in range(world)]
        merged = batched.lse_merge(torch.stack(parts)).view(q.shape).float()
        assert torch.max(torch.abs(merged - full)).item() < SCHED_TOL


def test_full_size_unit_properties_32k():
    """cfg2-sized units (32K context, reference tier maps): bit-exact codes/metadata for sampled
    units and decode within tolerance of the reference's f64 result."""
    import bench
    rng = np.random.default_rng(5)
    L, B, H, m, D, T = 1, 2, 8, 4, 128, 32768
    wls = [bench.load_workload(T, s) for s in range(B)]
    s = retrieval.search_batched(np.stack([w["emb"] for w in wls]), np.stack([w["norm"] for w in wls]),
                                 np.stack([w["q"] for w in wls]), np.array([w["qnorm"] for w in wls]))
    g = torch.Generator(device="cuda").manual_seed(3)
    k = torch.randn((L, B, T, H, D), generator=g, device="cuda", dtype=torch.float16)
    v = torch.randn((L, B, T, H, D), generator=g, device="cuda", dtype=torch.float16)
    q = torch.randn((L, B, H * m, D), generator=g, device="cuda", dtype=torch.float16)
    cache = batched.build_cache_batched(k, v, s)
    out = cache.decode(q).float().cpu().numpy()
    kh, vh, qh = k.cpu().numpy(), v.cpu().numpy(), q.cpu().numpy()
    for b, h in ((0, 0), (1, 5)):
        _check_unit(cache, 0, b, h, kh, vh, wls[b]["tiers"], qh[0, b, h * m:(h + 1) * m], out[0, b, h * m:(h + 1) * m])


def test_per_layer_pdl_launches_match_single_launch():
    rng = np.random.default_rng(31)
    L, B, H, m, D, N = 4, 2, 2, 4, 128, 24
    T = N * 32 + 5
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    q = torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16)).cuda()
    cache = batched.build_cache_batched(k, v, _search_from_tiers(rng.choice([0, 0, 1, 2], size=(B, N)).astype(np.uint8)))
    full = cache.decode(q).float()
    per = torch.empty_like(q)
    for l in range(L):
        cache.decode(q[l:l + 1], out=per[l:l + 1], layer=l, pdl=l > 0)
    assert torch.max(torch.abs(per.float() - full)).item() < SCHED_TOL
    for s in (1, 3, 16, 40):  # 40 > the merge's register fast path
        o = cache.decode(q, splits=s).float()
        assert torch.max(torch.abs(o - full)).item() < SCHED_TOL


def test_exact_mode_for_wide_scales_and_large_q():
    rng = np.random.default_rng(33)
    L, B, H, m, D, N = 1, 2, 2, 4, 128, 8
    T = N * 32
    k = (rng.normal(size=(L, B, T, H, D)) * 3).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v[0, 1, :, 1, :] *= 30000 / 4  # one unit with huge V spans
    tiers = rng.choice([0, 1], size=(B, N)).astype(np.uint8)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search_from_tiers(tiers))
    assert cache.wide_scale_units() >= 1
    for qscale in (1.0, 3000.0):  # |q| * scale_log2 > 1000 forces the unweighted mode too
        q = (rng.normal(size=(L, B, H * m, D)) * qscale).astype(np.float16)
        out = cache.decode(torch.from_numpy(q).cuda()).float().cpu().numpy()
        for b in range(B):
            for h in range(H):
                _check_unit(cache, 0, b, h, k, v, tiers[b], q[0, b, h * m:(h + 1) * m], out[0, b, h * m:(h + 1) * m])


def test_fp16_only_and_int_only_units_with_many_splits():
    rng = np.random.default_rng(35)
    L, B, H, m, D, N = 1, 2, 1, 4, 128, 12
    T = N * 32 + 3
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    tiers = np.stack([np.full(N, 2, np.uint8), np.full(N, 0, np.uint8)])
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search_from_tiers(tiers))
    assert cache.wide_scale_units() == 0
    q = rng.normal(size=(L, B, H * m, D)).astype(np.float16)
    for s in (1, 7, 25):
        out = cache.decode(torch.from_numpy(q).cuda(), splits=s).float().cpu().numpy()
        for b in range(B):
            _check_unit(cache, 0, b, 0, k, v, tiers[b], q[0, b, :m], out[0, b, :m])


@pytest.mark.parametrize("bits", [2, 4])
def test_adversarial_fp16_rows_through_fused_build(bits):
    """The reference's adversarial fp16 rows (grid midpoints, exact ties, subnormals, +-60000;
    tests/golden/make_golden.py) through the fused reorder/quantize/pack kernel (fast fp32
    candidate + guarded exact path, tile-native staging) and back through ckv_arena_export:
    packed words and f64 metadata bit-identical to the reference's quantize_groups/pack_codes."""
    g = load_golden("fp16_rows.npz")
    x = g["x16"]
    n = (x.shape[0] // 32) * 32
    rows = torch.from_numpy(x[:n]).cuda()
    k = rows.reshape(1, 1, n, 1, 128)
    v = torch.flip(rows, dims=[0]).contiguous().reshape(1, 1, n, 1, 128)  # different V rows
    tier = 0 if bits == 2 else 1
    cache = batched.build_cache_batched(k, v, _search_from_tiers(np.full((1, n // 32), tier, np.uint8)))
    ex = cache.export_unit(0, 0, 0)
    words = n * 128 * bits // 32
    kb, vb = (ex.k_q2, ex.v_q2) if bits == 2 else (ex.k_q4, ex.v_q4)
    assert np.array_equal(kb.packed, g[f"packed{bits}"][:words])
    assert np.array_equal(kb.scales.view(np.uint64), g[f"scales{bits}"][:n * 4].view(np.uint64))
    assert np.array_equal(kb.zero_points.view(np.uint64), g[f"zps{bits}"][:n * 4].view(np.uint64))
    want_v = O.quantize_groups(x[:n][::-1].astype(np.float64), bits, 32)
    assert np.array_equal(vb.packed, O.pack_codes(want_v[0].reshape(-1), bits))
    assert np.array_equal(vb.scales.view(np.uint64), want_v[1].view(np.uint64))


def test_layer_by_layer_build_and_per_layer_partials():
    """A cache built one layer at a time (build(..., layer=l)) equals the all-layers build, and
    per-layer decode_partial launches into slices of one buffer equal the single launch
    (the path bench.py's cfg3 uses for caches larger than their fp16 source)."""
    rng = np.random.default_rng(41)
    L, B, H, m, D, N = 3, 2, 2, 2, 128, 20
    T = N * 32 + 7
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    q = torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16)).cuda()
    s = _search_from_tiers(rng.choice([0, 0, 1, 2], size=(B, N)).astype(np.uint8))
    full = batched.build_cache_batched(k, v, s)
    counts = s.seg_counts.cpu().numpy()
    per = batched.BatchedKVCache(L, B, H, counts[:, 0], counts[:, 1], counts[:, 2], [T] * B, device=k.device)
    for l in range(L):
        per.build(k[l:l + 1], v[l:l + 1], s.perm, layer=l)
    assert torch.equal(full.tiles2, per.tiles2) and torch.equal(full.tiles4, per.tiles4)
    assert torch.equal(full.k["fp"], per.k["fp"]) and torch.equal(full.v["fp"], per.v["fp"])
    want = full.decode_partial(q)
    got = torch.empty_like(want)
    rows = B * H * m
    for l in range(L):
        per.decode_partial(q[l:l + 1], layer=l, pdl=l > 0, out=got[l * rows:(l + 1) * rows])
    assert torch.max(torch.abs(batched.lse_merge(got[None]).float() - batched.lse_merge(want[None]).float())).item() < SCHED_TOL


def test_decode_step_host_matches_device_decode():
    """decode_step_host (pinned host q -> overlapped uploads, per-layer PDL decode, overlapped
    downloads) returns exactly the device decode's output, over consecutive steps."""
    rng = np.random.default_rng(51)
    L, B, H, m, D, N = 5, 2, 2, 4, 128, 12
    T = N * 32 + 3
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    cache = batched.build_cache_batched(k, v, _search_from_tiers(rng.choice([0, 1, 2], size=(B, N)).astype(np.uint8)))
    for step in range(3):
        q = torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16))
        oh = torch.empty(q.shape, dtype=torch.float16).pin_memory()
        cache.decode_step_host(q.pin_memory(), oh, d2h_every=2, order_current=step == 0)
        if step:
            cache.host_step_ready.synchronize()
        torch.cuda.synchronize()
        want = cache.decode(q.cuda()).cpu()
        assert torch.equal(oh, want), step


def test_context_shorter_than_one_chunk():
    """A sequence with no full chunk (everything rides in the FP16 tail, harness.py:196-199)
    next to a normal one, built through the layout constructor (no search for the short one)."""
    rng = np.random.default_rng(61)
    L, B, H, m, D = 1, 2, 2, 4, 128
    ctx = np.array([20, 3 * 32 + 1])
    Tmax = int(ctx.max())
    k = rng.normal(size=(L, B, Tmax, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, Tmax, H, D)).astype(np.float16)
    tiers1 = np.array([0, 2, 1], np.uint8)
    counts = np.array([[0, 0, 0], np.bincount(tiers1, minlength=3)])
    perm = np.zeros((B, 3), np.int32)
    perm[1] = np.concatenate([np.nonzero(tiers1 == t)[0] for t in (0, 1, 2)])
    cache = batched.BatchedKVCache(L, B, H, counts[:, 0], counts[:, 1], counts[:, 2], ctx, 8, device=torch.device("cuda"))
    cache.build(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(perm).cuda())
    q = rng.normal(size=(L, B, H * m, D)).astype(np.float16)
    out = cache.decode(torch.from_numpy(q).cuda()).float().cpu().numpy()
    for b, tl in ((0, np.zeros(0, np.uint8)), (1, tiers1)):
        for h in range(H):
            oc = O.build_cache(k[0, b, :ctx[b], h].astype(np.float64), v[0, b, :ctx[b], h].astype(np.float64), tl, 32, 32)
            ref = O.mixed_decode_attention(q[0, b, h * m:(h + 1) * m].astype(np.float64), oc)
            err = np.max(np.abs(out[0, b, h * m:(h + 1) * m] - ref))
            assert err <= TOL_ABS and err / np.max(np.abs(ref)) <= TOL_REL, (b, h, err)


def test_decode_graph_replay_matches_eager():
    """decode_graph: the per-layer PDL-chained step captured in a CUDA graph gives the eager
    launches' output bit for bit, and follows in-place updates of q between replays."""
    rng = np.random.default_rng(71)
    L, B, H, m, D, N = 3, 2, 2, 4, 128, 10
    T = N * 32 + 5
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    cache = batched.build_cache_batched(k, v, _search_from_tiers(rng.choice([0, 1, 2], size=(B, N)).astype(np.uint8)))
    q = torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16)).cuda()
    out = torch.empty_like(q)
    g = cache.decode_graph(q, out, splits=3)
    for _ in range(2):
        g.replay()
        want = torch.empty_like(q)
        for l in range(L):
            cache.decode(q[l:l + 1], splits=3, out=want[l:l + 1], layer=l, pdl=l > 0)
        torch.cuda.synchronize()
        assert torch.equal(out, want)
        q.copy_(torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16)))


def test_decode_graph_sees_decode_appends():
    """A captured decode step keeps working across decode-token appends: the graph's launches
    read the sequence table (len_fp) on the device, so replays attend over the new tokens."""
    rng = np.random.default_rng(72)
    L, B, H, m, D, N = 2, 2, 2, 4, 128, 6
    T = N * 32 + 3
    k = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.normal(size=(L, B, T, H, D)).astype(np.float16)).cuda()
    cache = batched.build_cache_batched(k, v, _search_from_tiers(rng.choice([0, 1, 2], size=(B, N)).astype(np.uint8)),
                                        decode_capacity=16)
    q = torch.from_numpy(rng.normal(size=(L, B, H * m, D)).astype(np.float16)).cuda()
    out = torch.empty_like(q)
    g = cache.decode_graph(q, out, splits=2)
    for _ in range(5):
        cache.append(torch.from_numpy(rng.normal(size=(L, B, H, D)).astype(np.float16)).cuda(),
                     torch.from_numpy(rng.normal(size=(L, B, H, D)).astype(np.float16)).cuda())
        g.replay()
        want = cache.decode(q, splits=2)
        torch.cuda.synchronize()
        assert torch.equal(out, want)


@pytest.mark.parametrize("m", [12, 16])
def test_decode_more_than_eight_q_heads_per_kv_head(m):
    """GQA ratios above 8 (q rows per kv head beyond one launch's MMA columns) run as groups
    of <= 8 rows over the same cache."""
    rng = np.random.default_rng(80 + m)
    L, B, H, D, N = 1, 2, 2, 128, 9
    T = N * 32 + 4
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    tiers = rng.choice([0, 1, 2], size=(B, N)).astype(np.uint8)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search_from_tiers(tiers))
    q = rng.normal(size=(L, B, H * m, D)).astype(np.float16)
    out = cache.decode(torch.from_numpy(q).cuda()).float().cpu().numpy()
    for b in range(B):
        for h in range(H):
            _check_unit(cache, 0, b, h, k, v, tiers[b], q[0, b, h * m:(h + 1) * m], out[0, b, h * m:(h + 1) * m])


def test_reconstruct_and_token_order_tile_native():
    """BatchedKVCache.reconstruct (ckv_reconstruct: the tile-native arenas dequantized and
    scattered to original token order on the device) equals the reference's reconstruct of every
    exported unit bit for bit (f64), including a context tail and appended decode tokens; the
    per-sequence token_order equals the reference's."""
    from paper_2503_23294_b200 import kv_store
    rng = np.random.default_rng(123)
    L, B, H, D = 2, 3, 2, 128
    N, tail = 9, 11
    T = N * 32 + tail
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    tiers = rng.choice([0, 1, 2], size=(B, N), p=(0.5, 0.3, 0.2)).astype(np.uint8)
    s = retrieval.assign_tiers_batched(tiers.astype(np.float64), np.tile([[0.5, 1.5]], (B, 1)))
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), s,
                                        decode_capacity=8)
    for _ in range(3):
        kn = torch.from_numpy(rng.normal(size=(L, B, H, D)).astype(np.float16)).cuda()
        cache.append(kn, kn * 0.5)
    rk, rv = cache.reconstruct()
    rk, rv = rk.cpu().numpy(), rv.cpu().numpy()
    assert rk.shape == (L, B, T + 3, H, D)
    for l in range(L):
        for b in range(B):
            for h in range(H):
                ex = cache.export_unit(l, b, h)
                wk, wv = kv_store.reconstruct(ex)
                assert np.array_equal(rk[l, b, :, h], wk) and np.array_equal(rv[l, b, :, h], wv), (l, b, h)
                assert np.array_equal(cache.token_order(b), kv_store.token_order(ex))
    # FP16-tier and tail rows come back exactly; quantized rows within the group's half-step
    assert np.array_equal(rk[:, :, N * 32:T], k[:, :, N * 32:T].astype(np.float64))
    one = cache.reconstruct(layer=1, layers=1, t_out=T)[0].cpu().numpy()
    assert one.shape == (1, B, T, H, D) and np.array_equal(one[0], rk[1, :, :T])
