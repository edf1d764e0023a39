"""Decode precision across wide groups and large q.  Round 1's kernel routed units by
span_max x max|q| (log2-scaled q; a precise K path above 8), by max|q| (an exact mode above
1000) and by the quantize kernel's 4000 scale cutoff; the current kernel has one path (codes as
exact fp16 subnormals in the MMA, group scales in fp32: DESIGN §3 K3), and these former
boundaries stay as test points.  On both sides of each the output must meet the north_star
tolerance (1e-2 abs and 1e-2 of max|ref|) against the reference's f64 mixed_decode_attention on
the same fp16 inputs, with a peaky softmax (q aligned with a few keys)."""

import math

import numpy as np
import pytest
import torch

from oracle import ckv_oracle as O
from paper_2503_23294_b200 import batched, retrieval

pytestmark = pytest.mark.gpu

TOL = 1e-2
LOG2E = 1.4426950408889634


def _search(tiers):
    return retrieval.assign_tiers_batched(tiers.astype(np.float64), np.tile([[0.5, 1.5]], (tiers.shape[0], 1)))


def _unit_case(seed, T=4096, m=4, outlier=8.0):
    """One (layer, sequence) with two kv heads: K ~ N(0,1) with one channel per 32-wide group
    scaled by `outlier` (wide group spans), V ~ N(0,1), q built from a few keys (peaky)."""
    rng = np.random.default_rng(seed)
    n = T // 32
    k = rng.normal(size=(1, 1, T, 2, 128)).astype(np.float32)
    k[..., [3, 40, 77, 100]] *= outlier
    v = rng.normal(size=(1, 1, T, 2, 128)).astype(np.float32)
    q = np.zeros((1, 1, 2 * m, 128), np.float32)
    for h in range(2):
        for r in range(m):
            toks = rng.choice(T, size=3, replace=False)
            q[0, 0, h * m + r] = k[0, 0, toks, h].sum(axis=0) + 0.3 * rng.normal(size=128)
    tiers = rng.choice([0, 0, 0, 1, 2], size=(1, n)).astype(np.uint8)
    return k.astype(np.float16), v.astype(np.float16), q, tiers


def _scaled_q(q, factor):
    return (q * factor).astype(np.float16)


def _q_log2_max(q16, h, m):
    """max |fp16(q * log2(e) / sqrt(128))| over the unit's rows, as the kernel computes it."""
    rows = q16[0, 0, h * m:(h + 1) * m].astype(np.float32)
    return float(np.max(np.abs((rows * np.float32(LOG2E / math.sqrt(128))).astype(np.float16).astype(np.float32))))


def _run(k, v, q16, tiers, m):
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search(tiers))
    out = cache.decode(torch.from_numpy(q16).cuda(), splits=3).float().cpu().numpy()
    worst = 0.0
    for h in range(2):
        oc = O.build_cache(k[0, 0, :, h].astype(np.float64), v[0, 0, :, h].astype(np.float64), tiers[0], 32, 32)
        ref = O.mixed_decode_attention(q16[0, 0, h * m:(h + 1) * m].astype(np.float64), oc)
        got = out[0, 0, h * m:(h + 1) * m].astype(np.float64)
        err = np.max(np.abs(got - ref))
        assert err <= TOL, (h, err)
        worst = max(worst, err / max(np.max(np.abs(ref)), 1e-30))
    assert worst <= TOL, worst
    return cache


@pytest.mark.parametrize("m", [4, 8])
@pytest.mark.parametrize("product", [7.5, 8.5, 60.0])
def test_precise_threshold_both_sides(product, m):
    """span_max x max|q| just under, just over and far over round 1's precise-path threshold (8)."""
    k, v, q, tiers = _unit_case(11 + m, m=m)
    cache = batched.build_cache_batched(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), _search(tiers))
    span = cache.k["span_max"].view(torch.float32)[0, :, 0].cpu().numpy()
    f = product / max(float(span[h]) * _q_log2_max(q.astype(np.float16), h, m) for h in range(2))
    q16 = _scaled_q(q, f)
    got = max(float(span[h]) * _q_log2_max(q16, h, m) for h in range(2))
    assert abs(got - product) / product < 0.02, got
    _run(k, v, q16, tiers, m)


@pytest.mark.parametrize("qmax", [990.0, 1010.0])
def test_wide_q_boundary(qmax):
    """max|q| (log2-scaled) just under / over round 1's exact-mode threshold (1000)."""
    k, v, q, tiers = _unit_case(21, outlier=1.0)
    f = qmax / max(_q_log2_max(q.astype(np.float16), h, 4) for h in range(2))
    _run(k, v, _scaled_q(q, f), tiers, 4)


@pytest.mark.parametrize("scale", [3990.0, 4010.0])
def test_scale_cutoff_boundary(scale):
    """An INT2 group whose scale (span / 3) sits just under / over the 4000 cutoff: the unit's
    (diagnostic) span flag is set exactly above it, and the output meets the gate on both sides."""
    k, v, q, tiers = _unit_case(31, outlier=1.0)
    tiers[:] = 0  # all INT2 except the FP16 chunks the map would have: all quantized
    k[0, 0, 100, 0, 0] = np.float16(3 * scale + float(k[0, 0, 100, 0, 1:32].min()))
    cache = _run(k, v, _scaled_q(q, 0.05), tiers, 4)
    flags = cache.k["span_flags"][0, :, 0].cpu().numpy()
    assert bool(flags[0] & 1) == (scale > 4000), flags
