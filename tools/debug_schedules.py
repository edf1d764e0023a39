"""Debug aid: one small decode case through every schedule (warp plan, split 1/2/5) against the
oracle; prints max abs error per schedule and between schedules."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ckv_oracle as O  # noqa: E402
from paper_2503_23294_b200 import batched  # noqa: E402
from tests.test_gpu_batched import _search_from_tiers  # noqa: E402


def main(m=8, kind="int2", seed=None):
    rng = np.random.default_rng(hash((m, kind)) % 2**32 if seed is None else seed)
    L, B, H, D, N, tail = 2, 3, 2, 128, 20, 9
    T = N * 32 + tail
    k = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    v = rng.normal(size=(L, B, T, H, D)).astype(np.float16)
    q = (rng.normal(size=(L, B, H * m, D)) * 2).astype(np.float16)
    tiers = np.full((B, N), {"int2": 0, "int4": 1, "fp16": 2}[kind], np.uint8)
    kd, vd, qd = (torch.from_numpy(x).cuda() for x in (k, v, q))
    cache = batched.build_cache_batched(kd, vd, _search_from_tiers(tiers))
    outs = {"wp": cache.decode(qd, schedule="wp").float().cpu().numpy()}
    for s in (1, 2, 5):
        outs[f"split{s}"] = cache.decode(qd, splits=s, schedule="split").float().cpu().numpy()
    ref = np.zeros_like(outs["wp"])
    for l in range(L):
        for b in range(B):
            for h in range(H):
                oc = O.build_cache(k[l, b, :, h].astype(np.float64), v[l, b, :, h].astype(np.float64), tiers[b], 32, 32)
                ref[l, b, h * m:(h + 1) * m] = O.mixed_decode_attention(q[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
    for name, o in outs.items():
        e = np.abs(o - ref)
        idx = np.unravel_index(np.argmax(e), e.shape)
        print(f"{name}: max err vs oracle {e.max():.2e} at {idx}; vs wp {np.abs(o - outs['wp']).max():.2e}")


if __name__ == "__main__":
    main()
