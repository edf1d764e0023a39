"""cfg4 bitwidth-mix sweep: batch 64 x 16K, Llama-3-8B GQA (8 kv heads, m = 4), one layer per
launch; all-FP16, all-INT2 and the skewed reference maps (sequence b: 16K seed b % 8).
Prints algorithmic GB/s per map (decode only, device-timed, inputs > L2)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_23294_b200 import batched, retrieval  # noqa: E402


def run(kind, L=2, B=64, H=8, m=4, T=16384, steps=10):
    n = T // 32
    if kind == "skewed":
        maps = np.stack([bench.load_workload(T, b % 8)["tiers"] for b in range(B)])
    else:
        maps = np.full((B, n), 2 if kind == "all_fp16" else 0, np.uint8)
    s = retrieval.assign_tiers_batched(maps.astype(np.float64), np.tile([[0.5, 1.5]], (B, 1)))
    g = torch.Generator(device="cuda").manual_seed(5)
    k = torch.randn((L, B, T, H, 128), generator=g, device="cuda", dtype=torch.float16)
    v = torch.randn((L, B, T, H, 128), generator=g, device="cuda", dtype=torch.float16)
    cache = batched.build_cache_batched(k, v, s)
    cache.schedule = os.environ.get("CKV_SCHEDULE", "auto")
    del k, v
    q = torch.randn((L, B, H * m, 128), generator=g, device="cuda", dtype=torch.float16)
    out = torch.empty_like(q)
    step = lambda: [cache.decode(q[l:l + 1], out=out[l:l + 1], layer=l, pdl=l > 0) for l in range(L)]  # noqa: E731
    for _ in range(3):
        step()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / L)
    ms = statistics.median(ts)
    nbytes = cache.algorithmic_bytes(m) / L
    del cache
    torch.cuda.empty_cache()
    return {"map": kind, "ms_per_layer": round(ms, 4), "gb_per_layer": round(nbytes / 1e9, 3),
            "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1)}


if __name__ == "__main__":
    for kind in sys.argv[1:] or ("all_fp16", "all_int2", "skewed"):
        r = run(kind)
        r["schedule"] = os.environ.get("CKV_SCHEDULE", "auto")
        print(json.dumps(r))
