"""One cfg2 decode step (+ optional cfg5 prefill build) for ncu captures; prints nothing measured."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--prefill", action="store_true")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--schedule", choices=["auto", "wp", "split"], default="auto")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    bench.CFG2["layers"] = args.layers
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    m = q.shape[2] // cache.H
    splits = None if args.schedule != "split" else cache.default_splits(m, 1)  # None: the cache's schedule
    cache.schedule = args.schedule
    out = torch.empty_like(q)
    for l in range(cache.L):  # warm-up outside the profiled range
        cache.decode(q[l:l + 1], splits=splits, out=out[l:l + 1], layer=l, pdl=l > 0)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.steps):
        for l in range(cache.L):
            cache.decode(q[l:l + 1], splits=splits, out=out[l:l + 1], layer=l, pdl=l > 0)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    if args.prefill:
        del cache
        torch.cuda.empty_cache()
        bench.bench_prefill(torch, dev, steps=1, profile=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
