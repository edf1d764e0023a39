"""One cfg2 decode step (+ optional cfg5 prefill build) for ncu captures; prints nothing measured.
--chains 0 (default) runs the step as bench.py's default does: one micro-batch chain per
sequence, each its own sequence of per-layer launches (split schedule, chain_splits); --chains 1
the lockstep whole-batch per-layer launches (the cache's schedule)."""
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
    ap.add_argument("--chains", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    bench.CFG2["layers"] = args.layers
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    m = q.shape[2] // cache.H
    chains = cache.B if args.chains == 0 else args.chains
    ns = argparse.Namespace(schedule=args.schedule, splits=None, chains=chains)
    splits = bench.pick_splits(ns, cache, m)  # None: the warp plan
    out = torch.empty_like(q)
    streams = [torch.cuda.Stream(device=dev) for _ in range(chains)]
    cache._launch_layers(q, out, 0, cache.L, splits, None, chains, streams)  # warm-up outside the range
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.steps):
        cache._launch_layers(q, out, 0, cache.L, splits, None, chains, streams)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    if args.prefill:
        del cache
        torch.cuda.empty_cache()
        bench.bench_prefill(torch, dev, steps=1, profile=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
