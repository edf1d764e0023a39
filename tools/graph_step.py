"""cfg2 decode step captured in a CUDA graph (32 PDL-chained per-layer launches) vs eager."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    m = q.shape[2] // cache.H
    splits = cache.default_splits(m, 1)
    out = torch.empty_like(q)
    nbytes = cache.algorithmic_bytes(m)

    def step():
        for l in range(cache.L):
            cache.decode(q[l:l + 1], splits=splits, out=out[l:l + 1], layer=l, pdl=l > 0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    res = {}
    for name, fn in (("eager", step), ("graph", g.replay)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res[name] = {"ms": round(ms, 4), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1)}
    ref = out.clone()
    step()
    torch.cuda.synchronize()
    res["graph_equals_eager"] = bool(torch.equal(ref, out))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
