"""Probe (tuning aid): what the DecodeLoop's per-step input copies cost beside a plain graph
replay of the cfg2 default step, variants interleaved 5 times (the step time drifts upward as
the board reaches its power limit within ~0.3 s of load, so only interleaved variants compare;
see tools/sustained_probe.py)."""
import sys, os, torch, argparse
sys.path.insert(0, os.getcwd())
import bench
from paper_2503_23294_b200 import batched
dev = torch.device("cuda", 0)
cache, q, _ = bench.build_cfg2(torch, dev, 0)
cache.cap_fp = cache.cap_fp  # noqa
m = q.shape[2] // cache.H
ns = argparse.Namespace(schedule="auto", splits=None, chains=8)
splits = bench.pick_splits(ns, cache, m)
loop = batched.DecodeLoop(cache, m, splits=splits, chains=8)
L, B, H = cache.L, cache.B, cache.H
kn = torch.randn((L, B, H, 128), device=dev, dtype=torch.float16)
tiny = torch.zeros(16, device=dev)
def run(name, fn, n=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / n:.4f} ms", flush=True)
def replay(): cache.seq_host[:, 5] -= 0; loop.graph.replay()
# keep the cache size fixed: replays re-append into the same slot? no: use decode graph instead
out = torch.empty_like(q)
g = cache.decode_graph(q, out, splits=splits, chains=8)
variants = [("replay", g.replay),
            ("replay + tiny kernel", lambda: (tiny.add_(1), g.replay())),
            ("replay + 3 copies", lambda: (loop.q.copy_(q), loop.k_new.copy_(kn), loop.v_new.copy_(kn), g.replay())),
            ("replay + q copy", lambda: (loop.q.copy_(q), g.replay()))]
import collections
res = collections.defaultdict(list)
for rep in range(5):
    for name, fn in variants:
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 20)
for name, v in res.items():
    print(f"{name}: " + " ".join(f"{x:.4f}" for x in v))
