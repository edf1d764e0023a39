import sys, os, torch, argparse
sys.path.insert(0, os.getcwd())
import bench
from paper_2503_23294_b200 import batched
dev = torch.device("cuda", 0)
cache, q, _ = bench.build_cfg2(torch, dev, 0)
m = q.shape[2] // cache.H
ns = argparse.Namespace(schedule="auto", splits=None, chains=8)
splits = bench.pick_splits(ns, cache, m)
out = torch.empty_like(q)
def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
g = cache.decode_graph(q, out, splits=splits, chains=8)
print("step graph before appends: %.4f ms" % timeit(g.replay))
loop = batched.DecodeLoop(cache, m, splits=splits, chains=8)
L, B, H = cache.L, cache.B, cache.H
kn = torch.randn((L, B, H, 128), device=dev, dtype=torch.float16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
n = 100
for i in range(n): loop.step(q, kn, kn)
e1.record(); torch.cuda.synchronize()
print("DecodeLoop step (append + decode): %.4f ms" % (e0.elapsed_time(e1) / n))
g2 = cache.decode_graph(q, out, splits=splits, chains=8)
print("step graph after %d appends: %.4f ms" % (n, timeit(g2.replay)))
print("loop graph replay only (no input copies, no reserve; appends into the remaining capacity):")
e0.record()
for i in range(20):
    cache._reserve_decode_token(); loop.graph.replay()
e1.record(); torch.cuda.synchronize()
print("  %.4f ms" % (e0.elapsed_time(e1) / 20))
# the append alone, captured the same way
kn2 = torch.zeros((L, B, H, 128), device=dev, dtype=torch.float16)
side = torch.cuda.Stream(device=dev)
side.wait_stream(torch.cuda.current_stream())
ga = torch.cuda.CUDAGraph()
with torch.cuda.graph(ga, stream=side):
    cache._append_device(kn2, kn2)
torch.cuda.synchronize()
left = int((cache.cap_fp - cache.seq_host[:, 5]).min())
e0.record()
for i in range(min(10, left)):
    cache._reserve_decode_token(); ga.replay()
e1.record(); torch.cuda.synchronize()
print("append graph alone: %.4f ms" % (e0.elapsed_time(e1) / min(10, left)))
print("decode graph at the final state: %.4f ms" % timeit(g2.replay))
