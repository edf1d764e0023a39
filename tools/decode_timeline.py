"""Per-CTA timeline of one cfg2 decode step (per-layer PDL launches), from the kernel's
optional globaltimer trace (ckv_decode_set_trace).  Prints per-layer spans and where the
time of a layer goes: launch-to-wait, q staging, tiles, merge tail."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_23294_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--splits", type=int, default=None)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--single", action="store_true", help="one launch for all layers")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    bench.CFG2["layers"] = args.layers
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    m = q.shape[2] // cache.H
    splits = args.splits or cache.default_splits(m, 1)
    out = torch.empty_like(q)
    lib = _lib.load()
    lib.ckv_decode_set_trace.argtypes = [ctypes.c_void_p]

    def step():
        if args.single:
            cache.decode(q, out=out, splits=splits)
            return
        for l in range(cache.L):
            cache.decode(q[l:l + 1], splits=splits, out=out[l:l + 1], layer=l, pdl=l > 0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    buf = torch.zeros((200000, 16), dtype=torch.int64, device=dev)
    lib.ckv_decode_set_trace(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    lib.ckv_decode_set_trace(ctypes.c_void_p(0))
    t = buf.cpu().numpy()
    t = t[t[:, 0] != 0]
    t0 = t[:, 0].min()
    print(f"ctas {splits}; step {e0.elapsed_time(e1):.3f} ms (events, traced); {len(t)} CTAs")
    launches = sorted(set(t[:, 7].tolist()), key=lambda p: t[t[:, 7] == p, 0].min())
    print("layer ctas start[min,max] wait_done qsync_max tiles[med,max] tiles_end[min,max] end_max  (us)")
    ends = []
    for i, p in enumerate(launches):
        x = t[t[:, 7] == p]
        st, wt, qs, te, en = (x[:, k] - t0 for k in range(5))
        tt = te - qs
        ends.append(en.max())
        if i < 4 or i >= len(launches) - 2:
            print(f"{i:3d} {len(x):4d}  [{st.min()/1e3:8.1f},{st.max()/1e3:8.1f}] {wt.max()/1e3:8.1f} {qs.max()/1e3:8.1f} "
                  f"[{np.median(tt)/1e3:6.1f},{tt.max()/1e3:6.1f}] [{te.min()/1e3:8.1f},{te.max()/1e3:8.1f}] {en.max()/1e3:8.1f}")
    if len(ends) > 1:
        d = np.diff(ends) / 1e3
        print(f"layer-to-layer end spacing: median {np.median(d):.1f} us, mean {d.mean():.1f} us")
    tt = (t[:, 3] - t[:, 2]) / 1e3
    print("per-CTA qsync->tiles-end us: p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(tt, [10, 50, 90, 100])))
    tail = (t[:, 4] - t[:, 3]) / 1e3
    print("tiles-end -> exit (merge) us: p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(tail, [50, 90, 100])))
    ramp = (t[:, 2] - t[:, 1]) / 1e3
    print("wait -> first q staged us: p50 %.1f max %.1f" % tuple(np.percentile(ramp, [50, 100])))
    print("segments per CTA:", dict(zip(*[v.tolist() for v in np.unique(t[:, 8], return_counts=True)])))
    for p in launches[len(launches) // 2: len(launches) // 2 + 1]:
        x = t[t[:, 7] == p]
        sm_cnt = np.bincount(np.unique(x[:, 5], return_counts=True)[1])
        print("median layer: CTAs per SM histogram", sm_cnt.tolist())


if __name__ == "__main__":
    main()
