"""Where the time of the bench's default decode step goes (cfg2, one micro-batch chain per
sequence, split kernel): per-CTA globaltimer trace (ckv_decode_set_trace) of one traced step.
Prints the CTA-slot utilisation of the SMs over the step (4 resident CTAs per SM at most), the
share of CTA time spent in each phase (launch -> PDL wait, q staging, tiles, merge tail), and the
per-chain layer spacing."""
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
    ap.add_argument("--chains", type=int, default=8)
    ap.add_argument("--splits", type=int, default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    m = q.shape[2] // cache.H
    ns = argparse.Namespace(schedule="auto", splits=args.splits, chains=args.chains)
    splits = bench.pick_splits(ns, cache, m)
    out = torch.empty_like(q)
    streams = [torch.cuda.Stream(device=dev) for _ in range(args.chains)]  # eager warm-up only
    lib = _lib.load()
    lib.ckv_decode_set_trace.argtypes = [ctypes.c_void_p]

    def step():
        cache._launch_layers(q, out, 0, cache.L, splits, None, args.chains, streams)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    buf = torch.zeros((400000, 16), dtype=torch.int64, device=dev)
    # the trace pointer is a kernel parameter: arm it, then capture the step as the bench runs
    # it (one CUDA graph; eager chained launches are host-bound)
    lib.ckv_decode_set_trace(ctypes.c_void_p(buf.data_ptr()))
    g = cache.decode_graph(q, out, splits=splits, chains=args.chains)
    for _ in range(3):  # the first replays of a fresh graph launch its branches late (upload)
        g.replay()
    torch.cuda.synchronize()
    buf.zero_()
    g.replay()
    torch.cuda.synchronize()
    lib.ckv_decode_set_trace(ctypes.c_void_p(0))
    t = buf.cpu().numpy()
    t = t[t[:, 0] != 0]
    t0, t1 = t[:, 0].min(), t[:, 4].max()
    span = (t1 - t0) / 1e3
    print(f"chains {args.chains}, splits {splits}: traced step {span:.1f} us, {len(t)} CTAs")
    st, wt, qs, en = t[:, 0], t[:, 1], t[:, 2], t[:, 4]
    te = t[:, 12:16].max(1)  # last warp's tiles end
    life = (en - st).sum()
    for name, a, b in (("launch -> PDL wait done", st, wt), ("q staging", wt, qs), ("tiles", qs, te),
                       ("merge tail", te, en)):
        print(f"  {name:24s} {100 * (b - a).sum() / life:5.1f} % of CTA time, median {np.median(b - a) / 1e3:6.2f} us")
    t8, t9 = t[:, 8], t[:, 9]
    ok = (t8 > 0) & (t9 > 0)
    for name, a, b in (("finish warps + barrier", te, t8), ("park + in-CTA merge + partial", t8, t9),
                       ("arrival + final merge", t9, en)):
        print(f"    {name:30s} median {np.median((b - a)[ok]) / 1e3:6.2f} us, p90 {np.percentile((b - a)[ok], 90) / 1e3:6.2f}")
    sp = t[:, 12:16].max(1) - t[:, 12:16].min(1)
    print("warp spread of tile ends within a CTA us: p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(sp, [50, 90, 100]) / 1e3))
    # CTA-slot utilisation: resident CTAs per SM over time, vs the 4-slot capacity
    sms = np.unique(t[:, 5])
    grid = np.linspace(t0, t1, 2001)
    occ = np.zeros((len(sms), len(grid)))
    tiles = np.zeros_like(occ)
    for i, s in enumerate(sms):
        x = t[t[:, 5] == s]
        for r in x:
            occ[i] += (grid >= r[0]) & (grid < r[4])
            tiles[i] += (grid >= r[2]) & (grid < r[12:16].max())
    print(f"resident CTAs per SM (mean over the step): {occ.mean():.2f} of 4; in their tile phase: {tiles.mean():.2f}")
    q10 = np.percentile(occ.mean(0), [10, 50, 90])
    print(f"  across time: p10 {q10[0]:.2f} p50 {q10[1]:.2f} p90 {q10[2]:.2f}; first/last 5 % of the step: "
          f"{occ[:, :100].mean():.2f} / {occ[:, -100:].mean():.2f}")
    # per-chain layer spacing (launch id = (q pointer, first unit) -> chain by its sequence)
    seq_of = (t[:, 6] >> 40) // cache.H
    for c in range(min(args.chains, 2)):
        x = t[seq_of == c]
        ends = sorted({int(p): x[x[:, 7] == p, 4].max() for p in np.unique(x[:, 7])}.values())
        d = np.diff(ends) / 1e3
        print(f"chain {c}: {len(ends)} launches, end-to-end spacing median {np.median(d):.1f} us")
    # the step's ramp and drain: when every chain's first CTA starts / last CTA ends
    for c in range(min(args.chains, cache.B)):
        x = t[seq_of == c]
        print(f"chain {c}: first CTA start +{(x[:, 0].min() - t0) / 1e3:6.1f} us, first tiles +"
              f"{(x[:, 2].min() - t0) / 1e3:6.1f} us, last CTA end -{(t1 - x[:, 4].max()) / 1e3:6.1f} us")
    # how the chains drift apart: spread over chains of each layer's end time
    ptrs = np.unique(t[:, 7])
    lay = np.searchsorted(ptrs, t[:, 7])
    spread = []
    for l in range(len(ptrs)):
        e = [t[(lay == l) & (seq_of == c), 4].max() for c in range(min(args.chains, cache.B))
             if ((lay == l) & (seq_of == c)).any()]
        spread.append((max(e) - min(e)) / 1e3)
    print("spread of the chains' layer end times us, per layer: " + " ".join(f"{x:.0f}" for x in spread))
    bins = np.arange(0, 21)
    for name, ref, sgn in (("start", t0, 1), ("end", t1, -1)):
        row = []
        for i in bins[:-1]:
            a, b = (ref + i * 10000, ref + (i + 1) * 10000) if sgn > 0 else (ref - (i + 1) * 10000, ref - i * 10000)
            sel = (grid >= a) & (grid < b)
            row.append(occ[:, sel].mean() if sel.any() else float("nan"))
        print(f"resident CTAs per SM in 10 us bins from the step {name}: " + " ".join(f"{v:.2f}" for v in row))


if __name__ == "__main__":
    main()
