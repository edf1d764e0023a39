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
    print(f"splits {splits}; step {e0.elapsed_time(e1):.3f} ms (events, traced); {len(t)} CTAs")
    launches = sorted(set(t[:, 7].tolist()), key=lambda p: t[t[:, 7] == p, 0].min())
    prev_end = None
    rows = []
    for i, p in enumerate(launches):
        x = t[t[:, 7] == p]
        st, wt, qs, te, en = (x[:, k] - t0 for k in range(5))
        rows.append((i, len(x), st.min(), st.max(), wt.min(), wt.max(), qs.max(), np.median(te - qs),
                     (te - qs).max(), te.min(), te.max(), en.max(), np.median(en - te), (en - te).max()))
        prev_end = en.max()
    print("layer ctas start[min,max] wait_done[min,max] qsync_max tiles[med,max] tiles_end[min,max] end_max merge[med,max]  (us)")
    for r in rows:
        i, n = r[0], r[1]
        v = [x / 1e3 for x in r[2:]]
        print(f"{i:3d} {n:4d}  [{v[0]:8.1f},{v[1]:8.1f}] [{v[2]:8.1f},{v[3]:8.1f}] {v[4]:8.1f} [{v[5]:6.1f},{v[6]:6.1f}] "
              f"[{v[7]:8.1f},{v[8]:8.1f}] {v[9]:8.1f} [{v[10]:5.1f},{v[11]:5.1f}]")
    ends = [r[11] for r in rows]
    if len(ends) > 1:
        d = np.diff(ends) / 1e3
        print(f"layer-to-layer end spacing: median {np.median(d):.1f} us, mean {d.mean():.1f} us")
    # inside a layer: warp spread, local merge, arrival atomic, final split merge
    wt = t[:, 12:16]
    tiles_w = wt - t[:, 2:3]
    spread = wt.max(1) - wt.min(1)
    print("per-warp tile time us: p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(tiles_w, [10, 50, 90, 100]) / 1e3))
    print("warp spread within CTA us: p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(spread, [50, 90, 100]) / 1e3))
    print("local merge (all tiles -> before atomic) us: p50 %.1f max %.1f" % tuple(np.percentile(t[:, 9] - t[:, 8], [50, 100]) / 1e3))
    print("arrival atomic us: p50 %.1f max %.1f" % tuple(np.percentile(t[:, 10] - t[:, 9], [50, 100]) / 1e3))
    last = t[t[:, 11] == 1]
    if len(last):
        print("final split merge (last CTA) us: p50 %.1f max %.1f" % tuple(np.percentile(last[:, 4] - last[:, 10], [50, 100]) / 1e3))
    # per-SM speed: CTA tile time relative to its layer's median, averaged per SM over layers
    rel = np.zeros(len(t))
    for p in launches:
        sel = t[:, 7] == p
        d = (t[sel, 12:16].max(1) - t[sel, 2])
        rel[sel] = d / np.median(d)
    sms = np.unique(t[:, 5])
    half = [launches[: len(launches) // 2], launches[len(launches) // 2:]]
    a = np.array([[rel[(t[:, 5] == s) & np.isin(t[:, 7], h)].mean() for s in sms] for h in half])
    print("per-SM relative tile time: min %.3f max %.3f; correlation between layer halves %.2f" % (
        a.mean(0).min(), a.mean(0).max(), np.corrcoef(a[0], a[1])[0, 1]))
    order = np.argsort(a.mean(0))
    print("slowest SMs:", [(int(sms[k]), round(float(a.mean(0)[k]), 3)) for k in order[-8:]])
    print("fastest SMs:", [(int(sms[k]), round(float(a.mean(0)[k]), 3)) for k in order[:8]])
    # does the CTA count on an SM explain it?
    mid = launches[len(launches) // 2]
    x = t[t[:, 7] == mid]
    per_sm = {}
    for r in x:
        per_sm.setdefault(int(r[5]), []).append((r[12:16].max() - r[2]) / 1e3)
    by_n = {}
    for v in per_sm.values():
        by_n.setdefault(len(v), []).append(np.mean(v))
    print("median layer: tile time by CTAs/SM:", {k: round(float(np.mean(v)), 1) for k, v in by_n.items()})
    # variance decomposition over all layers: SM-level vs unit-level (CTAs of a unit share the
    # unit's data) vs residual, for CTAs on 4-CTA SMs
    nsplit = splits
    res = {"sm": [], "unit": []}
    for p_ in launches:
        x = t[t[:, 7] == p_]
        tt = x[:, 12:16].max(1) - x[:, 2]
        sm = x[:, 5]
        unit = x[:, 6] >> 40
        cnt = {k: v for k, v in zip(*np.unique(sm, return_counts=True))}
        keep = np.array([cnt[k] == 4 for k in sm])
        tt, sm, unit = tt[keep], sm[keep], unit[keep]
        dev = tt - tt.mean()
        sm_mean = {k: dev[sm == k].mean() for k in np.unique(sm)}
        un_mean = {k: dev[unit == k].mean() for k in np.unique(unit)}
        res["sm"].append(np.var([sm_mean[k] for k in sm]) / np.var(dev))
        res["unit"].append(np.var([un_mean[k] for k in unit]) / np.var(dev))
    print("variance share of per-SM means %.2f, of per-unit means %.2f (4-CTA SMs)" % (
        np.mean(res["sm"]), np.mean(res["unit"])))
    # per-tile cost regression (static split: CTA `split` of unit (b, h) takes the same share of
    # INT2, INT4 and FP16-region tiles): CTA tile time ~ t0 + c2 n2 + c4 n4 + cf nf
    if not args.single:
        sh = cache.seq_host.astype(np.int64)
        n2t, n4t, nft = sh[:, 1] // 16, sh[:, 3] // 16, (sh[:, 5] + 15) // 16
        S, H = splits, cache.H
        X, Y = [], []
        for p_ in launches:
            x = t[t[:, 7] == p_]
            for r in x:
                sp = (int(r[6]) >> 20) & 0xFFFFF; b = (int(r[6]) >> 40) // H
                f = lambda n: n * (sp + 1) // S - n * sp // S  # noqa: E731
                X.append([1.0, f(n2t[b]), f(n4t[b]), f(nft[b])])
                Y.append((r[12:16].max() - r[2]) / 1e3)
        X, Y = np.array(X, float), np.array(Y)
        coef, *_ = np.linalg.lstsq(X, Y, rcond=None)
        pred = X @ coef
        U = np.zeros((len(launches), cache.B, H))
        for li, p_ in enumerate(launches):
            x = t[t[:, 7] == p_]
            tt = x[:, 12:16].max(1) - x[:, 2]
            for r, v in zip(x, tt):
                u = int(r[6]) >> 40; b, h = u // H, u % H
                U[li, b, h] += v / S / 1e3
        U /= U.mean(axis=(1, 2), keepdims=True)
        half = len(launches) // 2
        print("per-unit relative time, correlation between layer halves: %.2f" % np.corrcoef(
            U[:half].mean(0).ravel(), U[half:].mean(0).ravel())[0, 1])
        print("mean over layers, rows = sequence b, cols = kv head h:")
        print(np.array2string(U.mean(0), precision=3))
        print("per-layer std of unit means %.3f; layer-to-layer std of a unit %.3f" % (
            U.std(axis=(1, 2)).mean(), U.std(axis=0).mean()))
        # relative CTA tile time by launch position (bins of 64 positions), median over layers
        P = []
        for p_ in launches:
            x = t[t[:, 7] == p_]
            tt = x[:, 12:16].max(1) - x[:, 2]
            P.append((x[:, 6] & 0xFFFFF, tt / np.median(tt)))
        pos = np.concatenate([a for a, _ in P]); rv = np.concatenate([b for _, b in P])
        nb = int(pos.max()) // 64 + 1
        print("relative CTA tile time by launch position / 64:",
              [round(float(np.mean(rv[pos // 64 == k])), 3) for k in range(nb)])
        print("tile-time model: t0 %.2f us, INT2 %.4f, INT4 %.4f, FP16 %.4f us/tile (per CTA); "
              "ratios INT4/INT2 %.2f FP16/INT2 %.2f; R^2 %.2f" % (
                  coef[0], coef[1], coef[2], coef[3], coef[2] / coef[1], coef[3] / coef[1],
                  1 - np.var(Y - pred) / np.var(Y)))


if __name__ == "__main__":
    main()
