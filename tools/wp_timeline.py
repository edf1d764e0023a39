"""Per-CTA timeline of one cfg2 decode step with the warp-plan kernel (per-layer launches):
where a layer's time goes (PDL release, q staging, tiles, in-CTA merge, arrival, final merge)."""
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
    dev = torch.device("cuda", 0)
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    out = torch.empty_like(q)
    lib = _lib.load()
    lib.ckv_decode_set_trace.argtypes = [ctypes.c_void_p]

    def step():
        for l in range(cache.L):
            cache.decode(q[l:l + 1], out=out[l:l + 1], layer=l, pdl=l > 0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    buf = torch.zeros((100000, 16), dtype=torch.int64, device=dev)
    lib.ckv_decode_set_trace(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    lib.ckv_decode_set_trace(ctypes.c_void_p(0))
    t = buf.cpu().numpy()
    t = t[t[:, 0] != 0]
    print(f"step {e0.elapsed_time(e1):.3f} ms (traced); {len(t)} CTAs")
    launches = sorted(set(t[:, 7].tolist()), key=lambda p: t[t[:, 7] == p, 0].min())
    t0 = t[:, 0].min()
    rel = lambda x: (x - t0) / 1e3  # noqa: E731
    rows = []
    for p in launches:
        x = t[t[:, 7] == p]
        rows.append([rel(x[:, 0].min()), rel(x[:, 0].max()), rel(x[:, 1].max()), rel(x[:, 2].max()),
                     rel(x[:, 3].min()), rel(x[:, 3].max()), rel(x[:, 4].max()),
                     np.median(x[:, 3] - x[:, 2]) / 1e3, np.median(x[:, 4] - x[:, 3]) / 1e3,
                     np.max(x[:, 4] - x[:, 3]) / 1e3])
    print("layer start[min,max] wait_max q_max tiles_end[min,max] end_max tiles_med merge[med,max] (us)")
    for i, r in enumerate(rows[:6] + rows[-2:]):
        print(i, " ".join(f"{v:8.1f}" for v in r))
    ends = np.array([r[6] for r in rows])
    print("layer-to-layer end spacing median %.1f us" % np.median(np.diff(ends)))
    w = t[:, 12:16] - t[:, 2:3]
    print("per-warp tile time us: p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(w, [10, 50, 90, 100]) / 1e3))
    spread = (t[:, 3] - t[:, 12:16].min(1)) / 1e3
    print("warp spread within CTA (last warp - earliest sampled) us: p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(spread, [50, 90, 100])))
    print("in-CTA merge us: p50 %.1f max %.1f" % tuple(np.percentile((t[:, 9] - t[:, 8]) / 1e3, [50, 100])))
    print("arrival us: p50 %.1f max %.1f" % tuple(np.percentile((t[:, 10] - t[:, 9]) / 1e3, [50, 100])))
    last = t[t[:, 11] > 0]
    print("final merges us (CTAs that complete units): p50 %.1f max %.1f" % tuple(np.percentile((last[:, 4] - last[:, 10]) / 1e3, [50, 100])))
    te = np.array([[rel(v) for v in t[t[:, 7] == p, 3]] for p in launches[1:-1]], dtype=object)
    spans = [max(x) - min(x) for x in te]
    print("per layer: last - first CTA tiles_end, median %.1f us" % np.median(spans))
    # release: earliest post-wait time of layer i+1 minus the last exit of layer i; late
    # starters: post-wait minus start of the 10% latest-starting CTAs
    rel_lat, late = [], []
    for i in range(1, len(launches) - 1):
        x, px = t[t[:, 7] == launches[i]], t[t[:, 7] == launches[i - 1]]
        rel_lat.append((x[:, 1].min() - px[:, 4].max()) / 1e3)
        k = max(1, len(x) // 10)
        idx = np.argsort(x[:, 0])[-k:]
        late.append(np.median(x[idx, 1] - x[idx, 0]) / 1e3)
    print("PDL release after the previous layer's last exit, median %.1f us; late starters start->wait %.1f us"
          % (np.median(rel_lat), np.median(late)))
    print("q staging (wait -> staged) per CTA p50 %.1f max %.1f us" % tuple(np.percentile((t[:, 2] - t[:, 1]) / 1e3, [50, 100])))
    # the critical CTA of each layer (latest exit): its phases relative to its own tiles end
    crit = []
    for i in range(1, len(launches) - 1):
        x = t[t[:, 7] == launches[i]]
        r = x[np.argmax(x[:, 4])]
        tmax = x[:, 3].max()
        crit.append([(r[3] - tmax) / 1e3, (r[8] - r[3]) / 1e3, (r[9] - r[8]) / 1e3, (r[10] - r[9]) / 1e3,
                     (r[4] - r[10]) / 1e3, r[11]])
    c = np.median(np.array(crit), axis=0)
    print("critical CTA (median over layers): tiles_end - layer tiles_end max %.1f, -> merge start %.1f, merge %.1f, "
          "publish %.1f, final %.1f us, completes %.0f units" % tuple(c))


if __name__ == "__main__":
    main()
