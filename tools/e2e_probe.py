"""Probe (tuning aid): where the cfg2 e2e step (decode_step_host: pinned host q -> device,
chained graph step, output -> pinned host) loses time against the device-only graph replay.
Variants interleaved (power state drifts, tools/sustained_probe.py), 20 steps each, with an idle
gap before every measurement:
  same graph      one graph replayed
  two graphs      the host API's two staging-buffer graphs alternated, no copies, no events
  events only     alternated graphs + the API's cross-stream event waits, no copies
  host API        decode_step_host (copies on their own streams)"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    m = q.shape[2] // cache.H
    ns = argparse.Namespace(schedule="auto", splits=None, chains=8)
    splits = bench.pick_splits(ns, cache, m)
    qh = q.cpu().pin_memory()
    oh = torch.empty(q.shape, dtype=torch.float16, pin_memory=True)
    cache.decode_step_host(qh, oh, splits=splits, order_current=False, chains=8)
    torch.cuda.synchronize()
    st = cache._host_step
    g0, g1 = st["graphs"][0][0], st["graphs"][1][0]
    side = torch.cuda.Stream(device=dev)
    n = 20

    def same():
        for _ in range(n):
            g0.replay()

    def two():
        for i in range(n):
            (g0 if i % 2 == 0 else g1).replay()

    def events():
        ms = torch.cuda.current_stream()
        for i in range(n):
            ev = torch.cuda.Event()
            ev.record(side)
            ms.wait_event(ev)
            (g0 if i % 2 == 0 else g1).replay()
            e2 = torch.cuda.Event()
            e2.record(ms)
            side.wait_event(e2)

    def host():
        for _ in range(n):
            cache.decode_step_host(qh, oh, splits=splits, order_current=False, chains=8)
        torch.cuda.current_stream().wait_event(cache.host_step_ready)

    res = {k: [] for k in ("same graph", "two graphs", "events only", "host API")}
    fns = dict(zip(res, (same, two, events, host)))
    for _ in range(3):
        for name, fn in fns.items():
            torch.cuda.synchronize()
            time.sleep(1.0)
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) / n)
    for name, v in res.items():
        print(f"{name:12s} ms/step: " + " ".join(f"{x:.4f}" for x in v))


if __name__ == "__main__":
    main()
