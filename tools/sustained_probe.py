"""Sustained decode (tuning aid): the cfg2 default step (8 micro-batch chains, one CUDA graph)
replayed back to back for ~6 s, timed per batch of 50 steps with CUDA events, with nvidia-smi
SM / memory clocks, power and throttle reasons sampled every 100 ms — how the rate moves from
the short bench window (20 steps) to sustained operation under the board's power limit."""
import argparse
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["chains", "lockstep", "single"], default="chains")
    ap.add_argument("--seconds", type=float, default=6.0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cache, q, _ = bench.build_cfg2(torch, dev, 0)
    m = q.shape[2] // cache.H
    chains = 8 if args.mode == "chains" else 1
    ns = argparse.Namespace(schedule="auto", splits=None, chains=chains)
    splits = bench.pick_splits(ns, cache, m)
    out = torch.empty_like(q)
    if args.mode == "single":
        sp = cache.default_splits(m, cache.L)

        class G:
            def replay(self):
                cache.decode(q, out=out, splits=sp)
        g = G()
    else:
        g = cache.decode_graph(q, out, splits=splits, chains=chains)
    print(f"mode {args.mode}")
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    time.sleep(2.0)  # idle first
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            r = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                                "clocks_event_reasons.active", "--format=csv,noheader,nounits"],
                               capture_output=True, text=True)
            samples.append((time.time(), r.stdout.strip()))
            time.sleep(0.1)

    th = threading.Thread(target=sampler)
    th.start()
    t0 = time.time()
    rows = []
    while time.time() - t0 < args.seconds:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        e1.synchronize()
        rows.append((time.time() - t0, e0.elapsed_time(e1) / 50))
    stop.set()
    th.join()
    nbytes = cache.algorithmic_bytes(m)
    print("t_s  ms_per_step  GB/s")
    for t, ms in rows[::4]:
        print(f"{t:5.2f}  {ms:.4f}  {nbytes / ms / 1e6:.0f}")
    print("nvidia-smi samples (t_s: sm MHz, mem MHz, W, C, reasons):")
    for t, s in samples[::3]:
        print(f"{t - t0:5.2f}: {s}")


if __name__ == "__main__":
    main()
