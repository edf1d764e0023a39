"""Benchmark of the Cocktail chunk-level KV-cache hot path on B200 (BASELINE.json metric).

Default (N=1): cfg2 — Llama-3-8B GQA shape (32 q / 8 kv heads, d128), 32 layers, 32K context,
batch 8.  Per-sequence tier maps come from Module I on the device (the reference's
synthetic workload + hashed-BoW embeddings, seeds 0-7, frozen in tests/golden/workloads.npz)
and are asserted equal to the reference's own maps.  K/V/q are synthetic fp16 N(0,1)
(random-init, no checkpoint).  One step = one decode step = mixed-precision attention over
all 32 layers, launched per layer as in a real model (32 launches).  The cache (7.1 GB of
quantized arenas) is larger than L2, so no flush is needed between steps.

Reported: whole-job algorithmic GB/s (SURVEY §8d bytes), tokens/s, roofline of the decode
kernel against MEASURED_PEAKS.json, an end-to-end figure through the public API with host
buffers, the CPU baseline (oracle restatement of the reference, timed on host cores), and a
prefill sub-object (cfg5-shaped search + reorder/quantize/pack, 128K x 32 layers x 8 kv heads).

N>1 (`--gpus N`: re-launches itself under torch.distributed.run when WORLD_SIZE is unset, one
rank per GPU): every rank owns its own batch of 8 sequences (batch-sharded, weak scaling, no
data-path collective); time is the max over ranks.  The N>1 line adds a `split_kv` object: cfg3
(128K, 40 layers x 40 heads) strong-scaled over the same ranks with sequence split-KV (per-layer
decode_partial launches, one NCCL all_gather of the (acc, m, l) partials, ckv_lse_merge; with
the local / exchange+merge split of the step time and the latency of one layer's exchange +
merge) and `head_shard`, the KV-head partition of the same cache (no collective).

--impl reference: the reference's CPU algorithm (oracle port of attention.py:63-90 over
quantizer.fqm / _numpy.py) on all host cores, same metric, bounded sample per step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "mixed-precision KV decode-attn GB/s (% HBM peak) and tokens/s at 1/2/4/8 B200"
WORKLOADS = os.path.join(ROOT, "tests", "golden", "workloads.npz")
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")

CFG2 = dict(layers=32, batch=8, kv_heads=8, q_per_kv=4, context=32768, head_dim=128)
CFG5 = dict(layers=32, batch=1, kv_heads=8, context=131072, head_dim=128)
CFG3 = dict(layers=40, batch=1, kv_heads=40, q_per_kv=1, context=131072, head_dim=128)
CFG4 = dict(layers=32, batch=64, kv_heads=8, q_per_kv=4, context=16384, head_dim=128)
CFG1 = dict(layers=1, batch=1, kv_heads=32, q_per_kv=1, context=4096, head_dim=128)


def load_workload(ctx, seed):
    with np.load(WORKLOADS) as z:
        idx = z[f"{ctx}_{seed}_idx"]
        val = z[f"{ctx}_{seed}_val"]
        n = idx.shape[0]
        emb = np.zeros((n, 256))
        rows = np.repeat(np.arange(n), idx.shape[1])
        nz = val.reshape(-1) != 0
        emb[rows[nz], idx.reshape(-1)[nz].astype(np.int64)] = val.reshape(-1)[nz]
        return dict(emb=emb, norm=z[f"{ctx}_{seed}_norm"], q=z[f"{ctx}_{seed}_q"],
                    qnorm=float(z[f"{ctx}_{seed}_qnorm"]), tiers=z[f"{ctx}_{seed}_tiers"])


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML) during the timed region: NVML is opened
    before the region starts, one sample is taken on entry, then every 5 ms, then on exit."""

    BITS = {"hw_slowdown": "nvmlClocksThrottleReasonHwSlowdown",
            "hw_thermal_slowdown": "nvmlClocksThrottleReasonHwThermalSlowdown",
            "sw_thermal_slowdown": "nvmlClocksThrottleReasonSwThermalSlowdown",
            "sw_power_cap": "nvmlClocksThrottleReasonSwPowerCap"}
    DEFAULT_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.error = None
        self._stop = threading.Event()
        self._t = None
        self._nv = self._hdl = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._hdl = nv.nvmlDeviceGetHandleByIndex(index)
            self._max = nv.nvmlDeviceGetMaxClockInfo(self._hdl, nv.NVML_CLOCK_SM)
            self._bits = {k: getattr(nv, a, self.DEFAULT_BITS[k]) for k, a in self.BITS.items()}
        except Exception as exc:  # no NVML: record why
            self.error = f"unsampled: {type(exc).__name__}"

    def _sample(self):
        nv = self._nv
        try:
            sm = nv.nvmlDeviceGetClockInfo(self._hdl, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._hdl)
            self.samples.append((sm, self._max, [k for k, b in self._bits.items() if r & b]))
        except Exception as exc:
            self.error = f"unsampled: {type(exc).__name__}"

    def _run(self):
        while not self._stop.wait(0.005):
            self._sample()

    def __enter__(self):
        if self._nv is not None:
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._t is not None:
            self._stop.set()
            self._t.join(timeout=10)
            self._sample()

    def summary(self):
        sm = [s[0] for s in self.samples if s[0] is not None]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.error or "unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples if s[1]),
                "reasons": sorted({r for s in self.samples for r in s[2]}), "samples": len(sm)}


def measured_peak_gbs(sustained=True):
    """HBM roofline denominator: MEASURED_PEAKS.json (driver-written) when present — its
    sustained copy figure for kernels timed inside a long step, the burst one otherwise —
    else the profiling guide's 6650 GB/s fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            data = json.load(fh)
        flat = {}

        def walk(d, pre=""):
            for k, v in d.items():
                if isinstance(v, dict):
                    walk(v, f"{pre}{k}.")
                elif isinstance(v, (int, float)) and not isinstance(v, bool):
                    flat[f"{pre}{k}"] = float(v)
        walk(data)
        hbm = {k: v for k, v in flat.items() if "hbm" in k.lower() and v > 0}
        if hbm:
            want = "sustain" if sustained else "burst"
            for k in sorted(hbm):
                if want in k.lower():
                    return hbm[k], f"measured ({k})"
            key = "hbm_gbs" if "hbm_gbs" in hbm else sorted(hbm)[0]
            return hbm[key], f"measured ({key})"
    return 6650.0, "fallback"


def profile_traffic(key):
    if os.path.exists(PROFILE_TRAFFIC):
        with open(PROFILE_TRAFFIC) as fh:
            return json.load(fh).get(key)
    return None


# ---------------------------------------------------------------------------------------
# CPU legs (oracle restatement of the reference; test infrastructure used as the baseline)

_CPU_UNITS = []  # prebuilt oracle caches of the CPU legs (inherited by forked pool workers)


def _cpu_decode(i):
    """Decode-only time of prebuilt unit i (the reference's mixed_decode_attention algorithm)."""
    from oracle import ckv_oracle as O
    q, cache = _CPU_UNITS[i]
    t0 = time.perf_counter()
    O.mixed_decode_attention(q, cache)
    t1 = time.perf_counter()
    nbytes = cache.len_2 * 96 + cache.len_4 * 160 + cache.len_fp * 512 + 2 * q.size * 2
    return t1 - t0, nbytes


def _cpu_build_units(n_units, ctx, m, rng):
    from oracle import ckv_oracle as O
    units = []
    for u in range(n_units):
        wl = load_workload(32768, u % 8) if ctx == 32768 else None
        tiers = wl["tiers"] if wl is not None else rng.choice([0, 1, 2], size=ctx // 32).astype(np.uint8)
        k = rng.standard_normal((ctx, 128)).astype(np.float16).astype(np.float64)
        v = rng.standard_normal((ctx, 128)).astype(np.float16).astype(np.float64)
        q = rng.standard_normal((m, 128)).astype(np.float16).astype(np.float64)
        units.append((q, O.build_cache(k, v, tiers, 32, 32)))
    return units


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_kernels():
    """Select the CPU leg's kernels: the reference's own compiled module (oracle/_ref, built by
    oracle/Makefile from /root/reference's _core.pyx) when present — kind "reference" — else
    the oracle's numpy restatement of the reference (kind "port")."""
    from oracle import ckv_oracle as O, ref_core
    mod = ref_core.load()
    O.use_reference_kernels(mod)
    return ("reference", "chunkkv.kernels._core (compiled reference, -O3 -ffp-contract=off) under the oracle's "
            "restatement of attention.py") if mod is not None else ("port", "oracle numpy restatement")


def cpu_baseline(seconds=12.0, processes=1, n_units=None):
    """Time the reference algorithm of mixed_decode_attention over cfg2 units (32K, m = 4):
    units prebuilt (build_cache is outside the timing), then decoded repeatedly — one process,
    or a fork pool of `processes` workers timed by the pool's wall clock — until `seconds`."""
    global _CPU_UNITS
    kind, kernels = cpu_kernels()
    n_units = n_units or max(2, processes)
    if len(_CPU_UNITS) < n_units:  # built once per process, reused by later calls
        _CPU_UNITS = _cpu_build_units(n_units, CFG2["context"], CFG2["q_per_kv"], np.random.default_rng(0))
    pool = None
    if processes > 1:
        import multiprocessing as mpx
        pool = mpx.get_context("fork").Pool(processes)
        pool.map(_cpu_decode, range(n_units))  # warm the workers
    done_bytes, wall, n_done = 0, 0.0, 0
    while wall < seconds:
        t0 = time.perf_counter()
        res = pool.map(_cpu_decode, range(n_units), chunksize=1) if pool else [_cpu_decode(i) for i in range(n_units)]
        wall += time.perf_counter() - t0
        done_bytes += sum(r[1] for r in res)
        n_done += len(res)
    if pool:
        pool.close()
        pool.join()
    return done_bytes / wall / 1e9, n_done, wall, kind, kernels


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's CPU implementation on all host cores; rank 0 only."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    steps_gbs = []
    kind = kernels = None
    for _ in range(args.warmup):
        cpu_baseline(seconds=0.5, processes=cores)
    for _ in range(args.steps):
        gbs, n, wall, kind, kernels = cpu_baseline(seconds=max(2.0, 20.0 / max(args.steps, 1)), processes=cores)
        steps_gbs.append(gbs)
    value = statistics.median(steps_gbs)
    sample = (f"{cores}-process fork pool over {cores} prebuilt cfg2 units (32K ctx, m=4, reference tier maps), "
              f"decode timed by the pool's wall clock, >= 2 s per step; kernels: {kernels}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: Llama-3-8B GQA 32q/8kv d128, 32 layers, 32K ctx, batch 8",
                   "sampled_units": True,
                   "same_config_note": "per-byte rate over sampled cfg2 units (BASELINE.md section 3 plan); "
                                       "the full step would take minutes on the CPU"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def pick_splits(args, cache, m, layers=1):
    """Decode schedule for a bench run: the warp plan (splits None) unless --schedule split or
    --splits is given, or the cache has no warp plan."""
    cache.schedule = args.schedule
    chains = getattr(args, "chains", 1)
    if chains > 1:  # micro-batch chains run the split kernel over (sequence, head) ranges
        if args.schedule == "wp" and chains <= cache.B and args.splits is None:
            return None
        return args.splits or cache.chain_splits(m)
    if args.schedule != "split" and args.splits is None and cache._use_wp(m, None, None, None) is not None:
        return None
    return args.splits or cache.default_splits(m, layers)


def auto_chains(batch):
    """Micro-batch chains of a decode step: up to 8 sequence ranges (one per sequence for the
    cfg2 batch of 8), each its own chain of per-layer launches on its own stream."""
    return max(1, min(int(batch), 8))


def launch_desc(chains):
    if chains == 1:
        return "per-layer (32 PDL-chained launches per step, replayed as one CUDA graph)"
    return (f"per-layer: {chains} micro-batch chains (sequence ranges) on their own streams, each 32 "
            f"PDL-chained per-layer launches (layer l+1 of a chain waits for its layer l); one CUDA graph per step")


def schedule_desc(cache, splits, chains=1):
    if splits is None:
        p = cache.warp_plan()
        nw = cache.wp_unit_warps
        desc = f"warp plan: {len(nw)} units x {int(nw.min())}-{int(nw.max())} warps, {p[1]} CTAs"
        if chains > 1:
            desc += f"; {chains} micro-batch chains, each its own warp plan per launch"
        return desc
    desc = f"split: {splits} CTAs of 4 warps per unit"
    if chains > 1:
        u = cache._chain_units(chains)
        b0, b1, h0, h1 = u[0]
        desc += (f"; {len(u)} micro-batch chains of {b1 - b0} sequence(s) x {h1 - h0} kv head(s), launches of "
                 f"{(b1 - b0) * (h1 - h0) * splits} CTAs")
    return desc


def build_cfg2(torch, dev, rank):
    from paper_2503_23294_b200 import batched, retrieval

    c = CFG2
    L, B, H, m, T, D = c["layers"], c["batch"], c["kv_heads"], c["q_per_kv"], c["context"], c["head_dim"]
    wls = [load_workload(T, (rank * B + b) % 8) for b in range(B)]
    emb = np.stack([w["emb"] for w in wls])
    norm = np.stack([w["norm"] for w in wls])
    qv = np.stack([w["q"] for w in wls])
    qn = np.array([w["qnorm"] for w in wls])
    search = retrieval.search_batched(emb, norm, qv, qn, 0.6, 0.1)
    tiers = search.tiers.cpu().numpy()
    ref_tiers = np.stack([w["tiers"] for w in wls])
    if not np.array_equal(tiers, ref_tiers):
        raise SystemExit("tier maps differ from the reference's (Module I parity failure)")
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    k = torch.randn((L, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    v = torch.randn((L, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    cache = batched.build_cache_batched(k, v, search, decode_capacity=128)
    # a few units' fp16 K/V kept on the host for the parity check of the timed cache
    samples = [(l, b, h, k[l, b, :, h].cpu().numpy(), v[l, b, :, h].cpu().numpy(), ref_tiers[b])
               for (l, b, h) in ((0, 0, 0), (L // 2, B - 1, H // 2), (L - 1, B // 2, H - 1))]
    del k, v
    q = torch.randn((L, B, H * m, D), generator=g, device=dev, dtype=torch.float16)
    cache.parity_samples = samples
    return cache, q, search


def sampled_parity(cache, q, out, m):
    """max relative error (|got - ref| / max|ref|) of sampled units of the timed cache's output
    against the reference algorithm (oracle) in f64 on the same fp16 inputs; outside the timed
    region."""
    from oracle import ckv_oracle as O
    qh, oh = q.cpu().numpy(), out.float().cpu().numpy()
    worst = 0.0
    for l, b, h, kh, vh, tiers in cache.parity_samples:
        oc = O.build_cache(kh.astype(np.float64), vh.astype(np.float64), tiers, 32, 32)
        ref = O.mixed_decode_attention(qh[l, b, h * m:(h + 1) * m].astype(np.float64), oc)
        got = oh[l, b, h * m:(h + 1) * m].astype(np.float64)
        worst = max(worst, float(np.max(np.abs(got - ref)) / np.max(np.abs(ref))))
    return worst


def bench_prefill(torch, dev, steps=3, profile=False):
    """cfg5-shaped prefill: search + reorder/quantize/pack of a 128K x 32-layer x 8-head cache."""
    from paper_2503_23294_b200 import batched, retrieval

    c = CFG5
    L, B, H, T, D = c["layers"], c["batch"], c["kv_heads"], c["context"], c["head_dim"]
    wl = load_workload(T, 0)
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    k = torch.randn((L, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    v = torch.randn((L, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    s = retrieval.search_batched(wl["emb"][None], wl["norm"][None], wl["q"][None], np.array([wl["qnorm"]]))
    if not np.array_equal(s.tiers.cpu().numpy()[0], wl["tiers"]):
        raise SystemExit("128K tier map differs from the reference's")
    counts = s.seg_counts.cpu().numpy()
    cache = batched.BatchedKVCache(L, B, H, counts[:, 0], counts[:, 1], counts[:, 2], [T], 0, device=dev)
    flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)  # read-based L2 flush (clean lines)
    times_build, times_search = [], []
    clk = ClockSampler(dev.index or 0)
    clk.__enter__()
    for i in range(steps + 2):
        flush.max()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        if profile and i == steps + 1:
            torch.cuda.profiler.start()
        e0.record()
        s2 = retrieval.search_batched(wl["emb"][None], wl["norm"][None], wl["q"][None],
                                      np.array([wl["qnorm"]]), check=False)
        e1.record()
        cache.build(k, v, s2.perm, check=False)
        e2.record()
        torch.cuda.synchronize()
        if profile and i == steps + 1:
            torch.cuda.profiler.stop()
        if i >= 2:
            times_search.append(e0.elapsed_time(e1))
            times_build.append(e1.elapsed_time(e2))
    clk.__exit__(None, None, None)
    tb = statistics.median(times_build) * 1e-3
    n2, n4, nf = (int(x) for x in counts[0])
    read = 2 * L * H * T * D * 2
    write = 2 * L * H * (n2 * 32 * 48 + n4 * 32 * 80 + (nf * 32 + (T - 32 * (n2 + n4 + nf))) * 256)
    peak, peak_kind = measured_peak_gbs(sustained=False)  # one kernel timed alone: burst figure
    ach = (read + write) / tb / 1e9
    del k, v, cache
    torch.cuda.empty_cache()
    text = bench_text_search(torch, T // 32)
    return {
        "workload": "cfg5: prefill search + reorder/quantize/pack, 128K ctx x 32 layers x 8 kv heads, b1",
        "tier_fractions": [round(x / (n2 + n4 + nf), 4) for x in (n2, n4, nf)],
        "quantize_ms": round(tb * 1e3, 3),
        "search_ms": round(statistics.median(times_search), 3),
        "search_note": "search_ms is the public search_batched call from host f64 embeddings "
                       "(includes their 8 MB host-to-device copy)",
        "bytes_read": read, "bytes_written": write,
        "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(ach / peak, 4), "peak_kind": peak_kind,
                     "traffic": profile_traffic("reorder_quantize_pack")},
        "clocks": clk.summary(),
        "text_search": text,
    }


def bench_text_search(torch, n_chunks, reps=5):
    """Texts -> tiers for one 128K context (n_chunks chunk texts of 32 synthetic words + a
    64-word query): the public search_texts call (UTF-8 packing, host-to-device copy, GPU
    hashed-BoW encode, search), wall clock with a device sync, beside the CPU restatement of
    the reference's per-text encoder on a sample of the same texts (extrapolated)."""
    from paper_2503_23294_b200 import retrieval

    rng = np.random.default_rng(5)
    words = rng.integers(0, 4096, size=(n_chunks, 32))
    chunks = [" ".join(f"w{int(x):05d}" for x in row) for row in words]
    query = " ".join(f"w{int(x):05d}" for x in rng.integers(0, 1024, size=64))
    enc = retrieval.HashedBowEncoder(seed=0)
    times = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = retrieval.search_texts([chunks], [query], 0.6, 0.1, enc, check=False)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    gpu_ms = statistics.median(times[1:]) * 1e3
    from oracle import ckv_oracle as O  # CPU baseline leg only

    sample = chunks[:512]
    t0 = time.perf_counter()
    for t in sample:
        O.bow_encode(t, 256, 0)
    cpu_ms = (time.perf_counter() - t0) * 1e3 * (n_chunks + 1) / len(sample)
    del r
    return {"chunks": n_chunks, "gpu_ms": round(gpu_ms, 3), "cpu_encode_ms": round(cpu_ms, 1),
            "note": "gpu_ms: search_texts from host strings to device tiers (encode + search); "
                    "cpu_encode_ms: the oracle port of HashedBowEncoder.encode (hashlib, 1 core) on "
                    "512 of the texts, scaled to all of them (encoding only)"}


def measure_cfg3(args, torch, dist, dev, rank, world, split="seq", steps=None, warmup=None):
    """cfg3: Llama-2-13B shape (40 layers x 40 MHA heads, d128), 128K context, batch 1, strong
    scaling of the fixed cache over the ranks (max-over-ranks device time).

    split="seq": sequence split-KV — every rank owns a chunk-aligned 1/N slice of each tier
    segment; a step is 40 per-layer decode_partial launches (PDL-chained, one CUDA graph), one
    all_gather of all layers' (acc, m, l) partials (NCCL over NVLink/NVSwitch) and the LSE merge.
    split="head": KV-head partition — every rank owns 40/N whole heads (all tokens); a step is
    40 per-layer decode launches; no collective.  Returns a dict of measurements (rank 0)."""
    from paper_2503_23294_b200 import batched, distributed, retrieval

    steps = args.steps if steps is None else steps
    warmup = max(args.warmup if warmup is None else warmup, 3)
    c = CFG3
    L, B, H, m, T, D = c["layers"], c["batch"], c["kv_heads"], c["q_per_kv"], c["context"], c["head_dim"]
    wl = load_workload(T, 0)
    search = retrieval.search_batched(wl["emb"][None], wl["norm"][None], wl["q"][None],
                                      np.array([wl["qnorm"]]), 0.6, 0.1)
    if not np.array_equal(search.tiers.cpu().numpy()[0], wl["tiers"]):
        raise SystemExit("128K tier map differs from the reference's")
    counts = search.seg_counts.cpu().numpy()
    h0, h1 = distributed.head_shard(H, world, rank) if split == "head" else (0, H)
    if split == "seq":
        cache, perm_r = distributed.sequence_shard_cache(search, L, H, [T], world, rank, decode_capacity=128,
                                                         device=dev)
    else:
        cache = batched.BatchedKVCache(L, B, h1 - h0, counts[:, 0], counts[:, 1], counts[:, 2], [T], 128,
                                       device=dev)
        perm_r = search.perm
    g = torch.Generator(device=dev)
    for l in range(L):  # the full context's K/V, one layer at a time (same data on every rank)
        g.manual_seed(4321 + l)
        k = torch.randn((1, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
        v = torch.randn((1, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
        cache.build(k[:, :, :, h0:h1], v[:, :, :, h0:h1], perm_r, layer=l)
        del k, v
    torch.cuda.empty_cache()
    g.manual_seed(99)
    q_all = torch.randn((L, B, H * m, D), generator=g, device=dev, dtype=torch.float16)
    q = q_all[:, :, h0 * m:h1 * m].contiguous()
    Hq = (h1 - h0) * m
    chains = args.chains if args.chains > 0 else 8  # micro-batch chains over the kv heads (batch 1)
    cargs = argparse.Namespace(**{**vars(args), "chains": chains})
    splits = pick_splits(cargs, cache, m)
    units = cache._chain_units(chains)
    chain_streams = [torch.cuda.Stream(device=dev) for _ in units]

    def partial_layers(qq, buf):
        """The step's per-layer decode_partial launches into buf: one PDL chain per kv-head range,
        each on its own stream (forked from / joined into the current stream)."""
        if len(units) == 1:
            for l in range(L):
                cache.decode_partial(qq[l:l + 1], splits=splits, layer=l, pdl=l > 0,
                                     out=buf[l * B * Hq:(l + 1) * B * Hq])
            return
        cur = torch.cuda.current_stream()
        for st in chain_streams:
            st.wait_stream(cur)
        for (_, _, ha, hb), st in zip(units, chain_streams):
            with torch.cuda.stream(st):
                for l in range(L):
                    cache.decode_partial(qq[l:l + 1], splits=splits, layer=l, pdl=l > 0,
                                         out=buf[l * B * Hq:(l + 1) * B * Hq], heads=(ha, hb))
        for st in chain_streams:
            cur.wait_stream(st)

    def barrier():
        if world > 1:
            dist.barrier()

    def sync_max(ms):
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def timed(fn, n):
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        return sync_max(e0.elapsed_time(e1) / n)

    res = {}
    if split == "seq":
        parts = torch.empty((L * B * Hq, D + 2), dtype=torch.float32, device=dev)

        def local_decode(qq):
            partial_layers(qq, parts)

        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            local_decode(q)
        torch.cuda.current_stream().wait_stream(side)
        local_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(local_graph, stream=side):  # the warm-up's stream: same workspaces
            local_decode(q)

        def step():
            local_graph.replay()
            gathered = distributed.exchange_partials(parts) if world > 1 else parts[None]
            return batched.lse_merge(gathered)

        layer_rows = parts[:B * Hq]

        def layer_merge():  # one layer's exchange + merge (the per-layer latency of SURVEY §7.8)
            gathered = distributed.exchange_partials(layer_rows) if world > 1 else layer_rows[None]
            return batched.lse_merge(gathered)

        for _ in range(warmup):
            step()
            layer_merge()
        # one layer's exchange + merge, 20 times in a CUDA graph (NCCL collectives capture), so
        # the figure is device latency, not Python launch overhead; eager when capture fails
        merge_fn, merge_reps = layer_merge, 1
        try:
            if world > 1 and dist.get_backend() != "nccl":
                raise RuntimeError("host-staged exchange (gloo): not capturable")
            side2 = torch.cuda.Stream(device=dev)
            side2.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side2):
                layer_merge()
            torch.cuda.current_stream().wait_stream(side2)
            mg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(mg):
                for _ in range(20):
                    layer_merge()
            mg.replay()
            merge_fn, merge_reps = mg.replay, 20
        except Exception:  # noqa: BLE001 (gloo test mode: no capture)
            torch.cuda.synchronize()
        with ClockSampler(dev.index or 0) as clk:
            ms = timed(step, steps)
        # the step's two parts measured inside the same kind of step (events between them, not a
        # difference of two separately timed loops): local decode | exchange + merge
        torch.cuda.synchronize()
        barrier()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        for e in ev:
            e[0].record()
            local_graph.replay()
            e[1].record()
            gathered = distributed.exchange_partials(parts) if world > 1 else parts[None]
            batched.lse_merge(gathered)
            e[2].record()
        torch.cuda.synchronize()
        barrier()
        res["local_decode_ms"] = round(sync_max(sum(e[0].elapsed_time(e[1]) for e in ev) / steps), 4)
        res["exchange_merge_ms"] = round(sync_max(sum(e[1].elapsed_time(e[2]) for e in ev) / steps), 4)
        res["per_layer_merge_us"] = round(1e3 * timed(merge_fn, max(steps, 20)) / merge_reps, 2)
        res["per_layer_merge_note"] = ("one layer's all_gather + ckv_lse_merge, " +
                                       ("CUDA-graph replayed" if merge_reps > 1 else "eager launches"))
        res["p2p"] = measure_p2p_exchange(torch, distributed, partial_layers, q, L, B, Hq, dev, steps, warmup,
                                          timed, barrier, sync_max)
        out_rows = L * B * Hq
        e2e_out = step
    else:
        out = torch.empty_like(q)
        graph = cache.decode_graph(q, out, splits=splits, chains=chains)
        for _ in range(warmup):
            graph.replay()
        with ClockSampler(dev.index or 0) as clk:
            ms = timed(graph.replay, steps)
        out_rows = L * B * Hq

        def e2e_out():
            graph.replay()
            return out

    my_bytes = cache.algorithmic_bytes(m)
    tot = torch.tensor([float(my_bytes)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tot)
    step_bytes = float(tot.item())

    # end to end: pinned host q -> device (this rank's q heads), step, output -> pinned host
    qh = q.cpu().pin_memory()
    oh = torch.empty((out_rows, D), dtype=torch.float16, pin_memory=True)

    if split == "head":
        # the public host-buffer API: uploads / downloads on their own copy streams overlapping
        # the chained per-layer launches (as the cfg2 line's e2e)
        oh = torch.empty(q.shape, dtype=torch.float16, pin_memory=True)

        def e2e_step():
            cache.decode_step_host(qh, oh, splits=splits, order_current=False, chains=chains)

        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e4.record()
        for _ in range(steps):
            e2e_step()
        torch.cuda.current_stream().wait_event(cache.host_step_ready)  # the last download is timed
        e5.record()
        torch.cuda.synchronize()
        barrier()
        e2e_ms = sync_max(e4.elapsed_time(e5) / steps)
    else:
        def e2e_step():
            q.copy_(qh, non_blocking=True)
            oh.copy_(e2e_out().reshape(out_rows, D), non_blocking=True)

        for _ in range(3):
            e2e_step()
        e2e_ms = timed(e2e_step, steps)
    # lockstep figure: every layer ONE launch over all of the rank's kv heads, so layer l+1
    # starts only after all of layer l (the dependency a batch-1 model step has: every head of
    # layer l+1 reads the whole layer-l output); the kv-head chains above relax it to "after
    # layer l of the same head range"
    if chains > 1:
        ls_args = argparse.Namespace(**{**vars(args), "chains": 1})
        ls_splits = pick_splits(ls_args, cache, m)  # the warp plan unless --splits / --schedule split
        if split == "seq":
            def ls_local(qq):
                for l in range(L):
                    cache.decode_partial(qq[l:l + 1], splits=ls_splits, layer=l, pdl=l > 0,
                                         out=parts[l * B * Hq:(l + 1) * B * Hq])

            side3 = torch.cuda.Stream(device=dev)
            side3.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side3):
                ls_local(q)
            torch.cuda.current_stream().wait_stream(side3)
            ls_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ls_graph, stream=side3):
                ls_local(q)

            def ls_step():
                ls_graph.replay()
                gathered = distributed.exchange_partials(parts) if world > 1 else parts[None]
                return batched.lse_merge(gathered)
        else:
            ls_out = torch.empty_like(q)
            ls_graph = cache.decode_graph(q, ls_out, splits=ls_splits)
            ls_step = ls_graph.replay
        for _ in range(warmup):
            ls_step()
        ls_ms = timed(ls_step, steps)
        res["lockstep_per_layer"] = {
            "value": round(step_bytes / (ls_ms * 1e-3) / 1e9, 2), "ms_per_step": round(ls_ms, 4),
            "launch": f"per-layer: {L} PDL-chained launches over all kv heads, one CUDA graph"
                      + (" + all_gather + merge" if split == "seq" else ""),
            "schedule": schedule_desc(cache, ls_splits)}
        del ls_graph
        cache.schedule = args.schedule
    counts0 = counts[0]
    res.update({
        "value": round(step_bytes / (ms * 1e-3) / 1e9, 2), "ms_per_step": round(ms, 4),
        "tokens_per_s": round(B / (ms * 1e-3), 1), "algorithmic_bytes_per_step": int(step_bytes),
        "splits": splits, "split": split, "schedule": schedule_desc(cache, splits, chains),
        "parallelism": f"{'seq-split' if split == 'seq' else 'head-shard'} x{world}",
        "per_rank_gbs": round(my_bytes / (ms * 1e-3) / 1e9, 1),
        "e2e": {"value": round(step_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": int(q.numel() * 2 * world), "d2h_bytes_per_step": int(oh.numel() * 2 * world)},
        "tier_fractions_int2_int4_fp16": [round(float(x) / counts0.sum(), 4) for x in counts0],
        "clocks": clk.summary(),
        "gpu_launches": steps * (L + (1 if split == "seq" else 0)),
    })
    del cache
    torch.cuda.empty_cache()
    return res


def measure_p2p_exchange(torch, distributed, partial_layers, q, L, B, Hq, dev, steps, warmup, timed, barrier,
                         sync_max):
    """cfg3 split-KV with the exchange over peer memory (distributed.P2PExchange: every rank's
    partials in a symmetric-memory buffer, one device barrier, ckv_lse_merge_ptrs reading all
    ranks' buffers over NVLink) instead of all_gather + merge: the step time, its local / barrier
    + merge parts (events inside the step) and one layer's barrier + merge latency.  Returns
    {"unavailable": why} when symmetric memory cannot be set up on these ranks.  A single-GPU
    run sets up a world-1 group for it (the path then measures its barrier + merge cost alone)."""
    import torch.distributed as tdist

    own_group = False
    try:
        if not tdist.is_initialized():
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            sk.close()
            tdist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
            own_group = True
        ex = distributed.P2PExchange(L * B * Hq, device=dev)
        graphs = []
        for i in range(2):  # one CUDA graph of the 40 local launches per buffer slot
            buf = ex.buffer(i)

            def local(qq, buf=buf):
                partial_layers(qq, buf)

            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                local(q)
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                local(q)
            graphs.append(g)

        def step():
            graphs[ex.i].replay()
            return ex.merge()

        for _ in range(warmup):
            step()
        ms = timed(step, steps)
        torch.cuda.synchronize()
        barrier()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        for e in ev:
            e[0].record()
            graphs[ex.i].replay()
            e[1].record()
            ex.merge()
            e[2].record()
        torch.cuda.synchronize()
        barrier()
        local_ms = sync_max(sum(e[0].elapsed_time(e[1]) for e in ev) / steps)
        xm_ms = sync_max(sum(e[1].elapsed_time(e[2]) for e in ev) / steps)
        ex1 = distributed.P2PExchange(B * Hq, device=dev)  # one layer's rows
        out1 = torch.empty((B * Hq, 128), dtype=torch.float16, device=dev)
        for _ in range(3):
            ex1.merge(out1)
        reps, fn = 1, (lambda: ex1.merge(out1))
        try:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for i in range(2):
                    ex1.merge(out1, i=i)
            torch.cuda.current_stream().wait_stream(side)
            mg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(mg):
                for r in range(20):
                    ex1.merge(out1, i=r % 2)
            mg.replay()
            reps, fn = 20, mg.replay
        except Exception:  # noqa: BLE001 (barrier not capturable here: eager launches)
            torch.cuda.synchronize()
        layer_us = 1e3 * timed(fn, max(steps, 20)) / reps
        return {"ms_per_step": round(ms, 4), "local_decode_ms": round(local_ms, 4),
                "exchange_merge_ms": round(xm_ms, 4), "per_layer_merge_us": round(layer_us, 2),
                "note": "partials in symmetric memory (torch.distributed._symmetric_memory), device barrier, "
                        "ckv_lse_merge_ptrs reading every rank's buffer over the peer mappings; per-layer: "
                        + ("CUDA-graph replayed" if reps > 1 else "eager launches")}
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    finally:
        if own_group:
            tdist.destroy_process_group()


def run_cfg3(args, torch, dist, dev, rank, world, local):
    """cfg3 line: --cfg3-split seq (sequence split-KV, default) or head (KV-head partition)."""
    r = measure_cfg3(args, torch, dist, dev, rank, world, split=args.cfg3_split)
    if rank == 0:
        peak, peak_kind = measured_peak_gbs()
        line = {
            "metric": METRIC, "value": r["value"], "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic (fp16 N(0,1) K/V/q; reference search tier map, 128K seed 0)",
            "config": {"workload": "cfg3: Llama-2-13B 40 layers x 40 MHA heads d128, 128K ctx, batch 1, "
                                   + ("sequence split-KV across the GPUs" if r["split"] == "seq"
                                      else "KV heads partitioned across the GPUs"),
                       "global_batch": CFG3["batch"], "seq_len": CFG3["context"], "parallelism": r["parallelism"],
                       "tier_fractions_int2_int4_fp16": r["tier_fractions_int2_int4_fp16"],
                       "launch": ("per-layer decode_partial (40 PDL-chained launches per kv-head chain, 8 chains on "
                                  "their own streams, one CUDA graph) + all_gather + merge" if r["split"] == "seq" else
                                  "per-layer decode (40 PDL-chained launches per kv-head chain, one CUDA graph), "
                                  "no collective")
                                 + "; a head range's layer l+1 waits for its own layer l only (a model step's "
                                   "layer l+1 needs all heads of layer l: lockstep_per_layer keeps that)",
                       "splits": r["splits"], "schedule": r["schedule"],
                       "l2": "inputs larger than L2 (21 GB of arenas over the ranks)"},
            "tokens_per_s": r["tokens_per_s"],
            "algorithmic_bytes_per_step": r["algorithmic_bytes_per_step"],
            "roofline": {"bound": "hbm", "achieved": r["per_rank_gbs"], "peak": peak, "unit": "GB/s",
                         "frac": round(r["per_rank_gbs"] / peak, 4), "peak_kind": peak_kind, "traffic": None},
            "e2e": r["e2e"], "gpu_launches": r["gpu_launches"], "clocks": r["clocks"],
        }
        for key in ("lockstep_per_layer", "local_decode_ms", "exchange_merge_ms", "per_layer_merge_us",
                    "per_layer_merge_note", "p2p"):
            if key in r:
                line[key] = r[key]
        if "ms_per_step" in (r.get("p2p") or {}):
            line["p2p"]["value"] = round(r["algorithmic_bytes_per_step"] / (r["p2p"]["ms_per_step"] * 1e-3) / 1e9, 2)
        print(json.dumps(line), flush=True)


def run_cfg4(args, torch, dist, dev, rank, world, local):
    """cfg4: batch 64 x 16K, Llama-3-8B GQA shape (32 layers, 8 kv heads, m = 4), the global
    batch sharded over the ranks (64/N whole sequences per GPU, no data-path collective; strong
    scaling of the fixed batch).  Tier maps (--cfg4-map): the reference's 16K maps (sequence
    b: seed b % 8, "skewed"), all-INT2 or all-FP16 — SURVEY's bitwidth-mix sweep.  The cache is
    built one layer at a time (the fp16 source of one layer is 4.3 GB)."""
    from paper_2503_23294_b200 import batched, distributed, retrieval

    c = CFG4
    L, Bg, H, m, T, D = c["layers"], c["batch"], c["kv_heads"], c["q_per_kv"], c["context"], c["head_dim"]
    lo, hi = distributed.batch_shard(Bg, world, rank)
    B = hi - lo
    n = T // 32
    if args.cfg4_map == "skewed":
        maps = np.stack([load_workload(T, b % 8)["tiers"] for b in range(lo, hi)])
    else:
        maps = np.full((B, n), 2 if args.cfg4_map == "all_fp16" else 0, np.uint8)
    search = retrieval.assign_tiers_batched(maps.astype(np.float64), np.tile([[0.5, 1.5]], (B, 1)))
    if not np.array_equal(search.tiers.cpu().numpy(), maps):
        raise SystemExit("cfg4 tier maps not reproduced")
    counts = search.seg_counts.cpu().numpy()
    cache = batched.BatchedKVCache(L, B, H, counts[:, 0], counts[:, 1], counts[:, 2], [T] * B, 128, device=dev)
    g = torch.Generator(device=dev)
    for l in range(L):
        g.manual_seed(7000 + 100 * rank + l)
        k = torch.randn((1, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
        v = torch.randn((1, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
        cache.build(k, v, search.perm, layer=l)
        del k, v
    torch.cuda.empty_cache()
    g.manual_seed(11 + rank)
    q = torch.randn((L, B, H * m, D), generator=g, device=dev, dtype=torch.float16)
    out = torch.empty_like(q)
    if args.chains == 0:
        args.chains = auto_chains(B)
    splits = pick_splits(args, cache, m)
    my_bytes = cache.algorithmic_bytes(m)

    graph = cache.decode_graph(q, out, splits=splits, chains=args.chains)  # the step's per-layer PDL-chained launches
    step = graph.replay

    def sync_max(ms):
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
    ms = sync_max(e0.elapsed_time(e1) / args.steps)
    qh = q.cpu().pin_memory()
    oh = torch.empty(q.shape, dtype=torch.float16, pin_memory=True)
    for _ in range(3):
        cache.decode_step_host(qh, oh, splits=splits, order_current=False, chains=args.chains)
    torch.cuda.synchronize()
    barrier()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record()
    for _ in range(args.steps):
        cache.decode_step_host(qh, oh, splits=splits, order_current=False, chains=args.chains)
    torch.cuda.current_stream().wait_event(cache.host_step_ready)
    e5.record()
    torch.cuda.synchronize()
    e2e_ms = sync_max(e4.elapsed_time(e5) / args.steps)
    tot = torch.tensor([float(my_bytes)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tot)
    step_bytes = float(tot.item())
    if rank == 0:
        peak, peak_kind = measured_peak_gbs()
        frac = counts.sum(axis=0) / counts.sum()
        line = {
            "metric": METRIC, "value": round(step_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
            "data": f"synthetic (fp16 N(0,1) K/V/q; tier maps: {args.cfg4_map})",
            "config": {"workload": f"cfg4: batch 64 x 16K, Llama-3-8B GQA 32q/8kv d128, 32 layers, map {args.cfg4_map}",
                       "global_batch": Bg, "seq_len": T, "parallelism": f"batch-shard x{world}",
                       "tier_fractions_int2_int4_fp16": [round(float(x), 4) for x in frac],
                       "launch": launch_desc(args.chains),
                       "splits": splits, "schedule": schedule_desc(cache, splits, args.chains),
                       "l2": "inputs larger than L2"},
            "tokens_per_s": round(Bg / (ms * 1e-3), 1),
            "algorithmic_bytes_per_step": int(step_bytes),
            "roofline": {"bound": "hbm", "achieved": round(my_bytes / (ms * 1e-3) / 1e9, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(my_bytes / (ms * 1e-3) / 1e9 / peak, 4),
                         "peak_kind": peak_kind, "traffic": None},
            "e2e": {"value": round(step_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": int(q.numel() * 2), "d2h_bytes_per_step": int(q.numel() * 2)},
            "gpu_launches": args.steps * L,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def run_cfg1(args, torch, dist, dev, rank, world, local):
    """cfg1: Llama-2-7B single layer (32 MHA heads, d128), 4K context, batch 1, the reference's
    4K tier map (106/20/2 chunks).  15 MB of arenas: L2-resident and launch-latency bound, so
    every timed launch follows an L2 flush (256 MB read); R (flush, decode) pairs minus R
    flushes, per decode (events tick in ~2 us steps).  Not a roofline target; replicas only at N > 1."""
    from paper_2503_23294_b200 import batched, retrieval

    c = CFG1
    L, B, H, m, T, D = c["layers"], c["batch"], c["kv_heads"], c["q_per_kv"], c["context"], c["head_dim"]
    wl = load_workload(T, 0)
    search = retrieval.search_batched(wl["emb"][None], wl["norm"][None], wl["q"][None],
                                      np.array([wl["qnorm"]]), 0.6, 0.1)
    if not np.array_equal(search.tiers.cpu().numpy()[0], wl["tiers"]):
        raise SystemExit("4K tier map differs from the reference's")
    g = torch.Generator(device=dev)
    g.manual_seed(17)
    k = torch.randn((L, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    v = torch.randn((L, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    cache = batched.build_cache_batched(k, v, search)
    del k, v
    q = torch.randn((L, B, H * m, D), generator=g, device=dev, dtype=torch.float16)
    out = torch.empty_like(q)
    splits = pick_splits(args, cache, m, 1)
    # L2 flush by READING 256 MB (a max-reduction): the decode then starts with L2 full of
    # clean lines of other data.  (A write-based flush leaves up to 126 MB of dirty lines whose
    # write-back the timed launch would pay for.)
    flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
    for _ in range(max(args.warmup, 3)):
        cache.decode(q, splits=splits, out=out)
    # CUDA events tick in ~2 us steps here, coarser than the decode itself: time R (flush,
    # decode) pairs and R flushes alone, each as one event-bracketed loop, and take the
    # difference per decode (the median over args.steps repetitions of the pair)
    R = 20

    def loop(with_decode):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(R):
            flush.max()
            if with_decode:
                cache.decode(q, splits=splits, out=out)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    times = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            times.append((loop(True) - loop(False)) / R)
    ms = statistics.median(times)
    qh = q.cpu().pin_memory()
    oh = torch.empty(q.shape, dtype=torch.float16, pin_memory=True)
    et = []
    for i in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(R):
            flush.max()
            cache.decode_step_host(qh, oh, splits=splits)
        e1.record()
        torch.cuda.synchronize()
        et.append((e0.elapsed_time(e1) - loop(False)) / R)
    e2e_ms = statistics.median(et)
    nbytes = cache.algorithmic_bytes(m)
    if rank == 0:
        peak, peak_kind = measured_peak_gbs(sustained=False)
        counts = search.seg_counts.cpu().numpy()[0]
        gbs = nbytes / (ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": round(world * gbs, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic (fp16 N(0,1) K/V/q; reference search tier map, 4K seed 0)",
            "config": {"workload": "cfg1: Llama-2-7B 1 layer x 32 MHA heads d128, 4K ctx, batch 1",
                       "global_batch": B * world, "seq_len": T, "parallelism": f"replicas x{world}",
                       "tier_chunks_int2_int4_fp16": [int(x) for x in counts], "splits": splits,
                       "schedule": schedule_desc(cache, splits),
                       "l2": "L2 flushed (256 MB read) before every timed launch"},
            "us_per_decode": round(ms * 1e3, 2),
            "algorithmic_bytes_per_step": int(nbytes),
            "roofline": {"bound": "latency", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "peak_kind": peak_kind, "traffic": None},
            "e2e": {"value": round(world * nbytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": int(q.numel() * 2), "d2h_bytes_per_step": int(q.numel() * 2)},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def run_cfg5(args, torch, dist, dev, rank, world, local):
    """cfg5 prefill sharded by layer: every rank runs the 128K search (its tier map
    is the reference's) and reorders / quantizes / packs its 32/N layers x 8 kv heads; no
    exchange.  Strong scaling of the fixed 32-layer build; max-over-ranks device time."""
    from paper_2503_23294_b200 import batched, distributed, retrieval

    c = CFG5
    L, B, H, T, D = c["layers"], c["batch"], c["kv_heads"], c["context"], c["head_dim"]
    lo, hi = distributed.layer_shard(L, world, rank)
    Ll = hi - lo
    wl = load_workload(T, 0)
    g = torch.Generator(device=dev)
    g.manual_seed(77 + rank)
    k = torch.randn((Ll, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    v = torch.randn((Ll, B, T, H, D), generator=g, device=dev, dtype=torch.float16)
    s = retrieval.search_batched(wl["emb"][None], wl["norm"][None], wl["q"][None], np.array([wl["qnorm"]]))
    if not np.array_equal(s.tiers.cpu().numpy()[0], wl["tiers"]):
        raise SystemExit("128K tier map differs from the reference's")
    counts = s.seg_counts.cpu().numpy()
    # search inputs resident on the device like the K/V (the timed region is device work only)
    dev_emb = [torch.as_tensor(x, device=dev) for x in (wl["emb"][None], wl["norm"][None], wl["q"][None],
                                                      np.array([wl["qnorm"]]))]
    cache = batched.BatchedKVCache(Ll, B, H, counts[:, 0], counts[:, 1], counts[:, 2], [T], 0, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    times = []
    with ClockSampler(local) as clk:
        for i in range(max(args.warmup, 3) + args.steps):
            flush.max()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s2 = retrieval.search_batched(*dev_emb, check=False)
            cache.build(k, v, s2.perm, check=False)
            e1.record()
            torch.cuda.synchronize()
            if i >= max(args.warmup, 3):
                times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n2, n4, nf = (int(x) for x in counts[0])
    read = 2 * L * H * T * D * 2
    write = 2 * L * H * (n2 * 32 * 48 + n4 * 32 * 80 + (nf * 32 + (T - 32 * (n2 + n4 + nf))) * 256)
    if rank == 0:
        peak, peak_kind = measured_peak_gbs(sustained=False)
        per_rank = (read + write) * Ll / L / (ms * 1e-3) / 1e9
        line = {
            "metric": "cfg5 prefill search + reorder/quantize/pack GB/s (% HBM peak)",
            "value": round((read + write) / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic (fp16 N(0,1) K/V; reference search tier map, 128K seed 0)",
            "config": {"workload": "cfg5: prefill search + reorder/quantize/pack, 128K ctx x 32 layers x 8 kv heads, b1",
                       "global_batch": B, "seq_len": T, "parallelism": f"layer-shard x{world}",
                       "l2": "L2 flushed (256 MB write) before every timed build"},
            "bytes_read": read, "bytes_written": write,
            "roofline": {"bound": "hbm", "achieved": round(per_rank, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(per_rank / peak, 4), "peak_kind": peak_kind,
                         "traffic": profile_traffic("reorder_quantize_pack")},
            "e2e": None,
            "gpu_launches": args.steps * 3,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--splits", type=int, default=None)
    ap.add_argument("--workload", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"], default="cfg2",
                    help="cfg2: batch-sharded 32K GQA decode (default); cfg3: 128K MHA decode with "
                         "sequence split-KV across the ranks (NCCL all-gather + LSE merge); cfg4: "
                         "batch 64 x 16K GQA decode sharded over the ranks (--cfg4-map); cfg1: the "
                         "4K single-layer MHA parity config (L2-flushed, latency bound); cfg5: the "
                         "128K prefill build with its layers sharded over the ranks")
    ap.add_argument("--cfg4-map", choices=["skewed", "all_int2", "all_fp16"], default="skewed")
    ap.add_argument("--cfg3-split", choices=["seq", "head"], default="seq",
                    help="cfg3 partition: sequence split-KV with NCCL LSE merge, or whole KV heads per GPU")
    ap.add_argument("--no-tpot", action="store_true", help="skip the 128-step decode loop (TPOT)")
    ap.add_argument("--no-sustained", action="store_true", help="skip the ~3 s sustained-rate run")
    ap.add_argument("--no-split-kv", action="store_true",
                    help="N>1 default line: skip the cfg3 split_kv / head_shard sub-objects")
    ap.add_argument("--schedule", choices=["auto", "wp", "split"], default="auto",
                    help="decode schedule of whole-batch launches: wp = warp plan (one 16-warp CTA per SM, "
                         "units split at warp granularity), split = 4-warp CTAs with --splits per unit, "
                         "auto = the warp plan unless the cache has fewer than 8 tiles per warp")
    ap.add_argument("--chains", type=int, default=0,
                    help="micro-batch chains per decode step (cfg2/cfg4): the batch is split into this "
                         "many sequence ranges, each its own chain of per-layer launches on its own "
                         "stream, so one range's layer boundary overlaps the others' work; 0 (default) = "
                         "one chain per sequence for cfg2, 1 for the other workloads")
    args = ap.parse_args()
    if args.chains == 0 and args.workload not in ("cfg2", "cfg3", "cfg4"):
        args.chains = 1

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched without torchrun: start one rank per GPU ourselves (127.0.0.1 rendezvous)
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus and os.environ.get("CKV_BENCH_SHARE_GPU") != "1":
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {n} GPU(s) visible")
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and rank == 0:
        print(f"bench.py: WORLD_SIZE {world} != --gpus {args.gpus}; using {world} ranks", file=sys.stderr)

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    # CKV_BENCH_SHARE_GPU=1 (test aid): every rank on cuda:0 over gloo, to exercise the N>1
    # control flow on a one-GPU box (its numbers are not measurements)
    share = os.environ.get("CKV_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    if args.workload in ("cfg1", "cfg3", "cfg4", "cfg5"):
        fn = {"cfg1": run_cfg1, "cfg3": run_cfg3, "cfg4": run_cfg4, "cfg5": run_cfg5}[args.workload]
        fn(args, torch, dist, dev, rank, world, local)
        if world > 1:
            dist.destroy_process_group()
        return

    from paper_2503_23294_b200 import batched as batched_mod

    cache, q, search = build_cfg2(torch, dev, rank)
    L, B = cache.L, cache.B
    m = q.shape[2] // cache.H
    if args.chains == 0:
        args.chains = auto_chains(B)
    splits = pick_splits(args, cache, m)
    wp = splits is None
    out = torch.empty_like(q)
    step_bytes = cache.algorithmic_bytes(m)

    chain_streams = [torch.cuda.Stream(device=dev) for _ in range(args.chains)]

    def eager_step():  # per-layer launches; layer l+1 overlaps its K/V prefetch with layer l
        cache._launch_layers(q, out, 0, L, splits, None, args.chains, chain_streams)

    # the same 32 PDL-chained launches captured once in a CUDA graph (a serving loop's decode
    # step); the eager figure is reported beside it
    graph = cache.decode_graph(q, out, splits=splits, chains=args.chains)
    step = graph.replay
    for _ in range(max(args.warmup, 3)):
        step()
        eager_step()
    torch.cuda.synchronize()
    barrier()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    sec = ms * 1e-3
    value = world * step_bytes / sec / 1e9
    tokens_per_s = world * B / sec

    def idle_gap():
        """Every figure below starts from the same power state as the headline window: after
        ~0.3 s of continuous load the board reaches its power limit (see `sustained`), so each
        one follows a 1 s idle gap."""
        torch.cuda.synchronize()
        time.sleep(1.0)
        barrier()

    # end to end through the public API: pinned host q -> H2D, decode (all layers), D2H
    # (decode_step_host: uploads / downloads overlap the per-layer launches on copy streams)
    idle_gap()
    qh = q.cpu().pin_memory()
    oh = torch.empty(q.shape, dtype=torch.float16, pin_memory=True)
    for _ in range(3):
        cache.decode_step_host(qh, oh, splits=splits, order_current=False, chains=args.chains)
    torch.cuda.synchronize()
    barrier()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record()
    for _ in range(args.steps):  # a step's downloads overlap the next step's first layers
        cache.decode_step_host(qh, oh, splits=splits, order_current=False, chains=args.chains)
    torch.cuda.current_stream().wait_event(cache.host_step_ready)  # the last download is timed
    e5.record()
    torch.cuda.synchronize()
    e2e_ms = e4.elapsed_time(e5) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_gbs = world * step_bytes / (e2e_ms * 1e-3) / 1e9

    # eager launches (no graph), same step
    idle_gap()
    e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e6.record()
    for _ in range(args.steps):
        eager_step()
    e7.record()
    torch.cuda.synchronize()
    eager_gbs = world * step_bytes / (e6.elapsed_time(e7) / args.steps * 1e-3) / 1e9

    # lockstep figure: the whole batch as ONE chain of per-layer launches (every layer waits for
    # the previous layer of every sequence), the schedule the cache would pick for it
    lockstep = None
    if args.chains > 1:
        ls_args = argparse.Namespace(**{**vars(args), "chains": 1})
        ls_splits = pick_splits(ls_args, cache, m)
        ls_graph = cache.decode_graph(q, out, splits=ls_splits)
        idle_gap()
        for _ in range(3):
            ls_graph.replay()
        torch.cuda.synchronize()
        barrier()
        with ClockSampler(local) as lclk:
            e10, e11 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e10.record()
            for _ in range(args.steps):
                ls_graph.replay()
            e11.record()
            torch.cuda.synchronize()
        ls_ms = e10.elapsed_time(e11) / args.steps
        if world > 1:
            t = torch.tensor([ls_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ls_ms = float(t.item())
        lockstep = {"value": round(world * step_bytes / (ls_ms * 1e-3) / 1e9, 2), "ms_per_step": round(ls_ms, 4),
                    "launch": launch_desc(1), "schedule": schedule_desc(cache, ls_splits),
                    "clocks": lclk.summary()}
        del ls_graph
        cache.schedule = args.schedule

    # single-launch (all 32 layers in one grid) figure for the same cache
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    single_splits = args.splits or cache.default_splits(m, L)  # split schedule: the faster one in one launch
    idle_gap()
    for _ in range(3):
        cache.decode(q, out=out, splits=single_splits)
    with ClockSampler(local) as fclk:
        e2.record()
        for _ in range(args.steps):
            cache.decode(q, out=out, splits=single_splits)
        e3.record()
        torch.cuda.synchronize()
    fused_gbs = step_bytes / (e2.elapsed_time(e3) / args.steps * 1e-3) / 1e9

    sched_desc = schedule_desc(cache, splits, args.chains)
    # parity of the timed cache: the graph step's output for sampled units vs the reference
    graph.replay()
    torch.cuda.synchronize()
    parity = sampled_parity(cache, q, out, m)

    # serving decode loop (TPOT): per step one appended token per (layer, sequence, kv head)
    # and the per-layer decode launches, all in one CUDA graph (batched.DecodeLoop); the cache
    # grows by 128 tokens per sequence, so this runs after the fixed-size measurements
    memory = cache.memory_footprint().as_dict()
    tpot = None
    if not args.no_tpot:
        n_tok = min(128, int((cache.cap_fp - cache.seq_host[:, 5]).min()))
        gt = torch.Generator(device=dev)
        gt.manual_seed(555 + rank)
        kn = torch.randn((n_tok, L, B, cache.H, 128), generator=gt, device=dev, dtype=torch.float16)
        vn = torch.randn((n_tok, L, B, cache.H, 128), generator=gt, device=dev, dtype=torch.float16)
        loop = batched_mod.DecodeLoop(cache, m, splits=splits, chains=args.chains)
        bytes0 = cache.algorithmic_bytes(m)
        idle_gap()
        e8, e9 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as tclk:
            e8.record()
            for i in range(n_tok):
                loop.step(q, kn[i], vn[i])
            e9.record()
            torch.cuda.synchronize()
        tp_ms = e8.elapsed_time(e9) / n_tok
        if world > 1:
            t = torch.tensor([tp_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tp_ms = float(t.item())
        mean_bytes = (bytes0 + cache.algorithmic_bytes(m)) / 2
        tpot = {"steps": n_tok, "ms_per_token": round(tp_ms, 4), "clocks": tclk.summary(),
                "tokens_per_s": round(world * B / (tp_ms * 1e-3), 1),
                "gbs": round(world * mean_bytes / (tp_ms * 1e-3) / 1e9, 2),
                "note": "batched.DecodeLoop: per step ckv_append_tokens (one new K/V row per unit) + the "
                        f"per-layer decode launches ({launch_desc(args.chains)}), one CUDA graph replay; the "
                        f"context grows from {CFG2['context']} to {CFG2['context'] + n_tok} tokens"}
        del kn, vn, loop

    # sustained rate: the same graph step back to back for ~2 s (the board settles at its power
    # limit), then ~1 s timed with clocks sampled — the short window above runs at boost clocks
    sustained = None
    if not args.no_sustained:
        s_bytes = cache.algorithmic_bytes(m)
        torch.cuda.synchronize()
        barrier()
        t_end = time.time() + 2.0
        while time.time() < t_end:
            for _ in range(50):
                step()
            torch.cuda.synchronize()
        n_s = max(1, int(round(1000.0 / ms)))
        with ClockSampler(local) as sclk:
            e12, e13 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e12.record()
            for _ in range(n_s):
                step()
            e13.record()
            torch.cuda.synchronize()
        s_ms = e12.elapsed_time(e13) / n_s
        if world > 1:
            t = torch.tensor([s_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            s_ms = float(t.item())
        sustained = {"value": round(world * s_bytes / (s_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                     "ms_per_step": round(s_ms, 4), "steps": n_s, "clocks": sclk.summary(),
                     "note": "the default graph step replayed back to back for 2 s untimed, then ~1 s timed "
                             "(after the TPOT appends: context + 128 tokens); the headline window is "
                             f"{args.steps} steps after an idle gap"}

    split_kv = None
    if world > 1 and not args.no_split_kv:
        # cfg3 (128K, 40 layers x 40 heads) on the same ranks: sequence split-KV with the NCCL
        # exchange + LSE merge, and the KV-head partition beside it (no collective)
        sk_steps = max(3, min(args.steps, 10))
        seq = measure_cfg3(args, torch, dist, dev, rank, world, "seq", steps=sk_steps)
        head = measure_cfg3(args, torch, dist, dev, rank, world, "head", steps=sk_steps)
        split_kv = {"workload": "cfg3: Llama-2-13B 40 layers x 40 MHA heads d128, 128K ctx, batch 1 (strong scaling)",
                    "value": seq["value"], "unit": "GB/s", "ms_per_step": seq["ms_per_step"],
                    "local_decode_ms": seq["local_decode_ms"], "exchange_merge_ms": seq["exchange_merge_ms"],
                    "per_layer_merge_us": seq["per_layer_merge_us"],
                    "per_layer_merge_note": seq["per_layer_merge_note"], "splits": seq["splits"],
                    "parallelism": seq["parallelism"], "e2e": seq["e2e"],
                    "lockstep_per_layer": seq.get("lockstep_per_layer"),
                    "head_shard": {"value": head["value"], "unit": "GB/s", "ms_per_step": head["ms_per_step"],
                                   "parallelism": head["parallelism"], "e2e": head["e2e"],
                                   "lockstep_per_layer": head.get("lockstep_per_layer")}}
        p2p = seq.get("p2p") or {}
        if "ms_per_step" in p2p:
            p2p["value"] = round(seq["algorithmic_bytes_per_step"] / (p2p["ms_per_step"] * 1e-3) / 1e9, 2)
        split_kv["p2p"] = p2p

    prefill = None
    if rank == 0 and world == 1 and not args.no_prefill:
        del cache
        torch.cuda.empty_cache()
        time.sleep(2.0)  # out of the power limit the sustained run left the board at
        prefill = bench_prefill(torch, dev)

    if rank == 0:
        peak, peak_kind = measured_peak_gbs()
        launches_per_step = L * args.chains  # the split merge happens inside the decode launch
        per_launch_bytes = step_bytes / launches_per_step
        achieved = per_launch_bytes / (ms * 1e-3 / launches_per_step) / 1e9
        counts = search.seg_counts.cpu().numpy()
        frac = counts.sum(axis=0) / counts.sum()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic (fp16 N(0,1) K/V/q; reference search tier maps, seeds 0-7)",
            "config": {"workload": "cfg2: Llama-3-8B GQA 32q/8kv d128, 32 layers, 32K ctx, batch 8 per GPU",
                       "global_batch": B * world, "seq_len": CFG2["context"], "parallelism": f"batch-shard x{world}",
                       "tier_fractions_int2_int4_fp16": [round(float(x), 4) for x in frac],
                       "launch": launch_desc(args.chains),
                       "splits": splits, "schedule": sched_desc,
                       "l2": "inputs larger than L2 (7.1 GB arenas vs 126 MB L2)"},
            "tokens_per_s": round(tokens_per_s, 1),
            "algorithmic_bytes_per_step": step_bytes,
            "eager_launches_gbs": round(eager_gbs, 2),
            "single_launch_all_layers_gbs": round(fused_gbs, 2),
            "single_launch_clocks": fclk.summary(),
            "lockstep_per_layer": lockstep,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                         "traffic": profile_traffic("decode_kernel" if args.chains == 1 else "decode_kernel_chain")},
            "e2e": {"value": round(e2e_gbs, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": int(q.numel() * 2), "d2h_bytes_per_step": int(q.numel() * 2)},
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk.summary(),
        }
        if prefill is not None:
            line["prefill"] = prefill
        if split_kv is not None:
            line["split_kv"] = split_kv
        line["memory"] = memory
        line["parity_sampled_max_rel"] = round(parity, 6)
        line["parity_note"] = ("3 units (layer, sequence, kv head) of the timed cfg2 cache, graph-step output vs "
                               "the reference algorithm in f64 (oracle), tolerance 1e-2")
        if tpot is not None:
            line["tpot"] = tpot
        if sustained is not None:
            line["sustained"] = sustained
        if world == 1 and not args.no_cpu_baseline:
            gbs, n, wall, kind, kernels = cpu_baseline(seconds=12.0, processes=1, n_units=4)
            line["cpu_baseline"] = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": kind,
                                    "cpu_model": cpu_model(),
                                    "sample": f"{n} decodes of 4 prebuilt cfg2 units (32K ctx, m=4) through "
                                              f"mixed_decode_attention, {wall:.1f} s single process; kernels: {kernels}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
