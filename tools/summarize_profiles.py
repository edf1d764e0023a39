"""Turn the ncu captures of a GPU session (gpurun_out/) into committed summaries (profiles/).

    python tools/summarize_profiles.py r01

Writes profiles/<tag>_ncu_summary.md (key metrics, stall mix, dynamic opcode mix per kernel),
profiles/<tag>_launches.csv (one decode step + one prefill build: every launch with its device
time; ncu serialises launches and runs them cold, so compare shares, not absolutes) and
profiles/traffic.json (DRAM bytes per launch, read by bench.py for roofline.traffic).
"""

from __future__ import annotations

import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (%)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (%)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe (%)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe (%)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe (%)"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid size"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("sm__cycles_active.min", "SM active cycles (min)"),
    ("sm__cycles_active.max", "SM active cycles (max)"),
]


def ncu(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"] +
                          (["--print-source", "sass"] if page == "source" else []),
                          capture_output=True, text=True).stdout


def summarize(rep):
    r = list(csv.reader(io.StringIO(ncu(rep, "raw"))))
    hdr, units, v = r[0], r[1], r[2]
    vals = dict(zip(hdr, v))
    unit = dict(zip(hdr, units))
    name = vals.get("Kernel Name", "?")
    metrics = {}
    for key, label in KEYS:
        if key in vals:
            metrics[label] = f"{vals[key]} {unit.get(key, '')}".strip()
    stalls = {}
    for h, x in vals.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(x.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    stall_mix = [(k, 100 * x / tot) for k, x in sorted(stalls.items(), key=lambda t: -t[1])[:10]]
    src = list(csv.reader(io.StringIO(ncu(rep, "source"))))
    ops = collections.Counter()
    total = 0
    if len(src) > 2:
        sh = src[1]
        idx = {h: i for i, h in enumerate(sh)}
        for row in src[2:]:
            if len(row) < len(sh):
                continue
            parts = row[idx["Source"]].strip().split()
            if not parts:
                continue
            op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
            try:
                n = int(row[idx["Instructions Executed"]] or 0)
            except ValueError:
                continue
            ops[op.split(".")[0]] += n
            total += n
    opmix = [(op, 100 * n / total) for op, n in ops.most_common(16)] if total else []
    dram = None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        dram = sum(float(vals[k].replace(",", "")) * scale[unit[k]]
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except (KeyError, ValueError):
        pass
    return name, metrics, stall_mix, opmix, dram


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary ({tag})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(`tools/gpu_round.sh`); one launch each.  Launch list: "
             f"`{tag}_launches.csv` (`--metrics gpu__time_duration.sum`).", ""]
    traffic = {}
    for rep, key, what in (
            ("decode_chain_prof.ncu-rep", "decode_kernel_chain",
             "the bench default: one (sequence, layer) launch of the split schedule in a micro-batch chain"),
            ("decode_prof.ncu-rep", "decode_kernel", "one lockstep per-layer launch (whole batch, warp plan)"),
            ("decode_split_prof.ncu-rep", "decode_kernel_split", "one lockstep per-layer launch (whole batch, split)"),
            ("quant_prof.ncu-rep", "reorder_quantize_pack", "the cfg5 build (128K x 32 layers x 8 heads)")):
        path = os.path.join(OUT, rep)
        if not os.path.exists(path):
            continue
        name, metrics, stalls, opmix, dram = summarize(path)
        traffic[key] = dram
        lines += [f"## {name}", "", f"{what}.", "", "| metric | value |", "|---|---|"]
        lines += [f"| {k} | {v} |" for k, v in metrics.items()]
        lines += ["", "Stall mix (sampled): " + ", ".join(f"{k} {x:.1f}%" for k, x in stalls), "",
                  "Dynamic opcode mix: " + ", ".join(f"{k} {x:.1f}%" for k, x in opmix), ""]
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if traffic:
        with open(os.path.join(PROF, "traffic.json"), "w") as fh:
            json.dump(traffic, fh, indent=1)
    src = os.path.join(OUT, "launches.csv")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(PROF, f"{tag}_launches.csv"))
        # per-kernel share of device time
        rows = list(csv.reader(open(src)))
        hdr_i = next((i for i, r in enumerate(rows) if "Kernel Name" in r), None)
        if hdr_i is not None:
            h = rows[hdr_i]
            ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
            agg = collections.Counter()
            cnt = collections.Counter()
            for r in rows[hdr_i + 1:]:
                if len(r) > vi and r[mi] == "gpu__time_duration.sum":
                    nm = r[ki].split("(")[0]
                    agg[nm] += float(r[vi].replace(",", ""))
                    cnt[nm] += 1
            tot = sum(agg.values()) or 1.0
            with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "a") as fh:
                fh.write("## Launch list (one decode step of 32 per-layer launches + one cfg5 prefill build)\n\n")
                fh.write("| kernel | launches | total device time | share |\n|---|---|---|---|\n")
                for nm, t in agg.most_common():
                    fh.write(f"| {nm} | {cnt[nm]} | {t:.1f} | {100 * t / tot:.1f}% |\n")
    print("wrote", os.path.join(PROF, f"{tag}_ncu_summary.md"))


if __name__ == "__main__":
    main()
