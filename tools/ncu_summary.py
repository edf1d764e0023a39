"""Summarise an ncu report: key metrics, stall reasons, dynamic opcode mix."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, v = r[0], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
for h, x in zip(hdr, v):
    if h in want:
        print(f"{h:60s} {x}")
d = {}
for h, x in zip(hdr, v):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        d[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(x.replace(",", ""))
tot = sum(d.values()) or 1
print("stalls:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in sorted(d.items(), key=lambda t: -t[1])[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hdr = r[1]
idx = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter()
total = 0
for row in r[2:]:
    if len(row) < len(hdr):
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
print("dynamic warp instructions", total)
print(", ".join(f"{op} {100*n/total:.1f}%" for op, n in ops.most_common(24)))
