#!/bin/bash
# initcheck with every report kept, aggregated by (kernel, source line, host frame)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool initcheck --print-limit 2000000 --target-processes all \
  python tools/sanitize_cases.py > gpurun_out/initcheck_full.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/initcheck_full.log
python - <<'PY'
import collections, re
txt = open("gpurun_out/initcheck_full.log").read()
blocks = txt.split("========= Uninitialized")[1:]
agg = collections.Counter()
for b in blocks:
    dev = re.search(r"Device Frame: ([^\(]*)\([^\n]*? in ([^\n]*)", b)
    host = re.findall(r"Host Frame: (\S+) in (\S+\.py:\d+)", b)
    size = re.search(r"memory read of size (\d+)", "Uninitialized" + b[:200])
    agg[(dev.group(1) if dev else "?", dev.group(2) if dev else "?", host[1] if len(host) > 1 else host[:1] and host[0])] += 1
with open("gpurun_out/initcheck_agg.txt", "w") as fh:
    fh.write(f"{len(blocks)} reports\n")
    for k, v in agg.most_common(40):
        fh.write(f"{v:8d}  {k}\n")
print(open("gpurun_out/initcheck_agg.txt").read())
PY
