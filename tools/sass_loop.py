"""Static look at the decode kernel's hot INT2 block: the longest straight-line SASS run with
>= 16 HMMA (the pipelined QK(i+1)/PV(i) body).  Prints its opcode histogram; no GPU needed."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2503_23294_b200/_lib/libckv.so"
fn = sys.argv[2] if len(sys.argv) > 2 else "decode_kernel"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
body, on = [], False
for line in sass.splitlines():
    if "Function : " in line:
        on = fn in line
        continue
    if on:
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for _, ins in body:
    m = re.search(r"BRA\S*\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", ins)
    if m and m.group(1):
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for addr, ins in body:
    if addr in targets and cur:
        blocks.append(cur); cur = []
    cur.append(ins)
    if re.search(r"\bBRA\b|\bEXIT\b", ins):
        blocks.append(cur); cur = []
if cur:
    blocks.append(cur)
hot = [b for b in blocks if sum("HMMA" in i for i in b) >= 16]
for b in sorted(hot, key=len)[:3]:
    c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0].split(".")[0] for i in b)
    print(len(b), "instrs:", dict(c.most_common()))
if "-v" in sys.argv:
    b = sorted(hot, key=len)[int(sys.argv[sys.argv.index("-v") + 1]) if len(sys.argv) > sys.argv.index("-v") + 1 else 1]
    for i in b:
        print("   ", i)
