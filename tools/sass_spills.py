"""Where do local-memory spills sit relative to the decode kernel's loops?  Prints each
backward-branch loop (address range, instruction count, HMMA count) with its STL/LDL count.
Usage: python tools/sass_spills.py [cubin or .so] [kernel substring]"""
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
loops = []
for a, ins in body:
    m = re.search(r"BRA\S*\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", ins)
    if m and m.group(1) and int(m.group(1), 16) < a:
        loops.append((int(m.group(1), 16), a))
spills = [(a, i) for a, i in body if re.search(r"\b(STL|LDL)\b", i)]
print(f"{len(body)} instructions, {len(spills)} STL/LDL")
for lo, hi in sorted(loops, key=lambda x: x[0]):
    ins = [i for a, i in body if lo <= a <= hi]
    n_h = sum("HMMA" in i for i in ins)
    n_s = sum(bool(re.search(r"\b(STL|LDL)\b", i)) for i in ins)
    if n_h or n_s:
        print(f"loop {lo:#x}-{hi:#x}: {len(ins)} instrs, {n_h} HMMA, {n_s} STL/LDL")
