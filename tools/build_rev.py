"""Build libckv.so from the csrc/ tree of a git revision into build/variants/<name>.so (A/B runs
against the working tree's kernel with tools/ab.sh).  Usage: python tools/build_rev.py REV NAME"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_23294_b200 import _build  # noqa: E402

rev, name = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as tmp:
    files = subprocess.run(["git", "-C", ROOT, "ls-tree", "--name-only", rev, "paper_2503_23294_b200/csrc/"],
                           capture_output=True, text=True, check=True).stdout.split()
    for f in files:
        data = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{f}"], capture_output=True, check=True).stdout
        with open(os.path.join(tmp, os.path.basename(f)), "wb") as fh:
            fh.write(data)
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = sorted(os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cu"))
    cmd = ["nvcc", *_build.NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", tmp, "-o", out, *srcs]
    subprocess.run(cmd, check=True)
    print(out)
