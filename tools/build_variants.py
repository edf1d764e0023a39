"""Build decode tuning variants of libckv.so into build/variants/<name>.so (A/B runs select one
with CKV_LIB_PATH).  Usage: python tools/build_variants.py name=DEF1,DEF2 name2=DEF3 ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_23294_b200 import _build  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    _build.build(out=out, defines=[d for d in defs.split(",") if d])
    return out


if __name__ == "__main__":
    with ThreadPoolExecutor(8) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print(o)
