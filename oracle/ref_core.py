"""Test infrastructure: the reference's own compiled kernel module (chunkkv.kernels._core,
built from /root/reference/pkg/src/chunkkv/kernels/_core.pyx by oracle/Makefile into
oracle/_ref/).  Only tests and bench.py's CPU legs load it; the product never does."""

from __future__ import annotations

import glob
import importlib.util
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
_mod = None


def load():
    """The compiled reference module, or None when oracle/_ref holds no build."""
    global _mod
    if _mod is not None:
        return _mod
    hits = sorted(glob.glob(os.path.join(REF_DIR, "_core*.so")))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_core", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    _mod = mod
    return mod
