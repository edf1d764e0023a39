"""ctypes binding of the C-ABI in include/ckv.h (the drop-in boundary).

The shared library is built in-tree by ``_build.build()`` into ``_lib/libckv.so``.
There is no fallback: if the library is missing or no CUDA device is present, the
calls raise.  Tensors are passed as raw device pointers plus sizes, together with
the current torch CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import re

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CKV_LIB_PATH") or os.path.join(_HERE, "_lib", "libckv.so")  # override: A/B builds (tuning aid)
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "ckv.h")

CKV_OK = 0
CKV_ERR_BITS = -1
CKV_ERR_GROUP = -2
CKV_ERR_SHAPE = -3
CKV_ERR_CAPACITY = -4
CKV_ERR_UNSUPPORTED = -5
CKV_ERR_ARG = -6
CKV_ERR_CUDA = -7

FLAG_NONFINITE = 1
FLAG_ZERO_QUERY = 2
FLAG_CROSSING = 4
FLAG_EMPTY_SCORES = 8
FLAG_NONFINITE_FP16 = 16

SEQ_FIELDS = 8  # CKV_SEQ_FIELDS
DECODE_PDL = 1  # CKV_DECODE_PDL
ABI_VERSION = 1  # ckv_abi_version() of the matching include/ckv.h

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_f32 = ctypes.c_float


class Arena(ctypes.Structure):
    """struct ckv_arena (include/ckv.h)."""

    _fields_ = [
        ("codes2", _vp), ("meta2", _vp), ("codes4", _vp), ("meta4", _vp), ("fp", _vp),
        ("span_flags", _vp), ("span_max", _vp), ("rows2", _i64), ("rows4", _i64), ("rows_fp", _i64),
    ]


_SIGNATURES = {
    "ckv_abi_version": ([], _i32),
    "ckv_status_string": ([_i32], ctypes.c_char_p),
    "ckv_quantize_groups_f64": ([_vp, _i64, _i64, _i32, _i64, _vp, _vp, _vp, _vp, _vp], _i32),
    "ckv_quantize_groups_f16": ([_vp, _i64, _i64, _i32, _i64, _vp, _vp, _vp, _vp, _vp], _i32),
    "ckv_pack_codes": ([_vp, _i64, _i32, _vp, _vp], _i32),
    "ckv_unpack_codes": ([_vp, _i64, _i32, _i64, _vp, _vp], _i32),
    "ckv_dequantize_codes_f64": ([_vp, _i64, _vp, _vp, _i64, _i64, _i32, _i64, _vp, _vp], _i32),
    "ckv_matmul_packed_f64": ([_vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _i32, _i64,
                               _i32, _vp, _i64, _i32, _vp], _i32),
    "ckv_matmul_f64": ([_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _i64, _i32, _vp], _i32),
    "ckv_scale_mask_softmax_f64": ([_vp, _i64, _i64, _f64, _vp, _vp], _i32),
    "ckv_scatter_rows_f64": ([_vp, _i64, _i64, _vp, _vp, _vp], _i32),
    "ckv_search": ([_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _f64, _f64, _vp, _vp, _vp, _vp, _vp,
                    _vp, _vp], _i32),
    "ckv_bow_encode": ([_vp, _vp, _i32, _i32, ctypes.c_char_p, _i32, _vp, _vp, _vp], _i32),
    "ckv_tfidf_encode": ([_vp, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp], _i32),
    "ckv_assign_tiers": ([_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "ckv_reorder_quantize_pack": ([_vp, _vp, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _vp, _i32,
                                   _vp, _i32, Arena, Arena, _vp, _vp], _i32),
    "ckv_append_tokens": ([_vp, _vp, _i32, _i32, _i32, _vp, Arena, Arena, _vp], _i32),
    "ckv_expand_meta": ([_vp, _i64, _i32, _vp, _vp, _vp], _i32),
    "ckv_arena_export": ([_vp, _vp, _i64, _i32, _i32, _i64, _vp, _vp, _vp], _i32),
    "ckv_reconstruct": ([Arena, Arena, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _i64, _i64, _i64, _i64, _i32,
                         _vp], _i32),
    "ckv_decode_workspace_bytes": ([_i32, _i32, _i32, _i32, _i32], _i64),
    "ckv_decode_ctas_per_sm": ([], _i32),
    "ckv_decode_attention": ([_vp, _i64, _i64, Arena, Arena, _vp, _i32, _i32, _i32, _i32, _f32, _i32,
                              _vp, _vp, _i64, _i64, _vp, _i32, _vp], _i32),
    "ckv_decode_attention_seqs": ([_vp, _i64, _i64, Arena, Arena, _vp, _i32, _i32, _i32, _i32, _i32, _i32,
                                   _f32, _i32, _vp, _vp, _i64, _i64, _vp, _i32, _vp], _i32),
    "ckv_decode_attention_range": ([_vp, _i64, _i64, Arena, Arena, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                    _i32, _f32, _i32, _vp, _vp, _i64, _i64, _vp, _i32, _vp], _i32),
    "ckv_decode_wp_workspace_bytes": ([_i32, _i32, _i32, _i32, _i32], _i64),
    "ckv_decode_wp_cta_warps": ([], _i32),
    "ckv_decode_wp_plan_ints": ([_i32], _i64),
    "ckv_decode_wp_plan": ([_vp, _i32, _i32, _vp, _i32, _vp, _vp, _vp], _i32),
    "ckv_decode_attention_wp": ([_vp, _i64, _i64, Arena, Arena, _vp, _i32, _i32, _i32, _i32, _f32, _vp, _i32, _i32,
                                 _i32, _vp, _vp, _i64, _i64, _vp, _i32, _vp], _i32),
    "ckv_decode_attention_wp_seqs": ([_vp, _i64, _i64, Arena, Arena, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _f32,
                                      _vp, _i32, _i32, _i32, _vp, _vp, _i64, _i64, _vp, _i32, _vp], _i32),
    "ckv_lse_merge": ([_vp, _i32, _i64, _vp, _vp], _i32),
    "ckv_lse_merge_ptrs": ([_vp, _i32, _i64, _vp, _vp], _i32),
}

_lib = None


def header_functions():
    """Names of every function declared in include/ckv.h."""
    with open(HEADER_PATH, "r", encoding="utf-8") as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*)\s+(ckv_\w+)\s*\(", text, re.M)))


def load():
    """Load libckv.so (no GPU needed to load).  Raises if the library was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__; __graft_entry__.build()')")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, ret) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ret
    if lib.ckv_abi_version() != ABI_VERSION:  # a stale build of another header revision
        raise RuntimeError(f"{LIB_PATH} has ABI {lib.ckv_abi_version()}, this package expects {ABI_VERSION}: rebuild")
    _lib = lib
    return lib


def device():
    """The CUDA device every call runs on.  No CPU fallback."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_23294_b200 requires a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return _vp(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return _vp(t.data_ptr())


def check(status):
    """Map a C-ABI status to the reference's exception types."""
    if status == CKV_OK:
        return
    msg = load().ckv_status_string(status).decode()
    if status in (CKV_ERR_BITS, CKV_ERR_GROUP, CKV_ERR_SHAPE, CKV_ERR_CAPACITY, CKV_ERR_ARG,
                  CKV_ERR_UNSUPPORTED):
        raise ValueError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    fn = getattr(load(), name)
    check(fn(*args))
