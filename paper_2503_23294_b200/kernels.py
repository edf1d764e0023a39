"""Kernel facade — the drop-in for ``chunkkv.kernels`` (kernels/__init__.py:9-57).

Same five callables with the same argument meaning, return types and ValueError
sites as the reference's numpy/Cython backends, executed by the sm_100a kernels in
libckv.so.  There is exactly one backend (``BACKEND``); no environment switch, no
CPU fallback.  Inputs may be numpy arrays or torch tensors (any device); outputs are
numpy arrays like the reference's.  The ``*_dev`` variants keep everything on the
GPU (torch CUDA tensors in and out) for callers that chain kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

ALLOWED_BITS = (2, 4)  # kernels/__init__.py:41
BACKEND = "cuda-sm100a"


def _check_bits(bits):
    # _numpy.py:14-16 / _core.pyx:21-24
    if bits not in ALLOWED_BITS:
        raise ValueError(f"bitwidth must be one of {ALLOWED_BITS}, got {bits}")


def to_dev(x, dtype):
    """numpy / torch -> contiguous CUDA tensor of `dtype` (copy only when needed)."""
    dev = _lib.device()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        arr = np.asarray(x)
        if dtype == torch.float64:
            arr = np.ascontiguousarray(arr, dtype=np.float64)
        elif dtype == torch.uint8:
            arr = np.ascontiguousarray(arr, dtype=np.uint8)
        elif dtype == torch.int32:  # packed u32 words travel as int32 bit patterns
            arr = np.ascontiguousarray(arr, dtype=np.uint32).view(np.int32)
        elif dtype == torch.int64:
            arr = np.ascontiguousarray(arr, dtype=np.int64)
        elif dtype == torch.float16:
            arr = np.ascontiguousarray(arr, dtype=np.float16)
        t = torch.from_numpy(arr)
    if t.dtype != dtype:
        if dtype == torch.int32 and t.dtype == torch.uint32:
            t = t.view(torch.int32)
        else:
            t = t.to(dtype)
    return t.to(dev, non_blocking=False).contiguous()


def words_np(t):
    """int32 device words -> numpy uint32."""
    return t.cpu().numpy().view(np.uint32)


def _flag_tensor():
    return torch.zeros(1, dtype=torch.int32, device=_lib.device())


# -- device-level ---------------------------------------------------------------

def quantize_groups_dev(x, bits, group_size):
    """x: 2D CUDA f64 (or f16) tensor -> (codes u8 [R, C], scales f64, zero_points f64, flag)."""
    _check_bits(bits)
    if group_size < 1:
        raise ValueError("group_size must be >= 1")
    if x.ndim != 2:
        raise ValueError("expected a 2D matrix")
    rows, cols = x.shape
    gpr = -(-cols // group_size) if cols else 0
    dev = x.device
    codes = torch.zeros((rows, cols), dtype=torch.uint8, device=dev)
    scales = torch.zeros(rows * gpr, dtype=torch.float64, device=dev)
    zps = torch.zeros(rows * gpr, dtype=torch.float64, device=dev)
    flag = _flag_tensor()
    fn = "ckv_quantize_groups_f16" if x.dtype == torch.float16 else "ckv_quantize_groups_f64"
    _lib.call(fn, _lib.ptr(x), rows, cols, bits, group_size, _lib.ptr(codes), _lib.ptr(scales),
              _lib.ptr(zps), _lib.ptr(flag), _lib.stream())
    return codes, scales, zps, flag


def pack_codes_dev(codes, bits):
    _check_bits(bits)
    codes = codes.reshape(-1)
    n = codes.numel()
    n_words = -(-n * bits // 32)
    packed = torch.zeros(n_words, dtype=torch.int32, device=codes.device)
    _lib.call("ckv_pack_codes", _lib.ptr(codes), n, bits, _lib.ptr(packed), _lib.stream())
    return packed


def unpack_codes_dev(packed, bits, count):
    _check_bits(bits)
    out = torch.zeros(count, dtype=torch.uint8, device=packed.device)
    _lib.call("ckv_unpack_codes", _lib.ptr(packed), packed.numel(), bits, count, _lib.ptr(out),
              _lib.stream())
    return out


def dequantize_codes_dev(packed, scales, zero_points, rows, cols, bits, group_size):
    _check_bits(bits)
    out = torch.zeros((rows, cols), dtype=torch.float64, device=packed.device)
    _lib.call("ckv_dequantize_codes_f64", _lib.ptr(packed), packed.numel(), _lib.ptr(scales),
              _lib.ptr(zero_points), rows, cols, bits, group_size, _lib.ptr(out), _lib.stream())
    return out


def matmul_packed_dev(a, packed, scales, zero_points, rows, cols, bits, group_size, transpose,
                      out=None, accumulate=False):
    _check_bits(bits)
    if a.ndim != 2:
        raise ValueError("expected a 2D left factor")
    inner = cols if transpose else rows
    if a.shape[1] != inner:
        raise ValueError(f"inner dimension mismatch: a has {a.shape[1]}, block provides {inner}")
    m = a.shape[0]
    n_out = rows if transpose else cols
    if out is None:
        out = torch.zeros((m, n_out), dtype=torch.float64, device=a.device)
    _lib.call("ckv_matmul_packed_f64", _lib.ptr(a), m, a.shape[1], a.stride(0), _lib.ptr(packed),
              packed.numel(), _lib.ptr(scales), _lib.ptr(zero_points), rows, cols, bits, group_size,
              int(bool(transpose)), _lib.ptr(out), out.stride(0), int(bool(accumulate)),
              _lib.stream())
    return out


def matmul_dev(a, b, transpose, out=None, accumulate=False):
    """Dense f64 product on the device: a @ b.T (transpose) or a @ b."""
    m, k = a.shape
    n = b.shape[0] if transpose else b.shape[1]
    if (b.shape[1] if transpose else b.shape[0]) != k:
        raise ValueError("inner dimension mismatch")
    if out is None:
        out = torch.zeros((m, n), dtype=torch.float64, device=a.device)
    _lib.call("ckv_matmul_f64", _lib.ptr(a), m, k, a.stride(0), _lib.ptr(b), n, b.stride(0),
              int(bool(transpose)), _lib.ptr(out), out.stride(0), int(bool(accumulate)), _lib.stream())
    return out


# -- reference-shaped (numpy in / numpy out) ----------------------------------------

def quantize_groups(x, bits, group_size):
    """_numpy.py:27-67 / _core.pyx:27-79 on the GPU; bit-identical codes and metadata."""
    _check_bits(bits)
    if group_size < 1:
        raise ValueError("group_size must be >= 1")
    xd = to_dev(x, torch.float64)
    if xd.ndim != 2:
        raise ValueError("expected a 2D matrix")
    codes, scales, zps, _ = quantize_groups_dev(xd, bits, group_size)
    return codes.cpu().numpy(), scales.cpu().numpy(), zps.cpu().numpy()


def pack_codes(codes, bits):
    """_numpy.py:70-86."""
    _check_bits(bits)
    return words_np(pack_codes_dev(to_dev(codes, torch.uint8).reshape(-1), bits))


def unpack_codes(packed, bits, count):
    """_numpy.py:89-99."""
    _check_bits(bits)
    p = to_dev(packed, torch.int32)
    if count > p.numel() * (32 // bits):
        raise ValueError("count exceeds packed capacity")
    return unpack_codes_dev(p, bits, count).cpu().numpy()


def dequantize_codes(packed, scales, zero_points, rows, cols, bits, group_size):
    """_numpy.py:102-112."""
    return dequantize_codes_dev(to_dev(packed, torch.int32), to_dev(scales, torch.float64),
                                to_dev(zero_points, torch.float64), rows, cols, bits,
                                group_size).cpu().numpy()


def matmul_packed(a, packed, scales, zero_points, rows, cols, bits, group_size, transpose):
    """_numpy.py:115-125: a @ dequantized (or its transpose), float64 accumulation."""
    a_np = np.asarray(a) if not isinstance(a, torch.Tensor) else a
    if a_np.ndim != 2:
        raise ValueError("expected a 2D left factor")
    return matmul_packed_dev(to_dev(a, torch.float64), to_dev(packed, torch.int32),
                             to_dev(scales, torch.float64), to_dev(zero_points, torch.float64),
                             rows, cols, bits, group_size, transpose).cpu().numpy()


__all__ = [
    "ALLOWED_BITS",
    "BACKEND",
    "dequantize_codes",
    "matmul_packed",
    "pack_codes",
    "quantize_groups",
    "unpack_codes",
]
