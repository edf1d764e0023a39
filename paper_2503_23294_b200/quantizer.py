"""Per-group asymmetric min-max quantization to 2 or 4 bits — drop-in for
``chunkkv.quantizer`` (quantizer.py:1-171), computed on the GPU.

A QuantizedBlock keeps the reference's host-visible fields (numpy ``packed``,
``scales``, ``zero_points``) and lazily mirrors them on the device so repeated fqm
calls do not re-upload.  Wire format identical to quantizer.py:126-171.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _lib, kernels

_HEADER = struct.Struct("<4I")


class QuantizedBlock:
    """Bit-packed integer matrix with per-group scale/zero-point metadata (quantizer.py:20-57)."""

    __slots__ = ("rows", "cols", "bitwidth", "group_size", "packed", "scales", "zero_points", "_dev")

    def __init__(self, rows, cols, bitwidth, group_size, packed, scales, zero_points):
        object.__setattr__(self, "rows", int(rows))
        object.__setattr__(self, "cols", int(cols))
        object.__setattr__(self, "bitwidth", int(bitwidth))
        object.__setattr__(self, "group_size", int(group_size))
        object.__setattr__(self, "packed", np.asarray(packed))
        object.__setattr__(self, "scales", np.asarray(scales))
        object.__setattr__(self, "zero_points", np.asarray(zero_points))
        object.__setattr__(self, "_dev", None)
        # quantizer.py:38-49
        if self.bitwidth not in kernels.ALLOWED_BITS:
            raise ValueError(f"bitwidth must be one of {kernels.ALLOWED_BITS}")
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.rows < 0 or self.cols < 0:
            raise ValueError("negative shape")
        n_words = -(-self.rows * self.cols * self.bitwidth // 32)
        if self.packed.shape != (n_words,):
            raise ValueError("packed length does not match shape")
        if self.scales.shape != (self.n_groups,) or self.zero_points.shape != (self.n_groups,):
            raise ValueError("metadata length does not match group count")

    def __setattr__(self, name, value):  # frozen, like the reference dataclass
        raise AttributeError("QuantizedBlock is immutable")

    def __eq__(self, other):
        if not isinstance(other, QuantizedBlock):
            return NotImplemented
        return serialize_block(self) == serialize_block(other)

    __hash__ = None

    def __repr__(self):
        return (f"QuantizedBlock(rows={self.rows}, cols={self.cols}, bitwidth={self.bitwidth}, "
                f"group_size={self.group_size})")

    @property
    def n_groups(self) -> int:
        return self.rows * (-(-self.cols // self.group_size))

    def storage_bytes(self) -> int:
        """Bytes held by packed words plus per-group metadata (quantizer.py:55-57)."""
        return self.packed.nbytes + self.scales.nbytes + self.zero_points.nbytes

    def device_tensors(self):
        """(packed int32, scales f64, zero_points f64) on the GPU, uploaded once."""
        if self._dev is None:
            object.__setattr__(self, "_dev", (
                kernels.to_dev(self.packed, torch.int32),
                kernels.to_dev(self.scales, torch.float64),
                kernels.to_dev(self.zero_points, torch.float64),
            ))
        return self._dev

    @classmethod
    def _from_device(cls, rows, cols, bitwidth, group_size, packed_d, scales_d, zps_d):
        blk = cls(rows, cols, bitwidth, group_size, kernels.words_np(packed_d),
                  scales_d.cpu().numpy(), zps_d.cpu().numpy())
        object.__setattr__(blk, "_dev", (packed_d, scales_d, zps_d))
        return blk


def quantize_dev(x, bitwidth, group_size=32) -> QuantizedBlock:
    """Quantize a 2D CUDA tensor (f64 or f16).  Raises ValueError on non-finite input."""
    if x.ndim != 2:
        raise ValueError("expected a 2D matrix")
    if bitwidth not in kernels.ALLOWED_BITS:
        raise ValueError(f"bitwidth must be one of {kernels.ALLOWED_BITS}, got {bitwidth}")
    if group_size < 1:
        raise ValueError("group_size must be >= 1")
    codes, scales, zps, flag = kernels.quantize_groups_dev(x, bitwidth, group_size)
    if x.numel() and int(flag.item()) & _lib.FLAG_NONFINITE:  # quantizer.py:71-72
        raise ValueError("matrix contains non-finite values")
    packed = kernels.pack_codes_dev(codes, bitwidth)
    return QuantizedBlock._from_device(x.shape[0], x.shape[1], bitwidth, group_size, packed, scales, zps)


def quantize(matrix, bitwidth, group_size=32) -> QuantizedBlock:
    """quantizer.py:60-83: scale = (M - m)/(2^b - 1), zero_point = m, code = round-half-up."""
    if not isinstance(matrix, torch.Tensor):
        arr = np.asarray(matrix, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("expected a 2D matrix")
    x = kernels.to_dev(matrix, torch.float64 if not (isinstance(matrix, torch.Tensor)
                                                     and matrix.dtype == torch.float16) else torch.float16)
    return quantize_dev(x, bitwidth, group_size)


def dequantize_dev(block: QuantizedBlock):
    p, s, z = block.device_tensors()
    return kernels.dequantize_codes_dev(p, s, z, block.rows, block.cols, block.bitwidth, block.group_size)


def dequantize(block: QuantizedBlock) -> np.ndarray:
    """quantizer.py:86-96."""
    return dequantize_dev(block).cpu().numpy()


def fqm_dev(a, block: QuantizedBlock, transpose_block=False, out=None, accumulate=False):
    if a.ndim != 2:
        raise ValueError("expected a 2D left factor")
    inner = block.cols if transpose_block else block.rows
    if a.shape[1] != inner:
        raise ValueError(f"inner dimension mismatch: a has {a.shape[1]}, block provides {inner}")
    p, s, z = block.device_tensors()
    return kernels.matmul_packed_dev(a, p, s, z, block.rows, block.cols, block.bitwidth,
                                     block.group_size, bool(transpose_block), out=out,
                                     accumulate=accumulate)


def fqm(a, block: QuantizedBlock, transpose_block=False) -> np.ndarray:
    """quantizer.py:99-123: a @ dequantize(block) (or its transpose), f64 accumulation."""
    if not isinstance(a, torch.Tensor):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("expected a 2D left factor")
    return fqm_dev(kernels.to_dev(a, torch.float64), block, transpose_block).cpu().numpy()


def serialize_block(block: QuantizedBlock) -> bytes:
    """quantizer.py:126-138: u32 header, f64 scales, f64 zero_points, u32 packed words (LE)."""
    header = _HEADER.pack(block.rows, block.cols, block.bitwidth, block.group_size)
    return b"".join((
        header,
        np.ascontiguousarray(block.scales, dtype="<f8").tobytes(),
        np.ascontiguousarray(block.zero_points, dtype="<f8").tobytes(),
        np.ascontiguousarray(block.packed, dtype="<u4").tobytes(),
    ))


def deserialize_block(buf, offset=0):
    """quantizer.py:141-171."""
    end = offset + _HEADER.size
    if end > len(buf):
        raise ValueError("truncated block header")
    rows, cols, bitwidth, group_size = _HEADER.unpack_from(buf, offset)
    if bitwidth not in kernels.ALLOWED_BITS:
        raise ValueError(f"bad bitwidth {bitwidth} in block header")
    if group_size < 1:
        raise ValueError("bad group_size in block header")
    n_groups = rows * (-(-cols // group_size))
    n_words = -(-rows * cols * bitwidth // 32)
    need = n_groups * 16 + n_words * 4
    if end + need > len(buf):
        raise ValueError("truncated block body")
    scales = np.frombuffer(buf, dtype="<f8", count=n_groups, offset=end).astype(np.float64)
    end += n_groups * 8
    zps = np.frombuffer(buf, dtype="<f8", count=n_groups, offset=end).astype(np.float64)
    end += n_groups * 8
    packed = np.frombuffer(buf, dtype="<u4", count=n_words, offset=end).astype(np.uint32)
    end += n_words * 4
    return QuantizedBlock(rows, cols, bitwidth, group_size, packed, scales, zps), end
