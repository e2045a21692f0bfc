"""TPK1 container -> device loader.

The reference's container (`container.py`) is a flat file of tensors:

    header:  magic b"TPK1" | version u32 = 1 | tensor_count u32            (container.py:1-17)
    record:  name_len u16 | name | dtype u8 | ndims u8 | dims u64 * ndims | data_len u64
             | zero padding to a 32-byte file offset | data                 (container.py:167-182)
    data:    F32/F16 raw; TQ2/TQ1 per 256-element block: payload then the binary16 scale
             (PackedMatrix.to_block_bytes, linear.py:73-82)

``read_container`` restates the reference parser with the same validation and the same error
types (container.py:34-57, 198-242), so callers written against the reference behave the
same.  ``load_to_device`` is the B200 addition: each quantized record's bytes go to the GPU
as they are and one kernel (``tr_repack_records``) de-interleaves payload and scale and
writes the T16 tiles; F16/F32 tensors become device tensors.  There is no host-side
unpacking and no CPU fallback.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .blocks import BLOCK_ELEMENTS, DType
from .device import TernaryWeight

MAGIC = b"TPK1"
VERSION = 1
DATA_ALIGN = 32

_HEADER = struct.Struct("<4sII")
_NAME_LEN = struct.Struct("<H")
_REC_FIXED = struct.Struct("<BB")
_U64 = struct.Struct("<Q")
_NUMPY_DTYPES = {DType.F32: np.dtype("<f4"), DType.F16: np.dtype("<f2")}


class ContainerError(Exception):
    """Base for container format failures (container.py:34-35)."""


class BadMagicError(ContainerError):
    pass


class VersionMismatchError(ContainerError):
    pass


class TruncatedError(ContainerError):
    pass


class SizeMismatchError(ContainerError):
    pass


def rows_cols(dims: Sequence[int]) -> tuple[int, int]:
    """Leading dims collapse into rows; the last dim is cols (container.py:60-65)."""
    rows = 1
    for d in dims[:-1]:
        rows *= d
    return rows, dims[-1]


def expected_data_len(dims: Sequence[int], dtype: DType) -> int:
    """Data-section bytes for a tensor of this shape and format (container.py:68-82)."""
    if len(dims) == 0 or any(d < 1 for d in dims):
        raise ValueError(f"dims must be positive, got {tuple(dims)}")
    if dtype.is_quantized:
        rows, cols = rows_cols(dims)
        return rows * (-(-cols // BLOCK_ELEMENTS)) * dtype.block_bytes
    count = 1
    for d in dims:
        count *= d
    return count * (4 if dtype is DType.F32 else 2)


@dataclass(frozen=True)
class TensorRecord:
    """One named tensor as stored (container.py:90-146); ``data`` is a zero-copy view."""

    name: str
    dtype: DType
    dims: tuple
    data: memoryview


class _Reader:
    def __init__(self, raw: memoryview):
        self.raw = raw
        self.pos = 0

    def take(self, n: int, what: str) -> memoryview:
        if self.pos + n > len(self.raw):
            raise TruncatedError(f"file ends inside {what}: need {n} bytes at offset {self.pos}, "
                                 f"have {len(self.raw) - self.pos}")
        chunk = self.raw[self.pos:self.pos + n]
        self.pos += n
        return chunk


def parse_container(raw: bytes) -> list[TensorRecord]:
    """Parse TPK1 bytes, validating exactly as the reference's read_container (container.py:198-242)."""
    rd = _Reader(memoryview(raw))
    magic, version, count = _HEADER.unpack(rd.take(_HEADER.size, "header"))
    if magic != MAGIC:
        raise BadMagicError(f"not a TPK1 file (magic {bytes(magic)!r})")
    if version != VERSION:
        raise VersionMismatchError(f"unsupported container version {version}")
    records = []
    for i in range(count):
        (name_len,) = _NAME_LEN.unpack(rd.take(_NAME_LEN.size, f"tensor {i} name length"))
        try:
            name = bytes(rd.take(name_len, f"tensor {i} name")).decode("utf-8")
        except UnicodeDecodeError as exc:
            raise ContainerError(f"tensor {i}: name is not valid UTF-8") from exc
        tag, ndims = _REC_FIXED.unpack(rd.take(_REC_FIXED.size, f"tensor {name!r} header"))
        try:
            dtype = DType(tag)
        except ValueError:
            raise ContainerError(f"tensor {name!r}: unknown dtype tag {tag}") from None
        if ndims == 0:
            raise ContainerError(f"tensor {name!r}: ndims must be >= 1")
        dims = tuple(_U64.unpack(rd.take(_U64.size, f"tensor {name!r} dims"))[0] for _ in range(ndims))
        (data_len,) = _U64.unpack(rd.take(_U64.size, f"tensor {name!r} data length"))
        rd.take(-rd.pos % DATA_ALIGN, f"tensor {name!r} alignment padding")
        data = rd.take(data_len, f"tensor {name!r} data")
        if any(d < 1 for d in dims):
            raise ContainerError(f"tensor {name!r}: dims {dims} must be positive")
        expected = expected_data_len(dims, dtype)
        if data_len != expected:
            raise SizeMismatchError(f"tensor {name!r}: data_len {data_len} but dims {dims} x {dtype.name} "
                                    f"require {expected}")
        records.append(TensorRecord(name=name, dtype=dtype, dims=dims, data=data))
    if rd.pos != len(rd.raw):
        raise ContainerError(f"{len(rd.raw) - rd.pos} trailing bytes after the last tensor")
    return records


def read_container(path) -> list[TensorRecord]:
    """Parse a TPK1 file (the reference's read_container contract)."""
    with open(path, "rb") as fh:
        return parse_container(fh.read())


def record_to_device(rec: TensorRecord, device="cuda"):
    """One record on the GPU: TQ2/TQ1 -> TernaryWeight (leading dims collapsed into rows);
    F16/F32 -> a device tensor in the stored shape."""
    dev = torch.device(device)
    if not rec.dtype.is_quantized:
        arr = np.frombuffer(rec.data, dtype=_NUMPY_DTYPES[rec.dtype]).reshape(rec.dims)
        return torch.from_numpy(arr.copy()).to(dev)
    rows, cols = rows_cols(rec.dims)
    records = torch.frombuffer(bytearray(rec.data), dtype=torch.uint8).to(dev)   # raw [payload | scale] records
    nbytes = _lib.lib().tr_layout_bytes(int(rec.dtype), rows, cols)
    data = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.call("tr_repack_records", int(rec.dtype), records.data_ptr(), rows, cols, data.data_ptr(),
                  _lib.stream_handle())
    nb, pb = -(-cols // BLOCK_ELEMENTS), rec.dtype.payload_bytes
    sbytes = records.view(rows, nb, pb + 2)[:, :, pb:]   # the scales' two bytes, in place
    s = (sbytes[..., 0].to(torch.int32) | (sbytes[..., 1].to(torch.int32) << 8))
    uniform = bool((s == s[:, :1]).all())
    return TernaryWeight(data, rows, cols, rec.dtype, uniform_scale=uniform)


def load_to_device(path, device="cuda") -> dict:
    """Every tensor of a TPK1 file on the GPU, by name (``record_to_device``)."""
    return {rec.name: record_to_device(rec, device) for rec in read_container(path)}
