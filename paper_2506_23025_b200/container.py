"""TPK1 container -> device loader.

File format (the reference's writer, container.py:1-17, 167-196): little-endian
``b"TPK1" | u32 version (1) | u32 count`` then ``count`` records of
``u16 name length | UTF-8 name | u8 dtype tag | u8 ndims | u64 dims[ndims] | u64 data length |
zero fill to a 32-byte file offset | data``.  Quantized data is rows x ceil(cols/256) blocks of
``payload | binary16 scale`` (PackedMatrix.to_block_bytes, linear.py:73-82).

The B200 part is ``record_to_device``: a quantized record's bytes go to the GPU untouched and
one kernel (``tr_repack_records``) splits payload from scale and writes the T16 tiles; F16 /
F32 tensors become device tensors.  It takes any record with ``name / dtype / dims / data``
(this module's ``TensorRecord`` or the reference's own ``tritpack.container.TensorRecord``).

``parse_container`` is a scanner of our own for the same byte format.  It raises the error
classes reference callers already catch (container.py:34-57: bad magic, version, truncation,
size mismatch, all ``ContainerError``), so code written against the reference reader keeps
its error handling.
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


class ContainerError(Exception):
    """Any malformed TPK1 input."""


class BadMagicError(ContainerError):
    """The first four bytes are not TPK1."""


class VersionMismatchError(ContainerError):
    """A version other than 1."""


class TruncatedError(ContainerError):
    """The input ends inside a field."""


class SizeMismatchError(ContainerError):
    """data length disagrees with dims x dtype."""


def rows_cols(dims: Sequence[int]) -> tuple[int, int]:
    """(product of the leading dims, last dim): how a quantized tensor is laid out as a matrix."""
    return int(np.prod(dims[:-1], dtype=np.int64)) if len(dims) > 1 else 1, int(dims[-1])


def expected_data_len(dims: Sequence[int], dtype: DType) -> int:
    """Bytes the data section of a `dims` tensor in `dtype` occupies."""
    if not dims or min(dims) < 1:
        raise ValueError(f"dims must be positive, got {tuple(dims)}")
    if dtype.is_quantized:
        rows, cols = rows_cols(dims)
        return rows * (-(-cols // BLOCK_ELEMENTS)) * dtype.block_bytes
    return int(np.prod(dims, dtype=np.int64)) * (4 if dtype is DType.F32 else 2)


@dataclass(frozen=True)
class TensorRecord:
    """One stored tensor; ``data`` is a zero-copy slice of the file bytes."""

    name: str
    dtype: DType
    dims: tuple
    data: memoryview


def parse_container(raw: bytes) -> list[TensorRecord]:
    """Scan TPK1 bytes into records, validating every field before it is used."""
    buf = memoryview(raw)
    end = len(buf)
    off = 0

    def take(n: int, field: str) -> memoryview:
        nonlocal off
        if n > end - off:
            raise TruncatedError(f"truncated at byte {off}: {field} needs {n} bytes, {end - off} left")
        piece = buf[off:off + n]
        off += n
        return piece

    def u(nbytes: int, field: str) -> int:
        return int.from_bytes(take(nbytes, field), "little")

    if bytes(take(4, "magic")) != MAGIC:
        raise BadMagicError(f"bad magic {bytes(buf[:4])!r}, expected {MAGIC!r}")
    version = u(4, "version")
    if version != VERSION:
        raise VersionMismatchError(f"container version {version} is not {VERSION}")
    out = []
    for idx in range(u(4, "tensor count")):
        raw_name = bytes(take(u(2, f"record {idx} name length"), f"record {idx} name"))
        try:
            name = raw_name.decode("utf-8")
        except UnicodeDecodeError as exc:
            raise ContainerError(f"record {idx}: name bytes are not UTF-8") from exc
        tag, ndims = u(1, f"{name}: dtype tag"), u(1, f"{name}: ndims")
        if tag not in {t.value for t in DType}:
            raise ContainerError(f"{name}: unknown dtype tag {tag}")
        if ndims < 1:
            raise ContainerError(f"{name}: ndims is 0 (need at least one dimension)")
        dims = struct.unpack(f"<{ndims}Q", take(8 * ndims, f"{name}: dims"))
        nbytes = u(8, f"{name}: data length")
        take((-off) % DATA_ALIGN, f"{name}: padding")
        data = take(nbytes, f"{name}: data")
        if min(dims) < 1:
            raise ContainerError(f"{name}: every dimension must be positive, got {dims}")
        dtype = DType(tag)
        want = expected_data_len(dims, dtype)
        if nbytes != want:
            raise SizeMismatchError(f"{name}: {nbytes} data bytes stored, {dtype.name} {dims} needs {want}")
        out.append(TensorRecord(name, dtype, tuple(dims), data))
    if off != end:
        raise ContainerError(f"{end - off} trailing bytes after record {len(out) - 1}")
    return out


def read_container(path) -> list[TensorRecord]:
    """``parse_container`` of a file's bytes."""
    with open(path, "rb") as fh:
        return parse_container(fh.read())


def record_to_device(rec: TensorRecord, device="cuda"):
    """One record on the GPU: TQ2/TQ1 -> TernaryWeight (leading dims collapsed into rows);
    F16/F32 -> a device tensor in the stored shape."""
    dev = torch.device(device)
    rec_dtype = DType(int(rec.dtype))   # (the reference's DType has the same tags, blocks.py:45-52)
    rec = TensorRecord(rec.name, rec_dtype, tuple(int(d) for d in rec.dims), memoryview(rec.data))
    if not rec.dtype.is_quantized:
        arr = np.frombuffer(rec.data, dtype="<f4" if rec.dtype is DType.F32 else "<f2").reshape(rec.dims)
        return torch.from_numpy(arr.copy()).to(dev)
    rows, cols = rows_cols(rec.dims)
    records = torch.frombuffer(bytearray(rec.data), dtype=torch.uint8).to(dev)   # raw [payload | scale] records
    nbytes = _lib.lib().tr_layout_bytes(int(rec.dtype), rows, cols)
    data = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.call("tr_repack_records", int(rec.dtype), records.data_ptr(), rows, cols, data.data_ptr(),
                  data.numel(), _lib.stream_handle())
    nb, pb = -(-cols // BLOCK_ELEMENTS), rec.dtype.payload_bytes
    sbytes = records.view(rows, nb, pb + 2)[:, :, pb:]   # the scales' two bytes, in place
    s = (sbytes[..., 0].to(torch.int32) | (sbytes[..., 1].to(torch.int32) << 8))
    uniform = bool((s == s[:, :1]).all())
    return TernaryWeight(data, rows, cols, rec.dtype, uniform_scale=uniform)


def load_to_device(path, device="cuda") -> dict:
    """Every tensor of a TPK1 file on the GPU, by name (``record_to_device``)."""
    return {rec.name: record_to_device(rec, device) for rec in read_container(path)}
