"""The reference kernel-module surface, executed on the B200.

Drop-in for tritpack._kernels / tritpack._kernels_py (reference
_kernels.pyx:23-227, _kernels_py.py:46-171): same names, argument meaning,
ownership (pack/unpack/quantize/dequantize allocate and return numpy arrays;
gemm_* write out[:, row0:row1] in place) and bit-identical results.  Each call
copies its numpy inputs to the device, runs the CUDA kernel through the
libtritrun C-ABI and copies the result back -- this module is the parity /
integration surface; the fast path is paper_2506_23025_b200.device.linear().

Frozen weights stay resident: ``PackedMatrix`` freezes its payload and fp32 scale
arrays (reference linear.py:58-62), so gemm_tq2 / gemm_tq1 upload a read-only
(payload, scales) pair once and reuse the device copy for every later call and
every row range ``linear.gemm(threads=N)`` shards it into (linear.py:155-166);
each call then moves only its activations in and its rows out.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np
import torch

from . import _lib


def _writable(a):
    """C-contiguous and writable (torch.from_numpy warns on read-only views, e.g. np.frombuffer)."""
    a = np.ascontiguousarray(a)
    return a if a.flags.writeable else a.copy()


NAME = "cuda"


def _dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(_writable(a)).cuda()


def _run(name: str, *args) -> None:
    _lib.call(name, *args, _lib.stream_handle())


def pack_base4(digits):
    d = _dev(np.asarray(digits, np.uint8).reshape(-1))
    out = torch.empty(d.numel() // 4, dtype=torch.uint8, device="cuda")
    _run("tr_pack_base4", d.data_ptr(), out.data_ptr(), out.numel())
    return out.cpu().numpy()


def unpack_base4(words):
    w = _dev(np.asarray(words, np.uint8).reshape(-1))
    out = torch.empty(4 * w.numel(), dtype=torch.uint8, device="cuda")
    _run("tr_unpack_base4", w.data_ptr(), out.data_ptr(), w.numel())
    return out.cpu().numpy()


def encode_base3(digits):
    d = _dev(np.asarray(digits, np.uint8).reshape(-1))
    out = torch.empty(d.numel() // 5, dtype=torch.uint8, device="cuda")
    _run("tr_encode_base3", d.data_ptr(), out.data_ptr(), out.numel())
    return out.cpu().numpy()


def decode_base3(codes):
    c = _dev(np.asarray(codes, np.uint8).reshape(-1))
    out = torch.empty(5 * c.numel(), dtype=torch.uint8, device="cuda")
    _run("tr_decode_base3", c.data_ptr(), out.data_ptr(), c.numel())
    return out.cpu().numpy()


def quantize_blocks(values):
    v = _dev(np.asarray(values, np.float32).reshape(-1, 256))
    nb = v.shape[0]
    digits = torch.empty((nb, 256), dtype=torch.uint8, device="cuda")
    scales = torch.empty(nb, dtype=torch.float32, device="cuda")
    _run("tr_quantize_blocks", v.data_ptr(), digits.data_ptr(), scales.data_ptr(), nb)
    return digits.cpu().numpy(), scales.cpu().numpy()


def dequantize_blocks(digits, scales):
    d = _dev(np.asarray(digits, np.uint8).reshape(-1, 256))
    s = _dev(np.asarray(scales, np.float32).reshape(-1))
    out = torch.empty(d.shape, dtype=torch.float32, device="cuda")
    _run("tr_dequantize_blocks", d.data_ptr(), s.data_ptr(), out.data_ptr(), d.shape[0])
    return out.cpu().numpy()


_RESIDENT: dict = {}              # id(payload) -> (weakref payload, weakref scales, device payload, device scales)
_RESIDENT_LOCK = threading.Lock()


def _frozen(a) -> bool:
    return isinstance(a, np.ndarray) and not a.flags.writeable and a.flags.c_contiguous


def _weights(payload, scales):
    """Device copies of (payload, fp32 scales); cached while both arrays are alive and read-only."""
    if not (_frozen(payload) and _frozen(scales) and scales.dtype == np.float32):
        return _dev(payload), _dev(np.asarray(scales, np.float32))
    key = id(payload)
    with _RESIDENT_LOCK:
        hit = _RESIDENT.get(key)
        if hit is not None and hit[0]() is payload and hit[1]() is scales:
            return hit[2], hit[3]
        dp, ds = _dev(payload), _dev(scales)
        try:
            wp = weakref.ref(payload, lambda _r, k=key: _RESIDENT.pop(k, None))
            ws = weakref.ref(scales)
        except TypeError:   # (views of foreign buffers may not take weak references)
            return dp, ds
        _RESIDENT[key] = (wp, ws, dp, ds)
        return dp, ds


def _gemm(fmt: int, payload, scales, x, out, row0: int, row1: int) -> None:
    rows, nb = scales.shape
    batch = x.shape[0]
    if row1 <= row0 or batch == 0:
        return
    p, s = _weights(payload, scales)
    xd = _dev(np.asarray(x, np.float32))
    o = torch.empty((batch, rows), dtype=torch.float32, device="cuda")
    _run("tr_gemm_exact", fmt, p.data_ptr(), s.data_ptr(), xd.data_ptr(), o.data_ptr(), rows, nb, batch,
         int(row0), int(row1))
    out[:, row0:row1] = o[:, row0:row1].cpu().numpy()


def gemm_tq2(payload, scales, x, out, row0, row1):
    """TQ2 rows [row0, row1) x activation batch -> out (bit-identical to _kernels.pyx:171-197)."""
    _gemm(_lib.FMT_TQ2, payload, scales, x, out, row0, row1)


def gemm_tq1(payload, scales, x, out, row0, row1):
    """TQ1 rows [row0, row1) x activation batch -> out (bit-identical to _kernels.pyx:200-227)."""
    _gemm(_lib.FMT_TQ1, payload, scales, x, out, row0, row1)
