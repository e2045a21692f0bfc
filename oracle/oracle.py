"""CPU oracle for the TriRun hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline.  The product package (paper_2506_23025_b200) never
imports it; its CUDA path fails loudly when the extension is missing.

Contents (each cites the reference code it restates; reference root is
/root/reference/pkg/src/tritpack/):

* ``kernels`` -- the reference kernel-module surface (_kernels_py.py:46-171,
  _kernels.pyx:23-227) backed by oracle/liboracle.so, a plain-C restatement
  (oracle/tritpack_oracle.c, -O3 -ffp-contract=off like setup.py:21).
* ``pack_matrix`` / ``dequantize_matrix`` / ``gemv_reference`` / ``gemm`` --
  numpy restatements of linear.py:98-208 and blocks.py:142-177 glue.
* ``ref_kernels()`` -- the reference's *own* compiled kernels, built from the
  reference sources into oracle/_ref/ by ``make -C oracle ref``; used to pin
  the restatement and as the ``kind: "reference"`` CPU baseline.

Parity is pinned: tests/test_oracle.py checks this module bit-for-bit against
tests/golden/*.npz (made by importing the reference, tests/golden/make_golden.py)
and against oracle/_ref on random inputs.
"""

from __future__ import annotations

import ctypes
import importlib.util
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BLOCK = 256
PAYLOAD_BYTES = {2: 64, 3: 52}   # DType.TQ2 / DType.TQ1 (blocks.py:45-76)
TQ2, TQ1 = 2, 3
_TQ1_PAD = 4                     # blocks.py:38 -- tail code holds 1 real trit + 4 pads

_lib = None


def build() -> None:
    """Compile oracle/liboracle.so (and oracle/_ref when the reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if os.path.exists("/root/reference/pkg/src/tritpack/_kernels.pyx"):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"PY={sys.executable}"], check=True)


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        p, i64 = ctypes.c_void_p, ctypes.c_int64
        for name in ("orc_pack_base4", "orc_unpack_base4", "orc_encode_base3", "orc_decode_base3"):
            getattr(lib, name).argtypes = [p, p, i64]
        lib.orc_quantize_blocks.argtypes = [p, p, p, i64]
        lib.orc_dequantize_blocks.argtypes = [p, p, p, i64]
        for name in ("orc_gemm_tq2", "orc_gemm_tq1"):
            getattr(lib, name).argtypes = [p, p, p, p, i64, i64, i64, i64, i64, p]
        lib.orc_gemv_f64.argtypes = [ctypes.c_int, p, p, p, p, i64, i64, i64, i64, i64]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# kernel-module surface (reference _kernels_py.py:46-171)
# ---------------------------------------------------------------------------

def pack_base4(digits):
    d = _c(digits, np.uint8).reshape(-1)
    out = np.empty(d.size // 4, np.uint8)
    _load().orc_pack_base4(_ptr(d), _ptr(out), out.size)
    return out


def unpack_base4(words):
    w = _c(words, np.uint8).reshape(-1)
    out = np.empty(4 * w.size, np.uint8)
    _load().orc_unpack_base4(_ptr(w), _ptr(out), w.size)
    return out


def encode_base3(digits):
    d = _c(digits, np.uint8).reshape(-1)
    out = np.empty(d.size // 5, np.uint8)
    _load().orc_encode_base3(_ptr(d), _ptr(out), out.size)
    return out


def decode_base3(codes):
    c = _c(codes, np.uint8).reshape(-1)
    out = np.empty(5 * c.size, np.uint8)
    _load().orc_decode_base3(_ptr(c), _ptr(out), c.size)
    return out


def quantize_blocks(values):
    v = _c(values, np.float32).reshape(-1, BLOCK)
    nb = v.shape[0]
    digits = np.empty((nb, BLOCK), np.uint8)
    scales = np.empty(nb, np.float32)
    _load().orc_quantize_blocks(_ptr(v), _ptr(digits), _ptr(scales), nb)
    return digits, scales


def dequantize_blocks(digits, scales):
    d = _c(digits, np.uint8).reshape(-1, BLOCK)
    s = _c(scales, np.float32).reshape(-1)
    out = np.empty(d.shape, np.float32)
    _load().orc_dequantize_blocks(_ptr(d), _ptr(s), _ptr(out), d.shape[0])
    return out


def _gemm_kernel(name):
    def kernel(payload, scales, x, out, row0, row1):
        rows, nb = scales.shape
        scratch = np.empty(nb * BLOCK, np.uint8)
        getattr(_load(), name)(_ptr(payload), _ptr(scales), _ptr(x), _ptr(out), rows, nb,
                               x.shape[0], int(row0), int(row1), _ptr(scratch))
    return kernel


gemm_tq2 = _gemm_kernel("orc_gemm_tq2")
gemm_tq1 = _gemm_kernel("orc_gemm_tq1")

kernels = SimpleNamespace(
    NAME="oracle", pack_base4=pack_base4, unpack_base4=unpack_base4,
    encode_base3=encode_base3, decode_base3=decode_base3,
    quantize_blocks=quantize_blocks, dequantize_blocks=dequantize_blocks,
    gemm_tq2=gemm_tq2, gemm_tq1=gemm_tq1,
)


def ref_kernels():
    """The reference's own compiled kernel module from oracle/_ref (None if not built)."""
    ref_dir = os.path.join(HERE, "_ref")
    for fn in os.listdir(ref_dir) if os.path.isdir(ref_dir) else ():
        if fn.startswith("_kernels") and fn.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_kernels", os.path.join(ref_dir, fn))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    return None


# ---------------------------------------------------------------------------
# array-level glue (reference blocks.py:142-177, linear.py:98-208)
# ---------------------------------------------------------------------------

def quantize_rows(values, fmt, kern=kernels):
    """blocks.py:142-161: quantize (nb,256) f32 -> (payload u8 (nb,pb), scales <f2 (nb,))."""
    digits, scales = kern.quantize_blocks(_c(values, np.float32))
    nb = digits.shape[0]
    if fmt == TQ2:
        payload = np.asarray(kern.pack_base4(digits.reshape(-1))).reshape(nb, 64)
    else:
        padded = np.concatenate([digits, np.ones((nb, _TQ1_PAD), np.uint8)], axis=1)
        payload = np.asarray(kern.encode_base3(np.ascontiguousarray(padded).reshape(-1))).reshape(nb, 52)
    return payload, np.asarray(scales).astype("<f2")


def pack_matrix(W, fmt, kern=kernels):
    """linear.py:98-120 -> (payload u8 (rows,nb,pb), scales <f2 (rows,nb))."""
    W = np.asarray(W, dtype=np.float32)
    if W.ndim != 2 or W.size == 0 or not np.isfinite(W).all():
        raise ValueError("expected a finite non-empty 2-D matrix")
    rows, cols = W.shape
    nb = -(-cols // BLOCK)
    padded = np.zeros((rows, nb * BLOCK), np.float32)
    padded[:, :cols] = W
    payload, scales = quantize_rows(padded.reshape(rows * nb, BLOCK), fmt, kern)
    return payload.reshape(rows, nb, PAYLOAD_BYTES[fmt]), scales.reshape(rows, nb)


def dequantize_matrix(payload, scales, cols, fmt, dtype=np.float64):
    """linear.py:177-198: independent decoder (TQ1 by the canonical division formula)."""
    rows, nb = scales.shape
    if fmt == TQ2:
        shifts = np.arange(4, dtype=np.uint8) * 2
        digits = (payload.reshape(rows, -1)[:, :, None] >> shifts) & 3
        digits = digits.reshape(rows, nb * BLOCK)
    else:
        codes = payload.reshape(rows, -1).astype(np.uint32)
        xq = (codes * 243 + 13) >> 8
        powers = np.array([81, 27, 9, 3, 1], dtype=np.uint32)
        digits = (xq[:, :, None] // powers) % 3
        digits = digits.reshape(rows, nb, 260)[:, :, :BLOCK].reshape(rows, nb * BLOCK)
    signs = digits.astype(dtype) - 1
    dense = signs.reshape(rows, nb, BLOCK) * scales.astype(dtype)[:, :, None]
    return dense.reshape(rows, nb * BLOCK)[:, :cols]


def gemv_reference(payload, scales, cols, fmt, x):
    """linear.py:201-208: dequantize fully, dense float64 product."""
    return dequantize_matrix(payload, scales, cols, fmt) @ np.asarray(x, np.float64)


def gemv_reference_batch(payload, scales, cols, fmt, X, threads=None):
    """linear.py:177-208 at full size: float64 W x for every row of X (batch, cols) without the
    dense matrix (oracle/tritpack_oracle.c orc_gemv_f64), rows sharded over host threads."""
    pay = _c(payload, np.uint8)
    sc = _c(np.asarray(scales).view(np.uint16), np.uint16)
    X = _c(np.atleast_2d(X), np.float64)
    rows = sc.shape[0]
    out = np.empty((X.shape[0], rows), np.float64)
    threads = threads or min(32, os.cpu_count() or 1)
    chunk = -(-rows // threads)
    lib = _load()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        futs = [pool.submit(lib.orc_gemv_f64, int(fmt), _ptr(pay), _ptr(sc), _ptr(X), _ptr(out), rows, int(cols),
                            X.shape[0], lo, min(lo + chunk, rows)) for lo in range(0, rows, chunk)]
        for f in futs:
            f.result()
    return out


def gemm(payload, scales, cols, fmt, X, threads=1, kern=kernels):
    """linear.py:137-166 harness: zero-pad x to the block grid, shard rows over threads."""
    X = _c(X, np.float32)
    rows, nb = scales.shape
    batch = X.shape[0]
    xpad = np.zeros((batch, nb * BLOCK), np.float32)
    xpad[:, :cols] = X
    out = np.empty((batch, rows), np.float32)
    s32 = _c(scales, np.float32)
    pay = _c(payload, np.uint8)
    kernel = kern.gemm_tq2 if fmt == TQ2 else kern.gemm_tq1
    if threads == 1 or rows == 1:
        kernel(pay, s32, xpad, out, 0, rows)
        return out
    chunk = -(-rows // threads)
    ranges = [(lo, min(lo + chunk, rows)) for lo in range(0, rows, chunk)]
    with ThreadPoolExecutor(max_workers=len(ranges)) as pool:
        for f in [pool.submit(kernel, pay, s32, xpad, out, lo, hi) for lo, hi in ranges]:
            f.result()
    return out
