"""ctypes binding of libtritrun.so (C-ABI declared in include/tritrun.h).

The library is built in-tree (``make -C paper_2506_23025_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the shared library is
missing or a call fails, this module raises -- the product path never drops to
a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRITRUN_LIB") or os.path.join(HERE, "libtritrun.so")   # override: dev A/B builds

FMT_TQ2 = 2   # blocks.DType.TQ2 (reference blocks.py:49-52)
FMT_TQ1 = 3
ACT_F16 = 1
ACT_BF16 = 2
LINEAR_PDL = 1
LINEAR_UNIFORM_SCALE = 2
LINEAR_FORCE_UMMA = 4
LINEAR_FORCE_GEMV = 8
LINEAR_GEMV_F16 = 16
LINEAR_COSCHEDULE = 32
LINEAR_EPI_SWIGLU = 64
LINEAR_OUT_F32 = 128
LINEAR_FULL_SM = 1 << 28
PRE_ADD_RMSNORM = 1
PRE_SILU_MUL = 2

_lock = threading.Lock()
_lib = None

_c_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int

class TrChainLayer(ctypes.Structure):
    """include/tritrun.h TrChainLayer: one product of a tr_linear_chain (with its fused producer)."""

    _fields_ = [("w", ctypes.c_void_p), ("x", ctypes.c_void_p), ("y", ctypes.c_void_p), ("ldx", ctypes.c_int64),
                ("ldy", ctypes.c_int64), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("pre_op", ctypes.c_int32), ("flags", ctypes.c_int32), ("delta", ctypes.c_void_p),
                ("gamma", ctypes.c_void_p), ("x_out", ctypes.c_void_p), ("eps", ctypes.c_float)]


_SIGS = {
    "tr_last_error": ([], ctypes.c_char_p),
    "tr_version": ([], _int),
    "tr_pack_base4": ([_c_p, _c_p, _i64, _c_p], _int),
    "tr_unpack_base4": ([_c_p, _c_p, _i64, _c_p], _int),
    "tr_encode_base3": ([_c_p, _c_p, _i64, _c_p], _int),
    "tr_decode_base3": ([_c_p, _c_p, _i64, _c_p], _int),
    "tr_quantize_blocks": ([_c_p, _c_p, _c_p, _i64, _c_p], _int),
    "tr_dequantize_blocks": ([_c_p, _c_p, _c_p, _i64, _c_p], _int),
    "tr_gemm_exact": ([_int, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, _i64, _i64, _c_p], _int),
    "tr_quantize_pack": ([_int, _c_p, _i64, _i64, _c_p, _c_p, _c_p], _int),
    "tr_layout_bytes": ([_int, _i64, _i64], _i64),
    "tr_repack": ([_int, _c_p, _c_p, _i64, _i64, _c_p, ctypes.c_size_t, _c_p], _int),
    "tr_unrepack": ([_int, _c_p, _i64, _i64, ctypes.c_size_t, _c_p, _c_p, _c_p], _int),
    "tr_dequant_dense": ([_int, _c_p, _c_p, _i64, _i64, _int, _c_p, _c_p], _int),
    "tr_linear_workspace_size": ([_int, _i64, _i64, _i64], ctypes.c_size_t),
    "tr_repack_records": ([_int, _c_p, _i64, _i64, _c_p, ctypes.c_size_t, _c_p], _int),
    "tr_linear": ([_int, _c_p, _c_p, _c_p, _i64, _i64, _i64, _int, _i64, _i64, _int, _c_p, ctypes.c_size_t,
                   _c_p], _int),
    "tr_linear_pre": ([_int, _c_p, _c_p, _c_p, _i64, _i64, _i64, _int, _i64, _i64, _int, _int, _c_p, _c_p, _c_p,
                       ctypes.c_float, _c_p], _int),
    "tr_linear_chain_workspace_size": ([_i64], ctypes.c_size_t),
    "tr_linear_chain_prepare": ([ctypes.POINTER(TrChainLayer), _i64, _i64, _c_p, ctypes.c_size_t], _int),
    "tr_linear_chain": ([_int, ctypes.POINTER(TrChainLayer), _i64, _i64, _int, _c_p, ctypes.c_size_t, _c_p], _int),
    "tr_add_rmsnorm": ([_int, _c_p, _c_p, _c_p, _c_p, _i64, _i64, ctypes.c_float, _c_p], _int),
    "tr_rope_kv": ([_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, _i64, _c_p], _int),
    "tr_greedy_next": ([_int, _c_p, _i64, _c_p, _i64, _c_p, _c_p, _c_p, _i64, _c_p, _c_p], _int),
    "tr_greedy_next_batch": ([_int, _c_p, _i64, _c_p, _i64, _c_p, _c_p, _c_p, _i64, _c_p, _i64, _c_p], _int),
    "tr_attn_decode_batch": ([_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, _i64, ctypes.c_float,
                              _c_p], _int),
    "tr_attn_decode": ([_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, ctypes.c_float, _c_p],
                       _int),
    "tr_silu_mul": ([_int, _c_p, _c_p, _i64, _i64, _c_p], _int),
    "tr_attn_decode_workspace_size": ([_i64, _i64, _i64], ctypes.c_size_t),
    "tr_qkv_attn_decode_workspace_size": ([_i64], ctypes.c_size_t),
    "tr_qkv_attn_decode": ([_int, _c_p, _c_p, _c_p, _c_p, _c_p, ctypes.c_float, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                            _c_p, _i64, _i64, _i64, ctypes.c_float, _c_p, ctypes.c_size_t, _int, _c_p], _int),
    "tr_attn_decode_split": ([_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, ctypes.c_float, _c_p,
                              ctypes.c_size_t, _c_p], _int),
}

EXPORTED = tuple(_SIGS)


class TriRunError(RuntimeError):
    """A libtritrun call rejected its arguments or a CUDA launch failed."""


def lib():
    """Load libtritrun.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                        "(or __graft_entry__.build()); there is no CPU fallback")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (args, res) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.argtypes = args
                    fn.restype = res
                _lib = handle
    return _lib


def call(name: str, *args) -> int:
    """Invoke a tr_* entry point; non-zero status raises TriRunError."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().tr_last_error().decode(errors="replace")
        raise TriRunError(f"{name} failed: {msg}")
    return rc


def call_nostream(name: str, *args) -> int:
    """Invoke a tr_* entry point that takes no stream argument."""
    return call(name, *args)


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
