"""CPU-only tests: the C-ABI library loads and exports every declared symbol, and
the host-side API logic (formats, PackedMatrix, backend selection, roofline
arithmetic) mirrors the reference.  No compute calls (no GPU here)."""

from __future__ import annotations

import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tritrun.h")).read()
    return sorted(set(re.findall(r"TR_API\s+[\w\s\*]+?\b(tr_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2506_23025_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.EXPORTED)
    assert _lib.lib().tr_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    from paper_2506_23025_b200 import _lib

    assert _lib.lib().tr_layout_bytes(2, 0, 5) == -1
    assert _lib.lib().tr_layout_bytes(2, 4096, 4096) == 16 * 256 * (1024 + 32)
    rc = _lib.lib().tr_linear(9, None, None, None, 1, 1, 1, 1, 1, 1, 0, None, 0, None)
    assert rc == -1 and b"fmt" in _lib.lib().tr_last_error()
    assert _lib.lib().tr_linear_workspace_size(2, 1, 4096, 4096) > 4096 * 4 // 16
    with pytest.raises(_lib.TriRunError):
        _lib.call("tr_quantize_pack", 7, None, 1, 1, None, None, None)


def test_dtype_mirror():
    from paper_2506_23025_b200 import DType

    assert (DType.TQ2.payload_bytes, DType.TQ2.block_bytes) == (64, 66)
    assert (DType.TQ1.payload_bytes, DType.TQ1.block_bytes) == (52, 54)
    assert DType.TQ2.bits_per_weight == Fraction(33, 16)
    assert DType.TQ1.bits_per_weight == Fraction(27, 16)
    assert DType.parse("tq1") is DType.TQ1
    with pytest.raises(ValueError):
        DType.parse("int8")
    with pytest.raises(ValueError):
        _ = DType.F32.payload_bytes


def test_packed_matrix_validation_and_block_bytes(golden):
    from paper_2506_23025_b200 import DType, PackedMatrix

    g = golden["linear"]
    pm = PackedMatrix(rows=37, cols=1500, fmt=DType.TQ1, payload=g["tq1_37x1500_payload"].copy(),
                      scales=g["tq1_37x1500_scales"].copy())
    assert pm.blocks_per_row == 6 and pm.weight_bytes == 37 * 6 * 54
    raw = pm.to_block_bytes()
    again = PackedMatrix.from_block_bytes(raw, 37, 1500, DType.TQ1)
    np.testing.assert_array_equal(again.payload, pm.payload)
    with pytest.raises(ValueError):
        pm.payload[0, 0, 0] = 1
    with pytest.raises(ValueError):
        PackedMatrix(rows=37, cols=1500, fmt=DType.TQ2, payload=pm.payload.copy(), scales=pm.scales.copy())
    with pytest.raises(ValueError):
        PackedMatrix.from_block_bytes(raw[:-1], 37, 1500, DType.TQ1)


def test_backend_selection(monkeypatch):
    from paper_2506_23025_b200 import backend

    assert backend.available() == ("cuda",)
    assert backend.resolve().NAME == "cuda"
    monkeypatch.setenv(backend.ENV_VAR, "python")
    with pytest.raises(ValueError):
        backend.default_name()
    monkeypatch.delenv(backend.ENV_VAR)
    with pytest.raises(ValueError):
        backend.resolve("fortran")


def test_critical_batch_and_weight_bytes():
    from paper_2506_23025_b200 import DType, critical_batch
    from paper_2506_23025_b200.perf import weight_bytes

    assert critical_batch(105, 2) == 13
    assert critical_batch(1678.2e12 / 6553e9, 2.0625) == 33
    assert weight_bytes(8, 300, DType.TQ2) == 1056 and weight_bytes(8, 300, DType.TQ1) == 864
    assert weight_bytes(8, 300, DType.F16) == 4800 and weight_bytes(8, 300, DType.F32) == 9600


def test_decode_entry_points_validate_without_gpu():
    """The round-2 decode entry points check their arguments before touching the GPU: wrong head
    size, cache length, batch bounds, workspace size and flag combinations come back as -1 with a
    message (the product path never silently falls back)."""
    from paper_2506_23025_b200 import _lib

    lib = _lib.lib()
    assert lib.tr_qkv_attn_decode_workspace_size(24) == 24 * 4
    assert lib.tr_qkv_attn_decode_workspace_size(0) == 0
    assert lib.tr_attn_decode_workspace_size(24, 128, 128) >= 0
    cases = [
        # (entry point, args, message fragment)
        ("tr_attn_decode_batch", (1, None, None, None, None, None, None, None, 2, 24, 64, 128, 0.1, None), b"head_dim"),
        ("tr_attn_decode_batch", (1, None, None, None, None, None, None, None, 0, 24, 128, 128, 0.1, None), b"batch"),
        ("tr_attn_decode_batch", (1, None, None, None, None, None, None, None, 2, 24, 128, 256, 0.1, None), b"max_seq"),
        ("tr_greedy_next_batch", (1, None, 0, None, 8, None, None, None, 16, None, 2, None), b"sizes"),
        ("tr_greedy_next_batch", (1, None, 100, None, 8, None, None, None, 16, None, 0, None), b"batch"),
        ("tr_qkv_attn_decode", (1, None, None, None, None, None, 1e-5, None, None, None, None, None, None, None,
                                24, 128, 128, 0.1, None, 0, 0, None), b"workspace"),
        ("tr_qkv_attn_decode", (3, None, None, None, None, None, 1e-5, None, None, None, None, None, None, None,
                                24, 128, 128, 0.1, None, 96, 0, None), b"act_dtype"),
        ("tr_attn_decode", (1, None, None, None, None, None, None, None, 24, 128, 512, 0.1, None), b"max_seq"),
    ]
    for name, args, frag in cases:
        rc = getattr(lib, name)(*args)
        assert rc == -1, name
        assert frag in lib.tr_last_error(), (name, lib.tr_last_error())
    # the SwiGLU epilogue never falls through to a path that does not know it
    flags = _lib.LINEAR_EPI_SWIGLU | _lib.LINEAR_FORCE_UMMA
    rc = lib.tr_linear(2, None, None, None, 1, 64, 64, 1, 64, 32, flags, None, 0, None)
    assert rc == -1
