"""Pin the CPU oracle (oracle/) against the reference before trusting it.

Two anchors:
  * golden fixtures produced by importing the reference (tests/golden/make_golden.py);
  * the reference's own compiled kernels in oracle/_ref (built from the reference
    sources by oracle/Makefile), compared bit-for-bit on random inputs.
Plus the reference's own hand-written golden vectors (test_codec.py:36-47,
166-177; test_blocks.py:131-154).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as orc

FMTS = {"tq2": orc.TQ2, "tq1": orc.TQ1}
SHAPES = [(1, 5), (2, 300), (3, 256), (6, 40), (16, 1000), (37, 1500), (64, 2048), (128, 512)]


def test_reference_vectors_base4():
    # test_codec.py:36-47 (trits -> digits = trit + 1)
    for trits, byte in (([-1, 0, 1, 1], 164), ([0, 0, 0, 0], 85), ([1, 1, 1, 1], 170), ([-1] * 4, 0)):
        d = (np.array(trits) + 1).astype(np.uint8)
        assert orc.pack_base4(d)[0] == byte
        np.testing.assert_array_equal(orc.unpack_base4(np.array([byte], np.uint8)), d)


def test_reference_vectors_tq1_blocks():
    # test_blocks.py:141-154: zero block = 52 x 0x80; all-absmax = 51 x 0xFF + 213
    p, s = orc.quantize_rows(np.zeros((1, 256), np.float32), orc.TQ1)
    assert p.tobytes() == bytes([128] * 52) and float(s[0]) == 0.0
    p, s = orc.quantize_rows(np.full((1, 256), 0.375, np.float32), orc.TQ1)
    assert p[0, :51].tobytes() == bytes([255] * 51) and p[0, 51] == 213
    # test_blocks.py:131-133: scale 1.0 stored as LE binary16 00 3c
    _, s = orc.quantize_rows(np.eye(1, 256, dtype=np.float32), orc.TQ2)
    assert s.tobytes() == b"\x00\x3c"


def test_codec_tables_match_golden(golden):
    g = golden["codec"]
    np.testing.assert_array_equal(orc.decode_base3(np.arange(256, dtype=np.uint8)).reshape(256, 5),
                                  g["decode_all_bytes"])
    np.testing.assert_array_equal(orc.encode_base3(g["encode_groups"].reshape(-1)), g["encode_codes"])
    np.testing.assert_array_equal(orc.pack_base4(g["base4_quads"].reshape(-1)), g["base4_bytes"])
    np.testing.assert_array_equal(orc.unpack_base4(np.arange(256, dtype=np.uint8)).reshape(256, 4),
                                  g["unpack_all_bytes"])


def test_algorithm1_differs_from_canonical_on_13_noncanonical_bytes(golden):
    # the mul decoder and the division decoder disagree exactly on
    # the 13 byte values the encoder never emits.
    mul = golden["codec"]["decode_all_bytes"].astype(np.int64)
    c = np.arange(256, dtype=np.int64)
    xq = (c * 243 + 13) >> 8
    canon = (xq[:, None] // np.array([81, 27, 9, 3, 1])) % 3
    differ = np.nonzero((mul != canon).any(axis=1))[0]
    assert differ.tolist() == [1, 20, 40, 60, 79, 99, 119, 138, 158, 178, 197, 217, 237]
    assert not set(differ) & set(golden["codec"]["encode_codes"].tolist())


def test_quantize_matches_golden(golden):
    g = golden["quantize"]
    dg, sc = orc.quantize_blocks(g["values"])
    np.testing.assert_array_equal(dg, g["digits"])
    np.testing.assert_array_equal(sc.view(np.uint32), g["scales_f32"].view(np.uint32))
    with np.errstate(over="ignore"):
        for fmt, key in ((orc.TQ2, "tq2"), (orc.TQ1, "tq1")):
            p, s = orc.quantize_rows(g["values"], fmt)
            np.testing.assert_array_equal(p, g[f"{key}_payload"])
            np.testing.assert_array_equal(s.view(np.uint16), g[f"{key}_scales"].view(np.uint16))
    out = orc.dequantize_blocks(g["dq_digits"], g["dq_scales"])
    np.testing.assert_array_equal(out.view(np.uint32), g["dq_out"].view(np.uint32))


@pytest.mark.parametrize("fmt", ["tq2", "tq1"])
@pytest.mark.parametrize("rows,cols", SHAPES)
def test_pack_gemm_reference_match_golden(golden, fmt, rows, cols):
    g = golden["linear"]
    key = f"{fmt}_{rows}x{cols}"
    payload, scales = orc.pack_matrix(g[f"W_{rows}x{cols}"], FMTS[fmt])
    np.testing.assert_array_equal(payload, g[key + "_payload"])
    np.testing.assert_array_equal(scales.view(np.uint16), g[key + "_scales"].view(np.uint16))
    Y = orc.gemm(payload, scales, cols, FMTS[fmt], g[key + "_X"])
    np.testing.assert_array_equal(Y.view(np.uint32), g[key + "_Y"].view(np.uint32))
    Yt = orc.gemm(payload, scales, cols, FMTS[fmt], g[key + "_X"], threads=3)
    np.testing.assert_array_equal(Yt.view(np.uint32), g[key + "_Y"].view(np.uint32))
    for j in range(3):
        ref = orc.gemv_reference(payload, scales, cols, FMTS[fmt], g[key + "_X"][j])
        np.testing.assert_array_equal(ref, g[key + "_ref"][j])
    if key + "_dense" in g:
        dense = orc.dequantize_matrix(payload, scales, cols, FMTS[fmt], np.float32)
        np.testing.assert_array_equal(dense, g[key + "_dense"])
    # the streaming float64 product used at full BASELINE sizes agrees with gemv_reference
    refb = orc.gemv_reference_batch(payload, scales, cols, FMTS[fmt], g[key + "_X"], threads=2)
    np.testing.assert_allclose(refb, g[key + "_ref"], rtol=1e-12, atol=1e-12 * np.abs(g[key + "_ref"]).max())


def test_ternarize_golden_is_numpy_pairwise_mean():
    """tests/golden/ternarize.npz (reference ternarize, blocks.py:220-236): gamma is eps + numpy's
    pairwise mean, the rule the product's host-side gamma follows."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "ternarize.npz"))
    keys = sorted(k[:-2] for k in g.files if k.endswith("_W"))
    assert len(keys) == 12
    for k in keys:
        eps = float(k.rsplit("_eps", 1)[1])
        W = np.asarray(g[k + "_W"], np.float64)
        assert float(g[k + "_gamma"]) == eps + float(np.mean(np.abs(W)))
        q = np.clip(W / float(g[k + "_gamma"]), -1.0, 1.0)
        np.testing.assert_array_equal((q >= 0.5).astype(np.int8) - (q <= -0.5).astype(np.int8), g[k + "_trits"])


ref_kernels = orc.ref_kernels()
needs_ref = pytest.mark.skipif(ref_kernels is None, reason="oracle/_ref not built (make -C oracle ref)")


@needs_ref
def test_oracle_matches_reference_build_elementwise():
    rng = np.random.default_rng(7)
    digits = rng.integers(0, 3, size=4 * 5 * 2000, dtype=np.uint8)
    np.testing.assert_array_equal(orc.pack_base4(digits), np.asarray(ref_kernels.pack_base4(digits)))
    np.testing.assert_array_equal(orc.encode_base3(digits), np.asarray(ref_kernels.encode_base3(digits)))
    codes = rng.integers(0, 256, size=5000, dtype=np.uint8)
    np.testing.assert_array_equal(orc.decode_base3(codes), np.asarray(ref_kernels.decode_base3(codes)))
    np.testing.assert_array_equal(orc.unpack_base4(codes), np.asarray(ref_kernels.unpack_base4(codes)))
    vals = rng.normal(size=(300, 256)).astype(np.float32) * rng.uniform(0, 5, size=(300, 1)).astype(np.float32)
    vals[0] = 0
    a, b = orc.quantize_blocks(vals)
    c, d = ref_kernels.quantize_blocks(vals)
    np.testing.assert_array_equal(a, np.asarray(c))
    np.testing.assert_array_equal(b.view(np.uint32), np.asarray(d).view(np.uint32))


@needs_ref
@pytest.mark.parametrize("fmt", [orc.TQ2, orc.TQ1])
def test_oracle_gemm_matches_reference_build(fmt):
    rng = np.random.default_rng(11 + fmt)
    rows, cols, batch = 57, 1300, 4
    W = rng.normal(size=(rows, cols)).astype(np.float32)
    payload, scales = orc.pack_matrix(W, fmt)
    X = rng.uniform(-2, 2, size=(batch, cols)).astype(np.float32)
    ours = orc.gemm(payload, scales, cols, fmt, X)
    theirs = orc.gemm(payload, scales, cols, fmt, X, kern=ref_kernels)
    np.testing.assert_array_equal(ours.view(np.uint32), theirs.view(np.uint32))
