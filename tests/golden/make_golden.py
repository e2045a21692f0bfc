"""Generate the golden fixtures in tests/golden/ by importing the REFERENCE package.

Run in the build container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py

It imports `tritpack` from /root/reference/pkg/src with TRITPACK_BACKEND=python
(the reference's numpy backend, bitwise-identical to its compiled one by the
contract in _kernels_py.py:1-30) and records inputs and outputs of the
functions on the TriRun hot path.  The committed .npz files are what the
oracle (oracle/) and the CUDA product are checked against.
"""

from __future__ import annotations

import itertools
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    os.environ["TRITPACK_BACKEND"] = "python"
    sys.path.insert(0, REF_SRC)
    from tritpack import backend
    from tritpack.blocks import DType, quantize_rows
    from tritpack.linear import gemm, gemv_reference, pack_matrix, dequantize_matrix

    kern = backend.resolve("python")

    # ---- codec tables -------------------------------------------------------
    groups = np.array(list(itertools.product(range(3), repeat=5)), dtype=np.uint8)  # 243 x 5
    quads = np.array(list(itertools.product(range(3), repeat=4)), dtype=np.uint8)   # 81 x 4
    np.savez_compressed(
        os.path.join(OUT, "codec.npz"),
        decode_all_bytes=kern.decode_base3(np.arange(256, dtype=np.uint8)).reshape(256, 5),
        encode_groups=groups,
        encode_codes=kern.encode_base3(groups.reshape(-1)),
        base4_quads=quads,
        base4_bytes=kern.pack_base4(quads.reshape(-1)),
        unpack_all_bytes=kern.unpack_base4(np.arange(256, dtype=np.uint8)).reshape(256, 4),
    )

    # ---- quantize edge cases (test_backends.py:120-132, test_blocks.py:93-154) ----
    rng = np.random.default_rng(62)
    vals = rng.normal(size=(16, 256)).astype(np.float32)
    vals[0] = 0.0
    vals[1, ::2] = -0.0
    vals[2] = 1e-38
    vals[3, 17] = -5.0
    vals[4, :5] = [0.5, -0.5, 0.4999999, -0.4999999, 1.0]
    vals[5] = 0.375
    vals[6] = (rng.integers(0, 3, 256) - 1) * np.float32(768.0)
    vals[7] = rng.uniform(-10, 10, 256)
    vals[8, :] = 65504.0 * 1.5  # scale overflows binary16 -> inf
    dg, sc = kern.quantize_blocks(vals)
    p2, s2 = quantize_rows(vals, DType.TQ2)
    p1, s1 = quantize_rows(vals, DType.TQ1)
    dq_digits = rng.integers(0, 3, size=(8, 256), dtype=np.uint8)
    dq_scales = rng.uniform(0, 2, size=8).astype(np.float32)
    dq_scales[:3] = 0.0
    np.savez_compressed(
        os.path.join(OUT, "quantize.npz"),
        values=vals, digits=dg, scales_f32=sc,
        tq2_payload=p2, tq2_scales=s2, tq1_payload=p1, tq1_scales=s1,
        dq_digits=dq_digits, dq_scales=dq_scales,
        dq_out=kern.dequantize_blocks(dq_digits, dq_scales),
    )

    # ---- pack_matrix + gemm + gemv_reference on the reference's test shapes ----
    cases = {}
    shapes = [(1, 5), (2, 300), (3, 256), (6, 40), (16, 1000), (37, 1500), (64, 2048), (128, 512)]
    for fmt in (DType.TQ2, DType.TQ1):
        for rows, cols in shapes:
            seed = rows * cols
            rng = np.random.default_rng(seed)
            if (rows, cols) == (128, 512):
                # BASELINE idiom: per-channel gamma_r * ternary T
                T = (rng.integers(0, 3, size=(rows, cols)) - 1).astype(np.float32)
                gam = np.float16(0.02 * (1.0 + rng.uniform(0, 1, size=(rows, 1)))).astype(np.float32)
                W = (gam * T).astype(np.float32)
            else:
                W = rng.normal(size=(rows, cols)).astype(np.float32)
                W[0, :] = 0.0 if rows > 2 else W[0, :]
            pm = pack_matrix(W, fmt)
            X = rng.uniform(-1.0, 1.0, size=(3, cols)).astype(np.float32)
            X[:, 0] = -0.0
            Y = gemm(pm, X)
            ref = np.stack([gemv_reference(pm, X[j]) for j in range(3)])
            key = f"{fmt.name.lower()}_{rows}x{cols}"
            cases[f"W_{rows}x{cols}"] = W  # same seed for both formats
            cases[key + "_payload"] = pm.payload
            cases[key + "_scales"] = pm.scales
            cases[key + "_X"] = X
            cases[key + "_Y"] = Y
            cases[key + "_ref"] = ref
            if rows * cols <= 20000:
                cases[key + "_dense"] = dequantize_matrix(pm, dtype=np.float32)
    np.savez_compressed(os.path.join(OUT, "linear.npz"), **cases)
    make_ternarize()
    print("wrote", sorted(f for f in os.listdir(OUT) if f.endswith(".npz")))


def make_ternarize() -> None:
    """ternarize (blocks.py:220-236): gamma = eps + mean|W| (numpy's pairwise float64 sum) and
    the trits, on shapes whose mean needs many partial sums (so the reduction order shows)."""
    sys.path.insert(0, REF_SRC)
    from tritpack.blocks import ternarize

    rng = np.random.default_rng(220)
    mats = {
        "normal_96x517": rng.normal(size=(96, 517)),
        "uniform_f32_65x257": rng.uniform(-3, 3, size=(65, 257)).astype(np.float32),
        "lognormal_8x4099": rng.lognormal(size=(8, 4099)) * rng.choice([-1.0, 1.0], size=(8, 4099)),
        "int_valued_31x33": rng.integers(-4, 5, size=(31, 33)).astype(np.float64),
        "zeros_4x4": np.zeros((4, 4)),
        "tiny_2x3": np.array([[1e-300, -1e-300, 0.0], [5e-6, -5e-6, 1e-5]]),
    }
    out = {}
    for name, W in mats.items():
        for eps in (1e-5, 0.25):
            r = ternarize(W, epsilon=eps)
            key = f"{name}_eps{eps:g}"
            out[key + "_W"] = W
            out[key + "_gamma"] = np.float64(r.gamma)
            out[key + "_trits"] = r.trits
    np.savez_compressed(os.path.join(OUT, "ternarize.npz"), **out)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ternarize":
    make_ternarize()
    sys.exit(0)


if __name__ == "__main__":
    main()
