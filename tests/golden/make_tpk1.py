"""Generate tests/golden/model.tpk1 (+ model_tpk1.npz) with the REFERENCE package's own writer.

Run in the build container (the reference is not present on the GPU box):

    python tests/golden/make_tpk1.py

The file is written by tritpack.container.write_container (container.py:167-182) from
tensors packed by tritpack.linear.pack_matrix; the .npz holds the reference's PackedMatrix
arrays and dense tensors, so the TPK1 loader is checked against the reference's own bytes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    os.environ["TRITPACK_BACKEND"] = "python"
    sys.path.insert(0, REF_SRC)
    from tritpack.blocks import DType
    from tritpack.container import TensorRecord, read_container, write_container
    from tritpack.linear import pack_matrix

    rng = np.random.default_rng(2506)

    def ternary(rows, cols, per_block=False):
        T = (rng.integers(0, 3, size=(rows, cols)) - 1).astype(np.float32)
        gam = np.float16(0.02 * (1 + rng.uniform(0, 1, size=(rows, 1)))).astype(np.float32)
        W = gam * T
        if per_block:
            nb = -(-cols // 256)
            W = W * np.repeat(rng.choice([1.0, 0.5, 0.25], size=(rows, nb)), 256, axis=1)[:, :cols].astype(np.float32)
        return W

    w_qkv = ternary(48, 300)             # stored as dims (3, 16, 300): leading dims collapse to 48 rows
    w_down = ternary(40, 700, True)      # TQ1, per-block scales
    w_up = ternary(130, 512, True)       # TQ2, per-block scales, rows not a multiple of 16
    embed = rng.normal(size=(10, 12)).astype(np.float16)
    norm = rng.normal(size=(12,)).astype(np.float32)
    pm_qkv, pm_down, pm_up = pack_matrix(w_qkv, DType.TQ2), pack_matrix(w_down, DType.TQ1), pack_matrix(w_up, DType.TQ2)
    recs = [
        TensorRecord.from_packed("layers.0.attn.qkv", pm_qkv, dims=(3, 16, 300)),
        TensorRecord.from_packed("layers.0.mlp.down", pm_down),
        TensorRecord.from_packed("layers.0.mlp.up", pm_up),
        TensorRecord.from_array("embed", embed),
        TensorRecord.from_array("norm", norm),
    ]
    path = os.path.join(OUT, "model.tpk1")
    write_container(path, recs)
    assert [r.name for r in read_container(path)] == [r.name for r in recs]
    np.savez_compressed(
        os.path.join(OUT, "model_tpk1.npz"),
        qkv_payload=pm_qkv.payload, qkv_scales=pm_qkv.scales.view(np.uint16),
        down_payload=pm_down.payload, down_scales=pm_down.scales.view(np.uint16),
        up_payload=pm_up.payload, up_scales=pm_up.scales.view(np.uint16),
        embed=embed, norm=norm)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
