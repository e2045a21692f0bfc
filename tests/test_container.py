"""TPK1 container parsing (CPU): the reference writer's own file, and the reference's failure modes
(test_container.py:194-340 restated)."""

from __future__ import annotations

import os
import struct

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def ct():
    from paper_2506_23025_b200 import container

    return container


def _block_bytes(payload, scales_u16):
    """PackedMatrix.to_block_bytes (linear.py:73-82): per block payload then the LE fp16 scale."""
    rows, nb, pb = payload.shape
    rec = np.zeros((rows, nb, pb + 2), np.uint8)
    rec[:, :, :pb] = payload
    rec[:, :, pb:] = scales_u16.astype("<u2").view(np.uint8).reshape(rows, nb, 2)
    return rec.tobytes()


def test_reference_written_file_parses(ct):
    g = np.load(os.path.join(GOLDEN, "model_tpk1.npz"))
    recs = ct.read_container(os.path.join(GOLDEN, "model.tpk1"))
    by = {r.name: r for r in recs}
    assert [r.name for r in recs] == ["layers.0.attn.qkv", "layers.0.mlp.down", "layers.0.mlp.up", "embed", "norm"]
    assert by["layers.0.attn.qkv"].dims == (3, 16, 300) and by["layers.0.attn.qkv"].dtype == ct.DType.TQ2
    assert by["layers.0.mlp.down"].dtype == ct.DType.TQ1 and by["layers.0.mlp.up"].dims == (130, 512)
    for key, name in [("qkv", "layers.0.attn.qkv"), ("down", "layers.0.mlp.down"), ("up", "layers.0.mlp.up")]:
        assert bytes(by[name].data) == _block_bytes(g[f"{key}_payload"], g[f"{key}_scales"])
    assert bytes(by["embed"].data) == g["embed"].astype("<f2").tobytes()
    assert bytes(by["norm"].data) == g["norm"].astype("<f4").tobytes()
    assert ct.expected_data_len((3, 16, 300), ct.DType.TQ2) == 48 * 2 * 66
    assert ct.rows_cols((3, 16, 300)) == (48, 300)


def _raw(name=b"w", tag=2, dims=(2, 256), data=None, version=1, magic=b"TPK1", count=1):
    """A hand-built single-record file (the reference test's _valid_raw shape)."""
    head = struct.pack("<4sII", magic, version, count)
    rec = struct.pack("<H", len(name)) + name + struct.pack("<BB", tag, len(dims))
    rec += b"".join(struct.pack("<Q", d) for d in dims)
    if data is None:
        data = bytes(2 * 66) if tag == 2 else bytes(4 * int(np.prod(dims)))
    rec += struct.pack("<Q", len(data))
    pos = len(head) + len(rec)
    return head + rec + b"\x00" * (-pos % 32) + data


def test_handcrafted_and_empty(ct):
    recs = ct.parse_container(_raw())
    assert recs[0].name == "w" and recs[0].dims == (2, 256) and len(recs[0].data) == 132
    assert ct.parse_container(struct.pack("<4sII", b"TPK1", 1, 0)) == []   # empty container: 12 bytes


def test_failure_modes(ct):
    with pytest.raises(ct.BadMagicError):
        ct.parse_container(_raw(magic=b"TPK2"))
    with pytest.raises(ct.VersionMismatchError):
        ct.parse_container(_raw(version=2))
    good = _raw()
    for cut in range(len(good)):
        with pytest.raises(ct.TruncatedError):
            ct.parse_container(good[:cut])
    with pytest.raises(ct.SizeMismatchError):
        ct.parse_container(_raw(data=bytes(131)))
    with pytest.raises(ct.ContainerError, match="unknown dtype"):
        ct.parse_container(_raw(tag=9))
    with pytest.raises(ct.ContainerError, match="ndims"):
        ct.parse_container(_raw(dims=()))
    with pytest.raises(ct.ContainerError, match="positive"):
        ct.parse_container(_raw(dims=(0, 256), data=b""))
    with pytest.raises(ct.ContainerError, match="trailing"):
        ct.parse_container(good + b"\x00")
    assert issubclass(ct.TruncatedError, ct.ContainerError)
