"""Tensor-parallel sharding.

CPU: world_size-2 gloo process groups exercise the column-/row-parallel host logic
and the collectives, with the oracle's exact fp32 matmul injected as the local
product (test infrastructure only).  GPU: shards run through the CUDA kernels on
one device and recombine to the single-GPU product; a world_size-1 NCCL group
runs the module classes end to end.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import oracle as orc


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _packed(rows, cols, seed):
    import paper_2506_23025_b200 as tp

    rng = np.random.default_rng(seed)
    W = rng.normal(size=(rows, cols)).astype(np.float32)
    payload, scales = orc.pack_matrix(W, orc.TQ2)
    return tp.PackedMatrix(rows=rows, cols=cols, fmt=tp.DType.TQ2, payload=payload, scales=scales)


def _oracle_linear(x, pm):
    import torch

    y = orc.gemm(pm.payload, pm.scales, pm.cols, int(pm.fmt), x.numpy().astype(np.float32))
    return torch.from_numpy(y)


def _worker(rank, world, port, shapes, batch, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_23025_b200.parallel import ColumnParallelTernaryLinear, RowParallelTernaryLinear

        for rows, cols in shapes:
            pm = _packed(rows, cols, 7)
            x = torch.from_numpy(np.random.default_rng(8).uniform(-1, 1, size=(batch, cols)).astype(np.float32))
            col = ColumnParallelTernaryLinear(pm, linear_fn=_oracle_linear, to_device=False)
            y_local = col(x)
            y_full = col(x, gather=True)
            row = RowParallelTernaryLinear(pm, linear_fn=_oracle_linear, to_device=False)
            y_row = row(x[:, row.c0:row.c1])
            q.put((rows, cols, rank, col.r0, col.r1, y_local.numpy(), y_full.numpy(), y_row.numpy()))
    finally:
        dist.destroy_process_group()


def test_tp_gloo_world2():
    import torch.multiprocessing as mp

    world, batch = 2, 3
    shapes = [(64, 1024), (37, 1500)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shapes, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world * len(shapes))]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rows, cols, rank, r0, r1, y_local, y_full, y_row in res:
        pm = _packed(rows, cols, 7)
        x = np.random.default_rng(8).uniform(-1, 1, size=(batch, cols)).astype(np.float32)
        ref = orc.gemm(pm.payload, pm.scales, cols, orc.TQ2, x)
        np.testing.assert_array_equal(y_local.view(np.uint32), np.ascontiguousarray(ref[:, r0:r1]).view(np.uint32))
        np.testing.assert_array_equal(y_full.view(np.uint32), ref.view(np.uint32))           # bitwise
        np.testing.assert_allclose(y_row, ref, rtol=1e-5, atol=1e-4)   # block-sum order differs


def _chain_worker(rank, world, port, q):
    """column-parallel (align=256) -> row-parallel with fp32 partials, the 70B MLP pattern."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_23025_b200.parallel import ColumnParallelTernaryLinear, RowParallelTernaryLinear

        up, down = _packed(1280, 300, 21), _packed(77, 1280, 22)   # 5 blocks of 256 rows over 2 ranks
        x = torch.from_numpy(np.random.default_rng(23).uniform(-1, 1, size=(2, 300)).astype(np.float32))
        col = ColumnParallelTernaryLinear(up, linear_fn=_oracle_linear, to_device=False, align=256)
        row = RowParallelTernaryLinear(down, linear_fn=_oracle_linear, to_device=False)
        h = col(x)
        assert (col.r0, col.r1) == (row.c0, row.c1)   # the column shard's outputs are the row shard's K
        y = row(h.half().float())   # activations between the layers as the GPU path carries them
        y16 = row(h.half(), fp32_partials=False)
        q.put((rank, col.r0, col.r1, y.numpy(), y16.float().numpy()))
    finally:
        dist.destroy_process_group()


def test_tp_gloo_world2_column_to_row_chain():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r0, r1) for _, r0, r1, _, _ in res] == [(0, 512), (512, 1280)]
    up, down = _packed(1280, 300, 21), _packed(77, 1280, 22)
    x = np.random.default_rng(23).uniform(-1, 1, size=(2, 300)).astype(np.float32)
    h = orc.gemm(up.payload, up.scales, 300, orc.TQ2, x).astype(np.float16).astype(np.float32)
    ref = orc.gemm(down.payload, down.scales, 1280, orc.TQ2, h).astype(np.float64)
    for _, _, _, y, y16 in res:
        np.testing.assert_array_equal(y, res[0][3])   # every rank holds the same all-reduced sum
        den = np.abs(ref).max(axis=1)
        assert (np.abs(y - ref).max(axis=1) / den).max() <= 1e-6     # fp32 partials: fp32 accuracy
        assert (np.abs(y16 - ref).max(axis=1) / den).max() <= 2e-3   # fp16 partials: stated fp16 error


def test_shard_geometry():
    from paper_2506_23025_b200.parallel import shard_bounds, shard_cols, shard_rows

    pm = _packed(10, 28672, 3)
    for tp_ in (1, 2, 4, 8):
        cols = [shard_cols(pm, tp_, i) for i in range(tp_)]
        assert [s.blocks_per_row for s, _, _ in cols] == [112 // tp_] * tp_
        assert cols[0][1] == 0 and cols[-1][2] == 28672
        rows = [shard_rows(pm, tp_ if tp_ <= 10 else 10, i) for i in range(tp_)]
        assert sum(s.rows for s in rows) == 10
    assert shard_bounds(28672, 8, 7) == (25088, 28672)
    # 256-aligned row shards line up with the row-parallel block shards (d_ff 9216, TP 8)
    assert [shard_bounds(9216, 8, i, 256) for i in (0, 7)] == [(0, 1024), (7936, 9216)]
    assert [shard_bounds(9216, 8, i, 256)[1] - shard_bounds(9216, 8, i, 256)[0] for i in range(8)] == \
        [(shard_bounds(36, 8, i)[1] - shard_bounds(36, 8, i)[0]) * 256 for i in range(8)]
    with pytest.raises(ValueError):
        shard_rows(_packed(2, 256, 1), 4, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("tp_", [2, 4, 8])
def test_tp_shards_recombine_on_gpu(tp_):
    import torch

    import paper_2506_23025_b200 as tp
    from paper_2506_23025_b200.parallel import shard_cols, shard_rows

    rows, cols = 1024, 28672 // 4
    pm = _packed(rows, cols, 11)
    w = pm.to_device()
    x = (torch.rand(4, cols, device="cuda") * 2 - 1).half()
    full = tp.linear(x, w).float()
    col = torch.cat([tp.linear(x, shard_rows(pm, tp_, i).to_device()) for i in range(tp_)], dim=1)
    assert torch.equal(col.float(), full)   # column-parallel: bitwise equal
    part = torch.zeros_like(full)
    for i in range(tp_):
        s, c0, c1 = shard_cols(pm, tp_, i)
        part += tp.linear(x[:, c0:c1].contiguous(), s.to_device()).float()
    err = ((part - full).abs().amax(1) / full.abs().amax(1)).max().item()
    assert err <= 2e-3, err


@pytest.mark.gpu
def test_tp_modules_nccl_world1():
    import torch
    import torch.distributed as dist

    import paper_2506_23025_b200 as tp
    from paper_2506_23025_b200.parallel import ColumnParallelTernaryLinear, RowParallelTernaryLinear

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        pm = _packed(512, 2048, 5)
        x = (torch.rand(2, 2048, device="cuda") * 2 - 1).half()
        ref = tp.linear(x, pm.to_device())
        assert torch.equal(ColumnParallelTernaryLinear(pm)(x, gather=True), ref)
        assert torch.equal(RowParallelTernaryLinear(pm)(x), ref)
    finally:
        dist.destroy_process_group()
