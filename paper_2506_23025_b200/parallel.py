"""Tensor-parallel ternary linears across the GPUs of one node.

The reference's only parallelism is host-thread row sharding (linear.py:132-166):
output rows are split into disjoint ranges and the result is bitwise independent
of the split.  Its multi-GPU generalisation:

* **column-parallel** (gate/up/qkv projections) -- rank i owns output rows
  [r0, r1) of the packed matrix (whole 256-blocks of every row, so the shard is an
  exact slice of ``PackedMatrix.payload`` / ``scales``).  No collective; the local
  output is bitwise equal to the same rows of the single-GPU product.
* **row-parallel** (down/o projections) -- rank i owns the 256-blocks
  [b0, b1) of every row (K split on block boundaries, the format's own
  granularity) and the matching columns of x.  Each rank produces a partial
  [batch, rows]; **one all-reduce (sum)** over NCCL/NVLink completes the product.
  The block-sum order changes, so parity with the single-GPU result is by
  tolerance.

Collectives go through ``torch.distributed`` (NCCL on B200 / NVSwitch, gloo in the
CPU tests).  The matmul itself is ``device.linear`` (the tcgen05 / mma.sync
kernels); ``linear_fn`` can be injected so the host logic is testable without a GPU.
"""

from __future__ import annotations

import numpy as np

from .blocks import BLOCK_ELEMENTS
from .packed_linear import PackedMatrix


def shard_bounds(n: int, parts: int, index: int, align: int = 1) -> tuple[int, int]:
    """[lo, hi) of the index-th of `parts` near-equal contiguous pieces of range(n), cut on
    multiples of `align` (the last piece takes the remainder)."""
    if not 0 <= index < parts:
        raise ValueError(f"shard index {index} out of range for {parts} parts")
    if align < 1:
        raise ValueError(f"align must be >= 1, got {align}")
    units = -(-n // align)
    lo, hi = (units * index) // parts * align, (units * (index + 1)) // parts * align
    return min(lo, n), min(hi, n)


def shard_rows(pm: PackedMatrix, parts: int, index: int, align: int = 1) -> PackedMatrix:
    """Column-parallel shard: output rows [r0, r1) (exact slice of the packed arrays).

    ``align=BLOCK_ELEMENTS`` cuts on 256-row boundaries, so the shard's outputs are exactly the
    256-blocks of K a following RowParallelTernaryLinear (shard_cols) owns on the same rank."""
    r0, r1 = shard_bounds(pm.rows, parts, index, align)
    if r1 <= r0:
        raise ValueError(f"{pm.rows} rows cannot be split into {parts} non-empty shards")
    return PackedMatrix(rows=r1 - r0, cols=pm.cols, fmt=pm.fmt, payload=np.array(pm.payload[r0:r1]),
                        scales=np.array(pm.scales[r0:r1]))


def shard_cols(pm: PackedMatrix, parts: int, index: int) -> tuple[PackedMatrix, int, int]:
    """Row-parallel shard: 256-blocks [b0, b1) of every row.

    Returns (shard, c0, c1): the shard multiplies x[:, c0:c1].  Only the last shard
    can carry the matrix's partial tail block.
    """
    nb = pm.blocks_per_row
    b0, b1 = shard_bounds(nb, parts, index)
    if b1 <= b0:
        raise ValueError(f"{nb} blocks per row cannot be split into {parts} non-empty shards")
    c0 = b0 * BLOCK_ELEMENTS
    c1 = min(b1 * BLOCK_ELEMENTS, pm.cols)
    shard = PackedMatrix(rows=pm.rows, cols=c1 - c0, fmt=pm.fmt, payload=np.array(pm.payload[:, b0:b1]),
                         scales=np.array(pm.scales[:, b0:b1]))
    return shard, c0, c1


def _dist():
    import torch.distributed as dist

    return dist


class ColumnParallelTernaryLinear:
    """y[:, r0:r1] = x @ W[r0:r1]^T on this rank; optionally all-gathered to the full y."""

    def __init__(self, pm: PackedMatrix, group=None, linear_fn=None, to_device=True, align: int = 1):
        """``align=BLOCK_ELEMENTS`` when the output feeds a RowParallelTernaryLinear (x_local = y)."""
        dist = _dist()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.rows, self.cols = pm.rows, pm.cols
        self.align = align
        self.r0, self.r1 = shard_bounds(pm.rows, self.world, self.rank, align)
        self.shard = shard_rows(pm, self.world, self.rank, align)
        self.weight = self.shard.to_device() if to_device else self.shard
        self.linear_fn = linear_fn

    def _mm(self, x):
        if self.linear_fn is not None:
            return self.linear_fn(x, self.weight)
        from .device import linear

        return linear(x, self.weight)

    def forward(self, x, gather: bool = False):
        y = self._mm(x)
        if not gather:
            return y
        import torch

        dist = _dist()
        # collectives need equal-sized pieces: pad every rank's rows to the largest shard
        bounds = [shard_bounds(self.rows, self.world, i, self.align) for i in range(self.world)]
        width = max(hi - lo for lo, hi in bounds)
        pad = torch.zeros((*y.shape[:-1], width), dtype=y.dtype, device=y.device)
        pad[..., : y.shape[-1]] = y
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[..., : hi - lo] for p, (lo, hi) in zip(parts, bounds)], dim=-1)

    __call__ = forward


class RowParallelTernaryLinear:
    """y = sum over ranks of x[:, c0:c1] @ W[:, c0:c1]^T -- one all-reduce after the local product.

    The local product keeps its fp32 accumulators (TR_LINEAR_OUT_F32) and the all-reduce sums
    fp32 partials; the sum is rounded once to the activation dtype.  With
    ``fp32_partials=False`` each partial is rounded to fp16/bf16 first (half the bytes on the
    wire, one extra rounding per rank: relative error up to world * 2^-11 for fp16).
    """

    def __init__(self, pm: PackedMatrix, group=None, linear_fn=None, to_device=True):
        dist = _dist()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.rows, self.cols = pm.rows, pm.cols
        self.shard, self.c0, self.c1 = shard_cols(pm, self.world, self.rank)
        self.weight = self.shard.to_device() if to_device else self.shard
        self.linear_fn = linear_fn

    def forward(self, x_local, allreduce: bool = True, fp32_partials: bool = True):
        """x_local: this rank's columns [..., c1 - c0] (e.g. the output of a column-parallel layer
        built with ``align=BLOCK_ELEMENTS``)."""
        import torch

        if x_local.shape[-1] != self.c1 - self.c0:
            raise ValueError(f"rank {self.rank} owns columns [{self.c0}, {self.c1}) "
                             f"({self.c1 - self.c0} wide), got activations {tuple(x_local.shape)}")
        if self.linear_fn is not None:
            y = self.linear_fn(x_local, self.weight)
            if fp32_partials:
                y = y.float()
        else:
            from .device import linear

            y = linear(x_local, self.weight, out_dtype=torch.float32 if fp32_partials else None)
        if allreduce and self.world > 1:
            _dist().all_reduce(y, group=self.group)
        return y.to(x_local.dtype) if fp32_partials else y

    __call__ = forward
