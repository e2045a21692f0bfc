"""GPU-resident ternary weights and the fp16/bf16 hot path (TriRun on B200).

New API (no reference analogue; SURVEY.md Appendix B "Recommended GPU
additions"): ``TernaryWeight`` holds a matrix in the device T16 layout
(DESIGN.md), ``linear(x, w)`` computes ``x @ W^T`` for fp16/bf16 activations
with fp32 accumulation (paper App. F semantics), ``TernaryLinear`` wraps it as
an nn.Module.  Everything dispatches to libtritrun.so; there is no CPU path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .blocks import BLOCK_ELEMENTS, DType


def _writable(a):
    """C-contiguous and writable (torch.from_numpy warns on read-only views, e.g. np.frombuffer)."""
    a = np.ascontiguousarray(a)
    return a if a.flags.writeable else a.copy()


_ACT = {torch.float16: _lib.ACT_F16, torch.bfloat16: _lib.ACT_BF16}

_WORKSPACES: dict = {}
_RETIRED_WORKSPACES: list = []


def workspace(nbytes: int, device=None, stream=None) -> torch.Tensor:
    """Per-(device, stream) zero-initialised workspace for tr_linear, grown on demand.

    The kernels leave its counter region zeroed, so one buffer serves every
    launch on that stream (including CUDA-graph replays, which bake the pointer in).
    """
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev.index, s.cuda_stream)
    buf = _WORKSPACES.get(key)
    if buf is None or buf.numel() < nbytes:
        size = max(nbytes, 1 << 20, 0 if buf is None else 2 * buf.numel())
        if buf is not None:   # a captured CUDA graph may still point at it: never free
            _RETIRED_WORKSPACES.append(buf)
        buf = torch.zeros(size, dtype=torch.uint8, device=dev)
        _WORKSPACES[key] = buf
    return buf


class TernaryWeight:
    """A rows x cols ternary matrix resident on one GPU in the T16 layout."""

    def __init__(self, data: torch.Tensor, rows: int, cols: int, fmt: DType, uniform_scale: bool = False):
        self.data = data
        self.rows = int(rows)
        self.cols = int(cols)
        self.fmt = DType(fmt)
        # every row has one scale for all its blocks (per-channel gamma): the tensor-core
        # path may then apply the scale once per row instead of once per 256-block
        self.uniform_scale = bool(uniform_scale)

    # -- construction ---------------------------------------------------------------
    @classmethod
    def from_device_packed(cls, payload: torch.Tensor, scales_f16: torch.Tensor, rows: int, cols: int,
                           fmt: DType = DType.TQ2) -> "TernaryWeight":
        """Repack device-resident reference-layout payload/scales (linear.py:29-95) into T16."""
        fmt = DType(fmt)
        nbytes = _lib.lib().tr_layout_bytes(int(fmt), rows, cols)
        if nbytes < 0:
            raise NotImplementedError(f"{fmt.name} has no device layout yet")
        data = torch.empty(nbytes, dtype=torch.uint8, device=payload.device)
        _lib.call("tr_repack", int(fmt), payload.data_ptr(), scales_f16.data_ptr(), rows, cols, data.data_ptr(),
                  data.numel(), _lib.stream_handle())
        s = scales_f16.view(torch.int16).reshape(rows, -1)
        uniform = bool((s == s[:, :1]).all())
        return cls(data, rows, cols, fmt, uniform_scale=uniform)

    @classmethod
    def from_packed(cls, pm) -> "TernaryWeight":
        """From a host PackedMatrix (the offline-packed checkpoint form)."""
        payload = torch.from_numpy(_writable(pm.payload)).cuda()
        scales = torch.from_numpy(_writable(pm.scales).view(np.uint16).view(np.float16)).cuda()
        return cls.from_device_packed(payload, scales, pm.rows, pm.cols, pm.fmt)

    @classmethod
    def from_float(cls, W: torch.Tensor, fmt: DType = DType.TQ2) -> "TernaryWeight":
        """Quantize + pack a dense device matrix (pack_matrix semantics) straight into T16."""
        W = W.detach().to(device="cuda", dtype=torch.float32).contiguous()
        rows, cols = W.shape
        nb = -(-cols // BLOCK_ELEMENTS)
        fmt = DType(fmt)
        payload = torch.empty((rows, nb, fmt.payload_bytes), dtype=torch.uint8, device=W.device)
        scales = torch.empty((rows, nb), dtype=torch.float16, device=W.device)
        _lib.call("tr_quantize_pack", int(fmt), W.data_ptr(), rows, cols, payload.data_ptr(), scales.data_ptr(),
                  _lib.stream_handle())
        return cls.from_device_packed(payload, scales, rows, cols, fmt)

    # -- inspection ---------------------------------------------------------------------
    @property
    def blocks_per_row(self) -> int:
        return -(-self.cols // BLOCK_ELEMENTS)

    @property
    def weight_bytes(self) -> int:
        """Algorithmic weight bytes per product (reference formula, linear.py:68-71)."""
        return self.rows * self.blocks_per_row * self.fmt.block_bytes

    def unpack(self):
        """Exact inverse of the repack: (payload u8 (rows,nb,pb), scales f16 (rows,nb)) on the device."""
        nb = self.blocks_per_row
        payload = torch.empty((self.rows, nb, self.fmt.payload_bytes), dtype=torch.uint8, device=self.data.device)
        scales = torch.empty((self.rows, nb), dtype=torch.float16, device=self.data.device)
        _lib.call("tr_unrepack", int(self.fmt), self.data.data_ptr(), self.rows, self.cols, self.data.numel(),
                  payload.data_ptr(),
                  scales.data_ptr(), _lib.stream_handle())
        return payload, scales

    def dequantize(self, dtype=torch.float16) -> torch.Tensor:
        """Dense (rows, cols) fp16/bf16 copy (values scale*(d-1), exact in fp16)."""
        payload, scales = self.unpack()
        out = torch.empty((self.rows, self.cols), dtype=dtype, device=self.data.device)
        _lib.call("tr_dequant_dense", int(self.fmt), payload.data_ptr(), scales.data_ptr(), self.rows, self.cols,
                  _ACT[dtype], out.data_ptr(), _lib.stream_handle())
        return out

    def __repr__(self) -> str:
        return f"TernaryWeight({self.rows}x{self.cols}, {self.fmt.name}, {self.data.numel()} B on {self.data.device})"


_PATHS = {"auto": 0, "umma": _lib.LINEAR_FORCE_UMMA, "gemv": _lib.LINEAR_FORCE_GEMV,
          "gemv_f16": _lib.LINEAR_FORCE_GEMV | _lib.LINEAR_GEMV_F16}


def linear(x: torch.Tensor, w: TernaryWeight, out: torch.Tensor | None = None, pdl: bool = False,
           ctas: int = 0, ws: torch.Tensor | None = None, path: str = "auto", ksplit: int = 0,
           cosched: bool = False, epi_swiglu: bool = False, out_dtype=None, full_sm: bool = False,
           _probe: int = 0) -> torch.Tensor:
    """y[..., rows] = x[..., cols] @ W^T for fp16/bf16 x on the GPU (TriRun hot path).

    Accumulation is fp32: per 256-block partial sums are scaled by the block's
    binary16 scale in fp32 and accumulated in ascending block order; the output
    is rounded once to x.dtype.  ``pdl`` launches with programmatic dependent
    launch (for CUDA-graph-chained layers).  Batches 1-2 run the decode GEMV (batch 2
    with a long, thinly spread K the GEMM), batches >= 3 the tcgen05 tensor-core GEMM (measured
    crossovers, ``tritrun.h``); ``path`` ("umma" / "gemv" / "gemv_f16") forces one.  ``ctas`` forces the GEMV's CTA count and ``ksplit`` the GEMM's
    K split (0 = automatic); ``ws`` overrides the per-stream workspace.
    ``cosched`` (TR_LINEAR_COSCHEDULE) marks a layer in a back-to-back GEMV chain: at batch 1
    the int8-slice GEMV then runs as half-SM CTAs so the next layer co-resides and prefetches.
    ``full_sm`` (TR_LINEAR_FULL_SM) asks for whole-SM 16-warp CTAs at batch 1 instead.
    ``epi_swiglu`` (TR_LINEAR_EPI_SWIGLU): W is a gate|up weight with 16-row tiles alternating
    gate / up (``interleave_gate_up``); the result is silu(gate) * up, rows // 2 wide.
    ``out_dtype=torch.float32`` (TR_LINEAR_OUT_F32) returns the fp32 accumulators unrounded --
    the row-parallel partials an all-reduce sums (parallel.RowParallelTernaryLinear).
    """
    if x.dtype not in _ACT:
        raise TypeError(f"activations must be float16 or bfloat16, got {x.dtype}")
    if not x.is_cuda:
        raise ValueError("activations must be on a CUDA device")
    if x.shape[-1] != w.cols:
        raise ValueError(f"activation shape {tuple(x.shape)} does not match cols={w.cols}")
    lead = x.shape[:-1]
    x2 = x.reshape(-1, w.cols)
    if x2.stride(-1) != 1:
        x2 = x2.contiguous()
    if w.fmt == DType.TQ1 and (x2.stride(0) % 8 or x2.data_ptr() % 16):
        # the TQ1 path reads activations by TMA: rows 16-byte aligned (pad the row pitch)
        xp = torch.zeros((x2.shape[0], -(-w.cols // 8) * 8), dtype=x2.dtype, device=x2.device)
        xp[:, : w.cols] = x2
        x2 = xp[:, : w.cols]
    batch = x2.shape[0]
    rows_out = w.rows // 2 if epi_swiglu else w.rows
    odt = x.dtype if out_dtype is None else out_dtype
    if odt not in (x.dtype, torch.float32):
        raise TypeError(f"out_dtype must be the activation dtype or float32, got {odt}")
    if out is None:
        out = torch.empty((*lead, rows_out), dtype=odt, device=x.device)
    elif out.dtype != odt:
        raise TypeError(f"out has dtype {out.dtype}, expected {odt}")
    y2 = out.view(-1, rows_out)
    flags = (_lib.LINEAR_PDL if pdl else 0) | (_lib.LINEAR_UNIFORM_SCALE if w.uniform_scale else 0) | _PATHS[path]
    if odt == torch.float32:
        flags |= _lib.LINEAR_OUT_F32
    if epi_swiglu:   # (the int8-slice GEMV or K5; tr_linear rejects the fp16 GEMV: TriRunError)
        flags |= _lib.LINEAR_EPI_SWIGLU
    if cosched:   # back-to-back GEMV chain: half-SM CTAs so consecutive layers co-reside
        flags |= _lib.LINEAR_COSCHEDULE
    if full_sm:
        flags |= _lib.LINEAR_FULL_SM
    # one knob: the GEMV's CTA count or the tensor-core GEMM's K split, whichever path runs
    flags |= ((int(ksplit or ctas)) & 0xFFFF) << 8
    flags |= (int(_probe) & 0xF) << 24   # development probes (see csrc); 0 in production
    need = _lib.lib().tr_linear_workspace_size(int(w.fmt), batch, w.rows, w.cols)
    if ws is None:
        ws = workspace(need, x.device)
    _lib.call("tr_linear", int(w.fmt), w.data.data_ptr(), x2.data_ptr(), y2.data_ptr(), batch, w.rows, w.cols,
              _ACT[x.dtype], x2.stride(0), y2.stride(0), flags, ws.data_ptr(), ws.numel(), _lib.stream_handle())
    return out


def linear_pre(x: torch.Tensor, w: TernaryWeight, pre: int, delta: torch.Tensor | None = None,
               gamma: torch.Tensor | None = None, x_out: torch.Tensor | None = None, eps: float = 1e-5,
               out: torch.Tensor | None = None, pdl: bool = False, cosched: bool = False,
               epi_swiglu: bool = False, full_sm: bool = False) -> torch.Tensor:
    """``linear`` with the producer of its input fused into the GEMV's activation staging.

    pre = _lib.PRE_ADD_RMSNORM: y = rmsnorm(x + delta) * gamma @ W^T, and x + delta is
    written to ``x_out`` (the residual stream; must not alias x).  pre = _lib.PRE_SILU_MUL:
    y = (silu(x[:, :cols]) * x[:, cols:]) @ W^T for a gate|up product x.  Batch 1..8.
    """
    x2 = x.reshape(-1, x.shape[-1])
    batch = x2.shape[0]
    if out is None:
        out = torch.empty((batch, w.rows // 2 if epi_swiglu else w.rows), dtype=x.dtype, device=x.device)
    ptr = lambda t: 0 if t is None else t.data_ptr()
    _lib.call("tr_linear_pre", int(w.fmt), w.data.data_ptr(), x2.data_ptr(), out.data_ptr(), batch, w.rows, w.cols,
              _ACT[x.dtype], x2.stride(0), out.stride(0),
              (_lib.LINEAR_PDL if pdl else 0) | (_lib.LINEAR_COSCHEDULE if cosched else 0)
              | (_lib.LINEAR_FULL_SM if full_sm else 0)
              | (_lib.LINEAR_EPI_SWIGLU if epi_swiglu else 0), int(pre), ptr(delta),
              ptr(gamma), ptr(x_out), float(eps), _lib.stream_handle())
    return out


class TernaryLinear(torch.nn.Module):
    """nn.Linear-shaped module over a TernaryWeight (no bias, like the paper's BitLinear layers)."""

    def __init__(self, weight: TernaryWeight):
        super().__init__()
        self.weight_t = weight
        self.in_features = weight.cols
        self.out_features = weight.rows

    @classmethod
    def from_linear(cls, lin: torch.nn.Linear, fmt: DType = DType.TQ2) -> "TernaryLinear":
        return cls(TernaryWeight.from_float(lin.weight, fmt))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return linear(x, self.weight_t)

    def extra_repr(self) -> str:
        return f"in_features={self.in_features}, out_features={self.out_features}, fmt={self.weight_t.fmt.name}"


def interleave_gate_up(W: torch.Tensor, d_ff: int) -> torch.Tensor:
    """Rows of a [gate (d_ff) ; up (d_ff)] matrix as 16-row tiles alternating gate / up (the
    layout TR_LINEAR_EPI_SWIGLU expects): tile 2p = gate rows 16p.., tile 2p+1 = up rows 16p..."""
    if d_ff % 16:
        raise ValueError(f"d_ff ({d_ff}) must be a multiple of 16")
    g, u = W[:d_ff].reshape(d_ff // 16, 16, -1), W[d_ff:2 * d_ff].reshape(d_ff // 16, 16, -1)
    return torch.stack((g, u), dim=1).reshape(2 * d_ff, -1)
