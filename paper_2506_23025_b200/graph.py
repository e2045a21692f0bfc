"""CUDA-graph execution of chained ternary linears (decode-style layer streams).

A decode step is a long chain of small, HBM-bound products; at batch 1 a
4096x4096 TQ2 GEMV moves only 4.3 MB (0.66 us at 6.5 TB/s), so launch
overhead and the DRAM-latency ramp of each kernel dominate unless the launches
are (a) captured once in a CUDA graph and (b) chained with programmatic
dependent launch, which lets layer i+1 fetch its weights while layer i
finishes (weights do not depend on the previous output; only x does).
``LinearStack`` is that executor; ``run_host`` is the end-to-end call with
host (pinned) buffers used by bench.py's e2e measurement.
"""

from __future__ import annotations

import torch

from . import _lib
from .blocks import DType
from .device import _ACT, TernaryWeight, linear


class Chain:
    """A dependent sequence of TQ2 products run as ONE persistent launch (tr_linear_chain, K6).

    ``ops`` are dicts: w (TernaryWeight), x, y (device tensors), and optionally pre
    (_lib.PRE_ADD_RMSNORM / PRE_SILU_MUL), delta, gamma, x_out, eps, epi_swiglu, out_f32 --
    the arguments of device.linear / linear_pre.  Up to 256 products, batch 1-4.  The
    buffers are bound once (the product table lives in the workspace); ``run()`` enqueues
    one launch on the current stream (graph-capturable).
    """

    def __init__(self, ops: list[dict], batch: int, dtype=torch.float16):
        if not 1 <= len(ops) <= 256:
            raise ValueError("a chain holds 1..256 products")
        self.ops = ops
        self.batch = int(batch)
        self.dtype = dtype
        table = []
        for op in ops:
            w, x, y = op["w"], op["x"], op["y"]
            if w.fmt is not DType.TQ2:
                raise ValueError("tr_linear_chain runs TQ2 weights")
            flags = (_lib.LINEAR_EPI_SWIGLU if op.get("epi_swiglu") else 0) | \
                    (_lib.LINEAR_OUT_F32 if op.get("out_f32") else 0)
            ptr = lambda t: 0 if t is None else t.data_ptr()
            table.append(_lib.TrChainLayer(w.data.data_ptr(), x.data_ptr(), y.data_ptr(), x.stride(0), y.stride(0),
                                           w.rows, w.cols, int(op.get("pre", 0)), flags, ptr(op.get("delta")),
                                           ptr(op.get("gamma")), ptr(op.get("x_out")), float(op.get("eps", 1e-5))))
        self._table = (_lib.TrChainLayer * len(table))(*table)
        dev = ops[0]["w"].data.device
        need = _lib.lib().tr_linear_chain_workspace_size(len(table))
        self._ws = torch.zeros(need, dtype=torch.uint8, device=dev)
        torch.cuda.synchronize(dev)
        _lib.call_nostream("tr_linear_chain_prepare", self._table, len(table), self.batch, self._ws.data_ptr(),
                           self._ws.numel())

    def run(self, pdl: bool = True, probe: int = 0, ns: int = 0, hold: int = 0) -> None:
        """``probe``/``ns``/``hold``: development knobs (trace stamps / skeleton probes, ring cap in 4 KiB,
        bulk-copy piece in KiB)."""
        _lib.call("tr_linear_chain", _ACT[self.dtype], self._table, len(self.ops), self.batch,
                  (_lib.LINEAR_PDL if pdl else 0) | ((probe & 0xF) << 24) | ((ns & 0xFF) << 8) | ((hold & 0xFF) << 16),
                  self._ws.data_ptr(), self._ws.numel(), _lib.stream_handle())

    def trace(self) -> torch.Tensor:
        """Development probe (run(probe=2)): int64 %globaltimer stamps [n_ops, n_ctas, 16] = (op start,
        inputs ready, staged, stored, warp 0 main loop done, slice landed, first x loads landed, slice
        issued, main loops joined, boundary tiles stored, all stored)."""
        n = len(self.ops)
        sms = torch.cuda.get_device_properties(self._ws.device).multi_processor_count
        tab = 4096 + 104 * n + 16 * n   # (counters | ChainOp 104 B each | ChainW 16 B each)
        off = (tab + 255) // 256 * 256
        return self._ws[off: off + n * sms * 128].view(torch.int64).view(n, sms, 16)


class LinearStack:
    """y = W_{n-1}( ... W_1(W_0 x)) over TernaryWeights, replayed from one CUDA graph.

    ``chain=True`` (batch <= 4, TQ2, <= 256 layers, each CTA's weight slice must fit the ring next
    to the staged activations): the whole stack is ONE persistent launch (K6, tr_linear_chain).
    Default: one PDL-chained tr_linear per layer (GEMV or tcgen05 GEMM by batch) -- measured as
    fast as K6 on the BASELINE stack (6.1 vs 6.5 us per layer), whose per-layer
    time is set by compute and synchronisation, not by the weight stream.
    """

    def __init__(self, weights: list[TernaryWeight], batch: int, dtype=torch.float16, pdl: bool = True,
                 chain: bool = False):
        if not weights:
            raise ValueError("empty stack")
        for a, b in zip(weights, weights[1:]):
            if a.rows != b.cols:
                raise ValueError(f"chain mismatch: {a.rows} outputs feed {b.cols} inputs")
        self.weights = weights
        self.batch = int(batch)
        self.dtype = dtype
        self.pdl = pdl
        dev = weights[0].data.device
        self.x = torch.zeros((self.batch, weights[0].cols), dtype=dtype, device=dev)
        self.bufs = [torch.empty((self.batch, w.rows), dtype=dtype, device=dev) for w in weights]
        self.chain = bool(chain)
        self._chain = None
        if self.chain:   # (tr_linear_chain_prepare rejects what K6 cannot run: TriRunError)
            ops, cur = [], self.x
            for w, out in zip(weights, self.bufs):
                ops.append({"w": w, "x": cur, "y": out})
                cur = out
            self._chain = Chain(ops, self.batch, dtype)
        self.stream = torch.cuda.Stream(device=dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            self._body()                      # warm-up (lazy kernel attribute setup) outside capture
            self.stream.synchronize()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._body()
        torch.cuda.synchronize(dev)

    def _body(self) -> None:
        if self.chain:
            self._chain.run(pdl=self.pdl)
            return
        cur = self.x
        for w, out in zip(self.weights, self.bufs):
            # back-to-back GEMVs: half-SM CTAs, so each layer's successor co-resides and
            # prefetches its weights while it computes (TR_LINEAR_COSCHEDULE)
            linear(cur, w, out=out, pdl=self.pdl, cosched=True)
            cur = out

    @property
    def out(self) -> torch.Tensor:
        return self.bufs[-1]

    @property
    def launches(self) -> int:
        return 1 if self.chain else len(self.weights)

    def algorithmic_bytes(self) -> int:
        """Weights by the reference formula (linear.py:68-71) + activations in + outputs out, per replay."""
        es = torch.finfo(self.dtype).bits // 8
        return sum(w.weight_bytes + self.batch * (w.cols + w.rows) * es for w in self.weights)

    def flops(self) -> int:
        return sum(2 * w.rows * w.cols * self.batch for w in self.weights)

    def replay(self) -> None:
        """Enqueue one pass on the current stream (no host sync)."""
        self.graph.replay()

    def run_host(self, x_host: torch.Tensor, y_host: torch.Tensor) -> None:
        """End-to-end, as a caller sees it: pinned host x -> device, graph replay, device -> pinned host
        y, and the host waits until y is there (returns with the result readable)."""
        self.x.copy_(x_host, non_blocking=True)
        self.graph.replay()
        y_host.copy_(self.out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
