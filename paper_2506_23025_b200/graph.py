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


class LinearStack:
    """y = W_{n-1}( ... W_1(W_0 x)) over TernaryWeights, replayed from one CUDA graph.

    Default: one PDL-chained tr_linear per layer (GEMV or tcgen05 GEMM by batch).
    ``chain=True`` (batch <= 8, TQ2) runs the whole stack as ONE persistent cooperative
    launch instead (tr_linear_chain: grid barriers between layers, weights prefetched
    across them) -- measured slower than the PDL chain in round 1 (11.4 vs 8.1 us per
    layer on the bench stack), so it is opt-in.
    """

    def __init__(self, weights: list[TernaryWeight], batch: int, dtype=torch.float16, pdl: bool = True,
                 chain: bool | None = None):
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
        if chain is None:
            chain = False
        chain = chain and self.batch <= 8 and all(w.fmt is DType.TQ2 for w in weights)
        self.chain = chain
        if chain:
            table = []
            cur = self.x
            for w, out in zip(weights, self.bufs):
                table.append(_lib.TrChainLayer(w.data.data_ptr(), cur.data_ptr(), out.data_ptr(), cur.stride(0),
                                               out.stride(0), w.rows, w.cols))
                cur = out
            self._table = (_lib.TrChainLayer * len(table))(*table)
            need = _lib.lib().tr_linear_chain_workspace_size(len(table))
            self._ws = torch.zeros(need, dtype=torch.uint8, device=dev)
            _lib.call_nostream("tr_linear_chain_prepare", self._table, len(table), self.batch, self._ws.data_ptr(),
                               self._ws.numel())
        self.stream = torch.cuda.Stream(device=dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            try:
                self._body()                  # warm-up (lazy kernel attribute setup) outside capture
            except _lib.TriRunError:
                if not self.chain:
                    raise
                self.chain = False            # e.g. activations too wide to stage: per-layer launches
                self._body()
            self.stream.synchronize()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._body()
        torch.cuda.synchronize(dev)

    def _body(self) -> None:
        if self.chain:
            _lib.call("tr_linear_chain", _ACT[self.dtype], self._table, len(self.weights), self.batch,
                      _lib.LINEAR_PDL if self.pdl else 0, self._ws.data_ptr(), self._ws.numel(), _lib.stream_handle())
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
        """End-to-end: pinned host x -> device, graph replay, device -> pinned host y (async on the current stream)."""
        self.x.copy_(x_host, non_blocking=True)
        self.graph.replay()
        y_host.copy_(self.out, non_blocking=True)
