"""TriLM-shaped decoder stack over the ternary linear path (BASELINE configs[2]).

The paper's end-to-end benchmark (serving metrics 669-680) decodes
with every transformer linear in TQ2 and fp16 embeddings / lm_head.  This module is
the decoder-layer linear dispatch around the hot path: per layer one fused QKV
projection, the attention output projection, one fused gate|up projection and the
down projection -- all ``device.linear`` (batch 1 -> the decode GEMV, the 64-token
prompt -> the tcgen05 GEMM) -- with residual-add + RMSNorm, rotary embedding + KV-cache
append, single-token attention and SwiGLU each one libtritrun kernel
(csrc/decode_ops.cu); ``fused=False`` runs the same glue as PyTorch ops (the
reference the tests compare against).

One decode step (all layers + lm_head + greedy argmax + cache update) is captured
in a CUDA graph whose inputs (token, position) live on the device and are advanced
by the graph itself, so N output tokens are N back-to-back graph replays with no
host round trip.  ``dense=True`` builds the fp16 cuBLAS twin on the same (exactly
dequantized) weights for the speed-up baseline.

Shape (SURVEY §8(d) shape note): d_model 3072, 30 layers, 24 heads x 128, SwiGLU
9216, vocab 32000, untied fp16 embedding / lm_head -> 3.877B parameters.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import _lib
from .blocks import DType
from .device import _ACT, TernaryWeight, interleave_gate_up, linear, linear_pre


@dataclass(frozen=True)
class DecoderConfig:
    d_model: int = 3072
    n_layers: int = 30
    n_heads: int = 24
    d_ff: int = 9216
    vocab: int = 32000
    max_seq: int = 128
    eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def n_params(self) -> int:
        d, f = self.d_model, self.d_ff
        return self.n_layers * (4 * d * d + 3 * d * f + 2 * d) + 2 * self.vocab * d + d

    def ternary_bytes(self) -> int:
        """Packed bytes of the ternary linears (reference formula, 66 B per 256 weights)."""
        d, f = self.d_model, self.d_ff
        per = lambda r, c: r * (-(-c // 256)) * 66
        return self.n_layers * (per(3 * d, d) + per(d, d) + per(2 * f, d) + per(d, f))


def _interleaved(w: TernaryWeight, d_ff: int) -> TernaryWeight:
    """The same packed gate|up weight with rows as alternating 16-row gate / up tiles."""
    payload, scales = w.unpack()
    idx = interleave_gate_up(torch.arange(2 * d_ff, device=payload.device).unsqueeze(1), d_ff).squeeze(1)
    return TernaryWeight.from_device_packed(payload[idx].contiguous(), scales[idx].contiguous(), w.rows, w.cols, w.fmt)


def _ternary(rows, cols, gen, device):
    """Random-init ternary matrix with per-channel fp16 gamma (the bench's synthetic weights)."""
    T = torch.randint(0, 3, (rows, cols), generator=gen, device=device, dtype=torch.int8).float() - 1
    gam = (0.02 * (1 + torch.rand((rows, 1), generator=gen, device=device))).half().float()
    return TernaryWeight.from_float(gam * T)


class TernaryDecoder:
    STEPS_PER_GRAPH = 8   # decode steps per CUDA-graph replay (decode(n) uses single steps for the remainder)

    def __init__(self, cfg: DecoderConfig = DecoderConfig(), device="cuda", seed: int = 0, dense: bool = False,
                 weights=None, dtype=torch.float16, fused: bool = True):
        self.cfg, self.device, self.dense, self.dtype = cfg, torch.device(device), dense, dtype
        self.fused = fused   # glue as libtritrun kernels (default) or PyTorch ops (reference for tests)
        d, f, L = cfg.d_model, cfg.d_ff, cfg.n_layers
        gen = torch.Generator(device=self.device).manual_seed(seed)
        if weights is None:   # ternary weights, built once and shared with a dense twin
            weights = {
                "layers": [{"qkv": _ternary(3 * d, d, gen, self.device), "o": _ternary(d, d, gen, self.device),
                            "gate_up": _ternary(2 * f, d, gen, self.device), "down": _ternary(d, f, gen, self.device)}
                           for _ in range(L)],
                "embed": (torch.randn((cfg.vocab, d), generator=gen, device=self.device) * 0.02).to(dtype),
                "lm_head": (torch.randn((cfg.vocab, d), generator=gen, device=self.device) * 0.02).to(dtype),
            }
        self.weights = weights
        if dense:   # fp16 cuBLAS twin: the exact dequantized values (scale * trit is exact in fp16)
            self.lin = [{k: w.dequantize(dtype) for k, w in lw.items()} for lw in weights["layers"]]
        else:
            self.lin = weights["layers"]
        # decode: gate|up rows as alternating 16-row gate / up tiles, so the GEMV's epilogue
        # emits silu(gate) * up and the down projection reads a plain activation (same trits
        # and scales, rows permuted on the device)
        self.gate_up_il = None
        if not dense and fused and f % 16 == 0 and all(lw["gate_up"].fmt is DType.TQ2 for lw in weights["layers"]):
            self.gate_up_il = [_interleaved(lw["gate_up"], f) for lw in weights["layers"]]
        self.norm_attn = [torch.ones(d, device=self.device, dtype=dtype) for _ in range(L)]
        self.norm_mlp = [torch.ones(d, device=self.device, dtype=dtype) for _ in range(L)]
        self.norm_out = torch.ones(d, device=self.device, dtype=dtype)
        H, D, S = cfg.n_heads, cfg.head_dim, cfg.max_seq
        self.k_cache = torch.zeros((L, H, S, D), device=self.device, dtype=dtype)
        self._attn_ws = torch.empty(max(1, _lib.lib().tr_attn_decode_workspace_size(H, D, S)), dtype=torch.uint8,
                                    device=self.device)
        self.v_cache = torch.zeros((L, H, S, D), device=self.device, dtype=dtype)
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, D, 2, device=self.device).float() / D))
        ang = torch.arange(S, device=self.device).float()[:, None] * inv[None, :]
        self.cos, self.sin = ang.cos().to(dtype), ang.sin().to(dtype)
        # device-resident decode state, advanced inside the captured graph
        self.tok = torch.zeros(1, dtype=torch.long, device=self.device)
        self.pos = torch.zeros(1, dtype=torch.long, device=self.device)
        self.out_tokens = torch.zeros(S, dtype=torch.long, device=self.device)
        self.h0 = torch.zeros((1, d), device=self.device, dtype=dtype)   # embedding row of the next token
        self._positions = torch.arange(S, device=self.device)
        # TR_LINEAR_COSCHEDULE per decode GEMV (qkv, o, gate_up, down): 8-warp CTAs (measured)
        self.cosched = (False, False, False, False)
        # TR_LINEAR_FULL_SM per decode GEMV (qkv, o, gate_up, down): 16-warp CTAs at batch 1.  The o
        # projection runs after the 24-CTA attention kernel, so it has the SMs to itself: 1091 vs
        # 1065 tok/s; the qkv GEMV must leave room for the attention kernel's early launch (16
        # warps: 1003); gate|up and down are 16-warp by shape already (scripts/dev/decode_width.py)
        self.full_sm = (False, True, False, False)
        # decode QKV GEMV + attention as one kernel (tr_qkv_attn_decode): off by default -- measured
        # slower inside the decode chain (its 16-warp CTAs keep the following o
        # projection from launching early); use_fused_attention(True) switches it on
        self.fused_attn = False
        self._fused_attn_ok = (not dense and fused and D == 128 and S <= 128
                               and all(lw["qkv"].fmt is DType.TQ2 for lw in weights["layers"]))
        self._qkv_attn_ws = torch.zeros(_lib.lib().tr_qkv_attn_decode_workspace_size(H), dtype=torch.uint8,
                                        device=self.device)   # per-head arrival counters (stay zero)
        self._prefill_graphs = {}
        self.graph = None
        self._host_pos = 0
        self.graph_multi = None    # STEPS_PER_GRAPH decode steps in one graph (no replay boundaries)

    def use_fused_attention(self, on: bool = True) -> None:
        """Decode steps run add + RMSNorm -> QKV GEMV -> attention as one kernel (tr_qkv_attn_decode);
        needs TQ2 QKV weights, head_dim 128 and max_seq <= 128.  Re-captures the decode graph."""
        if on and not self._fused_attn_ok:
            raise ValueError("fused QKV + attention needs ternary TQ2 QKV weights, head_dim 128 and max_seq <= 128")
        self.fused_attn = bool(on)
        self.graph = self.graph_multi = None

    # -- building blocks ----------------------------------------------------------------
    def _lin(self, x, w):
        return F.linear(x, w) if self.dense else linear(x, w, pdl=True)

    def _swiglu(self, i, xn):
        """silu(gate) * up of layer i's MLP for xn [T, d]: the gate|up product's own SwiGLU store on the
        interleaved weight (int8-slice GEMV or K5), else the product and tr_silu_mul."""
        if self.gate_up_il is not None and self.cfg.d_ff % 32 == 0:
            return linear(xn, self.gate_up_il[i], pdl=True, epi_swiglu=True)
        gu = self._lin(xn, self.lin[i]["gate_up"])
        a = torch.empty((xn.shape[0], self.cfg.d_ff), device=self.device, dtype=self.dtype)
        _lib.call("tr_silu_mul", _ACT[self.dtype], gu.data_ptr(), a.data_ptr(), xn.shape[0], self.cfg.d_ff,
                  _lib.stream_handle())
        return a

    def _rms(self, x, wgt):
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.cfg.eps)).to(self.dtype) * wgt

    def _rope(self, x, pos):   # x [T, H, D], pos [T]
        c, s = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        x1, x2 = x[..., 0::2], x[..., 1::2]
        return torch.stack((x1 * c - x2 * s, x1 * s + x2 * c), dim=-1).flatten(-2)

    def _layer(self, i, h, pos, T):
        cfg, lw = self.cfg, self.lin[i]
        H, D, d = cfg.n_heads, cfg.head_dim, cfg.d_model
        qkv = self._lin(self._rms(h, self.norm_attn[i]), lw["qkv"]).view(T, 3, H, D)
        q, k, v = self._rope(qkv[:, 0], pos), self._rope(qkv[:, 1], pos), qkv[:, 2]
        self.k_cache[i].index_copy_(1, pos, k.transpose(0, 1))
        self.v_cache[i].index_copy_(1, pos, v.transpose(0, 1))
        # attention over the static cache; positions after the query's are masked
        keys = torch.arange(cfg.max_seq, device=self.device)
        mask = keys[None, :] <= pos[:, None]                                  # [T, S]
        att = F.scaled_dot_product_attention(q.transpose(0, 1)[None], self.k_cache[i][None], self.v_cache[i][None],
                                             attn_mask=mask[None, None])      # [1, H, T, D]
        h = h + self._lin(att[0].transpose(0, 1).reshape(T, d), lw["o"])
        gu = self._lin(self._rms(h, self.norm_mlp[i]), lw["gate_up"])
        g, u = gu[:, : cfg.d_ff], gu[:, cfg.d_ff:]
        return h + self._lin(F.silu(g) * u, lw["down"])

    def forward(self, tokens, pos, h_in=None, from_start: bool = False):
        """tokens [T] at positions pos [T] -> logits of the last position [vocab] (fills the cache).
        h_in: the tokens' embedding rows when already gathered (the fused decode step).
        from_start: the caller guarantees pos = 0..T-1 (a prompt), so prompt attention is plain
        causal attention over the first T cache rows (the flash kernel, no mask tensor)."""
        if self.fused:
            return self._forward_fused(tokens, pos, h_in, from_start)
        T = tokens.shape[0]
        h = self.weights["embed"][tokens]
        for i in range(self.cfg.n_layers):
            h = self._layer(i, h, pos, T)
        h = self._rms(h[-1:], self.norm_out)
        return F.linear(h, self.weights["lm_head"])[0]

    def _forward_fused(self, tokens, pos, h_in=None, from_start=False):
        """Same computation with the glue as single kernels.  Decode (T = 1) of the ternary
        model folds residual-add + RMSNorm into the QKV / gate|up GEMVs and SwiGLU into the
        down GEMV (tr_linear_pre): 5 launches per layer."""
        cfg, act, st = self.cfg, _ACT[self.dtype], _lib.stream_handle()
        T = tokens.shape[0] if h_in is None else h_in.shape[0]
        d, H, D, S = cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.max_seq
        if T == 1 and not self.dense:
            return self._decode_step_fused(tokens, pos, h_in)
        # (h_in, the fused decode step's embedding buffer, doubles as the residual stream)
        h = (self.weights["embed"][tokens] if h_in is None else h_in).contiguous()
        xn = torch.empty_like(h)
        q = torch.empty((T, H, D), device=self.device, dtype=self.dtype)
        delta = None
        for i in range(cfg.n_layers):
            lw = self.lin[i]
            _lib.call("tr_add_rmsnorm", act, h.data_ptr(), 0 if delta is None else delta.data_ptr(),
                      self.norm_attn[i].data_ptr(), xn.data_ptr(), T, d, cfg.eps, st)
            qkv = self._lin(xn, lw["qkv"])
            if T == 1:   # rope + cache append + attention in one kernel
                att = torch.empty((1, d), device=self.device, dtype=self.dtype)
                _lib.call("tr_attn_decode", act, qkv.data_ptr(), pos.data_ptr(), self.cos.data_ptr(),
                          self.sin.data_ptr(), self.k_cache[i].data_ptr(), self.v_cache[i].data_ptr(), att.data_ptr(),
                          H, D, S, D ** -0.5, st)
            else:        # prompt: rope + cache append, then causal attention (not the decode hot path)
                _lib.call("tr_rope_kv", act, qkv.data_ptr(), pos.data_ptr(), self.cos.data_ptr(), self.sin.data_ptr(),
                          q.data_ptr(), self.k_cache[i].data_ptr(), self.v_cache[i].data_ptr(), T, H, D, S, st)
                if from_start:
                    att = F.scaled_dot_product_attention(q.transpose(0, 1)[None], self.k_cache[i][None, :, :T],
                                                         self.v_cache[i][None, :, :T], is_causal=True)
                else:
                    keys = torch.arange(S, device=self.device)
                    mask = keys[None, :] <= pos[:, None]
                    att = F.scaled_dot_product_attention(q.transpose(0, 1)[None], self.k_cache[i][None],
                                                         self.v_cache[i][None], attn_mask=mask[None, None])
                att = att[0].transpose(0, 1).reshape(T, d)
            o = self._lin(att, lw["o"])
            _lib.call("tr_add_rmsnorm", act, h.data_ptr(), o.data_ptr(), self.norm_mlp[i].data_ptr(), xn.data_ptr(),
                      T, d, cfg.eps, st)
            a = self._swiglu(i, xn)
            delta = self._lin(a, lw["down"])
        _lib.call("tr_add_rmsnorm", act, h.data_ptr(), delta.data_ptr(), self.norm_out.data_ptr(), xn.data_ptr(),
                  T, d, cfg.eps, st)
        return F.linear(xn[-1:], self.weights["lm_head"])[0]

    def _decode_step_fused(self, tokens, pos, h_in=None):
        cfg, act, st = self.cfg, _ACT[self.dtype], _lib.stream_handle()
        d, H, D, S = cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.max_seq
        h0 = self.weights["embed"][tokens].contiguous() if h_in is None else h_in
        hs = [h0, torch.empty((1, d), device=self.device, dtype=self.dtype)]
        cur, delta = 0, None
        for i in range(cfg.n_layers):
            lw = self.lin[i]
            # residual stream ping-pongs: the GEMV reads hs[cur] and stores hs[cur] + delta to hs[1 - cur]
            cs, fs = self.cosched, self.full_sm
            att = torch.empty((1, d), device=self.device, dtype=self.dtype)
            if self.fused_attn:   # add + RMSNorm -> QKV GEMV -> rotary, cache append, attention: one kernel
                qkv = torch.empty((1, 3 * d), device=self.device, dtype=self.dtype)
                w = lw["qkv"]
                _lib.call("tr_qkv_attn_decode", act, w.data.data_ptr(), hs[cur].data_ptr(),
                          0 if delta is None else delta.data_ptr(), self.norm_attn[i].data_ptr(),
                          hs[1 - cur].data_ptr(), cfg.eps, qkv.data_ptr(), pos.data_ptr(), self.cos.data_ptr(),
                          self.sin.data_ptr(), self.k_cache[i].data_ptr(), self.v_cache[i].data_ptr(),
                          att.data_ptr(), H, D, S, D ** -0.5, self._qkv_attn_ws.data_ptr(),
                          self._qkv_attn_ws.numel(), _lib.LINEAR_PDL, st)
                cur = 1 - cur
                o = linear(att, lw["o"], pdl=True, cosched=cs[1], full_sm=fs[1])
            else:
                o = self._qkv_attn_unfused(i, hs, cur, delta, pos, att)
                cur = 1 - cur
            if self.gate_up_il is not None:   # SwiGLU in the gate|up GEMV's epilogue
                act_ = linear_pre(hs[cur], self.gate_up_il[i], _lib.PRE_ADD_RMSNORM, o, self.norm_mlp[i],
                                  hs[1 - cur], cfg.eps, pdl=True, cosched=cs[2], epi_swiglu=True, full_sm=fs[2])
                cur = 1 - cur
                delta = linear(act_, lw["down"], pdl=True, cosched=cs[3], full_sm=fs[3])
            else:
                gu = linear_pre(hs[cur], lw["gate_up"], _lib.PRE_ADD_RMSNORM, o, self.norm_mlp[i], hs[1 - cur],
                                cfg.eps, pdl=True, cosched=cs[2])
                cur = 1 - cur
                delta = linear_pre(gu, lw["down"], _lib.PRE_SILU_MUL, pdl=True, cosched=cs[3])
        xn = torch.empty((1, d), device=self.device, dtype=self.dtype)
        _lib.call("tr_add_rmsnorm", act, hs[cur].data_ptr(), delta.data_ptr(), self.norm_out.data_ptr(), xn.data_ptr(),
                  1, d, cfg.eps, st)
        return F.linear(xn, self.weights["lm_head"])[0]

    def _qkv_attn_unfused(self, i, hs, cur, delta, pos, att):
        """QKV GEMV with the add + RMSNorm producer, then the attention kernel; returns o."""
        cfg, act, st, lw, cs = self.cfg, _ACT[self.dtype], _lib.stream_handle(), self.lin[i], self.cosched
        H, D, S = cfg.n_heads, cfg.head_dim, cfg.max_seq
        qkv = linear_pre(hs[cur], lw["qkv"], _lib.PRE_ADD_RMSNORM, delta, self.norm_attn[i], hs[1 - cur],
                         cfg.eps, pdl=True, cosched=cs[0], full_sm=self.full_sm[0])
        if S <= 128:   # one CTA per head holds the whole cache
            _lib.call("tr_attn_decode", act, qkv.data_ptr(), pos.data_ptr(), self.cos.data_ptr(),
                      self.sin.data_ptr(), self.k_cache[i].data_ptr(), self.v_cache[i].data_ptr(), att.data_ptr(),
                      H, D, S, D ** -0.5, st)
        else:          # split-KV over 128-key chunks, partial softmaxes merged
            _lib.call("tr_attn_decode_split", act, qkv.data_ptr(), pos.data_ptr(), self.cos.data_ptr(),
                      self.sin.data_ptr(), self.k_cache[i].data_ptr(), self.v_cache[i].data_ptr(), att.data_ptr(),
                      H, D, S, D ** -0.5, self._attn_ws.data_ptr(), self._attn_ws.numel(), st)
        return linear(att, lw["o"], pdl=True, cosched=cs[1], full_sm=self.full_sm[1])

    # -- serving --------------------------------------------------------------------------
    def prefill(self, prompt: torch.Tensor, graph: bool = True) -> None:
        """Run the prompt (one batched pass: the tcgen05 GEMM path) and seed the decode state.

        With ``graph`` the pass is captured once per prompt length as a CUDA graph (the prompt
        is copied into a static buffer) and replayed, so time-to-first-token is GPU time, not
        ~12 host launches per layer."""
        T = prompt.shape[0]
        if not graph:
            if T > self.cfg.max_seq:
                raise ValueError(f"prompt of {T} tokens exceeds max_seq={self.cfg.max_seq}")
            self._host_pos = T
            self._prefill_body(prompt)
            return
        if T > self.cfg.max_seq:
            raise ValueError(f"prompt of {T} tokens exceeds max_seq={self.cfg.max_seq}")
        self._host_pos = T
        if T not in self._prefill_graphs:
            buf = prompt.to(device=self.device, dtype=torch.long).clone()
            s = torch.cuda.Stream(device=self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))   # prompt / state writes queued before us
            with torch.cuda.stream(s):
                self._prefill_body(buf)   # warm-up outside capture (workspaces, lazy set-up)
                s.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self._prefill_body(buf)
            torch.cuda.synchronize(self.device)
            self._prefill_graphs[T] = (g, buf)
        g, buf = self._prefill_graphs[T]
        buf.copy_(prompt)
        g.replay()

    def _prefill_body(self, prompt: torch.Tensor) -> None:
        T = prompt.shape[0]
        logits = self.forward(prompt, self._positions[:T], from_start=True)
        self.tok.copy_(logits.argmax().view(1))
        self.pos.fill_(T)
        self.h0.copy_(self.weights["embed"][self.tok])

    def _decode_body(self):
        if self.fused:   # embedding row gathered by the previous step; greedy bookkeeping in one kernel
            logits = self.forward(self.tok, self.pos, self.h0)
            _lib.call("tr_greedy_next", _ACT[self.dtype], logits.data_ptr(), logits.shape[-1],
                      self.out_tokens.data_ptr(), self.out_tokens.shape[0], self.tok.data_ptr(), self.pos.data_ptr(),
                      self.weights["embed"].data_ptr(), self.cfg.d_model, self.h0.data_ptr(), _lib.stream_handle())
            return
        logits = self.forward(self.tok, self.pos)
        nxt = logits.argmax().view(1)
        self.out_tokens.index_copy_(0, self.pos, nxt)
        self.tok.copy_(nxt)
        self.pos.add_(1)

    def capture(self) -> None:
        """Capture one greedy decode step (state advanced on the device) as a CUDA graph."""
        cur = torch.cuda.current_stream(self.device)
        s = torch.cuda.Stream(device=self.device)
        saved = (self.tok.clone(), self.pos.clone(), self.k_cache.clone(), self.v_cache.clone(), self.h0.clone())
        s.wait_stream(cur)   # a queued prefill (and the clones above) complete before the warm-up step
        with torch.cuda.stream(s):
            self._decode_body()   # warm-up (lazy kernel set-up) outside capture
            s.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=s):
                self._decode_body()
            # the same step chained STEPS_PER_GRAPH times: the PDL chain runs on across steps
            # instead of draining at each replay boundary
            self.graph_multi = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph_multi, stream=s):
                for _ in range(self.STEPS_PER_GRAPH):
                    self._decode_body()
        torch.cuda.synchronize(self.device)
        cur.wait_stream(s)
        self.tok.copy_(saved[0])
        self.pos.copy_(saved[1])
        self.k_cache.copy_(saved[2])
        self.v_cache.copy_(saved[3])
        self.h0.copy_(saved[4])

    def decode(self, n: int) -> None:
        """n greedy decode steps as n graph replays (no host synchronisation).

        The position is tracked on the host too: stepping past ``cfg.max_seq`` raises instead of
        writing past the KV cache (the kernels also refuse rows >= max_seq)."""
        if self._host_pos + n > self.cfg.max_seq:
            raise ValueError(f"decode({n}) from position {self._host_pos} exceeds max_seq={self.cfg.max_seq}")
        if self.graph is None:
            self.capture()
        for _ in range(n // self.STEPS_PER_GRAPH):
            self.graph_multi.replay()
        for _ in range(n % self.STEPS_PER_GRAPH):
            self.graph.replay()
        self._host_pos += n

    def reset(self) -> None:
        self._host_pos = 0
        self.k_cache.zero_()
        self.v_cache.zero_()
        self.tok.zero_()
        self.pos.zero_()


class BatchedDecoder:
    """B independent sequences decoded together, one token each per step, on a TernaryDecoder's
    weights (or its dense fp16 twin's).  Every projection runs at batch B through ``tr_linear``'s
    dispatch (the int8-slice GEMV at batch 2, the tcgen05 GEMM beyond); attention and greedy
    selection run one CTA per (sequence, head) / sequence (``tr_attn_decode_batch``,
    ``tr_greedy_next_batch``).  Prompts of equal length; each sequence keeps its own KV cache rows
    [L, B, H, S, D] and position.  decode(n) replays one captured CUDA graph per step."""

    # batches up to this run the fused int8-slice step (_step_fused); from batch 3 the GEMM (K5, the
    # dispatch's choice there) with separate RMSNorm / SwiGLU kernels is faster: B=3 2236 -> 2286,
    # B=4 2988 -> 3041 tok/s; B=2 stays fused (1989 against 1714)
    FUSED_MAX_B = 2

    def __init__(self, base: TernaryDecoder, batch: int):
        if not base.fused:
            raise ValueError("BatchedDecoder runs on the fused (libtritrun glue) decoder")
        cfg = base.cfg
        self.base, self.B, self.cfg = base, int(batch), cfg
        L, H, S, D, d = cfg.n_layers, cfg.n_heads, cfg.max_seq, cfg.head_dim, cfg.d_model
        if D != 128 or S > 128:
            raise ValueError("batched decode attention: head_dim 128, max_seq <= 128")
        dev, dt = base.device, base.dtype
        self.k_cache = torch.zeros((L, self.B, H, S, D), device=dev, dtype=dt)
        self.v_cache = torch.zeros((L, self.B, H, S, D), device=dev, dtype=dt)
        self.tok = torch.zeros(self.B, dtype=torch.long, device=dev)
        self.pos = torch.zeros(self.B, dtype=torch.long, device=dev)
        self.out_tokens = torch.zeros((self.B, S), dtype=torch.long, device=dev)
        self.h0 = torch.zeros((self.B, d), device=dev, dtype=dt)
        self._host_pos = 0
        self.graph = None

    def reset(self) -> None:
        self._host_pos = 0
        self.k_cache.zero_()
        self.v_cache.zero_()
        self.tok.zero_()
        self.pos.zero_()
        self.graph = None

    def prefill(self, prompts: torch.Tensor) -> None:
        """prompts [B, T]: each sequence's prompt through the base decoder's prompt pass, into its
        own cache rows; seeds tok / pos / the next embedding row of every sequence."""
        base, T = self.base, prompts.shape[1]
        if prompts.shape[0] != self.B or T > self.cfg.max_seq:
            raise ValueError(f"prompts must be [{self.B}, T <= {self.cfg.max_seq}]")
        kc, vc = base.k_cache, base.v_cache
        try:
            for b in range(self.B):
                base.k_cache, base.v_cache = self.k_cache[:, b], self.v_cache[:, b]
                logits = base.forward(prompts[b].to(base.device), base._positions[:T], from_start=True)
                self.tok[b] = logits.argmax()
        finally:
            base.k_cache, base.v_cache = kc, vc
        self.pos.fill_(T)
        self.h0.copy_(base.weights["embed"][self.tok])
        self._host_pos = T
        self.graph = None

    def _step(self) -> None:
        base, cfg, B = self.base, self.cfg, self.B
        if B <= self.FUSED_MAX_B and not base.dense and base.gate_up_il is not None:
            return self._step_fused()
        act, st = _ACT[base.dtype], _lib.stream_handle()
        d, H, D, S = cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.max_seq
        h = self.h0
        xn = torch.empty((B, d), device=base.device, dtype=base.dtype)
        att = torch.empty((B, d), device=base.device, dtype=base.dtype)
        delta = None
        for i in range(cfg.n_layers):
            lw = base.lin[i]
            _lib.call("tr_add_rmsnorm", act, h.data_ptr(), 0 if delta is None else delta.data_ptr(),
                      base.norm_attn[i].data_ptr(), xn.data_ptr(), B, d, cfg.eps, st)
            qkv = base._lin(xn, lw["qkv"])
            _lib.call("tr_attn_decode_batch", act, qkv.data_ptr(), self.pos.data_ptr(), base.cos.data_ptr(),
                      base.sin.data_ptr(), self.k_cache[i].data_ptr(), self.v_cache[i].data_ptr(), att.data_ptr(),
                      B, H, D, S, D ** -0.5, st)
            o = base._lin(att, lw["o"])
            _lib.call("tr_add_rmsnorm", act, h.data_ptr(), o.data_ptr(), base.norm_mlp[i].data_ptr(), xn.data_ptr(),
                      B, d, cfg.eps, st)
            a = base._swiglu(i, xn)
            delta = base._lin(a, lw["down"])
        _lib.call("tr_add_rmsnorm", act, h.data_ptr(), delta.data_ptr(), base.norm_out.data_ptr(), xn.data_ptr(),
                  B, d, cfg.eps, st)
        logits = F.linear(xn, base.weights["lm_head"])
        self.last_logits = logits   # (the graph's buffer: the latest step's logits after a replay)
        _lib.call("tr_greedy_next_batch", act, logits.data_ptr(), logits.shape[-1], self.out_tokens.data_ptr(),
                  self.out_tokens.shape[1], self.tok.data_ptr(), self.pos.data_ptr(),
                  base.weights["embed"].data_ptr(), d, self.h0.data_ptr(), B, st)

    def _step_fused(self) -> None:
        """Batch 2 (up to FUSED_MAX_B) on the int8-slice GEMV: residual add + RMSNorm fused into the qkv and gate|up
        products, SwiGLU into gate|up's epilogue (the single-sequence decode step, batched)."""
        base, cfg, B = self.base, self.cfg, self.B
        act, st = _ACT[base.dtype], _lib.stream_handle()
        d, H, D, S = cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.max_seq
        hs = [self.h0, torch.empty((B, d), device=base.device, dtype=base.dtype)]
        att = torch.empty((B, d), device=base.device, dtype=base.dtype)
        cur, delta = 0, None
        for i in range(cfg.n_layers):
            lw = base.lin[i]
            qkv = linear_pre(hs[cur], lw["qkv"], _lib.PRE_ADD_RMSNORM, delta, base.norm_attn[i], hs[1 - cur], cfg.eps,
                             pdl=True)
            cur = 1 - cur
            _lib.call("tr_attn_decode_batch", act, qkv.data_ptr(), self.pos.data_ptr(), base.cos.data_ptr(),
                      base.sin.data_ptr(), self.k_cache[i].data_ptr(), self.v_cache[i].data_ptr(), att.data_ptr(),
                      B, H, D, S, D ** -0.5, st)
            o = linear(att, lw["o"], pdl=True)
            act_ = linear_pre(hs[cur], base.gate_up_il[i], _lib.PRE_ADD_RMSNORM, o, base.norm_mlp[i], hs[1 - cur],
                              cfg.eps, pdl=True, epi_swiglu=True)
            cur = 1 - cur
            delta = linear(act_, lw["down"], pdl=True)
        xn = torch.empty((B, d), device=base.device, dtype=base.dtype)
        _lib.call("tr_add_rmsnorm", act, hs[cur].data_ptr(), delta.data_ptr(), base.norm_out.data_ptr(), xn.data_ptr(),
                  B, d, cfg.eps, st)
        logits = F.linear(xn, base.weights["lm_head"])
        self.last_logits = logits
        _lib.call("tr_greedy_next_batch", act, logits.data_ptr(), logits.shape[-1], self.out_tokens.data_ptr(),
                  self.out_tokens.shape[1], self.tok.data_ptr(), self.pos.data_ptr(),
                  base.weights["embed"].data_ptr(), d, self.h0.data_ptr(), B, st)

    def capture(self) -> None:
        cur = torch.cuda.current_stream(self.base.device)
        s = torch.cuda.Stream(device=self.base.device)
        saved = (self.tok.clone(), self.pos.clone(), self.k_cache.clone(), self.v_cache.clone(), self.h0.clone(),
                 self.out_tokens.clone())
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            self._step()   # warm-up outside capture
            s.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=s):
                self._step()
        torch.cuda.synchronize(self.base.device)
        cur.wait_stream(s)
        for t, v in zip((self.tok, self.pos, self.k_cache, self.v_cache, self.h0, self.out_tokens), saved):
            t.copy_(v)

    def decode(self, n: int) -> None:
        """n greedy steps for every sequence (out_tokens[b, pos] holds sequence b's tokens)."""
        if self._host_pos + n > self.cfg.max_seq:
            raise ValueError(f"decode({n}) from position {self._host_pos} exceeds max_seq={self.cfg.max_seq}")
        if self.graph is None:
            self.capture()
        for _ in range(n):
            self.graph.replay()
        self._host_pos += n
