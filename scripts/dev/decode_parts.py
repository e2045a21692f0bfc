"""Dev: where one decode step's time goes -- CUDA-graph timings of each op type chained 30x (PDL)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200 import _lib
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder
from paper_2506_23025_b200.device import _ACT, linear, linear_pre

cfg = DecoderConfig()
m = TernaryDecoder(cfg)
d, f, H, D, S, L = cfg.d_model, cfg.d_ff, cfg.n_heads, cfg.head_dim, cfg.max_seq, cfg.n_layers
act, dev = _ACT[m.dtype], m.device
m.pos.fill_(64)
h = [torch.randn(1, d, device=dev).half() * 0.1 for _ in range(2)]
qkv = torch.randn(1, 3 * d, device=dev).half() * 0.1
att = torch.randn(1, d, device=dev).half() * 0.1
gu = torch.randn(1, 2 * f, device=dev).half() * 0.1
out_q = torch.empty(1, 3 * d, device=dev).half()
out_d = torch.empty(1, d, device=dev).half()
out_gu = torch.empty(1, 2 * f, device=dev).half()


def timeit(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): g.replay()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


st = lambda: _lib.stream_handle()
parts = {
    "qkv (rmsnorm fused)": lambda: [linear_pre(h[0], m.lin[i]["qkv"], _lib.PRE_ADD_RMSNORM, h[1], m.norm_attn[i], h[1 - 0] if False else h[1].clone() if False else out_d, cfg.eps, out=out_q, pdl=True) for i in range(L)],
    "attention": lambda: [_lib.call("tr_attn_decode", act, qkv.data_ptr(), m.pos.data_ptr(), m.cos.data_ptr(), m.sin.data_ptr(),
                                    m.k_cache[i].data_ptr(), m.v_cache[i].data_ptr(), att.data_ptr(), H, D, S, D ** -0.5, st()) for i in range(L)],
    "o": lambda: [linear(att, m.lin[i]["o"], out=out_d, pdl=True) for i in range(L)],
    "gate_up (rmsnorm fused)": lambda: [linear_pre(h[0], m.lin[i]["gate_up"], _lib.PRE_ADD_RMSNORM, h[1], m.norm_mlp[i], out_d, cfg.eps, out=out_gu, pdl=True) for i in range(L)],
    "down (swiglu fused)": lambda: [linear_pre(gu, m.lin[i]["down"], _lib.PRE_SILU_MUL, out=out_d, pdl=True) for i in range(L)],
}
if m.gate_up_il is not None:
    out_a = torch.empty(1, f, device=dev).half()
    parts["gate_up (rmsnorm + swiglu epilogue)"] = lambda: [linear_pre(h[0], m.gate_up_il[i], _lib.PRE_ADD_RMSNORM, h[1], m.norm_mlp[i], out_d, cfg.eps, out=out_a, pdl=True, epi_swiglu=True) for i in range(L)]
    parts["down (plain)"] = lambda: [linear(gu[:, :f], m.lin[i]["down"], out=out_d, pdl=True) for i in range(L)]
res = {k: round(timeit(v) / L, 2) for k, v in parts.items()}
m.reset(); m.prefill(torch.randint(0, cfg.vocab, (64,), device=dev)); m.capture()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): m.graph.replay()
e1.record(); e1.synchronize()
res["full step (ms)"] = round(e0.elapsed_time(e1) / 20, 4)
if m.gate_up_il is not None:   # A/B: the same model with the SwiGLU staged in the down GEMV
    m.gate_up_il = None
    m.reset(); m.prefill(torch.randint(0, cfg.vocab, (64,), device=dev)); m.capture()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20): m.graph.replay()
    e1.record(); e1.synchronize()
    res["full step, no epilogue (ms)"] = round(e0.elapsed_time(e1) / 20, 4)
res["sum of 30 layers (ms)"] = round(sum(v for k, v in res.items() if "ms" not in k and "epilogue" not in k and "plain" not in k) * L / 1e3, 4)
print(json.dumps(res))
