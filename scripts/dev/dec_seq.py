"""Dev: per-layer time of decode-op sequences chained 30x in one graph (PDL), to locate transition costs."""
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
hs = [torch.randn(1, d, device=dev).half() * 0.1 for _ in range(2)]
qkv = torch.empty(1, 3 * d, device=dev).half()
att = torch.randn(1, d, device=dev).half() * 0.1
o = torch.randn(1, d, device=dev).half() * 0.1
a = torch.randn(1, f, device=dev).half() * 0.1
dl = torch.randn(1, d, device=dev).half() * 0.1
st = lambda: _lib.stream_handle()
ops = {
    "q": lambda i: linear_pre(hs[0], m.lin[i]["qkv"], _lib.PRE_ADD_RMSNORM, dl, m.norm_attn[i], hs[1], cfg.eps, out=qkv, pdl=True),
    "A": lambda i: _lib.call("tr_attn_decode", act, qkv.data_ptr(), m.pos.data_ptr(), m.cos.data_ptr(), m.sin.data_ptr(),
                             m.k_cache[i].data_ptr(), m.v_cache[i].data_ptr(), att.data_ptr(), H, D, S, D ** -0.5, st()),
    "o": lambda i: linear(att, m.lin[i]["o"], out=o, pdl=True),
    "g": lambda i: linear_pre(hs[1], m.gate_up_il[i], _lib.PRE_ADD_RMSNORM, o, m.norm_mlp[i], hs[0], cfg.eps, out=a, pdl=True, epi_swiglu=True),
    "d": lambda i: linear(a, m.lin[i]["down"], out=dl, pdl=True),
}


def timeit(seq, n=20):
    fn = lambda: [ops[c](i) for i in range(L) for c in seq]
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
    return round(e0.elapsed_time(e1) * 1e3 / n / L, 2)


res = {seq: timeit(seq) for seq in sys.argv[1].split(",")}
print(json.dumps(res))
