"""Time the decode attention block input side: fused tr_qkv_attn_decode vs tr_linear_pre + tr_attn_decode
(H=24, D=128, S=128, pos=64), each as 30 back-to-back launches captured in a CUDA graph."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200 import _lib
from paper_2506_23025_b200.device import _ACT, linear_pre

H, D, S, L = 24, 128, 128, 30
d = H * D
tdt = torch.float16
act = _ACT[tdt]
ws = [tp.TernaryWeight.from_float(0.02 * torch.randint(-1, 2, (3 * d, d), device="cuda").float()) for _ in range(L)]
h = torch.randn((1, d), device="cuda").half()
hs = [h.clone(), h.clone()]
delta = (0.1 * torch.randn((1, d), device="cuda")).half()
gamma = torch.ones(d, device="cuda", dtype=tdt)
cos = torch.rand((S, D // 2), device="cuda").half()
sin = torch.rand((S, D // 2), device="cuda").half()
kc = torch.randn((L, H, S, D), device="cuda").half()
vc = torch.randn((L, H, S, D), device="cuda").half()
pos = torch.tensor([64], device="cuda")
qkv = torch.empty((1, 3 * d), device="cuda", dtype=tdt)
att = torch.empty((1, d), device="cuda", dtype=tdt)
cnt = torch.zeros(_lib.lib().tr_qkv_attn_decode_workspace_size(H), dtype=torch.uint8, device="cuda")


def fused(i, st, dbg=0, pp=pos):   # dbg: dev probe bits (16 = no L2 prefetch of the cache)
    _lib.call("tr_qkv_attn_decode", act, ws[i].data.data_ptr(), hs[i % 2].data_ptr(), delta.data_ptr(),
              gamma.data_ptr(), hs[1 - i % 2].data_ptr(), 1e-5, qkv.data_ptr(), pp.data_ptr(), cos.data_ptr(),
              sin.data_ptr(), kc[i].data_ptr(), vc[i].data_ptr(), att.data_ptr(), H, D, S, D ** -0.5,
              cnt.data_ptr(), cnt.numel(), _lib.LINEAR_PDL | (dbg << 16), st)


def gemv_only(i, st):
    linear_pre(hs[i % 2], ws[i], _lib.PRE_ADD_RMSNORM, delta, gamma, hs[1 - i % 2], 1e-5, pdl=True)


def unfused(i, st):
    q = linear_pre(hs[i % 2], ws[i], _lib.PRE_ADD_RMSNORM, delta, gamma, hs[1 - i % 2], 1e-5, pdl=True)
    _lib.call("tr_attn_decode", act, q.data_ptr(), pos.data_ptr(), cos.data_ptr(), sin.data_ptr(), kc[i].data_ptr(),
              vc[i].data_ptr(), att.data_ptr(), H, D, S, D ** -0.5, st)


def attn_only(i, st):
    _lib.call("tr_attn_decode", act, qkv.data_ptr(), pos.data_ptr(), cos.data_ptr(), sin.data_ptr(), kc[i].data_ptr(),
              vc[i].data_ptr(), att.data_ptr(), H, D, S, D ** -0.5, st)


pos_oor = torch.tensor([S], device="cuda")
xh = torch.randn((1, d), device="cuda").half()
res = {}
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
for name, f in (("fused", fused), ("fused_nopf", lambda i, st: fused(i, st, 16)),
                ("fused_oor", lambda i, st: fused(i, st, 0, pos_oor)),
                ("oor_noend", lambda i, st: fused(i, st, 128, pos_oor)),
                ("fused8", lambda i, st: fused(i, st, 256)),
                ("oor_std_noend", lambda i, st: fused(i, st, 64 | 128, pos_oor)),
                ("oor_std_noend_nopf", lambda i, st: fused(i, st, 64 | 128 | 16, pos_oor)),
                ("oor_noend_nopf", lambda i, st: fused(i, st, 128 | 16, pos_oor)),
                ("plain148", lambda i, st: tp.linear(xh, ws[i], out=qkv, pdl=True)),
                ("unfused", unfused), ("gemv_only", gemv_only), ("attn_only", attn_only)):
    if only and name not in only:
        continue
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st = _lib.stream_handle()
        for i in range(L):
            f(i, st)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(L):
                f(i, _lib.stream_handle())
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res[name] = round(e0.elapsed_time(e1) * 1000 / 20 / L, 2)
print(json.dumps(res))
