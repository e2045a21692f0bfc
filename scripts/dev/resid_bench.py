"""Dev: the residual-update forms against the old ones, 30-deep PDL graph chains (us per launch):
o projection (3072^2) plain vs tr_linear_resid; qkv GEMV (9216x3072) with the add+RMSNorm producer
vs TR_PRE_RMSNORM_TILES; both at the decoder's CTA widths."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200 import _lib
from paper_2506_23025_b200.device import linear_pre, linear_resid

L, d = 30, 3072
wo = [tp.TernaryWeight.from_float(0.02 * torch.randint(-1, 2, (d, d), device="cuda").float()) for _ in range(L)]
wq = [tp.TernaryWeight.from_float(0.02 * torch.randint(-1, 2, (3 * d, d), device="cuda").float()) for _ in range(L)]
x = torch.randn((1, d), device="cuda").half()
hs = [torch.randn((1, d), device="cuda").half() for _ in range(2)]
gam = torch.ones(d, device="cuda", dtype=torch.half)
ss = torch.rand(d // 16, device="cuda") * 100
y = torch.empty((1, d), device="cuda").half()
yq = torch.empty((1, 3 * d), device="cuda").half()
variants = {
    "o_plain_full": lambda i: tp.linear(x, wo[i], out=y, pdl=True, full_sm=True),
    "o_resid_full": lambda i: linear_resid(x, wo[i], hs[i % 2], hs[1 - i % 2], ss, out=y, pdl=True, full_sm=True),
    "o_plain_auto": lambda i: tp.linear(x, wo[i], out=y, pdl=True),
    "o_resid_auto": lambda i: linear_resid(x, wo[i], hs[i % 2], hs[1 - i % 2], ss, out=y, pdl=True),
    "qkv_pre1": lambda i: linear_pre(hs[i % 2], wq[i], _lib.PRE_ADD_RMSNORM, x, gam, hs[1 - i % 2], 1e-5, out=yq, pdl=True),
    "qkv_pre3": lambda i: linear_pre(hs[i % 2], wq[i], _lib.PRE_RMSNORM_TILES, ss, gam, None, 1e-5, out=yq, pdl=True),
    "qkv_plain": lambda i: tp.linear(hs[i % 2], wq[i], out=yq, pdl=True),
    "qkv_pre3_nostat": lambda i: _lib.call("tr_linear_pre", 2, wq[i].data.data_ptr(), hs[i % 2].data_ptr(), yq.data_ptr(),
                                           1, 3 * d, d, 1, d, 3 * d, _lib.LINEAR_PDL | ((8 << 12) << 8), 3,
                                           ss.data_ptr(), gam.data_ptr(), 0, 1e-5, _lib.stream_handle()),
}
res = {}
for name, f in variants.items():
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(L):
            f(i)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(L):
                f(i)
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
