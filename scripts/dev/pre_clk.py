"""Dev: per-warp SM-cycle phases (dbg=2 trace) of the plain int8-slice GEMV vs the add+RMSNorm producer
variant (the fused QKV kernel with its attention tail switched off), 9216x3072, 144 CTAs of 8 warps,
in a PDL graph chain: cycles from griddepcontrol.wait to x landed / staged / main loop done / stored."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200 import _lib
from paper_2506_23025_b200.device import _ACT

H, D, S, L, NW = 24, 128, 128, 6, 8
d = H * D
rows, cols = 3 * d, d
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(L)]
x = torch.randn(1, cols, device="cuda").half()
hs = [x.clone(), x.clone()]
delta = (0.1 * torch.randn((1, d), device="cuda")).half()
gamma = torch.ones(d, device="cuda", dtype=torch.half)
cs = torch.rand((S, D // 2), device="cuda").half()
kc = torch.randn((H, S, D), device="cuda").half()
att = torch.empty((1, d), device="cuda").half()
pos_oor = torch.tensor([S], device="cuda")
cnt = torch.zeros(4 * H, dtype=torch.uint8, device="cuda")
n = 148 * 8 * 4 + 148 * NW * 4 * 4 + rows + 64
ybig = [torch.zeros(1, n, device="cuda", dtype=torch.half) for _ in range(L)]


def plain(i):
    tp.linear(x, ws[i], out=ybig[i][:, :rows], pdl=True, ctas=(2 << 12) | 144, cosched=True)


def pre(i):
    _lib.call("tr_qkv_attn_decode", _ACT[torch.half], ws[i].data.data_ptr(), hs[i % 2].data_ptr(), delta.data_ptr(),
              gamma.data_ptr(), hs[1 - i % 2].data_ptr(), 1e-5, ybig[i].data_ptr(), pos_oor.data_ptr(), cs.data_ptr(),
              cs.data_ptr(), kc.data_ptr(), kc.data_ptr(), att.data_ptr(), H, D, S, D ** -0.5, cnt.data_ptr(),
              cnt.numel(), _lib.LINEAR_PDL | ((2 | 16 | 64 | 128) << 16), _lib.stream_handle())


for name, f in (("plain", plain), ("pre", pre)):
    s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(L):
            f(i)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(L):
                f(i)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    raw = [yb.view(torch.int64)[0].cpu().numpy() for yb in ybig]
    for i in (3, 4):
        wt = raw[i][148 * 8: 148 * 8 + 144 * NW * 4].reshape(144, NW, 4).astype(np.float64)
        ct = raw[i][: 144 * 8].reshape(144, 8).astype(np.float64)
        print(f"{name} layer {i}: " + "  ".join(
            f"{nm} med {np.median(wt[:, :, k]):.0f} max {wt[:, :, k].max():.0f}"
            for k, nm in ((3, "x_landed"), (1, "loop_done|pass1"), (2, "stored|synced"), (0, "staged"))) + " (cycles)"
            + f"  cta start->wait med {np.median(ct[:, 1] - ct[:, 0]):.0f} ns, start spread {ct[:, 0].max() - ct[:, 0].min():.0f} ns,"
            + f" end spread {ct[:, 3].max() - ct[:, 3].min():.0f} ns, wait-rel->end max {(ct[:, 3] - ct[:, 1].min()).max():.0f} ns")
