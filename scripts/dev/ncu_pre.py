"""Dev: ncu target -- linear_pre (SwiGLU or RMSNorm producer) on a decoder shape, rotating weights."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200 import _lib
from paper_2506_23025_b200.device import linear_pre
rows, cols, pre = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(8)]
if pre == 2:
    x = torch.randn(1, 2 * cols, device="cuda").half()
    for i in range(24): linear_pre(x, ws[i % 8], _lib.PRE_SILU_MUL)
else:
    x = torch.randn(1, cols, device="cuda").half(); d = torch.randn_like(x); g = torch.ones(cols, device="cuda").half()
    o = torch.empty_like(x)
    for i in range(24): linear_pre(x, ws[i % 8], _lib.PRE_ADD_RMSNORM, d, g, o)
torch.cuda.synchronize()
