"""Minimal launcher for ncu captures: rows cols batch [ctas] -> rotating-copy linear calls.
FMT=TQ1 in the environment packs 1.6-bit weights (K4 / K5 TQ1 paths)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_23025_b200 as tp
rows, cols, batch = (int(v) for v in sys.argv[1:4])
ctas = int(sys.argv[4]) if len(sys.argv) > 4 else 0
wb = rows * (-(-cols // 256)) * 66
copies = max(2, min(32, -(-3 * 126 * 2**20 // wb)))
def weight():   # the bench's synthetic weights: random trits, per-channel fp16 gamma
    T = torch.randint(-1, 2, (rows, cols), device="cuda").float()
    gam = (0.02 * (1 + torch.rand((rows, 1), device="cuda"))).half().float()
    return tp.TernaryWeight.from_float(gam * T, getattr(tp.DType, os.environ.get("FMT", "TQ2")))


ws = [weight() for _ in range(copies)]
x = torch.randn(batch, cols, device="cuda").half()
for i in range(3 * copies):
    tp.linear(x, ws[i % copies], ctas=ctas, cosched=os.environ.get("COSCHED") == "1")
torch.cuda.synchronize()
print("ok")
