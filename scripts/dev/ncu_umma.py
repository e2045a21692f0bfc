import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
rows, cols, b, ks = (int(v) for v in sys.argv[1:5])
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(3)]
x = torch.randn(b, cols, device="cuda").half()
for i in range(9):
    tp.linear(x, ws[i % 3], path="umma", ksplit=ks)
torch.cuda.synchronize()
