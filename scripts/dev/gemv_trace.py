"""Dev: per-CTA globaltimer trace of one GEMV launch (dbg bit 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import paper_2506_23025_b200 as tp
rows, cols, b, dbg = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(4)]
x = torch.randn(b, cols, device="cuda").half()
y = torch.zeros(max(b * rows, 148 * 32), device="cuda", dtype=torch.half)
for i in range(8):
    tp.linear(x, ws[i % 4], out=y[: b * rows].view(b, rows), ctas=(dbg << 12))
torch.cuda.synchronize()
t = y.view(torch.int64)[: 148 * 8].view(148, 8).cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
names = ["start", "after_wait", "after_csum", "first_chunk", "loop_end", "end"]
for k, n in enumerate(names):
    v = (t[:, k] - t0) / 1e3
    print(f"{n:12s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
