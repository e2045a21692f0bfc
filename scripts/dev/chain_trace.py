"""Dev: globaltimer stamps of consecutive PDL-chained GEMV layers (dbg bit 2 -> stamps into y)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import paper_2506_23025_b200 as tp
rows, cols, L = int(sys.argv[1]), int(sys.argv[2]), 8
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(L)]
x = torch.randn(1, cols, device="cuda").half() * 0.01
ybig = [torch.zeros(1, max(rows, 148 * 32) + 64, device="cuda", dtype=torch.half) for _ in range(L)]
ys = [yb[:, :rows] for yb in ybig]
def body(pdl):
    for i in range(L):
        tp.linear(x, ws[i], out=ys[i], pdl=pdl, ctas=(2 << 12))
for pdl in (True, False):
    s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        body(pdl); s.synchronize()
        with torch.cuda.graph(g, stream=s):
            body(pdl)
    torch.cuda.synchronize()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    t = np.stack([yb.view(torch.int64)[0, :148 * 8].view(148, 8).cpu().numpy() for yb in ybig]).astype(np.float64)
    t0 = t[0, :, 0].min()
    print("pdl", pdl)
    names = ["start", "waited", "csum", "chunk0", "loopend", "end"]
    for i in range(L):
        v = (t[i] - t0) / 1e3
        print(f" layer {i}: " + " ".join(f"{n}={np.median(v[:, k]):6.2f}/{v[:, k].max():6.2f}" for k, n in enumerate(names)))
