import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import paper_2506_23025_b200 as tp
rows, cols, L = int(sys.argv[1]), int(sys.argv[2]), 6
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(L)]
x = torch.randn(1, cols, device="cuda").half() * 0.01
ybig = [torch.zeros(1, 148 * 8 * 4 + 148 * 32 * 4 + rows + 64, device="cuda", dtype=torch.half) for _ in range(L)]
ys = [yb[:, :rows] for yb in ybig]
def body():
    for i in range(L):
        tp.linear(x, ws[i], out=ys[i], pdl=True, ctas=(2 << 12))
s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    body(); s.synchronize()
    with torch.cuda.graph(g, stream=s):
        body()
torch.cuda.synchronize()
for _ in range(3): g.replay()
torch.cuda.synchronize()
raw = [yb.view(torch.int64)[0].cpu().numpy().astype(np.float64) for yb in ybig]
t0 = raw[0][:148 * 8].reshape(148, 8)[:, 0].min()
for i in (2, 3):
    cta = raw[i][:148 * 8].reshape(148, 8)
    wl = raw[i][148 * 8: 148 * 8 + 148 * 32].reshape(148, 32)[:, :16]
    print(f"layer {i}: start {np.median(cta[:,0]-t0)/1e3:.2f}  waited {np.median(cta[:,1]-t0)/1e3:.2f}  csum {np.median(cta[:,2]-t0)/1e3:.2f}  chunk0 {np.median(cta[:,3]-t0)/1e3:.2f}  loop4 {np.median(cta[:,4]-t0)/1e3:.2f} sync6 {np.median(cta[:,6]-t0)/1e3:.2f}/{(cta[:,6]-t0).max()/1e3:.2f} end {np.median(cta[:,5]-t0)/1e3:.2f}/{(cta[:,5]-t0).max()/1e3:.2f}")
    for c in (0, 1, 77):
        print("   cta", c, "warp loop ends:", " ".join(f"{(v - t0)/1e3:.2f}" for v in wl[c]))
