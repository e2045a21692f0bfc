"""Dev: per-CTA / per-warp phase trace of the int8-slice GEMV in a PDL graph chain (dbg=2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import paper_2506_23025_b200 as tp
rows, cols, L = int(sys.argv[1]), int(sys.argv[2]), 6
extra = int(sys.argv[3]) if len(sys.argv) > 3 else 0
NW = 16
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(L)]
x = torch.randn(1, cols, device="cuda").half() * 0.01
n = 148 * 8 * 4 + 148 * NW * 4 * 4 + rows + 64
ybig = [torch.zeros(1, n, device="cuda", dtype=torch.half) for _ in range(L)]
ys = [yb[:, :rows] for yb in ybig]
def body():
    for i in range(L):
        tp.linear(x, ws[i], out=ys[i], pdl=True, ctas=((2 | extra) << 12))
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
for i in (2, 3, 4):
    cta = raw[i][:148 * 8].reshape(148, 8)
    wt = raw[i][148 * 8: 148 * 8 + 148 * NW * 4].reshape(148, NW, 4)
    med = lambda v: np.median(v - t0) / 1e3
    print(f"layer {i}: start {med(cta[:,0]):.2f} waited {med(cta[:,1]):.2f} staged {med(cta[:,2]):.2f} end {med(cta[:,3]):.2f}/{(cta[:,3]-t0).max()/1e3:.2f}"
          f" | warp x-landed {med(wt[:,:,3]):.2f} staged {med(wt[:,:,0]):.2f} loopend med {med(wt[:,:,1]):.2f} max {(wt[:,:,1]-t0).max()/1e3:.2f} done {med(wt[:,:,2]):.2f}")
