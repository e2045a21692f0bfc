"""Dev: per-warp SM-cycle phases of the int8-slice GEMV (dbg=2 trace) in a PDL graph chain of one shape:
cycles from griddepcontrol.wait to x landed / staged / main loop done / stored (median and max over warps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
import paper_2506_23025_b200 as tp
rows, cols, L = int(sys.argv[1]), int(sys.argv[2]), 6
NW = int(sys.argv[3]) if len(sys.argv) > 3 else 16
extra = (1 if NW == 16 else 0) | (int(sys.argv[4]) if len(sys.argv) > 4 else 0)   # + ring-order probe bits 4/8
fmt = getattr(tp.DType, os.environ.get("FMT", "TQ2"))
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02, fmt) for _ in range(L)]
x = torch.randn(1, cols, device="cuda").half() * 0.01
n = 148 * 8 * 4 + 148 * NW * 4 * 4 + rows + 64
ybig = [torch.zeros(1, n, device="cuda", dtype=torch.half) for _ in range(L)]
ys = [yb[:, :rows] for yb in ybig]
def body():
    for i in range(L):
        tp.linear(x, ws[i], out=ys[i], pdl=True, ctas=((2 | extra) << 12), cosched=(NW == 8))
s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    body(); s.synchronize()
    with torch.cuda.graph(g, stream=s):
        body()
torch.cuda.synchronize()
for _ in range(3): g.replay()
torch.cuda.synchronize()
raw = [yb.view(torch.int64)[0].cpu().numpy() for yb in ybig]
for i in (3,):
    wt = raw[i][148 * 8: 148 * 8 + 148 * NW * 4].reshape(148, NW, 4).astype(np.float64)
    names = ["staged", "loop_done", "stored", "x_landed"]
    print(f"{rows}x{cols} NW={NW} probe={extra & 12}: " + "  ".join(f"{nm} med {np.median(wt[:,:,k]):.0f} max {wt[:,:,k].max():.0f}"
                                               for k, nm in ((3, 'x_landed'), (0, 'staged'), (1, 'loop_done'), (2, 'stored'))) + " (cycles)")
