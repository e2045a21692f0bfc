import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200 import device, _lib
for rows, cols, batch in [(1, 5, 1), (1, 5, 32), (1, 5, 40), (2, 300, 40)]:
    W = torch.randn(rows, cols, device="cuda")
    w = tp.TernaryWeight.from_float(W)
    x = torch.randn(batch, cols, device="cuda").half()
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    y = tp.linear(x, w, ws=ws)
    torch.cuda.synchronize()
    v = ws.view(torch.int32)
    nz = torch.nonzero(v).flatten()
    print(rows, cols, batch, "need", _lib.lib().tr_linear_workspace_size(2, batch, rows, cols), "nonzero idx", nz[:10].tolist(), "n", nz.numel(),
          "vals", v[nz[:5]].tolist(), "asfloat", ws.view(torch.float32)[nz[:5]].tolist(), flush=True)
