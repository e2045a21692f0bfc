import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200 import device
torch.manual_seed(0)
for rows, cols, batch in [(4096, 4096, 1), (4096, 4096, 8), (512, 8192, 4), (11008, 4096, 1)]:
    g = torch.Generator(device="cuda").manual_seed(rows + cols + batch)
    Wf = torch.randn(rows, cols, generator=g, device="cuda")
    w = tp.TernaryWeight.from_float(Wf)
    x = (torch.rand(batch, cols, generator=g, device="cuda") * 2 - 1).half()
    ref = x.float() @ w.dequantize(torch.float16).float().T
    for rep in range(3):
        y = tp.linear(x, w).float()
        bad = ~torch.isfinite(y)
        err = ((y - ref).abs().amax(dim=1) / ref.abs().amax(dim=1)).max().item()
        nb = int(bad.sum())
        rows_bad = torch.nonzero(bad.any(0)).flatten()[:20].tolist()
        print(rows, cols, batch, "rep", rep, "err", err, "nonfinite", nb, "rows", rows_bad, flush=True)
    ws = device._WORKSPACES
    for k, v in ws.items():
        print("ws", k, v.numel(), "nonzero counters:", int((v[: (rows // 16) * 4].view(torch.int32) != 0).sum()))
