"""Diagnostics: time the GEMV with parts of the work disabled (dev tool)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_23025_b200 as tp
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe_gemv import graph_time

for (rows, cols) in [(28672, 8192), (8192, 8192)]:
    wb = rows * (-(-cols // 256)) * 66
    copies = max(2, min(64, -(-3 * 126 * 2**20 // wb)))
    ws = [tp.TernaryWeight.from_float(torch.randn(rows, cols, device="cuda")) for _ in range(copies)]
    for batch in (1, 8):
        x = torch.randn(batch, cols, device="cuda").half()
        out = torch.empty(batch, rows, device="cuda", dtype=torch.half)
        for dbg in (0, 1, 2):
            t = graph_time([(lambda w=w: tp.linear(x, w, out=out, pdl=True, _dbg=dbg)) for w in ws])
            print(json.dumps(dict(rows=rows, cols=cols, batch=batch, dbg=dbg, us=round(t / 1e3, 2), gbs=round(wb / t))), flush=True)
