"""Dev: per-layer time for one shape under variants (dbg bits via ctas<<12)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
rows, cols, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
wb = rows * (cols // 256) * 66
R = max(4, min(64, -(-3 * 126 * 2**20 // wb)))
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(R)]
x = torch.randn(b, cols, device="cuda").half()
ys = [torch.empty(b, rows, device="cuda", dtype=torch.half) for _ in range(R)]
for variant in [int(v) for v in sys.argv[4].split(",")]:
    for pdl in (False, True):
        s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=pdl, ctas=variant)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=pdl, ctas=variant)
        torch.cuda.synchronize()
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): g.replay()
        e1.record(); e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 10 / R
        print(json.dumps(dict(rows=rows, cols=cols, batch=b, variant=hex(variant), pdl=pdl, us=round(us, 3), gbs=round((wb + b*(rows+cols)*2) / us / 1e3, 1))), flush=True)
