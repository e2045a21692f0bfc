"""Dev: 8- vs 16-warp K3-S8 per decoder / BASELINE shape (graph + PDL chain of independent layers)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
for rows, cols in [(9216, 3072), (3072, 3072), (18432, 3072), (3072, 9216), (4096, 4096), (11008, 4096), (4096, 11008)]:
    wb = rows * (cols // 256) * 66
    R = max(4, min(64, -(-3 * 126 * 2**20 // wb)))
    ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(R)]
    x = torch.randn(1, cols, device="cuda").half()
    ys = [torch.empty(1, rows, device="cuda", dtype=torch.half) for _ in range(R)]
    res = {}
    for name, kw in [("auto", {}), ("w8", {"cosched": True}), ("w16", {"ctas": 1 << 12}),
                     ("auto_pre1", {"ctas": 8 << 12}), ("w8_pre1", {"cosched": True, "ctas": 8 << 12}),
                     ("w16_pre1", {"ctas": 9 << 12})]:
        s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, **kw)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, **kw)
        torch.cuda.synchronize()
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): g.replay()
        e1.record(); e1.synchronize()
        res[name] = round(e0.elapsed_time(e1) * 1e3 / 10 / R, 2)
    print(json.dumps({"shape": f"{rows}x{cols}", "us": res}), flush=True)
    del ws; torch.cuda.empty_cache()
