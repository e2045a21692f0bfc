"""Dev: per-layer time vs CTA count and warp variant (graph + PDL chain of independent layers)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
for rows, cols in [(4096, 4096), (11008, 4096), (4096, 11008), (3072, 3072), (3072, 9216)]:
    wb = rows * (cols // 256) * 66
    R = max(4, min(64, -(-3 * 126 * 2**20 // wb)))
    ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(R)]
    x = torch.randn(1, cols, device="cuda").half()
    ys = [torch.empty(1, rows, device="cuda", dtype=torch.half) for _ in range(R)]
    res = {}
    for ctas in (0, 96, 128, 192, 256, 296):
        for cs in (False, True):
            s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, ctas=ctas, cosched=cs)
                s.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, ctas=ctas, cosched=cs)
            torch.cuda.synchronize()
            for _ in range(3): g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): g.replay()
            e1.record(); e1.synchronize()
            res[f"{ctas}{'c' if cs else ''}"] = round(e0.elapsed_time(e1) * 1e3 / 10 / R, 2)
    print(json.dumps({"shape": f"{rows}x{cols}", "us": res}), flush=True)
    del ws; torch.cuda.empty_cache()
