"""Dev: K5 time vs K split (graph + PDL chain of independent layers), several shapes / batches."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp

shapes = [(4096, 4096), (11008, 4096), (4096, 11008), (8192, 8192), (28672, 8192)]
for rows, cols in shapes:
    wb = rows * (cols // 256) * 66
    R = max(4, min(32, -(-3 * 126 * 2**20 // wb)))
    ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(R)]
    for b in (16, 64, 128):
        x = torch.randn(b, cols, device="cuda").half()
        ys = [torch.empty(b, rows, device="cuda", dtype=torch.half) for _ in range(R)]
        out = {}
        for ks in (1, 2, 3, 4, 5, 6, 8, 0):
            s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, path="umma", ksplit=ks)
                s.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, path="umma", ksplit=ks)
            torch.cuda.synchronize()
            for _ in range(3): g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): g.replay()
            e1.record(); e1.synchronize()
            out[ks] = round(e0.elapsed_time(e1) * 1e3 / 10 / R, 2)
        print(json.dumps({"shape": f"{rows}x{cols}", "batch": b, "us_by_ks": out}), flush=True)
    del ws; torch.cuda.empty_cache()
