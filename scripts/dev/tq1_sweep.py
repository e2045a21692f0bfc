import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
rows, cols = 8192, 8192
for fmt, bpb in ((tp.DType.TQ1, 54), (tp.DType.TQ2, 66)):
    wb = rows * (cols // 256) * bpb
    R = max(4, min(32, -(-3 * 126 * 2**20 // wb)))
    def weight():
        T = torch.randint(-1, 2, (rows, cols), device="cuda").float()
        gam = (0.02 * (1 + torch.rand((rows, 1), device="cuda"))).half().float()
        return tp.TernaryWeight.from_float(gam * T, fmt)
    ws = [weight() for _ in range(R)]
    for b in (1, 8, 16, 64, 128):
        for path in (("umma",) if fmt is tp.DType.TQ1 else ("gemv", "umma")):
            if path == "gemv" and b > 8: continue
            x = torch.randn(b, cols, device="cuda").half()
            ys = [torch.empty(b, rows, device="cuda", dtype=torch.half) for _ in range(R)]
            s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, path=path)
                s.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, path=path)
            torch.cuda.synchronize()
            for _ in range(3): g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): g.replay()
            e1.record(); e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 10 / R
            print(json.dumps(dict(fmt=fmt.name, path=path, batch=b, us=round(us, 2), gbs=round((wb + b * (rows + cols) * 2) / us / 1e3, 1), tflops=round(2 * rows * cols * b / us / 1e6, 1))), flush=True)
    del ws
    torch.cuda.empty_cache()
