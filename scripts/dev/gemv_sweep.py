"""Dev: per-layer time of tr_linear over chained copies (CUDA graph, PDL), several shapes/batches."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200.graph import LinearStack

shapes = [(4096, 4096), (11008, 4096), (4096, 11008), (8192, 8192), (28672, 8192), (8192, 28672)]
batches = [int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16,32").split(",")]
paths = (sys.argv[2] if len(sys.argv) > 2 else "auto").split(",")
shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[3].split(",")] if len(sys.argv) > 3 else shapes
res = []
for rows, cols in shapes:
    wb = rows * (cols // 256) * 66
    R = max(4, min(64, -(-3 * 126 * 2**20 // wb)))
    # a square-chain requires rows == cols; use independent layers fed by the same x instead
    ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(R)]
    for b in batches:
        x = torch.randn(b, cols, device="cuda").half()
        ys = [torch.empty(b, rows, device="cuda", dtype=torch.half) for _ in range(R)]
        for pdl, path in [(True, p) for p in paths]:
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                for w, y in zip(ws, ys):
                    tp.linear(x, w, out=y, pdl=pdl, path=path)
                s.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for w, y in zip(ws, ys):
                        tp.linear(x, w, out=y, pdl=pdl, path=path)
            torch.cuda.synchronize()
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 10
            e0.record()
            for _ in range(n):
                g.replay()
            e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / n / R
            nbytes = wb + b * (rows + cols) * 2
            res.append(dict(rows=rows, cols=cols, batch=b, path=path, tflops=round(2*rows*cols*b/us/1e6, 1), us=round(us, 3), gbs=round(nbytes / us / 1e3, 1)))
            print(json.dumps(res[-1]), flush=True)
        # correctness spot check vs dense
        dense = ws[0].dequantize(torch.float16).float()
        ref = x.float() @ dense.T
        err = ((ys[0].float() - ref).abs().amax(1) / ref.abs().amax(1)).max().item()
        print(json.dumps(dict(rows=rows, cols=cols, batch=b, relerr=err)), flush=True)
    del ws
    torch.cuda.empty_cache()
