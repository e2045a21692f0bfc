import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp
rows, cols, b = (int(v) for v in sys.argv[1:4])
wb = rows * (cols // 256) * 66
R = max(3, min(32, -(-3 * 126 * 2**20 // wb)))
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(R)]
x = torch.randn(b, cols, device="cuda").half()
ys = [torch.empty(b, rows, device="cuda", dtype=torch.half) for _ in range(R)]
for probe in [int(v) for v in sys.argv[4].split(",")]:
    for ks in [int(v) for v in (sys.argv[5] if len(sys.argv) > 5 else "0").split(",")]:
        s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, path="umma", ksplit=ks, _probe=probe)
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                for w, y in zip(ws, ys): tp.linear(x, w, out=y, pdl=True, path="umma", ksplit=ks, _probe=probe)
        torch.cuda.synchronize()
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): g.replay()
        e1.record(); e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 10 / R
        print(json.dumps(dict(rows=rows, cols=cols, batch=b, probe=probe, ks=ks, us=round(us, 2), gbs=round(wb / us / 1e3, 1))), flush=True)
