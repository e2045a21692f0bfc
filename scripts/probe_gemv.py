"""Quick device-time probe of the GEMV path vs cuBLAS fp16 (dev tool, not the bench)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200.perf import time_rotating
import statistics

def run(rows, cols, batch, ks=0, copies=None):
    wb = rows * (-(-cols // 256)) * 66
    copies = copies or max(1, min(64, -(-3 * 126 * 2**20 // wb)))
    ws = [tp.TernaryWeight.from_float(torch.randn(rows, cols, device="cuda")) for _ in range(copies)]
    x = torch.randn(batch, cols, device="cuda").half()
    out = torch.empty(batch, rows, device="cuda", dtype=torch.half)
    t = statistics.median(time_rotating([(lambda w=w: tp.linear(x, w, out=out, ksplit=ks)) for w in ws], 50, 5))
    # graph of all copies back to back with PDL
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for w in ws: tp.linear(x, w, out=out, pdl=True, ksplit=ks)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for w in ws: tp.linear(x, w, out=out, pdl=True, ksplit=ks)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(10): g.replay()
    b.record(); b.synchronize()
    tg = a.elapsed_time(b) * 1e6 / 10 / copies
    d16 = [w.dequantize() for w in ws[:max(1, min(copies, -(-3 * 126 * 2**20 // (rows*cols*2))))]]
    tc = statistics.median(time_rotating([(lambda w=w: torch.nn.functional.linear(x, w)) for w in d16], 50, 5))
    return dict(rows=rows, cols=cols, batch=batch, ks=ks, us=t/1e3, gbs=wb/t, graph_us=tg/1e3, graph_gbs=wb/tg,
                cublas_us=tc/1e3, cublas_gbs=rows*cols*2/tc, speedup_graph=tc/tg)

for (r, c) in [(4096, 4096), (11008, 4096), (4096, 11008), (8192, 8192), (28672, 8192), (8192, 28672)]:
    for b in (1, 8, 16, 32):
        print(json.dumps(run(r, c, b)), flush=True)
