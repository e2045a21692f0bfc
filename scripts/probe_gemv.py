"""Device-time probe of the GEMV path vs cuBLAS fp16 (dev tool, not the bench).

usage: probe_gemv.py [shape-set] ; prints one JSON line per (shape, batch, rt, ks)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_23025_b200 as tp
from paper_2506_23025_b200.perf import time_rotating

def graph_time(fns, reps=10):
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for f in fns: f()
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for f in fns: f()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): g.replay()
    b.record(); b.synchronize()
    return a.elapsed_time(b) * 1e6 / reps / len(fns)

def run(rows, cols, batch, ks=0, cublas=True):
    wb = rows * (-(-cols // 256)) * 66
    copies = max(2, min(64, -(-3 * 126 * 2**20 // wb)))
    ws = [tp.TernaryWeight.from_float(torch.randn(rows, cols, device="cuda")) for _ in range(copies)]
    x = torch.randn(batch, cols, device="cuda").half()
    out = torch.empty(batch, rows, device="cuda", dtype=torch.half)
    t = statistics.median(time_rotating([(lambda w=w: tp.linear(x, w, out=out, ksplit=ks)) for w in ws], 30, 5))
    tg = graph_time([(lambda w=w: tp.linear(x, w, out=out, pdl=True, ksplit=ks)) for w in ws])
    r = dict(rows=rows, cols=cols, batch=batch, ks=ks, us=round(t/1e3, 2), gbs=round(wb/t), graph_us=round(tg/1e3, 2),
             graph_gbs=round(wb/tg))
    if cublas:
        n16 = max(2, min(copies, -(-3 * 126 * 2**20 // (rows*cols*2))))
        d16 = [w.dequantize() for w in ws[:n16]]
        tc = graph_time([(lambda w=w: torch.nn.functional.linear(x, w)) for w in d16])
        r.update(cublas_us=round(tc/1e3, 2), cublas_gbs=round(rows*cols*2/tc), speedup=round(tc/tg, 2))
    del ws
    torch.cuda.empty_cache()
    return r

def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "tune"
    if mode == "tune":
        for (r, c) in [(4096, 4096), (8192, 8192), (28672, 8192), (8192, 28672)]:
            for ks in (0, 1, 2, 4):
                print(json.dumps(run(r, c, 1, ks, cublas=(ks == 0))), flush=True)
    else:
        for (r, c) in [(4096, 4096), (11008, 4096), (4096, 11008), (8192, 8192), (28672, 8192), (8192, 28672)]:
            for b in (1, 4, 8, 16, 32):
                print(json.dumps(run(r, c, b)), flush=True)


if __name__ == "__main__":
    main()
