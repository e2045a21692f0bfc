"""Dev: the BASELINE stack (bench.py workload) with the GEMV grid at the SM count (default) or at the
fewest CTAs that keep the same most-tiles-per-CTA ("balanced": 4096 rows -> 128 CTAs of 2 tiles,
11008 rows -> 138 of 5), us per layer, PDL-chained graph; batch from argv (default 1,2)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
ws = bench.make_stack_weights(32, seed=1234)
out = {}
for b in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,2").split(",")]:
    x = bench.uniform_x(b, 4096, 4243)
    bufs = [torch.empty((b, w.rows), dtype=torch.float16, device="cuda") for w in ws]
    for name in ("default", "balanced"):
        def grid(w):
            if name == "default":
                return 0
            tiles = -(-w.rows // 16)
            per = -(-tiles // 148)
            return -(-tiles // per)
        def body():
            cur = x
            for w, o in zip(ws, bufs):
                tp.linear(cur, w, out=o, pdl=True, ctas=grid(w))
                cur = o
        s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            body(); s.synchronize()
            with torch.cuda.graph(g, stream=s):
                body()
        torch.cuda.synchronize()
        ms = bench.timed_graph(g.replay, 30, 5, None) / 30
        out[f"b{b}_{name}"] = round(ms * 1e3 / len(ws), 3)
print(json.dumps(out))
