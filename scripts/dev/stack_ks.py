"""Dev: the BASELINE stack at batch 16-128 (all K5) with the K split of the 4096-row shapes forced
(4096^2 / 4096x11008; 11008x4096 has 86 row tiles and runs unsplit), us per layer (PDL graph)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
ws = bench.make_stack_weights(32, seed=1234)
out = {}
for b in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "16,64,128").split(",")]:
    x = bench.uniform_x(b, 4096, 4243)
    bufs = [torch.empty((b, w.rows), dtype=torch.float16, device="cuda") for w in ws]
    for ks_a, ks_c in ((0, 0), (1, 1), (2, 2), (2, 4), (4, 2), (4, 8), (8, 4)):
        def body():
            cur = x
            for i, (w, o) in enumerate(zip(ws, bufs)):
                k = (ks_a, 0, ks_c)[i % 3]
                tp.linear(cur, w, out=o, pdl=True, ksplit=k)
                cur = o
        s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            body(); s.synchronize()
            with torch.cuda.graph(g, stream=s):
                body()
        torch.cuda.synchronize()
        ms = bench.timed_graph(g.replay, 20, 3, None) / 20
        out[f"b{b}_ks{ks_a}/{ks_c}"] = round(ms * 1e3 / len(ws), 3)
print(json.dumps(out))
