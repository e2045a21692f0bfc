"""Dev: the BASELINE stack (bench.py workload, batch 1) with each shape's GEMV CTA width chosen
independently: half-SM 8-warp CTAs (TR_LINEAR_COSCHEDULE) or whole-SM 16-warp (TR_LINEAR_FULL_SM);
us per layer (PDL graph)."""
import sys, os, json, itertools
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
ws = bench.make_stack_weights(32, seed=1234)
x = bench.uniform_x(1, 4096, 4243)
bufs = [torch.empty((1, w.rows), dtype=torch.float16, device="cuda") for w in ws]
out = {}
for modes in itertools.product("hf", repeat=3):   # per shape: 4096^2, 11008x4096, 4096x11008
    def body():
        cur = x
        for i, (w, o) in enumerate(zip(ws, bufs)):
            m = modes[i % 3]
            tp.linear(cur, w, out=o, pdl=True, cosched=m == "h", full_sm=m == "f")
            cur = o
    s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        body(); s.synchronize()
        with torch.cuda.graph(g, stream=s):
            body()
    torch.cuda.synchronize()
    ms = bench.timed_graph(g.replay, 30, 5, None) / 30
    out["".join(modes)] = round(ms * 1e3 / len(ws), 3)
print(json.dumps(out))
