"""Dev: the BASELINE stack (bench.py workload) as PDL-chained int8-slice GEMVs under ring-order
probes (tr_linear knob bits 12-15): us per layer for each variant."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
ws = bench.make_stack_weights(32, seed=1234)
x = bench.uniform_x(1, 4096, 4243)
bufs = [torch.empty((1, w.rows), dtype=torch.float16, device="cuda") for w in ws]
out = {}
for probe in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,4,8,12").split(",")]:
    for cos in (True, False):
        def body():
            cur = x
            for w, o in zip(ws, bufs):
                tp.linear(cur, w, out=o, pdl=True, cosched=cos, ctas=(probe << 12))
                cur = o
        s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            body(); s.synchronize()
            with torch.cuda.graph(g, stream=s):
                body()
        torch.cuda.synchronize()
        ms = bench.timed_graph(g.replay, 30, 5, None) / 30
        out[f"probe{probe}_{'cosched' if cos else 'auto'}"] = round(ms * 1e3 / len(ws), 3)
print(json.dumps(out))
