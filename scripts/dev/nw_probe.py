"""Dev: the BASELINE stack at batch 1-4 with the int8-slice GEMV at its automatic warp count or forced
to 16 warps (knob dbg 1), us per layer (PDL graph)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
ws = bench.make_stack_weights(32, seed=1234)
out = {}
for b in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4").split(",")]:
    x = bench.uniform_x(b, 4096, 4243)
    bufs = [torch.empty((b, w.rows), dtype=torch.float16, device="cuda") for w in ws]
    for name, knob, cos, path in (("auto", 0, False, "gemv"), ("cosched", 0, True, "gemv"), ("nw16", 1 << 12, False, "gemv"),
                                  ("dispatch_cosched", 0, True, "auto")):
        def body():
            cur = x
            for w, o in zip(ws, bufs):
                tp.linear(cur, w, out=o, pdl=True, ctas=knob, path=path, cosched=cos)
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
