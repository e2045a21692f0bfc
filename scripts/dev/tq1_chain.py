"""Dev: TQ1 (and TQ2) 8192^2 at batch 1 as a dependent PDL chain (each layer reads the previous
output), CTA width auto / half-SM (cosched) / whole-SM (full_sm): us per layer."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
out = {}
for fmt in (tp.DType.TQ1, tp.DType.TQ2):
    g = torch.Generator(device="cuda").manual_seed(7)
    ws = []
    for _ in range(12):
        T = torch.randint(0, 3, (8192, 8192), generator=g, device="cuda", dtype=torch.int8).float() - 1
        gam = (0.02 * (1 + torch.rand((8192, 1), generator=g, device="cuda"))).half().float()
        ws.append(tp.TernaryWeight.from_float(gam * T, fmt))
    x = bench.uniform_x(1, 8192, 11)
    bufs = [torch.empty((1, 8192), dtype=torch.float16, device="cuda") for _ in ws]
    for name, cs, fs in (("auto", False, False), ("half", True, False), ("full", False, True)):
        def body():
            cur = x
            for w, o in zip(ws, bufs):
                tp.linear(cur, w, out=o, pdl=True, cosched=cs, full_sm=fs)
                cur = o
        s = torch.cuda.Stream(); gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            body(); s.synchronize()
            with torch.cuda.graph(gr, stream=s):
                body()
        torch.cuda.synchronize()
        ms = bench.timed_graph(gr.replay, 20, 3, None) / 20
        out[f"{fmt.name}_{name}"] = round(ms * 1e3 / len(ws), 2)
    del ws
    torch.cuda.empty_cache()
print(json.dumps(out))
