"""Dev: K5 split-K sweep at the configs[1] shapes: per-layer us (graph + PDL, rotating copies > L2)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
res = {}
for rows, cols in ((11008, 4096), (4096, 4096), (4096, 11008)):
    g = torch.Generator(device="cuda").manual_seed(1)
    wb = rows * (cols // 256) * 66
    n = max(3, -(-3 * 126 * 2**20 // wb))
    ws = []
    for _ in range(n):
        T = torch.randint(0, 3, (rows, cols), generator=g, device="cuda", dtype=torch.int8).float() - 1
        gam = (0.02 * (1 + torch.rand((rows, 1), generator=g, device="cuda"))).half().float()
        ws.append(tp.TernaryWeight.from_float(gam * T))
    for b in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "16,32,64,128").split(",")]:
        x = bench.uniform_x(b, cols, b)
        row = {}
        for ks in range(0, 11):
            ys = [torch.empty((b, w.rows), dtype=torch.float16, device="cuda") for w in ws]
            s = torch.cuda.Stream(); gr = torch.cuda.CUDAGraph()
            def body():
                for w, y in zip(ws, ys):
                    tp.linear(x, w, out=y, pdl=True, path="umma", ksplit=ks)
            with torch.cuda.stream(s):
                body(); s.synchronize()
                with torch.cuda.graph(gr, stream=s):
                    body()
            torch.cuda.synchronize()
            ms = bench.timed_graph(gr.replay, 10, 3, None) / 10 / len(ws)
            row[ks] = round(ms * 1e3, 2)
        res[f"{rows}x{cols}_b{b}"] = row
    del ws
    torch.cuda.empty_cache()
print(json.dumps(res, indent=0))
