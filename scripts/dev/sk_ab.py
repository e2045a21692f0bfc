"""Dev A/B: K5 stream-K (default for uniform-scale products with fewer tiles than SMs) against the
even split-K plan (probe 8), per-layer us in a graph + PDL chain over rotating copies (> L2)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200 as tp

res = {}
for rows, cols in ((11008, 4096), (4096, 4096), (4096, 11008)):
    g = torch.Generator(device="cuda").manual_seed(1)
    n = max(3, -(-3 * 126 * 2**20 // (rows * (cols // 256) * 66)))
    ws = []
    for _ in range(n):
        T = torch.randint(0, 3, (rows, cols), generator=g, device="cuda", dtype=torch.int8).float() - 1
        gam = (0.02 * (1 + torch.rand((rows, 1), generator=g, device="cuda"))).half().float()
        ws.append(tp.TernaryWeight.from_float(gam * T))
    for b in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "16,32,64,128").split(",")]:
        x = (torch.rand(b, cols, generator=g, device="cuda") * 2 - 1).half()
        row = {}
        for name, probe in (("sk", 0), ("split", 8)):
            ys = [torch.empty((b, rows), dtype=torch.float16, device="cuda") for _ in ws]
            s = torch.cuda.Stream(); gr = torch.cuda.CUDAGraph()
            def body():
                for w, y in zip(ws, ys):
                    tp.linear(x, w, out=y, pdl=True, path="umma", _probe=probe)
            with torch.cuda.stream(s):
                body(); s.synchronize()
                with torch.cuda.graph(gr, stream=s):
                    body()
            torch.cuda.synchronize()
            for _ in range(3):
                gr.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                gr.replay()
            e1.record(); torch.cuda.synchronize()
            row[name] = round(e0.elapsed_time(e1) * 1000 / 10 / len(ws), 2)
            row[name + "_y"] = ys[0].float()
        d = (row.pop("sk_y") - row.pop("split_y")).abs().max().item()
        row["max_abs_diff"] = d
        res[f"{rows}x{cols}_b{b}"] = row
print(json.dumps(res, indent=0))
