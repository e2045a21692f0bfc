import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2506_23025_b200 as tp
g = torch.Generator(device="cuda").manual_seed(3)
res = {}
for rows, cols in ((28672, 8192), (8192, 28672)):
    ws = []
    for _ in range(4):
        T = torch.randint(0, 3, (rows, cols), generator=g, device="cuda", dtype=torch.int8).float() - 1
        ws.append(tp.TernaryWeight.from_float(0.02 * T))
    x = bench.uniform_x(1, cols, 5)
    res[f"{rows}x{cols}"] = round(bench._time_layers(ws, x) * 1e3, 2)
print(json.dumps(res))
