"""Dev: per-layer us by path at batch 2-12 on the configs[1] shapes (the GEMV / GEMM crossover)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
res = {}
for rows, cols in ((11008, 4096), (4096, 4096), (4096, 11008), (9216, 3072), (3072, 9216)):
    g = torch.Generator(device="cuda").manual_seed(1)
    wb = rows * (cols // 256) * 66
    n = max(3, -(-3 * 126 * 2**20 // wb))
    ws = []
    for _ in range(n):
        T = torch.randint(0, 3, (rows, cols), generator=g, device="cuda", dtype=torch.int8).float() - 1
        gam = (0.02 * (1 + torch.rand((rows, 1), generator=g, device="cuda"))).half().float()
        ws.append(tp.TernaryWeight.from_float(gam * T))
    for b in (2, 3, 4, 5, 6, 8, 12):
        x = bench.uniform_x(b, cols, b)
        row = {}
        for path in ("gemv", "gemv_f16", "umma"):
            try:
                row[path] = round(bench._time_layers(ws, x, path=path) * 1e3, 2)
            except Exception as e:
                row[path] = None
        res[f"{rows}x{cols}_b{b}"] = row
    del ws
    torch.cuda.empty_cache()
print(json.dumps(res))
