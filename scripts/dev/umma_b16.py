"""Dev: K5 per-layer us at b = 16 / 32 on the configs[1] shapes (graph + PDL, rotating copies > L2);
run under different TRITRUN_LIB builds for A/B; DT=bf16 for bfloat16 activations."""
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
    for b in (16, 32):
        x = bench.uniform_x(b, cols, b, torch.bfloat16 if os.environ.get("DT") == "bf16" else None)
        res[f"{rows}x{cols}_b{b}"] = round(bench._time_layers(ws, x, path="umma") * 1e3, 2)
    del ws
    torch.cuda.empty_cache()
print(os.environ.get("TRITRUN_LIB", "default"), json.dumps(res))
