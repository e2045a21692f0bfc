"""configs[3]: TQ1 8192x8192 per-layer time on K4 (GEMV) vs TQ2 on the same trits, batch 1-8."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2506_23025_b200 as tp

torch.cuda.set_device(0)
out = []
for fmt, bpb in ((tp.DType.TQ1, 54), (tp.DType.TQ2, 66)):
    g = torch.Generator(device="cuda").manual_seed(7)
    ws = []
    for _ in range(12):
        T = torch.randint(0, 3, (8192, 8192), generator=g, device="cuda", dtype=torch.int8).float() - 1
        gam = (0.02 * (1 + torch.rand((8192, 1), generator=g, device="cuda"))).half().float()
        ws.append(tp.TernaryWeight.from_float(gam * T, fmt))
    for b in (1, 2, 3, 4, 8):
        x = bench.uniform_x(b, 8192, 11 + b)
        for path in (("auto", "umma") if fmt is tp.DType.TQ1 and b <= 4 else ("auto",)):
            ms = bench._time_layers(ws, x, path=path)
            nbytes = 8192 * 32 * bpb + b * 16384 * 2
            out.append({"format": fmt.name, "batch": b, "path": path, "us": round(ms * 1e3, 2),
                        "gbs": round(nbytes / ms / 1e6, 1)})
    del ws
    torch.cuda.empty_cache()
print(json.dumps(out, indent=0))
