"""Per-warp timeline of one GEMV launch (globaltimer ns): start, after griddep wait,
after x staging, first data, loop end, after flushes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_23025_b200 as tp
for rows, cols, batch, dbg in [(28672, 8192, 1, 4), (28672, 8192, 1, 5), (4096, 4096, 1, 4)]:
    ws_list = [tp.TernaryWeight.from_float(torch.randn(rows, cols, device="cuda")) for _ in range(3)]
    x = torch.randn(batch, cols, device="cuda").half()
    buf = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    for i in range(3):
        tp.linear(x, ws_list[i % 3], ws=buf, _dbg=0)
    torch.cuda.synchronize()
    buf.zero_()
    tp.linear(x, ws_list[0], ws=buf, _dbg=dbg)
    torch.cuda.synchronize()
    ts = buf[256 * 1024 + (32 << 20):].view(torch.int64)[: 296 * 8 * 8].view(-1, 8)[:, :6].double()
    ts = ts[ts[:, 0] > 0]
    t0 = ts[:, 0].min()
    rel = (ts - t0) / 1000.0
    names = ["start", "griddep", "staged", "first", "loopend", "end"]
    q = lambda v: [round(float(torch.quantile(v, p)), 2) for p in (0.0, 0.5, 0.9, 1.0)]
    print(f"{rows}x{cols} b{batch} dbg{dbg}: warps {rel.shape[0]}  (us: min/median/p90/max)")
    for i, n in enumerate(names):
        print(f"   {n:8s} {q(rel[:, i])}")
