"""Dev: K5 CTA-0 clock trace (probe 4; needs a -DUMMA_TRACE=1 build: `bash scripts/dev/build_variant.sh trace
-DUMMA_TRACE=1`, then TRITRUN_LIB=scripts/dev/ab/trace/libtritrun.so): per block, cycles of activations landed / A decoded / MMAs issued
(MMA warp) and A buffer free / TMEM stores done (decode warp 0), relative to the first stamp."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2506_23025_b200 as tp

rows, cols, b = (int(v) for v in sys.argv[1:4])
torch.cuda.set_device(0)
ws = [tp.TernaryWeight.from_float(torch.randint(-1, 2, (rows, cols), device="cuda").float() * 0.02) for _ in range(4)]
x = (torch.rand(b, cols, device="cuda") * 2 - 1).to(torch.bfloat16 if os.environ.get("DT") == "bf16" else torch.half)
ys = [torch.zeros(b, rows, dtype=x.dtype, device="cuda") for _ in ws]
for rep in range(3):
    for w, y in zip(ws, ys):
        tp.linear(x, w, out=y, path="umma", _probe=4 | int(os.environ.get("PROBE", "0")), pdl=True)
torch.cuda.synchronize()
t = ys[-1].view(torch.int64).flatten()[: 64 * 8].cpu().numpy().reshape(64, 8)[:, :8].astype(np.float64)
nb = cols // 256
t = t[:nb]
t0 = t[t > 0].min()
t = t - t0
print(f"{rows}x{cols} b={b}: per block (cycles)  [act landed, A decoded, MMA issued | A free, st done (warp 0) | committed | st done warp 1, warp 6]")
for i in range(nb):
    print(i, " ".join(f"{v:8.0f}" for v in t[i]))
print("block period (MMA issued):", np.diff(t[:, 2]).round(0))
