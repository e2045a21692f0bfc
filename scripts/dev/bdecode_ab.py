"""Dev: BatchedDecoder tokens/s (ternary only) at B = 2, 3, 4, 8, 16 (bench.py's decode_batched leg; A/B via TRITRUN_LIB)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder, BatchedDecoder

torch.cuda.set_device(0)
cfg = DecoderConfig(max_seq=128)
tern = TernaryDecoder(cfg)
if os.environ.get("FUSED_MAX_B"):
    BatchedDecoder.FUSED_MAX_B = int(os.environ["FUSED_MAX_B"])
res = {}
for B in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,8,16").split(",")]:
    prompts = torch.randint(0, cfg.vocab, (B, 64), device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    bd = BatchedDecoder(tern, B)
    bd.prefill(prompts); bd.decode(1)
    best = None
    for _ in range(3):
        bd.prefill(prompts); bd.capture(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bd.decode(48); e1.record(); e1.synchronize()
        best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
    res[B] = round(B * 48 / best * 1e3, 1)
    del bd
print(os.environ.get("TRITRUN_LIB", "default"), json.dumps(res))
