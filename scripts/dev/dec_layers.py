"""Dev: decode-step time against layer count (graph replays): the tail (0 layers) and the per-layer slope."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder
res = {}
for L in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,2,10,30").split(",")]:
    cfg = DecoderConfig(n_layers=L, max_seq=128)
    m = TernaryDecoder(cfg)
    m.reset(); m.prefill(torch.randint(0, cfg.vocab, (64,), device="cuda")); m.capture()
    for _ in range(5): m.graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): m.graph.replay()
    e1.record(); e1.synchronize()
    res[L] = round(e0.elapsed_time(e1) * 1e3 / 20, 1)
    del m; torch.cuda.empty_cache()
print(json.dumps({"step_us_by_layers": res}))
