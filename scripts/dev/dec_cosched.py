"""Dev: decode-step time for several TR_LINEAR_COSCHEDULE settings of the 4 decode GEMVs."""
import os, sys, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder
cfg = DecoderConfig()
m = TernaryDecoder(cfg)
prompt = torch.randint(0, cfg.vocab, (64,), device="cuda")
for combo in [(0,0,0,0),(1,1,1,1),(1,1,0,0),(0,0,1,1),(1,0,0,0),(0,1,0,0),(0,0,1,0),(0,0,0,1)]:
    m.cosched = tuple(bool(c) for c in combo)
    m.graph = None
    m.reset(); m.prefill(prompt); m.capture()
    ts = []
    for _ in range(3):
        m.reset(); m.prefill(prompt); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); m.decode(48); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 48)
    print(json.dumps({"cosched": combo, "ms_per_token": round(min(ts), 4)}), flush=True)
