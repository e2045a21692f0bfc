"""Dev: decode tok/s (bench.py's decode leg) by decode steps per CUDA graph replay."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder

cfg = DecoderConfig(max_seq=128)
prompt = torch.randint(0, cfg.vocab, (64,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
m = TernaryDecoder(cfg)
res = {}
for k in (8, 16, 32, 64):
    m.STEPS_PER_GRAPH = k
    m.graph = m.graph_multi = None
    m.reset(); m.prefill(prompt); m.capture()
    best = None
    for _ in range(3):
        m.reset(); torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); m.prefill(prompt); e[1].record(); m.decode(64); e[2].record(); e[2].synchronize()
        t = e[1].elapsed_time(e[2])
        best = t if best is None or t < best else best
    res[k] = round(64 / best * 1e3, 1)
print(json.dumps(res))
