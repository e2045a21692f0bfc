"""Dev: decode tok/s (bench.py's decode leg) over the fused-attention switch and the GEMV CTA width
(TR_LINEAR_FULL_SM / TR_LINEAR_COSCHEDULE) of the decode projections."""
import os, sys, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder

cfg = DecoderConfig(max_seq=128)
prompt = torch.randint(0, cfg.vocab, (64,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
m = TernaryDecoder(cfg)
res = {}
for fa in (False,):
    for fs in [(False, True, False, False), (True, True, False, False), (False, False, False, False)]:
        m.use_fused_attention(fa)
        m.full_sm = fs
        m.cosched = (False, False, False, False)
        m.reset(); m.prefill(prompt); m.capture()
        best = None
        for _ in range(3):
            m.reset(); torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(); m.prefill(prompt); e[1].record(); m.decode(64); e[2].record(); e[2].synchronize()
            t = e[1].elapsed_time(e[2])
            best = t if best is None or t < best else best
        res[f"fa={int(fa)} full_sm={''.join(str(int(v)) for v in fs)}"] = round(64 / best * 1e3, 1)
print(json.dumps(res))
