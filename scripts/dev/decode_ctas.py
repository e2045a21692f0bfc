"""Dev: decode tok/s with the down projection (3072x8192: 192 tiles, 2 on the busiest CTA) and the o
projection (3072^2) on fewer CTAs, leaving SMs free for the next kernel's early launch."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_23025_b200.decoder as dec
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder

cfg = DecoderConfig(max_seq=128)
prompt = torch.randint(0, cfg.vocab, (64,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
m = TernaryDecoder(cfg)
orig = dec.linear
res = {}
for down_ctas in (0, 96, 120):
    for o_ctas in (0, 96, 128):
        def patched(x, w, *a, **k):
            if w.rows == 3072 and w.cols == 8192 and down_ctas:
                k["ctas"] = down_ctas
            if w.rows == 3072 and w.cols == 3072 and o_ctas:
                k["ctas"] = o_ctas
            return orig(x, w, *a, **k)
        dec.linear = patched
        m.graph = m.graph_multi = None
        m.reset(); m.prefill(prompt); m.capture()
        best = None
        for _ in range(3):
            m.reset(); torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(); m.prefill(prompt); e[1].record(); m.decode(64); e[2].record(); e[2].synchronize()
            t = e[1].elapsed_time(e[2])
            best = t if best is None or t < best else best
        res[f"down{down_ctas}_o{o_ctas}"] = round(64 / best * 1e3, 1)
dec.linear = orig
print(json.dumps(res))
