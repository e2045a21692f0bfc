"""Dev A/B of decode variants on the TriLM-3.9B-shaped decoder (bench.py's decode leg): fused
QKV + attention kernel on / off, tokens/s over 64 greedy steps (best of 3), interleaved runs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder

cfg = DecoderConfig(max_seq=128)
prompt = torch.randint(0, cfg.vocab, (64,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
m = TernaryDecoder(cfg)


def measure(fa):
    m.use_fused_attention(fa)
    m.reset(); m.prefill(prompt); m.capture()
    best = None
    for _ in range(3):
        m.reset()
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); m.prefill(prompt); e[1].record(); m.decode(64); e[2].record(); e[2].synchronize()
        cur = e[1].elapsed_time(e[2])
        best = cur if best is None or cur < best else best
    toks = m.out_tokens[64:128].clone()
    return round(64 / best * 1e3, 1), toks


res = {}
for rep in range(2):
    for fa in (False, True):
        tps, toks = measure(fa)
        res.setdefault(f"fused_attn={fa}", []).append(tps)
        res.setdefault(f"tokens_{fa}", toks)
same = torch.equal(res.pop("tokens_False"), res.pop("tokens_True"))
print(json.dumps({**res, "same_tokens": same}))
