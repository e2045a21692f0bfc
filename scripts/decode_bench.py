"""Config (3): TriLM-3.9B-shaped decoder, 64-token prompt + 64 greedy output tokens, ternary vs fp16 cuBLAS.

Prints one JSON line: TTFT (prefill) and decode tokens/s for both, and the speed-up.
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder

p = argparse.ArgumentParser()
p.add_argument("--layers", type=int, default=30)
p.add_argument("--prompt", type=int, default=64)
p.add_argument("--gen", type=int, default=64)
p.add_argument("--reps", type=int, default=5)
a = p.parse_args()
cfg = DecoderConfig(n_layers=a.layers, max_seq=a.prompt + a.gen)
torch.cuda.set_device(0)
prompt = torch.randint(0, cfg.vocab, (a.prompt,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))


def first_logits(model):   # the first decode step's logits (eager), for the logit-level comparison
    model.reset()
    model.prefill(prompt, graph=False)
    return model.forward(model.tok, model.pos).float()


def measure(model):
    model.reset()
    model.prefill(prompt)
    model.capture()
    ttft, dec = [], []
    for _ in range(a.reps):
        model.reset()
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        model.prefill(prompt)
        e[1].record()
        model.decode(a.gen)
        e[2].record()
        e[2].synchronize()
        ttft.append(e[0].elapsed_time(e[1]))
        dec.append(e[1].elapsed_time(e[2]))
    ttft.sort(); dec.sort()
    return ttft[len(ttft) // 2], dec[len(dec) // 2], model.out_tokens[a.prompt:a.prompt + a.gen].clone()


tern = TernaryDecoder(cfg)
t_ttft, t_dec, t_out = measure(tern)
t_logits = first_logits(tern)
dense = TernaryDecoder(cfg, dense=True, weights=tern.weights)
del tern
d_ttft, d_dec, d_out = measure(dense)
d_logits = first_logits(dense)
top2 = d_logits.topk(2).values
agree = int((t_out == d_out).sum())
res = {"config": "trilm_3.9b_decoder", "layers": cfg.n_layers, "params": cfg.n_params(), "prompt": a.prompt,
       "generated": a.gen, "ternary_bytes_per_token": cfg.ternary_bytes() + cfg.vocab * cfg.d_model * 2,
       "ternary": {"ttft_ms": round(t_ttft, 3), "decode_ms": round(t_dec, 3), "tokens_per_s": round(a.gen / t_dec * 1e3, 1)},
       "fp16_cublas": {"ttft_ms": round(d_ttft, 3), "decode_ms": round(d_dec, 3), "tokens_per_s": round(a.gen / d_dec * 1e3, 1)},
       "decode_speedup": round(d_dec / t_dec, 3), "ttft_speedup": round(d_ttft / t_ttft, 3),
       # random weights give near-tied top logits, so greedy tokens diverge under any change of
       # accumulation order; the logits of the first decode step are the parity number
       "first_step_logits_rel_err": round(float((t_logits - d_logits).abs().max() / d_logits.abs().max()), 5),
       "first_step_top2_gap": round(float(top2[0] - top2[1]), 5),
       "greedy_tokens_agree": f"{agree}/{a.gen}"}
print(json.dumps(res), flush=True)
