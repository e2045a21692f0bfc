"""Dev: greedy tokens of the 3.9B-shaped decoder with / without the SwiGLU epilogue vs the dense twin."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder

cfg = DecoderConfig(max_seq=128)
prompt = torch.randint(0, cfg.vocab, (64,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
m = TernaryDecoder(cfg)
def run(model):
    model.reset(); model.graph = None; model.prefill(prompt)
    first = model.forward(model.tok, model.pos).float()
    top = first.topk(2).values
    model.reset(); model.prefill(prompt); model.decode(64)
    return model.out_tokens[64:128].clone(), first, float(top[0] - top[1])
t_epi, l_epi, gap = run(m)
il = m.gate_up_il; m.gate_up_il = None
t_no, l_no, _ = run(m)
dense = TernaryDecoder(cfg, dense=True, weights=m.weights)
t_d, l_d, gap_d = run(dense)
rel = lambda a, b: float((a - b).abs().max() / b.abs().max())
print(json.dumps({"epi_vs_dense": int((t_epi == t_d).sum()), "noepi_vs_dense": int((t_no == t_d).sum()),
                  "epi_vs_noepi": int((t_epi == t_no).sum()), "gap_top2": gap, "gap_dense": gap_d,
                  "logit_rel_epi_dense": rel(l_epi, l_d), "logit_rel_noepi_dense": rel(l_no, l_d),
                  "argmax": [int(l_epi.argmax()), int(l_no.argmax()), int(l_d.argmax())]}))
