import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder
cfg = DecoderConfig(n_layers=4, max_seq=128)
m = TernaryDecoder(cfg)
prompt = torch.randint(0, cfg.vocab, (64,), device="cuda")
m.prefill(prompt)
torch.cuda.synchronize()
for _ in range(2):
    m._decode_body()
torch.cuda.synchronize()
