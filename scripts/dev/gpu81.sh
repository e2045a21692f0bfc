#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "decoder" 2>&1 | tail -1
timeout 600 python scripts/decode_bench.py 2>&1 | tail -1
git_multi=1 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2506_23025_b200.decoder import DecoderConfig, TernaryDecoder
cfg = DecoderConfig(max_seq=128)
m = TernaryDecoder(cfg)
p = torch.randint(0, cfg.vocab, (64,), device='cuda')
for spg in (1, 8):
    m.STEPS_PER_GRAPH = spg; m.graph = None
    m.reset(); m.prefill(p); m.capture()
    ts = []
    for _ in range(3):
        m.reset(); m.prefill(p); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); m.decode(64); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) / 64)
    print('steps_per_graph', spg, 'ms/token', round(min(ts), 4), m.out_tokens[64:72].tolist())
"
