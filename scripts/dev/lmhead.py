"""Dev: time the decoder's fp16 lm_head GEMV (cuBLAS) and the decode tail, CUDA-graphed."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import torch.nn.functional as F
W = [torch.randn(32000, 3072, device="cuda").half() * 0.02 for _ in range(4)]
x = torch.randn(1, 3072, device="cuda").half()
def timeit(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): g.replay()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n
us = timeit(lambda: [F.linear(x, w) for w in W]) / 4
print(json.dumps({"lm_head_us": round(us, 2), "gbs": round(32000 * 3072 * 2 / us / 1e3, 1)}))
