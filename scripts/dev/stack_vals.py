import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2506_23025_b200.graph import LinearStack
ws = bench.make_stack_weights(32, seed=1234)
for dt in (torch.float16, torch.bfloat16):
    for b in (1, 16):
        st = LinearStack(ws, batch=b, dtype=dt)
        st.x.copy_(bench.uniform_x(b, st.x.shape[1], 4242 + b, dt))
        st.replay(); torch.cuda.synchronize()
        am = [float(o.float().abs().max()) for o in st.bufs]
        fin = [bool(torch.isfinite(o).all()) for o in st.bufs]
        print(dt, b, "absmax layers 0,1,2,5,10,30,60,95:", [f"{am[i]:.3g}" for i in (0,1,2,5,10,30,60,95)], "first nonfinite:", fin.index(False) if False in fin else None)
