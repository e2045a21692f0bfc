"""One K6 chain launch over the BASELINE stack (R replicas) for an ncu capture."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2506_23025_b200.graph import LinearStack

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
torch.cuda.set_device(0)
ws = bench.make_stack_weights(reps, seed=1234)
st = LinearStack(ws, batch=1, chain=True)
st.x.copy_(bench.uniform_x(1, 4096, 4243))
for _ in range(4):
    st._chain.run()
torch.cuda.synchronize()
