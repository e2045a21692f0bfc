"""Dev: the bench's BASELINE stack (32 replicas of the three configs[1] shapes) ms per replay at the
given batches, ternary only (A/B via TRITRUN_LIB); argv[2] = bf16 for bfloat16 activations."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2506_23025_b200.graph import LinearStack

torch.cuda.set_device(0)
ws = bench.make_stack_weights(32, seed=1234)
dt = torch.bfloat16 if len(sys.argv) > 2 and sys.argv[2] == "bf16" else torch.float16
out = {}
for b in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4,8,16,32").split(",")]:
    st = LinearStack(ws, batch=b, dtype=dt)
    st.x.copy_(bench.uniform_x(b, st.x.shape[1], 4242 + b, dt))
    out[b] = round(min(bench.timed_graph(st.replay, 20, 3, None) / 20 for _ in range(3)), 4)
    del st
print(os.environ.get("TRITRUN_LIB", "default"), json.dumps(out))
