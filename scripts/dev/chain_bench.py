"""K6 persistent chain vs the PDL chain on the BASELINE stack (bench.py's workload), plus a
%globaltimer trace of the chain: per op, wait / staging / compute+store spans (us)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2506_23025_b200.graph import LinearStack

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 32
batches = [int(b) for b in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1"])]
torch.cuda.set_device(0)
ws = bench.make_stack_weights(reps, seed=1234)
out = {}
for b in batches:
    for chain in (False, True):
        st = LinearStack(ws, batch=b, chain=chain)
        st.x.copy_(bench.uniform_x(b, 4096, 4243))
        ms = bench.timed_graph(st.replay, 30, 5, None) / 30
        out[f"b{b}_{'chain' if chain else 'pdl'}"] = {"ms": round(ms, 4), "us_per_layer": round(ms * 1e3 / len(ws), 3),
                                                      "gbs": round(st.algorithmic_bytes() / ms / 1e6, 1)}
        if chain and b == batches[0]:
            ch = st._chain
            ch.run(probe=2)
            torch.cuda.synchronize()
            tr = ch.trace().cpu().double()
            t0 = tr[0, :, 0].min()
            tr = (tr - t0) / 1e3
            n = tr.shape[0]
            rows = []
            for l in range(min(n, 9)):
                rows.append({"op": l, "start_max": round(tr[l, :, 0].max().item(), 2),
                             "ready_min": round(tr[l, :, 1].min().item(), 2), "ready_max": round(tr[l, :, 1].max().item(), 2),
                             "staged_avg": round((tr[l, :, 2] - tr[l, :, 1]).mean().item(), 3),
                             "compute_avg": round((tr[l, :, 3] - tr[l, :, 2]).mean().item(), 3),
                             "compute_max": round((tr[l, :, 3] - tr[l, :, 2]).max().item(), 3),
                             "stored_max": round(tr[l, :, 3].max().item(), 2)})
            out["trace_first_ops"] = rows
            out["trace_total_us"] = round(tr[n - 1, :, 3].max().item(), 2)
            per = [(tr[l, :, 3].max() - tr[l - 1, :, 3].max()).item() for l in range(1, n)]
            out["trace_us_per_op_avg"] = round(sum(per) / len(per), 3)
            out["trace_wait_avg"] = round(sum((tr[l, :, 1].min() - tr[l - 1, :, 3].max()).item() for l in range(1, n)) / (n - 1), 3)
        del st
        torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
