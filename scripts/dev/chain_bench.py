"""K6 persistent chain vs the PDL chain on the BASELINE stack (bench.py's workload): timing over
ring depths / refill hold windows, and a %globaltimer breakdown per op (median over CTAs, us)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2506_23025_b200.graph import LinearStack

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 32
b = int(sys.argv[2]) if len(sys.argv) > 2 else 1
variants = [tuple(int(v) for v in s.split(":")) for s in (sys.argv[3] if len(sys.argv) > 3 else "0:0:0").split(",")]
variants = [v + (0,) * (3 - len(v)) for v in variants]
torch.cuda.set_device(0)
ws = bench.make_stack_weights(reps, seed=1234)
out = {}
st = LinearStack(ws, batch=b, chain=False)
st.x.copy_(bench.uniform_x(b, 4096, 4243))
ms = bench.timed_graph(st.replay, 30, 5, None) / 30
out["pdl"] = {"us_per_layer": round(ms * 1e3 / len(ws), 3), "gbs": round(st.algorithmic_bytes() / ms / 1e6, 1)}
nbytes = st.algorithmic_bytes()
del st
st = LinearStack(ws, batch=b, chain=True)
st.x.copy_(bench.uniform_x(b, 4096, 4243))
ch = st._chain
for ns, hold, probe in variants:
    run = lambda: ch.run(ns=ns, hold=hold, probe=probe)
    try:
        ms = bench.timed_graph(run, 20, 3, None) / 20
    except Exception as e:
        out[f"chain_ns{ns}_probe{probe}"] = {"error": str(e)[:200]}
        continue
    key = f"chain_ns{ns}_hold{hold}_probe{probe}"
    out[key] = {"us_per_layer": round(ms * 1e3 / len(ws), 3), "gbs": round(nbytes / ms / 1e6, 1)}
    ch.run(probe=2 | probe, ns=ns, hold=hold)
    torch.cuda.synchronize()
    tr = ch.trace().cpu().double() / 1e3
    n = tr.shape[0]
    med = lambda t: round(t.median().item(), 3)
    rows = {}
    for kind, idx in (("4096x4096", range(3, n, 3)), ("11008x4096", range(4, n, 3)), ("4096x11008", range(5, n, 3))):
        idx = list(idx)
        prev_stored = torch.stack([tr[l - 1, :, 3].max() for l in idx])
        rows[kind] = {
            "wait_after_prev_done": med(torch.stack([tr[l, :, 1].median() for l in idx]) - prev_stored),
            "staging": med(torch.stack([(tr[l, :, 2] - tr[l, :, 1]).median() for l in idx])),
            "x_load_w0": med(torch.stack([(tr[l, :, 6] - tr[l, :, 1]).median() for l in idx])),
            "first_slot_wait_w0": med(torch.stack([(tr[l, :, 5] - tr[l, :, 2]).median() for l in idx])),
            "w0_issue_lead": med(torch.stack([(tr[l, :, 2] - tr[l, :, 7]).median() for l in idx])),
            "w0_issue_to_land": med(torch.stack([(tr[l, :, 5] - tr[l, :, 7]).median() for l in idx])),
            "mainloop_w0": med(torch.stack([(tr[l, :, 4] - tr[l, :, 2]).median() for l in idx])),
            "tail_store": med(torch.stack([(tr[l, :, 3] - tr[l, :, 4]).median() for l in idx])),
            "t_join": med(torch.stack([(tr[l, :, 8] - tr[l, :, 4]).median() for l in idx])),
            "t_reduce": med(torch.stack([(tr[l, :, 9] - tr[l, :, 8]).median() for l in idx])),
            "t_sync2": med(torch.stack([(tr[l, :, 10] - tr[l, :, 9]).median() for l in idx])),
            "t_release": med(torch.stack([(tr[l, :, 3] - tr[l, :, 10]).median() for l in idx])),
            "op_span": med(torch.stack([tr[l, :, 3].max() - prev for l, prev in zip(idx, prev_stored)])),
        }
    out[key]["trace"] = rows
print(json.dumps(out, indent=1))
