"""Dev: summarize an ncu report: key metrics, stall reasons, top stalled SASS lines by region."""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_read.sum.per_second', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'smsp__warps_active.avg.per_cycle_active', 'launch__grid_size', 'launch__block_size']
for i, n in enumerate(h):
    if n in keys:
        print(f"{n:70s} {u[i]:10s} {v[i]}")
st = sorted([(float(v[i] or 0), n) for i, n in enumerate(h) if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued')], reverse=True)
print("stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_','')}={int(x)}" for x, n in st[:12]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(src.splitlines()))
h = r[1]; rows = r[2:]
ia = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
sc = [i for i, n in enumerate(h) if n.startswith('stall_') and 'Not Issued' not in n]
tot = sum(float(x[ia] or 0) for x in rows)
print("total samples", tot)
top = sorted(rows, key=lambda x: -float(x[ia] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for x in top:
    s = float(x[ia] or 0)
    stl = sorted([(float(x[i] or 0), h[i]) for i in sc], reverse=True)[:2]
    print(f"{int(x[0],16)&0xffff:6x} {s:5.0f} {x[ie]:>7s} {x[1][:70]:70s}", [(n[6:], int(q)) for q, n in stl if q > 0])
