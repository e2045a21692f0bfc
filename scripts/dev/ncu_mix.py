"""Dev: instruction mix of an ncu report grouped by execution count (loop level)."""
import csv, subprocess, sys
from collections import Counter, defaultdict
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(src.splitlines()))
h = r[1]; rows = r[2:]
ie = h.index("Instructions Executed"); ia = h.index("Warp Stall Sampling (All Samples)")
by = defaultdict(Counter); samp = Counter(); tot = 0
for x in rows:
    n = int(float(x[ie] or 0))
    if n == 0: continue
    t = x[1].split()
    op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    by[n][op] += 1; samp[n] += float(x[ia] or 0); tot += n
print("total warp-instructions", tot)
for n in sorted(by, key=lambda n: -n * sum(by[n].values()))[:8]:
    c = by[n]
    print(f"count {n:8d}: {sum(c.values()):4d} instrs/iter, {n*sum(c.values())/tot*100:5.1f}% of instrs, samples {samp[n]:.0f}:",
          ", ".join(f"{k}={v}" for k, v in c.most_common(14)))
