"""Summarise gpurun_out/ (scripts/profile_round.sh) into profiles/: launch list, ncu full captures, bench line."""
import csv, collections, json, shutil, subprocess, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hdr = None
d = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    rec = dict(zip(hdr, r))
    d[(rec["Kernel Name"].split("(")[0], rec["Grid Size"], rec["Block Size"])].append(float(rec["Metric Value"].replace(",", "")))
lines = ["kernel,grid,block,launches,mean_us,min_us,max_us"]
for (n, g, b), v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{n},{g},{b},{len(v)},{sum(v)/len(v)/1e3:.3f},{min(v)/1e3:.3f},{max(v)/1e3:.3f}")
open(f"profiles/{tag}_launches_bench.csv", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return dict(zip(r[0], r[2]))


keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
summ = {}
import os

for name, rep, shape in [("gemv", "gpurun_out/prof_gemv.ncu-rep", "rows 11008 x cols 4096, batch 1, fp16"),
                         ("umma", "gpurun_out/prof_umma.ncu-rep", "rows 11008 x cols 4096, batch 128, fp16"),
                         ("umma_b16", "gpurun_out/prof_u16.ncu-rep", "rows 11008 x cols 4096, batch 16, fp16"),
                         ("gemv_tq1", "gpurun_out/prof_q1.ncu-rep", "TQ1 rows 8192 x cols 8192, batch 1, fp16"),
                         ("chain", "gpurun_out/prof_chain.ncu-rep",
                          "K6 chain, 8 replicas of (4096x4096, 11008x4096, 4096x11008), batch 1, fp16")]:
    if not os.path.exists(rep):
        continue
    m = raw(rep)
    e = {"kernel": (m.get("Kernel Name") or m.get("Function Name") or "").split("(")[0]}
    e.update({k: m.get(k) for k in keys})
    e["shape"] = shape
    e["units"] = "time us, dram bytes MB, smem KB (ncu --set full, one launch, cold, --clock-control none)"
    summ[name] = e
json.dump(summ, open(f"profiles/{tag}_ncu_full_summary.json", "w"), indent=1)
print(json.dumps(summ, indent=1))
shutil.copy("gpurun_out/bench.json", f"profiles/{tag}_bench.json")
