"""Summarise an ncu report (run here, no GPU): key metrics + top stall PCs."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25

def run(*a):
    return subprocess.run(["ncu", "-i", rep] + list(a), capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, u = raw[0], raw[1]
# several launches in the report: summarise the longest one
it = h.index("gpu__time_duration.sum")
pick = max(range(2, len(raw)), key=lambda i: float(raw[i][it].replace(",", "") or 0))
v = raw[pick]
if len(raw) > 3:
    print(f"(longest of {len(raw) - 2} captured launches: #{pick - 2})")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "lts__t_bytes.sum",
        "smsp__sass_branch_targets_threads_divergent.sum", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in want:
    if k in h:
        i = h.index(k)
        print(f"{k:60s} {v[i]:>16s} {u[i]}")
stalls = [(k, v[i]) for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x or 0)) for k, x in stalls), key=lambda t: -t[1])
tot = sum(x for _, x in stalls) or 1
print("stall samples:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in stalls[:8]))
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
# the source page lists every captured launch (and each non-inlined device
# function) as its own section: keep the sections of the chosen launch
heads = [i for i, r in enumerate(src) if "Source" in r and "Instructions Executed" in r]
nlaunch = max(1, len(raw) - 2)
per = max(1, len(heads) // nlaunch)
mine = heads[(pick - 2) * per:(pick - 1) * per] or heads[:1]
hh = src[mine[0]]
data = []
for hi in mine:
    end = next((j for j in heads if j > hi), len(src))
    data += [r for r in src[hi + 1:end] if len(r) == len(hh) and "Source" not in r]
iS, iE, iW = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
print("top stall PCs:" + ("" if nlaunch == 1 else " (source page of an imported multi-launch report: the CLI gives the first launch's)"))
for r in sorted(data, key=lambda r: -float(r[iW] or 0))[:top]:
    print(f"  {float(r[iE] or 0):12.0f} {float(r[iW] or 0):8.0f}  {r[iS][:100]}")
