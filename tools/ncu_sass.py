"""Per-instruction SASS listing of an ncu report with executed counts and stall samples
(source page).  usage: ncu_sass.py REPORT [min_count]"""
import csv, subprocess, sys
rep = sys.argv[1]; mn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if "Source" in r][0]
h = rows[hi]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= iE: continue
    e = int(r[iE] or 0); tot += e
    if e >= mn: print(str(e).rjust(10), str(r[iW]).rjust(6), r[iS].strip()[:100])
print("total", tot)
