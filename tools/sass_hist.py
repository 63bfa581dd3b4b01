"""Opcode histogram (executed warp instructions per key) of one kernel of an
ncu report.  usage: sass_hist.py REPORT KERNEL_REGEX NKEYS [min_count]"""
import collections, csv, re, subprocess, sys
rep, kre, nkeys = sys.argv[1], sys.argv[2], float(sys.argv[3])
mn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if "Source" in r][0]
h = rows[hi]
iS, iE = h.index("Source"), h.index("Instructions Executed")
agg = collections.Counter(); tot = 0
for r in rows[hi + 1:]:
    if len(r) <= iE or not r[iE].isdigit(): continue
    c = int(r[iE]); tot += c
    if c < mn: continue
    toks = r[iS].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    agg[op] += c
for op, c in agg.most_common(40):
    print(f"{op:24s} {c / 1e6:8.2f}M {c * 32 / nkeys:6.2f}/key")
print(f"total {tot / 1e6:.1f}M warp instructions = {tot * 32 / nkeys:.1f} per key")
