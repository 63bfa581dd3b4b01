"""Stall reasons per CUDA source line of one kernel (ncu source page, cuda,sass
view; line rows carry the line totals).  usage: ncu_linestalls.py REPORT KERNEL_REGEX [top]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]; top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = [r for r in rows if len(r) > 8 and r[0] == "Line No"][0]
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
fname = None; res = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0].isdigit():
        num = lambda x: int(x) if x.isdigit() else 0
        tot = num(r[4])
        if tot:
            st = sorted(((num(r[i]), h[i][6:]) for i in cols), reverse=True)[:3]
            res.append((tot, f"{fname}:{r[0]}", r[1].strip()[:60], st))
for tot, loc, src, st in sorted(res, reverse=True)[:top]:
    print(f"{tot:6d} {loc:24s} {' '.join(f'{n}={v}' for v, n in st):50s} {src}")
