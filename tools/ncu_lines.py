"""Per-CUDA-source-line instruction counts and stall samples of an ncu report
(source page, cuda,sass view).  usage: ncu_lines.py REPORT [top]"""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
KF = (["-k", "regex:" + __import__("os").environ["NCU_K"]] if __import__("os").environ.get("NCU_K") else [])
out = subprocess.run(["ncu", "-i", rep] + KF + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []; fname = None; tot = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        e = int(r[7] or 0); w = int(r[4] or 0); tot += e
        res.append((e, w, f"{fname}:{r[0]}", r[1].strip()[:90]))
res.sort(key=lambda x: -x[0])
print("total", tot)
for e, w, loc, src in res[:top]:
    print(f"{e:>11} {100*e/tot:5.1f}% {w:>6} {loc:<28} {src}")
