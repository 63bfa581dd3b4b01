"""Map ncu SASS-page stall samples to CUDA source lines (run here, no GPU).
usage: sass_lines.py report.ncu-rep kernel_substring cubin [top]"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, ksub, cubin = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# split per function
funcs = re.split(r"\n\s*\.text\.", dis)
body = None
for f in funcs:
    name = f.split(":", 1)[0]
    if ksub in name:
        body = f
        break
assert body, "kernel not found"
line_of = {}
cur = None
for ln in body.splitlines():
    m = re.search(r'line (\d+)', ln)
    if "## File" in ln and m:
        fm = re.search(r'File "([^"]+)"', ln)
        cur = (fm.group(1).split("/")[-1] if fm else "?") + ":" + m.group(1)
    m2 = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m2 and cur:
        line_of[int(m2.group(1), 16)] = cur
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                                capture_output=True, text=True).stdout)))
h = src[1]; data = src[2:]
iA, iE, iW = 0, h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = min(int(r[iA], 16) for r in data)
agg = defaultdict(lambda: [0.0, 0.0])
for r in data:
    off = int(r[iA], 16) - base
    key = line_of.get(off, "?")
    agg[key][0] += float(r[iE] or 0)
    agg[key][1] += float(r[iW] or 0)
tot = sum(v[1] for v in agg.values()) or 1
toti = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot:.0f} total warp-inst {toti:.0f}")
for k, (e, w) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"  {k:32s} inst {e:12.0f} ({100*e/toti:4.1f}%)  stall {w:8.0f} ({100*w/tot:4.1f}%)")
