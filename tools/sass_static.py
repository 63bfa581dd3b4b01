"""Static SASS opcode histogram of one kernel of a cubin, split by the
source file:line each instruction maps to (nvdisasm -g); a line filter
restricts it to a region (e.g. a loop body).
usage: sass_static.py CUBIN KERNEL_SUBSTR [FILE:LO-HI ...]"""
import collections, re, subprocess, sys
cub, ksub = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    f, r = a.split(":"); lo, hi = r.split("-"); ranges.append((f, int(lo), int(hi)))
out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
cur_fn = None; loc = None; agg = collections.Counter(); n = 0
for line in out.splitlines():
    m = re.match(r'\s*\.text\.(\S+):', line) or re.match(r'^(_Z\S+):', line)
    if m: cur_fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m: loc = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if cur_fn is None or ksub not in cur_fn: continue
    m = re.match(r'\s*/\*[0-9a-f]{4,}\*/\s+(.*?);', line)
    if not m: continue
    ins = m.group(1).strip()
    if ranges and not (loc and any(loc[0] == f and lo <= loc[1] <= hi for f, lo, hi in ranges)): continue
    toks = ins.split(); op = toks[1] if toks[0].startswith("@") else toks[0]
    agg[op] += 1; n += 1
for op, c in agg.most_common(): print(f"{op:24s} {c}")
print("total", n)
