"""Group a kernel's SASS (ncu source page) by execution count: how many
instructions run per round / per unit / per key.  usage: ncu_execgroups.py REPORT KERNEL_REGEX"""
import collections, csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "-k", "regex:" + sys.argv[2], "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(out.splitlines()) if len(r) > 6 and r[0].startswith("0x")]
seen = set(); uniq = []
for r in rows:   # (the page may list the code twice)
    if r[0] in seen: continue
    seen.add(r[0]); uniq.append(r)
byc = collections.defaultdict(list); tot = 0; samp = 0
for r in uniq:
    c = int(r[5]) if r[5].isdigit() else 0
    tot += c; samp += int(r[2] or 0)
    byc[c].append(r)
print(f"total {tot / 1e6:.1f}M warp instructions, {samp} stall samples")
for c, rs in sorted(byc.items(), key=lambda kv: -kv[0] * len(kv[1]))[:12]:
    ops = collections.Counter((r[1].split()[1] if r[1].split()[0].startswith("@") else r[1].split()[0]).split(".")[0] for r in rs)
    s = sum(int(r[2] or 0) for r in rs)
    print(f"x{c:9d}: {len(rs):4d} instrs {c * len(rs) / tot * 100:5.1f}% of instrs, {s / max(samp, 1) * 100:5.1f}% of samples: "
          + " ".join(f"{k}:{v}" for k, v in ops.most_common(10)))
