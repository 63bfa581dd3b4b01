"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, summed device time and share.  Run here (no GPU)."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "").split("<")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[iv].replace(",", "")) / 1e6   # ns -> ms
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    tot = sum(v for _, v in agg.values())
    print(f"| kernel | launches | ms (sum) | share |\n|---|---:|---:|---:|")
    for k, (c, v) in sorted(agg.items(), key=lambda t: -t[1][1]):
        print(f"| {k} | {c} | {v:.3f} | {100 * v / tot:.1f}% |")
    print(f"| total | {sum(c for c, _ in agg.values())} | {tot:.3f} | |")
