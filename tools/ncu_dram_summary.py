"""Summarise an ncu launch list with gpu__time_duration.sum and
dram__bytes_{read,write}.sum (one c2 sort, host-driven loop): per kernel the
launches, summed device time and DRAM bytes per launch; writes the JSON that
bench.py reads for roofline.traffic.  usage: ncu_dram_summary.py CSV OUT.json"""
import collections, csv, json, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iid, im, iv = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    key = (r[iid], r[ik])
    per.setdefault(key, {})[r[im]] = float(r[iv].replace(",", ""))
agg = collections.OrderedDict()
for (lid, name), m in per.items():
    k = name.split("(")[0].replace("void ", "").split("<")[0].replace("bq::", "")
    a = agg.setdefault(k, {"launches": 0, "active_launches": 0, "ms": 0.0, "dram_read": 0.0, "dram_write": 0.0})
    a["launches"] += 1
    a["active_launches"] += m.get("gpu__time_duration.sum", 0.0) > 20000   # > 20 us: not a no-op level
    a["ms"] += m.get("gpu__time_duration.sum", 0.0) / 1e6
    a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
    a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
out = {}
for k, a in agg.items():
    out[k] = dict(a, dram_bytes_total=a["dram_read"] + a["dram_write"],
                  note="DRAM bytes of all launches of one sort (the level loop's trailing no-op levels move none)")
json.dump(out, open(sys.argv[2], "w"), indent=1)
tot = sum(a["ms"] for a in agg.values())
print("| kernel | launches | ms (sum) | share | DRAM GB read | DRAM GB write |\n|---|---:|---:|---:|---:|---:|")
for k, a in sorted(agg.items(), key=lambda t: -t[1]["ms"]):
    print(f"| {k} | {a['launches']} | {a['ms']:.3f} | {100 * a['ms'] / tot:.1f}% | {a['dram_read'] / 1e9:.3f} | {a['dram_write'] / 1e9:.3f} |")
