"""Per-launch lines (second half of the list: the measured sort) of an ncu
launch list with time and DRAM bytes.  usage: launch_detail.py CSV [min_us]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iv, im, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
d, order = {}, []
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    k = r[iid]
    if k not in d:
        d[k] = {"name": r[ik].split("(")[0].replace("void ", "").replace("bq::", "")[:48]}
        order.append(k)
    d[k][r[im]] = float(r[iv].replace(",", ""))
for k in order[len(order) // 2:]:
    x = d[k]
    t = x["gpu__time_duration.sum"] / 1e3
    if t >= mn:
        rb, wb = x.get("dram__bytes_read.sum", 0) / 1e9, x.get("dram__bytes_write.sum", 0) / 1e9
        print(f"{x['name']:48s} {t:8.1f} us  R {rb:6.3f} W {wb:6.3f} GB  {(rb + wb) / t * 1e6:6.0f} GB/s")
