"""Copy the round's evidence from gpurun_out/ (tools/gpu_prof_final.sh) into
profiles/r02/ and write the launch-list and ncu summaries (run here, no GPU)."""
import collections, csv, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", "r02")
run = lambda *a: subprocess.run([sys.executable] + list(a), capture_output=True, text=True, cwd=ROOT).stdout


def launches(path, second_half):
    """per-launch dicts (name, ms, read GB, write GB) of an ncu launch list"""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, im, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
    d, order = {}, []
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        if r[iid] not in d:
            d[r[iid]] = {"name": r[ik].split("(")[0].replace("void ", "").replace("bq::", "").split("<")[0]}
            order.append(r[iid])
        d[r[iid]][r[im]] = float(r[iv].replace(",", ""))
    if second_half:
        order = order[len(order) // 2:]
    return [dict(name=d[k]["name"], ms=d[k].get("gpu__time_duration.sum", 0) / 1e6,
                 rd=d[k].get("dram__bytes_read.sum", 0) / 1e9, wr=d[k].get("dram__bytes_write.sum", 0) / 1e9)
            for k in order]


def table(ls):
    agg = collections.OrderedDict()
    for l in ls:
        a = agg.setdefault(l["name"], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += l["ms"]
        a[2] += l["rd"]
        a[3] += l["wr"]
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | ms (sum) | share | DRAM GB read | DRAM GB write |", "|---|---:|---:|---:|---:|---:|"]
    for k, a in sorted(agg.items(), key=lambda t: -t[1][1]):
        out.append(f"| {k} | {a[0]} | {a[1]:.3f} | {100 * a[1] / tot:.1f}% | {a[2]:.3f} | {a[3]:.3f} |")
    out.append(f"| total | {sum(a[0] for a in agg.values())} | {tot:.3f} | | | |")
    return "\n".join(out)


shutil.copy(os.path.join(G, "bench_final.json"), os.path.join(P, "bench_current.json"))
shutil.copy(os.path.join(G, "cfg_final.jsonl"), os.path.join(P, "configs_timing.jsonl"))
shutil.copy(os.path.join(G, "launches_c2_final.csv"), os.path.join(P, "launches_c2_sort_dram.csv"))
run("tools/ncu_dram_summary.py", os.path.join(P, "launches_c2_sort_dram.csv"), os.path.join(P, "ncu_sort_dram.json"))
open(os.path.join(P, "launches_c2_sort_dram.md"), "w").write(
    "# One c2 sort (2^28 int32), ncu launch list with DRAM bytes\n\n"
    "Host-driven level loop (the graph's kernels), `tools/gpu_prof_final.sh`; cold and serialised.\n\n"
    + table(launches(os.path.join(P, "launches_c2_sort_dram.csv"), False)) + "\n")
for c, what in (("c3", "2^27 float64"), ("c5", "2^26 32-byte records (key+index pairs)")):
    shutil.copy(os.path.join(G, f"launches_{c}_final.csv"), os.path.join(P, f"launches_{c}_sort_dram.csv"))
    ls = launches(os.path.join(P, f"launches_{c}_sort_dram.csv"), True)
    big = "\n".join(f"| {l['name']} | {1e3 * l['ms']:.1f} | {l['rd']:.3f} | {l['wr']:.3f} | "
                    f"{1e3 * (l['rd'] + l['wr']) / l['ms'] if l['ms'] else 0:.0f} |" for l in ls if l["ms"] > 0.015)
    open(os.path.join(P, f"launches_{c}_sort_dram.md"), "w").write(
        f"# One {c} sort ({what}), ncu launch list with DRAM bytes\n\n"
        "Host-driven level loop, second of two sorts (`tools/one_sort.py`); cold and serialised.\n\n"
        + table(ls) + "\n\nLaunches over 15 us:\n\n| kernel | us | DRAM GB read | DRAM GB write | GB/s |\n"
        "|---|---:|---:|---:|---:|\n" + big + "\n")
parts = []
for rep, title, k in (("final_mw8i", "k_mw8w_count / k_mw8t_scatter<KI32> (level 0 of the c2 sort)", None),
                      ("final_leaf", "k_leaf<KI32, 512> (c2, the largest leaf launch)", None),
                      ("final_mw8w", "k_mw8w_count / k_mw8t_scatter<KF64> (level 0 of the c3 sort)", None)):
    path = os.path.join(G, rep + ".ncu-rep")
    parts.append(f"## {title}\n\n```\n{run('tools/ncu_brief.py', path)}```\n")
    parts.append(f"Instructions by source line (top 20):\n\n```\n{run('tools/ncu_lines.py', path, '20')}```\n")
open(os.path.join(P, "ncu_full_r02.md"), "w").write(
    "# ncu --set full captures (r02, final kernels)\n\n`tools/gpu_prof_final.sh`; "
    "`tools/ncu_brief.py` and `tools/ncu_lines.py` over the reports.\n\n" + "\n".join(parts))
print("ok")
