"""Copy the latest bench / launch list / ncu summaries from gpurun_out/ into
profiles/r01/ and regenerate profiles/r01/current.md (run here, no GPU)."""
import json, os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", "r01")
for src, dst in [("bench.json", "bench_current.json"), ("bench_ref.json", "bench_reference.json"),
                 ("launches_sort.csv", "current_launches_sort.csv"), ("cfg_now.jsonl", "configs_timing.jsonl")]:
    shutil.copy(os.path.join(G, src), os.path.join(P, dst))
run = lambda *a: subprocess.run([sys.executable] + list(a), capture_output=True, text=True, cwd=ROOT).stdout
launch = run("tools/launch_summary.py", os.path.join(P, "current_launches_sort.csv"))
part = run("tools/ncu_summary.py", os.path.join(G, "prof_part.ncu-rep"), "10")
leaf = run("tools/ncu_summary.py", os.path.join(G, "prof_leaf.ncu-rep"), "6")
b = json.load(open(os.path.join(P, "bench_current.json")))
r = json.load(open(os.path.join(P, "bench_reference.json")))
rf, pp = b["roofline"], b["partition_pass"]
cfg = [json.loads(l) for l in open(os.path.join(P, "configs_timing.jsonl")) if l.strip()]
rows = "\n".join(f"| {c['config']}{' ' + c['ordering'] if 'ordering' in c else ''} | {c['n']} | {c['ms']} | {c['Gkeys_s']} | {c['levels']} | {c['element_passes']} |" for c in cfg)
md = f"""# r01 (current): c2 sort, n = 2^28 int32, SAMPLE64 pivots

Bench line (`bench_current.json`): {b['value']:.2f} Gkeys/s, {b['ms_per_step']:.2f} ms per step,
{b['passes_per_element']:.2f} element-passes; partition kernel in the sort
{rf['achieved']:.0f} GB/s = {rf['frac']:.3f} of the measured {rf['peak']} GB/s copy bandwidth
({rf['launch_ms_avg']:.3f} ms per launch, {rf['launches_per_step']} launches, {100 * rf['share_of_step']:.0f} % of the step);
one isolated pass {pp['gbs_median']:.0f} GB/s ({pp['frac_median']:.3f}); bq_partition_i32 (in place, N2)
{pp['inplace_ms_median']:.3f} ms; e2e (host buffers, PCIe) {b['e2e']['value']:.2f} Gkeys/s; clocks
{b['clocks']['sm_mhz']:.0f} MHz, throttle reasons {b['clocks']['reasons']}.  Reference arm (the oracle on
{r['cpu_baseline']['cores']} host core): {r['value']:.4f} Gkeys/s (`bench_reference.json`).

All BASELINE configs at full size (`tools/time_configs.py`, CUDA events, median; `configs_timing.jsonl`):

| config | n | ms | Gkeys/s | levels | element-passes |
|---|---:|---:|---:|---:|---:|
{rows}

Launch list of one c2 sort + 2 single passes (`tools/gpu_cmd_prof.sh`, ncu
`gpu__time_duration.sum`, cold and serialised; `current_launches_sort.csv`):

{launch}
## k_part_fast, one 2^28 pass (ncu --set full)

```
{part}```

## k_leaf<KI32, 13> (ncu --set full; the longest captured launch)

```
{leaf}```
"""
open(os.path.join(P, "current.md"), "w").write(md)
print("ok")
