"""Time bq_sort on every BASELINE.json config at its full size (CUDA events,
device-resident input restored before each run); prints one JSON line per
config.  usage: time_configs.py [--ways W] [--records R] [--configs c1,c5,...]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bqgen
import paper_1604_06697_b200 as bq

ap = argparse.ArgumentParser()
ap.add_argument("--ways", type=int, default=0)
ap.add_argument("--records", type=int, default=0)
ap.add_argument("--configs", default="")
args = ap.parse_args()
ways = args.ways
cases = [("c1", {}), ("c2", {}), ("c3", {"ordering": "random"}), ("c3", {"ordering": "ascending"}),
         ("c3", {"ordering": "descending"}), ("c3", {"ordering": "swapped"}), ("c4a", {}), ("c4b", {}), ("c5", {})]
for name, kw in cases:
    if args.configs and name not in args.configs.split(","):
        continue
    a = bqgen.config(name, seed=1, **kw)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    src = torch.from_numpy(a).cuda()
    dst = torch.empty_like(src)
    ws = bq.workspace(bq.kind_of(src), len(src))
    ts = []
    for i in range(4):
        dst.copy_(src)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bq.bq_sort_ex(dst, ws=ws, ways=ways, records=args.records, stats=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    dst.copy_(src)
    st = bq.bq_sort_ex(dst, ws=ws, ways=ways, records=args.records)
    ms = sorted(ts[1:])[1]
    n = len(src)
    print(json.dumps({"config": name, **kw, "records": args.records, "n": n, "ms": round(ms, 3), "Gkeys_s": round(n / ms / 1e6, 2),
                      "levels": st["levels"], "element_passes": round(st["element_passes"] / n, 2),
                      "all_ms": [round(t, 3) for t in ts], "fallback_segments": st["fallback_segments"],
                      "leaves": st.get("leaves"), "kernel_launches": st.get("kernel_launches")}), flush=True)
    del src, dst, ws
    torch.cuda.empty_cache()
