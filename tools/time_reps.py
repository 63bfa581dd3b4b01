"""c2 sort repeated R times (CUDA events), prints min/median/max and outliers."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bqgen
import paper_1604_06697_b200 as bq
R = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
a = bqgen.config(cfg, seed=1)
if a.dtype.name == "uint64":
    a = a.view("int64")
src = torch.from_numpy(a).cuda()
t = torch.empty_like(src)
ws = bq.workspace(bq.kind_of(src), len(src))
ts = []
for i in range(R):
    t.copy_(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bq.bq_sort_ex(t, ws=ws); e1.record(); torch.cuda.synchronize()
    ts.append(round(e0.elapsed_time(e1), 3))
s = sorted(ts)
print(json.dumps({"cfg": cfg, "lib": os.path.basename(bq.LIB_PATH), "min": s[0], "med": s[len(s)//2], "max": s[-1], "all": ts}))
