"""Time the out-of-place partition pass and one full sort at n = 2^28 int32."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import bqgen
import paper_1604_06697_b200 as bq
n = 1 << 28
ORD = bool(int(os.environ.get('BQ_ORDERED', '0')))
a = bqgen.i32_full(n, 1)
src = torch.from_numpy(a).cuda(); dst = torch.empty_like(src)
ws = bq.workspace(bq.BQ_I32, n); c = torch.zeros(3, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
pv = bq.bq_pivot_i32(src, 0, ws=ws)
ts = []
for i in range(8):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bq.bq_partition_pass(src, dst, pv, c, ordered=ORD, ws=ws); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts[2:])
st = []
for i in range(3):
    dst.copy_(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s = bq.bq_sort_ex(dst, ws=ws, timing=True, ordered=ORD); e1.record(); torch.cuda.synchronize()
    st.append((e0.elapsed_time(e1), s["partition_ms"], s["partition_bytes"]))
ok = bool(torch.equal(dst, torch.sort(src)[0]))
sm, pm, pb = st[-1]
print(json.dumps({"pass_ms": ms, "pass_gbs": 8 * n / ms / 1e6, "sort_ms": sm, "part_ms": pm,
                  "part_gbs": pb / pm / 1e6, "sort_ok": ok}))
