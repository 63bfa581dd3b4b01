"""Breakdown of the c5 records sort and the records partition pass."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as bq
n = 1 << 26
src = torch.from_numpy(bqgen.rec32(n, 1).view(np.int64)).cuda()
dst = torch.empty_like(src)
ws = bq.workspace(bq.BQ_REC32, n)
for i in range(3):
    dst.copy_(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); st = bq.bq_sort_ex(dst, ws=ws, timing=True); e1.record(); torch.cuda.synchronize()
print(json.dumps({"sort_ms": e0.elapsed_time(e1), "part_ms": st["partition_ms"], "part_GBps": st["partition_bytes"] / st["partition_ms"] / 1e6, "levels": st["levels"]}))
counts = torch.zeros(3, dtype=torch.int64, device="cuda")
pv = bq.pivot(src, bq.BQ_PIVOT_MO3, ws=ws)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(6):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bq.bq_partition_pass(src, dst, pv, counts, ordered=True, ws=ws); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts[1:])
print(json.dumps({"rec_pass_ms": ms, "rec_pass_GBps": 64 * n / ms / 1e6}))
