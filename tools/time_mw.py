"""Time the c2 sort (n = 2^28 int32) with binary and with multiway passes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bqgen
import paper_1604_06697_b200 as bq
n = 1 << 28
src = torch.from_numpy(bqgen.i32_full(n, 1)).cuda()
dst = torch.empty_like(src)
ws = bq.workspace(bq.BQ_I32, n)
ref = torch.sort(src)[0]
for ways in (2, 8, 16):
    ts = []
    for i in range(4):
        dst.copy_(src)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); st = bq.bq_sort_ex(dst, ws=ws, ways=ways); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"ways": ways, "ms": ts[1:], "ok": bool(torch.equal(dst, ref)), "levels": st["levels"],
                      "element_passes": st["element_passes"] / n}), flush=True)
