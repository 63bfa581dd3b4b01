"""GPU debug: out-of-place pass and sort vs plain definitions at growing n."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as bq

def three(a, p):
    return np.concatenate([a[a < p], a[a == p], a[a > p][::-1]])

for lg in [12, 14, 16, 18, 20, 22, 24, 26]:
    n = (1 << lg) + 7
    a = bqgen.i32_full(n, lg)
    src = torch.from_numpy(a).cuda(); dst = torch.empty_like(src)
    c = torch.zeros(3, dtype=torch.int64, device="cuda")
    p = int(a[n // 2])
    bq.bq_partition_pass(src, dst, p, c); torch.cuda.synchronize()
    got = dst.cpu().numpy(); exp = three(a, np.int32(p))
    bad = np.nonzero(got != exp)[0]
    print("pass", lg, c.tolist(), (int((a<p).sum()), int((a==p).sum())), "mismatches", len(bad), bad[:5], flush=True)
    t = src.clone(); st = bq.bq_sort_ex(t)
    got = t.cpu().numpy(); exp = np.sort(a)
    bad = np.nonzero(got != exp)[0]
    print("sort", lg, "levels", st["levels"], "mismatches", len(bad), bad[:5], flush=True)
