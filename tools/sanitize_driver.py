"""Small-n workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kind through the sort (graph or host-driven loop, binary / 8-way /
16-way / ordered, the depth-cap fallback), the out-of-place pass (fast and
ordered), the in-place partition, the batched pass and the pivots; results
checked against torch / numpy.  usage: sanitize_driver.py [--small]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bqgen
import paper_1604_06697_b200 as bq

small = "--small" in sys.argv
N = 70_001 if small else 200_003
fails = []


def check(name, ok):
    print(name, "ok" if ok else "MISMATCH", flush=True)
    if not ok:
        fails.append(name)


def dev(a):
    if a.dtype == np.uint64 and a.ndim == 1:
        return torch.from_numpy(a).cuda()
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def keys_sorted(t, a):
    got = t.cpu().numpy()
    if a.ndim == 2:
        return np.array_equal(got[:, 0].view(np.uint64), np.sort(a[:, 0]))
    if a.dtype == np.float64:
        b = np.sort(a)
        return np.array_equal(got.view(np.uint64), b.view(np.uint64)) or np.array_equal(got, b)
    return np.array_equal(got, np.sort(a))


inputs = {
    "i32": bqgen.i32_full(N, 3),
    "u64": bqgen.u64(N, 4),
    "f64": bqgen.f64(N, 5) * 2.0 - 1.0,
    "rec32": bqgen.rec32(N // 2, 6),
}
for kind, a in inputs.items():
    for ways in ([0, 2, 8, 16] if kind != "rec32" else [0]):
        for ordered in (False, True):
            t = dev(a)
            bq.bq_sort_ex(t, ways=ways, ordered=ordered)
            check(f"sort {kind} ways={ways} ordered={ordered}", keys_sorted(t, a))
    t = dev(a)
    bq.bq_sort_ex(t, depth_limit=1, ways=2)
    check(f"sort {kind} depth_limit=1 (fallback)", keys_sorted(t, a))
a = bqgen.rec32(N // 2, 7)
t = dev(a)
bq.bq_sort_ex(t, records=bq.RECORDS_DIRECT)
check("sort rec32 direct", keys_sorted(t, a))
# duplicates (equal bands, k_fill) and the leaf classes
a = bqgen.i32_range(N, 5, 8)
t = dev(a)
bq.bq_sort_ex(t)
check("sort i32 dups", keys_sorted(t, a))
for n in (1, 2, 33, 1000, 31744, 31745):
    a = bqgen.i32_full(n, n)
    t = dev(a)
    bq.bq_sort_i32(t)
    torch.cuda.synchronize()
    check(f"sort i32 n={n}", keys_sorted(t, a))
# passes, in-place partition, segments, pivots
a = bqgen.i32_full(N, 9)
src = dev(a)
dst = torch.empty_like(src)
c = torch.zeros(3, dtype=torch.int64, device="cuda")
p = bq.bq_pivot_i32(src, bq.BQ_PIVOT_MO3)
for ordered in (False, True):
    bq.bq_partition_pass(src, dst, p, c, ordered=ordered)
    torch.cuda.synchronize()
    check(f"pass i32 ordered={ordered}", c[0].item() == int((a < p).sum()))
t = dev(a)
s, e = bq.bq_partition_i32(t, p)
check("inplace i32", s == int((a < p).sum()) and e == int((a == p).sum()))
for kind, arr in (("f64", bqgen.f64(N, 10)), ("rec32", bqgen.rec32(N // 2, 11))):
    t = dev(arr)
    pv = bq.pivot(t, bq.BQ_PIVOT_SAMPLE64)
    s, e = bq.partition(t, pv)
    keys = arr[:, 0] if arr.ndim == 2 else arr
    check(f"inplace {kind}", s == int((keys < pv).sum()))
begins, lens = [0, 1000, 50000], [1000, 40000, 30000]
pivs = [int(a[b]) for b in begins]
c3 = torch.zeros(9, dtype=torch.int64, device="cuda")
bq.bq_partition_segments(src, dst, begins, lens, pivs, c3, ordered=True)
check("segments", all(c3[3 * i].item() == int((a[b:b + l] < pv).sum()) for i, (b, l, pv) in enumerate(zip(begins, lens, pivs))))
torch.cuda.synchronize()
print("FAILS", fails, flush=True)
sys.exit(1 if fails else 0)
