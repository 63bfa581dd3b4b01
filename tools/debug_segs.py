"""GPU debug: batched multi-segment pass vs the per-segment three-list definition."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as bq

def three(a, p):
    return np.concatenate([a[a < p], a[a == p], a[a > p][::-1]])

rng = np.random.default_rng(0)
for n, nseg in [(1 << 22, 2), (1 << 22, 4), (1 << 22, 8), (1 << 22, 16), (1 << 22, 100), (1 << 20, 64), (1 << 24, 8)]:
    a = bqgen.i32_full(n, nseg)
    cuts = np.sort(rng.choice(np.arange(1, n), size=nseg - 1, replace=False))
    bounds = np.concatenate([[0], cuts, [n]])
    begins, lens = bounds[:-1], np.diff(bounds)
    pivots = [int(a[b + l // 2]) for b, l in zip(begins, lens)]
    src = torch.from_numpy(a).cuda(); dst = torch.zeros_like(src)
    c = torch.zeros(3 * nseg, dtype=torch.int64, device="cuda")
    bq.bq_partition_segments(src, dst, begins, lens, pivots, c)
    got = dst.cpu().numpy(); cc = c.cpu().numpy().reshape(-1, 3)
    nbad, nbadc = 0, 0
    for i, (b, l, p) in enumerate(zip(begins, lens, pivots)):
        seg = a[b:b + l]
        exp = three(seg, np.int32(p))
        if not np.array_equal(got[b:b + l], exp):
            nbad += 1
            if nbad <= 3:
                d = np.nonzero(got[b:b + l] != exp)[0]
                print("  seg", i, "b", b, "len", l, "first bad", d[:4], "nbad", len(d), "L", int((seg < p).sum()))
        if tuple(cc[i]) != (int((seg < p).sum()), int((seg == p).sum()), int((seg > p).sum())):
            nbadc += 1
    print("n", n, "nseg", nseg, "bad segments", nbad, "bad counts", nbadc, flush=True)
