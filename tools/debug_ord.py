"""Debug the ordered multi-segment pass (k_part_ord)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as B
from gpu_util import three_list, to_dev, to_host
for kind, n in [("i32", (1 << 24) + 5), ("i32", (1 << 23) + 5), ("u64", (1 << 20) + 5), ("u64", (1 << 21) + 5), ("u64", 600000)]:
    for nseg in [1, 2, 3]:
        rng = np.random.default_rng(nseg)
        a = bqgen.i32_full(n, nseg) if kind == "i32" else bqgen.u64(n, nseg)
        cuts = np.sort(rng.choice(np.arange(1, n), size=nseg, replace=False)) if nseg > 1 else np.array([], dtype=np.int64)
        bounds = np.concatenate([[0], cuts, [n]])
        begins = bounds[:-1]; lens = np.diff(bounds)
        pivots = [a[b + rng.integers(0, l)] for b, l in zip(begins, lens)]
        src = to_dev(a); dst = torch.zeros_like(src)
        counts = torch.zeros(3 * len(begins), dtype=torch.int64, device="cuda")
        B.bq_partition_segments(src, dst, begins, lens, pivots, counts)
        got = to_host(dst, a)
        bad = []
        for i, (b, l, p) in enumerate(zip(begins, lens, pivots)):
            exp = three_list(a[b:b + l], p)
            g = got[b:b + l]
            if not np.array_equal(g, exp):
                d = np.nonzero(g != exp)[0]
                L = int((a[b:b+l] < p).sum()); E = int((a[b:b+l] == p).sum())
                bad.append((i, int(b), int(l), L, E, int(d[0]), int(d[-1]), len(d), bool(np.array_equal(np.sort(g), np.sort(exp)))))
        print(kind, n, nseg, "OK" if not bad else bad[:3], flush=True)
