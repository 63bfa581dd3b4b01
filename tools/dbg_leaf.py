"""Leaf debug: sort int32 arrays of several sizes, compare with torch.sort, report mismatches."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as bq
for n, ways in [(1 << 20, 2), (1 << 22, 2), (1 << 24, 2), (1 << 26, 2), (1 << 28, 0), (1 << 22, 8)]:
    a = bqgen.i32_full(n, seed=1)
    t = torch.from_numpy(a).cuda()
    ref = torch.sort(t)[0]
    st = bq.bq_sort_ex(t, ways=ways)
    bad = (t != ref).nonzero().flatten()
    print(n, ways, "mismatches", bad.numel(), "leaves", st["leaves"], "levels", st["levels"], flush=True)
    if bad.numel():
        b0 = int(bad[0]); b1 = int(bad[-1])
        print("  first", b0, "last", b1, "span", b1 - b0, flush=True)
        # runs of mismatches
        d = torch.diff(bad)
        brk = (d > 1).nonzero().flatten()
        starts = [b0] + [int(bad[i + 1]) for i in brk[:20]]
        print("  run starts", starts[:20], "nruns", brk.numel() + 1, flush=True)
        print("  got", t[b0:b0 + 8].tolist(), "ref", ref[b0:b0 + 8].tolist(), flush=True)
