"""Profiling driver: a few out-of-place partition passes of config 2
(n = 2^28 int32, Mo3 pivot) and optionally one full sort, for ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bqgen
import paper_1604_06697_b200 as bq

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 28)
ap.add_argument("--passes", type=int, default=4)
ap.add_argument("--sort", type=int, default=0)
ap.add_argument("--kind", default="i32")
ap.add_argument("--fast", type=int, default=0, help="1: atomic-cursor (sort) placement")
ap.add_argument("--ways", type=int, default=0)
a = ap.parse_args()
if a.kind == "i32":
    src = torch.from_numpy(bqgen.i32_full(a.n, 1)).cuda()
elif a.kind == "f64":
    src = torch.from_numpy(bqgen.f64(a.n, 1)).cuda()
else:
    src = torch.from_numpy(bqgen.rec32(a.n, 1).view("int64")).cuda()
dst = torch.empty_like(src)
ws = bq.workspace(bq.kind_of(src), a.n)
counts = torch.zeros(3, dtype=torch.int64, device="cuda")
pv = bq.pivot(src, bq.BQ_PIVOT_MO3, ws=ws)
for _ in range(a.passes):
    bq.bq_partition_pass(src, dst, pv, counts, ordered=not a.fast, ws=ws)
for _ in range(a.sort):
    dst.copy_(src)
    st = bq.bq_sort_ex(dst, ws=ws, ways=a.ways)
torch.cuda.synchronize()
print("counts", counts.tolist(), "ok")
