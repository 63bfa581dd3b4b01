"""One bq_sort of a BASELINE config at full size after one untimed warm-up
sort (for ncu launch lists).  usage: one_sort.py CONFIG [--ways W]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bqgen
import paper_1604_06697_b200 as bq

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--ways", type=int, default=0)
args = ap.parse_args()
a = bqgen.config(args.config, seed=1)
if a.dtype == np.uint64:
    a = a.view(np.int64)
src = torch.from_numpy(a).cuda()
dst = torch.empty_like(src)
ws = bq.workspace(bq.kind_of(src), len(src))
for _ in range(2):
    dst.copy_(src)
    bq.bq_sort_ex(dst, ws=ws, ways=args.ways, stats=False)
torch.cuda.synchronize()
print("ok", args.config)
