import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as bq
n = (1 << 22) + 7
a = bqgen.i32_full(n, 22)
exp = np.sort(a)
for dl in list(range(1, 18)) + [-1]:
    t = torch.from_numpy(a).cuda()
    st = bq.bq_sort_ex(t, depth_limit=dl)
    got = t.cpu().numpy()
    bad = np.nonzero(got != exp)[0]
    print("depth_limit", dl, "levels", st["levels"], "fb", st["fallback_segments"], "mismatch", len(bad), bad[:3], flush=True)
