import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as bq
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22) + 7
dl = int(sys.argv[2]) if len(sys.argv) > 2 else 4
a = bqgen.i32_full(n, 22)
t = torch.from_numpy(a).cuda()
st = bq.bq_sort_ex(t, depth_limit=dl)
got = t.cpu().numpy()
bad = np.nonzero(got != np.sort(a))[0]
print("n", n, "depth_limit", dl, "levels", st["levels"], "mismatch", len(bad), bad[:3], flush=True)
