import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from test_gpu_parity import make, LEAF, check_sorted_equal
from gpu_util import to_dev, to_host
import paper_1604_06697_b200 as B
for kind in ["i32", "f64", "rec32"]:
    n = 10 * LEAF[kind] + 7
    a = make(kind, n, seed=9)
    for ways, limits in [(2, [0, 1, 2]), (16, [0, 1])]:
        for limit in limits:
            t = to_dev(a)
            st = B.bq_sort_ex(t, depth_limit=limit, ways=ways)
            check_sorted_equal(kind, to_host(t, a), a)
            print(kind, ways, limit, st["fallback_segments"], st["levels"], st["leaves"], flush=True)
