"""Debug the 8-way scatter: sort permutations with ways=8 and report what the
output lost or duplicated.  usage: dbg_mw8t.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1604_06697_b200 as bq
for lg in (13, 15, 16, 18, 20):
    n = 1 << lg
    rng = np.random.default_rng(lg)
    a = rng.permutation(n).astype(np.int32)
    t = torch.from_numpy(a).cuda()
    st = bq.bq_sort_ex(t, ways=8)
    g = t.cpu().numpy()
    ok = np.array_equal(g, np.arange(n, dtype=np.int32))
    ms = np.array_equal(np.sort(g), np.arange(n, dtype=np.int32))
    bad = np.nonzero(g != np.arange(n))[0]
    cnt = np.bincount(g.astype(np.int64) % n, minlength=n) if len(g) else None
    print(lg, "ok", ok, "multiset", ms, "nbad", len(bad), "first", bad[:8].tolist(), "vals", g[bad[:8]].tolist(),
          "missing", int((cnt == 0).sum()), "dup", int((cnt > 1).sum()), "levels", st.get("levels"),
          "ep", st.get("element_passes"), flush=True)
for lg in (15, 18, 20, 22):
    n = 1 << lg
    rng = np.random.default_rng(lg)
    a = np.empty((n, 2), dtype=np.uint64); a[:, 0] = rng.permutation(n).astype(np.uint64) * 7919; a[:, 1] = np.arange(n, dtype=np.uint64)
    t = torch.from_numpy(a.view(np.int64)).cuda()
    try:
        st = bq.bq_sort_ex(t, ways=8)
        g = t.cpu().numpy().view(np.uint64)
        ok = np.array_equal(g[:, 0], np.sort(a[:, 0]))
        ms = np.array_equal(np.sort(g[:, 1]), np.arange(n, dtype=np.uint64))
        print("pairs", lg, "ok", ok, "idx multiset", ms, "levels", st.get("levels"), flush=True)
    except Exception as e:
        print("pairs", lg, "ERR", str(e)[:200], flush=True)
        break
