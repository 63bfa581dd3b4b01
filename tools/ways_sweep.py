"""Sort time by ways (2 / 8 / 16) across n for int32, uint64 and key+index
pairs (CUDA events, median of 5): the data behind the default `ways`."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bqgen
import paper_1604_06697_b200 as bq
LOGS = [int(x) for x in os.environ.get("SWEEP_LOGS", "16,18,20,22,24,26,28").split(",")]
KINDS = os.environ.get("SWEEP_KINDS", "i32,u64,pair").split(",")
for kind in KINDS:
    for lg in LOGS:
        n = 1 << lg
        if kind == "u64" and lg > 27 or kind == "pair" and lg > 26:
            continue
        if kind == "i32":
            h = torch.from_numpy(bqgen.i32_full(n, 1))
        elif kind == "u64":
            h = torch.from_numpy(bqgen.u64(n, 1).view(np.int64)).view(torch.uint64)
        else:
            a = np.empty((n, 2), dtype=np.uint64); a[:, 0] = bqgen.u64(n, 1); a[:, 1] = np.arange(n, dtype=np.uint64)
            h = torch.from_numpy(a.view(np.int64))  # (n, 2): key+index pairs
        src = h.cuda(); t = torch.empty_like(src); ws = bq.workspace(bq.kind_of(src), n)
        res = {}
        for w in (2, 8, 16):
            ts = []
            for i in range(6):
                t.copy_(src)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); bq.bq_sort_ex(t, ws=ws, ways=w); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[w] = round(sorted(ts[1:])[2], 3)
        print(json.dumps({"kind": kind, "log2n": lg, "ms": res}), flush=True)
        del src, t, ws; torch.cuda.empty_cache()
