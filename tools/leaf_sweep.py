"""Sort time by leaf_max (the BQ_LEAF_MAX override of driver.cuh's
leaf_max_for) and by the loop batch's extra levels across small n (CUDA
events, median of 7; every result checked against torch.sort): the data
behind leaf_max_for's small-input rule."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bqgen
import paper_1604_06697_b200 as bq
LOGS = [int(x) for x in os.environ.get("SWEEP_LOGS", "16,17,18,19,20,21,22,23,24").split(",")]
KINDS = os.environ.get("SWEEP_KINDS", "i32,u64").split(",")
LMS = [int(x) for x in os.environ.get("SWEEP_LMS", "0,16,8,4,2").split(",")]   # 0 = built-in rule, else IPT * 32 * x
EXTRAS = [int(x) for x in os.environ.get("SWEEP_EXTRAS", "0,1").split(",")]
WAYS = [int(x) for x in os.environ.get("SWEEP_WAYS", "0").split(",")]
for kind in KINDS:
    for lg in LOGS:
        n = 1 << lg
        if kind == "i32":
            h = torch.from_numpy(bqgen.i32_full(n, 1))
        else:
            h = torch.from_numpy(bqgen.u64(n, 1).view(np.int64)).view(torch.uint64)
        src = h.cuda()
        ref = torch.sort(src)[0] if kind == "i32" else None
        t = torch.empty_like(src)
        S = bq.leaf_elems(bq.kind_of(src))
        res = {}
        for x in LMS:
            for ex in EXTRAS:
                for w in WAYS:
                    if x:
                        os.environ["BQ_LEAF_MAX"] = str(S // 32 * x)
                    else:
                        os.environ.pop("BQ_LEAF_MAX", None)
                    os.environ["BQ_BATCH_EXTRA"] = str(ex)
                    ws = bq.workspace(bq.kind_of(src), n)
                    ts = []
                    for i in range(8):
                        t.copy_(src)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(); bq.bq_sort_ex(t, ws=ws, ways=w); e1.record(); torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    if ref is not None:
                        assert torch.equal(t, ref), (kind, lg, x, ex, w)
                    else:
                        d = t.cpu().numpy()
                        assert (d[1:] >= d[:-1]).all(), (kind, lg, x, ex, w)
                    res[f"lm{x}_e{ex}_w{w}"] = round(sorted(ts[1:])[3], 4)
                    del ws
        print(json.dumps({"kind": kind, "log2n": lg, "S": S, "ms": res}), flush=True)
        del src, t; torch.cuda.empty_cache()
