"""Probe for staggered groups: G independent slices of the c2 input sorted by G
host threads on G streams, thread k starting k*delay ms after thread 0, so one
slice's ALU-bound leaf sorts can overlap the next slice's HBM-bound level
passes.  Wall clock (device synchronised), median of 5."""
import os, sys, threading, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bqgen
import paper_1604_06697_b200 as bq
n = 1 << 28
h = torch.from_numpy(bqgen.i32_full(n, 1)).cuda()
t = torch.empty_like(h)
wsf = bq.workspace(bq.BQ_I32, n)
res = {}
def timed(fn, reps=5):
    out = []
    for _ in range(reps + 1):
        t.copy_(h); torch.cuda.synchronize()
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
    out = sorted(out[1:]); return round(out[len(out) // 2], 3)
res["one"] = timed(lambda: bq.bq_sort_ex(t, ws=wsf))
for G in (2, 4):
    m = n // G
    wss = [bq.workspace(bq.BQ_I32, m) for _ in range(G)]
    sts = [torch.cuda.Stream() for _ in range(G)]
    for d in (0.0, 1.0, 2.0, 3.0):
        def run():
            th = [threading.Thread(target=lambda k=k: (time.sleep(k * d / 1e3),
                  bq.bq_sort_ex(t[k * m:(k + 1) * m], ws=wss[k], stream=sts[k]))) for k in range(G)]
            for x in th: x.start()
            for x in th: x.join()
        res[f"G{G}_d{d}"] = timed(run)
    del wss
print(json.dumps({"lib": os.path.basename(bq.LIB_PATH), **res}))
