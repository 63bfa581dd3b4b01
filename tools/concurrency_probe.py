"""Probe: does sorting independent halves concurrently (two host threads, two
streams) overlap one half's ALU-bound leaf sorts with the other half's
HBM-bound partition levels?  Prints wall-clock ms (device synchronised) of
  - one 2^28 int32 sort,
  - two 2^27 sorts one after the other,
  - two 2^27 sorts concurrently.
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bqgen
import paper_1604_06697_b200 as bq

n = 1 << 28
h = torch.from_numpy(bqgen.i32_full(n, 1)).cuda()
t = torch.empty_like(h)
ws = bq.workspace(bq.BQ_I32, n)
half = n // 2
wsa, wsb = bq.workspace(bq.BQ_I32, half), bq.workspace(bq.BQ_I32, half)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    out = []
    for _ in range(reps + 1):
        t.copy_(h)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
    out = sorted(out[1:])
    return out[len(out) // 2]


def one():
    bq.bq_sort_ex(t, ws=ws)


def seq():
    bq.bq_sort_ex(t[:half], ws=wsa, stream=sa)
    bq.bq_sort_ex(t[half:], ws=wsb, stream=sb)


def conc():
    th = [threading.Thread(target=lambda: bq.bq_sort_ex(t[:half], ws=wsa, stream=sa)),
          threading.Thread(target=lambda: bq.bq_sort_ex(t[half:], ws=wsb, stream=sb))]
    for x in th:
        x.start()
    for x in th:
        x.join()


print("one 2^28        ms", round(timed(one), 3))
print("two 2^27 seq    ms", round(timed(seq), 3))
print("two 2^27 conc   ms", round(timed(conc), 3))


def stag(delay_ms):
    def run():
        ta = threading.Thread(target=lambda: bq.bq_sort_ex(t[:half], ws=wsa, stream=sa))
        tb = threading.Thread(target=lambda: (time.sleep(delay_ms / 1e3), bq.bq_sort_ex(t[half:], ws=wsb, stream=sb)))
        ta.start()
        tb.start()
        ta.join()
        tb.join()
    return run


for d in (1.5, 2.5, 3.0, 3.5, 4.0):
    print(f"staggered {d} ms ms", round(timed(stag(d)), 3))
