"""Time N2's in-place partition (bq_partition_inplace) against the
out-of-place pass (bq_partition_pass, fast and ordered) on config 2's input
(n = 2^28 int32, Mo3 pivot) and the other kinds at 2^27 / 2^25 elements.
CUDA events on the current stream; the input is restored from a pristine copy
before every timed call (the copy is outside the timed region).  Prints one
JSON line per (kind, variant)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bqgen
import paper_1604_06697_b200 as bq

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--kinds", default="i32,u64,f64,rec32")
ap.add_argument("--only", default="", help="time just this variant")
a = ap.parse_args()

cases = [("i32", 1 << 28), ("u64", 1 << 27), ("f64", 1 << 27), ("rec32", 1 << 25)]
for kind, n in cases:
    if kind not in a.kinds.split(","):
        continue
    if kind == "i32":
        h = torch.from_numpy(bqgen.i32_full(n, 1))
    elif kind == "u64":
        h = torch.from_numpy(bqgen.u64(n, 1).view("int64"))
    elif kind == "f64":
        h = torch.from_numpy(bqgen.f64(n, 1))
    else:
        h = torch.from_numpy(bqgen.rec32(n, 1).view("int64"))
    src = h.cuda()
    t = torch.empty_like(src)
    dst = torch.empty_like(src)
    k = bq.kind_of(src)
    ws = bq.workspace(k, n)
    iws = torch.empty(bq.bq_inplace_workspace_bytes(k, n), dtype=torch.uint8, device="cuda")
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    pv = bq.pivot(src, bq.BQ_PIVOT_MO3, ws=ws)
    nbytes = src.numel() * src.element_size()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        ms = []
        for r in range(a.reps + 1):
            t.copy_(src)
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r:
                ms.append(e0.elapsed_time(e1))
        ms.sort()
        return ms[len(ms) // 2]

    fns = {
        "inplace": lambda: bq.bq_partition_inplace(t, pv, ws=iws),
        "pass_fast": lambda: bq.bq_partition_pass(t, dst, pv, counts, ordered=False, ws=ws),
        "pass_ordered": lambda: bq.bq_partition_pass(t, dst, pv, counts, ordered=True, ws=ws),
        "partition_api": lambda: bq.partition(t, pv, ws=ws),   # ordered pass + copy-back (n scratch)
    }
    res = {name: timed(fn) for name, fn in fns.items() if not a.only or name == a.only}
    for name, ms in res.items():
        print(json.dumps({"kind": kind, "n": n, "variant": name, "ms": round(ms, 4),
                          "tb_s_rw": round(2 * nbytes / ms / 1e9, 3),
                          "workspace_mb": round((iws.numel() if name == "inplace" else ws.numel()) / 2**20, 1)}))
    del src, t, dst, ws, iws
    torch.cuda.empty_cache()
