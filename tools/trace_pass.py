"""Per-tile phase trace of one partition pass (needs a -DBQ_TRACE build via BQ_LIB)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bqgen
import paper_1604_06697_b200 as bq
from paper_1604_06697_b200 import bq as B
n = 1 << 28
a = bqgen.i32_full(n, 1)
src = torch.from_numpy(a).cuda(); dst = torch.empty_like(src)
ws = bq.workspace(bq.BQ_I32, n); c = torch.zeros(3, dtype=torch.int64, device="cuda")
pv = bq.bq_pivot_i32(src, 0, ws=ws)
for _ in range(3):
    bq.bq_partition_pass(src, dst, pv, c, ordered=bool(int(os.environ.get('BQ_ORDERED', '0'))), ws=ws)
torch.cuda.synchronize()
ntiles = n // 4096
buf = np.zeros((1 << 17, 8), dtype=np.uint64)
B._lib.bq_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert B._lib.bq_debug_trace(buf.ctypes.data, buf.nbytes) == 0
tr = buf[:ntiles].astype(np.int64)
t0 = tr[:, 6].min()
issue, pub, cdone, start, b1, b3 = (tr[:, 6] - t0, tr[:, 5] - t0, tr[:, 4] - t0, tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 3] - t0)
pub = np.where(tr[:, 5] > 0, pub, cdone)
def pct(x):
    return {p: round(float(np.percentile(x, p)), 3) for p in (10, 50, 90, 99)}
out = {
    "span_us": float((b3.max() - issue.min()) / 1e3),
    "issue_to_agg_us": pct((pub - issue) / 1e3),
    "agg_to_lookback_done_us": pct((cdone - pub) / 1e3),
    "lookback_done_to_consumer_start_us": pct((start - cdone) / 1e3),
    "start_to_B1_us": pct((b1 - start) / 1e3),
    "B1_to_B2_us": pct((b3 - b1) / 1e3),
    "issue_to_B2_us": pct((b3 - issue) / 1e3),
}
cta = tr[:, 7] & 0xffffffff
order = np.lexsort((b3, cta))
gaps = np.diff(b3[order])[np.diff(cta[order]) == 0]
out["cta_tile_period_us"] = pct(gaps / 1e3)
print(json.dumps(out, indent=1))
# how late are the predecessors' aggregates relative to the tile's own?
from numpy.lib.stride_tricks import sliding_window_view
W = 256
aggv = pub.astype(np.int64)
mx = sliding_window_view(np.concatenate([np.full(W, aggv.min()), aggv]), W)[:-1].max(axis=1)
lag = (mx[:len(aggv)] - aggv)[W:]
claim_order = np.all(np.diff(issue) >= -2000)
extra = {"pred_agg_lag_us": pct(lag / 1e3), "issue_monotone_within_2us": bool(claim_order),
         "issue_jitter_us": pct((np.maximum.accumulate(issue) - issue) / 1e3),
         "agg_minus_issue_p999_us": float(np.percentile((pub - issue) / 1e3, 99.9)),
         "lookback_minus_agg_p10_90": [float(np.percentile((cdone - pub) / 1e3, q)) for q in (10, 50, 90)]}
print(json.dumps(extra))

scan_start = tr[:, 2] - t0; scan_end = tr[:, 1] - t0
hasscan = (tr[:, 2] > 0)
info = tr[:, 7].astype(np.uint64)
nret = ((info >> np.uint64(40)) & np.uint64(0x7fffff)).astype(np.int64)
nround = ((info >> np.uint64(32)) & np.uint64(0xff)).astype(np.int64)
m = hasscan
print(json.dumps({"claim_to_scan_start_us": pct(((scan_start - issue) / 1e3)[m]),
                  "scan_us": pct(((scan_end - scan_start) / 1e3)[m]),
                  "scan_end_minus_agg_us": pct(((scan_end - pub) / 1e3)[m]),
                  "retries": pct(nret[m]), "rounds": pct(nround[m])}))
