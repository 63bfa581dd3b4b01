"""Repeated c2 sorts: per run the device time (CUDA events), the host time
of the call, and NVML SM clock / throttle reasons right after it — to tell
device slowdowns from host-side gaps between the level batches."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bqgen
import pynvml
import paper_1604_06697_b200 as bq
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 60
a = bqgen.config("c2", seed=1)
src = torch.from_numpy(a).cuda()
t = torch.empty_like(src)
ws = bq.workspace(bq.kind_of(src), len(src))
rows = []
for i in range(R):
    t.copy_(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(); st = bq.bq_sort_ex(t, ws=ws); e1.record()
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    clk = pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM)
    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hdl)
    rows.append((round(e0.elapsed_time(e1), 3), round((h1 - h0) * 1e3, 3), clk, rs, st["levels"]))
ev = sorted(r[0] for r in rows)
print(json.dumps({"med": ev[len(ev) // 2], "slow": [r for r in rows if r[0] > 1.2 * ev[len(ev) // 2]]}))
