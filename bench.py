#!/usr/bin/env python
"""bench.py — BASELINE.json's metric on one B200 (or N independent replicas).

Metric: "sort Gkeys/s at n=2^28 int32 (1 B200); partition-pass HBM GB/s vs
peak".  A *step* is one full bq_sort (every hot-path row a1-a9) of config 2:
n = 2^28 int32 keys, i.i.d. uniform over the full int32 range (bqgen, seeded;
synthetic like the paper's mt19937 inputs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl bq|reference]

Timing (device, CUDA events on the stream the library launches on):
  * value / ms_per_step: sum over the K timed steps of the event time around
    the bq_sort call; before each step the input is restored from a pristine
    device copy outside the events.  Inputs (1 GiB) are larger than the
    126 MB L2, and the restore copy streams 2 GiB through it as well.
  * roofline: the kernel family with the largest share of the step (the
    library's timing mode records CUDA events around the binary partition,
    multiway count/scatter and leaf launches, bq_sort_options.timing);
    achieved = its algorithmic bytes per sort / its summed launch time;
    roofline_by_kernel lists every family.
  * partition_pass: BASELINE.md's roofline measurement — 10 single out-of-place
    passes over the pristine input around its Mo3 pivot, L2 flushed before each.
  * e2e: bq_sort_host (H2D from pinned memory + sort + D2H) per step; value =
    K such steps software-pipelined over three streams (one step's H2D runs
    under another's sort and D2H), e2e.serial = one step at a time.
  * cpu_baseline: the oracle (oracle/, single-threaded) on a bounded sample.
Multi-GPU (--gpus N under torchrun): replicas only — every rank
sorts its own copy; the time is the max over ranks; value = N*n / time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_FULL = 1 << 28
WORKLOAD = "c2: int32 keys, n=2^28, iid uniform over the full int32 range (seeded SplitMix64); full bq_sort"
METRIC = "sort Gkeys/s at n=2^28 int32 (1 B200); partition-pass HBM GB/s vs peak"
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_traffic(kernel):
    """DRAM bytes (read + write) of all launches of `kernel` inside one c2
    sort and its active launches, from the committed ncu capture summary."""
    p = os.path.join(ROOT, "profiles", "r02", "ncu_sort_dram.json")
    try:
        with open(p) as f:
            d = json.load(f)[kernel]
        return d["dram_bytes_total"], max(d["active_launches"], 1), "profiles/r02/ncu_sort_dram.json"
    except Exception:
        return None, None, None


def partition_pass_by_config(bq, bqgen, dev, stream, passes, peak):
    """north_star: "each partition pass at >= 60% of B200 peak HBM bandwidth" on
    every config.  Binary passes: BASELINE.md's measurement (10 single
    out-of-place passes around the Mo3 pivot of the pristine input, L2 flushed
    before each, median).  Multiway (8-way, the sort's default for 64-bit keys
    and key+index pairs): every multiway level of a sort of the config (count +
    scan + scatter, CUDA events), algorithmic bytes 2 w per element like a
    binary pass (the count pass's extra read counts against it)."""
    import numpy as np
    import torch
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def entry(ms, nbytes, **kw):
        gbs = nbytes / (ms * 1e-3) / 1e9
        return dict(kw, ms_median=ms, bytes=nbytes, gbs=gbs, frac_of_measured=gbs / peak,
                    frac_of_8tbs=gbs / 8000.0, meets_bar=gbs >= 4800.0)

    def time_passes(src, dst, pv, ordered, ws):
        counts = torch.zeros(3, dtype=torch.int64, device=dev)
        times = []
        for _ in range(passes + 1):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            bq.bq_partition_pass(src, dst, pv, counts, ordered=ordered, ws=ws, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        return statistics.median(times[1:])

    def time_mw(data, src, ws):
        st = []
        for _ in range(3):
            data.copy_(src)
            flush.fill_(1)
            st.append(bq.bq_sort_ex(data, timing=True, ws=ws, stream=stream))
        ms = statistics.median(s["multiway_ms"] for s in st)
        return ms, st[-1]["multiway_element_passes"], st[-1], {
            "scatter_ms": statistics.median(s["mw_scatter_ms"] for s in st),
            "count_scan_ms": statistics.median(s["mw_count_ms"] for s in st)}

    def mw_entry(ms, ep, st, parts, w, **kw):
        """an 8-way level: 2 w per element-pass against the whole level (the
        count's extra read counts against it), and each kernel on its own bytes
        (scatter: read + write, count: read)"""
        e = entry(ms, 2 * w * ep, element_passes=ep, levels=st["levels"], **kw)
        sc, cn = parts["scatter_ms"], parts["count_scan_ms"]
        moved = 3 * w * ep / (ms * 1e-3) / 1e9
        e["level_bytes_moved_frac_of_measured"] = moved / peak
        # the same bar on the bytes the level's two passes really move (count:
        # one read; scatter: read + write), and per kernel — `meets_bar` above
        # stays the strict reading (2 w per element-pass over the whole level)
        e["level_bytes_moved_frac_of_8tbs"] = moved / 8000.0
        e["meets_bar_by_bytes_moved"] = moved / 8000.0 >= 0.6
        sg, cg = 2 * w * ep / (sc * 1e-3) / 1e9, w * ep / (cn * 1e-3) / 1e9
        e["scatter"] = {"ms": sc, "gbs": sg, "frac_of_measured": sg / peak, "frac_of_8tbs": sg / 8000.0,
                        "meets_bar": sg / 8000.0 >= 0.6}
        e["count_scan"] = {"ms": cn, "gbs": cg, "frac_of_measured": cg / peak, "frac_of_8tbs": cg / 8000.0,
                           "meets_bar": cg / 8000.0 >= 0.6}
        return e

    out = {}
    # c3: float64, n = 2^27, random
    a = bqgen.config("c3", seed=1, ordering="random")
    n3 = len(a)
    src = torch.from_numpy(a).to(dev)
    dst = torch.empty_like(src)
    ws = bq.workspace(bq.BQ_F64, n3, dev)
    pv = bq.bq_pivot_f64(src, bq.BQ_PIVOT_MO3, ws=ws, stream=stream)
    out["c3_f64_binary_pass"] = entry(time_passes(src, dst, pv, False, ws), 16 * n3, n=n3)
    out["c3_f64_8way_levels"] = mw_entry(*time_mw(dst, src, ws), 8, n=n3)
    del src, dst, ws
    # c2: int32, n = 2^28: the sort's 8-way levels (its default)
    a = bqgen.config("c2", seed=1)
    n2 = len(a)
    src = torch.from_numpy(a).to(dev)
    dst = torch.empty_like(src)
    ws = bq.workspace(bq.BQ_I32, n2, dev)
    out["c2_i32_8way_levels"] = mw_entry(*time_mw(dst, src, ws), 4, n=n2)
    del src, dst, ws
    # c4a: int32, n = 2^28, 16384 distinct values
    a = bqgen.config("c4a", seed=1)
    n4 = len(a)
    src = torch.from_numpy(a).to(dev)
    dst = torch.empty_like(src)
    ws = bq.workspace(bq.BQ_I32, n4, dev)
    pv = bq.bq_pivot_i32(src, bq.BQ_PIVOT_MO3, ws=ws, stream=stream)
    out["c4a_i32_binary_pass"] = entry(time_passes(src, dst, pv, False, ws), 8 * n4, n=n4)
    del src, dst, ws
    # c5: 32-byte records, n = 2^26: the records pass, the key+index pairs' pass
    # and the pairs' 8-way levels (the records sort's default path)
    r = bqgen.config("c5", seed=1)
    n5 = len(r)
    src = torch.from_numpy(r.view(np.int64)).to(dev)
    dst = torch.empty_like(src)
    ws = bq.workspace(bq.BQ_REC32, n5, dev)
    pv = bq.bq_pivot_records(src, bq.BQ_PIVOT_MO3, ws=ws, stream=stream)
    out["c5_rec32_pass"] = entry(time_passes(src, dst, pv, True, ws), 64 * n5, n=n5,
                                 note="records: the standalone pass is the three-way ordered placement")
    out["c5_pairs_8way_levels"] = mw_entry(*time_mw(dst, src, ws), 16, n=n5,
                                           note="key+index pairs (16 B) of the records sort")
    pairs = torch.empty((n5, 2), dtype=torch.int64, device=dev)
    pairs[:, 0] = src[:, 0]
    pairs[:, 1] = torch.arange(n5, dtype=torch.int64, device=dev)
    pdst = torch.empty_like(pairs)
    del dst
    out["c5_pairs_pass"] = entry(time_passes(pairs, pdst, pv, True, ws), 32 * n5, n=n5,
                                 note="pairs: the standalone pass is the three-way ordered placement")
    del src, pairs, pdst, ws, flush
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------ distributed ----

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def reduce_max(value: float, world: int, device=None) -> float:
    """Max over ranks (replica timing).  Works for nccl (device tensor) and gloo."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate(n_per_rank: int, ms_total_max: float, steps: int, world: int):
    """Whole-job throughput of `world` replicas each sorting n_per_rank keys per
    step: (Gkeys/s, ms_per_step)."""
    ms_per_step = ms_total_max / steps
    return world * n_per_rank / (ms_per_step * 1e-3) / 1e9, ms_per_step


# ---------------------------------------------------------------- clocks -----

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.offset = 0
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # nvidia-smi's start-up (driver attach) stalls CUDA calls of this
        # process for tens of ms (measured: two 9 ms steps took 21-26 ms when
        # it started inside the timed region); its steady 100 ms polling does
        # not.  Wait for its first sample before the timed region begins.
        t0 = time.time()
        while time.time() - t0 < 5.0:
            self.f.flush()
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.05)
        time.sleep(0.2)
        self.f.flush()
        self.offset = os.path.getsize(self.path)   # samples from here on fall in (or just after) the timed region

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        def parse(text):
            out = []
            for line in text.splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    out.append(parts)
            return out
        text = open(self.path).read()
        rows = parse(text[getattr(self, "offset", 0):]) or parse(text)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------- cpu baselines ---

def e2e_pipelined(bq, torch, keys_np, data, ws, stream, dev, n, args):
    """K end-to-end sorts through the public API, software-pipelined over S = 3
    streams (step i on stream i mod S, each stream with its own device buffer
    and workspace): every step copies its own input from pinned host memory
    (H2D), sorts it (bq_sort_ex, the graph launch) and reads the whole result
    back (D2H).  The H2D copies are chained across steps, and so are the D2H
    copies, so each link carries one copy at a time and step i+1's H2D runs
    under step i's sort and D2H (PCIe is full duplex).  Each step has its own
    pinned input/output buffer, filled before the timed region.  Time: CUDA
    events from before the first copy to the end of the last D2H."""
    import numpy as np
    S = 3
    K = max(S, args.e2e_pipe_steps)
    hosts = [torch.from_numpy(keys_np).pin_memory() for _ in range(K)]
    devs = [data] + [torch.empty_like(data) for _ in range(S - 1)]
    wss = [ws] + [bq.workspace(bq.BQ_I32, n, dev) for _ in range(S - 1)]
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(S - 1)]
    for j in range(S):   # warm-up: each buffer set's sort graph is instantiated here
        devs[j].copy_(torch.from_numpy(keys_np).to(dev))
        bq.bq_sort_ex(devs[j], pivot_rule=args.pivot_rule, ws=wss[j], stream=streams[j], stats=False)
    torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    start, end = ev(), ev()
    start.record(streams[0])
    prev_h2d = prev_d2h = start
    for i in range(K):
        st, d = streams[i % S], devs[i % S]
        st.wait_event(prev_h2d)
        with torch.cuda.stream(st):
            d.copy_(hosts[i], non_blocking=True)
        prev_h2d = ev()
        prev_h2d.record(st)
        bq.bq_sort_ex(d, pivot_rule=args.pivot_rule, ws=wss[i % S], stream=st, stats=False)
        st.wait_event(prev_d2h)
        with torch.cuda.stream(st):
            hosts[i].copy_(d, non_blocking=True)
        prev_d2h = ev()
        prev_d2h.record(st)
    streams[0].wait_event(prev_d2h)
    end.record(streams[0])
    torch.cuda.synchronize()
    ms_total = start.elapsed_time(end)
    ok = all(bool(np.all(h.numpy()[1:] >= h.numpy()[:-1])) for h in (hosts[0], hosts[-1]))
    if not ok:
        raise RuntimeError("pipelined e2e: a result is not sorted")
    return {"steps": K, "streams": S, "ms_total": ms_total, "results_sorted": ok,
            "how": "K steps (H2D of the step's own pinned input, bq_sort_ex, D2H of its result) "
                   "on 3 streams with their own buffers; H2D copies chained, D2H copies chained; "
                   "events from before the first copy to the end of the last D2H"}


def host_facts():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "usable_cores": usable}


def cpu_baseline(keys_np, sample_n: int):
    """The oracle (as it stands) and std::sort, single-threaded, on the first
    sample_n keys of the workload (the full c2 n by default)."""
    import oracle
    s = keys_np[:sample_n].copy()
    t0 = time.perf_counter()
    out = oracle.sort(s, inplace=True)
    t_or = time.perf_counter() - t0
    s2 = keys_np[:sample_n].copy()
    t0 = time.perf_counter()
    oracle.std_sort(s2, inplace=True)
    t_std = time.perf_counter() - t0
    import numpy as np
    assert np.array_equal(out, s2)
    full = sample_n == len(keys_np)
    return {"value": sample_n / t_or / 1e9, "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
            "sample": (f"the whole c2 input (n = 2^{int(math.log2(sample_n))})" if full else
                       f"first {sample_n} keys of the c2 input (2^{int(math.log2(sample_n))})") + ", one run",
            "seconds": t_or, "host": host_facts(),
            "std_sort": {"value": sample_n / t_std / 1e9, "unit": "Gkeys/s", "cores": 1, "seconds": t_std}}


# ------------------------------------------------------------- reference -----

def run_reference(args, rank, world):
    """--impl reference: the oracle (CPU, as it stands) on bounded samples of the
    same workload.  Under torchrun only rank 0 runs and prints."""
    if rank != 0:
        return 0
    import numpy as np
    import bqgen
    import oracle
    sample = 1 << 22
    keys = bqgen.i32_full(sample, 1)
    for _ in range(args.warmup):
        oracle.sort(keys)
    ts = []
    for _ in range(args.steps):
        s = keys.copy()
        t0 = time.perf_counter()
        oracle.sort(s, inplace=True)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * sum(ts) / len(ts)
    value = sample / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gkeys/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": f"each step sorts the first 2^22 keys of the c2 input"},
        "cpu_baseline": {"value": value, "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
                         "sample": "first 2^22 keys of the c2 input per step", "host": host_facts()},
        "e2e": {"value": value, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- main ----

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bq", choices=["bq", "reference"])
    ap.add_argument("--n", type=int, default=N_FULL, help="keys per GPU (default 2^28)")
    ap.add_argument("--pivot-rule", type=int, default=2, help="0 Mo3, 1 ninther, 2 median of a 64-key sample")
    ap.add_argument("--passes", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-pipe-steps", type=int, default=-1,
                    help="end-to-end sorts pipelined over three streams (0: serial e2e only; default 12 at N=1, 6 per rank above)")
    ap.add_argument("--cpu-sample", type=int, default=1 << 28)
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config partition-pass table")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    args = ap.parse_args()
    if args.e2e_pipe_steps < 0:
        args.e2e_pipe_steps = 12 if int(os.environ.get("WORLD_SIZE", "1")) == 1 else 6
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import bqgen
    import paper_1604_06697_b200 as bq

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    n = args.n
    keys_np = bqgen.i32_full(n, seed=1 + rank)
    src = torch.from_numpy(keys_np).to(dev)
    data = torch.empty_like(src)
    ws = bq.workspace(bq.BQ_I32, n, dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        # the product path: fully asynchronous graph launch, no host wait
        bq.bq_sort_ex(data, pivot_rule=args.pivot_rule, ws=ws, stream=stream, stats=False)

    for _ in range(args.warmup):
        data.copy_(src)
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        data.copy_(src)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_total = sum(step_ms)
    ms_total_max = reduce_max(ms_total, world, dev)
    value, ms_per_step = aggregate(n, ms_total_max, args.steps, world)

    verified = None
    if not args.no_verify:
        ref = torch.sort(src)[0]          # a library routine (CUB radix sort), test-only check
        verified = bool(torch.equal(ref, data))
        del ref

    # statistics of one (untimed) step: the device counters of the same sort
    data.copy_(src)
    last = bq.bq_sort_ex(data, pivot_rule=args.pivot_rule, ws=ws, stream=stream)

    # roofline of the dominant kernel: the sort's host-driven mode
    # (bq_sort_options.timing; same kernels, same levels as the graph) records
    # CUDA events on the launching streams around the binary partition
    # launches, the multiway count + scan and scatter launches of every level
    # and the leaf launches; the kernel with the largest share of the step is
    # reported, every kernel family in roofline_by_kernel
    peak, peak_src = load_peak()
    tstats = []
    for _ in range(3):
        data.copy_(src)
        tstats.append(bq.bq_sort_ex(data, pivot_rule=args.pivot_rule, timing=True, ws=ws, stream=stream))
    avg = lambda k: sum(s[k] for s in tstats) / len(tstats)
    mwp = avg("multiway_element_passes")
    fams = {
        "k_part_fast": ("tile partition pass (binary levels)", avg("partition_bytes"), avg("partition_ms"),
                        "HBM (0.92 of the copy bandwidth in r02 session 1)"),
        "k_mw8t_scatter": ("8-way scatter (multiway levels): read + write of every key", 8.0 * mwp,
                           avg("mw_scatter_ms"), "issue: ~45 instructions per key, ALU pipe 60 % (ncu, profiles/r02)"),
        "k_mw8w_count": ("8-way count + scan (multiway levels): read of every key", 4.0 * mwp, avg("mw_count_ms"),
                         "issue / HBM (ncu, profiles/r02)"),
        "k_leaf": ("leaf sort (a8): read + write of every leaf key", 8.0 * N_FULL, avg("leaf_ms"),
                   "shared memory: 78 % of the wavefront rate, issue 55 % (ncu, profiles/r02/ncu_full_r02.md)"),
    }
    by_kernel = {}
    for kname, (desc, nbytes, ms, bound) in fams.items():
        if ms <= 0 or nbytes <= 0:
            continue
        ach = nbytes / (ms * 1e-3) / 1e9
        by_kernel[kname] = {"what": desc, "bytes_per_sort": nbytes, "ms_per_sort": ms, "achieved": ach,
                            "frac": ach / peak, "share_of_step": ms / ms_per_step, "bound_by": bound}
    # the dominant family: the largest summed kernel time in the committed ncu
    # launch list of one c2 sort (serialised, per-kernel durations); the
    # timing mode's leaf span also holds the leaf classes' launch gaps and
    # tails, so its shares are only the fallback
    dom_src = "timing mode"
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ncu_sort_dram.json")) as f:
            nc = json.load(f)
        cand = {k: nc[k]["ms"] for k in by_kernel if k in nc}
        dom = max(cand, key=cand.get)
        dom_src = "ncu launch list (profiles/r02/ncu_sort_dram.json): " + ", ".join(
            f"{k} {v:.3f} ms" for k, v in sorted(cand.items(), key=lambda kv: -kv[1]))
    except Exception:
        dom = max(by_kernel, key=lambda k: by_kernel[k]["ms_per_sort"])
    dk = by_kernel[dom]
    traffic_total, active, traffic_src = load_traffic(dom)   # one whole c2 sort under ncu (same input, same levels)
    roofline = {
        "bound": "hbm", "achieved": dk["achieved"], "peak": peak, "unit": "GB/s", "frac": dk["frac"],
        "peak_source": peak_src,
        "kernel": dom + " (" + dk["what"] + ")",
        "dominant_by": dom_src,
        "algorithmic_bytes_per_sort": dk["bytes_per_sort"],
        "ms_per_sort": dk["ms_per_sort"],
        "share_of_step": dk["share_of_step"],
        "active_launches": active,
        "algorithmic_bytes_per_launch": dk["bytes_per_sort"] / active if active else None,
        "traffic": traffic_total / active if traffic_total else None,
        "traffic_per": "active launch (ncu, one whole c2 sort: the kernel's DRAM read + write over its launches "
                       "longer than 20 us; algorithmic_bytes_per_launch uses the same divisor)",
        "traffic_source": traffic_src,
        "how": "CUDA events on the launching stream around every launch of the kernel family (bq_sort_options."
               "timing: the host-driven level loop, same kernels as the graph), averaged over 3 sorts; "
               "achieved = algorithmic bytes / that time; share = that time / ms_per_step",
    }

    # BASELINE.md partition-pass measurement: 10 single passes, L2 flushed
    ppass = None
    if args.passes > 0:
        pv = bq.bq_pivot_i32(src, bq.BQ_PIVOT_MO3, ws=ws, stream=stream)
        counts = torch.zeros(3, dtype=torch.int64, device=dev)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        def passes(ordered):
            times = []
            for _ in range(args.passes + 1):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                bq.bq_partition_pass(src, data, pv, counts, ordered=ordered, ws=ws, stream=stream)
                b.record(stream)
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
            return times[1:]
        times = passes(False)          # the sort's placement (atomic cursor)
        times_ord = passes(True)       # the deterministic layout (decoupled look-back)
        times_ip = []                  # bq_partition_i32: the in-place block partition (N2)
        for _ in range(args.passes + 1):
            data.copy_(src)
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            bq.bq_partition_i32(data, pv, ws=ws, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            times_ip.append(a.elapsed_time(b))
        times_ip = times_ip[1:]
        del flush
        pbytes = 2 * 4 * n
        med, mn = statistics.median(times), min(times)
        c = counts.cpu().tolist()
        ppass = {"passes": args.passes, "bytes": pbytes, "pivot": pv, "split": c[0], "n_equal": c[1],
                 "ms_median": med, "ms_min": mn,
                 "gbs_median": pbytes / (med * 1e-3) / 1e9, "gbs_max": pbytes / (mn * 1e-3) / 1e9,
                 "frac_median": pbytes / (med * 1e-3) / 1e9 / peak,
                 "frac_of_8tbs_median": pbytes / (med * 1e-3) / 1e9 / 8000.0,
                 "ordered_ms_median": statistics.median(times_ord),
                 "ordered_gbs_median": pbytes / (statistics.median(times_ord) * 1e-3) / 1e9,
                 "inplace_ms_median": statistics.median(times_ip),
                 "inplace_gbs_median": pbytes / (statistics.median(times_ip) * 1e-3) / 1e9,
                 "note": "one bq_partition_pass (partition kernel + per-segment counts + band kernel) "
                         "over the pristine c2 input around its Mo3 pivot, atomic-cursor placement as "
                         "in the sort; L2 flushed (512 MiB write) before each; ordered_* = the "
                         "deterministic decoupled look-back placement (bq_partition_pass ordered=1); "
                         "inplace_* = bq_partition_i32, the in-place block partition (N2) with its "
                         "equal band, input restored before each call"}

    by_config = None
    if args.passes > 0 and not args.no_configs and rank == 0:
        by_config = partition_pass_by_config(bq, bqgen, dev, stream, args.passes, peak)

    # end to end through the public API with host buffers
    e2e = None
    if args.e2e_steps > 0:
        host = torch.from_numpy(keys_np.copy()).pin_memory()
        t_e2e = []
        for i in range(args.e2e_steps + 1):
            host.copy_(torch.from_numpy(keys_np))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            bq.bq_sort_host(host, data, pivot_rule=args.pivot_rule, ws=ws, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            if i > 0:
                t_e2e.append(a.elapsed_time(b))
        e2e_ms = reduce_max(sum(t_e2e), world, dev) / len(t_e2e)
        serial = {"value": world * n / (e2e_ms * 1e-3) / 1e9, "unit": "Gkeys/s", "ms_per_step": e2e_ms,
                  "how": "one stream: each step's H2D, sort and D2H back to back (bq_sort_host)"}
        e2e = {"value": serial["value"], "unit": "Gkeys/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n, "ms_per_step": e2e_ms,
               "serial": serial}
        if args.e2e_pipe_steps > 0:
            try:
                pipe = e2e_pipelined(bq, torch, keys_np, data, ws, stream, dev, n, args)
                pipe_ms = pipe["ms_total"] / pipe["steps"]
            except (RuntimeError, MemoryError) as ex:   # e.g. pinned host memory exhausted
                pipe, pipe_ms = {"error": str(ex)[:200]}, float("inf")
            # (every rank reaches the reduction, a failed one with inf)
            pipe_ms = reduce_max(pipe_ms, world, dev)
            if "error" not in pipe and math.isfinite(pipe_ms):
                pipe.update({"value": world * n / (pipe_ms * 1e-3) / 1e9, "unit": "Gkeys/s",
                             "ms_per_step": pipe_ms})
                e2e.update({"value": pipe["value"], "ms_per_step": pipe_ms, "pipelined": pipe})
            else:
                e2e["pipelined"] = pipe

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(keys_np, min(args.cpu_sample, n))

    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_per_gpu": n, "pivot_rule": ["mo3", "ninther", "sample64"][args.pivot_rule],
                   "parallelism": f"replicas{world}" if world > 1 else "1gpu",
                   "l2": "inputs (1 GiB) larger than L2 (126 MB); restore copy between steps is untimed",
                   "timing": "sum of per-step CUDA events around bq_sort (the asynchronous graph launch) "
                             "on the launch stream"},
        "roofline": roofline,
        "roofline_by_kernel": by_kernel,
        "partition_pass": ppass,
        "partition_pass_by_config": by_config,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(last["kernel_launches"]) * args.steps,
        "clocks": clk,
        "sort_stats": {k: last[k] for k in ("levels", "partition_launches", "kernel_launches", "element_passes",
                                            "partitioned_segments", "leaves", "fallback_segments",
                                            "band_elements")},
        "passes_per_element": last["element_passes"] / n,
        "verified_vs_torch_sort": verified,
        "step_ms": step_ms,
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
