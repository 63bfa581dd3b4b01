"""Full-size parity (-m gpu): BASELINE.json's five configs at their stated n,
in the launch configuration bench.py times (bq_sort_ex defaults: ninther
pivots, atomic-cursor placement, persistent partition CTAs).

north_star target: "bit-exact sorted output versus the CPU oracle on all five
configs".  The oracle (single-threaded CPU BlockQuicksort) finishes 2^28 int32
keys in about ten seconds, so every config is compared with it in full, byte
for byte; on top of that the plain definition of sorted position is checked
on sampled outputs (#{a < out[i]} <= i < #{a <= out[i]}) and each config's
closed form where it has one (SURVEY §8(c) "Sort" pins).
"""
import numpy as np
import pytest
import torch

import bqgen
import oracle
from gpu_util import to_dev, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def B(bq):
    assert torch.cuda.is_available()
    return bq


def sampled_ranks(inp_keys, out_keys, samples=12, seed=0):
    rng = np.random.default_rng(seed)
    n = len(out_keys)
    for i in rng.integers(0, n, size=samples):
        v = out_keys[i]
        lo = int(np.count_nonzero(inp_keys < v))
        hi = int(np.count_nonzero(inp_keys <= v))
        assert lo <= i < hi, (i, lo, hi)


def run_sort(B, a):
    t = to_dev(a)
    st = B.bq_sort_ex(t)
    got = to_host(t, a)
    del t
    torch.cuda.empty_cache()
    return got, st


@pytest.mark.parametrize("name", ["c1", "c2", "c4a", "c4b"])
def test_full_int32_configs(B, name):
    a = bqgen.config(name, seed=1)
    got, st = run_sort(B, a)
    exp = oracle.sort(a)
    assert np.array_equal(got, exp)                     # bit-exact vs oracle
    assert st["fallback_segments"] == 0
    sampled_ranks(a, got)
    if name == "c1":
        assert np.array_equal(got, np.arange(len(a), dtype=np.int32))
    elif name == "c4a":
        counts = np.bincount(a, minlength=int(a.max()) + 1)
        assert np.array_equal(got, np.repeat(np.arange(len(counts), dtype=np.int32), counts))
    elif name == "c4b":
        assert np.array_equal(got, a) and st["levels"] == 1


@pytest.mark.parametrize("ordering", ["random", "ascending", "descending", "swapped"])
def test_full_c3_float64(B, ordering):
    a = bqgen.config("c3", seed=1, ordering=ordering)
    got, st = run_sort(B, a)
    assert np.array_equal(got.view(np.uint64), oracle.sort(a).view(np.uint64))
    assert st["fallback_segments"] == 0
    sampled_ranks(a, got)
    if ordering != "random":
        assert np.array_equal(got, bqgen.f64(len(a), 1, "ascending"))   # closed form (R11)


def test_full_c5_records(B):
    a = bqgen.config("c5", seed=1)
    got, st = run_sort(B, a)
    exp = oracle.sort(a)
    assert np.array_equal(got[:, 0], exp[:, 0])
    idx = got[:, 1].astype(np.int64)
    assert np.array_equal(np.sort(idx), np.arange(len(a)))
    assert (got[:, 1] == got[:, 2]).all() and (got[:, 2] == got[:, 3]).all()
    assert np.array_equal(got[:, 0], a[idx, 0])
    sampled_ranks(a[:, 0], got[:, 0])


def test_full_c2_partition(B):
    """BASELINE config 2's roofline unit: one three-way partition of 2^28
    int32 keys around the Mo3 pivot, checked against the oracle's counts and
    the band predicates."""
    a = bqgen.config("c2", seed=1)
    t = to_dev(a)
    p = B.bq_pivot_i32(t, B.BQ_PIVOT_MO3)
    assert p == oracle.pivot(a, oracle.MO3)
    split, neq = B.bq_partition_i32(t, p)
    assert split == int(np.count_nonzero(a < p)) and neq == int(np.count_nonzero(a == p))
    assert bool((t[:split] < p).all()) and bool((t[split:split + neq] == p).all())
    assert bool((t[split + neq:] > p).all())
    got = t.cpu().numpy()
    assert np.array_equal(np.sort(got), np.sort(a))


def test_sort_2pow30_int32(B):
    """Beyond the configs: n = 2^30 int32 (4 GiB + 4 GiB workspace) exercises
    the 32-bit segment offsets, tile counts and packed per-tile counters at
    scale; checked against torch.sort (a library radix sort) and by sampled
    ranks on the device."""
    n = 1 << 30
    g = torch.Generator(device="cuda").manual_seed(11)
    src = torch.randint(-(1 << 31), (1 << 31) - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    ref = torch.sort(src)[0]
    t = src.clone()
    st = B.bq_sort_ex(t)
    assert bool(torch.equal(t, ref))
    assert st["fallback_segments"] == 0
    del ref
    for i in [0, 12345, n // 3, n - 1]:
        v = t[i]
        assert int((src < v).sum()) <= i < int((src <= v).sum())


NMAX = (1 << 31) - 1   # include/bq.h: n <= 2^31 - 1


def _free_cuda():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def test_sort_max_n_int32(B):
    """The largest n the C-ABI accepts (2^31 - 1 int32 keys, 8 GiB + 8 GiB of
    workspace): equal to torch.sort (a library radix sort), sampled ranks on
    the device."""
    g = torch.Generator(device="cuda").manual_seed(12)
    src = torch.randint(-(1 << 31), (1 << 31) - 1, (NMAX,), dtype=torch.int32, device="cuda", generator=g)
    t = src.clone()
    st = B.bq_sort_ex(t)
    assert st["fallback_segments"] == 0
    ref = torch.sort(src)[0]
    assert bool(torch.equal(t, ref))
    del ref
    for i in [0, 777, NMAX // 2, NMAX - 1]:
        v = t[i]
        assert int((src < v).sum()) <= i < int((src <= v).sum())
    del src, t
    _free_cuda()


def test_sort_max_n_uint64(B):
    """2^31 - 1 uint64 keys (16 GiB), top bit clear so torch's int64 sort
    orders them the same way; the default 8-way passes at the size limit."""
    g = torch.Generator(device="cuda").manual_seed(13)
    src = torch.randint(0, (1 << 62) - 1, (NMAX,), dtype=torch.int64, device="cuda", generator=g)
    t = src.clone()
    st = B.bq_sort_ex(t.view(torch.uint64))
    assert st["fallback_segments"] == 0
    ref = torch.sort(src)[0]
    assert bool(torch.equal(t, ref))
    del src, t, ref
    _free_cuda()


def test_partition_max_n_int32(B):
    """bq_partition_i32 (in place, N2) at 2^31 - 1 keys: the split and the
    equal count equal the plain counts, the three bands hold, and the multiset
    is unchanged (compared sorted)."""
    g = torch.Generator(device="cuda").manual_seed(14)
    src = torch.randint(-1000, 1000, (NMAX,), dtype=torch.int32, device="cuda", generator=g)
    t = src.clone()
    p = 17
    split, neq = B.bq_partition_i32(t, p)
    assert split == int((src < p).sum()) and neq == int((src == p).sum())
    assert bool((t[:split] < p).all()) and bool((t[split:split + neq] == p).all())
    assert bool((t[split + neq:] > p).all())
    assert bool(torch.equal(torch.bincount(t.long() + 1000, minlength=2000),
                            torch.bincount(src.long() + 1000, minlength=2000)))
    del src, t
    _free_cuda()


def test_sort_records_2pow30(B):
    """2^30 records (32 GiB) through the default key+index path: the keys come
    out equal to torch.sort of the keys, every record travels whole (its
    payload words are functions of its key and original position), and the
    positions form a permutation (each names a record with that key)."""
    n = 1 << 30
    g = torch.Generator(device="cuda").manual_seed(15)
    r = torch.empty((n, 4), dtype=torch.int64, device="cuda")
    r[:, 0] = torch.randint(0, 1 << 40, (n,), dtype=torch.int64, device="cuda", generator=g)
    r[:, 1] = torch.arange(n, dtype=torch.int64, device="cuda")
    r[:, 2] = r[:, 0] ^ 0x5A5A5A5A
    r[:, 3] = r[:, 1] * 3
    keys = r[:, 0].clone()
    st = B.bq_sort_ex(r)
    assert st["fallback_segments"] == 0
    assert bool(torch.equal(r[:, 0], torch.sort(keys)[0]))
    assert bool(torch.equal(r[:, 2], r[:, 0] ^ 0x5A5A5A5A)) and bool(torch.equal(r[:, 3], r[:, 1] * 3))
    assert bool(torch.equal(keys[r[:, 1]], r[:, 0]))
    seen = torch.zeros(n, dtype=torch.bool, device="cuda")
    seen[r[:, 1]] = True
    assert bool(seen.all())
    del r, keys, seen
    _free_cuda()
