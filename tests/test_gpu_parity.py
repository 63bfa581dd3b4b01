"""Parity of the CUDA path (through the C-ABI) against the CPU oracle (-m gpu).

Bars: everything here is integer / byte work, so every
comparison is bit-exact — float64 is compared by bit pattern, records by key
sequence plus the payload rule of SURVEY §8(c) (the order inside runs of
equal keys is unspecified, as in Quicksort).
"""
import numpy as np
import pytest
import torch

import bqgen
import oracle
from gpu_util import three_list, to_dev, to_host

pytestmark = pytest.mark.gpu

import paper_1604_06697_b200 as _bq

# tile T and leaf S per kind (csrc/common.cuh Tune<>, queried through the C-ABI)
TILE = {k: _bq.tile_elems(_bq.KIND[k]) for k in ("i32", "u64", "f64", "rec32")}
LEAF = {k: _bq.leaf_elems(_bq.KIND[k]) for k in ("i32", "u64", "f64", "rec32")}


def edge_sizes(kind):
    T, S = TILE[kind], LEAF[kind]
    return sorted({0, 1, 2, 3, 31, 32, 33, T - 1, T, T + 1, 2 * T - 1, 2 * T + 1,
                   S - 1, S, S + 1, 3 * S + 7, (1 << 16) + 3})


def make(kind, n, seed=1, dist="random"):
    if kind == "i32":
        if dist == "dups":
            return bqgen.i32_range(n, 17, seed) - 8
        return bqgen.i32_full(n, seed)
    if kind == "u64":
        if dist == "dups":
            return bqgen.u64(n, seed) >> np.uint64(60)
        return bqgen.u64(n, seed)
    if kind == "f64":
        a = bqgen.f64(n, seed) * 2.0 - 1.0
        if dist == "dups":
            a = np.round(a, 1)
            a[a == 0] = 0.0
            a[::5] = -0.0      # signed zeros: -0.0 < +0.0 (R9)
        return a
    if kind == "rec32":
        return bqgen.rec32(n, seed, dup_keys=23 if dist == "dups" else None)
    raise KeyError(kind)


def keys_of(a):
    return a[:, 0] if a.ndim == 2 else a


def f64_key(a):
    """The totalOrder rank key of doubles, for the three-list layout pin."""
    b = a.view(np.uint64)
    return np.where(b >> np.uint64(63), ~b, b | np.uint64(1 << 63))


def check_sorted_equal(kind, got, inp):
    exp = oracle.sort(inp)
    if kind == "rec32":
        assert np.array_equal(got[:, 0], exp[:, 0])
        idx = got[:, 1].astype(np.int64)
        assert np.array_equal(np.sort(idx), np.arange(len(inp)))
        assert (got[:, 1] == got[:, 2]).all() and (got[:, 2] == got[:, 3]).all()
        assert np.array_equal(got[:, 0], inp[idx, 0])
    elif kind == "f64":
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    else:
        assert np.array_equal(got, exp)


@pytest.fixture(scope="module")
def B(bq):
    assert torch.cuda.is_available()
    return bq


# ------------------------------------------------------------------ sort ------

@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
@pytest.mark.parametrize("dist", ["random", "dups"])
def test_sort_edge_sizes(B, kind, dist):
    for n in edge_sizes(kind):
        a = make(kind, n, seed=n + 11, dist=dist)
        t = to_dev(a)
        B.sort(t)
        check_sorted_equal(kind, to_host(t, a), a)


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
@pytest.mark.parametrize("rule", [0, 1, 2])
def test_sort_medium(B, kind, rule):
    for n in [100003, (1 << 20) + 17]:
        a = make(kind, n, seed=7)
        t = to_dev(a)
        st = B.bq_sort_ex(t, pivot_rule=rule)
        check_sorted_equal(kind, to_host(t, a), a)
        assert st["levels"] >= 1 and st["fallback_segments"] == 0


@pytest.mark.parametrize("kind", ["i32", "u64", "f64"])
def test_sort_unaligned_pointer(B, kind):
    for n in [5000, 70001]:
        a = make(kind, n, seed=3)
        t = to_dev(a, offset=1)
        assert t.data_ptr() % 16 != 0
        B.sort(t)
        check_sorted_equal(kind, to_host(t, a), a)


@pytest.mark.parametrize("kind", ["i32", "u64", "f64"])
def test_sort_multiway_unaligned_pointer(B, kind):
    """8-way levels over a buffer that is not 16-byte aligned: the scatter
    without bulk copies (k_mw8w_scatter) places the keys; aligned, the same
    input goes through the TMA-staged scatter (k_mw8t_scatter)."""
    for n in [300007, (1 << 20) + 5]:
        a = make(kind, n, seed=11)
        for off in (1, 0):
            t = to_dev(a, offset=off)
            assert (t.data_ptr() % 16 != 0) == (off == 1)
            st = B.bq_sort_ex(t, ways=8)
            check_sorted_equal(kind, to_host(t, a), a)
            assert st["multiway_element_passes"] > 0 and st["fallback_segments"] == 0


def test_sort_configs_reduced(B):
    n = 1 << 20
    for name in ["c1", "c2", "c4a", "c4b", "c5"]:
        a = bqgen.config(name, n, seed=2)
        t = to_dev(a)
        B.sort(t)
        check_sorted_equal("rec32" if name == "c5" else "i32", to_host(t, a), a)
    for ordering in ["random", "ascending", "descending", "swapped"]:
        a = bqgen.config("c3", n, seed=2, ordering=ordering)
        t = to_dev(a)
        st = B.bq_sort_ex(t)
        got = to_host(t, a)
        check_sorted_equal("f64", got, a)
        if ordering != "random":
            assert np.array_equal(got, bqgen.f64(n, 2, "ascending"))   # closed form


def test_sort_closed_forms(B):
    n = (1 << 20) + 3
    a = bqgen.i32_perm(n, 5)
    t = to_dev(a)
    B.sort(t)
    assert np.array_equal(t.cpu().numpy(), np.arange(n, dtype=np.int32))
    c = bqgen.i32_const(n)
    t = to_dev(c)
    st = B.bq_sort_ex(t)
    assert np.array_equal(t.cpu().numpy(), c)
    assert st["levels"] == 1 and st["band_elements"] == n


def test_sort_special_f64(B):
    table = np.array([0xfff0000000000000, 0xffefffffffffffff, 0xbff0000000000000, 0x8010000000000000,
                      0x8000000000000001, 0x8000000000000000, 0x0, 0x1, 0x0010000000000000,
                      0x3ff0000000000000, 0x7fefffffffffffff, 0x7ff0000000000000],
                     dtype=np.uint64).view(np.float64)
    rng = np.random.default_rng(3)
    for n in [12, 1000, 50000]:
        a = table[rng.integers(0, len(table), size=n)]
        t = to_dev(a)
        B.sort(t)
        got = t.cpu().numpy()
        assert np.array_equal(got.view(np.uint64), oracle.sort(a).view(np.uint64))


@pytest.mark.parametrize("kind", ["i32", "f64", "rec32"])
def test_depth_cap_fallback(B, kind):
    # a tiny Introsort limit sends segments to the merge-based fallback (a9):
    # binary passes at n ~ 10 S leave segments longer than S down to depth 2;
    # 16-way passes at n ~ 40 S leave children of ~2.5 S at depth 1
    for ways, limits, m in [(2, [0, 1, 2], 10), (16, [0, 1], 40)]:
        n = m * LEAF[kind] + 7
        a = make(kind, n, seed=9)
        for limit in limits:
            t = to_dev(a)
            st = B.bq_sort_ex(t, depth_limit=limit, ways=ways)
            check_sorted_equal(kind, to_host(t, a), a)
            assert st["fallback_segments"] >= 1


def test_sort_deterministic(B):
    # the ordered (decoupled look-back) placement fixes the layout of every
    # pass, so even the order of equal-key records is reproducible; the default
    # atomic-cursor placement only guarantees the sorted keys (R10)
    a = make("rec32", 200000, seed=4, dist="dups")
    outs = []
    for _ in range(2):
        t = to_dev(a)
        B.bq_sort_ex(t, ordered=True)
        outs.append(t.cpu().numpy())
        check_sorted_equal("rec32", outs[-1], a)
    assert np.array_equal(outs[0], outs[1])
    t = to_dev(a)
    B.bq_sort_ex(t)
    check_sorted_equal("rec32", to_host(t, a), a)


# ------------------------------------------------------------- partition ------

def _pivots(kind, a):
    k = keys_of(a)
    if len(k) == 0:
        return [0]
    ps = [k[len(k) // 2], k.min(), k.max()]
    if kind == "i32":
        ps += [np.int32(0), np.int32(-(1 << 31)), np.int32((1 << 31) - 1)]
    elif kind in ("u64", "rec32"):
        ps += [np.uint64(0), np.uint64(1 << 63), np.uint64((1 << 64) - 1)]
    else:
        ps += [0.0, -0.0, 0.5, -2.0]
    return ps


def _bands_ok(kind, a, got, pv, split, neq):
    """The partition invariants (the unique part of a partition's output):
    the three bands hold exactly the keys <, == and > the pivot, and the
    multiset (for records: every row whole) is preserved."""
    if kind == "f64":
        k, pk = f64_key(got), f64_key(np.array([pv]))[0]
        assert np.array_equal(np.sort(got.view(np.uint64)), np.sort(a.view(np.uint64)))
    elif kind == "rec32":
        k, pk = got[:, 0], np.uint64(pv)
        idx = got[:, 1].astype(np.int64)
        assert np.array_equal(np.sort(idx), np.arange(len(a)))
        assert (got[:, 1] == got[:, 2]).all() and (got[:, 2] == got[:, 3]).all()
        assert np.array_equal(got[:, 0], a[idx, 0])
    else:
        k, pk = got, np.array(pv, dtype=a.dtype)
        assert np.array_equal(np.sort(got), np.sort(a))
    assert (k[:split] < pk).all() and (k[split:split + neq] == pk).all() and (k[split + neq:] > pk).all()


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
@pytest.mark.parametrize("dist", ["random", "dups"])
def test_partition_vs_oracle(B, kind, dist):
    """bq_partition_* (in place, N2): split and n_equal exactly the oracle's,
    the band invariants and the multiset; the ordered out-of-place pass on the
    same input: exactly the oracle's deterministic layout (the three-list
    definition, gpu_util.three_list)."""
    for n in edge_sizes(kind):
        a = make(kind, n, seed=n + 5, dist=dist)
        for p in _pivots(kind, a):
            pv = float(p) if kind == "f64" else int(p)
            _, s_o, e_o = oracle.partition(a, pv)
            t = to_dev(a)
            split, neq = B.partition(t, pv)
            assert (split, neq) == (s_o, e_o)
            _bands_ok(kind, a, to_host(t, a), pv, split, neq)
            if n == 0:
                continue
            src = to_dev(a)
            dst = torch.empty_like(src)
            counts = torch.zeros(3, dtype=torch.int64, device="cuda")
            B.bq_partition_pass(src, dst, pv, counts, ordered=True)
            assert counts.cpu().tolist()[:2] == [s_o, e_o]
            got = to_host(dst, a)
            if kind == "f64":
                exp = three_list(a, f64_key(np.array([pv]))[0], key=f64_key)
                assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
            elif kind == "rec32":
                exp = three_list(a, np.uint64(pv), key=lambda x: x[:, 0])
                assert np.array_equal(got, exp)
            else:
                exp = three_list(a, np.array(pv, dtype=a.dtype))
                assert np.array_equal(got, exp)


def test_partition_config1_closed_form(B):
    a = bqgen.config("c1")
    t = to_dev(a)
    p = B.bq_pivot_i32(t, B.BQ_PIVOT_MO3)
    assert p == oracle.pivot(a, oracle.MO3)
    split, neq = B.bq_partition_i32(t, p)
    assert split == p and neq == 1          # permutation of 0..n-1
    got = t.cpu().numpy()
    assert (got[:split] < p).all() and got[split] == p and (got[split + 1:] > p).all()


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
def test_partition_pass_out_of_place(B, kind):
    n = (1 << 18) + 77
    a = make(kind, n, seed=21, dist="dups")
    src = to_dev(a)
    dst = torch.empty_like(src)
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    p = keys_of(a)[n // 3]
    pv = float(p) if kind == "f64" else int(p)
    B.bq_partition_pass(src, dst, pv, counts)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(src, a), a)            # src untouched
    _, s_o, e_o = oracle.partition(a, pv)
    c = counts.cpu().numpy()
    assert (c[0], c[1], c[2]) == (s_o, e_o, n - s_o - e_o)
    got = to_host(dst, a)
    if kind == "f64":
        exp = three_list(a, f64_key(np.array([pv]))[0], key=f64_key)
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    elif kind == "rec32":
        assert np.array_equal(got, three_list(a, np.uint64(pv), key=lambda x: x[:, 0]))
    else:
        assert np.array_equal(got, three_list(a, np.array(pv, dtype=a.dtype)))


@pytest.mark.parametrize("kind", ["i32", "u64", "f64"])
@pytest.mark.parametrize("n", [1, 4097, (1 << 20) + 3, (1 << 23) + 5])
def test_partition_pass_fast_mode(B, kind, n):
    """Atomic-cursor placement (the sort's default): tiles land in completion
    order, so check the plain definition: bands, counts and the multiset; and
    that every tile's < run is a contiguous, in-order subsequence."""
    a = make(kind, n, seed=n + 3, dist="dups")
    src = to_dev(a)
    dst = torch.empty_like(src)
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    p = keys_of(a)[n // 2]
    pv = float(p) if kind == "f64" else int(p)
    B.bq_partition_pass(src, dst, pv, counts, ordered=False)
    got = to_host(dst, a)
    if kind == "f64":
        ka, kg, pk = f64_key(a), f64_key(got), f64_key(np.array([pv]))[0]
    else:
        ka, kg, pk = a, got, np.array(pv, dtype=a.dtype)
    s_, e_ = int((ka < pk).sum()), int((ka == pk).sum())
    assert counts.cpu().tolist() == [s_, e_, n - s_ - e_]
    assert (kg[:s_] < pk).all() and (kg[s_:s_ + e_] == pk).all() and (kg[s_ + e_:] > pk).all()
    assert np.array_equal(np.sort(kg), np.sort(ka))


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
def test_partition_pass_persistent_reuse(B, kind):
    # enough tiles that every persistent CTA cycles its TMA ring many times
    n = ((1 << 23) if kind != "rec32" else (1 << 21)) + 13
    a = make(kind, n, seed=31)
    src = to_dev(a)
    dst = torch.empty_like(src)
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    p = keys_of(a)[7]
    pv = float(p) if kind == "f64" else int(p)
    B.bq_partition_pass(src, dst, pv, counts)
    got = to_host(dst, a)
    if kind == "f64":
        exp = three_list(a, f64_key(np.array([pv]))[0], key=f64_key)
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    elif kind == "rec32":
        assert np.array_equal(got, three_list(a, np.uint64(pv), key=lambda x: x[:, 0]))
    else:
        assert np.array_equal(got, three_list(a, np.array(pv, dtype=a.dtype)))


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
@pytest.mark.parametrize("nseg", [2, 8, 37, 100])
def test_partition_segments(B, kind, nseg):
    """One breadth-first level of many segments at once (segment boundaries
    inside tiles, every alignment), each against its own three-list layout."""
    rng = np.random.default_rng(nseg)
    n = (1 << 22) + 5 if kind != "rec32" else (1 << 20) + 5
    a = make(kind, n, seed=nseg, dist="dups" if nseg % 2 else "random")
    cuts = np.sort(rng.choice(np.arange(1, n), size=nseg, replace=False))
    bounds = np.concatenate([[0], cuts, [n]])
    keep = rng.random(nseg + 1) < 0.8            # leave some gaps uncovered
    begins = bounds[:-1][keep]
    lens = np.diff(bounds)[keep]
    k = keys_of(a)
    pivots = [k[b + rng.integers(0, l)] for b, l in zip(begins, lens)]
    src = to_dev(a)
    dst = torch.zeros_like(src)
    counts = torch.zeros(3 * len(begins), dtype=torch.int64, device="cuda")
    B.bq_partition_segments(src, dst, begins, lens, pivots, counts)
    got = to_host(dst, a)
    c = counts.cpu().numpy().reshape(-1, 3)
    for i, (b, l, p) in enumerate(zip(begins, lens, pivots)):
        seg = a[b:b + l]
        if kind == "f64":
            exp = three_list(seg, f64_key(np.array([p]))[0], key=f64_key)
            assert np.array_equal(got[b:b + l].view(np.uint64), exp.view(np.uint64)), i
            sk, pk = f64_key(seg), f64_key(np.array([p]))[0]
        elif kind == "rec32":
            exp = three_list(seg, p, key=lambda x: x[:, 0])
            assert np.array_equal(got[b:b + l], exp), i
            sk, pk = seg[:, 0], p
        else:
            exp = three_list(seg, p)
            assert np.array_equal(got[b:b + l], exp), i
            sk, pk = seg, p
        assert tuple(c[i]) == (int((sk < pk).sum()), int((sk == pk).sum()), int((sk > pk).sum())), i


def test_sort_large_levels(B):
    # many multi-segment levels with persistent CTAs: the shape that exposed
    # the staging-overflow bug (DESIGN.md log)
    for lg in [22, 24]:
        a = bqgen.i32_full((1 << lg) + 7, lg)
        t = to_dev(a)
        B.sort(t)
        assert np.array_equal(t.cpu().numpy(), np.sort(a))


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
def test_pivot_rules(B, kind):
    for n in [1, 2, 3, 8, 9, 10, 63, 64, 65, 1000, 123457]:
        a = make(kind, n, seed=n)
        t = to_dev(a)
        for rule in [0, 1, 2]:
            got = B.pivot(t, rule)
            exp = oracle.pivot(a, rule)
            if kind == "f64":
                assert np.array([got]).view(np.uint64)[0] == np.array([exp]).view(np.uint64)[0]
            else:
                assert got == exp


def test_errors_are_loud(B):
    t = torch.zeros(10, dtype=torch.int32, device="cuda")
    small_ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(B.BQError):
        B.bq_sort_i32(t, ws=small_ws)
    with pytest.raises(B.BQError):
        B.bq_partition_f64(torch.zeros(4, dtype=torch.float64, device="cuda"), float("nan"))


def test_sort_host_e2e(B):
    a = bqgen.i32_full((1 << 20) + 9, 13)
    host = torch.from_numpy(a.copy()).pin_memory()
    dev = torch.empty_like(host, device="cuda")
    B.bq_sort_host(host, dev)
    assert np.array_equal(host.numpy(), oracle.sort(a))


# ------------------------------------- the paper's structured inputs (N3) ------

PATTERNS = ["imodsqrt", "square", "pow8", "sorted", "reversed", "rotation",
            "swaps_sqrt", "swaps_n", "swaps_nlogn", "halfhalf", "zeroone"]


def pattern_as(kind, p):
    """The int32 pattern mapped order-preservingly into each kind (u64 above
    2^63 and f64 negatives exercise the unsigned compare and the H0 codec)."""
    if kind == "i32":
        return p
    if kind == "u64":
        return p.astype(np.uint64) + np.uint64(1 << 63)
    if kind == "f64":
        return p.astype(np.float64) * 0.25 - 1000.0
    r = np.empty((len(p), 4), dtype=np.uint64)
    r[:, 0] = p.astype(np.uint64) * np.uint64(3)
    r[:, 1] = r[:, 2] = r[:, 3] = np.arange(len(p), dtype=np.uint64)
    return r


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
@pytest.mark.parametrize("name", PATTERNS)
def test_sort_patterns(B, kind, name):
    for n in [(1 << 16) + 3, (1 << 20) + 1]:
        if name == "swaps_nlogn" and n > (1 << 17):
            continue                       # the generator itself is O(n log n) serial swaps
        a = pattern_as(kind, bqgen.i32_pattern(name, n, seed=3))
        for rule in [1, 2]:
            t = to_dev(a)
            st = B.bq_sort_ex(t, pivot_rule=rule)
            check_sorted_equal(kind, to_host(t, a), a)
            if rule == 2:
                # the jittered sample keeps periodic inputs off the depth cap
                # (the paper's deterministic ninther may fall back on them,
                # which is exactly what the Introsort limit is for)
                assert st["fallback_segments"] == 0


@pytest.mark.parametrize("name", ["pow8", "halfhalf", "rotation"])
def test_sort_patterns_ordered_placement(B, name):
    a = bqgen.i32_pattern(name, (1 << 20) + 5, seed=4)
    t = to_dev(a)
    B.bq_sort_ex(t, ordered=True)
    assert np.array_equal(t.cpu().numpy(), oracle.sort(a))


# ------------------------------------------ multi-pivot block partition (N4) ---

@pytest.mark.parametrize("ways", [8, 16])
@pytest.mark.parametrize("kind", ["i32", "u64", "f64"])
@pytest.mark.parametrize("dist", ["random", "dups"])
def test_sort_multiway(B, kind, dist, ways):
    for n in [S_ + 1 for S_ in (LEAF[kind],)] + [100003, (1 << 20) + 17, (1 << 22) + 3]:
        a = make(kind, n, seed=n % 97, dist=dist)
        t = to_dev(a)
        st = B.bq_sort_ex(t, ways=ways)
        check_sorted_equal(kind, to_host(t, a), a)
        assert st["fallback_segments"] == 0


@pytest.mark.parametrize("ways", [8, 16])
@pytest.mark.parametrize("name", PATTERNS)
def test_sort_multiway_patterns(B, name, ways):
    for n in [(1 << 16) + 3, (1 << 20) + 1]:
        if name == "swaps_nlogn" and n > (1 << 17):
            continue
        a = bqgen.i32_pattern(name, n, seed=3)
        t = to_dev(a)
        st = B.bq_sort_ex(t, ways=ways)
        assert np.array_equal(t.cpu().numpy(), oracle.sort(a))
        assert st["fallback_segments"] == 0


@pytest.mark.parametrize("ways", [8, 16])
def test_sort_multiway_configs(B, ways):
    for name in ["c1", "c2", "c4a", "c4b"]:
        a = bqgen.config(name, 1 << 21, seed=5)
        t = to_dev(a)
        B.bq_sort_ex(t, ways=ways)
        assert np.array_equal(t.cpu().numpy(), oracle.sort(a))
    for ordering in ["random", "ascending", "descending", "swapped"]:
        a = bqgen.config("c3", 1 << 20, seed=5, ordering=ordering)
        t = to_dev(a)
        B.bq_sort_ex(t, ways=ways)
        assert np.array_equal(t.cpu().numpy().view(np.uint64), oracle.sort(a).view(np.uint64))


def test_concurrent_sorts_on_streams(B):
    """bq.h: concurrent calls on disjoint data with distinct workspaces are
    safe.  Four host threads sort four arrays (all kinds) at once, each on its
    own stream; every result is checked against the oracle."""
    import threading
    cases = [("i32", 1 << 20), ("u64", (1 << 19) + 5), ("f64", 3 << 18), ("rec32", 1 << 18)]
    arrays = [make(kind, n, seed=n, dist="random") for kind, n in cases]
    tens = [to_dev(a) for a in arrays]
    streams = [torch.cuda.Stream() for _ in cases]
    errors = []

    def work(i):
        try:
            for _ in range(3):
                t = tens[i]
                with torch.cuda.stream(streams[i]):
                    t.copy_(to_dev(arrays[i]))
                    B.bq_sort_ex(t, stream=streams[i])
        except Exception as e:   # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for (kind, _), a, t in zip(cases, arrays, tens):
        check_sorted_equal(kind, to_host(t, a), a)


def _total_order_key(bits):
    """IEEE 754 totalOrder as an unsigned key: negative values (sign bit set,
    NaNs included) reversed below the positive ones."""
    bits = bits.astype(np.uint64)
    neg = (bits >> np.uint64(63)) == 1
    return np.where(neg, ~bits, bits | np.uint64(1 << 63))


@pytest.mark.parametrize("ways", [0, 2])
def test_sort_nan_inputs_total_order(B, ways):
    """NaNs are outside the contract (include/bq.h) but must not break the
    sort: the output is a permutation of the input bit patterns, ordered by
    IEEE 754 totalOrder (quiet and signalling NaNs of both signs beyond the
    infinities), for the multi-pivot and the binary passes."""
    rng = np.random.default_rng(21)
    specials = np.array([0x7ff8000000000000, 0xfff8000000000000, 0x7ff0000000000001, 0xfff0000000000001,
                         0x7fffffffffffffff, 0x7ff0000000000000, 0xfff0000000000000, 0x8000000000000000, 0],
                        dtype=np.uint64)
    for n in [9, 5000, 300_001]:
        bits = rng.normal(size=n).view(np.uint64).copy()
        pick = rng.random(n) < 0.2
        bits[pick] = specials[rng.integers(0, len(specials), size=int(pick.sum()))]
        a = bits.view(np.float64)
        t = to_dev(a)
        st = B.bq_sort_ex(t, ways=ways)
        assert st["fallback_segments"] == 0
        got = t.cpu().numpy().view(np.uint64)
        assert np.array_equal(np.sort(got), np.sort(bits))
        k = _total_order_key(got)
        assert bool((k[1:] >= k[:-1]).all())


@pytest.mark.parametrize("frac", [1.0001, 1.1, 1.45, 1.65])
def test_leaf_aware_split(B, frac):
    """R22: an int32 segment one pass from its leaves (S < n <= 2(S - n/16))
    is split at the sample quantile that leaves about S - n/16 keys on the
    left: one binary pass still yields exactly two leaves (the quantile never
    pushes the larger child past S) and the output equals the oracle's."""
    n = int(LEAF["i32"] * frac) + 1
    a = make("i32", n, seed=n)
    t = to_dev(a)
    st = B.bq_sort_ex(t, ways=2)
    check_sorted_equal("i32", to_host(t, a), a)
    assert st["levels"] == 1 and st["leaves"] == 2 and st["fallback_segments"] == 0


def test_async_graph_sorts_and_cache(B):
    """bq_sort_* is enqueued without a host wait (a CUDA-graph level loop,
    DESIGN.md §7): sorts on a side stream, the stream synchronised only at the
    end; graphs are cached per (buffers, n, options) — a re-used buffer with new
    contents, new buffers, and more distinct configurations than cache slots
    (eviction) all sort correctly."""
    s = torch.cuda.Stream()
    arrs = [make("i32", 200_003 + 977 * k, seed=k) for k in range(40)]
    outs = []
    with torch.cuda.stream(s):
        for k, a in enumerate(arrs):
            t = to_dev(a)
            B.bq_sort_i32(t, stream=s)            # no stats: fully asynchronous
            outs.append(t)
        t0 = outs[0]
        t0.copy_(to_dev(arrs[1][: len(arrs[0])]))  # same buffer, new contents: cached graph
        B.bq_sort_i32(t0, stream=s)
    s.synchronize()
    for k in range(1, len(arrs)):
        assert np.array_equal(to_host(outs[k], arrs[k]), oracle.sort(arrs[k]))
    assert np.array_equal(to_host(outs[0], arrs[0]), oracle.sort(arrs[1][: len(arrs[0])]))


@pytest.mark.parametrize("kind", ["i32", "f64", "rec32"])
def test_host_loop_matches_graph(B, kind):
    """The host-driven level loop (timing=True: CUDA events per partition
    launch) runs the same kernels as the graph: same levels and sorted keys."""
    a = make(kind, 12 * LEAF[kind] + 5, seed=21)
    t1, t2 = to_dev(a), to_dev(a)
    s1 = B.bq_sort_ex(t1)
    s2 = B.bq_sort_ex(t2, timing=True)
    check_sorted_equal(kind, to_host(t1, a), a)
    check_sorted_equal(kind, to_host(t2, a), a)
    assert s1["levels"] == s2["levels"] and s1["element_passes"] == s2["element_passes"]
    assert s2["partition_ms"] > 0


def mo3_adversary(n, S, depth):
    """int32 keys on which the GPU's Mo3 rule with the ordered layout ([< in
    input order | = | > in reverse input order], bq.h) picks, in every level,
    the second smallest key of the segment as pivot: the samples at positions
    b, b + len/2 get the two smallest remaining values, the one at e - 1 a
    larger one, so each level peels two keys off — a median-of-3 killer
    (Introsort's motivation) for this partition."""
    val = np.full(n, -1, dtype=np.int64)
    seg = np.arange(n)
    nxt = 0
    for _ in range(depth + 1):
        L = len(seg)
        if L <= S:
            break
        val[seg[0]], val[seg[L // 2]] = nxt, nxt + 1
        nxt += 2
        keep = np.ones(L, dtype=bool)
        keep[0] = keep[L // 2] = False
        seg = seg[keep][::-1]
    rest = np.flatnonzero(val < 0)
    val[rest] = nxt + np.arange(len(rest))
    return val.astype(np.int32)


def test_depth_cap_natural_trigger(B):
    """a9 fires without a forced limit: on a Mo3 killer the recursion reaches
    the Introsort depth 2 floor(log2 n) + 3 and the capped
    segment is finished by the fallback; the output equals the oracle's."""
    n = 1 << 17
    a = mo3_adversary(n, LEAF["i32"], oracle.depth_limit(n))
    t = to_dev(a)
    st = B.bq_sort_ex(t, pivot_rule=B.BQ_PIVOT_MO3, ordered=True, ways=2)
    assert st["fallback_segments"] >= 1
    assert st["levels"] >= oracle.depth_limit(n)
    check_sorted_equal("i32", to_host(t, a), a)


@pytest.mark.parametrize("kind", ["i32", "u64", "f64"])
def test_duplicate_check_at_leaf_boundary(B, kind):
    """R23: a leaf-sized segment whose 64-key sample holds few distinct keys is
    partitioned three-way once more (its repeated keys become an equal band)
    instead of being merge-sorted: leaves of 3 distinct values; the output
    equals the oracle's and most keys were placed by the band fill."""
    S = LEAF[kind]
    n = 6 * S + 11
    base = make(kind, n, seed=31)
    vals = np.sort(base[:3]) if kind != "u64" else np.sort(base[:3])
    rng = np.random.default_rng(5)
    a = vals[rng.integers(0, 3, size=n)]
    t = to_dev(a)
    st = B.bq_sort_ex(t, ways=2)
    check_sorted_equal(kind, to_host(t, a), a)
    assert st["band_elements"] >= n // 2


@pytest.mark.parametrize("kind", ["i32", "f64", "rec32"])
@pytest.mark.parametrize("div", [16, 4])
def test_leaf_max_override(B, kind, div, monkeypatch):
    """driver.cuh's leaf_max_for: a plan with a smaller leaf bound (the
    BQ_LEAF_MAX override tools/leaf_sweep.py uses) sizes its own workspace,
    runs more levels, and sorts to the oracle's output; dups exercise the
    equal bands and the binary segments under the smaller bound."""
    lm = LEAF[kind] // div
    for dist in ("random", "dups"):
        a = make(kind, 40 * LEAF[kind] + 13, seed=17, dist=dist)
        base = B.bq_sort_ex(to_dev(a))
        monkeypatch.setenv("BQ_LEAF_MAX", str(lm))
        t = to_dev(a)
        st = B.bq_sort_ex(t)
        monkeypatch.delenv("BQ_LEAF_MAX")
        check_sorted_equal(kind, to_host(t, a), a)
        assert st["fallback_segments"] == 0
        if dist == "random":
            assert st["leaves"] > base["leaves"]


@pytest.mark.parametrize("kind", ["i32", "u64", "f64"])
def test_equal_bands_in_place_and_filled(B, kind):
    """a6: (1) an input of one repeated key is its own equal band — the pass
    finds L = G = 0 with the source in the user buffer and writes nothing
    (band_in_place); (2) a long band between smaller and larger keys (E above
    the inline limit, odd offsets, a buffer off 16-byte alignment) is written
    by k_fill's 16-byte stores with scalar head and tail; (3) few distinct
    values: single-value segments end the recursion at both buffer parities."""
    S = LEAF[kind]
    base = make(kind, 4096, seed=41)
    v = np.sort(base)[2048]
    for n in (S + 1, 5 * S + 3, (1 << 20) + 7):
        a = np.full(n, v, dtype=base.dtype)
        for off in (0, 1):
            t = to_dev(a, offset=off)
            st = B.bq_sort_ex(t, ways=2)
            check_sorted_equal(kind, to_host(t, a), a)
            assert st["band_elements"] == n and st["leaves"] == 0
    rng = np.random.default_rng(9)
    lo, hi = base[base < v][:1001], base[base > v][:777]
    for E in ((1 << 16) + 1, 300001):
        a = np.concatenate([lo, np.full(E, v, dtype=base.dtype), hi])
        rng.shuffle(a)
        for off in (0, 1):
            for ways in (2, 8):
                t = to_dev(a, offset=off)
                st = B.bq_sort_ex(t, ways=ways)
                check_sorted_equal(kind, to_host(t, a), a)
                assert st["band_elements"] >= E
    vals = np.sort(base)[::512]   # 8 distinct values
    a = vals[rng.integers(0, len(vals), size=12 * S + 5)]
    for ways in (2, 8):
        t = to_dev(a)
        st = B.bq_sort_ex(t, ways=ways)
        check_sorted_equal(kind, to_host(t, a), a)
        assert st["band_elements"] >= len(a) // 2
