"""N2: the in-place block partition, bq_partition_inplace, vs
the oracle (-m gpu).

The in-place variant places keys by block swaps (Alg. 3), so the
order inside each band is unspecified; what is unique is checked exactly —
split and n_equal against oracle.partition (bit-exact counts), the three band
predicates, the multiset, and for records that every row travels whole.  Its
workspace is O(#CTAs * T), independent of n (the paper's in-place property,
P:157-161), which is pinned too.
"""
import numpy as np
import pytest
import torch

import bqgen
import oracle
from gpu_util import to_dev, to_host
from test_gpu_parity import TILE, _pivots, edge_sizes, f64_key, keys_of, make

pytestmark = pytest.mark.gpu

KINDS = ["i32", "u64", "f64", "rec32"]


@pytest.fixture(scope="module")
def B(bq):
    assert torch.cuda.is_available()
    return bq


def _key(kind, a):
    if kind == "f64":
        return f64_key(a)
    return keys_of(a)


def _pk(kind, pv):
    if kind == "f64":
        return f64_key(np.array([pv]))[0]
    if kind == "i32":
        return np.int32(pv)
    return np.uint64(pv)


def check(B, kind, a, pv):
    t = to_dev(a)
    split, neq = B.bq_partition_inplace(t, pv)
    _, s_o, e_o = oracle.partition(a, pv)
    assert (split, neq) == (s_o, e_o)
    got = to_host(t, a)
    k, pk = _key(kind, got), _pk(kind, pv)
    assert (k[:split] < pk).all()
    assert (k[split:split + neq] == pk).all()
    assert (k[split + neq:] > pk).all()
    if kind == "rec32":
        idx = got[:, 1].astype(np.int64)
        assert np.array_equal(np.sort(idx), np.arange(len(a)))
        assert (got[:, 1] == got[:, 2]).all() and (got[:, 2] == got[:, 3]).all()
        assert np.array_equal(got[:, 0], a[idx, 0])
    elif kind == "f64":
        assert np.array_equal(np.sort(got.view(np.uint64)), np.sort(a.view(np.uint64)))
    else:
        assert np.array_equal(np.sort(got), np.sort(a))
    return split, neq


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("dist", ["random", "dups"])
def test_inplace_vs_oracle_edge_sizes(B, kind, dist):
    for n in edge_sizes(kind):
        a = make(kind, n, seed=n + 9, dist=dist)
        for p in _pivots(kind, a):
            check(B, kind, a, float(p) if kind == "f64" else int(p))


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n_tiles", [7, 150, 1185, 3001])
def test_inplace_many_blocks(B, kind, n_tiles):
    """More blocks than resident CTAs (148 x occupancy) and a ragged tail, so
    blocks are claimed repeatedly from both sides and leftovers occur."""
    n = n_tiles * TILE[kind] + 37
    for dist in ("random", "dups"):
        a = make(kind, n, seed=n_tiles, dist=dist)
        k = keys_of(a)
        p = k[len(k) // 3]
        check(B, kind, a, float(p) if kind == "f64" else int(p))


@pytest.mark.parametrize("kind", ["i32", "f64"])
@pytest.mark.parametrize("pattern", ["ascending", "descending", "all_left", "all_right", "all_equal"])
def test_inplace_skewed(B, kind, pattern):
    """One-sided inputs: all blocks neutralize from one end (the claim word
    must not run past the meeting point), sorted / reverse-sorted ranges
    (nothing / everything misplaced), and a constant range (only the equal
    band)."""
    n = 2000 * TILE[kind] + 11
    a = make(kind, n, seed=5)
    srt = np.sort(a)
    if pattern == "ascending":
        a, p = srt, srt[n // 2]
    elif pattern == "descending":
        a, p = srt[::-1].copy(), srt[n // 2]
    elif pattern == "all_left":
        p = srt[-1]
    elif pattern == "all_right":
        p = srt[0]
    else:
        a = np.full(n, srt[n // 2], dtype=a.dtype)
        p = a[0]
    check(B, kind, a, float(p) if kind == "f64" else int(p))


def test_inplace_absent_pivot_and_extremes(B):
    n = 1500 * TILE["u64"] + 5
    a = make("u64", n, seed=3)
    for pv in [0, (1 << 64) - 1, int(np.sort(a)[n // 2]) + 1]:
        check(B, "u64", a, pv)


def test_inplace_workspace_is_independent_of_n(B):
    """The paper's in-place property: the workspace does not grow with n
    (bounded by #CTAs blocks plus the cleanup's small buffers)."""
    w1 = B.bq_inplace_workspace_bytes(B.BQ_I32, 1 << 24)
    w2 = B.bq_inplace_workspace_bytes(B.BQ_I32, 1 << 30)
    assert w1 == w2
    assert w2 < (1 << 24) * 4
    assert B.bq_inplace_workspace_bytes(B.BQ_I32, 100) < w1


def test_inplace_c2_full(B):
    """BASELINE config 2 at full size, in place, around the oracle's Mo3 pivot."""
    a = bqgen.config("c2", seed=1)
    t = to_dev(a)
    p = B.bq_pivot_i32(t, B.BQ_PIVOT_MO3)
    split, neq = B.bq_partition_inplace(t, p)
    assert split == int(np.count_nonzero(a < p)) and neq == int(np.count_nonzero(a == p))
    assert bool((t[:split] < p).all()) and bool((t[split:split + neq] == p).all())
    assert bool((t[split + neq:] > p).all())
    got = t.cpu().numpy()
    assert np.array_equal(np.sort(got), np.sort(a))


def test_inplace_invalid_arguments(B):
    t = torch.zeros(10, dtype=torch.float64, device="cuda")
    with pytest.raises(Exception):
        B.bq_partition_inplace(t, float("nan"))
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(Exception):
        B.bq_partition_inplace(torch.zeros(1 << 16, dtype=torch.int32, device="cuda"), 0, ws=small)


@pytest.mark.parametrize("kind,offset", [("i32", 1), ("i32", 2), ("i32", 3), ("u64", 1), ("f64", 1)])
def test_inplace_unaligned_start(B, kind, offset):
    """A range that does not start on 16 bytes: the head before the first
    aligned block goes to the cleanup (with every lv < head / lv >= head case
    of the final fix-up: pivots at the minimum, inside, and above)."""
    for n in [2, offset + 1, 5 * TILE[kind] + 3, 301 * TILE[kind] + 9]:
        a = make(kind, n, seed=n + offset, dist="dups")
        srt = np.sort(keys_of(a))
        for p in [srt[0], srt[len(srt) // 2], srt[-1]]:
            pv = float(p) if kind == "f64" else int(p)
            t = to_dev(a, offset=offset)
            split, neq = B.bq_partition_inplace(t, pv)
            _, s_o, e_o = oracle.partition(a, pv)
            assert (split, neq) == (s_o, e_o)
            got = to_host(t, a)
            k, pk = _key(kind, got), _pk(kind, pv)
            assert (k[:split] < pk).all() and (k[split:split + neq] == pk).all() and (k[split + neq:] > pk).all()
            assert np.array_equal(np.sort(_key(kind, got)), np.sort(_key(kind, a)))


@pytest.mark.parametrize("kind,n", [("i32", 1 << 25), ("u64", 1 << 24), ("f64", 1 << 24), ("rec32", 1 << 22)])
@pytest.mark.parametrize("nvals", [4, 64])
def test_inplace_equal_band_both_ways(B, kind, n, nvals):
    """The equal band is formed by compaction when it fits the cleanup
    lists, otherwise by a second block pass (mode 1: left <=> key <= p):
    4 distinct keys puts n/4 keys in the band (> the list capacity, second
    pass), 64 puts n/64 (compaction)."""
    a = make(kind, n, seed=nvals)
    if kind == "rec32":
        a[:, 0] = a[:, 0] % np.uint64(nvals)
    elif kind == "f64":
        a = np.floor(a * nvals / 2) / nvals
    else:
        a = (a % nvals).astype(a.dtype)
    k = keys_of(a)
    p = np.sort(k)[len(k) // 2]
    split, neq = check(B, kind, a, float(p) if kind == "f64" else int(p))
    assert neq > n // (2 * nvals)


@pytest.mark.parametrize("kind", ["i32", "u64", "rec32"])
def test_inplace_equal_band_geometries(B, kind):
    """The equal band from pass 0's recorded positions (no scan of the right
    part) across many geometries: random sizes (ragged tails), unaligned
    starts (heads), pivots anywhere (the head and tail fix-ups, leftover blocks
    moved out of the right window with their recorded keys), and a few to a
    few thousand keys equal to the pivot."""
    rng = np.random.default_rng(17)
    T = TILE[kind]
    for case in range(24):
        n = int(rng.integers(T, 600 * T)) + int(rng.integers(0, T))
        offset = int(rng.integers(0, 4)) if kind != "rec32" else 0
        a = make(kind, n, seed=case + 100)
        k = keys_of(a)
        # plant copies of one key (1 .. ~n/64 of them) at random positions
        p = k[int(rng.integers(0, n))]
        m = int(rng.integers(1, max(2, n // 64)))
        pos = rng.integers(0, n, size=m)
        if kind == "rec32":
            a[pos, 0] = p
        else:
            a[pos] = p
        pv = int(p)
        t = to_dev(a, offset=offset)
        split, neq = B.bq_partition_inplace(t, pv)
        _, s_o, e_o = oracle.partition(a, pv)
        assert (split, neq) == (s_o, e_o), case
        got = to_host(t, a)
        kk, pk = _key(kind, got), _pk(kind, pv)
        assert (kk[:split] < pk).all() and (kk[split:split + neq] == pk).all() and (kk[split + neq:] > pk).all()
        assert np.array_equal(np.sort(_key(kind, got)), np.sort(_key(kind, a)))
