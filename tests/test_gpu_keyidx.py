"""N3: the key+index record variant (-m gpu).

bq_keyidx16 pairs are sorted by key (only the key is compared);
the records sort's default path sorts (key, position) pairs and gathers every
record once.  Bars: keys bit-exact against the oracle's sort of the same keys;
every pair / record travels whole (its index or payload still belongs to its
key); the payload permutation is a permutation.
"""
import numpy as np
import pytest
import torch

import bqgen
import oracle
from gpu_util import to_dev, to_host
from test_gpu_parity import check_sorted_equal, make

pytestmark = pytest.mark.gpu

import paper_1604_06697_b200 as _bq

T_PAIR, S_PAIR = _bq.tile_elems(_bq.BQ_KEYIDX16), _bq.leaf_elems(_bq.BQ_KEYIDX16)


@pytest.fixture(scope="module")
def B(bq):
    assert torch.cuda.is_available()
    return bq


def pairs_from(keys):
    n = len(keys)
    a = np.empty((n, 2), dtype=np.uint64)
    a[:, 0] = keys
    a[:, 1] = np.arange(n, dtype=np.uint64) * np.uint64(7) + np.uint64(3)
    return a


def check_pairs(a, got):
    exp_keys = oracle.sort(a[:, 0].copy())
    assert np.array_equal(got[:, 0], exp_keys)
    pos = (got[:, 1] - np.uint64(3)) // np.uint64(7)
    assert np.array_equal(np.sort(pos), np.arange(len(a), dtype=np.uint64))
    assert np.array_equal(a[pos.astype(np.int64), 0], got[:, 0])


def edge_sizes():
    return sorted({0, 1, 2, 31, 33, T_PAIR - 1, T_PAIR + 1, S_PAIR - 1, S_PAIR, S_PAIR + 1,
                   3 * S_PAIR + 7, (1 << 16) + 3, (1 << 20) + 11})


@pytest.mark.parametrize("ways", [0, 2, 16])
@pytest.mark.parametrize("dist", ["random", "dups", "sorted", "reversed"])
def test_sort_keyidx16(B, dist, ways):
    """Pairs sort by the multi-pivot passes by default (8-way, N4), by binary
    two-way passes with ways = 2, 16-way with ways = 16."""
    for n in edge_sizes():
        k = bqgen.u64(n, n + 1)
        if dist == "dups":
            k = k % np.uint64(13)
        elif dist == "sorted":
            k = np.sort(k)
        elif dist == "reversed":
            k = np.sort(k)[::-1].copy()
        a = pairs_from(k)
        t = to_dev(a)
        st = B.bq_sort_ex(t, ways=ways)
        assert st["fallback_segments"] == 0
        check_pairs(a, to_host(t, a))


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("dist", ["random", "dups"])
def test_records_both_paths(B, path, dist):
    """bq_sort_options.records: 1 moves the records every pass, 2 (and the
    default 0) sorts key+index pairs and gathers once; sizes around the
    key+index threshold (2 x the records leaf size) and beyond."""
    for n in [0, 1, 4095, 4096, 4097, 3 * 4096 + 5, (1 << 18) + 9, (1 << 21) + 1]:
        a = make("rec32", n, seed=n + path, dist=dist)
        t = to_dev(a)
        st = B.bq_sort_ex(t, records=path)
        assert st["fallback_segments"] == 0
        check_sorted_equal("rec32", to_host(t, a), a)


def test_records_default_is_keyidx(B):
    """The default records path reports the pair sort's statistics: 16-byte
    elements moved per pass."""
    n = 1 << 20
    a = make("rec32", n, seed=4)
    t = to_dev(a)
    st = B.bq_sort_ex(t, timing=True)
    check_sorted_equal("rec32", to_host(t, a), a)
    # partition_bytes covers the binary passes; multiway levels are counted apart
    binary = st["element_passes"] - st["multiway_element_passes"]
    assert st["partition_bytes"] == pytest.approx(2 * 16 * binary)
    assert st["multiway_element_passes"] > 0 and st["multiway_ms"] > 0
    t2 = to_dev(a)
    st2 = B.bq_sort_ex(t2, timing=True, records=B.RECORDS_DIRECT)
    assert st2["partition_bytes"] == pytest.approx(2 * 32 * st2["element_passes"])
    assert np.array_equal(to_host(t2, a)[:, 0], to_host(t, a)[:, 0])


def test_records_workspace_covers_keyidx(B):
    n = 1 << 20
    need = B.bq_workspace_bytes(B.BQ_REC32, n)
    # 16n pairs + the pair sort's layout (16n scratch + O(n/T)) + the 32n copy (bq.h)
    assert need >= 16 * n + 16 * n + 32 * n
    a = make("rec32", n, seed=8)
    t = to_dev(a)
    small = torch.empty(need - 256, dtype=torch.uint8, device="cuda")
    with pytest.raises(Exception):
        B.bq_sort_ex(t, ws=small)


def test_keyidx16_partition_and_inplace(B):
    n = 300 * T_PAIR + 17
    k = bqgen.u64(n, 5) % np.uint64(1000)
    a = pairs_from(k)
    p = int(np.sort(k)[n // 2])
    src = to_dev(a)
    dst = torch.empty_like(src)
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    B.bq_partition_pass(src, dst, p, counts)
    lt, eq = int((k < p).sum()), int((k == p).sum())
    assert counts.cpu().tolist() == [lt, eq, n - lt - eq]
    got = to_host(dst, a)
    assert (got[:lt, 0] < p).all() and (got[lt:lt + eq, 0] == p).all() and (got[lt + eq:, 0] > p).all()
    t = to_dev(a)
    split, neq = B.bq_partition_inplace(t, p)
    assert (split, neq) == (lt, eq)
    g2 = to_host(t, a)
    assert (g2[:lt, 0] < p).all() and (g2[lt:lt + eq, 0] == p).all() and (g2[lt + eq:, 0] > p).all()
    assert np.array_equal(np.sort(g2[:, 1]), np.sort(a[:, 1]))
