"""N1, second half: the subtree pass (-m gpu).

With bq_sort_options.subtree, segments of S < len <= SUB elements (SUB = 96 KB
of elements) are finished depth-first by one CTA in shared memory; their
pieces of <= S go to the leaf sorts.  Bars: the sorted output is bit-exact
against the oracle for every kind, at sizes around S and SUB (the root itself
may be a subtree), on duplicate-heavy and patterned inputs, with the depth cap
reached inside a subtree, and with the ordered placement.
"""
import numpy as np
import pytest
import torch

import bqgen
import oracle
from gpu_util import to_dev, to_host
from test_gpu_parity import LEAF, check_sorted_equal, make

pytestmark = pytest.mark.gpu

SUB = {"i32": 24576, "u64": 12288, "f64": 12288, "rec32": 3072}


@pytest.fixture(scope="module")
def B(bq):
    assert torch.cuda.is_available()
    return bq


def sizes(kind):
    S, U = LEAF[kind], SUB[kind]
    return sorted({S + 1, S + 17, (S + U) // 2, U - 1, U, U + 1, 2 * U + 3, 7 * U + 11, (1 << 20) + 5})


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
@pytest.mark.parametrize("dist", ["random", "dups"])
def test_subtree_sort_vs_oracle(B, kind, dist):
    for n in sizes(kind):
        a = make(kind, n, seed=n + 3, dist=dist)
        t = to_dev(a)
        st = B.bq_sort_ex(t, subtree=True)
        check_sorted_equal(kind, to_host(t, a), a)
        assert st["fallback_segments"] == 0


@pytest.mark.parametrize("kind", ["i32", "f64"])
@pytest.mark.parametrize("pattern", ["sorted", "reversed", "rotation", "imodsqrt", "halfhalf", "zeroone"])
def test_subtree_patterns(B, kind, pattern):
    n = (1 << 21) + 7
    a = bqgen.i32_pattern(pattern, n, 9)
    if kind == "f64":
        a = a.astype(np.float64) * 0.5
    t = to_dev(a)
    B.bq_sort_ex(t, subtree=True)
    check_sorted_equal(kind, to_host(t, a), a)


def test_subtree_depth_cap_inside(B):
    """A small depth limit makes segments around the subtree size hit the cap
    (at the level passes or inside a subtree, depending on the pivots the
    atomic placement leads to): they go to the fallback sort, and the output
    is still exact."""
    n = 200_000
    a = make("i32", n, seed=12)
    t = to_dev(a)
    st = B.bq_sort_ex(t, subtree=True, depth_limit=4, ways=2)
    check_sorted_equal("i32", to_host(t, a), a)
    assert st["fallback_segments"] > 0


def test_subtree_ordered_is_deterministic(B):
    a = make("rec32", (1 << 18) + 3, seed=5, dist="dups")
    outs = []
    for _ in range(2):
        t = to_dev(a)
        B.bq_sort_ex(t, subtree=True, ordered=True, records=B.RECORDS_DIRECT)
        outs.append(to_host(t, a))
    assert np.array_equal(outs[0], outs[1])
    check_sorted_equal("rec32", outs[0], a)


def test_subtree_c2_full(B):
    """BASELINE config 2 at full size through the subtree pass."""
    a = bqgen.config("c2", seed=1)
    t = to_dev(a)
    st = B.bq_sort_ex(t, subtree=True)
    got = to_host(t, a)
    del t
    torch.cuda.empty_cache()
    assert np.array_equal(got, oracle.sort(a))
    assert st["fallback_segments"] == 0
