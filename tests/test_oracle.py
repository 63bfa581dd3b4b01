"""Pins for oracle/ (CPU, -m "not gpu").

The oracle is checked against things other than itself: worked examples the
paper/SPEC print (tests/golden/), brute force over all small inputs against
the plain definitions (sortedness, the partition predicate of P:262-266,
split = #less), library routines (numpy's sort, libstdc++ std::sort), closed
forms of the config inputs, and invariants the paper states (comparison
count of the simple block partition, stack bound, depth limit).
"""
import itertools
import json
import math
import os
import struct

import numpy as np
import pytest

import bqgen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------- golden ----

def test_golden_median_of_3():
    for ex in _golden()["median_of_3"]:
        a = np.array(ex["input"], dtype=np.int32)
        assert oracle.pivot(a, oracle.MO3) == ex["pivot_value"], ex["cite"]


def test_golden_block_partition():
    for ex in _golden()["block_partition"]:
        if "input" in ex:
            a = np.array(ex["input"], dtype=np.int32)
        else:
            a = np.full(ex["input_fill"]["n"], ex["input_fill"]["value"], dtype=np.int32)
        out, cut, cmp = oracle.block_partition(a, ex["pivot_index"], ex["block"])
        assert cut == ex["cut"], ex["cite"]
        assert cmp == ex["comparisons"], ex["cite"]


def test_golden_sort():
    for ex in _golden()["sort"]:
        a = np.array(ex["input"], dtype=np.int32)
        assert oracle.sort(a).tolist() == ex["output"], ex["cite"]


def test_golden_depth_limit():
    for ex in _golden()["depth_limit"]:
        assert oracle.depth_limit(ex["n"]) == ex["limit"], ex["cite"]


def _f64_table():
    vals = []
    with open(os.path.join(GOLDEN, "f64_total_order.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            vals.append(int(line.split()[0], 16))
    return np.array(vals, dtype=np.uint64).view(np.float64)


def test_golden_f64_total_order():
    table = _f64_table()
    rng = np.random.default_rng(5)
    for _ in range(50):
        perm = rng.permutation(len(table))
        # repeat values too, so equal keys (incl. both zeros) are exercised
        a = np.concatenate([table[perm], table[perm[: len(table) // 2]]])
        out = oracle.sort(a, cutoff=3)
        exp = np.sort(np.concatenate([np.arange(len(table)), perm[: len(table) // 2]]))
        assert out.view(np.uint64).tolist() == table[exp].view(np.uint64).tolist()


# ---------------------------------------------------- brute force, tiny n ----

def _check_partition_predicate(inp, out, cut, pivot):
    assert out[cut] == pivot
    assert all(x <= pivot for x in out[:cut])
    assert all(x >= pivot for x in out[cut + 1:])
    assert sorted(out.tolist()) == sorted(inp.tolist())


@pytest.mark.parametrize("block", [1, 2, 4, 128])
def test_block_partition_all_permutations(block):
    # P:262-266 partition predicate, S:76/S:117 exactly len-1 comparisons
    for n in range(1, 8):
        for perm in itertools.permutations(range(n)):
            inp = np.array(perm, dtype=np.int32)
            for pi in range(n):
                out, cut, cmp = oracle.block_partition(inp, pi, block)
                _check_partition_predicate(inp, out, cut, inp[pi])
                assert cut == inp[pi]            # distinct keys: cut = rank(p)
                assert cmp == n - 1


@pytest.mark.parametrize("block", [1, 2, 128])
def test_block_partition_duplicate_words(block):
    for n in range(1, 8):
        for w in itertools.product(range(3), repeat=n):
            inp = np.array(w, dtype=np.int32)
            for pi in range(n):
                out, cut, cmp = oracle.block_partition(inp, pi, block)
                _check_partition_predicate(inp, out, cut, inp[pi])
                assert cmp == n - 1


@pytest.mark.parametrize("block", [1, 2, 128])
def test_value_partition_words(block):
    # O-partition: split = #{k < p}, n_equal = #{k == p}, three bands, multiset
    for n in range(0, 7):
        for w in itertools.product(range(4), repeat=n):
            inp = np.array(w, dtype=np.int32)
            for p in range(-1, 5):
                out, s, e = oracle.partition(inp, p, block)
                assert s == sum(1 for x in w if x < p)
                assert e == sum(1 for x in w if x == p)
                assert all(x < p for x in out[:s])
                assert all(x == p for x in out[s:s + e])
                assert all(x > p for x in out[s + e:])
                assert sorted(out.tolist()) == sorted(w)


@pytest.mark.parametrize("block", [1, 2, 128])
def test_sort_all_permutations(block):
    # cutoff 3 so the partition path runs on tiny inputs (SURVEY §8(c) amb. 16)
    for n in range(0, 8):
        ident = list(range(n))
        for perm in itertools.permutations(range(n)):
            out = oracle.sort(np.array(perm, dtype=np.int32), block=block, cutoff=3)
            assert out.tolist() == ident


@pytest.mark.parametrize("block", [1, 2, 128])
def test_sort_duplicate_words(block):
    for n in range(0, 8):
        for w in itertools.product(range(3), repeat=n):
            out = oracle.sort(np.array(w, dtype=np.int32), block=block, cutoff=3)
            assert out.tolist() == sorted(w)


def test_sort_all_permutations_n8():
    for perm in itertools.permutations(range(8)):
        out = oracle.sort(np.array(perm, dtype=np.int32), block=2, cutoff=3)
        assert out.tolist() == list(range(8))


# --------------------------------------------- library routines, larger n ----

SIZES = [17, 100, 255, 256, 257, 1000, 4097, 65536 + 3, 300000]


@pytest.mark.parametrize("n", SIZES)
def test_sort_i32_vs_numpy(n):
    a = bqgen.i32_full(n, seed=n)
    out = oracle.sort(a)
    assert np.array_equal(out, np.sort(a, kind="stable"))
    assert np.array_equal(out, oracle.std_sort(a))


@pytest.mark.parametrize("n", SIZES)
def test_sort_u64_vs_numpy(n):
    a = bqgen.u64(n, seed=n)
    assert (a >= np.uint64(1 << 63)).any() or n < 100   # unsigned-compare trap
    out = oracle.sort(a)
    assert np.array_equal(out, np.sort(a))


@pytest.mark.parametrize("n", SIZES)
def test_sort_f64_vs_numpy(n):
    a = bqgen.f64(n, seed=n) * 2.0 - 1.0     # negatives included, no -0.0
    a[::7] = np.round(a[::7], 2)             # and some duplicates
    a[a == 0] = 0.0                          # rounding can make -0.0
    assert not np.signbit(a[a == 0]).any()
    out = oracle.sort(a)
    assert np.array_equal(out.view(np.uint64), np.sort(a).view(np.uint64))


def test_sort_f64_signed_zeros():
    a = np.array([0.0, -0.0] * 40 + [1.0, -1.0] * 10, dtype=np.float64)
    out = oracle.sort(a)
    bits = out.view(np.uint64)
    # totalOrder: all -1.0, then all -0.0, then all +0.0, then 1.0
    exp = np.concatenate([np.full(10, -1.0), np.full(40, -0.0), np.full(40, 0.0), np.full(10, 1.0)])
    assert bits.tolist() == exp.view(np.uint64).tolist()


@pytest.mark.parametrize("n,dup", [(1000, None), (65539, None), (20000, 50), (5000, 1)])
def test_sort_rec32(n, dup):
    a = bqgen.rec32(n, seed=3, dup_keys=dup)
    out = oracle.sort(a)
    assert np.array_equal(out[:, 0], np.sort(a[:, 0]))
    idx = out[:, 1].astype(np.int64)
    assert np.array_equal(np.sort(idx), np.arange(n))            # a permutation
    assert (out[:, 1] == out[:, 2]).all() and (out[:, 2] == out[:, 3]).all()
    assert np.array_equal(out[:, 0], a[idx, 0])                  # payload matches key


@pytest.mark.parametrize("kind", ["i32", "u64", "f64", "rec32"])
def test_value_partition_random(kind):
    n = 50000
    if kind == "i32":
        a = bqgen.i32_range(n, 300, seed=2)
        keys, p = a, 150
    elif kind == "u64":
        a = bqgen.u64(n, seed=2) >> np.uint64(55)
        keys, p = a, int(a[17])
    elif kind == "f64":
        a = np.round(bqgen.f64(n, seed=2), 3)
        keys, p = a, float(a[5])
    else:
        a = bqgen.rec32(n, seed=2, dup_keys=200)
        keys, p = a[:, 0], int(a[9, 0])
    out, s, e = oracle.partition(a, p)
    ok = out[:, 0] if kind == "rec32" else out
    pv = np.array(p, dtype=keys.dtype)
    assert s == int((keys < pv).sum()) and e == int((keys == pv).sum())
    assert (ok[:s] < pv).all() and (ok[s:s + e] == pv).all() and (ok[s + e:] > pv).all()
    if kind == "rec32":
        assert np.array_equal(np.sort(out[:, 1]), np.arange(n, dtype=np.uint64))
    else:
        assert np.array_equal(np.sort(out), np.sort(a))


# ------------------------------------------------ pivot sample rules --------

def test_pivot_rules_vs_median():
    rng = np.random.default_rng(1)
    for n in [3, 4, 8, 9, 10, 100, 12345]:
        for _ in range(20):
            a = rng.integers(-50, 50, size=n).astype(np.int32)
            samp = [a[0], a[n // 2], a[n - 1]]
            assert oracle.pivot(a, oracle.MO3) == int(np.median(samp))
            if n >= 9:
                pos = [(k * (n - 1)) // 8 for k in range(9)]
                meds = [int(np.median([a[pos[3 * g + j]] for j in range(3)])) for g in range(3)]
                assert oracle.pivot(a, oracle.NINTHER) == int(np.median(meds))


def test_pivot_sample64_closed_forms():
    # R18/R19: the lower median of 64 keys, key j drawn from the j-th of 64
    # equal strata.  On an ascending array the sample is ascending, so the
    # pivot lies in stratum 31; on a descending one the 32nd smallest sampled
    # key comes from stratum 32.
    for n in [64, 65, 1000, 12345, 1 << 20]:
        asc = np.arange(n, dtype=np.int32) * 3 - 7
        p = oracle.pivot(asc, oracle.SAMPLE64)
        assert asc[(31 * n) >> 6] <= p <= asc[((32 * n) >> 6) - 1]
        desc = asc[::-1].copy()
        q = oracle.pivot(desc, oracle.SAMPLE64)
        assert desc[((33 * n) >> 6) - 1] <= q <= desc[(32 * n) >> 6]
    for n in [1, 2, 5, 63]:     # short segments: strata of length 0 or 1
        a = np.arange(n, dtype=np.int32)
        assert 0 <= oracle.pivot(a, oracle.SAMPLE64) < n
    # all keys equal: the pivot is that key; u64 keys above 2^63 compare unsigned
    assert oracle.pivot(np.full(500, 9, dtype=np.int32), oracle.SAMPLE64) == 9
    u = np.arange(6400, dtype=np.uint64) + np.uint64(1 << 63)
    assert u[3100] <= oracle.pivot(u, oracle.SAMPLE64) <= u[3199]
    # the jitter defeats periodic inputs: on i mod 100 with n = 64 * 100 an
    # equidistant sample would see one value 64 times
    per = (np.arange(6400) % 100).astype(np.int32)
    assert 30 <= oracle.pivot(per, oracle.SAMPLE64) <= 70


# ------------------------------------------ closed forms of config inputs ----

def test_closed_form_c1():
    a = bqgen.config("c1", 1 << 16, seed=4)
    assert np.array_equal(oracle.sort(a), np.arange(1 << 16, dtype=np.int32))
    p = oracle.pivot(a, oracle.MO3)
    out, s, e = oracle.partition(a, p)
    assert s == p and e == 1          # a permutation of 0..n-1: split == p


def test_closed_form_c3_orderings():
    n = 1 << 15
    asc = bqgen.f64(n, 3, "ascending")
    assert (np.diff(asc) > 0).all()
    assert np.array_equal(oracle.sort(asc), asc)
    assert np.array_equal(oracle.sort(bqgen.f64(n, 3, "descending")), asc)
    assert np.array_equal(oracle.sort(bqgen.f64(n, 3, "swapped")), asc)


def test_closed_form_c4():
    n = 1 << 16
    a = bqgen.config("c4a", n, seed=2)
    m = math.isqrt(n)
    hist = np.bincount(a, minlength=m)
    exp = np.repeat(np.arange(m, dtype=np.int32), hist)
    assert np.array_equal(oracle.sort(a), exp)
    b = bqgen.config("c4b", n)
    assert np.array_equal(oracle.sort(b), b)
    out, s, e = oracle.partition(b, bqgen.CONST_KEY)
    assert (s, e) == (0, n)


# ---------------------------------------- paper invariants / faithfulness ----

def test_comparison_constant_band():
    g = _golden()["comparison_constant"]
    n = g["n"]
    a = bqgen.i32_perm(n, seed=1)
    out, st = oracle.sort(a, stats=True)
    c = st["comparisons"] / (n * math.log2(n))
    assert g["lo"] <= c <= g["hi"], (c, g["cite"])


@pytest.mark.parametrize("shape", ["perm", "asc", "desc", "swapped", "fewdistinct", "const"])
def test_stack_bound_and_no_heapsort(shape):
    # S:119 stack <= ceil(log2 n)+1; no Introsort fallback on config shapes
    n = 1 << 16
    a = {"perm": lambda: bqgen.i32_perm(n, 7),
         "asc": lambda: bqgen.f64(n, 7, "ascending"),
         "desc": lambda: bqgen.f64(n, 7, "descending"),
         "swapped": lambda: bqgen.f64(n, 7, "swapped"),
         "fewdistinct": lambda: bqgen.config("c4a", n, 7),
         "const": lambda: bqgen.i32_const(n)}[shape]()
    out, st = oracle.sort(a, stats=True)
    assert st["max_stack"] <= math.ceil(math.log2(n)) + 1
    assert st["heapsort_calls"] == 0
    assert np.array_equal(out, np.sort(a))


def test_heapsort_fallback_path():
    # depth limit 0 sends every sub-array > cutoff to Heapsort
    a = bqgen.i32_full(5000, seed=9)
    out, st = oracle.sort(a, depth_limit=0, stats=True)
    assert st["heapsort_calls"] == 1 and st["partitions"] == 0
    assert np.array_equal(out, np.sort(a))
    out, st = oracle.sort(a, depth_limit=3, stats=True)
    assert st["heapsort_calls"] >= 1
    assert np.array_equal(out, np.sort(a))


def test_helpers_sort():
    for f in (oracle.heapsort, oracle.insertion_sort):
        for n in [0, 1, 2, 3, 16, 17, 500]:
            a = bqgen.i32_full(n, seed=n + 1)
            assert np.array_equal(f(a), np.sort(a))


# ------------------------------------------- the paper's structured inputs ----

@pytest.mark.parametrize("name", ["imodsqrt", "square", "pow8", "sorted", "reversed", "rotation",
                                  "swaps_sqrt", "swaps_n", "swaps_nlogn", "halfhalf", "zeroone"])
def test_sort_patterns(name):
    for n in [17, 1 << 12, (1 << 16) + 3]:
        a = bqgen.i32_pattern(name, n, seed=2)
        out, st = oracle.sort(a, stats=True)
        assert np.array_equal(out, np.sort(a))
        assert st["max_stack"] <= int(np.ceil(np.log2(n))) + 1


def test_oracle_splitmix64_known_answer():
    """The oracle's own SplitMix64 output function (SAMPLE64's sample
    positions, R19): the published first output of SplitMix64 from state 0
    (Vigna, splitmix64.c: 0xE220A8397B1DCDAF), mix(0) = 0, and agreement with
    the independent copy in bqgen (whose stream is mix(mix(seed) + (i+1)*gamma))."""
    import bqgen
    g, m64 = 0x9E3779B97F4A7C15, (1 << 64) - 1
    assert oracle.splitmix64_mix(g) == 0xE220A8397B1DCDAF
    assert oracle.splitmix64_mix(0) == 0
    for seed in (0, 1, 7, 12345):
        s = oracle.splitmix64_mix(seed)
        for i in range(4):
            assert bqgen.u64_at(seed, i) == oracle.splitmix64_mix((s + (i + 1) * g) & m64)
