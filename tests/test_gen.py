"""bqgen: the shared seeded input generators (CPU)."""
import math

import numpy as np

import bqgen

M64 = (1 << 64) - 1


def _splitmix_mix(z):
    # SplitMix64 finaliser (Steele, Lea & Flood 2014) for a known-answer check
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_splitmix_known_answer():
    # Vigna's splitmix64.c with state x: next() = mix(x += gamma).  Our stream
    # seeds the state with mix(seed); check the counter form matches.
    for seed in [0, 1, 12345]:
        x = _splitmix_mix(seed)
        for i in range(5):
            x = (x + 0x9E3779B97F4A7C15) & M64
            assert bqgen.u64_at(seed, i) == _splitmix_mix(x)
    assert bqgen.u64(3, seed=1).tolist() == [bqgen.u64_at(1, i) for i in range(3)]
    # published first output of SplitMix64 from state 0 (Vigna): 0xE220A8397B1DCDAF
    assert _splitmix_mix(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF


def test_deterministic_and_seeded():
    assert np.array_equal(bqgen.i32_full(1000, 3), bqgen.i32_full(1000, 3))
    assert not np.array_equal(bqgen.i32_full(1000, 3), bqgen.i32_full(1000, 4))


def test_perm_is_permutation():
    for n in [0, 1, 2, 1000, 1 << 16]:
        a = bqgen.i32_perm(n, 2)
        assert np.array_equal(np.sort(a), np.arange(n, dtype=np.int32))
    assert not np.array_equal(bqgen.i32_perm(1000, 2), np.arange(1000))


def test_full_range_signed():
    a = bqgen.i32_full(1 << 16, 1)
    assert (a < 0).any() and (a > 0).any()


def test_range_and_const():
    n = 1 << 16
    a = bqgen.config("c4a", n)
    assert a.min() >= 0 and a.max() < math.isqrt(n)
    assert len(np.unique(a)) == math.isqrt(n)
    assert (bqgen.config("c4b", 100) == bqgen.CONST_KEY).all()


def test_f64_orderings():
    n = 1 << 14
    r = bqgen.f64(n, 1)
    assert (r >= 0).all() and (r < 1).all() and not np.signbit(r).any()
    asc = bqgen.f64(n, 1, "ascending")
    assert (np.diff(asc) > 0).all() and asc[0] >= 0 and asc[-1] < 1
    assert np.array_equal(bqgen.f64(n, 1, "descending"), asc[::-1])
    sw = bqgen.f64(1 << 20, 1, "swapped")
    asc2 = bqgen.f64(1 << 20, 1, "ascending")
    frac = (sw != asc2).mean()
    assert 0.008 < frac < 0.0101        # ~1% displaced (2*n/200 minus collisions)


def test_rec32_payload():
    a = bqgen.rec32(1000, 5)
    assert (a[:, 1] == np.arange(1000)).all()
    assert (a[:, 1] == a[:, 2]).all() and (a[:, 2] == a[:, 3]).all()
    d = bqgen.rec32(1000, 5, dup_keys=10)
    assert d[:, 0].max() < 10
