"""Seeded synthetic inputs shaped like BASELINE.json's five configs.

A module of its own (see bqgen.c): it holds none of the sorting method's
arithmetic and imports neither ``oracle`` nor the CUDA package.  Generation is
done in C (``libbqgen.so``, built by ``__graft_entry__.build()`` or lazily by
``tools.build``) because config 2 asks for 2^28 keys.

Config recipes:

=====  ==========================================================  =========
cfg    input                                                       paper
=====  ==========================================================  =========
c1     int32 Fisher-Yates permutation of 0..n-1, n=2^20             Fig. 5
c2     int32 i.i.d. uniform over the full int32 range, n=2^28       Fig. 5
c3     float64 uniform [0,1), n=2^27: random/asc/desc/1%-swapped   Figs. 9-10
c4a    int32 uniform over {0..floor(sqrt n)-1}, n=2^28              Fig. 6
c4b    int32 all equal (0x2A2A2A2A), n=2^28                         Fig. 11
c5     32 B records {u64 key, payload i,i,i}, n=2^26               Fig. 8
=====  ==========================================================  =========
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libbqgen.so")
_lib = None

CONST_KEY = 0x2A2A2A2A


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            from tools import build as _b
            _b.build_gen()
        lib = ctypes.CDLL(_LIB_PATH)
        u64, sz, vp = ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p
        lib.bqgen_u64_at.restype = u64
        lib.bqgen_u64_at.argtypes = [u64, u64]
        for name, args in {
            "bqgen_u64": [u64, sz, vp],
            "bqgen_i32_full": [u64, sz, vp],
            "bqgen_i32_range": [u64, sz, ctypes.c_uint32, vp],
            "bqgen_i32_const": [sz, ctypes.c_int32, vp],
            "bqgen_i32_perm": [u64, sz, vp],
            "bqgen_f64_unit": [u64, sz, vp],
            "bqgen_f64_ascending": [u64, sz, vp],
            "bqgen_f64_descending": [u64, sz, vp],
            "bqgen_f64_swapped": [u64, sz, vp],
            "bqgen_rec32": [u64, sz, vp],
            "bqgen_rec32_dupkeys": [u64, sz, u64, vp],
        }.items():
            f = getattr(lib, name)
            f.restype = None
            f.argtypes = args
        lib.bqgen_i32_pattern.restype = ctypes.c_int
        lib.bqgen_i32_pattern.argtypes = [ctypes.c_int, u64, sz, vp]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def u64_at(seed: int, i: int) -> int:
    return int(_load().bqgen_u64_at(seed, i))


def u64(n: int, seed: int = 1) -> np.ndarray:
    a = np.empty(n, dtype=np.uint64)
    _load().bqgen_u64(seed, n, _ptr(a))
    return a


def i32_full(n: int, seed: int = 1) -> np.ndarray:
    a = np.empty(n, dtype=np.int32)
    _load().bqgen_i32_full(seed, n, _ptr(a))
    return a


def i32_range(n: int, m: int, seed: int = 1) -> np.ndarray:
    a = np.empty(n, dtype=np.int32)
    _load().bqgen_i32_range(seed, n, m, _ptr(a))
    return a


def i32_const(n: int, value: int = CONST_KEY) -> np.ndarray:
    a = np.empty(n, dtype=np.int32)
    _load().bqgen_i32_const(n, value, _ptr(a))
    return a


def i32_perm(n: int, seed: int = 1) -> np.ndarray:
    a = np.empty(n, dtype=np.int32)
    _load().bqgen_i32_perm(seed, n, _ptr(a))
    return a


def f64(n: int, seed: int = 1, ordering: str = "random") -> np.ndarray:
    a = np.empty(n, dtype=np.float64)
    fn = {
        "random": _load().bqgen_f64_unit,
        "ascending": _load().bqgen_f64_ascending,
        "descending": _load().bqgen_f64_descending,
        "swapped": _load().bqgen_f64_swapped,
    }[ordering]
    fn(seed, n, _ptr(a))
    return a


def rec32(n: int, seed: int = 1, dup_keys: int | None = None) -> np.ndarray:
    """Records as an (n, 4) uint64 array: column 0 = key, 1..3 = payload."""
    a = np.empty((n, 4), dtype=np.uint64)
    if dup_keys is None:
        _load().bqgen_rec32(seed, n, _ptr(a))
    else:
        _load().bqgen_rec32_dupkeys(seed, n, dup_keys, _ptr(a))
    return a


# --- BASELINE.json configs ---------------------------------------------------

CONFIG_N = {"c1": 1 << 20, "c2": 1 << 28, "c3": 1 << 27, "c4a": 1 << 28,
            "c4b": 1 << 28, "c5": 1 << 26}
CONFIG_KIND = {"c1": "i32", "c2": "i32", "c3": "f64", "c4a": "i32",
               "c4b": "i32", "c5": "rec32"}


def config(name: str, n: int | None = None, seed: int = 1,
           ordering: str = "random") -> np.ndarray:
    """Input of BASELINE.json config `name` at size n (default: full size)."""
    if n is None:
        n = CONFIG_N[name]
    if name == "c1":
        return i32_perm(n, seed)
    if name == "c2":
        return i32_full(n, seed)
    if name == "c3":
        return f64(n, seed, ordering)
    if name == "c4a":
        return i32_range(n, max(1, math.isqrt(n)), seed)
    if name == "c4b":
        return i32_const(n)
    if name == "c5":
        return rec32(n, seed)
    raise KeyError(name)


# --- the paper's structured workloads (bqgen.c) -----------

PATTERNS = ("imodsqrt", "square", "pow8", "sorted", "reversed", "rotation",
            "swaps_sqrt", "swaps_n", "swaps_nlogn", "halfhalf", "zeroone")


def i32_pattern(name: str, n: int, seed: int = 1) -> np.ndarray:
    """int32 input of one of the paper's Fig. 7/9/10/11 patterns."""
    a = np.empty(n, dtype=np.int32)
    rc = _load().bqgen_i32_pattern(PATTERNS.index(name), seed, n, _ptr(a))
    if rc != 0:
        raise ValueError(name)
    return a
