"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``liboracle.so`` (bq_oracle.cpp + stdsort_ref.cpp), the
plain single-threaded CPU BlockQuicksort written from the paper.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package; the product path
(``paper_1604_06697_b200``) never does and never falls back to it.

All functions work in place on numpy arrays (a private copy is made unless
``inplace=True``) and return the result.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

KINDS = ("i32", "u64", "f64", "rec32")
_DTYPES = {"i32": np.int32, "u64": np.uint64, "f64": np.float64}
MO3, NINTHER, SAMPLE64 = 0, 1, 2


class OracleOpts(ctypes.Structure):
    _fields_ = [("block", ctypes.c_longlong), ("cutoff", ctypes.c_longlong),
                ("depth_limit", ctypes.c_int)]


class OracleStats(ctypes.Structure):
    _fields_ = [("comparisons", ctypes.c_uint64), ("partitions", ctypes.c_uint64),
                ("heapsort_calls", ctypes.c_uint64), ("insertion_calls", ctypes.c_uint64),
                ("max_stack", ctypes.c_uint64)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


_SCALAR = {"i32": ctypes.c_int32, "u64": ctypes.c_uint64, "f64": ctypes.c_double,
           "rec32": ctypes.c_uint64}


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            from tools import build as _b
            _b.build_oracle()
        lib = ctypes.CDLL(_LIB_PATH)
        vp, ll = ctypes.c_void_p, ctypes.c_longlong
        for k in KINDS:
            f = getattr(lib, f"bq_oracle_sort_{k}")
            f.restype, f.argtypes = None, [vp, ll, ctypes.POINTER(OracleOpts), ctypes.POINTER(OracleStats)]
            f = getattr(lib, f"bq_oracle_block_partition_{k}")
            f.restype, f.argtypes = ll, [vp, ll, ll, ll, ctypes.POINTER(ctypes.c_ulonglong)]
            f = getattr(lib, f"bq_oracle_partition_{k}")
            f.restype, f.argtypes = None, [vp, ll, _SCALAR[k], ll, ctypes.POINTER(ll), ctypes.POINTER(ll)]
            f = getattr(lib, f"bq_oracle_pivot_{k}")
            f.restype, f.argtypes = _SCALAR[k], [vp, ll, ctypes.c_int]
            f = getattr(lib, f"bq_std_sort_{k}")
            f.restype, f.argtypes = None, [vp, ll]
            if k != "rec32":
                for nm in ("heapsort", "insertion_sort"):
                    f = getattr(lib, f"bq_oracle_{nm}_{k}")
                    f.restype, f.argtypes = None, [vp, ll]
        lib.bq_oracle_depth_limit.restype = ctypes.c_int
        lib.bq_oracle_depth_limit.argtypes = [ll]
        lib.bq_oracle_splitmix64_mix.restype = ctypes.c_uint64
        lib.bq_oracle_splitmix64_mix.argtypes = [ctypes.c_uint64]
        _lib = lib
    return _lib


def kind_of(a: np.ndarray) -> str:
    if a.ndim == 2 and a.shape[1] == 4 and a.dtype == np.uint64:
        return "rec32"
    for k, dt in _DTYPES.items():
        if a.dtype == dt:
            return k
    raise TypeError(f"unsupported array {a.dtype} {a.shape}")


def _prep(a, inplace):
    if not inplace:
        a = np.array(a, copy=True, order="C")
    assert a.flags["C_CONTIGUOUS"]
    return a


def sort(a: np.ndarray, block: int = 128, cutoff: int = 16, depth_limit: int = -1,
         inplace: bool = False, stats: bool = False):
    """O-sort: the paper's BlockQuicksort (simple variant) on a copy of `a`."""
    k = kind_of(a)
    a = _prep(a, inplace)
    o = OracleOpts(block, cutoff, depth_limit)
    st = OracleStats()
    getattr(_load(), f"bq_oracle_sort_{k}")(a.ctypes.data, len(a), ctypes.byref(o), ctypes.byref(st))
    return (a, st.as_dict()) if stats else a


def block_partition(a: np.ndarray, pivot_index: int, block: int = 128, inplace: bool = False):
    """Paper-form element-pivot block partition (Appendix B).
    Returns (array, cut, comparisons)."""
    k = kind_of(a)
    a = _prep(a, inplace)
    c = ctypes.c_ulonglong(0)
    cut = getattr(_load(), f"bq_oracle_block_partition_{k}")(a.ctypes.data, len(a), pivot_index,
                                                             block, ctypes.byref(c))
    return a, int(cut), int(c.value)


def partition(a: np.ndarray, pivot, block: int = 128, inplace: bool = False):
    """O-partition: value pivot, canonical three-way output.
    Returns (array, split, n_equal).  For records `pivot` is a key."""
    k = kind_of(a)
    a = _prep(a, inplace)
    s, e = ctypes.c_longlong(0), ctypes.c_longlong(0)
    getattr(_load(), f"bq_oracle_partition_{k}")(a.ctypes.data, len(a), _SCALAR[k](pivot), block,
                                                  ctypes.byref(s), ctypes.byref(e))
    return a, int(s.value), int(e.value)


def pivot(a: np.ndarray, rule: int = MO3):
    """Pivot value of the Mo3 (rule 0), ninther (rule 1) or 64-key sample
    median (rule 2) rule."""
    k = kind_of(a)
    a = np.ascontiguousarray(a)
    v = getattr(_load(), f"bq_oracle_pivot_{k}")(a.ctypes.data, len(a), rule)
    return v


def heapsort(a: np.ndarray):
    k = kind_of(a)
    a = _prep(a, False)
    getattr(_load(), f"bq_oracle_heapsort_{k}")(a.ctypes.data, len(a))
    return a


def insertion_sort(a: np.ndarray):
    k = kind_of(a)
    a = _prep(a, False)
    getattr(_load(), f"bq_oracle_insertion_sort_{k}")(a.ctypes.data, len(a))
    return a


def std_sort(a: np.ndarray, inplace: bool = False):
    """libstdc++ std::sort (a library routine, not the oracle)."""
    k = kind_of(a)
    a = _prep(a, inplace)
    getattr(_load(), f"bq_std_sort_{k}")(a.ctypes.data, len(a))
    return a


def depth_limit(n: int) -> int:
    return int(_load().bq_oracle_depth_limit(n))


def splitmix64_mix(z: int) -> int:
    """The oracle's SplitMix64 output function (R19), for its known-answer test."""
    return int(_load().bq_oracle_splitmix64_mix(z))
