"""Python binding of libbq.so — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C-ABI
(include/bq.h); this module only turns torch tensors into device pointers and
the current CUDA stream into a ``cudaStream_t``.  There is no CPU fallback:
if ``libbq.so`` is missing or fails to load, importing this module raises.

Function names are the C names.  Tensors must be CUDA, contiguous, and of the
kind's dtype: int32 (``i32``), uint64 (``u64``; a 1-D int64 tensor is refused,
since its order would be ambiguous — pass ``t.view(torch.uint64)``), float64
(``f64``), records as an (n, 4) uint64/int64 tensor whose column 0 is the
unsigned key (``rec32``, 32 bytes per row), and key+index pairs as an (n, 2)
uint64/int64 tensor (``keyidx16``: key, index).  Every call runs on the
tensor's device (device guard) and on the given stream (default: that
device's current stream); a workspace the binding allocates is allocated on
that stream, so the caching allocator reuses it only after the call's work.
"""
from __future__ import annotations

import ctypes
import functools
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# BQ_LIB may point at a tuning variant of the same library (tools/tune.py)
LIB_PATH = os.environ.get("BQ_LIB", os.path.join(_HERE, "libbq.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

BQ_OK, BQ_ERR_INVALID_ARGUMENT, BQ_ERR_WORKSPACE, BQ_ERR_CUDA, BQ_ERR_UNSUPPORTED = range(5)
BQ_I32, BQ_U64, BQ_F64, BQ_REC32, BQ_KEYIDX16 = range(5)
BQ_PIVOT_MO3, BQ_PIVOT_NINTHER, BQ_PIVOT_SAMPLE64 = range(3)
KIND = {"i32": BQ_I32, "u64": BQ_U64, "f64": BQ_F64, "rec32": BQ_REC32, "keyidx16": BQ_KEYIDX16}
WIDTH = {BQ_I32: 4, BQ_U64: 8, BQ_F64: 8, BQ_REC32: 32, BQ_KEYIDX16: 16}
# bq_sort_options.records: the records sort path
RECORDS_DEFAULT, RECORDS_DIRECT, RECORDS_KEYIDX = 0, 1, 2


class bq_sort_options(ctypes.Structure):
    _fields_ = [("pivot_rule", ctypes.c_int32), ("depth_limit", ctypes.c_int32),
                ("timing", ctypes.c_int32), ("ordered", ctypes.c_int32), ("ways", ctypes.c_int32),
                ("records", ctypes.c_int32), ("subtree", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1)]


class bq_sort_stats(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_uint32), ("partition_launches", ctypes.c_uint32),
                ("kernel_launches", ctypes.c_uint32), ("reserved0", ctypes.c_uint32),
                ("element_passes", ctypes.c_uint64), ("partitioned_segments", ctypes.c_uint64),
                ("leaves", ctypes.c_uint64), ("fallback_segments", ctypes.c_uint64),
                ("band_elements", ctypes.c_uint64), ("partition_ms", ctypes.c_double),
                ("partition_bytes", ctypes.c_double), ("multiway_ms", ctypes.c_double),
                ("multiway_element_passes", ctypes.c_uint64), ("mw_count_ms", ctypes.c_double),
                ("mw_scatter_ms", ctypes.c_double), ("leaf_ms", ctypes.c_double)]

    def as_dict(self):
        return {f: (getattr(self, f) if not isinstance(getattr(self, f), ctypes.Array) else None)
                for f, _ in self._fields_}


_vp, _sz, _st = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
_psz = ctypes.POINTER(ctypes.c_size_t)

_SIGS = {
    "bq_workspace_bytes": (_sz, [_st, _sz]),
    "bq_pivot_i32": (_st, [_vp, _sz, _st, ctypes.POINTER(ctypes.c_int32), _vp, _sz, _vp]),
    "bq_pivot_u64": (_st, [_vp, _sz, _st, ctypes.POINTER(ctypes.c_uint64), _vp, _sz, _vp]),
    "bq_pivot_f64": (_st, [_vp, _sz, _st, ctypes.POINTER(ctypes.c_double), _vp, _sz, _vp]),
    "bq_pivot_records": (_st, [_vp, _sz, _st, ctypes.POINTER(ctypes.c_uint64), _vp, _sz, _vp]),
    "bq_partition_i32": (_st, [_vp, _sz, ctypes.c_int32, _psz, _psz, _vp, _sz, _vp]),
    "bq_partition_u64": (_st, [_vp, _sz, ctypes.c_uint64, _psz, _psz, _vp, _sz, _vp]),
    "bq_partition_f64": (_st, [_vp, _sz, ctypes.c_double, _psz, _psz, _vp, _sz, _vp]),
    "bq_partition_records": (_st, [_vp, _sz, ctypes.c_uint64, _psz, _psz, _vp, _sz, _vp]),
    "bq_partition_pass": (_st, [_st, _vp, _vp, _sz, _vp, _vp, _st, _vp, _sz, _vp]),
    "bq_inplace_workspace_bytes": (_sz, [_st, _sz]),
    "bq_partition_inplace": (_st, [_st, _vp, _sz, _vp, _psz, _psz, _vp, _sz, _vp]),
    "bq_partition_segments": (_st, [_st, _vp, _vp, _sz, _vp, _vp, _vp, _sz, _vp, _st, _vp, _sz, _vp]),
    "bq_sort_i32": (_st, [_vp, _sz, _vp, _sz, _vp]),
    "bq_sort_u64": (_st, [_vp, _sz, _vp, _sz, _vp]),
    "bq_sort_f64": (_st, [_vp, _sz, _vp, _sz, _vp]),
    "bq_sort_records": (_st, [_vp, _sz, _vp, _sz, _vp]),
    "bq_sort_ex": (_st, [_st, _vp, _sz, ctypes.POINTER(bq_sort_options),
                         ctypes.POINTER(bq_sort_stats), _vp, _sz, _vp]),
    "bq_sort_host": (_st, [_st, _vp, _sz, _vp, ctypes.POINTER(bq_sort_options), _vp, _sz, _vp]),
    "bq_status_string": (ctypes.c_char_p, [_st]),
    "bq_last_error": (ctypes.c_char_p, []),
    "bq_version": (ctypes.c_int, []),
    "bq_tile_elems": (_sz, [_st]),
    "bq_leaf_elems": (_sz, [_st]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args


class BQError(RuntimeError):
    def __init__(self, status: int):
        self.status = status
        msg = _lib.bq_status_string(status).decode()
        detail = _lib.bq_last_error().decode()
        super().__init__(f"{msg}: {detail}" if detail else msg)


def _check(status: int):
    if status != BQ_OK:
        raise BQError(status)


# --- marshalling helpers -------------------------------------------------------

def kind_of(t: torch.Tensor) -> int:
    if t.dim() == 2 and t.shape[1] == 4 and t.dtype in (torch.uint64, torch.int64):
        return BQ_REC32
    if t.dim() == 2 and t.shape[1] == 2 and t.dtype in (torch.uint64, torch.int64):
        return BQ_KEYIDX16
    if t.dtype == torch.int32:
        return BQ_I32
    if t.dtype == torch.uint64:
        return BQ_U64
    if t.dtype == torch.int64 and t.dim() == 1:
        raise TypeError("1-D int64 keys are ambiguous (libbq sorts uint64 keys unsigned): "
                        "pass t.view(torch.uint64)")
    if t.dtype == torch.float64:
        return BQ_F64
    raise TypeError(f"unsupported tensor {t.dtype} {tuple(t.shape)}")


def _n(t: torch.Tensor) -> int:
    return t.shape[0] if t.dim() >= 1 else 0


def _dev(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _torch_stream(stream):
    if stream is None:
        return torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream))


def _guard(fn):
    """Run an entry point on the device of its first CUDA tensor argument
    (libbq launches on the current device)."""
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        for x in args:
            if isinstance(x, torch.Tensor) and x.is_cuda:
                with torch.cuda.device(x.device):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)
    return wrapper


def _same(a: torch.Tensor, b: torch.Tensor, what: str):
    if a.shape != b.shape or a.dtype != b.dtype:
        raise ValueError(f"{what}: shape/dtype {tuple(b.shape)} {b.dtype} != {tuple(a.shape)} {a.dtype}")


def _counts(d_counts: torch.Tensor, nseg: int):
    if not (isinstance(d_counts, torch.Tensor) and d_counts.is_cuda and d_counts.is_contiguous()
            and d_counts.dtype in (torch.int64, torch.uint64) and d_counts.numel() >= 3 * nseg):
        raise ValueError(f"d_counts must be a contiguous CUDA int64/uint64 tensor of >= {3 * nseg} elements")


def workspace_bytes(kind: int, n: int) -> int:
    return int(_lib.bq_workspace_bytes(kind, n))


def bq_workspace_bytes(kind: int, n: int) -> int:
    return workspace_bytes(kind, n)


def workspace(kind: int, n: int, device=None) -> torch.Tensor:
    """A device workspace tensor of bq_workspace_bytes(kind, n) bytes."""
    return torch.empty(workspace_bytes(kind, n), dtype=torch.uint8,
                       device=device if device is not None else "cuda")


def _ws(ws, kind, n, like, stream=None):
    if ws is None:
        with torch.cuda.stream(_torch_stream(stream)):
            ws = workspace(kind, n, like.device)
    elif not ws.is_cuda or ws.device != like.device:
        raise ValueError("the workspace must be on the data's device")
    return ws.data_ptr(), ws.numel() * ws.element_size()


# --- entry points ---------------------------------------------------------------

@_guard
def _pivot(name, ctype, t, rule, ws, stream):
    kind = kind_of(t)
    w, wb = _ws(ws, kind, _n(t), t, stream)
    out = ctype()
    _check(getattr(_lib, name)(_dev(t), _n(t), rule, ctypes.byref(out), w, wb, _stream(stream)))
    return out.value


@_guard
def bq_pivot_i32(keys, rule=BQ_PIVOT_MO3, ws=None, stream=None):
    return _pivot("bq_pivot_i32", ctypes.c_int32, keys, rule, ws, stream)


@_guard
def bq_pivot_u64(keys, rule=BQ_PIVOT_MO3, ws=None, stream=None):
    return _pivot("bq_pivot_u64", ctypes.c_uint64, keys, rule, ws, stream)


@_guard
def bq_pivot_f64(keys, rule=BQ_PIVOT_MO3, ws=None, stream=None):
    return _pivot("bq_pivot_f64", ctypes.c_double, keys, rule, ws, stream)


@_guard
def bq_pivot_records(recs, rule=BQ_PIVOT_MO3, ws=None, stream=None):
    return _pivot("bq_pivot_records", ctypes.c_uint64, recs, rule, ws, stream)


@_guard
def _partition(name, cpivot, t, pivot, ws, stream):
    kind = kind_of(t)
    w, wb = _ws(ws, kind, _n(t), t, stream)
    s, e = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(getattr(_lib, name)(_dev(t), _n(t), cpivot(pivot), ctypes.byref(s), ctypes.byref(e),
                               w, wb, _stream(stream)))
    return s.value, e.value


@_guard
def bq_partition_i32(keys, pivot, ws=None, stream=None):
    return _partition("bq_partition_i32", ctypes.c_int32, keys, pivot, ws, stream)


@_guard
def bq_partition_u64(keys, pivot, ws=None, stream=None):
    return _partition("bq_partition_u64", ctypes.c_uint64, keys, pivot, ws, stream)


@_guard
def bq_partition_f64(keys, pivot, ws=None, stream=None):
    return _partition("bq_partition_f64", ctypes.c_double, keys, pivot, ws, stream)


@_guard
def bq_partition_records(recs, pivot_key, ws=None, stream=None):
    return _partition("bq_partition_records", ctypes.c_uint64, recs, pivot_key, ws, stream)


_PIVOT_CTYPE = {BQ_I32: ctypes.c_int32, BQ_U64: ctypes.c_uint64, BQ_F64: ctypes.c_double,
                BQ_REC32: ctypes.c_uint64, BQ_KEYIDX16: ctypes.c_uint64}


@_guard
def bq_partition_pass(src, dst, pivot, d_counts, ordered=True, ws=None, stream=None):
    """Asynchronous out-of-place pass; d_counts is a CUDA uint64/int64 tensor of >= 3."""
    kind = kind_of(src)
    _same(src, dst, "dst")
    _counts(d_counts, 1)
    w, wb = _ws(ws, kind, _n(src), src, stream)
    pv = _PIVOT_CTYPE[kind](pivot)
    _check(_lib.bq_partition_pass(kind, _dev(src), _dev(dst), _n(src), ctypes.byref(pv),
                                  _dev(d_counts), int(ordered), w, wb, _stream(stream)))


def bq_inplace_workspace_bytes(kind: int, n: int) -> int:
    return int(_lib.bq_inplace_workspace_bytes(kind, n))


@_guard
def bq_partition_inplace(data, pivot, ws=None, stream=None):
    """In-place three-way partition with a small workspace (N2); returns
    (split, n_equal).  The order inside each band is unspecified."""
    kind = kind_of(data)
    if ws is None:
        with torch.cuda.stream(_torch_stream(stream)):
            ws = torch.empty(bq_inplace_workspace_bytes(kind, _n(data)), dtype=torch.uint8, device=data.device)
    pv = _PIVOT_CTYPE[kind](pivot)
    s, e = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(_lib.bq_partition_inplace(kind, _dev(data), _n(data), ctypes.byref(pv), ctypes.byref(s),
                                     ctypes.byref(e), ws.data_ptr(), ws.numel() * ws.element_size(),
                                     _stream(stream)))
    return s.value, e.value


@_guard
def bq_partition_segments(src, dst, begins, lens, pivots, d_counts, ordered=True, ws=None, stream=None):
    """Batched pass over disjoint segments; begins/lens/pivots are host sequences,
    d_counts a CUDA int64 tensor of >= 3*len(begins).  Synchronises the stream."""
    import numpy as np
    kind = kind_of(src)
    _same(src, dst, "dst")
    nseg = len(begins)
    if not (len(lens) == nseg and len(pivots) == nseg):
        raise ValueError("begins, lens and pivots must have the same length")
    _counts(d_counts, nseg)
    w, wb = _ws(ws, kind, _n(src), src, stream)
    b = np.ascontiguousarray(np.asarray(begins, dtype=np.uint32))
    ln = np.ascontiguousarray(np.asarray(lens, dtype=np.uint32))
    pdt = {BQ_I32: np.int32, BQ_U64: np.uint64, BQ_F64: np.float64, BQ_REC32: np.uint64,
           BQ_KEYIDX16: np.uint64}[kind]
    pv = np.ascontiguousarray(np.asarray(pivots).astype(pdt))
    _check(_lib.bq_partition_segments(kind, _dev(src), _dev(dst), _n(src), b.ctypes.data, ln.ctypes.data,
                                      pv.ctypes.data, nseg, _dev(d_counts), int(ordered), w, wb,
                                      _stream(stream)))


_SORT_KIND = {"bq_sort_i32": BQ_I32, "bq_sort_u64": BQ_U64, "bq_sort_f64": BQ_F64, "bq_sort_records": BQ_REC32}


@_guard
def _sort(name, t, ws, stream):
    kind = kind_of(t)
    if kind != _SORT_KIND[name]:
        raise TypeError(f"{name}: tensor of kind {kind}")
    w, wb = _ws(ws, kind, _n(t), t, stream)
    _check(getattr(_lib, name)(_dev(t), _n(t), w, wb, _stream(stream)))
    return t


@_guard
def bq_sort_i32(keys, ws=None, stream=None):
    return _sort("bq_sort_i32", keys, ws, stream)


@_guard
def bq_sort_u64(keys, ws=None, stream=None):
    return _sort("bq_sort_u64", keys, ws, stream)


@_guard
def bq_sort_f64(keys, ws=None, stream=None):
    return _sort("bq_sort_f64", keys, ws, stream)


@_guard
def bq_sort_records(recs, ws=None, stream=None):
    return _sort("bq_sort_records", recs, ws, stream)


def _opts(pivot_rule, depth_limit, timing, ordered=False, ways=0, records=0, subtree=False):
    o = bq_sort_options()
    o.records = int(records)
    o.subtree = int(subtree)
    o.pivot_rule = pivot_rule
    o.depth_limit = depth_limit
    o.timing = int(timing)
    o.ordered = int(ordered)
    o.ways = int(ways)
    return o


@_guard
def bq_sort_ex(data, pivot_rule=BQ_PIVOT_SAMPLE64, depth_limit=-1, timing=False, ordered=False, ways=0,
               records=RECORDS_DEFAULT, subtree=False, ws=None, stream=None, stats=True):
    """Kind-generic sort; returns the bq_sort_stats as a dict (stats=True: the
    call then waits for the stream to read the device counters; stats=False:
    fully asynchronous, returns None).  ways: 0 the default per kind (binary
    for int32 and records, 8-way for 64-bit keys and key+index pairs), 2
    binary, 8 or 16 multi-pivot passes.  records: RECORDS_DEFAULT /
    RECORDS_KEYIDX sort (key, index) pairs and gather the records once,
    RECORDS_DIRECT moves the records in every pass.  subtree: ignored (ABI
    field kept)."""
    kind = kind_of(data)
    w, wb = _ws(ws, kind, _n(data), data, stream)
    o = _opts(pivot_rule, depth_limit, timing, ordered, ways, records, subtree)
    st = bq_sort_stats() if stats else None
    _check(_lib.bq_sort_ex(kind, _dev(data), _n(data), ctypes.byref(o), ctypes.byref(st) if stats else None,
                           w, wb, _stream(stream)))
    return st.as_dict() if stats else None


@_guard
def bq_sort_host(host, dev, pivot_rule=BQ_PIVOT_SAMPLE64, ways=0, ws=None, stream=None):
    """End-to-end sort of a host (ideally pinned) tensor through dev (same shape/dtype)."""
    kind = kind_of(dev)
    if host.is_cuda or not host.is_contiguous():
        raise ValueError("host must be a contiguous CPU tensor")
    _same(dev, host, "host")
    w, wb = _ws(ws, kind, _n(dev), dev, stream)
    o = _opts(pivot_rule, -1, False, False, ways)
    _check(_lib.bq_sort_host(kind, host.data_ptr(), _n(dev), _dev(dev), ctypes.byref(o), w, wb,
                             _stream(stream)))
    return host


# --- conveniences ---------------------------------------------------------------

_SORT_BY_KIND = {BQ_I32: bq_sort_i32, BQ_U64: bq_sort_u64, BQ_F64: bq_sort_f64,
                 BQ_REC32: bq_sort_records}
_PART_BY_KIND = {BQ_I32: bq_partition_i32, BQ_U64: bq_partition_u64, BQ_F64: bq_partition_f64,
                 BQ_REC32: bq_partition_records}
_PIVOT_BY_KIND = {BQ_I32: bq_pivot_i32, BQ_U64: bq_pivot_u64, BQ_F64: bq_pivot_f64,
                  BQ_REC32: bq_pivot_records}


def sort(t, ws=None, stream=None):
    """Sort a CUDA tensor in place (kind from dtype/shape)."""
    return _SORT_BY_KIND[kind_of(t)](t, ws, stream)


def partition(t, pivot, ws=None, stream=None):
    return _PART_BY_KIND[kind_of(t)](t, pivot, ws, stream)


def pivot(t, rule=BQ_PIVOT_MO3, ws=None, stream=None):
    return _PIVOT_BY_KIND[kind_of(t)](t, rule, ws, stream)


def version() -> int:
    return int(_lib.bq_version())


def tile_elems(kind: int) -> int:
    """Partition tile T of `kind` (bq_tile_elems)."""
    return int(_lib.bq_tile_elems(kind))


def leaf_elems(kind: int) -> int:
    """Leaf size S of `kind` (bq_leaf_elems): segments of <= S elements are
    finished by the shared-memory leaf sort."""
    return int(_lib.bq_leaf_elems(kind))
