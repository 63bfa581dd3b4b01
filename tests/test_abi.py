"""The C-ABI library (CPU, -m "not gpu"): it builds, loads, and exports every
symbol include/bq.h declares; argument validation needs no GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bq.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"BQ_API\s+[\w\s\*]+?\b(bq_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from tools import build
    path = build.build_bq()
    return ctypes.CDLL(path), path


def test_header_declares_entry_points():
    names = _declared()
    for must in ["bq_workspace_bytes", "bq_partition_i32", "bq_partition_u64", "bq_partition_f64",
                 "bq_sort_i32", "bq_sort_u64", "bq_sort_f64", "bq_sort_records", "bq_pivot_i32",
                 "bq_partition_pass", "bq_sort_ex", "bq_sort_host", "bq_last_error"]:
        assert must in names


def test_exports_every_declared_symbol(lib):
    so, path = lib
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bq_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    for n in _declared():
        getattr(so, n)
    # nothing but the C-ABI is exported
    assert all(e in _declared() for e in exported), sorted(exported - set(_declared()))


def test_sm100a_cubin(lib):
    _, path = lib
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls(lib):
    so, _ = lib
    so.bq_workspace_bytes.restype = ctypes.c_size_t
    so.bq_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_size_t]
    n = 1 << 20
    for kind, w in [(0, 4), (1, 8), (2, 8), (3, 32)]:
        b = so.bq_workspace_bytes(kind, n)
        # n*w scratch + O(n/T); below ~5M elements the in-place partition's
        # two cleanup buffers (2*n*w) can be the larger need
        assert n * w <= b < 2 * n * w + n * w // 4 + (1 << 16)
        if kind == 3:
            # records (bq.h): the key+index path's 16n pairs + the pair sort's
            # layout (16n scratch + O(n/T)) + the 32n copy of the records
            assert so.bq_workspace_bytes(kind, 1 << 28) < (1 << 28) * 68
        else:
            assert so.bq_workspace_bytes(kind, 1 << 28) < (1 << 28) * w * 5 // 4 + (1 << 26)
    so.bq_status_string.restype = ctypes.c_char_p
    assert so.bq_status_string(0) == b"BQ_OK"
    assert so.bq_status_string(4) == b"BQ_ERR_UNSUPPORTED"
    assert so.bq_version() >= 100


def test_argument_validation_without_gpu(lib):
    so, _ = lib
    vp, sz = ctypes.c_void_p, ctypes.c_size_t
    so.bq_sort_i32.argtypes = [vp, sz, vp, sz, vp]
    so.bq_last_error.restype = ctypes.c_char_p
    assert so.bq_sort_i32(None, 1 << 31, None, 0, None) == 1          # n >= 2^31
    assert so.bq_sort_i32(None, 10, None, 0, None) == 1               # NULL data
    assert so.bq_sort_i32(ctypes.c_void_p(256), 10, None, 0, None) == 2   # no workspace
    assert b"workspace" in so.bq_last_error()


def test_product_path_never_touches_oracle():
    pkg = os.path.join(ROOT, "paper_1604_06697_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "bq_oracle" not in txt, f


def test_workspace_sizes_of_the_next_rows(lib):
    """Host-only sizing of the §8(f) rows: the key+index kind, the records
    workspace covering the key+index path, and the in-place partition's
    workspace, which does not grow with n (N2)."""
    so, _ = lib
    for f in (so.bq_workspace_bytes, so.bq_inplace_workspace_bytes):
        f.restype = ctypes.c_size_t
        f.argtypes = [ctypes.c_int, ctypes.c_size_t]
    n = 1 << 22
    pair = so.bq_workspace_bytes(4, n)
    assert 16 * n <= pair < 16 * n + 4 * n
    rec = so.bq_workspace_bytes(3, n)
    assert rec >= 16 * n + pair + 4 * n
    assert so.bq_workspace_bytes(5, n) == 0                       # unknown kind
    for kind in range(5):
        small = so.bq_inplace_workspace_bytes(kind, 1000)
        big = so.bq_inplace_workspace_bytes(kind, 1 << 30)
        assert 0 < small <= big == so.bq_inplace_workspace_bytes(kind, 1 << 28)
        assert big < (64 << 20)


def test_options_struct_layout():
    """bq_sort_options / bq_sort_stats as the binding declares them match the
    header's field lists (eight int32 options; the stats' sizes)."""
    import paper_1604_06697_b200.bq as b
    src = open(HEADER).read()
    body = src[src.index("typedef struct {\n    int32_t pivot_rule;"):src.index("} bq_sort_options;")]
    n_fields = sum(int(m.group(2) or 1) for m in re.finditer(r"int32_t (\w+)(?:\[(\d+)\])?;", body))
    assert ctypes.sizeof(b.bq_sort_options) == 4 * n_fields == 32
    assert [f for f, _ in b.bq_sort_options._fields_][:7] == ["pivot_rule", "depth_limit", "timing", "ordered",
                                                               "ways", "records", "subtree"]
    body = src[src.index("typedef struct {\n    uint32_t levels;"):src.index("} bq_sort_stats;")]
    size = {"uint32_t": 4, "uint64_t": 8, "double": 8}
    fields = re.findall(r"^\s*(uint32_t|uint64_t|double) (\w+);", body, re.M)
    assert [f for f, _ in b.bq_sort_stats._fields_] == [nm for _, nm in fields]
    assert ctypes.sizeof(b.bq_sort_stats) == sum(size[t] for t, _ in fields) == 112


def test_binding_refuses_ambiguous_int64():
    """A 1-D int64 tensor has no unambiguous order for libbq (uint64 keys are
    compared unsigned): the binding refuses it; uint64, int32,
    float64 and the 2-D record/pair shapes map to their kinds."""
    import torch
    import pytest
    import paper_1604_06697_b200 as bq
    with pytest.raises(TypeError):
        bq.kind_of(torch.zeros(4, dtype=torch.int64))
    assert bq.kind_of(torch.zeros(4, dtype=torch.uint64)) == bq.BQ_U64
    assert bq.kind_of(torch.zeros(4, dtype=torch.int32)) == bq.BQ_I32
    assert bq.kind_of(torch.zeros(4, dtype=torch.float64)) == bq.BQ_F64
    assert bq.kind_of(torch.zeros((4, 4), dtype=torch.int64)) == bq.BQ_REC32
    assert bq.kind_of(torch.zeros((4, 2), dtype=torch.int64)) == bq.BQ_KEYIDX16


def test_workspace_follows_the_leaf_bound(lib, monkeypatch):
    """driver.cuh leaf_max_for: the plan's leaf bound sizes the workspace (more
    segments and leaves under a smaller bound); the BQ_LEAF_MAX override is
    clamped to [2 warps' keys, S] and a malformed value leaves the default."""
    so, _ = lib
    so.bq_workspace_bytes.restype = ctypes.c_size_t
    so.bq_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_size_t]
    so.bq_leaf_elems.restype = ctypes.c_size_t
    so.bq_leaf_elems.argtypes = [ctypes.c_int]
    n = 1 << 24
    for kind in (0, 1, 2):
        S = so.bq_leaf_elems(kind)
        monkeypatch.delenv("BQ_LEAF_MAX", raising=False)
        base = so.bq_workspace_bytes(kind, n)
        monkeypatch.setenv("BQ_LEAF_MAX", str(S // 8))
        small = so.bq_workspace_bytes(kind, n)
        monkeypatch.setenv("BQ_LEAF_MAX", "1")            # clamped up to IPT * 64
        tiny = so.bq_workspace_bytes(kind, n)
        monkeypatch.setenv("BQ_LEAF_MAX", str(S // 16))   # = IPT * 64
        assert so.bq_workspace_bytes(kind, n) == tiny
        assert base < small < tiny
        for bad in ("0", "-5", "abc", str(10 * S)):       # ignored / clamped down to S
            monkeypatch.setenv("BQ_LEAF_MAX", bad)
            assert so.bq_workspace_bytes(kind, n) == base
