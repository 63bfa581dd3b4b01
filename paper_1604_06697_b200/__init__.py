"""paper_1604_06697_b200 — BlockQuicksort's hot path, B200-native (sm_100a).

The block-partition step of Edelkamp & Weiß (arXiv 1604.06697) as hand-written
CUDA behind a C-ABI (``include/bq.h``, ``libbq.so``), driven into a full
three-way Quicksort/Introsort.  This package is only the thin ctypes binding
(``bq``); see DESIGN.md.
"""
from . import bq  # noqa: F401  (raises ImportError when libbq.so is missing)
from .bq import (  # noqa: F401
    BQ_F64, BQ_I32, BQ_KEYIDX16, BQ_PIVOT_MO3, BQ_PIVOT_NINTHER, BQ_PIVOT_SAMPLE64, BQ_REC32, BQ_U64, BQError,
    bq_partition_f64, bq_partition_i32, bq_partition_inplace, bq_partition_pass, bq_inplace_workspace_bytes, bq_partition_records, bq_partition_segments,
    bq_partition_u64,
    bq_pivot_f64, bq_pivot_i32, bq_pivot_records, bq_pivot_u64, bq_sort_ex, bq_sort_f64,
    bq_sort_host, bq_sort_i32, bq_sort_records, bq_sort_u64, bq_workspace_bytes, kind_of, partition,
    pivot, sort, workspace, workspace_bytes, tile_elems, leaf_elems, KIND, RECORDS_DEFAULT, RECORDS_DIRECT, RECORDS_KEYIDX,
)

LIB_PATH = bq.LIB_PATH
