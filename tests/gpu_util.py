"""Helpers shared by the -m gpu tests (test infrastructure)."""
import numpy as np
import torch


def to_dev(a: np.ndarray, offset: int = 0) -> torch.Tensor:
    """numpy -> contiguous CUDA tensor of the matching kind: u64 keys as
    torch.uint64, records (2-D) as int64 rows whose column 0 the binding reads
    as the unsigned key.  offset > 0 returns a view starting `offset` elements
    into a larger allocation (unaligned-pointer tests)."""
    if a.dtype == np.uint64 and a.ndim == 2:
        a = a.view(np.int64)
    if offset:
        a = np.concatenate([np.zeros((offset,) + a.shape[1:], dtype=a.dtype), a])
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t[offset:] if offset else t


def to_host(t: torch.Tensor, like: np.ndarray) -> np.ndarray:
    out = t.cpu().numpy()
    if like.dtype == np.uint64:
        out = out.view(np.uint64)
    return out


def three_list(a: np.ndarray, p, key=None):
    """The plain definition of the GPU partition layout (bq.h): keys < p in
    input order, keys == p, keys > p in reverse input order."""
    k = a if key is None else key(a)
    return np.concatenate([a[k < p], a[k == p], a[k > p][::-1]])
