"""Host <-> device helpers for the drop-in API edge (numpy in, numpy out).

Matrices cross the edge as float64; column-major (F-order) d x d matrices are
uploaded as the row-major bytes of their transpose so the device sees the same
column-major layout as the C ABI.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def torch():
    import torch as _t

    return _t


def device():
    _lib.require_cuda()
    t = torch()
    return t.device("cuda", t.cuda.current_device())


def to_dev(a, dtype=None):
    """C-order upload of a numpy array (float64 unless dtype given)."""
    t = torch()
    a = np.ascontiguousarray(a, dtype=np.float64 if dtype is None else dtype)
    return t.from_numpy(a).to(device())


def colmajor_to_dev(M):
    """Upload a square matrix so the device buffer is its column-major layout."""
    M = np.asarray(M, dtype=np.float64)
    return to_dev(np.ascontiguousarray(M.T))


def colmajor_to_host(t, d):
    """Download a column-major d x d device buffer as an F-ordered numpy matrix."""
    a = t.reshape(d, d).cpu().numpy()  # row-major view of the transpose
    return np.asfortranarray(a.T)


def empty(shape, dtype=None):
    t = torch()
    return t.empty(shape, dtype=t.float64 if dtype is None else dtype, device=device())


def zeros(shape, dtype=None):
    t = torch()
    return t.zeros(shape, dtype=t.float64 if dtype is None else dtype, device=device())


def workspace(nbytes):
    t = torch()
    return t.empty((max(int(nbytes), 16),), dtype=t.uint8, device=device())
