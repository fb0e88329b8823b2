"""B200-native piCholesky cross-validation path (arXiv 1404.0466).

A drop-in for the hot path of the reference package ``ridgepath``
(``cvsearch.grid_search_pichol`` and the functions it calls): the same module
names (``linalg``, ``trivec``, ``pichol``, ``ridge``, ``cvsearch``, ``errors``),
signatures, dataclasses and exceptions, with the arithmetic in hand-written
FP64 sm_100a CUDA kernels reached through the C ABI in
``include/ridgepath_b200.h`` (``libridgepath_b200.so``). There is no CPU
fallback: compute entry points raise ``DeviceError`` without the library or a
GPU.
"""

from . import configs, cvsearch, errors, linalg, pichol, ridge, trivec
from .errors import (
    BadFormat,
    DeviceError,
    DimensionMismatch,
    HypothesisViolated,
    NotPositiveDefinite,
    NotSymmetric,
    NumericalError,
    RidgepathError,
    SingularInterpolant,
    UsageError,
)

__version__ = "0.1.0"

__all__ = [
    "configs",
    "cvsearch",
    "errors",
    "linalg",
    "pichol",
    "ridge",
    "trivec",
    "BadFormat",
    "DeviceError",
    "DimensionMismatch",
    "HypothesisViolated",
    "NotPositiveDefinite",
    "NotSymmetric",
    "NumericalError",
    "RidgepathError",
    "SingularInterpolant",
    "UsageError",
    "__version__",
]
