"""Batch container of the reference (proj/include/dyngraph/csr.hpp:12-88), host side.

`CsrBatch` is the drop-in input format: offsets span the whole vertex count.
The O(batch) COO form is what the measured entry points take; `csr_from_pairs`
is kept because the reference's callers build batches with it.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .errors import DataError


class BatchKind(Enum):  # csr.hpp:12
    Insert = 0
    Delete = 1


@dataclass
class CsrBatch:  # csr.hpp:17-25
    kind: BatchKind = BatchKind.Insert
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, dtype=np.uint64))
    destinations: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint32))

    def vertex_count(self) -> int:
        return 0 if len(self.offsets) == 0 else len(self.offsets) - 1

    def edge_count(self) -> int:
        return int(len(self.destinations))

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])


def csr_from_pairs(kind: BatchKind, vertex_count: int, src, dst) -> CsrBatch:
    """Stable grouping by source (csr.hpp:29-45): destinations keep input order."""
    src = np.asarray(src, dtype=np.uint32)
    dst = np.asarray(dst, dtype=np.uint32)
    if src.shape != dst.shape:
        raise DataError("csr_from_pairs: src/dst length mismatch")
    if len(src) and int(src.max()) >= vertex_count:
        raise DataError("csr_from_pairs: source out of range")
    counts = np.bincount(src, minlength=vertex_count).astype(np.uint64)
    offsets = np.zeros(vertex_count + 1, dtype=np.uint64)
    np.cumsum(counts, out=offsets[1:])
    order = np.argsort(src, kind="stable")
    return CsrBatch(kind, offsets, np.ascontiguousarray(dst[order]))


def compute_block_size(first_batch: CsrBatch) -> int:
    """Average degree of the non-empty sources, rounded half up, >= 1 (csr.hpp:77-88)."""
    deg = np.diff(first_batch.offsets.astype(np.int64))
    nonzero = int((deg > 0).sum())
    if nonzero == 0:
        raise DataError("compute_block_size: first batch contains no edges")
    total = first_batch.edge_count()
    rounded = (total + nonzero // 2) // nonzero
    return max(1, int(rounded))
