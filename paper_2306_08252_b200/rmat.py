"""numpy twin of the counter-based R-MAT generator (csrc/dg_kernels.cuh rmat_edge)."""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
IDX_MUL = np.uint64(0xD1342543DE82EF95)


def thresholds(a: float = 0.57, b: float = 0.19, c: float = 0.19):
    """32-bit fixed-point cumulative thresholds (a, a+b, a+b+c), computed exactly from
    integer per-mille inputs so every twin agrees."""
    pa, pb, pc = round(a * 1000), round(b * 1000), round(c * 1000)
    f = lambda pm: (pm * (1 << 32)) // 1000
    return int(f(pa)), int(f(pa + pb)), int(f(pa + pb + pc))


def _mix64(x: np.ndarray) -> np.ndarray:
    x = x + GOLDEN
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def rmat_edges(scale: int, seed: int, first_index: int, n: int, thr=None):
    """Edges [first_index, first_index + n) of the (scale, seed) R-MAT stream."""
    ta, tab, tabc = thr or thresholds()
    with np.errstate(over="ignore"):
        idx = np.arange(first_index, first_index + n, dtype=np.uint64)
        base = _mix64(np.uint64(seed) ^ (idx * IDX_MUL))
        s = np.zeros(n, dtype=np.uint32)
        d = np.zeros(n, dtype=np.uint32)
        for level in range(0, scale, 2):
            h = _mix64(base + np.uint64(level >> 1) * GOLDEN)
            halves = [(h & np.uint64(0xFFFFFFFF)).astype(np.uint32), (h >> np.uint64(32)).astype(np.uint32)]
            for half in range(2):
                if level + half >= scale:
                    break
                r = halves[half]
                sb = (r >= np.uint32(tab)).astype(np.uint32)
                db = (((r >= np.uint32(ta)) & (r < np.uint32(tab))) | (r >= np.uint32(tabc))).astype(np.uint32)
                s = (s << np.uint32(1)) | sb
                d = (d << np.uint32(1)) | db
    return s, d
