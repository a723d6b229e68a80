"""Random op scripts following the reference's verify workload mix
(proj/include/dyngraph/verify.hpp:135-265): 55% insert (<= 4096 pairs from
alive sources), 25% delete (70% from the edge log, 30% arbitrary), 10% add
1-64 vertices, 10% delete 1-4 vertices (+ a dead id 25% of the time), plus a
query sample at the end.  The RNG is numpy's, so scripts are reproducible from
the seed but not bit-identical to the reference's mt19937_64 stream; the
op mix and ranges are.
"""
from __future__ import annotations

import numpy as np


def make_workload(seed: int, max_vertices: int = 4096, max_edges: int = 100000,
                  max_insert: int = 4096, steps_lo: int = 4, steps_hi: int = 24):
    rng = np.random.default_rng(seed)
    v0 = int(1 + rng.integers(0, 256))
    block_size = int(1 + rng.integers(0, 8))
    reclaim = bool(rng.integers(0, 2) == 0)
    cfg = {"v0": v0, "block_size": block_size, "reclaim": reclaim,
           "workers": int(1 + rng.integers(0, 3)),
           "arena_bytes": 8 << 20, "initial_fraction": 0.002 + int(rng.integers(0, 32)) / 1000.0}
    size = v0
    alive = list(range(v0))
    dead = []
    log_s, log_d = [], []
    budget = int(min(max_edges, 200 + rng.integers(0, max_edges)))
    inserted = 0
    script = []
    for _ in range(int(rng.integers(steps_lo, steps_hi))):
        roll = int(rng.integers(0, 100))
        if not alive and roll < 80:
            roll = 90
        if roll < 55:
            if inserted >= budget or not alive:
                continue
            k = int(min(1 + rng.integers(0, max_insert), budget - inserted))
            al = np.asarray(alive, np.uint32)
            s = al[rng.integers(0, len(al), k)]
            d = rng.integers(0, size, k).astype(np.uint32)
            script.append(("insert", s, d))
            log_s.append(s); log_d.append(d)
            inserted += k
        elif roll < 80:
            if not log_s:
                continue
            ls, ld = np.concatenate(log_s), np.concatenate(log_d)
            k = int(1 + rng.integers(0, min(len(ls), 2048)))
            pick = rng.integers(0, len(ls), k)
            s, d = ls[pick].copy(), ld[pick].copy()
            arb = rng.integers(0, 10, k) >= 7
            s[arb] = rng.integers(0, size, int(arb.sum())).astype(np.uint32)
            d[arb] = rng.integers(0, size, int(arb.sum())).astype(np.uint32)
            script.append(("delete", s, d))
        elif roll < 90:
            if size >= max_vertices:
                continue
            count = int(min(1 + rng.integers(0, 64), max_vertices - size))
            script.append(("add_vertices", count))
            alive.extend(range(size, size + count))
            size += count
        else:
            if not alive:
                continue
            count = int(1 + rng.integers(0, 4))
            ids = [alive[int(rng.integers(0, len(alive)))] for _ in range(count)]
            if rng.integers(0, 4) == 0 and dead:
                ids.append(dead[0])
            script.append(("del_vertices", np.asarray(ids, np.uint32)))
            for i in ids:
                if i in alive:
                    alive.remove(i)
                    dead.append(i)
        script.append(("check",))
    # query sample: every logged edge candidate + random pairs (oracle.hpp:141-160)
    if log_s:
        ls, ld = np.concatenate(log_s), np.concatenate(log_d)
        pick = rng.integers(0, len(ls), min(len(ls), 512))
        qs = np.concatenate([ls[pick], rng.integers(0, size + 4, 256).astype(np.uint32)])
        qd = np.concatenate([ld[pick], rng.integers(0, size + 4, 256).astype(np.uint32)])
    else:
        qs = rng.integers(0, size + 4, 256).astype(np.uint32)
        qd = rng.integers(0, size + 4, 256).astype(np.uint32)
    script.append(("query", qs, qd))
    return cfg, script
