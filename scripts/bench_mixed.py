#!/usr/bin/env python
"""BASELINE config 5: mixed interleaved insert / delete / query stream with vertex add / remove and
block reclamation, batch sizes 1K-100K (latency regime).  Follows the op mix of the reference's
random workloads (verify.hpp:179-259: 55 % insert, 25 % delete of which 70 % from the edge log,
10 % add 1-64 vertices, 10 % remove 1-4 vertices) plus a query batch after every update batch.
Every op goes through the public synchronous API with HOST batches, so a latency includes the
H2D copy of the batch and the status read-back.  Reports p50 / p99 per op and batch size.

    python scripts/bench_mixed.py [--scale 20] [--ops 400] [--cpu-ops 40] > profiles/rNN_mixed.json

The CPU reference (oracle/_ref, or the oracle port) runs the first --cpu-ops ops of the same stream
for the latency columns beside it, and the final graph digest is compared over that prefix."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def make_stream(scale, n_ops, seed=0x5EED):
    from paper_2306_08252_b200 import rmat
    rng = np.random.default_rng(seed)
    V = 1 << scale
    sizes = [1000, 3000, 10000, 30000, 100000]
    ops, log_s, log_d, cursor, size_v = [], [], [], 0, V
    for i in range(n_ops):
        roll = rng.random()
        b = int(rng.choice(sizes))
        if roll < 0.55 or not log_s:
            s, d = rmat.rmat_edges(scale, 2, cursor, b)
            cursor += b
            ops.append(("insert", s, d)); log_s.append(s); log_d.append(d)
        elif roll < 0.80:
            k = int(rng.integers(0, len(log_s)))
            n_log = min(b * 7 // 10, log_s[k].size)
            s = np.concatenate([log_s[k][:n_log], rng.integers(0, V, b - n_log).astype(np.uint32)])
            d = np.concatenate([log_d[k][:n_log], rng.integers(0, V, b - n_log).astype(np.uint32)])
            ops.append(("delete", s, d))
        elif roll < 0.90:
            c = int(rng.integers(1, 65))
            ops.append(("add_vertices", c)); size_v += c
        else:
            ids = rng.integers(V, max(V + 1, size_v), int(rng.integers(1, 5))).astype(np.uint32)   # only added vertices: sources of the stream stay alive
            ops.append(("del_vertices", ids))
        if ops[-1][0] in ("insert", "delete"):
            q = min(b, 10000)
            ops.append(("query", ops[-1][1][:q].copy(), rng.integers(0, V, q).astype(np.uint32)))
    return ops


def run(g, ops, is_gpu):
    lat = []
    for op in ops:
        t0 = time.perf_counter()
        if op[0] == "insert":
            g.insert_pairs(op[1], op[2])
        elif op[0] == "delete":
            g.delete_pairs(op[1], op[2])
        elif op[0] == "query":
            (g.query_edges if is_gpu else g.query)(op[1], op[2])
        elif op[0] == "add_vertices":
            g.insert_vertices(op[1])
        else:
            g.delete_vertices(op[1])
        lat.append((op[0], op[1].size if op[0] in ("insert", "delete", "query") else 0, (time.perf_counter() - t0) * 1e3))
    return lat


def summarize(lat):
    out = {}
    for kind in ("insert", "delete", "query", "add_vertices", "del_vertices"):
        for size in sorted({n for k, n, _ in lat if k == kind}):
            ms = np.array([t for k, n, t in lat if k == kind and n == size])
            key = f"{kind}@{size}" if size else kind
            out[key] = {"n": int(ms.size), "p50_ms": round(float(np.percentile(ms, 50)), 4), "p99_ms": round(float(np.percentile(ms, 99)), 4),
                        "medges_s_p50": round(size / np.percentile(ms, 50) / 1e3, 1) if size else None}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ops", type=int, default=400)
    ap.add_argument("--cpu-ops", type=int, default=40)
    a = ap.parse_args()
    import torch
    from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat
    V, E = 1 << a.scale, 16 << a.scale
    ops = make_stream(a.scale, a.ops)
    bs, bd = rmat.rmat_edges(a.scale, 1, 0, E)
    g = DynamicGraph(GraphConfig(pool_blocks=int(E / 32 * 1.5) + V, pool_max_blocks=int(E / 32 * 4) + 2 * V), V, 32)
    g.insert_pairs(bs, bd)
    run(g, ops[:20], True)          # warm-up on a prefix (workspace growth, module load) ...
    g.close()
    g = DynamicGraph(GraphConfig(pool_blocks=int(E / 32 * 1.5) + V, pool_max_blocks=int(E / 32 * 4) + 2 * V), V, 32)
    g.insert_pairs(bs, bd)          # ... then the measured run on a fresh graph
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lat = run(g, ops, True)
    wall = time.perf_counter() - t0
    updates = sum(n for k, n, _ in lat if k in ("insert", "delete"))
    res = {"workload": f"config 5: R-MAT s{a.scale} base ({E} edges), {len(ops)} interleaved ops (55/25/10/10 mix + a query batch per update), "
                       "batch sizes 1K-100K, reclaim on, growing pool; host batches through the synchronous public API",
           "gpu": summarize(lat), "gpu_total_s": round(wall, 4), "gpu_update_medges_s": round(updates / wall / 1e6, 1),
           "stats": {k: g.stats()[k] for k in ("active_edges", "pool_blocks_created", "pool_blocks_in_use", "growth_count", "logical_size")}}
    # CPU reference beside it on a prefix of the same stream (a fresh pair of graphs so the digests compare)
    from tests.drivers import CpuGraph, load_oracle, load_ref
    ref = load_ref()
    lib, prefix = (ref, "ref") if ref is not None else (load_oracle(), "orc")
    import os
    o = CpuGraph(lib, prefix, V, 32, 8 << 30, 0.5, True, os.cpu_count() or 1)
    o.insert_pairs(bs, bd)
    g2 = DynamicGraph(GraphConfig(pool_blocks=int(E / 32 * 1.5) + V, pool_max_blocks=int(E / 32 * 4) + 2 * V), V, 32)
    g2.insert_pairs(bs, bd)
    n_cpu = min(a.cpu_ops, len(ops))
    t0 = time.perf_counter()
    lat_cpu = run(o, ops[:n_cpu], False)
    cpu_wall = time.perf_counter() - t0
    run(g2, ops[:n_cpu], True)
    same = (g2.active_edges() == o.active_edges() and g2.logical_size() == o.logical_size() and
            np.array_equal(np.asarray(g2.degrees(), np.uint64), np.asarray(o.degrees(), np.uint64)))
    res["cpu_reference"] = {"kind": "reference" if ref is not None else "port", "cores": os.cpu_count(), "ops": n_cpu,
                            "latency": summarize(lat_cpu), "total_s": round(cpu_wall, 3),
                            "state_matches_gpu_after_prefix": bool(same)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
