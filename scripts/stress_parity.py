#!/usr/bin/env python
"""Randomised parity soak (GPU vs the oracle port): the reference's verify op mix (tests/workloads.py)
over many seeds with the knobs the unit tests only sample — native and odd block sizes, both COO
grouping strategies, CSR and COO entry points, fixed and growing pools, larger batches.  Prints one
line per failure and a summary; exit code 1 on any mismatch.

    python scripts/stress_parity.py --seeds 400 [--first 5000]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=200)
    ap.add_argument("--first", type=int, default=5000)
    a = ap.parse_args()
    from paper_2306_08252_b200 import BatchKind, DynamicGraph, GraphConfig, csr_from_pairs
    from tests.drivers import CpuGraph, GpuGraph, assert_same, load_oracle, run_script
    from tests.workloads import make_workload
    orc = load_oracle()
    fails, t0 = 0, time.time()
    for seed in range(a.first, a.first + a.seeds):
        rng = np.random.default_rng(seed ^ 0xABCDEF)
        cfg, script = make_workload(seed, max_vertices=6000, max_edges=int(rng.choice([3000, 30000, 150000])),
                                    max_insert=int(rng.choice([512, 4096, 40000])))
        B = int(rng.choice([32, 32, 32, 1, 2, 7, 15, 16, 31, 33, 48, 64]))
        cfg["block_size"] = B
        group = str(rng.choice(["auto", "radix", "count"]))
        grow = bool(rng.integers(0, 2))
        # turn some COO inserts / deletes into their CSR forms (sizes follow the logical size at that point)
        size, out = cfg["v0"], []
        for op in script:
            if op[0] == "add_vertices":
                size += op[1]
            if op[0] in ("insert", "delete") and rng.integers(0, 3) == 0 and len(op[1]) and int(op[1].max()) < size:
                b = csr_from_pairs(BatchKind.Insert if op[0] == "insert" else BatchKind.Delete, size, op[1], op[2])
                out.append((op[0] + "_csr", b.offsets, b.destinations))
            else:
                out.append(op)
        g = GpuGraph.__new__(GpuGraph)
        pool = 1 << 16
        g.g = DynamicGraph(GraphConfig(pool_blocks=(64 if grow else pool * (4 if B < 4 else 1)), pool_max_blocks=(pool * 8 if grow else 0),
                                       reclaim_on_delete=cfg["reclaim"], group=group), cfg["v0"], B)
        o = CpuGraph(orc, "orc", cfg["v0"], B, 1 << 30, 0.5, cfg["reclaim"], 1)
        try:
            assert_same(run_script(g, out), run_script(o, out), f"seed {seed}")
        except AssertionError as e:
            fails += 1
            print(f"FAIL seed={seed} B={B} group={group} grow={grow}: {str(e)[:200]}", flush=True)
        finally:
            g.close(); o.close()
    print(f"stress_parity: {a.seeds} seeds, {fails} failures, {time.time() - t0:.0f} s")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
