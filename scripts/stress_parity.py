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
    ap.add_argument("--hubs", action="store_true",
                    help="hub-heavy scripts instead of the verify mix: few vertices, zipf sources, 50K-400K-entry batches "
                         "(chains of thousands of blocks, table tiers with several 4096-target slices, heavy CSR items)")
    ap.add_argument("--submit", action="store_true",
                    help="streams of SUBMITTED COO updates (dg_submit_*_coo, no host wait between ops, one flush per stream; some "
                         "streams carry a rejected batch in the middle): final canonical state against the oracle port")
    a = ap.parse_args()
    from paper_2306_08252_b200 import BatchKind, DynamicGraph, GraphConfig, csr_from_pairs
    from tests.drivers import CpuGraph, GpuGraph, assert_same, load_oracle, run_script
    from tests.workloads import make_workload
    orc = load_oracle()
    fails, t0 = 0, time.time()
    if a.submit:
        import torch
        from paper_2306_08252_b200 import DataError, EngineError

        def dev(x):
            return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).cuda()
        for seed in range(a.first, a.first + a.seeds):
            rng = np.random.default_rng(seed)
            V = int(rng.choice([60, 900, 6000, 50000]))
            B = int(rng.choice([32, 32, 32, 5, 33]))
            grow = bool(rng.integers(0, 3) == 0)
            g = DynamicGraph(GraphConfig(pool_blocks=(512 if grow else 1 << 21), pool_max_blocks=(1 << 21 if grow else 0),
                                         group=str(rng.choice(["auto", "radix", "count"])),
                                         submit_inputs_ready=bool(rng.integers(0, 4) != 0)), V, B)
            o = CpuGraph(orc, "orc", V, B, 2 << 30, 0.5, True, 1)
            keep, log, what = [], [], ""
            try:
                for stream in range(int(rng.integers(1, 4))):
                    n_ops = int(rng.integers(2, 9))
                    bad_at = int(rng.integers(0, n_ops)) if rng.integers(0, 4) == 0 else -1
                    applied_expect, failed, reported = 0, False, False
                    for it in range(n_ops):
                        n = int(rng.choice([1, 300, 20000, 120000]))
                        s = (rng.zipf(float(rng.choice([1.2, 1.6])), n) % V).astype(np.uint32)
                        d = rng.integers(0, V, n).astype(np.uint32)
                        kind = "insert" if not log or rng.random() < 0.55 else "delete"
                        if kind == "delete":
                            ps, pd = log[int(rng.integers(0, len(log)))]
                            k = min(n, len(ps)) * 7 // 10
                            s[:k], d[:k] = ps[:k], pd[:k]
                        if it == bad_at:
                            d = d.copy(); d[int(rng.integers(0, n))] = V + 3   # csr.hpp:67-72: the whole batch is rejected
                        ds, dd = dev(s), dev(d)
                        keep.append((ds, dd))
                        try:
                            (g.submit_insert_pairs if kind == "insert" else g.submit_delete_pairs)(ds, dd)
                        except DataError:
                            failed = reported = True
                            break
                        if it == bad_at:
                            failed = True   # (reported by a later submit or by the flush; nothing behind it may run)
                        elif not failed:
                            (o.insert_pairs if kind == "insert" else o.delete_pairs)(s, d)
                            applied_expect += 1
                            if kind == "insert":
                                log.append((s, d))
                    try:
                        n_applied = g.flush()
                    except DataError:
                        reported = True
                        n_applied = g.flush()
                    assert reported == failed, "a rejected batch was not reported (or a good stream was)"
                    assert n_applied == applied_expect, f"applied {n_applied} != {applied_expect}"
                    assert g.active_edges() == o.active_edges(), "active edges"
                    assert np.array_equal(np.asarray(g.degrees()), np.asarray(o.degrees())), "degrees"
                ga, oa = g.export_csr(), o.export_csr()
                assert np.array_equal(ga[0], oa[0]) and np.array_equal(ga[1], oa[1]), "adjacency"
            except (AssertionError, EngineError) as e:
                fails += 1
                print(f"FAIL submit seed={seed} V={V} B={B} grow={grow}: {str(e)[:200]}", flush=True)
            finally:
                g.close(); o.close()
        print(f"stress_parity --submit: {a.seeds} seeds, {fails} failures, {time.time() - t0:.0f} s")
        return 1 if fails else 0
    if a.hubs:
        for seed in range(a.first, a.first + a.seeds):
            rng = np.random.default_rng(seed)
            V = int(rng.choice([50, 700, 5000, 40000]))
            B = int(rng.choice([32, 32, 32, 8, 33]))
            zipf = float(rng.choice([1.1, 1.3, 1.8]))
            script, log = [], []
            for it in range(int(rng.integers(4, 9))):
                n = int(rng.choice([50000, 150000, 400000]))
                s = (rng.zipf(zipf, n) % V).astype(np.uint32)
                d = rng.integers(0, V, n).astype(np.uint32)
                kind = "insert" if it < 2 or rng.random() < 0.55 else "delete"
                if kind == "delete":
                    ps, pd = log[int(rng.integers(0, len(log)))]
                    k = min(n, len(ps)) * 7 // 10
                    s[:k], d[:k] = ps[:k], pd[:k]
                else:
                    log.append((s, d))
                if rng.integers(0, 3) == 0:
                    b = csr_from_pairs(BatchKind.Insert if kind == "insert" else BatchKind.Delete, V, s, d)
                    script.append((kind + "_csr", b.offsets, b.destinations))
                else:
                    script.append((kind, s, d))
                script.append(("check",))
            qs, qd = log[0][0][:20000].copy(), log[0][1][:20000].copy()
            qd[::3] = rng.integers(0, V, len(qd[::3])).astype(np.uint32)
            script.append(("query", qs, qd))
            grow = bool(rng.integers(0, 2))
            g = GpuGraph.__new__(GpuGraph)
            g.g = DynamicGraph(GraphConfig(pool_blocks=(256 if grow else 1 << 19), pool_max_blocks=(1 << 20 if grow else 0),
                                           group=str(rng.choice(["auto", "radix", "count"]))), V, B)
            o = CpuGraph(orc, "orc", V, B, 4 << 30, 0.5, True, 1)
            try:
                assert_same(run_script(g, script), run_script(o, script), f"hub seed {seed}")
            except AssertionError as e:
                fails += 1
                print(f"FAIL hub seed={seed} V={V} B={B} zipf={zipf} grow={grow}: {str(e)[:200]}", flush=True)
            finally:
                g.close(); o.close()
        print(f"stress_parity --hubs: {a.seeds} seeds, {fails} failures, {time.time() - t0:.0f} s")
        return 1 if fails else 0
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
