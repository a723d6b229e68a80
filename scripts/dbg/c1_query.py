import sys, time, os
sys.path.insert(0, ".")
import numpy as np
from paper_2306_08252_b200 import BatchKind, DynamicGraph, GraphConfig, compute_block_size, csr_from_pairs
from paper_2306_08252_b200 import io as dio
V, E = 65536, 1000000
s, d = dio.synth_uniform_pairs(V, E, 0xBEEF)
base = csr_from_pairs(BatchKind.Insert, V, s, d)
rng = np.random.default_rng(0xBEEF)
pick = rng.integers(0, E, 50000)
qs = np.concatenate([s[pick], rng.integers(0, V, 50000).astype(np.uint32)])
qd = np.concatenate([d[pick], rng.integers(0, V, 50000).astype(np.uint32)])
for B in (15, 32):
    g = DynamicGraph(GraphConfig(pool_blocks=1 << 18), V, B)
    g.bulk_init(base.offsets, base.destinations)
    for rep in range(3):
        t = time.perf_counter(); a = g.query_edges(qs, qd); dt = (time.perf_counter() - t) * 1e3
        print("B", B, "query ms", round(dt, 3), "hits", int(np.asarray(a).sum()), g.last_op_report()["kernel_launches"], flush=True)
    g.profile_enable(True); g.query_edges(qs, qd); g.profile_enable(False)
    for k, (ms, n) in sorted(g.profile_report().items(), key=lambda kv: -kv[1][0])[:6]:
        print("   ", k, round(ms * 1e3, 1), "us x", n)
    g.close()
print("--- after 10 x 10K inserts (the bench_c1 sequence)")
us, ud = dio.synth_uniform_pairs(V, 100000, 0xBEEF + 1)
for rep in range(2):
    g = DynamicGraph(GraphConfig(pool_blocks=1 << 18), V, 15)
    g.bulk_init(base.offsets, base.destinations)
    for i in range(10):
        g.insert_pairs(us[i * 10000:(i + 1) * 10000], ud[i * 10000:(i + 1) * 10000])
    os.environ["X"] = "1"
    t = time.perf_counter(); a = g.query_edges(qs, qd); dt = (time.perf_counter() - t) * 1e3
    print("query ms", round(dt, 3), g.last_op_report(), flush=True)
    t = time.perf_counter(); a = g.query_edges(qs, qd); dt = (time.perf_counter() - t) * 1e3
    print("query again ms", round(dt, 3), flush=True)
    g.profile_enable(True); g.query_edges(qs, qd); g.profile_enable(False)
    for k, (ms, n) in sorted(g.profile_report().items(), key=lambda kv: -kv[1][0])[:4]:
        print("   ", k, round(ms * 1e3, 1), "us x", n)
    g.close()
