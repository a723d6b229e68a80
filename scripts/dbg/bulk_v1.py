import numpy as np, sys
sys.path.insert(0, ".")
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, BatchKind, CsrBatch
V = 1
off = np.array([0, 32], np.uint64)
dst = np.zeros(32, np.uint32)
g = DynamicGraph(GraphConfig(pool_blocks=4096), V, 32)
for bad_at in [0, 31, 16, 0]:
    bad = dst.copy(); bad[bad_at] = 10
    try:
        g.insert_batch(CsrBatch(BatchKind.Insert, off, bad))
        print("accepted?!")
    except Exception as e:
        print("rejected:", e, g.stats()["queue_front"], g.active_edges())
try:
    g.insert_batch(CsrBatch(BatchKind.Insert, off, dst))
    print("good ok", g.active_edges())
except Exception as e:
    print("good rejected:", e)
