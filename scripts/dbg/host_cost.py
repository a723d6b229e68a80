"""Host cost of one submitted op (no blocking: bursts of 6 ops after a flush)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat
scale, b = 22, 1_000_000
V, E = 1 << scale, 16 << scale
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
with torch.cuda.stream(stream):
    g = DynamicGraph(GraphConfig(device=0, pool_blocks=int((E // 32 + V) * 1.25) + 4096 + 125000, stream=stream.cuda_stream), V, 32)
    src = torch.empty(E, dtype=torch.int32, device=dev); dst = torch.empty(E, dtype=torch.int32, device=dev)
    thr = rmat.thresholds()
    g.gen_rmat(scale, 1, 0, src, dst, thr)
    off = torch.empty(V + 1, dtype=torch.int64, device=dev); out = torch.empty(E, dtype=torch.int32, device=dev)
    g.coo_to_csr(src, dst, V, off, out)
    g.bulk_init(off, out)
    bs = []
    for i in range(6):
        s = torch.empty(b, dtype=torch.int32, device=dev); d = torch.empty(b, dtype=torch.int32, device=dev)
        g.gen_rmat(scale, 2, i * b, s, d, thr)
        bs.append((s, d))
    for s, d in bs[:2]:
        g.insert_pairs(s, d); g.delete_pairs(s, d)
    ti, td = [], []
    for rep in range(10):
        g.flush(); torch.cuda.synchronize()
        for i in range(3):
            s, d = bs[i]
            t0 = time.perf_counter(); g.submit_insert_pairs(s, d); t1 = time.perf_counter(); g.submit_delete_pairs(s, d); t2 = time.perf_counter()
            ti.append((t1 - t0) * 1e6); td.append((t2 - t1) * 1e6)
    g.flush()
    print("submit insert host us: median %.1f min %.1f" % (np.median(ti), min(ti)))
    print("submit delete host us: median %.1f min %.1f" % (np.median(td), min(td)))
    t0 = time.perf_counter()
    for _ in range(1000): g.pending_ops()
    print("ctypes call us: %.2f" % ((time.perf_counter() - t0) * 1e3))
