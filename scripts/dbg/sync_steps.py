"""Per-step device time of the synchronous calls, first and second pass over the same batches."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat
scale, b, K = 22, 1_000_000, 8
V, E = 1 << scale, 16 << scale
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
with torch.cuda.stream(stream):
    g = DynamicGraph(GraphConfig(device=0, pool_blocks=int((E // 32 + V) * 1.25) + 4096 + 125000, stream=stream.cuda_stream,
                                 workspace_bytes=48 * V + 8 * (E // 32) + (64 << 20)), V, 32)
    src = torch.empty(E, dtype=torch.int32, device=dev); dst = torch.empty(E, dtype=torch.int32, device=dev)
    thr = rmat.thresholds()
    g.gen_rmat(scale, 1, 0, src, dst, thr)
    off = torch.empty(V + 1, dtype=torch.int64, device=dev); out = torch.empty(E, dtype=torch.int32, device=dev)
    g.coo_to_csr(src, dst, V, off, out)
    g.bulk_init(off, out)
    del src, dst
    bs = []
    for i in range(K):
        s = torch.empty(b, dtype=torch.int32, device=dev); d = torch.empty(b, dtype=torch.int32, device=dev)
        g.gen_rmat(scale, 2, i * b, s, d, thr); bs.append((s, d))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    import os
    for p in range(3):
        if os.environ.get("PROF"):
            g.profile_enable(True)
        row = []
        for i in range(K):
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream); g.insert_pairs(*bs[i]); e[1].record(stream); g.delete_pairs(*bs[i]); e[2].record(stream); e[2].synchronize()
            row.append((round(e[0].elapsed_time(e[1]) * 1e3), round(e[1].elapsed_time(e[2]) * 1e3)))
        if os.environ.get("PROF"):
            g.profile_enable(False)
            rep = g.profile_report()
            print("   ", {k: round(ms / n * 1e3, 1) for k, (ms, n) in sorted(rep.items(), key=lambda kv: -kv[1][0])[:16]})
        print("pass", p, row, "ws MB", g.memory()["workspace_bytes"] >> 20, flush=True)
