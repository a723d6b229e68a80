import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat
scale, b, K = 22, 1_000_000, 6
V, E = 1 << scale, 16 << scale
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
copy_stream = torch.cuda.Stream(device=dev)
with torch.cuda.stream(stream):
    g = DynamicGraph(GraphConfig(device=0, pool_blocks=int((E // 32 + V) * 1.25) + 4096 + 125000, stream=stream.cuda_stream), V, 32)
    src = torch.empty(E, dtype=torch.int32, device=dev); dst = torch.empty(E, dtype=torch.int32, device=dev)
    thr = rmat.thresholds()
    g.gen_rmat(scale, 1, 0, src, dst, thr)
    off = torch.empty(V + 1, dtype=torch.int64, device=dev); out = torch.empty(E, dtype=torch.int32, device=dev)
    g.coo_to_csr(src, dst, V, off, out); g.bulk_init(off, out)
    del src, dst
    bs = []
    for i in range(K):
        s = torch.empty(b, dtype=torch.int32, device=dev); d = torch.empty(b, dtype=torch.int32, device=dev)
        g.gen_rmat(scale, 2, i * b, s, d, thr); bs.append((s, d))
    stream.synchronize()
    hbuf = torch.empty(2 * b, dtype=torch.int32).pin_memory()
    dbuf = torch.empty(2 * b, dtype=torch.int32, device=dev)
    for with_copies in (False, True):
        print("copies beside:", with_copies, file=sys.stderr, flush=True)
        for i in range(K):
            g.insert_pairs(*bs[i])
            torch.cuda.synchronize()
            if with_copies:
                with torch.cuda.stream(copy_stream):
                    for _ in range(3):
                        dbuf.copy_(hbuf, non_blocking=True)
            g.delete_pairs(*bs[i])
            torch.cuda.synchronize()
