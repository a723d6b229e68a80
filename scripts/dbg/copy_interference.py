"""Do H2D copies and the update kernels slow each other down?  Device-resident submitted steps with and without an
independent stream of pinned H2D copies beside them."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat
scale, b, K = 22, 1_000_000, 20
V, E = 1 << scale, 16 << scale
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
copy_stream = torch.cuda.Stream(device=dev)
with torch.cuda.stream(stream):
    g = DynamicGraph(GraphConfig(device=0, pool_blocks=int((E // 32 + V) * 1.25) + 4096 + 125000, stream=stream.cuda_stream,
                                 submit_inputs_ready=True), V, 32)
    src = torch.empty(E, dtype=torch.int32, device=dev); dst = torch.empty(E, dtype=torch.int32, device=dev)
    thr = rmat.thresholds()
    g.gen_rmat(scale, 1, 0, src, dst, thr)
    off = torch.empty(V + 1, dtype=torch.int64, device=dev); out = torch.empty(E, dtype=torch.int32, device=dev)
    g.coo_to_csr(src, dst, V, off, out); g.bulk_init(off, out)
    del src, dst
    bs = []
    for i in range(K + 3):
        s = torch.empty(b, dtype=torch.int32, device=dev); d = torch.empty(b, dtype=torch.int32, device=dev)
        g.gen_rmat(scale, 2, i * b, s, d, thr); bs.append((s, d))
    stream.synchronize()
    for i in range(3):
        g.insert_pairs(*bs[i]); g.delete_pairs(*bs[i])
    hbuf = torch.empty(2 * b, dtype=torch.int32).pin_memory()
    dbuf = torch.empty(2 * b, dtype=torch.int32, device=dev)
    for with_copies in (False, True, False, True):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if with_copies:
            with torch.cuda.stream(copy_stream):
                c0.record(copy_stream)
                for _ in range(2 * K):
                    dbuf.copy_(hbuf, non_blocking=True)
                c1.record(copy_stream)
        for i in range(3, 3 + K):
            g.submit_insert_pairs(*bs[i]); g.submit_delete_pairs(*bs[i])
        g.flush()
        e1.record(stream); e1.synchronize(); torch.cuda.synchronize()
        msg = f"copies beside: {with_copies}  compute {e0.elapsed_time(e1) / K:.3f} ms/step"
        if with_copies:
            msg += f"   copies {c0.elapsed_time(c1) / K:.3f} ms per 16 MB = {2 * K * 8 * b / (c0.elapsed_time(c1) * 1e-3) / 1e9:.1f} GB/s"
        print(msg, flush=True)

    # which op suffers?  inserts only / deletes only (the other half outside the timed region)
    for kind in ("insert", "delete"):
        for with_copies in (False, True):
            tot = 0.0
            for i in range(3, 3 + K):
                if kind == "delete":
                    g.insert_pairs(*bs[i])
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if with_copies:
                    with torch.cuda.stream(copy_stream):
                        for _ in range(3):
                            dbuf.copy_(hbuf, non_blocking=True)
                e0.record(stream)
                (g.submit_insert_pairs if kind == "insert" else g.submit_delete_pairs)(*bs[i])
                e1.record(stream); g.flush(); e1.synchronize(); torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
                if kind == "insert":
                    g.delete_pairs(*bs[i])
            print(f"{kind} alone, copies beside: {with_copies}  {tot / K * 1e3:.0f} us per op", flush=True)
