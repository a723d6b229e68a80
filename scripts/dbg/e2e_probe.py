"""Where does the e2e step time go?  Same stream of host batches through the ingest queue with different depths,
and the same ops submitted from DEVICE batches (no copies) in one timed region."""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat, csr_from_pairs, BatchKind
scale, b, K, W = 22, 1_000_000, 20, 3
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
    del src, dst
    batches, host = [], []
    for i in range(K + W):
        s = torch.empty(b, dtype=torch.int32, device=dev); d = torch.empty(b, dtype=torch.int32, device=dev)
        g.gen_rmat(scale, 2, i * b, s, d, thr)
        batches.append((s, d))
        hs = torch.empty(b, dtype=torch.int32).pin_memory(); hd = torch.empty(b, dtype=torch.int32).pin_memory()
        hs.copy_(s); hd.copy_(d)
        host.append((hs.numpy().view(np.uint32), hd.numpy().view(np.uint32)))
    stream.synchronize()
    def timed(fn, label):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record(stream)
        t_host = fn()
        e1.record(stream); e1.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        print(f"{label:44s} device {e0.elapsed_time(e1) / K:.3f} ms/step  wall {wall / K:.3f} ms/step  host-enqueue {t_host / K:.3f} ms/step", flush=True)
    def dev_submit():
        t0 = time.perf_counter()
        for i in range(W, W + K):
            s, d = batches[i]
            g.submit_insert_pairs(s, d); g.submit_delete_pairs(s, d)
        th = (time.perf_counter() - t0) * 1e3
        g.flush()
        return th
    for i in range(W):
        g.insert_pairs(*batches[i]); g.delete_pairs(*batches[i])
    timed(dev_submit, "device batches, submitted, one region")
    timed(dev_submit, "device batches, submitted, one region")
    for depth in (2, 3, 4, 6):
        q = g.ingest(b, depth=depth)
        def run():
            t0 = time.perf_counter()
            for i in range(W, W + K):
                hs, hd = host[i]
                q.submit("insert", hs, hd); q.submit("delete", hs, hd)
            th = (time.perf_counter() - t0) * 1e3
            q.flush()
            return th
        run()
        timed(run, f"host batches, ingest depth {depth}")
        q.close()
    # raw H2D rate
    t = torch.empty(b, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(40):
        t.copy_(torch.from_numpy(host[i % len(host)][0].view(np.int32)), non_blocking=True)
    e1.record(stream); e1.synchronize()
    print(f"raw H2D: {40 * 4 * b / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
