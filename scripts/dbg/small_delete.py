import sys, time, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat
scale = 20
V, E = 1 << scale, 16 << scale
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
with torch.cuda.stream(stream):
    g = DynamicGraph(GraphConfig(device=0, pool_blocks=int((E // 32 + V) * 1.5), stream=stream.cuda_stream), V, 32)
    src = torch.empty(E, dtype=torch.int32, device=dev); dst = torch.empty(E, dtype=torch.int32, device=dev)
    thr = rmat.thresholds()
    g.gen_rmat(scale, 1, 0, src, dst, thr)
    g.insert_pairs(src, dst)
    for n in (1000, 10000, 100000):
        hs = np.empty(n, np.uint32); hd = np.empty(n, np.uint32)
        lat_i, lat_d = [], []
        for i in range(30):
            s = torch.empty(n, dtype=torch.int32, device=dev); d = torch.empty(n, dtype=torch.int32, device=dev)
            g.gen_rmat(scale, 7 + n, i * n, s, d, thr)
            hs[:] = s.cpu().numpy().view(np.uint32); hd[:] = d.cpu().numpy().view(np.uint32)
            stream.synchronize()
            t = time.perf_counter(); g.insert_pairs(hs, hd); lat_i.append((time.perf_counter() - t) * 1e6)
            t = time.perf_counter(); g.delete_pairs(hs, hd); lat_d.append((time.perf_counter() - t) * 1e6)
        print(n, "insert p50 %.0f us  delete p50 %.0f us  (%d launches)" % (np.median(lat_i), np.median(lat_d), g.last_op_report()["kernel_launches"]), flush=True)
