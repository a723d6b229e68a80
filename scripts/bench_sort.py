#!/usr/bin/env python
"""Radix-sort pass timing: dg_coo_to_csr over an R-MAT edge list (pack + ceil(scale / 8) Onesweep passes).
    python scripts/bench_sort.py [scale] [edge_factor]"""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 16
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
with torch.cuda.stream(stream):
    V, E = 1 << scale, ef << scale
    g = DynamicGraph(GraphConfig(device=0, pool_blocks=1024, stream=stream.cuda_stream), 1, 1)
    src = torch.empty(E, dtype=torch.int32, device=dev); dst = torch.empty(E, dtype=torch.int32, device=dev)
    g.gen_rmat(scale, 1, 0, src, dst, rmat.thresholds())
    off = torch.empty(V + 1, dtype=torch.int64, device=dev); out = torch.empty(E, dtype=torch.int32, device=dev)
    for _ in range(2):
        g.coo_to_csr(src, dst, V, off, out)
    g.profile_enable(True)
    for _ in range(3):
        g.coo_to_csr(src, dst, V, off, out)
    g.profile_enable(False)
    rep = g.profile_report()
    for k, (ms, n) in sorted(rep.items(), key=lambda kv: -kv[1][0]):
        line = f"{k:32s} {ms / n * 1e3:9.1f} us/launch x{n}"
        if k.startswith("sort_pass"):
            line += f"   {16 * E / (ms / n * 1e-3) / 1e9:7.0f} GB/s = {16 * E / (ms / n * 1e-3) / 1e9 / peak:.2f} of measured HBM peak ({E} keys)"
        print(line)
    # stable grouping check against torch
    o = off.cpu().numpy(); d = out.cpu().numpy()
    s_cpu, d_cpu = src.cpu().numpy(), dst.cpu().numpy()
    import numpy as np
    order = np.argsort(s_cpu.view(np.uint32), kind="stable")
    assert np.array_equal(d, d_cpu[order]), "stable grouping mismatch"
    assert o[-1] == E
    print("stable order ok")
