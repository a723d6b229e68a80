"""Regenerates tests/golden/*.npz by running the UNMODIFIED reference
(oracle/_ref/libdyngraph_ref.so, built from /root/reference/proj/include by
oracle/Makefile).  Run in the build container only:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures hold the op scripts AND the reference's observations (status
codes, skipped ids, query answers, final canonical state), so they pin both
the oracle restatement (CPU tests) and the CUDA path (GPU tests) without
/root/reference being present.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from tests.drivers import CpuGraph, load_ref, run_script  # noqa: E402
from tests.golden_io import save_cases  # noqa: E402
from tests.workloads import make_workload  # noqa: E402
from tests.known_answers import KNOWN_ANSWER_SCRIPTS  # noqa: E402

OUT = Path(__file__).resolve().parent


IO_SYNTH = [(0, 100, 500, 42), (1, 100, 500, 42), (1, 4096, 20000, 7), (0, 64, 300, 5)]
IO_BATCHES = [(3, 0, 3, 0, 1), (3, 7, 3, 1, 3), (2, 0, 2, 1, 9), (0, 13, 0, 1, 42)]   # (synth idx, batch, -, shuffled, seed)
# (kind, V, E, seed, batch, ops, shuffled, block_size, query_sample, arena_bytes)
IO_RUNS = [(0, 64, 512, 1, 100, 2, 0, 0, 200, 1 << 20), (1, 256, 3000, 7, 0, 1, 0, 0, 101, 1 << 22),
           (0, 500, 4000, 3, 333, 0, 1, 4, 64, 1 << 22), (1, 1000, 10000, 11, 1000, 2, 1, 0, 1000, 1 << 24)]


def make_io_golden(ref):
    """io-side goldens (io/synthetic.hpp, io/batching.hpp, io/workload.hpp) from the reference itself."""
    import ctypes as C
    vp = C.c_void_p
    ref.ref_make_batches_flat.restype = C.c_longlong
    out = {}
    synth = []
    for i, (kind, v, e, seed) in enumerate(IO_SYNTH):
        off = np.zeros(v + 1, np.uint64); dst = np.zeros(e, np.uint32)
        assert ref.ref_synth_csr(kind, C.c_uint64(v), C.c_uint64(e), C.c_uint64(seed), vp(off.ctypes.data), vp(dst.ctypes.data)) == 0
        out[f"synth{i}_off"], out[f"synth{i}_dst"] = off, dst
        synth.append((v, off, dst))
    for i, (si, batch, _, shuffled, seed) in enumerate(IO_BATCHES):
        v, off, dst = synth[si]
        e = dst.size
        so = np.zeros(e, np.uint32); do = np.zeros(e, np.uint32); sizes = np.zeros(e + 1, np.uint64)
        nb = ref.ref_make_batches_flat(C.c_uint64(v), vp(off.ctypes.data), vp(dst.ctypes.data), C.c_uint64(e), C.c_uint64(batch),
                                       shuffled, C.c_uint64(seed), vp(so.ctypes.data), vp(do.ctypes.data), vp(sizes.ctypes.data))
        assert nb > 0
        out[f"batch{i}_src"], out[f"batch{i}_dst"], out[f"batch{i}_sizes"] = so, do, sizes[:nb]
    for i, (kind, v, e, seed, batch, ops, shuffled, bs, qn, arena) in enumerate(IO_RUNS):
        res = np.zeros(8, np.uint64); ph = C.create_string_buffer(1 << 16)
        rc = ref.ref_run_workload_synth(kind, C.c_uint64(v), C.c_uint64(e), C.c_uint64(seed), C.c_uint64(batch), ops, shuffled,
                                        C.c_uint32(bs), C.c_uint64(qn), C.c_uint64(arena), vp(res.ctypes.data), ph, C.c_uint64(1 << 16))
        assert rc == 0, rc
        out[f"run{i}_res"] = res
        out[f"run{i}_phases"] = np.frombuffer(ph.value, dtype=np.uint8).copy()
    np.savez_compressed(OUT / "ref_io.npz", **out)


def main():
    ref = load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref/libdyngraph_ref.so missing: run `make -C oracle ref` first")
    cases = []
    for seed in range(1000, 1024):
        cfg, script = make_workload(seed, max_vertices=1024, max_edges=4000, max_insert=600)
        g = CpuGraph(ref, "ref", cfg["v0"], cfg["block_size"], cfg["arena_bytes"],
                     cfg["initial_fraction"], cfg["reclaim"], cfg["workers"])
        cases.append({"cfg": cfg, "script": script, "expect": run_script(g, script)})
        g.close()
    save_cases(OUT / "ref_workloads.npz", cases)
    ka = []
    for name, cfg, script in KNOWN_ANSWER_SCRIPTS:
        g = CpuGraph(ref, "ref", cfg["v0"], cfg["block_size"], cfg.get("arena_bytes", 1 << 20),
                     cfg.get("initial_fraction", 0.5), cfg.get("reclaim", True), 1)
        c = dict(cfg)
        c["name"] = name
        ka.append({"cfg": c, "script": script, "expect": run_script(g, script)})
        g.close()
    save_cases(OUT / "ref_known_answers.npz", ka)
    # config-1 input checksum: synth_uniform(65536, 1000000, 0xbeef) (acceptance_test.cpp:241)
    import ctypes as C
    s = np.zeros(1000000, np.uint32); d = np.zeros(1000000, np.uint32)
    ref.ref_synth_uniform_pairs(65536, 1000000, 0xBEEF, C.c_void_p(s.ctypes.data), C.c_void_p(d.ctypes.data))
    # the COO restatement must be the reference's own graph: same CSR as dyngraph::io::synth_uniform
    off = np.zeros(65537, np.uint64); dd = np.zeros(1000000, np.uint32)
    assert ref.ref_synth_csr(0, C.c_uint64(65536), C.c_uint64(1000000), C.c_uint64(0xBEEF), C.c_void_p(off.ctypes.data),
                             C.c_void_p(dd.ctypes.data)) == 0
    order = np.argsort(s, kind="stable")
    assert np.array_equal(dd, d[order]) and np.array_equal(np.diff(off.astype(np.int64)), np.bincount(s, minlength=65536))
    np.savez_compressed(OUT / "synth_uniform_beef.npz", head_src=s[:64], head_dst=d[:64],
                        sum_src=np.uint64(s.astype(np.uint64).sum()), sum_dst=np.uint64(d.astype(np.uint64).sum()),
                        xor_src=np.bitwise_xor.reduce(s), xor_dst=np.bitwise_xor.reduce(d))
    make_io_golden(ref)
    print("wrote", [p.name for p in OUT.glob("*.npz")])


if __name__ == "__main__":
    main()
