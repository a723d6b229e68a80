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
    np.savez_compressed(OUT / "synth_uniform_beef.npz", head_src=s[:64], head_dst=d[:64],
                        sum_src=np.uint64(s.astype(np.uint64).sum()), sum_dst=np.uint64(d.astype(np.uint64).sum()),
                        xor_src=np.bitwise_xor.reduce(s), xor_dst=np.bitwise_xor.reduce(d))
    print("wrote", [p.name for p in OUT.glob("*.npz")])


if __name__ == "__main__":
    main()
