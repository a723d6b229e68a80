"""Test drivers: one interface over the three implementations.

  CpuGraph(lib, prefix)  — oracle/liboracle.so (prefix "orc", the C restatement)
                           or oracle/_ref/libdyngraph_ref.so (prefix "ref", the
                           unmodified reference headers behind oracle/ref_shim.cpp)
  GpuGraph               — the product, through paper_2306_08252_b200 (C ABI)

`run_script` applies one op script to any of them and returns everything the
reference's oracle_compare (oracle.hpp:98-163) looks at, so parity is a
dictionary comparison.  TEST INFRASTRUCTURE: only tests/, smoke() and the
bench's cpu_baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"
ORACLE_SO = ORACLE_DIR / "liboracle.so"
REF_SO = ORACLE_DIR / "_ref" / "libdyngraph_ref.so"

_vp = C.c_void_p


def build_oracle(force: bool = False):
    src = ORACLE_DIR / "dyngraph_oracle.c"
    if force or not ORACLE_SO.exists() or ORACLE_SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(ORACLE_DIR), "liboracle.so"], check=True, capture_output=True)
    return ORACLE_SO


def _bind(lib, prefix: str):
    sig = {
        "create": (_vp, [C.c_uint64, C.c_double, C.c_int, C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(C.c_int)]),
        "destroy": (None, [_vp]),
        "last_error": (C.c_char_p, [_vp]),
        "insert_csr": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_uint64]),
        "delete_csr": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_uint64]),
        "insert_coo": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.POINTER(C.c_double)]),
        "delete_coo": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.POINTER(C.c_double)]),
        "query": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _vp]),
        "insert_vertices": (C.c_int, [_vp, C.c_uint64]),
        "delete_vertices": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.POINTER(C.c_uint64)]),
        "block_size": (C.c_uint32, [_vp]),
        "logical_size": (C.c_uint64, [_vp]),
        "vertex_capacity": (C.c_uint64, [_vp]),
        "alive_vertices": (C.c_uint64, [_vp]),
        "active_edges": (C.c_uint64, [_vp]),
        "vertex_alive": (C.c_int, [_vp, C.c_uint32]),
        "queue_size": (C.c_uint64, [_vp]),
        "blocks_in_use": (C.c_uint64, [_vp]),
        "degrees": (C.c_int, [_vp, _vp]),
        "export_csr": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int]),
        "digest": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "plan_batch": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_uint64, _vp, _vp, _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, f"{prefix}_{name}")
        fn.restype, fn.argtypes = res, args
    return lib


def load_oracle():
    build_oracle()
    lib = _bind(C.CDLL(str(ORACLE_SO)), "orc")
    lib.orc_gen_rmat.restype = None
    lib.orc_gen_rmat.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp]
    lib.orc_synth_uniform_pairs.restype = None
    lib.orc_synth_uniform_pairs.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp]
    return lib


def load_ref():
    if not REF_SO.exists():
        return None
    lib = _bind(C.CDLL(str(REF_SO)), "ref")
    lib.ref_synth_uniform_pairs.restype = C.c_int
    lib.ref_synth_uniform_pairs.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp]
    lib.ref_compute_block_size_coo.restype = C.c_int
    lib.ref_compute_block_size_coo.argtypes = [C.c_uint64, _vp, _vp, C.c_uint64, C.POINTER(C.c_uint32)]
    return lib


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _u32(x):
    return np.ascontiguousarray(x, dtype=np.uint32)


class CpuGraph:
    """Oracle restatement ("orc") or the real reference ("ref") behind one interface."""

    def __init__(self, lib, prefix, v0, block_size, arena_bytes=8 << 30, initial_fraction=0.5,
                 reclaim=True, workers=1):
        self.lib, self.pfx = lib, prefix
        err = C.c_int()
        self.h = self._f("create")(arena_bytes, initial_fraction, int(reclaim), workers, v0, block_size, C.byref(err))
        self.create_rc = err.value
        if not self.h:
            raise RuntimeError(f"create failed rc={err.value}: {self._f('last_error')(None).decode()}")

    def _f(self, name):
        return getattr(self.lib, f"{self.pfx}_{name}")

    def close(self):
        if self.h:
            self._f("destroy")(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # ops return the status code (0 / 2 / 3)
    def insert_pairs(self, src, dst, seconds=None):
        s, d = _u32(src), _u32(dst)
        return self._f("insert_coo")(self.h, _p(s), _p(d), len(s), seconds)

    def delete_pairs(self, src, dst, seconds=None):
        s, d = _u32(src), _u32(dst)
        return self._f("delete_coo")(self.h, _p(s), _p(d), len(s), seconds)

    def insert_csr(self, offsets, dsts):
        o, d = np.ascontiguousarray(offsets, np.uint64), _u32(dsts)
        return self._f("insert_csr")(self.h, _p(o), len(o), _p(d), len(d))

    def delete_csr(self, offsets, dsts):
        o, d = np.ascontiguousarray(offsets, np.uint64), _u32(dsts)
        return self._f("delete_csr")(self.h, _p(o), len(o), _p(d), len(d))

    def plan_batch(self, offsets, dsts):
        """(rc, blocks_required, prefix_sum, space_remaining) of plan_batch (graph.hpp:135-160)"""
        o, d = np.ascontiguousarray(offsets, np.uint64), _u32(dsts)
        n = max(len(o) - 1, 0)
        req, pre, space = np.zeros(n, np.uint64), np.zeros(n, np.uint64), np.zeros(n, np.uint32)
        rc = self._f("plan_batch")(self.h, _p(o), len(o), _p(d), len(d), _p(req), _p(pre), _p(space))
        return rc, req, pre, space

    def query(self, src, dst):
        s, d = _u32(src), _u32(dst)
        out = np.zeros(len(s), np.uint8)
        self._f("query")(self.h, _p(s), _p(d), len(s), _p(out))
        return out

    def insert_vertices(self, count):
        return self._f("insert_vertices")(self.h, count)

    def delete_vertices(self, ids):
        a = _u32(ids)
        sk = np.zeros(max(1, len(a)), np.uint32)
        ns = C.c_uint64()
        rc = self._f("delete_vertices")(self.h, _p(a), len(a), _p(sk), C.byref(ns))
        return rc, [int(x) for x in sk[: ns.value]]

    def logical_size(self): return int(self._f("logical_size")(self.h))
    def vertex_capacity(self): return int(self._f("vertex_capacity")(self.h))
    def alive_vertices(self): return int(self._f("alive_vertices")(self.h))
    def active_edges(self): return int(self._f("active_edges")(self.h))
    def block_size(self): return int(self._f("block_size")(self.h))
    def queue_size(self): return int(self._f("queue_size")(self.h))
    def blocks_in_use(self): return int(self._f("blocks_in_use")(self.h))
    def vertex_alive(self, v): return bool(self._f("vertex_alive")(self.h, v))
    def last_error(self): return self._f("last_error")(self.h).decode()

    def alive_vector(self):
        n = self.logical_size()
        return np.array([self._f("vertex_alive")(self.h, v) for v in range(n)], dtype=np.uint8)

    def degrees(self):
        out = np.zeros(self.logical_size(), np.uint64)
        self._f("degrees")(self.h, _p(out))
        return out

    def digest(self):
        """(sum over live entries of mix64(v << 32 | dst), live entries) -- the twin of DynamicGraph.digest()"""
        d, n = C.c_uint64(), C.c_uint64()
        assert self._f("digest")(self.h, C.byref(d), C.byref(n)) == 0
        return int(d.value), int(n.value)

    def export_csr(self, sorted=True):
        n = self.logical_size()
        off = np.zeros(n + 1, np.uint64)
        self._f("export_csr")(self.h, _p(off), None, 0, int(sorted))
        d = np.zeros(int(off[n]), np.uint32)
        self._f("export_csr")(self.h, _p(off), _p(d) if len(d) else None, len(d), int(sorted))
        return off, d


class GpuGraph:
    """The product behind the same interface (status codes instead of exceptions)."""

    def __init__(self, v0, block_size, pool_blocks=1 << 16, reclaim=True, group="auto", **_):
        from paper_2306_08252_b200 import DynamicGraph, GraphConfig
        self.g = DynamicGraph(GraphConfig(pool_blocks=pool_blocks, reclaim_on_delete=reclaim, group=group),
                              v0, block_size)

    def close(self):
        self.g.close()

    def _rc(self, fn, *a):
        from paper_2306_08252_b200 import DataError, EngineError
        try:
            fn(*a)
            return 0
        except DataError:
            return 2
        except EngineError:
            return 3

    def insert_pairs(self, src, dst, seconds=None): return self._rc(self.g.insert_pairs, _u32(src), _u32(dst))
    def delete_pairs(self, src, dst, seconds=None): return self._rc(self.g.delete_pairs, _u32(src), _u32(dst))

    def insert_csr(self, offsets, dsts):
        from paper_2306_08252_b200 import BatchKind, CsrBatch
        return self._rc(self.g.insert_batch, CsrBatch(BatchKind.Insert, np.asarray(offsets, np.uint64), _u32(dsts)))

    def delete_csr(self, offsets, dsts):
        from paper_2306_08252_b200 import BatchKind, CsrBatch
        return self._rc(self.g.delete_batch, CsrBatch(BatchKind.Delete, np.asarray(offsets, np.uint64), _u32(dsts)))

    def query(self, src, dst): return self.g.query_edges(_u32(src), _u32(dst))
    def insert_vertices(self, count): return self._rc(self.g.insert_vertices, count)
    def delete_vertices(self, ids): return 0, self.g.delete_vertices(_u32(ids))
    def logical_size(self): return self.g.logical_size()
    def vertex_capacity(self): return self.g.vertex_capacity()
    def alive_vertices(self): return self.g.alive_vertices()
    def active_edges(self): return self.g.active_edges()
    def block_size(self): return self.g.block_size()
    def vertex_alive(self, v): return self.g.vertex_alive(v)
    def queue_size(self): return self.g.stats()["pool_queue_size"]
    def blocks_in_use(self): return self.g.stats()["pool_blocks_in_use"]
    def alive_vector(self):
        return np.array([self.g.vertex_alive(v) for v in range(self.g.logical_size())], dtype=np.uint8)
    def degrees(self): return self.g.degrees()
    def export_csr(self, sorted=True): return self.g.export_csr(sorted=sorted)


def canonical_state(g) -> dict:
    """What oracle_compare looks at (oracle.hpp:98-163), as plain arrays."""
    off, dst = g.export_csr(sorted=True)
    return {
        "logical_size": g.logical_size(),
        "capacity": g.vertex_capacity(),
        "alive_vertices": g.alive_vertices(),
        "active_edges": g.active_edges(),
        "alive": g.alive_vector(),
        "degrees": np.asarray(g.degrees(), np.uint64),
        "offsets": np.asarray(off, np.uint64),
        "destinations": np.asarray(dst, np.uint32),
    }


def run_script(g, script) -> dict:
    """Apply an op script; returns per-op observations + the final canonical state."""
    obs = []
    for op in script:
        kind = op[0]
        if kind == "insert":
            obs.append(("rc", g.insert_pairs(op[1], op[2])))
        elif kind == "delete":
            obs.append(("rc", g.delete_pairs(op[1], op[2])))
        elif kind == "insert_csr":
            obs.append(("rc", g.insert_csr(op[1], op[2])))
        elif kind == "delete_csr":
            obs.append(("rc", g.delete_csr(op[1], op[2])))
        elif kind == "add_vertices":
            obs.append(("rc", g.insert_vertices(op[1])))
        elif kind == "del_vertices":
            rc, skipped = g.delete_vertices(op[1])
            obs.append(("skipped", tuple(skipped)))
        elif kind == "query":
            obs.append(("answers", np.asarray(g.query(op[1], op[2]), np.uint8).tobytes()))
        elif kind == "check":
            obs.append(("edges", g.active_edges(), g.logical_size(), g.alive_vertices()))
        else:
            raise ValueError(kind)
    return {"obs": obs, "state": canonical_state(g)}


def assert_same(a: dict, b: dict, what=""):
    assert len(a["obs"]) == len(b["obs"]), what
    for i, (x, y) in enumerate(zip(a["obs"], b["obs"])):
        assert x == y, f"{what}: op {i} differs: {x[:2]} vs {y[:2]}"
    sa, sb = a["state"], b["state"]
    for k in ("logical_size", "capacity", "alive_vertices", "active_edges"):
        assert sa[k] == sb[k], f"{what}: {k}: {sa[k]} vs {sb[k]}"
    for k in ("alive", "degrees", "offsets", "destinations"):
        assert np.array_equal(sa[k], sb[k]), f"{what}: {k} differs"
