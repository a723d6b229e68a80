"""Host-side mirror of the reference's operator API over the CUDA library.

`DynamicGraph` has the method names, argument meaning and error behaviour of
`class dyngraph::DynamicGraph` (proj/include/dyngraph/graph.hpp:80-317); every
method is a thin call through the C ABI (include/dyngraph_b200.h) into
hand-written sm_100a kernels.  Bulk arguments may be numpy arrays (host) or
CUDA torch tensors (device, used in place).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .csr import BatchKind, CsrBatch
from .errors import CudaError, DataError, EngineError, Error


@dataclass
class GraphConfig:
    """graph.hpp:23-28.  `pool_bytes`/`pool_blocks` replace arena_bytes * initial_fraction."""
    device: int = 0
    pool_bytes: int = 0          # 0 => library default (1 GiB)
    pool_blocks: int = 0         # exact block count; overrides pool_bytes
    reclaim_on_delete: bool = True
    stream: int = 0              # cudaStream_t handle; 0 => library-owned stream
    group: str = "auto"          # how COO batches are grouped by source: "auto" | "radix" | "count"
    # submit_*_pairs: the device arrays are complete when the call is made (nothing enqueued on the graph's stream
    # produces them), so an op's first kernel may start beside the previous op's last (DG_FLAG_SUBMIT_INPUTS_READY)
    submit_inputs_ready: bool = False
    auto_block_native: bool = False   # block_size 0: a computed size in [24, 48] becomes the native 32 (DG_FLAG_AUTO_BLOCK_NATIVE)
    workspace_bytes: int = 0     # per-op scratch reserved at construction (0 => grown on first use)
    # GrowthPolicy (block_pool.hpp:18-29): pool_max_blocks is the arena's role (0 => fixed pool)
    pool_max_blocks: int = 0
    trigger_fraction: float = 0.0   # 0 => 0.8
    growth_fraction: float = 0.0    # 0 => 0.25


def _is_device(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


class _Arg:
    """Keeps the backing array alive and exposes (pointer, mem-space)."""

    def __init__(self, x, dtype):
        if _is_device(x):
            import torch
            want = {np.uint32: (torch.int32, torch.uint32), np.uint64: (torch.int64, torch.uint64),
                    np.uint8: (torch.uint8,)}[dtype]
            if x.dtype not in want:
                raise DataError(f"device tensor must be one of {want}, got {x.dtype}")
            if not x.is_contiguous():
                x = x.contiguous()
            self.keep = x
            self.ptr = C.c_void_p(x.data_ptr())
            self.mem = _lib.DG_MEM_DEVICE
            self.n = x.numel()
        else:
            a = np.ascontiguousarray(x, dtype=dtype)
            self.keep = a
            self.ptr = C.c_void_p(a.ctypes.data)
            self.mem = _lib.DG_MEM_HOST
            self.n = a.size


@dataclass
class BatchPlan:
    """graph.hpp:33-39."""
    blocks_required: np.ndarray
    prefix_sum: np.ndarray
    space_remaining: np.ndarray

    def total_blocks(self) -> int:
        return int(self.prefix_sum[-1]) if len(self.prefix_sum) else 0


class DynamicGraph:
    def __init__(self, config: GraphConfig | None, initial_vertex_count: int, block_size: int):
        self._lib = _lib.load()
        cfg = config or GraphConfig()
        c = _lib.DgConfig()
        c.device = cfg.device
        c.flags = 0 if cfg.reclaim_on_delete else _lib.DG_FLAG_NO_RECLAIM
        c.flags |= {"auto": 0, "radix": _lib.DG_FLAG_GROUP_RADIX, "count": _lib.DG_FLAG_GROUP_COUNT}[cfg.group]
        if cfg.auto_block_native:
            c.flags |= _lib.DG_FLAG_AUTO_BLOCK_NATIVE
        if cfg.submit_inputs_ready:
            c.flags |= _lib.DG_FLAG_SUBMIT_INPUTS_READY
        c.pool_bytes = cfg.pool_bytes
        c.pool_blocks = cfg.pool_blocks
        c.stream = cfg.stream or None
        c.workspace_bytes = cfg.workspace_bytes
        c.pool_max_blocks = cfg.pool_max_blocks
        c.trigger_fraction = cfg.trigger_fraction
        c.growth_fraction = cfg.growth_fraction
        self._h = C.c_void_p()
        rc = self._lib.dg_create(C.byref(c), initial_vertex_count, block_size, C.byref(self._h))
        if rc != 0:
            self._h = C.c_void_p()
            self._raise(rc, None)

    # -- plumbing -------------------------------------------------------------
    def _raise(self, rc: int, h):
        msg = self._lib.dg_last_error(h).decode(errors="replace")
        cls = {_lib.DG_ERR_DATA: DataError, _lib.DG_ERR_ENGINE: EngineError,
               _lib.DG_ERR_CUDA: CudaError}.get(rc, Error)
        raise cls(msg)

    def _check(self, rc: int):
        if rc != 0:
            self._raise(rc, self._h)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h:
            self._lib.dg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- observables (graph.hpp:96-108) ------------------------------------------
    def block_size(self) -> int: return int(self._lib.dg_block_size(self._h))
    def logical_size(self) -> int: return int(self._lib.dg_logical_size(self._h))
    def vertex_capacity(self) -> int: return int(self._lib.dg_vertex_capacity(self._h))
    def alive_vertices(self) -> int: return int(self._lib.dg_alive_vertices(self._h))
    def active_edges(self) -> int: return int(self._lib.dg_active_edges(self._h))
    def vertex_alive(self, v: int) -> bool:
        return 0 <= v < 2**32 and bool(self._lib.dg_vertex_alive(self._h, v))
    def stream(self) -> int: return int(self._lib.dg_stream(self._h) or 0)
    def synchronize(self): self._check(self._lib.dg_synchronize(self._h))

    # -- batch updates -------------------------------------------------------------
    def insert_batch(self, batch: CsrBatch):
        """graph.hpp:167-188."""
        if batch.kind != BatchKind.Insert:
            raise DataError("plan_batch: expected an insert batch")  # graph.hpp:136-138
        off, dst = _Arg(batch.offsets, np.uint64), _Arg(batch.destinations, np.uint32)
        self._check(self._lib.dg_insert_batch_csr(self._h, off.ptr, off.n, dst.ptr, dst.n, dst.mem))

    def delete_batch(self, batch: CsrBatch):
        """graph.hpp:195-222."""
        if batch.kind != BatchKind.Delete:
            raise DataError("delete_batch: expected a delete batch")  # graph.hpp:196-198
        off, dst = _Arg(batch.offsets, np.uint64), _Arg(batch.destinations, np.uint32)
        self._check(self._lib.dg_delete_batch_csr(self._h, off.ptr, off.n, dst.ptr, dst.n, dst.mem))

    def plan_batch(self, batch: CsrBatch) -> "BatchPlan":
        """graph.hpp:135-160: validation of an insert batch + its BatchPlan (nothing is mutated)."""
        if batch.kind != BatchKind.Insert:
            raise DataError("plan_batch: expected an insert batch")  # graph.hpp:136-138
        off, dst = _Arg(np.asarray(batch.offsets), np.uint64), _Arg(np.asarray(batch.destinations), np.uint32)
        n = max(off.n - 1, 0)
        req, pre, space = np.zeros(n, np.uint64), np.zeros(n, np.uint64), np.zeros(n, np.uint32)
        total = C.c_uint64()
        self._check(self._lib.dg_plan_batch_csr(self._h, off.ptr, off.n, dst.ptr, dst.n, _lib.DG_MEM_HOST,
                                                C.c_void_p(req.ctypes.data), C.c_void_p(pre.ctypes.data),
                                                C.c_void_p(space.ctypes.data), C.byref(total)))
        return BatchPlan(req, pre, space)

    def bulk_init(self, offsets, destinations):
        """ctor + first insert_batch of the whole graph (io/workload.hpp:113-139)."""
        off, dst = _Arg(offsets, np.uint64), _Arg(destinations, np.uint32)
        if off.mem != dst.mem:
            raise DataError("bulk_init: offsets and destinations must live in the same memory space")
        self._check(self._lib.dg_bulk_init_csr(self._h, off.ptr, off.n, dst.ptr, dst.n, dst.mem))

    def insert_pairs(self, src, dst):
        """insert_batch(csr_from_pairs(Insert, V, pairs)) in O(batch) (csr.hpp:29-45)."""
        s, d = self._pair_args(src, dst)
        self._check(self._lib.dg_insert_batch_coo(self._h, s.ptr, d.ptr, s.n, s.mem))

    def delete_pairs(self, src, dst):
        s, d = self._pair_args(src, dst)
        self._check(self._lib.dg_delete_batch_coo(self._h, s.ptr, d.ptr, s.n, s.mem))

    # -- submitted updates (dg_submit_*_coo / dg_flush: no host wait per batch) -----------------
    def submit_insert_pairs(self, src, dst) -> int:
        """insert_pairs without waiting for the op: DEVICE arrays that stay alive until flush().  Returns the
        op's ticket (0: the call had to run it synchronously).  A failure surfaces at flush() or at the next
        call of any kind; ops submitted behind a failed one are not applied (graph.hpp:168-171)."""
        return self._submit(self._lib.dg_submit_insert_coo, src, dst)

    def submit_delete_pairs(self, src, dst) -> int:
        return self._submit(self._lib.dg_submit_delete_coo, src, dst)

    def _submit(self, fn, src, dst) -> int:
        s, d = self._pair_args(src, dst)
        if s.mem != _lib.DG_MEM_DEVICE:
            raise DataError("submit: device arrays only (host batches go through ingest())")
        t = C.c_uint64()
        self._check(fn(self._h, s.ptr, d.ptr, s.n, C.byref(t)))
        return int(t.value)

    def flush(self) -> int:
        """Waits for every submitted op; raises the first failure; returns how many ops were applied since the last
        flush() that returned (a flush that raises keeps its count for the next one: after a failure, call flush()
        once more to learn how many ops went in before the failed one)."""
        n = C.c_uint64()
        rc = self._lib.dg_flush(self._h, C.byref(n))
        self._applied_pending = getattr(self, "_applied_pending", 0) + int(n.value)
        self._check(rc)
        out, self._applied_pending = self._applied_pending, 0
        return out

    def pending_ops(self) -> int:
        return int(self._lib.dg_pending_ops(self._h))

    @staticmethod
    def _pair_args(src, dst):
        s, d = _Arg(src, np.uint32), _Arg(dst, np.uint32)
        if s.n != d.n or s.mem != d.mem:
            raise DataError("pairs: src/dst must have equal length and memory space")
        return s, d

    # -- queries -----------------------------------------------------------------------
    def query_edges(self, src, dst):
        """Batched query_edge (graph.hpp:228-241); returns uint8 answers."""
        s, d = self._pair_args(src, dst)
        if s.mem == _lib.DG_MEM_DEVICE:
            import torch
            out = torch.empty(s.n, dtype=torch.uint8, device=s.keep.device)
            self._check(self._lib.dg_query_edges(self._h, s.ptr, d.ptr, s.n, C.c_void_p(out.data_ptr()), s.mem))
            return out
        out = np.zeros(s.n, dtype=np.uint8)
        self._check(self._lib.dg_query_edges(self._h, s.ptr, d.ptr, s.n, C.c_void_p(out.ctypes.data), s.mem))
        return out

    def query_edge(self, source: int, destination: int) -> bool:
        if not (0 <= source < 2**32 and 0 <= destination < 2**32):
            return False
        return bool(self.query_edges(np.array([source], np.uint32), np.array([destination], np.uint32))[0])

    def export_csr(self, sorted: bool = True):
        """active_destinations of every vertex as one CSR (graph.hpp:116-129)."""
        n = self.logical_size()
        offsets = np.zeros(n + 1, dtype=np.uint64)
        self._check(self._lib.dg_export_csr(self._h, C.c_void_p(offsets.ctypes.data), None, 0,
                                            int(sorted), _lib.DG_MEM_HOST))
        total = int(offsets[n])
        dsts = np.zeros(total, dtype=np.uint32)
        if total:
            self._check(self._lib.dg_export_csr(self._h, C.c_void_p(offsets.ctypes.data),
                                                C.c_void_p(dsts.ctypes.data), total, int(sorted),
                                                _lib.DG_MEM_HOST))
        return offsets, dsts

    def active_destinations(self, v: int) -> np.ndarray:
        """Live destinations of ONE vertex in traversal order (graph.hpp:116-129): dg_active_destinations."""
        if v < 0 or v >= self.logical_size():
            return np.zeros(0, dtype=np.uint32)
        n = C.c_uint64()
        out = np.zeros(64, dtype=np.uint32)
        rc = self._lib.dg_active_destinations(self._h, v, C.c_void_p(out.ctypes.data), out.size, C.byref(n), _lib.DG_MEM_HOST)
        if rc == _lib.DG_ERR_DATA and n.value > out.size:   # the degree came back: once more with room for it
            out = np.zeros(int(n.value), dtype=np.uint32)
            rc = self._lib.dg_active_destinations(self._h, v, C.c_void_p(out.ctypes.data), out.size, C.byref(n), _lib.DG_MEM_HOST)
        self._check(rc)
        return out[:int(n.value)]

    def degrees(self) -> np.ndarray:
        out = np.zeros(self.logical_size(), dtype=np.uint64)
        self._check(self._lib.dg_degrees(self._h, C.c_void_p(out.ctypes.data), _lib.DG_MEM_HOST))
        return out

    def digest(self):
        d, n = C.c_uint64(), C.c_uint64()
        self._check(self._lib.dg_digest(self._h, C.byref(d), C.byref(n)))
        return int(d.value), int(n.value)

    # -- vertex updates -------------------------------------------------------------------
    def insert_vertices(self, count: int):
        self._check(self._lib.dg_insert_vertices(self._h, count))

    def delete_vertices(self, ids) -> list[int]:
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        skipped = np.zeros(max(1, a.size), dtype=np.uint32)
        ns = C.c_uint64()
        self._check(self._lib.dg_delete_vertices(self._h, C.c_void_p(a.ctypes.data), a.size,
                                                 C.c_void_p(skipped.ctypes.data), C.byref(ns)))
        return [int(x) for x in skipped[: ns.value]]

    # -- pipelined host batches ------------------------------------------------------------------
    def ingest(self, max_entries: int, depth: int = 2, synchronous: bool = False) -> "BatchIngest":
        """Ingest queue for a stream of HOST batches: the copy of the next batch overlaps the
        current op (the loop of io/workload.hpp:141-155, with the PCIe copy taken off its path)."""
        return BatchIngest(self, max_entries, depth, synchronous)

    # -- reports -----------------------------------------------------------------------------
    def stats(self) -> dict:
        st = _lib.DgStats()
        self._check(self._lib.dg_stats_get(self._h, C.byref(st)))
        d = {n: int(getattr(st, n)) for n, _ in st._fields_ if n != "reserved"}
        d["hole_ratio"] = 0.0 if d["occupied_slots"] == 0 else d["hole_slots"] / d["occupied_slots"]
        return d

    def memory(self) -> dict:
        m = _lib.DgMemory()
        self._check(self._lib.dg_memory_get(self._h, C.byref(m)))
        d = {n: int(getattr(m, n)) for n, _ in m._fields_}
        d["total"] = d["dictionary_bytes"] + d["sentinel_bytes"] + d["pool_bytes"] + d["queue_bytes"]
        return d

    def last_op_report(self) -> dict:
        r = _lib.DgOpReport()
        self._check(self._lib.dg_last_op_report(self._h, C.byref(r)))
        return {n: int(getattr(r, n)) for n, _ in r._fields_}

    def profile_enable(self, on: bool = True):
        self._check(self._lib.dg_profile_enable(self._h, int(on)))

    def profile_report(self) -> dict:
        """kernel name -> (total_ms, launches) since profiling was enabled."""
        out = {}
        for line in self._lib.dg_profile_report(self._h).decode().splitlines():
            name, ms, cnt = line.split("\t")
            out[name] = (float(ms), int(cnt))
        return out

    # -- input-side helpers --------------------------------------------------------------------
    def compute_block_size_pairs(self, src) -> int:
        s = _Arg(src, np.uint32)
        out = C.c_uint32()
        self._check(self._lib.dg_compute_block_size_coo(self._h, s.ptr, s.n, s.mem, C.byref(out)))
        return int(out.value)

    def gen_rmat(self, scale: int, seed: int, first_index: int, src_dev, dst_dev, thresholds):
        s, d = _Arg(src_dev, np.uint32), _Arg(dst_dev, np.uint32)
        if s.mem != _lib.DG_MEM_DEVICE or d.mem != _lib.DG_MEM_DEVICE:
            raise DataError("gen_rmat writes device tensors")
        ta, tab, tabc = thresholds
        self._check(self._lib.dg_gen_rmat(self._h, scale, seed, first_index, s.n, ta, tab, tabc, s.ptr, d.ptr))

    def coo_to_csr(self, src, dst, vertex_count: int, offsets_dev, destinations_dev):
        s, d = self._pair_args(src, dst)
        o, dd = _Arg(offsets_dev, np.uint64), _Arg(destinations_dev, np.uint32)
        self._check(self._lib.dg_coo_to_csr(self._h, s.ptr, d.ptr, s.n, s.mem, vertex_count, o.ptr, dd.ptr))


class BatchIngest:
    """`submit("insert" | "delete", src, dst)` applies host batches in order, exactly like calling
    insert_pairs / delete_pairs one after the other, without a host wait per batch: the copy of a batch goes
    to one of `depth` device slots on its own stream and the op is SUBMITTED behind it (dg_ingest_submit_*),
    so copies, ops and the host loop overlap.  A failing batch raises from a later submit or from flush();
    batches submitted behind it are not applied (the reference loop would have stopped there too) and
    `applied` tells how many were.  Host arrays are kept alive here until their op has certainly run
    (pinned memory makes the copy asynchronous).  `synchronous=True` keeps the round-1 behaviour: one host
    wait per op, `depth - 1` copies in flight behind the running op."""

    def __init__(self, graph: DynamicGraph, max_entries: int, depth: int = 2, synchronous: bool = False):
        self._g = graph
        self._lib = graph._lib
        self._max_entries = max_entries
        self._depth = depth
        self._sync = synchronous
        self._q = None
        self._open()
        self._pending = []   # synchronous mode: (kind, slot, keep-alive arrays)
        self._keep = []      # submitted mode: host arrays of the last depth + 8 batches
        self.applied = 0

    def _open(self):
        q = C.c_void_p()
        self._g._check(self._lib.dg_ingest_create(self._g._h, self._max_entries, self._depth, C.byref(q)))
        self._q = q

    def close(self):
        if self._q:
            self._lib.dg_ingest_destroy(self._q)
            self._q = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _run_oldest(self):
        kind, slot, _keep = self._pending.pop(0)
        fn = self._lib.dg_ingest_insert if kind == "insert" else self._lib.dg_ingest_delete
        rc = fn(self._q, slot)
        if rc != 0:
            self._pending.clear()
            self._lib.dg_ingest_reset(self._q)   # drop whatever is still staged
            self._g._check(rc)
        self.applied += 1
        return rc

    def submit(self, kind: str, src, dst):
        if kind not in ("insert", "delete"):
            raise DataError("ingest: kind must be 'insert' or 'delete'")
        s = np.ascontiguousarray(src, dtype=np.uint32)
        d = np.ascontiguousarray(dst, dtype=np.uint32)
        if s.size != d.size:
            raise DataError("pairs: src/dst must have equal length")
        if self._sync and len(self._pending) == self._depth:
            self._run_oldest()
        slot = C.c_uint32()
        self._g._check(self._lib.dg_ingest_stage_coo(self._q, C.c_void_p(s.ctypes.data), C.c_void_p(d.ctypes.data),
                                                     s.size, C.byref(slot)))
        if self._sync:
            self._pending.append((kind, int(slot.value), (s, d)))
            if len(self._pending) == self._depth:   # keep depth - 1 copies in flight behind the running op
                self._run_oldest()
            return
        # (at most `depth` staged + 7 submitted ops are ever unfinished: older host arrays can go)
        self._keep.append((s, d))
        if len(self._keep) > self._depth + 8:
            self._keep.pop(0)
        fn = self._lib.dg_ingest_submit_insert if kind == "insert" else self._lib.dg_ingest_submit_delete
        t = C.c_uint64()
        rc = fn(self._q, int(slot.value), C.byref(t))
        if rc != 0:
            self._lib.dg_ingest_reset(self._q)
            self._collect()
            self._g._check(rc)

    def _collect(self):
        n = C.c_uint64()
        rc = self._lib.dg_flush(self._g._h, C.byref(n))
        self.applied += int(n.value)
        self._keep.clear()
        return rc

    def flush(self):
        while self._pending:
            self._run_oldest()
        if not self._sync:
            self._g._check(self._collect())
