"""Source-partitioned multi-GPU store (nothing like it in the reference).

One process per GPU.  Vertex v is owned by rank `perm(v) mod world` and lives
there under local id `perm(v) // world`, where `perm` is the fixed mixing
bijection of include/dyngraph_b200.h (`dg_owner_perm`): R-MAT sources with
equal low bits carry ~44 % of the edges, so `v mod world` would be badly skewed.
Each rank owns an ordinary single-GPU `DynamicGraph` (its own dictionary, block
pool and free ring) over its local ids; destinations stay GLOBAL ids.

Every batch op routes its pairs to the owners, then runs the single-GPU op on
what was received; queries send their 1-byte answers back.  Two exchanges:

  exchange="p2p"  (default when every peer is reachable over CUDA IPC / NVLink)
      ONE kernel (`dg_exchange_push_coo`) computes each pair's owner and stores
      it straight into the owner's receive buffer (peer-mapped memory, slots
      reserved with a warp-aggregated system-scope atomicAdd on the owner's
      cursor) — routing and transfer fused, no pack / count exchange / unpack.
      The status all-reduce that agrees on validation doubles as the barrier
      that publishes the round.  Answers go back the same way
      (`dg_exchange_push_answers`).
  exchange="nccl"
      `dg_route_coo` (owner-bucket partition on the device) -> count exchange ->
      payload all-to-all (`torch.distributed`) -> reverse all-to-all for answers.

Validation failures are agreed with one all-reduce(MAX) BEFORE any rank mutates
(batch atomicity, reference graph.hpp:168-171).

The exchange itself (`exchange_buckets`) is device-agnostic so the host logic
is covered by world_size-2 gloo tests on CPU tensors; the product path only
ever feeds it CUDA tensors produced by the CUDA library.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import DataError, EngineError, Error
from .graph import DynamicGraph, GraphConfig


# ---- host twins of owner_perm (csrc/dg_kernels.cuh) ---------------------------------------------
def owner_bits(vertex_count: int) -> int:
    return max(1, int(vertex_count - 1).bit_length())


def owner_perm_np(v: np.ndarray, bits: int) -> np.ndarray:
    """numpy twin of dg_owner_perm: a bijection on [0, 2^bits)."""
    if bits == 0:
        return v.astype(np.uint32)
    mask = np.uint64(0xFFFFFFFF if bits >= 32 else (1 << bits) - 1)
    sh = np.uint64((bits + 1) // 2)
    x = v.astype(np.uint64) & mask
    x = (x * np.uint64(0x9E3779B1)) & mask
    x ^= x >> sh
    x = (x * np.uint64(0x85EBCA6B)) & mask
    x ^= x >> sh
    return x.astype(np.uint32)


def owner_of_np(v: np.ndarray, bits: int, world: int):
    p = owner_perm_np(v, bits)
    return (p % np.uint32(world)).astype(np.uint32), (p // np.uint32(world)).astype(np.uint32)


def local_vertex_count(vertex_count: int, world: int) -> int:
    bits = owner_bits(vertex_count)
    return ((1 << bits) + world - 1) // world


# ---- the collective --------------------------------------------------------------------------------
def exchange_buckets(tensors, send_counts, group=None):
    """All-to-all of owner-grouped buckets.

    `tensors` are 1-D tensors of equal length laid out as world consecutive
    buckets of sizes `send_counts` (a python list / 1-D int64 CPU tensor).
    Returns (received tensors, recv_counts list).  Works for gloo/CPU and
    nccl/CUDA tensors alike."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    send_counts = [int(c) for c in send_counts]
    assert len(send_counts) == world
    dev = tensors[0].device
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(c) for c in rc.tolist()]
    out = []
    for t in tensors:
        r = torch.empty(sum(recv_counts), dtype=t.dtype, device=dev)
        dist.all_to_all_single(r, t, output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
        out.append(r)
    return out, recv_counts


def agree_status(code: int, device, group=None) -> int:
    """max over ranks of a status code (0 ok / 2 data / 3 engine / 4 cuda)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(code)], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


_STATUS_EXC = {_lib.DG_ERR_DATA: DataError, _lib.DG_ERR_ENGINE: EngineError}


class ShardedDynamicGraph:
    """The operator API of DynamicGraph over `world` source-partitioned GPUs."""

    def __init__(self, config: GraphConfig | None, vertex_count: int, block_size: int,
                 torch_stream=None, group=None, exchange: str = "p2p", exchange_capacity: int = 1 << 22):
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            raise EngineError("ShardedDynamicGraph needs an initialised torch.distributed process group")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.vertex_count = int(vertex_count)
        self.bits = owner_bits(self.vertex_count)
        cfg = config or GraphConfig()
        self.device = torch.device("cuda", cfg.device)
        self.torch_stream = torch_stream
        self.local = DynamicGraph(cfg, local_vertex_count(self.vertex_count, self.world), block_size)
        lib = self.local._lib
        rc = lib.dg_set_dst_limit(self.local._h, self.vertex_count)
        if rc != 0:
            raise DataError("dst limit")
        self._lib = lib
        self._x = None
        if exchange == "p2p":
            self._setup_p2p(int(exchange_capacity))

    def close(self):
        if self._x is not None:
            self._lib.dg_exchange_destroy(self._x)
            self._x = None
        self.local.close()

    # -- fused routing + exchange over peer memory ----------------------------------------------------
    def _setup_p2p(self, capacity: int):
        import torch.distributed as dist

        x = C.c_void_p()
        rc = self._lib.dg_exchange_create(self.local._h, self.rank, self.world, capacity, C.byref(x))
        if agree_status(rc, self.device, self.group) != 0:
            raise EngineError("sharded store: could not create the peer-memory exchange buffers")
        handle = C.create_string_buffer(_lib.DG_IPC_HANDLE_BYTES)
        self.local._check(self._lib.dg_exchange_ipc_handle(x, handle))
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=self.group)
        rc = 0
        for peer, raw in enumerate(handles):
            if peer != self.rank:
                rc = max(rc, self._lib.dg_exchange_set_peer(x, peer, C.create_string_buffer(raw, len(raw))))
        if agree_status(rc, self.device, self.group) != 0:
            self._lib.dg_exchange_destroy(x)
            raise EngineError("sharded store: a peer's exchange buffer could not be mapped (CUDA IPC); "
                              "use exchange='nccl'")
        self._x = x

    def _push(self, src, dst):
        """One exchange round; returns (n_received, src_ptr, dst_ptr, idx_ptr, from_ptr)."""
        lib = self._lib
        rc = lib.dg_exchange_reset(self._x)
        agree_status(rc, self.device, self.group)     # barrier: every cursor is zero before anyone pushes
        rc = lib.dg_exchange_push_coo(self._x, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), src.numel(),
                                      self.bits, self.vertex_count)
        rc = agree_status(rc, self.device, self.group)  # barrier: every push has landed (each rank synchronised)
        if rc != 0:
            raise _STATUS_EXC.get(rc, Error)("sharded batch: a rank rejected the batch while routing "
                                              "(source id out of range or receive buffer full)")
        n = C.c_uint64()
        ps, pd, pi, pf = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        self.local._check(lib.dg_exchange_received(self._x, C.byref(n), C.byref(ps), C.byref(pd), C.byref(pi), C.byref(pf)))
        return int(n.value), ps, pd, pi, pf

    def _apply_ptr(self, fn, ps, pd, n):
        code = fn(self.local._h, ps, pd, n, _lib.DG_MEM_DEVICE) if n else 0
        msg = self._lib.dg_last_error(self.local._h).decode(errors="replace") if code else ""
        agreed = agree_status(code, self.device, self.group)
        if agreed != 0:
            raise _STATUS_EXC.get(agreed, Error)(msg or "sharded batch: rejected on another rank")

    # -- routing -------------------------------------------------------------------------------------
    def _route(self, src, dst):
        """Device partition by owner; returns (src_local, dst, index, counts) or raises DataError
        on every rank if any rank saw a source outside the graph."""
        import torch

        n = src.numel()
        out_s = torch.empty(n, dtype=torch.int32, device=self.device)
        out_d = torch.empty(n, dtype=torch.int32, device=self.device)
        out_i = torch.empty(n, dtype=torch.int32, device=self.device)
        counts = (C.c_uint64 * self.world)()
        rc = self._lib.dg_route_coo(self.local._h, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), n,
                                    self.world, self.bits, self.vertex_count, C.c_void_p(out_s.data_ptr()),
                                    C.c_void_p(out_d.data_ptr()), C.c_void_p(out_i.data_ptr()), counts)
        rc = agree_status(rc, self.device, self.group)
        if rc != 0:
            raise _STATUS_EXC.get(rc, Error)("sharded batch: a rank rejected the batch while routing "
                                              "(source id out of range)")
        return out_s, out_d, out_i, [int(c) for c in counts]

    def _exchange(self, tensors, counts):
        import torch

        # the route kernels ran on the graph's stream; the collective runs on torch's current one
        self.local.synchronize()
        return exchange_buckets(tensors, counts, self.group)

    def _apply(self, fn, s, d):
        """Run the local op; agree on the outcome so every rank raises or none does."""
        code, msg = 0, ""
        try:
            fn(s, d)
        except DataError as e:
            code, msg = _lib.DG_ERR_DATA, str(e)
        except EngineError as e:
            code, msg = _lib.DG_ERR_ENGINE, str(e)
        agreed = agree_status(code, self.device, self.group)
        if agreed != 0:
            raise _STATUS_EXC.get(agreed, Error)(msg or "sharded batch: rejected on another rank")

    # -- operator API (graph.hpp:167-241) ------------------------------------------------------------------
    def insert_pairs(self, src, dst):
        if self._x is not None:
            n, ps, pd, _, _ = self._push(src, dst)
            return self._apply_ptr(self._lib.dg_insert_batch_coo, ps, pd, n)
        s, d, _, counts = self._route(src, dst)
        (rs, rd), _ = self._exchange([s, d], counts)
        self._apply(self.local.insert_pairs, rs, rd)

    def delete_pairs(self, src, dst):
        if self._x is not None:
            n, ps, pd, _, _ = self._push(src, dst)
            return self._apply_ptr(self._lib.dg_delete_batch_coo, ps, pd, n)
        s, d, _, counts = self._route(src, dst)
        (rs, rd), _ = self._exchange([s, d], counts)
        self._apply(self.local.delete_pairs, rs, rd)

    def query_edges(self, src, dst):
        """Answers in the caller's order on the calling rank (uint8 CUDA tensor)."""
        import torch

        n = src.numel()
        # unknown sources answer 0 (graph.hpp:229): clamp them to a vertex id and mask afterwards
        known = (src.to(torch.int64) & 0xFFFFFFFF) < self.vertex_count
        src_c = torch.where(known, src, torch.zeros_like(src))
        if self._x is not None:
            nr, ps, pd, _, _ = self._push(src_c, dst)
            ans = torch.zeros(max(nr, 1), dtype=torch.uint8, device=self.device)
            rc = self._lib.dg_query_edges(self.local._h, ps, pd, nr, C.c_void_p(ans.data_ptr()), _lib.DG_MEM_DEVICE) if nr else 0
            rc = max(rc, self._lib.dg_exchange_push_answers(self._x, C.c_void_p(ans.data_ptr()), nr))
            if agree_status(rc, self.device, self.group) != 0:   # barrier: every answer has landed
                raise EngineError("sharded query failed on a rank")
            out = torch.empty(n, dtype=torch.uint8, device=self.device)
            self.local._check(self._lib.dg_exchange_answers(self._x, C.c_void_p(out.data_ptr()), n, _lib.DG_MEM_DEVICE))
            return out * known.to(torch.uint8)
        s, d, idx, counts = self._route(src_c, dst)
        (rs, rd), recv_counts = self._exchange([s, d], counts)
        ans = self.local.query_edges(rs, rd) if rs.numel() else torch.empty(0, dtype=torch.uint8, device=self.device)
        self.local.synchronize()
        (back,), _ = exchange_buckets([ans], recv_counts, self.group)
        out = torch.zeros(n, dtype=torch.uint8, device=self.device)
        out[idx.to(torch.int64)] = back
        return out * known.to(torch.uint8)

    # -- observables: sums / maxima over ranks ---------------------------------------------------------------
    def _sum(self, x: int) -> int:
        import torch
        import torch.distributed as dist

        t = torch.tensor([int(x)], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def logical_size(self) -> int:
        return self.vertex_count

    def active_edges(self) -> int:
        return self._sum(self.local.active_edges())

    def digest(self):
        d, n = self.local_digest_global()
        import torch
        import torch.distributed as dist

        t = torch.tensor([d - (1 << 64) if d >= (1 << 63) else d, n], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)  # wraps mod 2^64 like the device sum
        return int(t[0].item()) & ((1 << 64) - 1), int(t[1].item())

    def local_digest_global(self):
        """Digest of this rank's entries expressed over GLOBAL (src, dst) ids, so the sum over ranks
        equals the single-GPU dg_digest of the same multiset."""
        off, dst = self.local.export_csr(sorted=False)
        deg = np.diff(off.astype(np.int64))
        lid = np.repeat(np.arange(len(deg), dtype=np.uint64), deg)
        p = lid * np.uint64(self.world) + np.uint64(self.rank)
        gsrc = np.array([self._lib.dg_owner_perm_inv(int(x), self.bits) for x in np.unique(p)], dtype=np.uint64)
        lut = dict(zip(np.unique(p).tolist(), gsrc.tolist()))
        g = np.array([lut[int(x)] for x in p], dtype=np.uint64) if len(p) else np.zeros(0, np.uint64)
        with np.errstate(over="ignore"):
            x = (g << np.uint64(32)) | dst.astype(np.uint64)
            x = x + np.uint64(0x9E3779B97F4A7C15)
            x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            x = x ^ (x >> np.uint64(31))
            return int(x.sum(dtype=np.uint64)) if len(x) else 0, int(len(x))
