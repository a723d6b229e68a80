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
      The whole round protocol runs ON THE DEVICE: arrival and status counters
      live in the peer-mapped buffers (system-scope atomics, a one-warp waiting
      kernel, two buffer sets alternating between rounds), so a batch costs NO
      host collective.  Answers go back the same way.
  exchange="nccl"
      `dg_route_coo` (owner-bucket partition on the device) -> count exchange ->
      payload all-to-all (`torch.distributed`) -> reverse all-to-all for answers.

Batch atomicity across ranks (reference graph.hpp:168-171: a rejected batch
leaves the graph unchanged): every rank validates and plans what it received,
the statuses are agreed, and only an all-clear lets any rank mutate — on the
device inside the op for p2p (`exchange_agree_kernel`), with
`dg_check_batch_coo` + one all-reduce(MAX) for nccl.

Vertex ids: the owner permutation is a bijection on [0, 2^bits), fixed at
creation (`reserve_vertices` leaves room to grow); `insert_vertices` is
replicated metadata, `delete_vertices` routes every id to its owner.

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


def owner_perm_inv_np(p: np.ndarray, bits: int) -> np.ndarray:
    """numpy twin of dg_owner_perm_inv."""
    if bits == 0:
        return p.astype(np.uint32)
    mask = np.uint64(0xFFFFFFFF if bits >= 32 else (1 << bits) - 1)
    sh = np.uint64((bits + 1) // 2)

    def inv32(a):
        x = a
        for _ in range(5):
            x = (x * ((2 - a * x) & 0xFFFFFFFF)) & 0xFFFFFFFF
        return x
    x = p.astype(np.uint64) & mask
    x ^= x >> sh
    x = (x * np.uint64(inv32(0x85EBCA6B))) & mask
    x ^= x >> sh
    x = (x * np.uint64(inv32(0x9E3779B1))) & mask
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
                 torch_stream=None, group=None, exchange: str = "p2p", exchange_capacity: int = 1 << 22,
                 reserve_vertices: int = 0):
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            raise EngineError("ShardedDynamicGraph needs an initialised torch.distributed process group")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.vertex_count = int(vertex_count)
        # the permutation's domain is fixed for the life of the store: vertices can be added up to 2^bits
        self.bits = owner_bits(max(self.vertex_count, int(reserve_vertices), 1))
        self.retired = 0
        cfg = config or GraphConfig()
        self.device = torch.device("cuda", cfg.device)
        self.torch_stream = torch_stream
        self.local = DynamicGraph(cfg, ((1 << self.bits) + self.world - 1) // self.world, block_size)
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

    def _raise(self, rc: int, msg: str = ""):
        raise _STATUS_EXC.get(rc, Error)(msg or self._lib.dg_last_error(self.local._h).decode(errors="replace")
                                         or "sharded batch: rejected on another rank")

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
        dist.all_gather_object(handles, handle.raw, group=self.group)   # (also the barrier: every buffer is zeroed)
        rc = 0
        for peer, raw in enumerate(handles):
            if peer != self.rank:
                rc = max(rc, self._lib.dg_exchange_set_peer(x, peer, C.create_string_buffer(raw, len(raw))))
        if agree_status(rc, self.device, self.group) != 0:
            self._lib.dg_exchange_destroy(x)
            raise EngineError("sharded store: a peer's exchange buffer could not be mapped (CUDA IPC); "
                              "use exchange='nccl'")
        self._lib.dg_exchange_attach(x, 1)   # local ops agree their status with the peers on the device
        self._x = x

    def _sync_inputs(self):
        """Tensors handed in were produced on torch's current stream; the graph runs on its own."""
        import torch
        if self.torch_stream is None or self.torch_stream.cuda_stream != self._lib.dg_stream(self.local._h):
            torch.cuda.current_stream(self.device).synchronize()

    def _push(self, src, dst):
        """One exchange round up to the reception; returns (n_received, src_ptr, dst_ptr, idx_ptr, from_ptr).
        No host collective: arrival and status travel through the peer-mapped round words."""
        lib = self._lib
        self._sync_inputs()
        lib.dg_exchange_push_coo(self._x, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), src.numel(),
                                 self.bits, self.vertex_count)   # (a local rejection comes back agreed below)
        n = C.c_uint64()
        ps, pd, pi, pf = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        rc = lib.dg_exchange_received(self._x, C.byref(n), C.byref(ps), C.byref(pd), C.byref(pi), C.byref(pf))
        if rc != 0:   # the same status on every rank: nobody applies anything
            msg = lib.dg_last_error(self.local._h).decode(errors="replace")
            lib.dg_exchange_end_round(self._x)
            self._raise(rc, msg)
        return int(n.value), ps, pd, pi, pf

    def _apply_ptr(self, fn, ps, pd, n):
        """The local op on what was received; its validation / plan status is agreed with the peers ON THE DEVICE
        before anything mutates (dg_exchange_attach), so the return code is already the agreed one."""
        lib = self._lib
        if n:
            rc = fn(self.local._h, ps, pd, n, _lib.DG_MEM_DEVICE)
        else:
            agreed = C.c_int()
            rc = lib.dg_exchange_agree(self._x, 0, C.byref(agreed))
        msg = lib.dg_last_error(self.local._h).decode(errors="replace") if rc else ""
        lib.dg_exchange_end_round(self._x)
        if rc != 0:
            self._raise(rc, msg)

    # -- routing -------------------------------------------------------------------------------------
    def _route(self, src, dst):
        """Device partition by owner; returns (src_local, dst, index, counts) or raises DataError
        on every rank if any rank saw a source outside the graph."""
        import torch

        n = src.numel()
        self._sync_inputs()
        out_s = torch.empty(n, dtype=torch.int32, device=self.device)
        out_d = torch.empty(n, dtype=torch.int32, device=self.device)
        out_i = torch.empty(n, dtype=torch.int32, device=self.device)
        torch.cuda.current_stream(self.device).synchronize()
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
        # the route kernels ran on the graph's stream; the collective runs on torch's current one
        self.local.synchronize()
        return exchange_buckets(tensors, counts, self.group)

    def _apply(self, fn, s, d, is_insert: bool):
        """NCCL exchange: validate + plan on every rank (dg_check_batch_coo, nothing mutates), agree, then apply —
        a batch is applied on every rank or on none (graph.hpp:168-171)."""
        import torch
        torch.cuda.current_stream(self.device).synchronize()   # (the all-to-all wrote s / d on torch's stream)
        n = s.numel()
        rc = self._lib.dg_check_batch_coo(self.local._h, C.c_void_p(s.data_ptr()), C.c_void_p(d.data_ptr()), n,
                                          int(is_insert), _lib.DG_MEM_DEVICE) if n else 0
        msg = self._lib.dg_last_error(self.local._h).decode(errors="replace") if rc else ""
        agreed = agree_status(rc, self.device, self.group)
        if agreed != 0:
            self._raise(agreed, msg if rc == agreed else "sharded batch: rejected on another rank")
        if n:
            fn(s, d)

    # -- operator API (graph.hpp:167-241) ------------------------------------------------------------------
    def insert_pairs(self, src, dst):
        if self._x is not None:
            n, ps, pd, _, _ = self._push(src, dst)
            return self._apply_ptr(self._lib.dg_insert_batch_coo, ps, pd, n)
        s, d, _, counts = self._route(src, dst)
        (rs, rd), _ = self._exchange([s, d], counts)
        self._apply(self.local.insert_pairs, rs, rd, True)

    def delete_pairs(self, src, dst):
        if self._x is not None:
            n, ps, pd, _, _ = self._push(src, dst)
            return self._apply_ptr(self._lib.dg_delete_batch_coo, ps, pd, n)
        s, d, _, counts = self._route(src, dst)
        (rs, rd), _ = self._exchange([s, d], counts)
        self._apply(self.local.delete_pairs, rs, rd, False)

    def bulk_init(self, offsets, destinations):
        """This rank's part of the base graph as a CSR over GLOBAL vertex ids (offsets: vertex_count + 1 int64,
        destinations: int32; CUDA tensors): expanded to pairs and routed like any insert batch (io/workload.hpp:113-139
        bulk-builds with one insert_batch of the whole graph)."""
        import torch
        deg = (offsets[1:] - offsets[:-1]).to(torch.int64)
        src = torch.repeat_interleave(torch.arange(self.vertex_count, dtype=torch.int32, device=self.device), deg)
        self.insert_pairs(src, destinations)

    def query_edges(self, src, dst):
        """Answers in the caller's order on the calling rank (uint8 CUDA tensor)."""
        import torch

        n = src.numel()
        # unknown sources answer 0 (graph.hpp:229): clamp them to a vertex id and mask afterwards
        known = (src.to(torch.int64) & 0xFFFFFFFF) < self.vertex_count
        src_c = torch.where(known, src, torch.zeros_like(src))
        if self._x is not None:
            lib = self._lib
            nr, ps, pd, _, _ = self._push(src_c, dst)
            # (empty: dg_query_edges writes every answer; no fill on torch's stream can land after them)
            ans = torch.empty(max(nr, 1), dtype=torch.uint8, device=self.device)
            torch.cuda.current_stream(self.device).synchronize()
            rc = lib.dg_query_edges(self.local._h, ps, pd, nr, C.c_void_p(ans.data_ptr()), _lib.DG_MEM_DEVICE) if nr else 0
            lib.dg_exchange_push_answers(self._x, C.c_void_p(ans.data_ptr()), nr if rc == 0 else 0)
            out = torch.empty(n, dtype=torch.uint8, device=self.device)
            torch.cuda.current_stream(self.device).synchronize()
            rc2 = lib.dg_exchange_answers(self._x, C.c_void_p(out.data_ptr()), n, _lib.DG_MEM_DEVICE)
            lib.dg_exchange_end_round(self._x)
            if rc or rc2:
                raise EngineError("sharded query failed on a rank")
            return out * known.to(torch.uint8)
        s, d, idx, counts = self._route(src_c, dst)
        (rs, rd), recv_counts = self._exchange([s, d], counts)
        torch.cuda.current_stream(self.device).synchronize()
        ans = self.local.query_edges(rs, rd) if rs.numel() else torch.empty(0, dtype=torch.uint8, device=self.device)
        self.local.synchronize()
        (back,), _ = exchange_buckets([ans], recv_counts, self.group)
        out = torch.zeros(n, dtype=torch.uint8, device=self.device)
        out[idx.to(torch.int64)] = back
        return out * known.to(torch.uint8)

    # -- vertex updates (graph.hpp:246, :252-276) --------------------------------------------------------------
    def insert_vertices(self, count: int):
        """Replicated metadata: every rank calls it with the same count.  The new ids already have their slots (the
        owner permutation covers [0, 2^bits)); beyond that the store cannot grow."""
        count = int(count)
        if count == 0:
            return
        if self.vertex_count + count > (1 << self.bits):
            raise EngineError(f"sharded store: vertex capacity 2^{self.bits} was fixed at creation "
                              f"(pass reserve_vertices to leave room)")
        self.vertex_count += count
        if self._lib.dg_set_dst_limit(self.local._h, self.vertex_count) != 0:
            raise DataError("dst limit")

    def delete_vertices(self, ids) -> np.ndarray:
        """Every rank passes the SAME id list; each retires the vertices it owns.  Returns the skipped ids (unknown,
        already dead, repeated in the call) in encounter order, identical on every rank (graph.hpp:255-259)."""
        import torch
        import torch.distributed as dist

        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint32))
        skipped_mask = np.zeros(len(ids), dtype=np.int32)
        known = ids < self.vertex_count
        if self.rank == 0:
            skipped_mask[~known] = 1
        own, loc = owner_of_np(np.where(known, ids, 0).astype(np.uint32), self.bits, self.world)
        mine = np.nonzero(known & (own == self.rank))[0]
        if len(mine):
            # positions this rank skips: already dead, or seen earlier in the call (graph.hpp:255-259)
            seen = set()
            for i in mine:
                l = int(loc[i])
                if l in seen or not self.local.vertex_alive(l):
                    skipped_mask[i] = 1
                seen.add(l)
            local_skipped = self.local.delete_vertices(loc[mine])
            if len(local_skipped) != int(skipped_mask[mine].sum()):
                raise EngineError("sharded delete_vertices: shard and host mirror disagree")
        t = torch.from_numpy(skipped_mask).to(self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        mask = t.cpu().numpy() > 0
        self.retired += int((~mask).sum())
        return ids[mask]

    # -- observables: sums / maxima over ranks ---------------------------------------------------------------
    def _sum(self, x: int) -> int:
        import torch
        import torch.distributed as dist

        t = torch.tensor([int(x)], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def logical_size(self) -> int:
        return self.vertex_count

    def vertex_capacity(self) -> int:
        return 1 << self.bits

    def alive_vertices(self) -> int:
        return self.vertex_count - self.retired

    def active_edges(self) -> int:
        return self._sum(self.local.active_edges())

    def degrees(self):
        """sentinel_of(v).active_edge_count for every GLOBAL v < vertex_count (int64 CUDA tensor, the same on every rank)."""
        import torch
        import torch.distributed as dist

        loc = torch.from_numpy(self.local.degrees().astype(np.int64)).to(self.device)
        # local id l of this rank is vertex perm_inv(l * world + rank)
        lid = np.arange(len(loc), dtype=np.uint64) * np.uint64(self.world) + np.uint64(self.rank)
        valid = lid < (1 << self.bits)
        gid = owner_perm_inv_np(lid[valid].astype(np.uint32), self.bits).astype(np.int64)
        keep = gid < self.vertex_count
        out = torch.zeros(self.vertex_count, dtype=torch.int64, device=self.device)
        out[torch.from_numpy(gid[keep]).to(self.device)] = loc[torch.from_numpy(np.nonzero(valid)[0][keep]).to(self.device)]
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)
        return out

    def digest(self):
        """Sum over the ranks of each shard's digest over GLOBAL ids (computed on the device: dg_digest_global)."""
        import torch
        import torch.distributed as dist

        d, n = C.c_uint64(), C.c_uint64()
        self.local._check(self._lib.dg_digest_global(self.local._h, self.rank, self.world, self.bits, C.byref(d), C.byref(n)))
        dv = int(d.value)
        t = torch.tensor([dv - (1 << 64) if dv >= (1 << 63) else dv, int(n.value)], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)  # wraps mod 2^64 like the device sum
        return int(t[0].item()) & ((1 << 64) - 1), int(t[1].item())
