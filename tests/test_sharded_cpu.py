"""Host-side logic of the source-partitioned multi-GPU path, world_size 2 over gloo (CPU).

The CUDA pieces (dg_route_coo, the per-rank store) are replaced by their CPU
checkers here — numpy routing with the owner permutation twin and the oracle as
the per-rank store — so what is covered is the partition function, the count +
payload all-to-all, the answer return path and the status agreement.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_08252_b200 import _lib
from paper_2306_08252_b200.sharded import (agree_status, exchange_buckets, local_vertex_count, owner_bits,
                                           owner_of_np, owner_perm_np)
from tests.drivers import CpuGraph, load_oracle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_owner_perm_twin_matches_library_and_is_a_bijection():
    lib = _lib.load()
    for bits in (1, 2, 5, 10, 16, 22):
        n = min(1 << bits, 1 << 12)
        v = np.unique(np.concatenate([np.arange(n, dtype=np.uint32),
                                      np.random.default_rng(bits).integers(0, 1 << bits, 512).astype(np.uint32)]))
        p = owner_perm_np(v, bits)
        assert all(int(lib.dg_owner_perm(int(a), bits)) == int(b) for a, b in zip(v[:300], p[:300]))
        assert all(int(lib.dg_owner_perm_inv(int(b), bits)) == int(a) for a, b in zip(v[:300], p[:300]))
        if (1 << bits) <= (1 << 12):
            assert len(np.unique(p)) == len(v)
            assert p.max() < (1 << bits)


def test_owner_hash_balances_rmat_sources():
    from paper_2306_08252_b200 import rmat
    s, _ = rmat.rmat_edges(16, 1, 0, 1 << 18)
    own, _ = owner_of_np(s, 16, 8)
    counts = np.bincount(own, minlength=8)
    naive = np.bincount(s % 8, minlength=8)
    assert counts.max() / counts.mean() < 1.35, counts          # hashed: near-even
    assert naive.max() / naive.mean() > 2.0, naive              # v mod 8: the skew the hash removes


def _route_np(src, dst, bits, world):
    own, loc = owner_of_np(src, bits, world)
    order = np.argsort(own, kind="stable")
    counts = np.bincount(own, minlength=world)
    return loc[order], dst[order], order.astype(np.int64), counts


def _worker(rank, world, port, V, B, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = load_oracle()
        bits = owner_bits(V)
        # destinations stay GLOBAL ids: the CUDA store lifts its range check with dg_set_dst_limit; the
        # oracle stand-in is simply given V vertices (local ids are < local_vertex_count <= V)
        assert local_vertex_count(V, world) <= V
        store = CpuGraph(orc, "orc", V, B, 1 << 26)
        rng = np.random.default_rng(seed * 100 + rank)
        log = []
        for it in range(6):
            n = int(rng.integers(1, 3000))
            s = rng.integers(0, V, n).astype(np.uint32)
            d = rng.integers(0, V, n).astype(np.uint32)
            kind = "insert" if it % 3 != 2 else "delete"
            if kind == "delete" and log:
                ls, ld = log[-1]
                k = min(len(ls), n) // 2
                s[:k], d[:k] = ls[:k], ld[:k]
            log.append((s.copy(), d.copy()))
            ls_, d_, _, counts = _route_np(s, d, bits, world)
            (rs, rd), rc = exchange_buckets([torch.from_numpy(ls_.astype(np.int64)), torch.from_numpy(d_.astype(np.int64))],
                                            counts.tolist())
            assert sum(rc) == rs.numel()
            fn = store.insert_pairs if kind == "insert" else store.delete_pairs
            code = fn(rs.numpy().astype(np.uint32), rd.numpy().astype(np.uint32))
            assert agree_status(code, torch.device("cpu")) == 0
            q.put(("op", rank, it, kind, s, d))
        # query round trip: answers come back in the caller's order
        qs = rng.integers(0, V, 500).astype(np.uint32)
        qd = rng.integers(0, V, 500).astype(np.uint32)
        qs[:100], qd[:100] = log[0][0][:100], log[0][1][:100]
        ls_, d_, order, counts = _route_np(qs, qd, bits, world)
        (rs, rd), rc = exchange_buckets([torch.from_numpy(ls_.astype(np.int64)), torch.from_numpy(d_.astype(np.int64))],
                                        counts.tolist())
        ans = store.query(rs.numpy().astype(np.uint32), rd.numpy().astype(np.uint32))
        (back,), _ = exchange_buckets([torch.from_numpy(ans)], rc)
        out = np.zeros(len(qs), np.uint8)
        out[order] = back.numpy()
        q.put(("query", rank, qs, qd, out))
        # status agreement: one failing rank fails everyone
        assert agree_status(2 if rank == 1 else 0, torch.device("cpu")) == 2
        # batch atomicity ACROSS ranks (graph.hpp:168-171): check on every rank -> agree -> apply.  One bad
        # destination inside the share of whichever rank owns its source: the other rank's share is valid, yet
        # neither rank may apply anything.
        before = (store.active_edges(), store.degrees().copy())
        bs = np.arange(40, dtype=np.uint32) + 7
        bd = np.full(40, 3, dtype=np.uint32)
        if rank == 0:
            bd[11] = V + 5
        ls_, d_, _, counts = _route_np(bs, bd, bits, world)
        (rs, rd), _ = exchange_buckets([torch.from_numpy(ls_.astype(np.int64)), torch.from_numpy(d_.astype(np.int64))],
                                       counts.tolist())
        check = 2 if (rd.numpy() >= V).any() else 0           # the CPU stand-in of dg_check_batch_coo
        agreed = agree_status(check, torch.device("cpu"))
        assert agreed == 2
        if agreed == 0:
            store.insert_pairs(rs.numpy().astype(np.uint32), rd.numpy().astype(np.uint32))
        assert store.active_edges() == before[0] and np.array_equal(store.degrees(), before[1])
        q.put(("atomic", rank, int(check)))
        # export this rank's shard in GLOBAL ids
        off, dst = store.export_csr(sorted=True)
        lib = _lib.load()
        edges = []
        for lid in range(len(off) - 1):
            if off[lid + 1] > off[lid]:
                gsrc = int(lib.dg_owner_perm_inv(lid * world + rank, bits))
                edges.append((gsrc, dst[int(off[lid]):int(off[lid + 1])].copy()))
        q.put(("shard", rank, edges, store.active_edges()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 2])
def test_two_rank_routed_store_equals_single_store(seed):
    world, V, B = 2, 1000, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, B, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = []
    expected = world * (6 + 1 + 1 + 1)
    while len(msgs) < expected:
        msgs.append(q.get(timeout=120))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # replay on ONE oracle store: per iteration, rank 0's batch then rank 1's (disjoint sources per
    # owner make the order between ranks irrelevant for the multiset)
    orc = load_oracle()
    single = CpuGraph(orc, "orc", V, B, 1 << 26)
    ops = sorted([m for m in msgs if m[0] == "op"], key=lambda m: (m[2], m[1]))
    for _, _, _, kind, s, d in ops:
        assert (single.insert_pairs if kind == "insert" else single.delete_pairs)(s, d) == 0
    off, dst = single.export_csr(sorted=True)
    shards = [m for m in msgs if m[0] == "shard"]
    assert sum(m[3] for m in shards) == single.active_edges()
    seen = {}
    for _, _, edges, _ in shards:
        for gsrc, dsts in edges:
            assert gsrc not in seen
            seen[gsrc] = dsts
    for v in range(V):
        want = dst[int(off[v]):int(off[v + 1])]
        got = seen.get(v, np.zeros(0, np.uint32))
        assert np.array_equal(want, got), v
    for _, _, qs, qd, out in [m for m in msgs if m[0] == "query"]:
        assert np.array_equal(single.query(qs, qd), out)
    # the bad destination reached exactly ONE rank's share; both ranks held back (asserted in the workers)
    assert sorted(m[2] for m in msgs if m[0] == "atomic") == [0, 2]
