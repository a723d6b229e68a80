#!/usr/bin/env python
"""bench.py — batch edge insert/delete throughput on R-MAT scale 22 (BASELINE.json config[1]).

    python bench.py --gpus N --steps K --warmup W            # the CUDA path (this repo)
    python bench.py --impl reference --gpus N --steps K ...  # the reference's CPU path

One STEP = one pass of the hot path over one batch: the insert of a 1M-pair
R-MAT batch followed by the delete of the same batch, on a graph bulk-built from
the 16*2^22-edge R-MAT base (so a step processes 2*batch edge updates and the
graph keeps its size from step to step).  Every step uses a distinct batch.
Printed: ONE JSON line (rank 0).

  value      whole-job Medges/s with the batch already resident in HBM
             (CUDA events on the graph's stream, sum over the K steps, max over ranks);
             the two ops of a step are SUBMITTED (`dg_submit_insert_coo`,
             `dg_submit_delete_coo`: validated and applied on the device in stream order,
             no host wait between them) and flushed inside the step's bracket;
             `sync_calls` is the same pass through `dg_insert_batch_coo` /
             `dg_delete_batch_coo` (one host wait per op)
  e2e        the same steps through the public API with HOST (pinned) batches:
             the H2D copy of the pairs and the D2H read of the op status are inside
             the timed region
  roofline   the dominant kernel of the step (per-kernel CUDA-event timing via
             dg_profile_enable in a separate pass over the same steps): algorithmic
             bytes per launch / average launch duration vs MEASURED_PEAKS.json
  cpu_baseline  oracle/_ref (the unmodified reference, when it was compiled) or the
             oracle port, timed on this box's host cores on a bounded sample

N > 1 (torchrun): vertices are hash-partitioned by source over the ranks
(paper_2306_08252_b200.sharded); every rank generates its own 1M-pair slice of
the update stream and 16*2^22 base edges of a scale-(22+log2 N) graph, routes
them to the owners with an NCCL all-to-all and applies what it receives —
weak scaling, per-GPU work fixed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "batch edge insert+delete throughput (batch=1M, R-MAT s22)"
UNIT = "Medges/s"
STATUS_BYTES = 256  # sizeof(DeviceState) + sizeof(OpState): the per-op D2H status read (csrc/dg_api.cu op_end)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scale", type=int, default=22, help="R-MAT scale per GPU (22 = BASELINE config[1])")
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--block-size", type=int, default=32,
                    help="edge-block size B; 32 = one 128-byte line (0 = the reference's compute_block_size rule)")
    ap.add_argument("--pool-initial-fraction", type=float, default=0.0,
                    help="start with this fraction of the pre-sized pool and let the growth policy (80 %% trigger / 25 %% "
                         "rounds / on-demand, block_pool.hpp:162-189) commit the rest in place; 0 = pre-sized, no growth")
    ap.add_argument("--group", default="auto", choices=["auto", "count", "radix"],
                    help="how COO batches are grouped by source (GraphConfig.group); auto = chosen per batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=0,
                    help="batches in the cpu_baseline sample; 0 = all warm-up + timed batches, which also makes the "
                         "final states comparable (the `parity` block)")
    return ap.parse_args()


# --------------------------------------------------------------------------------------
# clocks (B200_PROFILING.md "clocks DURING the timed region")
# --------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock / throttle reasons sampled every 20 ms through NVML while the passes run."""

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[int, int, float, int]] = []
        self._stop = threading.Event()
        self.thread = None
        self.err = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:  # NVML missing: report it, never fail the bench
            self.err = f"nvml unavailable: {e}"

    def _run(self):
        nv, h = self.nv, self.handle
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((sm, mx, pw, rs))
            except Exception as e:
                self.err = str(e)
                return
            time.sleep(0.02)

    def stop(self) -> dict:
        self._stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"]}
        nv = self.nv
        names = {"hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                 "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                 "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                 "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4)}
        allbits = 0
        for smp in self.samples:
            allbits |= smp[3]
        sm = sorted(x[0] for x in self.samples)
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": max(x[1] for x in self.samples),
                "power_w_max": max(x[2] for x in self.samples), "samples": len(sm),
                "reasons": sorted(k for k, bit in names.items() if allbits & bit)}


# --------------------------------------------------------------------------------------
# algorithmic bytes per kernel launch
# --------------------------------------------------------------------------------------
def kernel_bytes(name: str, rep: dict, B: int) -> float | None:
    """Algorithmic HBM bytes of ONE launch of `name`.

    b = batch entries, T = touched sources, W = blocks of touched chains,
    S = slots of touched chains, M = compaction moves (all from dg_last_op_report)."""
    b, T = rep["batch_entries"], rep["touched_sources"]
    W, S, M = rep["blocks_scanned"], rep["slots_scanned"], rep["moved"]
    SL, ST = rep.get("slots_scanned_long", 0), rep.get("slots_scanned_tiny", 0)
    SF = rep.get("slots_scanned_fused", 0)
    if name.startswith("fused_delete"):
        # slab slots of the warp-owned sources + their next links + targets + per-source state (read + repaired)
        return 4 * SF + 4 * (SF // B) + 8 * b + 32 * T
    # the hub tiers: slab slots of the tier + handles + masks (their share of the 8b target bytes is not reported
    # per tier and is left out rather than charged three times)
    if name.startswith("match_long"):
        return 4 * SL + 8 * (SL // B)
    if name.startswith("match_med"):
        SM = S - SL - ST - SF
        return 4 * SM + 8 * (SM // B)
    if name.startswith("match_tiny"):
        return 4 * ST + 12 * (ST // B)
    if name.startswith("delete_holes_kernel"):
        return 12 * W + 8 * M + 32 * T                   # worklist + masks, hole records, per-source repair
    if name.startswith("delete_moves_kernel"):
        return 8 * W + 16 * M
    if name.startswith("sort_pass_kernel"):
        return 16 * b                                    # 8 B key read + 8 B key write
    if name.startswith("pack_coo_kernel"):
        return 16 * b                                    # 2 x u32 in, u64 key out
    if name.startswith("scan_kernel"):
        return 16 * b                                    # the largest scan of an op (run detection over the keys)
    if name.startswith("alloc_kernel<group"):
        return 4 * rep.get("vertices", 0) + 40 * T       # per-vertex counters + per-run outputs
    if name.startswith("alloc_kernel"):
        return 24 * T
    if name.startswith("group_"):
        return 16 * b
    if name.startswith("enumerate_"):
        return 12 * W + 12 * T                           # next[] reads + worklist writes
    if name.startswith("append_"):
        return 16 * b + 32 * T + 4 * (T + b // B)
    return None


# --------------------------------------------------------------------------------------
# CPU baseline (reference arm and the cpu_baseline leg)
# --------------------------------------------------------------------------------------
def cpu_reference_run(scale: int, edge_factor: int, batch: int, warmup: int, steps: int, threads: int,
                      block_size: int = 32, want_state: bool = False):
    """Times the reference's CPU implementation of the step on this host.

    Uses oracle/_ref/libdyngraph_ref.so (the unmodified reference headers behind
    oracle/ref_shim.cpp) when it was compiled, else the oracle port.  Batch
    construction (csr_from_pairs) is outside the timed region, as in the
    reference's own harness."""
    import ctypes as C
    import numpy as np
    from tests.drivers import CpuGraph, load_oracle, load_ref
    from paper_2306_08252_b200 import rmat

    orc = load_oracle()
    ref = load_ref()
    lib, pfx, kind = (ref, "ref", "reference") if ref is not None else (orc, "orc", "port")
    V, E = 1 << scale, edge_factor << scale
    thr = rmat.thresholds()

    def gen(seed, first, n):
        s, d = np.empty(n, np.uint32), np.empty(n, np.uint32)
        orc.orc_gen_rmat(scale, seed, first, n, thr[0], thr[1], thr[2],
                         C.c_void_p(s.ctypes.data), C.c_void_p(d.ctypes.data))
        return s, d

    bs, bd = gen(1, 0, E)
    B = block_size
    if B == 0 and ref is not None:
        out = C.c_uint32()
        if ref.ref_compute_block_size_coo(V, C.c_void_p(bs.ctypes.data), C.c_void_p(bd.ctypes.data), E, C.byref(out)) == 0:
            B = int(out.value)
    arena = max(8 << 30, 48 * E)  # 8 GiB at s22 (proj/README.md:111-113)
    t0 = time.perf_counter()
    g = CpuGraph(lib, pfx, V, B, arena, 0.5, True, threads)
    init_s = time.perf_counter() - t0
    sec = C.c_double()
    rc = g.insert_pairs(bs, bd, C.byref(sec))
    assert rc == 0, g.last_error()
    bulk_s = sec.value
    del bs, bd
    t_ins = t_del = 0.0
    for i in range(warmup + steps):
        s, d = gen(2, i * batch, batch)
        assert g.insert_pairs(s, d, C.byref(sec)) == 0
        ti = sec.value
        assert g.delete_pairs(s, d, C.byref(sec)) == 0
        td = sec.value
        if i >= warmup:
            t_ins += ti
            t_del += td
    state = None
    if want_state:   # observables oracle_compare checks (oracle.hpp:98-163), in their scale-independent form
        dg, ne = g.digest()
        state = {"active_edges": g.active_edges(), "digest": dg, "entries": ne, "degrees": g.degrees(),
                 "alive_vertices": g.alive_vertices(), "logical_size": g.logical_size()}
    g.close()
    total = t_ins + t_del
    return {
        "state": state,
        "kind": kind, "cores": threads, "block_size": B,
        "value": 2 * batch * steps / total / 1e6, "unit": UNIT,
        "insert_medges_s": batch * steps / t_ins / 1e6, "delete_medges_s": batch * steps / t_del / 1e6,
        "init_ms": init_s * 1e3, "bulk_insert_ms": bulk_s * 1e3, "ms_per_step": total / steps * 1e3,
        "sample": f"R-MAT s{scale} base graph ({E} edges) + {steps} steps of insert+delete batch={batch} "
                  f"after {warmup} warm-up, workers={threads}, batch construction untimed",
    }


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    # the B200 arm's config at N GPUs is weak-scaled (scale + log2 N, batch * N); the CPU run is a BOUNDED
    # sample of it (at most scale 24 / 4M-entry batches: ~2 minutes on 16 cores), described in `sample`
    world = max(1, args.gpus)
    ref_scale = min(args.scale + int(math.log2(world)), max(args.scale, 24))
    ref_batch = min(args.batch * world, max(args.batch, 4_000_000))
    r = cpu_reference_run(ref_scale, args.edge_factor, ref_batch, args.warmup, args.steps, threads, args.block_size)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(args, world, r["block_size"]),
        "insert_medges_s": r["insert_medges_s"], "delete_medges_s": r["delete_medges_s"],
        "bulk_init_ms": r["init_ms"] + r["bulk_insert_ms"],
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line)
    return 0


def workload_config(args, world: int, B: int, exchange: str = "p2p") -> dict:
    scale = args.scale + int(math.log2(world))
    return {
        "workload": f"R-MAT scale {scale} (a,b,c,d=.57,.19,.19,.05; V={1 << scale}, base E={args.edge_factor << scale}) "
                    f"bulk init + per step: insert batch={args.batch * world} then delete the same batch",
        "batch": args.batch * world, "scale": scale, "edge_factor": args.edge_factor, "block_size": B,
        "parallelism": "single GPU" if world == 1 else
        (f"source-hash partition over {world} GPUs, fused owner-routing + exchange kernel over peer memory (NVLink P2P)"
         if exchange == "p2p" else f"source-hash partition over {world} GPUs, device owner-bucket partition + NCCL all-to-all"),
        "l2": "256 MiB memset between steps (untimed) flushes L2; distinct batch every step",
    }


# --------------------------------------------------------------------------------------
# the CUDA arm
# --------------------------------------------------------------------------------------
def run_b200_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device — the product has no CPU path")
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("bench.py --gpus N>1 must be launched with torch.distributed.run (one rank per GPU)")
    # DG_BENCH_ONE_DEVICE=1: functional check of the N > 1 flow where only one GPU exists — every rank
    # uses cuda:0 and gloo carries the collectives (NCCL refuses two ranks on one device); the peers'
    # buffers are still mapped through CUDA IPC.  Timings of such a run mean nothing.
    one_device = bool(os.environ.get("DG_BENCH_ONE_DEVICE"))
    if one_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    force_sharded = bool(os.environ.get("DG_FORCE_SHARDED"))   # exercise the multi-GPU path on one GPU
    if world > 1 or force_sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        if one_device:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    from paper_2306_08252_b200 import DynamicGraph, GraphConfig, rmat
    from paper_2306_08252_b200._lib import load
    load()  # fail loudly if the CUDA library is missing

    scale = args.scale + int(math.log2(world))
    V = 1 << scale
    E_local = args.edge_factor << args.scale          # base edges GENERATED per rank
    b = args.batch                                    # update pairs GENERATED per rank per step
    thr = rmat.thresholds()
    stream = torch.cuda.Stream(device=dev)
    K, W = args.steps, args.warmup
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in peaks else "6650 GB/s (of fallback)"

    with torch.cuda.stream(stream):
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

        def i32(n):
            return torch.empty(n, dtype=torch.int32, device=dev)

        exchange_used = "p2p"
        # ---- graph construction + bulk init (timed) --------------------------------------
        if world == 1 and not os.environ.get("DG_FORCE_SHARDED"):
            gen = DynamicGraph(GraphConfig(device=local, pool_blocks=1024, stream=stream.cuda_stream), 1, 1)
            src, dst = i32(E_local), i32(E_local)
            gen.gen_rmat(scale, 1, 0, src, dst, thr)
            # 0 => compute_block_size (csr.hpp:77-88) on the base graph
            B = args.block_size or gen.compute_block_size_pairs(src)
            off = torch.empty(V + 1, dtype=torch.int64, device=dev)
            csr_dst = i32(E_local)
            gen.coo_to_csr(src, dst, V, off, csr_dst)
            del src, dst
            pool_blocks = int((E_local // B + V) * 1.25) + (4 * b) // B + 4096
            grow = {}
            if args.pool_initial_fraction > 0:   # queue pressure: the pool grows while the graph is built
                grow = {"pool_max_blocks": pool_blocks}
                pool_blocks = max(1024, int(pool_blocks * args.pool_initial_fraction))
            ws_hint = 48 * V + 8 * (E_local // B) + (64 << 20)   # scratch of the bulk build, reserved at create
            bulk_ms = []
            g = None
            for rep in range(3):
                if g is not None:
                    g.close()
                t0 = time.perf_counter()
                # (submit_inputs_ready: the update batches are generated and the stream synchronised before any timed pass)
                g = DynamicGraph(GraphConfig(device=local, pool_blocks=pool_blocks, stream=stream.cuda_stream,
                                             workspace_bytes=ws_hint, group=args.group, submit_inputs_ready=True, **grow), V, B)
                create_ms = (time.perf_counter() - t0) * 1e3
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                flush.zero_()
                e0.record(stream)
                g.bulk_init(off, csr_dst)
                e1.record(stream)
                stream.synchronize()
                bulk_ms.append((create_ms, e0.elapsed_time(e1)))
            bulk_rep = g.last_op_report()
            st = g.stats()
            bulk_kernels = None
            if not args.no_profile:   # one more, untimed, build with per-kernel events
                g.close()
                # (submit_inputs_ready: the update batches are generated and the stream synchronised before any timed pass)
                g = DynamicGraph(GraphConfig(device=local, pool_blocks=pool_blocks, stream=stream.cuda_stream,
                                             workspace_bytes=ws_hint, group=args.group, submit_inputs_ready=True, **grow), V, B)
                g.profile_enable(True)
                g.bulk_init(off, csr_dst)
                g.profile_enable(False)
                bulk_kernels = {k: round(ms * 1e3, 1) for k, (ms, _) in g.profile_report().items()}
            del off, csr_dst
            sharded = None
        else:
            from paper_2306_08252_b200.sharded import ShardedDynamicGraph
            gen = DynamicGraph(GraphConfig(device=local, pool_blocks=1024, stream=stream.cuda_stream), 1, 1)
            src, dst = i32(E_local), i32(E_local)
            gen.gen_rmat(scale, 1, rank * E_local, src, dst, thr)
            B = args.block_size or 2 * args.edge_factor
            pool_blocks = int((E_local // B + V // world) * 1.6) + (8 * b) // B + 4096
            # fused owner-routing + exchange over peer memory (default); the receive buffer holds one round
            # (the bulk build goes through it in one piece): 1.25x the per-rank share + slack.  The NCCL
            # all-to-all baseline takes over when the peer mapping cannot be set up or the store built
            # through the fused exchange does not hold exactly the edges that were generated (multiset
            # insert keeps every copy: the global live-edge count must equal world * E_local).
            from paper_2306_08252_b200 import EngineError
            want_exchange = os.environ.get("DG_EXCHANGE", "p2p")
            for exchange in ([want_exchange, "nccl"] if want_exchange != "nccl" else ["nccl"]):
                t0 = time.perf_counter()
                try:
                    sharded = ShardedDynamicGraph(GraphConfig(device=local, pool_blocks=pool_blocks, stream=stream.cuda_stream),
                                                  V, B, torch_stream=stream, exchange=exchange,
                                                  exchange_capacity=int(1.25 * max(E_local, b)) + (1 << 20))
                except EngineError as exc:   # (agreed by every rank: agree_status inside the constructor)
                    if rank == 0:
                        print(f"[bench] exchange={exchange} unavailable: {exc}", file=sys.stderr)
                    continue
                create_ms = (time.perf_counter() - t0) * 1e3
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                dist.barrier(); torch.cuda.synchronize()
                e0.record(stream)
                sharded.insert_pairs(src, dst)
                e1.record(stream)
                stream.synchronize()
                bulk_ms = [(create_ms, e0.elapsed_time(e1))]
                if sharded.active_edges() == world * E_local:
                    exchange_used = exchange
                    break
                if rank == 0:
                    print(f"[bench] exchange={exchange}: live edges {sharded.active_edges()} != {world * E_local}; falling back", file=sys.stderr)
                sharded.close()
                sharded = None
            if sharded is None:
                raise SystemExit("bench: the sharded store could not be built with any exchange")
            bulk_kernels = None
            g = sharded.local
            bulk_rep = g.last_op_report()
            st = g.stats()
            del src, dst

        # ---- update batches (device + pinned host copies) ---------------------------------------
        # A batch's FIRST application is the real workload: its delete also removes the base graph's own copies of
        # the pairs (~2.7 % of an R-MAT batch), which sit in the middle of chains and force compaction moves; a
        # second application of the same batch finds nothing but what it just appended.  So every headline pass
        # gets a set of batches no earlier pass has touched: set 0 the synchronous calls (and, second-hand, the
        # split / report / per-kernel passes), set 1 the submitted pass (`value`), set 2 the ingest-queue pass (`e2e`).
        nb = K + W
        n_sets = 3 if sharded is None else 1
        batches = []
        for i in range(n_sets * nb):
            s, d = i32(b), i32(b)
            gen.gen_rmat(scale, 2, (i * world + rank) * b, s, d, thr)
            batches.append((s, d))
        stream.synchronize()
        host_batches = [None] * len(batches)
        if not args.no_e2e:
            for j in ([k for k in range(nb)] + ([2 * nb + k for k in range(nb)] if n_sets == 3 else [])):
                s, d = batches[j]
                hs = torch.empty(b, dtype=torch.int32).pin_memory()
                hd = torch.empty(b, dtype=torch.int32).pin_memory()
                hs.copy_(s); hd.copy_(d)
                host_batches[j] = (hs.numpy().view(np.uint32), hd.numpy().view(np.uint32))
        target = sharded if sharded is not None else g

        def step(i, host=False, reports=False, submit=False, bset=0):
            s, d = (host_batches if host else batches)[bset * nb + i]
            if host and sharded is not None:   # the sharded API takes device tensors: the H2D copy is explicit
                s = torch.from_numpy(s.view(np.int32)).to(dev, non_blocking=True)
                d = torch.from_numpy(d.view(np.int32)).to(dev, non_blocking=True)
            if submit:   # dg_submit_*_coo: both ops enqueued without a host wait; the caller flushes
                g.submit_insert_pairs(s, d)
                g.submit_delete_pairs(s, d)
                return None, None
            target.insert_pairs(s, d)
            r_ins = g.last_op_report() if reports else None   # (kept out of the timed passes: host work between ops)
            target.delete_pairs(s, d)
            return r_ins, (g.last_op_report() if reports else None)

        def timed_pass(host: bool, submit: bool = False, bset: int = 0):
            """W warm-up + K timed steps; returns (sum of per-step device ms, per-step list, reports)."""
            for i in range(W):
                step(i, host, submit=submit, bset=bset)
            if submit:
                g.flush()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            per, reps = [], []
            t_wall = time.perf_counter()
            for i in range(W, W + K):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                reps.append(step(i, host, submit=submit, bset=bset))
                e1.record(stream)
                if submit:
                    assert g.flush() == 2   # both status read-backs are inside the bracket; raises if an op failed
                e1.synchronize()
                per.append(e0.elapsed_time(e1))
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t_wall) * 1e3
            total = torch.tensor([sum(per)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(total, op=dist.ReduceOp.MAX)
            return float(total.item()), per, reps, wall

        # split insert / delete device times (one extra untimed-for-the-metric pass of event pairs)
        def split_pass():
            ins = dele = 0.0
            for i in range(W, W + K):
                s, d = batches[i]
                flush.zero_()
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(stream); target.insert_pairs(s, d); e1.record(stream)
                target.delete_pairs(s, d); e2.record(stream); e2.synchronize()
                ins += e0.elapsed_time(e1); dele += e1.elapsed_time(e2)
            return ins, dele

        clocks = ClockSampler(local)
        clocks.start()
        # headline: the two ops of a step SUBMITTED back to back (no host round trip between insert and delete);
        # the same step through the synchronous calls is reported beside it
        sync_total_ms, _, _, sync_wall_ms = timed_pass(host=False)
        if sharded is None:
            total_ms, per_step, _, wall_ms = timed_pass(host=False, submit=True, bset=1)
            value_api = "dg_submit_insert_coo + dg_submit_delete_coo per step, dg_flush per step (device-resident batches)"
        else:
            total_ms, per_step, wall_ms = sync_total_ms, None, sync_wall_ms
            value_api = "ShardedDynamicGraph.insert_pairs / delete_pairs (synchronous per op)"
        reps = [step(i, reports=True) for i in range(W, W + K)]   # same batches again, untimed: op reports
        launches = sum(r[0]["kernel_launches"] + r[1]["kernel_launches"] for r in reps)
        if sharded is None:
            launches += 2 * K   # the timed pass submits its ops: one op_arm_kernel per op on top of the op's own kernels
        ins_ms, del_ms = split_pass()
        e2e = None
        if not args.no_e2e:
            # (1) the synchronous public calls, one per op, host batch in -> status out
            sync_ms, _, _, _ = timed_pass(host=True)
            e2e = {"value": 2 * b * world * K / (sync_ms * 1e-3) / 1e6, "unit": UNIT,
                   "ms_per_step": sync_ms / K,
                   "h2d_bytes_per_step": 2 * 8 * b, "d2h_bytes_per_step": 2 * STATUS_BYTES,
                   "api": "DynamicGraph.insert_pairs/delete_pairs -> dg_insert_batch_coo/dg_delete_batch_coo(DG_MEM_HOST), pinned host batches"}
            if sharded is None:
                # (2) the same stream of host batches through the ingest queue (dg_ingest_*): the copy of
                # batch k+1 overlaps op k.  One timed region over all K steps (no per-step brackets: the
                # copies cross step boundaries), every H2D copy and status read-back inside it; no L2
                # flush in this pass — every step's inputs come from host memory and a step touches
                # more graph data (> 230 MB) than the L2 holds.
                q = g.ingest(b, depth=int(os.environ.get("DG_E2E_DEPTH", "3")))
                for i in range(W):
                    hs, hd = host_batches[2 * nb + i]
                    q.submit("insert", hs, hd); q.submit("delete", hs, hd)
                q.flush()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                e0.record(stream)
                for i in range(W, W + K):
                    hs, hd = host_batches[2 * nb + i]
                    q.submit("insert", hs, hd); q.submit("delete", hs, hd)
                q.flush()
                e1.record(stream)
                e1.synchronize()
                pipe_wall = (time.perf_counter() - t0) * 1e3
                pipe_ms = max(e0.elapsed_time(e1), pipe_wall)   # the copy stream may start before e0 lands: take the larger
                q.close()
                e2e = {"value": 2 * b * K / (pipe_ms * 1e-3) / 1e6, "unit": UNIT, "ms_per_step": pipe_ms / K,
                       "h2d_bytes_per_step": 2 * 8 * b, "d2h_bytes_per_step": 2 * STATUS_BYTES,
                       "api": "BatchIngest.submit -> dg_ingest_stage_coo + dg_ingest_submit_insert/_delete, one dg_flush at the end: "
                              "pinned host batches, copies on their own stream overlapped with the ops, no host wait per "
                              "batch, one timed region over all steps",
                       "sync_api": {"value": 2 * b * K / (sync_ms * 1e-3) / 1e6, "ms_per_step": sync_ms / K,
                                    "api": "DynamicGraph.insert_pairs/delete_pairs(DG_MEM_HOST), copy serialised with the op"}}

        # ---- per-kernel timing pass (CUDA events around every launch) ---------------------------
        roofline, kernels = None, None
        if not args.no_profile:
            g.profile_enable(True)
            prof_reps = [step(i, reports=True) for i in range(W, W + K)]
            g.profile_enable(False)
            prof = g.profile_report()
            tot = sum(ms for ms, _ in prof.values()) or 1.0
            kernels = {k: {"ms_per_step": ms / K, "launches_per_step": n / K, "share": ms / tot}
                       for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0])}
            top = max(prof.items(), key=lambda kv: kv[1][0])
            name, (ms, n) = top
            # delete-side kernels use the delete report, insert-side the insert report
            ins_side = name.startswith(("append_", "alloc_kernel<group+plan"))
            per_launch = [kernel_bytes(name, r[0] if ins_side else r[1], B) for r in prof_reps]
            if per_launch[0] is not None and n:
                bytes_launch = sum(per_launch) / len(per_launch)
                avg_ms = ms / n
                ach = bytes_launch / (avg_ms * 1e-3) / 1e9
                traffic = None
                try:   # dram__bytes_read+write per launch of this kernel from the committed ncu --set full capture —
                    # only when that capture was taken on THIS workload (scale, batch, block size)
                    tfile = sorted((ROOT / "profiles").glob("*traffic.json"))[-1]
                    tj = json.loads(tfile.read_text())
                    if tj.get("workload") == {"scale": scale, "batch": b, "block_size": B, "n_gpus": world}:
                        traffic = tj.get(name.split("<")[0])
                except Exception:
                    pass
                roofline = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                            "frac": ach / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                            "bytes_per_launch": bytes_launch, "avg_launch_ms": avg_ms,
                            "launches_per_step": n / K, "share_of_step": ms / tot}

        clock_rec = clocks.stop()   # sampled over the timed, split, e2e and per-kernel passes
        final_st = g.stats()
        digest = g.digest()
        gpu_degrees = g.degrees() if sharded is None else None
        global_edges = sharded.active_edges() if sharded is not None else final_st["active_edges"]   # (collective)

    value = 2 * b * world * K / (total_ms * 1e-3) / 1e6
    r_ins, r_del = reps[-1]
    # op-level algorithmic bytes: insert 12b + 32T; delete 8b + 4S + S/8 + 32T
    a_ins = 12 * r_ins["batch_entries"] + 32 * r_ins["touched_sources"]
    a_del = 8 * r_del["batch_entries"] + 4 * r_del["slots_scanned"] + r_del["slots_scanned"] / 8 + 32 * r_del["touched_sources"]
    a_bulk = 8 * (V // world + 1) + 4 * bulk_rep["batch_entries"] * 2 + 16 * (V // world) + 8 * st["pool_blocks_in_use"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic", "config": workload_config(args, world, B, exchange_used),
        "insert_medges_s": b * world * K / (ins_ms * 1e-3) / 1e6, "delete_medges_s": b * world * K / (del_ms * 1e-3) / 1e6,
        "insert_ms": ins_ms / K, "delete_ms": del_ms / K,
        "bulk_init_ms": min(m for _, m in bulk_ms), "create_ms": min(c for c, _ in bulk_ms),
        "op_hbm": {"insert_gbs": a_ins / (ins_ms / K * 1e-3) / 1e9, "delete_gbs": a_del / (del_ms / K * 1e-3) / 1e9,
                   "bulk_init_gbs": a_bulk / (min(m for _, m in bulk_ms) * 1e-3) / 1e9, "peak_gbs": hbm_peak},
        "op_report": {"insert": r_ins, "delete": r_del},
        "graph": {"active_edges": global_edges, "rank0_active_edges": final_st["active_edges"],
                  "blocks_in_use": final_st["pool_blocks_in_use"],
                  "max_degree": final_st["max_degree"], "digest": f"{digest[0]:016x}",
                  "pool_blocks_created": final_st["pool_blocks_created"], "growth_count": final_st["growth_count"],
                  "memory": g.memory()},
        "wall_ms_per_step": wall_ms / K, "value_api": value_api,
        "passes": "every headline pass applies batches for the FIRST time (a delete then also removes the base graph's copies "
                  "of its pairs, mid-chain: compaction moves): sync_calls = set 0, value = set 1 (submitted), e2e = set 2 "
                  "(ingest queue); insert_ms / delete_ms, op_report, kernels and roofline come from later passes over set 0 "
                  "(second application: deletes only find what the step appended)",
        "sync_calls": {"value": 2 * b * world * K / (sync_total_ms * 1e-3) / 1e6, "ms_per_step": sync_total_ms / K,
                       "wall_ms_per_step": sync_wall_ms / K,
                       "api": "dg_insert_batch_coo + dg_delete_batch_coo (one host wait per op)"},
        "bulk_init_kernels_us": bulk_kernels, "clocks": clock_rec, "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "kernels": kernels,
    }
    parity_failed = False
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # The reference applies the SAME batches (every set, W + K each, once each: repeating a step on the GPU
            # does not change the outcome — a delete removes every copy of its pairs, base copies included) to
            # the SAME base graph; both stores must then hold the same multiset: live-edge count, per-vertex
            # degrees and the digest over (source, destination) copies.  Untimed on the GPU side.
            full = args.cpu_steps == 0
            r = cpu_reference_run(args.scale, args.edge_factor, args.batch, 0 if full else 1, n_sets * (K + W) if full else args.cpu_steps,
                                  os.cpu_count() or 1, B, want_state=full)
            line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                     "insert_medges_s", "delete_medges_s", "bulk_insert_ms", "init_ms")}
            if full and r["state"] is not None and gpu_degrees is not None:
                st_ref = r["state"]
                deg_equal = bool(np.array_equal(np.asarray(gpu_degrees, dtype=np.uint64), np.asarray(st_ref["degrees"], dtype=np.uint64)))
                ok = (deg_equal and st_ref["active_edges"] == final_st["active_edges"] and st_ref["digest"] == digest[0]
                      and st_ref["entries"] == digest[1] and st_ref["alive_vertices"] == final_st["alive_vertices"]
                      and st_ref["logical_size"] == final_st["logical_size"])
                line["parity"] = {"ok": ok, "against": r["kind"], "batches_applied": n_sets * (K + W),
                                  "active_edges": [final_st["active_edges"], st_ref["active_edges"]],
                                  "digest": [f"{digest[0]:016x}", f"{st_ref['digest']:016x}"],
                                  "entries": [digest[1], st_ref["entries"]], "degrees_equal": deg_equal,
                                  "what": "GPU store after every pass of this run vs the reference after the same base graph + "
                                          "the same batches: live edges, per-vertex degrees, digest of all (src, dst) copies"}
                parity_failed = not ok
        except Exception as e:  # the baseline is reported, never required for the CUDA number
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable",
                                    "sample": f"failed: {e}"}
    if rank == 0:
        emit(line)
    if world > 1 or force_sharded:
        dist.destroy_process_group()
    if parity_failed:
        print("bench.py: PARITY FAILURE against the reference (see the `parity` block)", file=sys.stderr)
        return 3
    return 0


_JSON_OUT = None   # the process's real stdout; everything else that writes to fd 1 goes to stderr


def emit(line: dict):
    print(json.dumps(line), file=_JSON_OUT or sys.stdout, flush=True)


def main():
    global _JSON_OUT
    args = parse_args()
    # stdout must carry exactly ONE JSON line: libraries that write to fd 1 on their own (NCCL prints its
    # version banner there) are moved to stderr for the whole run
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
