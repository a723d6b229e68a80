// dg_kernels.cuh — the graph kernels of libdyngraph_b200 (sm_100a).
//
// Data layout in HBM (SURVEY.md §8a maps each piece to the reference type it
// replaces):
//   vertex dictionary (a5, a4)  SoA: head[cap], tail[cap], deg[cap] (u32) and
//                               an alive bitmap (u32 words)
//   edge blocks (a2, a3)        dst slab u32[NB * B] + next[NB]; chains are
//                               kept COMPACT: every block but the tail is
//                               full, so deg alone gives block count and the
//                               tail fill (the reference's occupied/active
//                               counters and last_insert_offset are derived)
//   edge queue (a6)             ring u32[NB] of free handles with unwrapped
//                               64-bit front/rear cursors in DeviceState
//
// All kernels are memory-bound integer work: no tensor cores.  Work is
// decomposed FLAT (one warp per edge block / append unit) so R-MAT hubs do
// not serialise; the only chain walk (enumerate_walk_kernel) confirms up to
// 32 consecutive handles per round trip.
#pragma once

#include "dg_device.cuh"

namespace dg {

struct GraphView {
  uint32_t* head;
  uint32_t* tail;
  uint32_t* deg;
  uint32_t* alive;  // bitmap
  uint32_t* slab;
  uint32_t* next;
  uint32_t* ring;
  unsigned long long ring_cap;  // == NB
  unsigned long long ring_identity;  // ring[p] == p for every queue position p below this (never-recycled prefix)
  uint32_t B;
  int bsh;             // log2(B) when B is a power of two, else -1
  uint32_t mw;         // 32-bit match-mask words per block: ceil(B / 32)
  uint32_t size;       // logical size at launch
  uint32_t dst_limit;  // destinations must be < dst_limit (== size single-GPU)
  int reclaim;
  DeviceState* st;
};

struct BatchView {
  const unsigned long long* keys;  // sorted (src<<32|dst), or nullptr on the CSR path
  const uint32_t* dsts;            // CSR path values, or nullptr
  const uint32_t* run_src;         // nullptr => run r is vertex r
  const uint32_t* run_start;       // first entry of run r
  const uint32_t* run_end;         // one past its last entry (== run_start + 1 when runs are laid out in order)
};

__device__ __forceinline__ uint32_t batch_value(const BatchView& b, uint32_t i) {
  return b.keys ? (uint32_t)b.keys[i] : b.dsts[i];
}
__device__ __forceinline__ uint32_t batch_src(const BatchView& b, uint32_t r) {
  return b.run_src ? b.run_src[r] : r;
}
__device__ __forceinline__ uint32_t run_len(const BatchView& b, uint32_t r) {
  return b.run_end[r] - b.run_start[r];
}
__device__ __forceinline__ uint32_t ceil_div(uint32_t a, uint32_t b) { return (a + b - 1) / b; }
// x / B and ceil(x / B) with the shift fast path (B = 32 is the native block: one 128-byte line)
__device__ __forceinline__ uint32_t div_b(const GraphView& g, uint32_t x) {
  return g.bsh >= 0 ? (x >> g.bsh) : (x / g.B);
}
__device__ __forceinline__ uint32_t blocks_for(const GraphView& g, uint32_t x) {
  return div_b(g, x + g.B - 1);
}

__device__ __forceinline__ unsigned long long block_reduce_sum(unsigned long long v,
                                                               unsigned long long* s_warp) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  __syncthreads();
  if (lane_id() == 0) s_warp[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_warp[w];
  return t;  // valid in thread 0
}

// ---- asynchronous global -> shared staging (LDGSTS) -------------------------------
// The match kernels stage up to 32 edge blocks of 128 bytes per warp in shared
// memory: the copies are all issued before anything waits (no registers tied
// up, no unrolled code), then a rolled loop consumes them.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// Stages blocks u in [0, 32) whose bit is set in `want` (B = 32): handle of
// block u in lane u; 8 lanes move one 128-byte block, 4 blocks per instruction.
// Layout: the 16-byte chunk c of block u sits at chunk position (c + u) & 7 of
// row u, so that afterwards LANE u can read ITS block with eight conflict-free
// 16-byte shared loads (block_chunk) — the compare then runs one block per
// lane with no cross-lane traffic.
__device__ __forceinline__ void stage_blocks32(const GraphView& g, uint32_t (*dst)[32], uint32_t hd_lane,
                                               unsigned want) {
  const int lane = lane_id();
  const int sub = lane >> 3, c = lane & 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int u = 4 * i + sub;
    const uint32_t hu = __shfl_sync(kFull, hd_lane, u);
    if ((want >> u) & 1u) cp_async16(&dst[u][((c + u) & 7) * 4], g.slab + (unsigned long long)hu * 32u + c * 4);
  }
}
__device__ __forceinline__ uint4 block_chunk(uint32_t (*stg)[32], int u, int c) {
  return *reinterpret_cast<const uint4*>(&stg[u][((c + u) & 7) * 4]);
}
__device__ __forceinline__ uint32_t block_slot(uint32_t (*stg)[32], int u, uint32_t s) {
  return stg[u][((((s >> 2) + u) & 7) << 2) | (s & 3)];
}
// Any block size: pass p stages words [32p, min(32p + 32, B)) of up to 32 blocks into the same
// swizzled rows, one 4-byte cp.async per lane and block (blocks of B != 32 words are not 16-byte
// aligned), so the lane-per-block compare below runs unchanged on 32-word rows; a block of B > 32
// slots takes ceil(B / 32) passes and one 32-bit mask word per pass.
__device__ __forceinline__ void stage_rows32(const GraphView& g, uint32_t (*dst)[32], uint32_t hd_lane,
                                             unsigned want, uint32_t p) {
  const int lane = lane_id();
  const uint32_t nwords = min(32u, g.B - 32u * p);
#pragma unroll 4
  for (int u = 0; u < 32; ++u) {
    const uint32_t hu = __shfl_sync(kFull, hd_lane, u);
    if (((want >> u) & 1u) && (uint32_t)lane < nwords)
      cp_async4(&dst[u][(((((uint32_t)lane >> 2) + u) & 7) << 2) | ((uint32_t)lane & 3)],
                g.slab + (unsigned long long)hu * g.B + 32u * p + lane);
  }
}
__device__ __forceinline__ uint32_t low_bits32(uint32_t n) { return n >= 32u ? 0xFFFFFFFFu : ((1u << n) - 1u); }
// second, independent hash for the membership filters
__device__ __forceinline__ uint32_t filter_hash(uint32_t x, int bits) { return (x * 0x85EBCA6Bu) >> (32 - bits); }

// ---------------------------------------------------------------------------
// submitted (asynchronous) ops: arming the op words on the device
// ---------------------------------------------------------------------------
// A submitted op does not wait for the host between ops, so "a failed batch reports before the next
// one mutates" (graph.hpp:168-171) is kept on the device: the op words of the NEXT op are installed by
// this one-thread kernel (they travel as the kernel argument — no host buffer to keep alive), which
// first looks at the words the previous op left behind.  chain != 0: the previous op of the stream was
// submitted too and has not been reported — if it failed (or an earlier one did: the poison word),
// this op starts out rejected and every kernel of it returns at its first line.
// pre: the words an EARLY group_count of this op reported into (it ran beside the previous op's last kernel, before
// these op words existed): its verdict is merged here.
__global__ void op_arm_kernel(OpState fresh, DeviceState* st, OpState* op, int chain, const OpState* pre) {
  if (pre != nullptr && pre->err != 0) {
    fresh.err = pre->err;
    fresh.err_detail = pre->err_detail;
    fresh.err_index = pre->err_index;
  }
  if (chain && (st->poison != 0 || op->err != 0)) {
    st->poison = 1;
    fresh.err = 3u;   // DG_ERR_ENGINE
    fresh.err_detail = kErrSkipped;
  } else {
    st->poison = 0;
  }
  *op = fresh;
}

// The op's status {DeviceState, OpState} goes to its pinned host slot by STORES from this one-warp kernel (mapped
// host memory), not by a device-to-host memcpy: a copy-engine transfer queues behind whatever the engine is busy
// with — next to an ingest queue streaming 8 MB batches, a 256-byte status copy waited ~150 us per op and serialised
// the ops with the batch copies.
__global__ void op_publish_kernel(const unsigned long long* __restrict__ dev_words, unsigned long long* host_words, int n_words) {
  for (int i = threadIdx.x; i < n_words; i += blockDim.x) host_words[i] = dev_words[i];
  __threadfence_system();
}

__global__ void op_pre_arm_kernel(OpState* pre) {
  pre->err = 0u;
  pre->err_detail = 0u;
  pre->err_index = ~0ull;
}

// ---------------------------------------------------------------------------
// init
// ---------------------------------------------------------------------------
// block_pool.hpp:242-247 pushes one handle per block; here one coalesced store.
__global__ void ring_fill_kernel(uint32_t* __restrict__ ring, unsigned long long nb) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (unsigned long long)gridDim.x * blockDim.x)
    ring[i] = (uint32_t)i;
}

// Pool growth (try_grow, block_pool.hpp:252-264): the queue window [front, rear) moves to a ring
// of the new capacity and the `grant` new handles are pushed behind it.
__global__ void ring_relayout_kernel(const uint32_t* __restrict__ old_ring, unsigned long long old_cap,
                                     uint32_t* __restrict__ new_ring, unsigned long long new_cap,
                                     unsigned long long front, unsigned long long rear,
                                     uint32_t first_new, unsigned long long grant) {
  const unsigned long long live = rear - front;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < live + grant;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long pos = front + i;
    new_ring[pos % new_cap] = i < live ? old_ring[pos % old_cap] : first_new + (uint32_t)(i - live);
  }
}

// vertex_dictionary.hpp:84-91 (append_slots): fresh alive vertices with empty
// sentinels for ids [first, first + count).
__global__ void vertex_init_kernel(GraphView g, uint32_t first, uint32_t count) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += gridDim.x * blockDim.x) {
    const uint32_t v = first + i;
    g.head[v] = kNull;
    g.tail[v] = kNull;
    g.deg[v] = 0;
    atomicOr(&g.alive[v >> 5], 1u << (v & 31));
  }
}

// ---------------------------------------------------------------------------
// COO staging: validate + pack (src,dst) -> 64-bit keys
// ---------------------------------------------------------------------------
enum PackMode : int { kPackInsert = 0, kPackDelete = 1, kPackQuery = 2 };

// csr.hpp:67-72 (destination range), graph.hpp:322-327 (dead source on insert).
// Query mode never fails: ids outside the graph are clamped to values no
// stored entry can equal (graph.hpp:229 unknown source -> false).
// The radix-sort digit histograms of the keys are accumulated in the same
// pass (hist != nullptr), so the sort never re-reads the batch for them.
template <int kMode, bool kWithIndex>
__global__ void __launch_bounds__(256)
pack_coo_kernel(GraphView g, const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                uint32_t n, unsigned long long* __restrict__ keys, uint32_t* __restrict__ index,
                SortPlan plan, unsigned int* __restrict__ hist, OpState* op) {
  __shared__ unsigned int s_hist[kMaxPasses * kRadix];
  if (hist != nullptr) hist_clear(s_hist, plan);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = src[i], d = dst[i];
    if (kMode == kPackQuery) {
      if (s >= g.size) s = g.size;
      if (d >= g.dst_limit) d = g.dst_limit;
    } else {
      if (s >= g.size) {
        set_error(op, 2, kErrSrcRange, i);
        s = 0;
      } else if (kMode == kPackInsert && !bit_test(g.alive, s)) {
        set_error(op, 2, kErrDeadSource, i);
      }
      if (d >= g.dst_limit) set_error(op, 2, kErrDstRange, i);
    }
    const unsigned long long k = ((unsigned long long)s << 32) | d;
    keys[i] = k;
    if (kWithIndex) index[i] = i;
    if (hist != nullptr) hist_add(s_hist, plan, k);
  }
  if (hist != nullptr) hist_flush(s_hist, plan, hist);
}

// ---------------------------------------------------------------------------
// COO staging, counting variant: group the batch by source with a per-vertex
// counter array instead of a radix sort — count, scan over the vertices,
// scatter.  Used when the vertex count is within a small multiple of the batch
// (the scan is O(V)); the radix path covers small batches on large graphs.
// The order of a source's entries inside its group is the arrival order of the
// atomics, which the multiset semantics do not observe.
// ---------------------------------------------------------------------------
// Counter slot of a source.  Low vertex ids are the hubs of an R-MAT graph: a
// direct index would pile 10+% of the atomics onto a handful of 128-byte lines
// (measured: 26.5 us vs 16.3 us per 1M atomics), so the index is scattered by an
// odd multiplier — a bijection on [0, 2^bits).  Slot 2^bits collects the unknown
// sources a query batch is clamped to.
struct GroupIndex {
  uint32_t mask;   // 2^bits - 1, 2^bits >= vertex count
  uint32_t size;   // vertex count
  __device__ __forceinline__ uint32_t operator()(uint32_t s) const {
    return s >= size ? mask + 1u : ((s * 0x9E3779B1u) & mask);
  }
};

// validate (csr.hpp:67-72, graph.hpp:322-327) + count entries per source.
// Four entries per thread, each stage issued for all four before the next
// (loads -> alive-bit loads -> atomics), so the dependent round trips overlap.
constexpr int kGroupItems = 4;
template <int kMode>
__global__ void __launch_bounds__(256)
group_count_kernel(GraphView g, GroupIndex gi, const uint32_t* __restrict__ src,
                   const uint32_t* __restrict__ dst, uint32_t n, uint32_t* __restrict__ cnt,
                   uint32_t* __restrict__ rank, OpState* op) {
  const uint32_t base = blockIdx.x * (256 * kGroupItems) + threadIdx.x;
  const uint32_t op_err = op->err;   // (an op submitted behind a failed one starts out rejected; tested after the first loads are in flight)
  uint32_t s[kGroupItems], d[kGroupItems];
  bool ok[kGroupItems];
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) {
    const uint32_t i = base + q * 256;
    ok[q] = i < n;
    s[q] = ok[q] ? src[i] : 0u;
    d[q] = ok[q] ? dst[i] : 0u;
  }
  if (op_err) return;
  uint32_t aw[kGroupItems];
  if (kMode == kPackInsert) {
#pragma unroll
    for (int q = 0; q < kGroupItems; ++q) aw[q] = (ok[q] && s[q] < g.size) ? g.alive[s[q] >> 5] : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) {
    if (!ok[q]) continue;
    const uint32_t i = base + q * 256;
    if (kMode == kPackQuery) {
      if (s[q] >= g.size) s[q] = g.size;  // cnt has size + 1 entries: the extra one collects unknown sources
    } else {
      if (s[q] >= g.size) {
        set_error(op, 2, kErrSrcRange, i);
        ok[q] = false;
      } else if (kMode == kPackInsert && !((aw[q] >> (s[q] & 31)) & 1u)) {
        set_error(op, 2, kErrDeadSource, i);
        ok[q] = false;
      }
      if (d[q] >= g.dst_limit) {
        set_error(op, 2, kErrDstRange, i);
        ok[q] = false;
      }
    }
  }
  // the returned count is the entry's rank inside its source's group
  uint32_t rk[kGroupItems];
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q)
    if (ok[q]) rk[q] = atomicAdd(&cnt[gi(s[q])], 1u);
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q)
    if (ok[q]) rank[base + q * 256] = rk[q];
}

template <int kMode, bool kWithIndex>
__global__ void __launch_bounds__(256)
group_scatter_kernel(GraphView g, GroupIndex gi, const uint32_t* __restrict__ src,
                     const uint32_t* __restrict__ dst, uint32_t n, const uint32_t* __restrict__ start,
                     const uint32_t* __restrict__ rank, uint32_t* __restrict__ out_dst,
                     uint32_t* __restrict__ out_index, OpState* op) {
  if (op->err) return;  // a rejected batch was counted only partially
  const uint32_t base = blockIdx.x * (256 * kGroupItems) + threadIdx.x;
  uint32_t s[kGroupItems], d[kGroupItems], pos[kGroupItems];
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) {
    const uint32_t i = base + q * 256;
    s[q] = i < n ? src[i] : 0u;
    d[q] = i < n ? dst[i] : 0u;
    pos[q] = i < n ? rank[i] : 0u;
    if (kMode == kPackQuery) {
      if (s[q] >= g.size) s[q] = g.size;
      if (d[q] >= g.dst_limit) d[q] = g.dst_limit;
    }
  }
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q)
    if (base + q * 256 < n) pos[q] += start[gi(s[q])];
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) {
    if (base + q * 256 < n) {
      out_dst[pos[q]] = d[q];
      if (kWithIndex) out_index[pos[q]] = base + q * 256;
    }
  }
  // consumers that started beside this kernel (fused_delete_kernel) wait for the count of finished CTAs
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&op->scatter_ctas, 1u);
  }
}

// ---------------------------------------------------------------------------
// run detection over sorted keys (scan functors)
// ---------------------------------------------------------------------------
struct RunsIn {
  const unsigned long long* keys;
  __device__ unsigned long long operator()(unsigned long long i) const {
    if (i == 0) return 1ull;
    return (uint32_t)(keys[i] >> 32) != (uint32_t)(keys[i - 1] >> 32) ? 1ull : 0ull;
  }
};
struct RunsOut {
  const unsigned long long* keys;
  uint32_t* run_start;
  uint32_t* run_src;
  __device__ void operator()(unsigned long long i, unsigned long long excl,
                             unsigned long long v) const {
    if (v) {
      run_start[excl] = (uint32_t)i;
      run_src[excl] = (uint32_t)(keys[i] >> 32);
    }
  }
};
struct RunsFin {
  uint32_t* run_start;
  OpState* op;
  uint32_t n;
  __device__ void operator()(unsigned long long total) const {
    run_start[total] = n;
    op->n_runs = total;
  }
};

// ---------------------------------------------------------------------------
// CSR batch validation (csr.hpp:49-73 + graph.hpp:320-328)
// ---------------------------------------------------------------------------
__global__ void csr_validate_offsets_kernel(GraphView g, const unsigned long long* __restrict__ offsets,
                                            uint32_t n_offsets, unsigned long long n_edges,
                                            int check_dead_source, uint32_t* __restrict__ run_start,
                                            OpState* op) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_offsets;
       i += gridDim.x * blockDim.x) {
    const unsigned long long o = offsets[i];
    if (i == 0 && o != 0) set_error(op, 2, kErrOffsetsStart, 0);
    if (i + 1 == n_offsets && o != n_edges) set_error(op, 2, kErrOffsetsEnd, i);
    if (i + 1 < n_offsets) {
      const unsigned long long nx = offsets[i + 1];
      if (nx < o) set_error(op, 2, kErrOffsetsMonotone, i + 1);
      else if (check_dead_source && nx > o && !bit_test(g.alive, i))
        set_error(op, 2, kErrDeadSource, i);
    }
    run_start[i] = (uint32_t)(o > n_edges ? n_edges : o);
  }
}

__global__ void validate_dsts_kernel(GraphView g, const uint32_t* __restrict__ dsts, uint32_t n,
                                     OpState* op) {
  bool bad = false;
  uint32_t first_bad = 0xFFFFFFFFu;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (dsts[i] >= g.dst_limit && !bad) {
      bad = true;
      first_bad = i;
    }
  }
  if (bad) set_error(op, 2, kErrDstRange, first_bad);
}

// Number of vertices with a non-empty run (compute_block_size, csr.hpp:79-81).
__global__ void count_nonzero_runs_kernel(const uint32_t* __restrict__ run_start, uint32_t n_runs,
                                          OpState* op) {
  __shared__ unsigned long long s_warp[32];
  unsigned long long c = 0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_runs; r += gridDim.x * blockDim.x)
    c += run_start[r + 1] > run_start[r];
  const unsigned long long t = block_reduce_sum(c, s_warp);
  if (threadIdx.x == 0 && t) atomicAdd(&op->aux0, t);
}

// CSR -> sorted-by-source keys (delete path needs (src,dst) keys to sort).
// One warp per 32 consecutive edges; the warp finds the run range once.
__global__ void csr_expand_kernel(const uint32_t* __restrict__ run_start, uint32_t n_runs,
                                  const uint32_t* __restrict__ dsts, uint32_t n,
                                  unsigned long long* __restrict__ keys, const OpState* op) {
  if (op->err) return;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nchunks = (n + 31) / 32;
  for (uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nwarps) {
    const uint32_t i0 = c * 32;
    const uint32_t i1 = min(n, i0 + 32) - 1;
    const uint32_t r_lo = warp_find_run(run_start, n_runs, i0);
    const uint32_t r_hi = warp_find_run(run_start, n_runs, i1);
    const uint32_t i = i0 + lane_id();
    if (i < n) {
      // largest r in [r_lo, r_hi] with run_start[r] <= i
      uint32_t lo = r_lo, hi = r_hi + 1;
      while (hi - lo > 1) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (run_start[mid] <= i) lo = mid; else hi = mid;
      }
      keys[i] = ((unsigned long long)lo << 32) | dsts[i];
    }
  }
}

// ---------------------------------------------------------------------------
// insert: plan (graph.hpp:135-160).  Everything the plan hands out is a
// disjoint range (append units, queue positions, and — on the counting path —
// run slots and group slots), so it runs as ONE alloc_kernel pass:
//   word a = [63:32] touched sources (runs), [31:0] batch entries
//   word b = [63:32] append units,           [31:0] fresh blocks
// (The In functors are PURE loads: the kernel issues a thread's 8 items back to
// back, and a store in between would serialise them.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long plan_word(const GraphView& g, uint32_t d, uint32_t c) {
  // space left in the tail block == block_size - last_insert_offset (graph.hpp:149-150)
  const uint32_t nb = blocks_for(g, d);
  const uint32_t space = nb * g.B - d;
  const uint32_t fill = min(c, space);
  const uint32_t need = blocks_for(g, c - fill);  // graph.hpp:152-153
  const uint32_t units = need + (fill > 0 ? 1u : 0u);
  return ((unsigned long long)units << 32) | need;
}

// BatchPlan as the reference returns it (graph.hpp:33-39, :135-160): per vertex the free slots of its last-insert
// block, the fresh blocks the batch needs, and their INCLUSIVE prefix sum in vertex order (the pop schedule) — an
// ordered scan, unlike the range allocation the ops themselves use.
struct BatchPlanIn {
  GraphView g;
  const uint32_t* run_start;   // 32-bit copy of the validated offsets
  __device__ unsigned long long operator()(unsigned long long v) const {
    const uint32_t c = run_start[v + 1] - run_start[v];
    return plan_word(g, g.deg[v], c) & 0xFFFFFFFFull;
  }
};
struct BatchPlanOut {
  GraphView g;
  unsigned long long* blocks_required;
  unsigned long long* prefix_sum;
  uint32_t* space_remaining;
  __device__ void operator()(unsigned long long v, unsigned long long excl, unsigned long long need) const {
    const uint32_t d = g.deg[v];
    blocks_required[v] = need;
    prefix_sum[v] = excl + need;
    space_remaining[v] = blocks_for(g, d) * g.B - d;   // block_size - last_insert_offset; 0 without a block (graph.hpp:149-150)
  }
};
struct BatchPlanFin {
  OpState* op;
  __device__ void operator()(unsigned long long total) const { op->total_need = total; }
};

struct PlanAux {
  uint32_t d, tail;  // degree / tail block of the source before the batch
};
struct PlanArrays {
  uint32_t* run_deg;   // snapshots of deg/tail: append publishes the new values while other
  uint32_t* run_tail;  // units of the same source still need the old ones
  uint32_t* unit_off;
  uint32_t* blk_off;
  uint32_t* unit_run;  // every unit records its run so the append kernel never searches
  __device__ void write(uint32_t r, const PlanAux& x, unsigned long long excl_b, unsigned long long val_b) const {
    run_deg[r] = x.d;
    run_tail[r] = x.tail;
    const uint32_t uo = (uint32_t)(excl_b >> 32);
    unit_off[r] = uo;
    blk_off[r] = (uint32_t)excl_b;
    const uint32_t units = (uint32_t)(val_b >> 32);
    for (uint32_t j = 0; j < units; ++j) unit_run[uo + j] = r;
  }
};

// plan over already-grouped runs (radix path, CSR batches)
struct PlanIn {
  using Aux = PlanAux;
  GraphView g;
  BatchView b;
  __device__ Sum2 operator()(unsigned long long r64, Aux& x) const {
    const uint32_t r = (uint32_t)r64;
    const uint32_t c = run_len(b, r);
    const uint32_t v = batch_src(b, r);
    x.d = c ? g.deg[v] : 0u;
    x.tail = c ? g.tail[v] : kNull;
    return Sum2{0ull, c ? plan_word(g, x.d, c) : 0ull};
  }
};
struct PlanOut {
  PlanArrays arr;
  __device__ void operator()(unsigned long long r, unsigned long long, unsigned long long excl_b,
                             Sum2 v, const PlanAux& x) const {
    arr.write((uint32_t)r, x, excl_b, v.b);
  }
};
// plan fused with the counting group-by: one pass over the batch ENTRIES.  The
// entry that drew rank 0 in group_count_kernel speaks for its source: it reads
// the source's count and state and takes the source's queue positions — no
// pass over the vertices, no run list.  What the append needs per source goes
// to `info`, indexed like the counters.
struct SourceInfo {   // 16 bytes, one gather per entry in append_entries_kernel
  uint32_t d;         // degree before the batch
  uint32_t tail;      // tail block before the batch
  uint32_t blk_off;   // first queue position (relative to the old front) of its fresh blocks
  uint32_t c;         // entries the batch holds for it
};
struct GroupPlanIn {
  using Aux = PlanAux;
  GraphView g;
  GroupIndex gi;
  const uint32_t* src;
  const uint32_t* rank;
  const uint32_t* cnt;
  __device__ Sum2 operator()(unsigned long long i, Aux& x) const {
    const uint32_t s = src[i];
    const bool rep = rank[i] == 0;
    const uint32_t c = rep ? cnt[gi(s)] : 0u;
    x.d = rep ? g.deg[s] : 0u;
    x.tail = rep ? g.tail[s] : kNull;
    return Sum2{c ? ((1ull << 32) | c) : 0ull, c ? (plan_word(g, x.d, c) & 0xFFFFFFFFull) : 0ull};
  }
};
struct GroupPlanOut {
  GroupIndex gi;
  const uint32_t* src;
  uint4* info;
  uint32_t* cnt;   // the source's counter is handed back zeroed (the counter array is never cleared between ops)
  __device__ void operator()(unsigned long long i, unsigned long long, unsigned long long excl_b,
                             Sum2 val, const PlanAux& x) const {
    const uint32_t c = (uint32_t)val.a;
    if (c == 0) return;
    const uint32_t slot = gi(src[i]);
    info[slot] = make_uint4(x.d, x.tail, (uint32_t)excl_b, c);
    cnt[slot] = 0u;
  }
};
struct PlanFin {
  GraphView g;
  OpState* op;
  unsigned long long n_edges;
  int set_runs;        // counting path: the pass also counted the runs
  int commit_globals;  // COO path: validation is complete, commit here; CSR path: commit_insert_kernel
  __device__ void operator()(unsigned long long total_a, unsigned long long total_b, unsigned int) const {
    const unsigned long long need = total_b & 0xFFFFFFFFull;
    const unsigned long long units = total_b >> 32;
    if (set_runs) op->n_runs = total_a >> 32;
    op->n_units = units;
    op->total_need = need;
    op->n_edges = n_edges;
    DeviceState* st = g.st;
    // ensure_available (block_pool.hpp:177-189): fail BEFORE any mutation
    if (need > st->rear - st->front) {
      op->err = 3;
      op->err_detail = kErrPoolUnderflow;
      op->err_index = need - (st->rear - st->front);
      return;
    }
    op->front_old = st->front;
    if (commit_globals) {
      st->front += need;              // commit_front (block_pool.hpp:162-166)
      st->active_edges += n_edges;    // graph.hpp:186
    }
  }
};

// ring slot of queue position front_old + off, off < ring_cap (pop_range, block_pool.hpp:148-158).
// lap0: front_old < ring_identity, i.e. the queue still serves never-recycled handles.  Positions
// below ring_identity were written once (ring[p] = p, ring_fill_kernel / pool growth) and can only
// be overwritten by pushes a full lap later, so there the handle IS the position: no load, no
// dependent latency (a fresh pool behaves like a bump allocator until its first wrap).
__device__ __forceinline__ uint32_t ring_at(const GraphView& g, unsigned long long base_mod,
                                            unsigned long long off, bool lap0 = false) {
  unsigned long long i = base_mod + off;
  if (lap0 && i < g.ring_identity) return (uint32_t)i;
  if (i >= g.ring_cap) i -= g.ring_cap;
  return g.ring[i];
}

// ---------------------------------------------------------------------------
// insert: append (graph.hpp:333-372).  A unit is either the free tail of a
// source's last block or one fresh block.  A warp takes 32 consecutive units:
// each lane resolves ONE unit's metadata and links (one round of independent
// loads for 32 units), then the warp copies the 32 units' entries with
// coalesced loads/stores, four units in flight.
//   kValidateDst: CSR path — the destination range check (csr.hpp:67-72) is
//     fused into this single pass over the batch; entries land only in free
//     slots (tail space beyond deg, blocks still owned by the queue), so a
//     late failure leaves nothing observable and commit_insert_kernel never runs.
//   kCommit: COO path — validation finished before the sort, so the last unit
//     of a source publishes deg/tail here.
// ---------------------------------------------------------------------------
template <bool kValidateDst, bool kCommit>
__global__ void __launch_bounds__(256)
append_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ unit_off,
              const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ unit_run,
              const uint32_t* __restrict__ run_deg, const uint32_t* __restrict__ run_tail,
              OpState* op) {
  if (op->err) return;
  const uint32_t U = (uint32_t)op->n_units;
  const unsigned long long base_mod = op->front_old % g.ring_cap;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (uint32_t u0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u; u0 < U; u0 += nwarps * 32u) {
    const uint32_t u = u0 + lane;
    uint32_t blk = 0, off0 = 0, src0 = 0, cnt = 0;
    if (u < U) {
      const uint32_t r = unit_run[u];
      const uint32_t j = u - unit_off[r];
      const uint32_t v = batch_src(b, r);
      const uint32_t rs = b.run_start[r];
      const uint32_t c = b.run_end[r] - rs;
      const uint32_t d = run_deg[r];
      const uint32_t nb_old = blocks_for(g, d);
      const uint32_t space = nb_old * g.B - d;
      const uint32_t fill = min(c, space);
      const uint32_t has_fill = fill > 0 ? 1u : 0u;
      const uint32_t need = blocks_for(g, c - fill);
      if (has_fill && j == 0) {
        blk = run_tail[r];                 // resume at the last-insert position (graph.hpp:344-349)
        off0 = d - (nb_old - 1) * g.B;
        src0 = rs;
        cnt = fill;
      } else {
        const uint32_t f = j - has_fill;
        const unsigned long long o = (unsigned long long)blk_off[r] + f;
        blk = ring_at(g, base_mod, o);
        off0 = 0;
        src0 = rs + fill + f * g.B;
        cnt = min(g.B, c - fill - f * g.B);
        const uint32_t prev = (f == 0) ? (nb_old > 0 ? run_tail[r] : kNull) : ring_at(g, base_mod, o - 1);
        if (prev == kNull) g.head[v] = blk; else g.next[prev] = blk;
        if (f == need - 1) {
          g.next[blk] = kNull;
          if (kCommit) g.tail[v] = blk;
        }
      }
      if (kCommit && j == need + has_fill - 1) g.deg[v] = d + c;
    }
    const uint32_t nvalid = min(32u, U - u0);
    constexpr int kFly = 8;  // units in flight per warp (16 measured slower: registers)
    for (uint32_t l0 = 0; l0 < nvalid; l0 += kFly) {
      uint32_t vb[kFly], vo[kFly], vs[kFly], vc[kFly], val[kFly];
#pragma unroll
      for (int q = 0; q < kFly; ++q) {
        const int l = (int)(l0 + q) & 31;
        vb[q] = __shfl_sync(kFull, blk, l);
        vo[q] = __shfl_sync(kFull, off0, l);
        vs[q] = __shfl_sync(kFull, src0, l);
        const uint32_t cq = __shfl_sync(kFull, cnt, l);
        vc[q] = (l0 + q < nvalid) ? cq : 0u;
      }
#pragma unroll
      for (int q = 0; q < kFly; ++q)
        if ((uint32_t)lane < vc[q]) val[q] = batch_value(b, vs[q] + lane);
#pragma unroll
      for (int q = 0; q < kFly; ++q) {
        if ((uint32_t)lane < vc[q]) {
          if (kValidateDst && val[q] >= g.dst_limit) set_error(op, 2, kErrDstRange, vs[q] + lane);
          g.slab[(unsigned long long)vb[q] * g.B + vo[q] + lane] = val[q];
        }
      }
#pragma unroll
      for (int q = 0; q < kFly; ++q) {
        for (uint32_t s = 32 + lane; s < vc[q]; s += 32) {  // blocks wider than a warp
          const uint32_t x = batch_value(b, vs[q] + s);
          if (kValidateDst && x >= g.dst_limit) set_error(op, 2, kErrDstRange, vs[q] + s);
          g.slab[(unsigned long long)vb[q] * g.B + vo[q] + s] = x;
        }
      }
    }
  }
}

// insert, counting path: append straight from the COO batch, one thread per
// ENTRY, four entries per thread with each stage issued for all four (entry ->
// source info gather -> queue handle -> slab store).  The entry's rank inside
// its source fixes its slot: position = old degree + rank.  The entry landing in
// slot 0 of a fresh block links that block; the last entry publishes degree and
// tail (graph.hpp:333-372 without a grouped copy of the batch and without a
// unit list).
__global__ void __launch_bounds__(256)
append_entries_kernel(GraphView g, GroupIndex gi, const uint32_t* __restrict__ src,
                      const uint32_t* __restrict__ dst, const uint32_t* __restrict__ rank, uint32_t n,
                      const uint4* __restrict__ info, OpState* op) {
  if (op->err) return;
  const unsigned long long base_mod = op->front_old % g.ring_cap;
  const bool lap0 = op->front_old < g.ring_identity;
  const uint32_t base = blockIdx.x * (256 * kGroupItems) + threadIdx.x;
  uint32_t s[kGroupItems], d[kGroupItems], rk[kGroupItems];
  uint4 in[kGroupItems];
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) {
    const uint32_t i = base + q * 256;
    s[q] = i < n ? src[i] : 0u;
    d[q] = i < n ? dst[i] : 0u;
    rk[q] = i < n ? rank[i] : 0u;
  }
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) in[q] = (base + q * 256 < n) ? info[gi(s[q])] : make_uint4(0, 0, 0, 0);
  uint32_t blk[kGroupItems], prev[kGroupItems], slot[kGroupItems];
  bool fresh[kGroupItems];
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) {
    const uint32_t d_old = in[q].x;
    const uint32_t nb_old = blocks_for(g, d_old);
    const uint32_t p = d_old + rk[q];
    const uint32_t kb = div_b(g, p);
    slot[q] = p - kb * g.B;
    fresh[q] = kb >= nb_old;
    blk[q] = in[q].y;   // the old tail block (the only old block with room: chains are compact)
    prev[q] = kNull;
    if (base + q * 256 < n && fresh[q]) {
      const unsigned long long o = (unsigned long long)in[q].z + (kb - nb_old);
      blk[q] = ring_at(g, base_mod, o, lap0);
      if (slot[q] == 0) prev[q] = (kb == nb_old) ? (nb_old > 0 ? in[q].y : kNull) : ring_at(g, base_mod, o - 1, lap0);
    }
  }
#pragma unroll
  for (int q = 0; q < kGroupItems; ++q) {
    if (base + q * 256 >= n) continue;
    g.slab[(unsigned long long)blk[q] * g.B + slot[q]] = d[q];
    if (fresh[q] && slot[q] == 0) {
      if (prev[q] == kNull) g.head[s[q]] = blk[q]; else g.next[prev[q]] = blk[q];
    }
    if (rk[q] == in[q].w - 1) {   // the source's last entry
      g.deg[s[q]] = in[q].x + in[q].w;
      if (fresh[q]) {
        g.next[blk[q]] = kNull;
        g.tail[s[q]] = blk[q];
      }
    }
  }
}

// CSR path commit: runs only when every check passed (validate-then-mutate,
// graph.hpp:168-171): publishes deg/tail per source and the queue front /
// live-edge count (block_pool.hpp:162-166, graph.hpp:186).
__global__ void __launch_bounds__(256)
commit_insert_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ blk_off,
                     const uint32_t* __restrict__ run_deg, OpState* op) {
  if (op->err) return;
  const uint32_t T = (uint32_t)op->n_runs;
  const unsigned long long base_mod = op->front_old % g.ring_cap;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < T; r += gridDim.x * blockDim.x) {
    const uint32_t c = run_len(b, r);
    if (c == 0) continue;
    const uint32_t v = batch_src(b, r);
    const uint32_t d = run_deg[r];
    const uint32_t nb_old = blocks_for(g, d);
    const uint32_t fill = min(c, nb_old * g.B - d);
    const uint32_t need = blocks_for(g, c - fill);
    g.deg[v] = d + c;
    if (need > 0) g.tail[v] = ring_at(g, base_mod, (unsigned long long)blk_off[r] + need - 1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g.st->front += op->total_need;
    g.st->active_edges += op->n_edges;
  }
}

// ---------------------------------------------------------------------------
// CSR insert / bulk init, native block size (B = 32): plan + ONE append pass.
//
//   csr plan   (alloc_kernel<CsrPlan*>) one pass over the vertices: validates the
//              offsets (csr.hpp:49-66, graph.hpp:322-327), computes the fresh
//              blocks every source needs (plan_batch, graph.hpp:135-160), hands
//              out queue positions, and lists (vertex, 32-unit chunk) items for
//              sources with more than kCsrHeavy entries.
//   csr append (csr_append_kernel) a warp owns 32 consecutive vertices: their
//              entries are ONE contiguous range of the batch, staged into the
//              warp's shared-memory buffer by a TMA bulk copy
//              (cp.async.bulk global -> shared, completion on an mbarrier) while
//              the lanes resolve queue handles and links; the units (tail fill
//              or one fresh block) are then written as full-sector 128-byte
//              stores straight from shared memory.  Heavy sources are split into
//              items of 32 units so a hub is spread over the whole grid.
//              The destination range check (csr.hpp:67-72) rides in this pass and
//              deg/tail/front are published by it; if a bad destination shows up
//              the host runs csr_rollback_kernel, so a rejected batch still
//              leaves the graph unchanged (graph.hpp:168-171).
// ---------------------------------------------------------------------------
constexpr uint32_t kCsrStage = 1024;   // entries staged per round (4 KB per warp)
constexpr uint32_t kCsrHeavy = 128;    // sources with more entries become items of up to 32 units (balance: hubs spread over the grid)
constexpr int kCsrWarps = 8;

struct __align__(16) CsrItem {   // 32 bytes: one 32-unit chunk of a heavy source, self-contained (one load)
  uint32_t v, chunk, d, tail;    // d / tail: the source's state BEFORE the batch
  unsigned long long o0;         // first batch entry of the source
  uint32_t c, bo;                // its batch entries / first queue position
};

// Plan pass: one thread handles kCsrPlanItems vertices, strided by the CTA size so every load is
// coalesced.  Fresh blocks and heavy items are two 32-bit counts packed in ONE 64-bit word
// ([63:32] items, [31:0] blocks): one CTA scan, one atomicAdd per tile on the packed cursor
// (ranges only need to be disjoint, not ordered).  There is no finishing step here: the append
// pass reads the packed totals itself, so no tile ever waits on a fence.
// scratch: [0] packed cursor, [1] finished CTAs of the append pass; zeroed before the launch.
constexpr int kCsrPlanItems = 4;
constexpr int kCsrPlanTile = 256 * kCsrPlanItems;
// kFresh: the pool is untouched (bulk init proper), so every source is empty — its degree and tail are not read.
template <bool kFresh>
__global__ void __launch_bounds__(256)
csr_plan_kernel(GraphView g, const unsigned long long* __restrict__ off, uint32_t V, unsigned long long n_edges,
                uint32_t* __restrict__ blk_off, CsrItem* __restrict__ items, unsigned long long items_cap,
                unsigned long long* scratch, OpState* op) {
  __shared__ unsigned long long s_warp[8];
  __shared__ unsigned long long s_base;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t v0 = blockIdx.x * kCsrPlanTile + threadIdx.x;
  unsigned long long o0[kCsrPlanItems], o1[kCsrPlanItems];
  uint32_t dg[kCsrPlanItems], aw[kCsrPlanItems];
#pragma unroll
  for (int j = 0; j < kCsrPlanItems; ++j) {   // every load independent of the others
    const uint32_t v = v0 + j * 256;
    const bool in = v < V;
    o0[j] = in ? off[v] : 0ull;
    o1[j] = in ? off[v + 1] : 0ull;
    dg[j] = (in && !kFresh) ? g.deg[v] : 0u;
    aw[j] = in ? g.alive[v >> 5] : 0xFFFFFFFFu;
  }
  unsigned long long w[kCsrPlanItems], sum = 0;
  uint32_t cc[kCsrPlanItems];
#pragma unroll
  for (int j = 0; j < kCsrPlanItems; ++j) {
    const uint32_t v = v0 + j * 256;
    bool ok = v < V;
    if (ok) {   // csr.hpp:49-66, graph.hpp:322-327
      if (v == 0 && o0[j] != 0) { set_error(op, 2, kErrOffsetsStart, 0); ok = false; }
      if (v + 1 == V && o1[j] != n_edges) { set_error(op, 2, kErrOffsetsEnd, V); ok = false; }
      if (o1[j] < o0[j]) { set_error(op, 2, kErrOffsetsMonotone, v + 1); ok = false; }
      if (o1[j] > n_edges) ok = false;   // (non-monotone or bad end: reported where it happens)
    }
    const uint32_t c = ok ? (uint32_t)(o1[j] - o0[j]) : 0u;
    if (c > 0 && !((aw[j] >> (v & 31)) & 1u)) set_error(op, 2, kErrDeadSource, v);
    cc[j] = c;
    const unsigned long long pw = c ? plan_word(g, dg[j], c) : 0ull;   // [63:32] units, [31:0] fresh blocks
    const uint32_t n_it = (c > kCsrHeavy) ? ((uint32_t)(pw >> 32) + 31u) / 32u : 0u;
    w[j] = ((unsigned long long)n_it << 32) | (pw & 0xFFFFFFFFull);
    sum += w[j];
  }
  unsigned long long incl = sum;
#pragma unroll
  for (int dl = 1; dl < 32; dl <<= 1) {
    const unsigned long long t = __shfl_up_sync(kFull, incl, dl);
    if (lane >= dl) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  unsigned long long warp_excl = 0, tile_sum = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const unsigned long long sw = s_warp[k];
    if (k < warp) warp_excl += sw;
    tile_sum += sw;
  }
  if (threadIdx.x == 0) s_base = tile_sum ? atomicAdd(&scratch[0], tile_sum) : 0ull;
  __syncthreads();
  unsigned long long run = s_base + warp_excl + (incl - sum);
#pragma unroll
  for (int j = 0; j < kCsrPlanItems; ++j) {
    const uint32_t v = v0 + j * 256;
    if (v < V) {
      blk_off[v] = (uint32_t)run;
      const uint32_t n_it = (uint32_t)(w[j] >> 32);
      const unsigned long long ib = run >> 32;
      if (n_it != 0 && ib + n_it <= items_cap) {   // (overflow only with broken offsets: already an error)
        const uint32_t tl = kFresh ? kNull : g.tail[v];
        for (uint32_t k = 0; k < n_it; ++k) items[ib + k] = CsrItem{v, k, dg[j], tl, o0[j], cc[j], (uint32_t)run};
      }
    }
    run += w[j];
  }
}

// ---- mbarrier + TMA bulk copy (global -> shared) ---------------------------------
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}
// bytes: multiple of 16; both addresses 16-byte aligned
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

// Stages batch entries [e0, e1) (e1 - e0 <= kCsrStage) into `stage`; returns the
// index in `stage` of entry e0.  The 16-byte-aligned interior goes through one
// TMA bulk copy (waited for with csr_stage_wait), the unaligned tail (<= 3
// entries) and ranges inside a single 16-byte chunk through the lanes.
__device__ __forceinline__ uint32_t csr_stage_issue(uint32_t* stage, unsigned long long* bar, const uint32_t* __restrict__ dsts,
                                                    unsigned long long e0, unsigned long long e1, bool& armed) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(dsts + e0);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(dsts + e1);
  const uintptr_t A = a0 & ~(uintptr_t)15, Z = a1 & ~(uintptr_t)15;
  const uint32_t lead = (uint32_t)((a0 - A) >> 2);
  armed = Z > A;
  const int lane = lane_id();
  if (armed && lane == 0) {
    const unsigned bytes = (unsigned)(Z - A);
    mbar_expect_tx(bar, bytes);
    tma_load_1d(stage, reinterpret_cast<const void*>(A), bytes, bar);
  }
  // the rest: [max(a0, Z), a1) — at most 3 entries
  const uintptr_t t0 = a0 > Z ? a0 : Z;
  const uint32_t nt = (uint32_t)((a1 - t0) >> 2);
  if ((uint32_t)lane < nt) cp_async4(&stage[((t0 - A) >> 2) + lane], reinterpret_cast<const void*>(t0 + 4u * lane));
  return lead;
}

// One batch of up to 32 append units, one per lane (blk / off0 / srel / cnt; cnt = 0: no unit),
// written from the staging buffer.  Fresh blocks (off0 == 0) go out FOUR PER INSTRUCTION: eight
// lanes own one block, each lane a 16-byte quarter-sector-aligned chunk (st.global.v4), padded
// with kTomb up to the next 32-byte sector so no partial sector is ever written.  Slots beyond a
// unit's entries are free slots of that block (nothing reads past deg), so padding is invisible.
// Tail fills (off0 != 0, at most one per source) take a scalar path.  Returns through `bad` the
// smallest batch index of an out-of-range destination seen by this lane (csr.hpp:67-72).
__device__ __forceinline__ void csr_write_units(const GraphView& g, const uint32_t* stage, uint32_t nunits, uint32_t blk,
                                                uint32_t off0, uint32_t srel, uint32_t cnt,
                                                unsigned long long stage_entry0, unsigned long long& bad) {
  const int lane = lane_id();
  const int sub = lane >> 3, c8 = lane & 7;
  const bool is_fill = cnt > 0 && off0 != 0;
  // [11:0] srel, [17:12] cnt, [23:18] padded end (0 for fills and empty lanes: skipped by the fast loop)
  const uint32_t pad_end = (cnt > 0 && !is_fill) ? min(32u, (cnt + 7u) & ~7u) : 0u;
  const uint32_t pack = srel | (cnt << 12) | (pad_end << 18);
  const uint32_t limit = g.dst_limit;
  for (uint32_t q0 = 0; q0 < nunits; q0 += 4) {
    const uint32_t bq = __shfl_sync(kFull, blk, q0 + sub);
    const uint32_t pq = __shfl_sync(kFull, pack, q0 + sub);
    const uint32_t sq = pq & 0xFFFu, cq = (pq >> 12) & 63u, pe = pq >> 18;
    const uint32_t s0 = 4u * c8;
    if (s0 < pe) {
      const uint32_t* src = stage + sq + s0;
      uint4 v;
      v.x = src[0]; v.y = src[1]; v.z = src[2]; v.w = src[3];
      const uint32_t nv = cq - min(cq, s0);   // valid words of this chunk (>= 4: all)
      // branch-free: out-of-range test on the real entries, then kTomb padding (selects)
      const bool b0 = v.x >= limit && nv > 0, b1 = v.y >= limit && nv > 1, b2 = v.z >= limit && nv > 2, b3 = v.w >= limit && nv > 3;
      if (nv < 1) v.x = kTomb;
      if (nv < 2) v.y = kTomb;
      if (nv < 3) v.z = kTomb;
      if (nv < 4) v.w = kTomb;
      if (b0 | b1 | b2 | b3) {
        const unsigned long long e = stage_entry0 + sq + s0 + (b0 ? 0u : b1 ? 1u : b2 ? 2u : 3u);
        bad = min(bad, e);
      }
      *reinterpret_cast<uint4*>(g.slab + (unsigned long long)bq * 32u + s0) = v;
    }
  }
  unsigned fills = __ballot_sync(kFull, is_fill);
  while (fills) {
    const int q = __ffs(fills) - 1;
    fills &= fills - 1;
    const uint32_t bq = __shfl_sync(kFull, blk, q);
    const uint32_t oq = __shfl_sync(kFull, off0, q);
    const uint32_t sq = __shfl_sync(kFull, srel, q);
    const uint32_t cq = __shfl_sync(kFull, cnt, q);
    if ((uint32_t)lane < cq) {
      const uint32_t val = stage[sq + lane];
      if (val >= limit) bad = min(bad, stage_entry0 + sq + lane);
      g.slab[(unsigned long long)bq * 32u + oq + lane] = val;
    }
  }
}

// Unit j of a source with c batch entries, degree d and tail block tl before the batch, first
// queue position bo: resolves its block, links it, and returns where its entries sit.
// src_rel0: index in the staging buffer of the source's first batch entry.
__device__ __forceinline__ void csr_resolve_unit(const GraphView& g, unsigned long long base_mod, bool lap0, uint32_t v, uint32_t j,
                                                 uint32_t c, uint32_t d, uint32_t tl, uint32_t bo, uint32_t src_rel0,
                                                 uint32_t& blk, uint32_t& off0, uint32_t& srel, uint32_t& cnt) {
  const uint32_t nb_old = (d + 31u) >> 5;
  const uint32_t space = nb_old * 32u - d;
  const uint32_t fill = min(c, space);
  const uint32_t has_fill = fill > 0 ? 1u : 0u;
  const uint32_t need = (c - fill + 31u) >> 5;
  if (has_fill && j == 0) {
    blk = tl;                      // resume at the last-insert position (graph.hpp:344-349)
    off0 = d - (nb_old - 1u) * 32u;
    srel = src_rel0;
    cnt = fill;
  } else {
    const uint32_t f = j - has_fill;
    const unsigned long long o = (unsigned long long)bo + f;
    blk = ring_at(g, base_mod, o, lap0);
    off0 = 0;
    srel = src_rel0 + fill + f * 32u;
    cnt = min(32u, c - fill - f * 32u);
    const uint32_t prev = (f == 0) ? (nb_old > 0 ? tl : kNull) : ring_at(g, base_mod, o - 1, lap0);
    if (prev == kNull) g.head[v] = blk; else g.next[prev] = blk;
    if (f == need - 1) g.next[blk] = kNull;
  }
}

// Work unit w of the append pass: w < n_items is heavy item w, otherwise vertex group w - n_items.
// Its metadata is two 16-byte registers, loaded one unit ahead of its use:
//   item : a = {v, chunk, d, tail}           b = {o0.lo, o0.hi, c, bo}
//   group: a = {o0.lo, o0.hi, o1.lo, o1.hi}  b = {d, tail, bo, -} of the lane's vertex
struct CsrWork {
  uint4 a, b;
};
__device__ __forceinline__ CsrWork csr_load_work(const GraphView& g, const unsigned long long* __restrict__ off,
                                                 const uint32_t* __restrict__ blk_off, const CsrItem* __restrict__ items,
                                                 uint32_t V, uint32_t n_items, uint32_t w, uint32_t total) {
  CsrWork r{make_uint4(0, 0, 0, 0), make_uint4(0, kNull, 0, 0)};
  if (w >= total) return r;
  if (w < n_items) {
    const uint4* p = reinterpret_cast<const uint4*>(items + w);
    r.a = p[0];
    r.b = p[1];
  } else {
    const uint32_t v = (w - n_items) * 32u + lane_id();
    if (v < V) {   // five independent loads
      const unsigned long long o0 = off[v], o1 = off[v + 1];
      r.a = make_uint4((uint32_t)o0, (uint32_t)(o0 >> 32), (uint32_t)o1, (uint32_t)(o1 >> 32));
      r.b = make_uint4(g.deg[v], g.tail[v], blk_off[v], 0u);
    }
  }
  return r;
}

__global__ void __launch_bounds__(kCsrWarps * 32, 4)
csr_append_kernel(GraphView g, const unsigned long long* __restrict__ off, const uint32_t* __restrict__ dsts, uint32_t V,
                  const uint32_t* __restrict__ blk_off, const CsrItem* __restrict__ items, unsigned long long n_edges,
                  unsigned long long* scratch, OpState* op) {
  // op->err can only hold a PLAN error here: this pass reports bad destinations through
  // op->bad_index and turns them into an error once every CTA has finished.
  if (op->err) return;
  const unsigned long long plan_tot = scratch[0];            // [63:32] heavy items, [31:0] fresh blocks
  const unsigned long long need = plan_tot & 0xFFFFFFFFull;
  const unsigned long long front_old = g.st->front;           // (published by the last CTA only)
  if (need > g.st->rear - front_old) {                        // ensure_available (block_pool.hpp:177-189)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      op->err_detail = kErrPoolUnderflow;
      op->err_index = need - (g.st->rear - front_old);
      __threadfence();
      op->err = 3;
    }
    return;
  }
  __shared__ __align__(16) uint32_t s_stage[kCsrWarps][kCsrStage + 40];   // + alignment lead (<= 3) + the padded read of the last unit
  __shared__ unsigned long long s_bar[kCsrWarps];
  __shared__ uint8_t s_owner[kCsrWarps][256];   // <= 32 x (ceil(kCsrHeavy / 32) + 1) units per round
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  uint32_t* stage = s_stage[warp];
  unsigned long long* bar = &s_bar[warp];
  uint8_t* owner = s_owner[warp];
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;
  unsigned long long bad = ~0ull;   // smallest out-of-range destination index this lane saw
  const unsigned long long base_mod = front_old % g.ring_cap;
  const bool lap0 = front_old < g.ring_identity;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t n_items = (uint32_t)(plan_tot >> 32);
  const uint32_t total = n_items + (V + 31u) / 32u;

  // Work units (heavy items first, then vertex groups) differ 30x in size, so warps take them in
  // chunks of kCsrChunk consecutive units from a device cursor (one same-address atomic per chunk:
  // ~0.5 G/s of those is all the L2 gives).  The next chunk's ticket is requested when a chunk
  // starts and the next unit's metadata is loaded one unit ahead: neither is ever waited for.
  constexpr uint32_t kCsrChunk = 4;
  uint32_t w_cur = gw * kCsrChunk, w_nxt = w_cur + 1;
  uint32_t ticket = 0;
  CsrWork nxt = csr_load_work(g, off, blk_off, items, V, n_items, w_cur, total);
  while (w_cur < total) {
    if ((w_cur % kCsrChunk) == 0 && lane == 0) ticket = nwarps + atomicAdd(&op->med_cursor, 1u);
    if ((w_nxt % kCsrChunk) == 0) w_nxt = __shfl_sync(kFull, ticket, 0) * kCsrChunk;
    const CsrWork cur = nxt;
    nxt = csr_load_work(g, off, blk_off, items, V, n_items, w_nxt, total);
    if (w_cur < n_items) {
      // ---- heavy item: 32 consecutive units of one source
      const uint32_t v = cur.a.x, chunk = cur.a.y, d = cur.a.z, tl = cur.a.w;
      const unsigned long long o0 = ((unsigned long long)cur.b.y << 32) | cur.b.x;
      const uint32_t c = cur.b.z, bo = cur.b.w;
      const uint32_t nb_old = (d + 31u) >> 5;
      const uint32_t fill = min(c, nb_old * 32u - d);
      const uint32_t has_fill = fill > 0 ? 1u : 0u;
      const uint32_t nu = ((c - fill + 31u) >> 5) + has_fill;
      const uint32_t j0 = chunk * 32u;
      const uint32_t nunits = min(32u, nu - j0);
      // entries of units [j0, j0 + nunits)
      const uint32_t f0 = j0 == 0 ? 0u : fill + (j0 - has_fill) * 32u;
      const uint32_t j1 = j0 + nunits;
      const uint32_t f1 = min(c, fill + (j1 - has_fill) * 32u);
      bool armed;
      const uint32_t lead = csr_stage_issue(stage, bar, dsts, o0 + f0, o0 + f1, armed);
      uint32_t blk = 0, o_ = 0, srel = 0, cnt = 0;
      if ((uint32_t)lane < nunits)
        csr_resolve_unit(g, base_mod, lap0, v, j0 + lane, c, d, tl, bo, lead - f0, blk, o_, srel, cnt);
      cp_async_wait_all();
      if (armed) { mbar_wait(bar, phase); phase ^= 1u; }
      __syncwarp();
      csr_write_units(g, stage, nunits, blk, o_, srel, cnt, o0 + f0 - lead, bad);
      __syncwarp();
    } else {
      // ---- group of 32 consecutive vertices, one per lane
      const uint32_t grp = w_cur - n_items;
      const uint32_t v = grp * 32u + lane;
      const bool valid = v < V;
      const unsigned long long o0 = ((unsigned long long)cur.a.y << 32) | cur.a.x;
      const unsigned long long o1 = ((unsigned long long)cur.a.w << 32) | cur.a.z;
      const uint32_t c = (uint32_t)(o1 - o0);
      const uint32_t d = c ? cur.b.x : 0u, tl = cur.b.y, bo = cur.b.z;
      const uint32_t nb_old = (d + 31u) >> 5;
      const uint32_t fill = min(c, nb_old * 32u - d);
      const uint32_t has_fill = fill > 0 ? 1u : 0u;
      const uint32_t need = (c - fill + 31u) >> 5;
      const bool heavy = c > kCsrHeavy;
      const bool light = c > 0 && !heavy;
      // the source's new state (insert_adjacency, graph.hpp:367-371): the tail handle is requested
      // now and published at the end of the group, off the critical path
      if (c > 0) g.deg[v] = d + c;
      uint32_t tail_new = kNull;
      if (need > 0) tail_new = ring_at(g, base_mod, (unsigned long long)bo + need - 1, lap0);
      const unsigned lightmask = __ballot_sync(kFull, light);
      if (lightmask != 0) {
        const unsigned heavymask = __ballot_sync(kFull, heavy);
        const uint32_t cl = light ? c : 0u;
        uint32_t cincl = cl;
#pragma unroll
        for (int dl = 1; dl < 32; dl <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, cincl, dl);
          if (lane >= dl) cincl += t;
        }
        const uint32_t nu = light ? need + has_fill : 0u;
        uint32_t pos = 0;
        while (pos < 32) {
          const unsigned rem = lightmask & (0xFFFFFFFFu << pos);
          if (rem == 0) break;
          const int a = __ffs(rem) - 1;
          const uint32_t cbase = __shfl_sync(kFull, cincl - cl, a);
          const unsigned hv_after = heavymask & (0xFFFFFFFFu << a);
          const int hb = hv_after ? __ffs(hv_after) - 1 : 32;
          const bool okl = valid && lane >= a && lane < hb && (cincl - cbase) <= kCsrStage;
          const unsigned okmask = __ballot_sync(kFull, okl);
          const int lb = a + __popc(okmask);   // the eligible lanes are a contiguous run starting at a
          const unsigned long long e0 = __shfl_sync(kFull, o0, a);
          const unsigned long long e1 = __shfl_sync(kFull, o1, lb - 1);
          bool armed;
          const uint32_t lead = csr_stage_issue(stage, bar, dsts, e0, e1, armed);
          const bool in_round = lane >= a && lane < lb;
          const uint32_t nur = in_round ? nu : 0u;
          uint32_t uincl = nur;
#pragma unroll
          for (int dl = 1; dl < 32; dl <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, uincl, dl);
            if (lane >= dl) uincl += t;
          }
          const uint32_t uexcl = uincl - nur;
          const uint32_t U = __shfl_sync(kFull, uincl, 31);
          for (uint32_t j = 0; j < nur; ++j) owner[uexcl + j] = (uint8_t)lane;
          __syncwarp();
          bool waited = false;
          for (uint32_t ub = 0; ub < U; ub += 32) {
            const uint32_t u = ub + lane;
            const int L = (u < U) ? owner[u] : 0;
            const unsigned long long oL = __shfl_sync(kFull, o0, L);
            const uint32_t cL = __shfl_sync(kFull, c, L);
            const uint32_t dL = __shfl_sync(kFull, d, L);
            const uint32_t tlL = __shfl_sync(kFull, tl, L);
            const uint32_t boL = __shfl_sync(kFull, bo, L);
            const uint32_t ueL = __shfl_sync(kFull, uexcl, L);
            uint32_t blk = 0, o_ = 0, srel = 0, cnt = 0;
            if (u < U)
              csr_resolve_unit(g, base_mod, lap0, grp * 32u + L, u - ueL, cL, dL, tlL, boL, (uint32_t)(oL - e0) + lead, blk, o_, srel, cnt);
            if (!waited) {
              cp_async_wait_all();
              if (armed) { mbar_wait(bar, phase); phase ^= 1u; }
              waited = true;
            }
            __syncwarp();
            csr_write_units(g, stage, min(32u, U - ub), blk, o_, srel, cnt, e0 - lead, bad);
          }
          __syncwarp();
          pos = (uint32_t)lb;
        }
      }
      if (need > 0) g.tail[v] = tail_new;
    }
    w_cur = w_nxt;
    w_nxt = w_cur + 1;
  }
  if (bad != ~0ull) atomicMin(&op->bad_index, bad);
  // the last CTA to finish publishes the queue front / live-edge count and the verdict
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&scratch[1], 1ull) == gridDim.x - 1) {
      __threadfence();
      op->total_need = need;
      op->n_items = n_items;
      op->n_edges = n_edges;
      op->front_old = front_old;
      g.st->front = front_old + need;      // commit_front (block_pool.hpp:162-166)
      g.st->active_edges += n_edges;       // graph.hpp:186
      op->committed = 1;
      const unsigned long long b = ld_volatile_u64(&op->bad_index);
      if (b != ~0ull) {
        op->err_detail = kErrDstRange;
        op->err_index = b;
        op->err = 2;
      }
    }
  }
}

// Error path of the fused CSR append: a destination failed the range check after
// deg/tail/front were published.  Restores every source's degree and tail (the old
// tail is re-found by walking the chain) and the global counters, so the rejected
// batch leaves the graph unchanged (graph.hpp:168-171).
__global__ void __launch_bounds__(256)
csr_rollback_kernel(GraphView g, const unsigned long long* __restrict__ off, uint32_t V, OpState* op) {
  if (!op->committed) return;   // (the append pass never ran: nothing was published)
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(off[v + 1] - off[v]);
    if (c == 0) continue;
    const uint32_t d = g.deg[v] - c;
    const uint32_t nb_old = (d + 31u) >> 5;
    const uint32_t fill = min(c, nb_old * 32u - d);
    g.deg[v] = d;
    if (c > fill) {   // fresh blocks were linked: the tail moved
      uint32_t t = kNull;
      if (nb_old > 0) {
        t = g.head[v];
        for (uint32_t k = 1; k < nb_old; ++k) t = g.next[t];
        g.next[t] = kNull;
      } else {
        g.head[v] = kNull;
      }
      g.tail[v] = t;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g.st->front -= op->total_need;
    g.st->active_edges -= op->n_edges;
  }
}

// ---------------------------------------------------------------------------
// Bulk init proper: the CSR insert into a pool nothing was ever popped from (ctor + first insert_batch,
// io/workload.hpp:113-139).  Every source is empty (no tail to resume) and the queue still serves
// ring[p] == p, so a source's chain is the handle range [front + blk_off[v], + ceil(c / 32)) and the
// whole op is a segmented copy of the destination array into the slab with every source padded to a
// block boundary.  That needs none of the staging / unit resolution of csr_append_kernel:
//   heavy item (32 blocks of one source): row r of the item is dsts[src + 32 r + lane] -> one coalesced
//     128-byte load and one coalesced 128-byte store per block, eight rows in flight per warp;
//   vertex group (32 consecutive vertices, lane = vertex): the lanes publish deg / head / tail and the links
//     of their (<= 4) blocks and describe each block in shared memory {first entry, handle, count}; the warp
//     then copies block after block with lane = slot, four blocks in flight.
// ~15 warp instructions per block instead of ~45.  Same plan (csr_plan_kernel), same validation (the range
// check of csr.hpp:67-72 rides on the copy), same finish protocol and rollback as csr_append_kernel.
// ---------------------------------------------------------------------------
constexpr int kBulkWarps = 8;
__global__ void __launch_bounds__(kBulkWarps * 32)
csr_bulk_kernel(GraphView g, const unsigned long long* __restrict__ off, const uint32_t* __restrict__ dsts, uint32_t V,
                const uint32_t* __restrict__ blk_off, const CsrItem* __restrict__ items, unsigned long long n_edges,
                unsigned long long* scratch, OpState* op) {
  if (op->err) return;
  const unsigned long long plan_tot = scratch[0];            // [63:32] heavy items, [31:0] fresh blocks
  const unsigned long long need = plan_tot & 0xFFFFFFFFull;
  const unsigned long long front_old = g.st->front;
  if (need > g.st->rear - front_old) {                        // ensure_available (block_pool.hpp:177-189)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      op->err_detail = kErrPoolUnderflow;
      op->err_index = need - (g.st->rear - front_old);
      __threadfence();
      op->err = 3;
    }
    return;
  }
  __shared__ uint4 s_desc[kBulkWarps][32 * 4 + 8];   // {first batch entry, handle, entries, entries padded to a sector} per block of the group
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  uint4* desc = s_desc[warp];
  const uint32_t limit = g.dst_limit;
  const uint32_t h_base = (uint32_t)front_old;   // (handle of queue position p is p: the caller checked the pool is untouched)
  uint32_t bad = 0xFFFFFFFFu;   // smallest batch index of an out-of-range destination seen by this lane (n_edges < 2^31)
  const uint32_t* src_lane = dsts + lane;
  uint32_t* out_lane = g.slab + lane;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t n_items = (uint32_t)(plan_tot >> 32);
  const uint32_t total = n_items + (V + 31u) / 32u;
  constexpr uint32_t kChunk = 4;   // units per ticket (one same-address atomic per chunk)
  constexpr int kRows = 16;        // item rows in flight per warp (2 KB)
  constexpr int kBlocks = 8;       // group blocks in flight per warp
  uint32_t w_cur = gw * kChunk, w_nxt = w_cur + 1;
  uint32_t ticket = 0;
  while (w_cur < total) {
    if ((w_cur % kChunk) == 0 && lane == 0) ticket = nwarps + atomicAdd(&op->med_cursor, 1u);
    if ((w_nxt % kChunk) == 0) w_nxt = __shfl_sync(kFull, ticket, 0) * kChunk;
    if (w_cur < n_items) {
      // ---- heavy item: up to 32 consecutive blocks of one source, a straight copy.  Slots past the source's
      // entries are free (nothing reads past deg): they are filled with 0 up to the next 32-byte sector so no
      // partial sector is written, and the range check needs no validity mask.
      const uint4* ip = reinterpret_cast<const uint4*>(items + w_cur);
      const uint4 ia = ip[0], ib = ip[1];
      const uint32_t chunk = ia.y, o0 = ib.x, c = ib.z, bo = ib.w;
      const uint32_t nb = (c + 31u) >> 5;
      const uint32_t j0 = chunk * 32u;
      const uint32_t rows = min(32u, nb - j0);
      const uint32_t rem = c - j0 * 32u;            // entries from the item's first row on
      const uint32_t first = o0 + j0 * 32u;
      const uint32_t* src = src_lane + first;
      const uint32_t h0 = h_base + bo + j0;
      uint32_t* out = out_lane + (unsigned long long)h0 * 32u;
      if ((uint32_t)lane < rows) g.next[h0 + lane] = (j0 + lane + 1u == nb) ? kNull : h0 + lane + 1u;
      const uint32_t full = min(rows, rem >> 5) & ~(uint32_t)(kRows - 1);   // rows of complete 16-row batches
      uint32_t r0 = 0;
#pragma unroll 1
      for (; r0 < full; r0 += kRows) {   // every slot of these rows holds an entry: no masks
        uint32_t x[kRows];
#pragma unroll
        for (int q = 0; q < kRows; ++q) x[q] = src[(r0 + q) * 32u];
#pragma unroll
        for (int q = 0; q < kRows; ++q) {
          if (x[q] >= limit) bad = min(bad, first + (r0 + q) * 32u + lane);
          out[(r0 + q) * 32u] = x[q];
        }
      }
      const uint32_t pad_end = min(rows * 32u, (rem + 7u) & ~7u);
#pragma unroll 1
      for (; r0 < rows; r0 += 4) {
        uint32_t x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t idx = (r0 + q) * 32u + lane;
          x[q] = idx < rem ? src[(r0 + q) * 32u] : 0u;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t idx = (r0 + q) * 32u + lane;
          if (x[q] >= limit) bad = min(bad, first + idx);
          if (idx < pad_end) out[(r0 + q) * 32u] = x[q];
        }
      }
    } else {
      // ---- group of 32 consecutive vertices, lane = vertex
      const uint32_t v = (w_cur - n_items) * 32u + lane;
      const bool valid = v < V;
      const uint32_t o0 = valid ? (uint32_t)off[v] : 0u;
      const uint32_t o1 = valid ? (uint32_t)off[v + 1] : 0u;
      const uint32_t bo = valid ? blk_off[v] : 0u;
      const uint32_t c = o1 - o0;
      const uint32_t nb = (c + 31u) >> 5;
      const uint32_t h0 = h_base + bo;
      if (c > 0) {   // insert_adjacency on an empty source (graph.hpp:333-372)
        g.deg[v] = c;
        g.head[v] = h0;
        g.tail[v] = h0 + nb - 1u;
      }
      const uint32_t nbl = c > kCsrHeavy ? 0u : nb;   // (heavy sources were listed as items by the plan)
      uint32_t uincl = nbl;
#pragma unroll
      for (int dl = 1; dl < 32; dl <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, uincl, dl);
        if (lane >= dl) uincl += t;
      }
      const uint32_t uexcl = uincl - nbl;
      const uint32_t U = __shfl_sync(kFull, uincl, 31);
#pragma unroll 1
      for (uint32_t j = 0; j < nbl; ++j) {
        const uint32_t cnt = min(32u, c - j * 32u);
        desc[uexcl + j] = make_uint4(o0 + j * 32u, h0 + j, cnt, (cnt + 7u) & ~7u);
        g.next[h0 + j] = (j + 1u == nbl) ? kNull : h0 + j + 1u;
      }
      if (lane < kBlocks) desc[U + lane] = make_uint4(0u, 0u, 0u, 0u);   // the last batch reads past U: empty blocks
      __syncwarp();
#pragma unroll 1
      for (uint32_t u0 = 0; u0 < U; u0 += kBlocks) {
        uint32_t x[kBlocks];
#pragma unroll
        for (int q = 0; q < kBlocks; ++q) {
          const uint4 dq = desc[u0 + q];
          x[q] = (uint32_t)lane < dq.z ? src_lane[dq.x] : 0u;
        }
#pragma unroll
        for (int q = 0; q < kBlocks; ++q) {
          const uint4 dq = desc[u0 + q];
          if (x[q] >= limit) bad = min(bad, dq.x + lane);
          if ((uint32_t)lane < dq.w) out_lane[(unsigned long long)dq.y * 32u] = x[q];
        }
      }
      __syncwarp();   // the descriptors are rewritten by the next group
    }
    w_cur = w_nxt;
    w_nxt = w_cur + 1;
  }
  if (bad != 0xFFFFFFFFu) atomicMin(&op->bad_index, (unsigned long long)bad);
  // the last CTA to finish publishes the queue front / live-edge count and the verdict
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&scratch[1], 1ull) == gridDim.x - 1) {
      __threadfence();
      op->total_need = need;
      op->n_items = n_items;
      op->n_edges = n_edges;
      op->front_old = front_old;
      g.st->front = front_old + need;      // commit_front (block_pool.hpp:162-166)
      g.st->active_edges += n_edges;       // graph.hpp:186
      op->committed = 1;
      const unsigned long long b = ld_volatile_u64(&op->bad_index);
      if (b != ~0ull) {
        op->err_detail = kErrDstRange;
        op->err_index = b;
        op->err = 2;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// chain enumeration: touched sources -> flat list of their blocks (+ the CTA
// work items of the long-chain match path)
// ---------------------------------------------------------------------------
constexpr uint32_t kLaneWalk = 16;       // chains up to this many blocks are walked by one lane
constexpr uint32_t kHugeWalk = 1024;     // longer chains are walked by a whole CTA, 1024 links per round trip
// Match tiers by the number of targets k the batch holds for a source:
//   k <= kTinyTargets               thread-per-block register compare (match_tiny_kernel)
//   kTinyTargets < k <= kMedTargets a warp per 32-block chunk, per-warp shared-memory table
//   k > kMedTargets                 a CTA per 256-block chunk, CTA-wide shared-memory table
constexpr uint32_t kTinyTargets = 8;
constexpr uint32_t kMedTargets = 128;
constexpr uint32_t kMedChunk = 32;       // blocks per warp item of the medium path
// wl_run entries carry the tier in the top bit (set = NOT tiny) so the tiny
// kernel decides from its first load; runs index fewer than 2^31 entries.
constexpr uint32_t kTierBit = 0x80000000u;
constexpr uint32_t kRunMask = 0x7FFFFFFFu;
__device__ __forceinline__ uint32_t run_tag(const BatchView& b, uint32_t r) {
  if (b.run_start == nullptr) return r;
  return (run_len(b, r) > kTinyTargets) ? (r | kTierBit) : r;
}
constexpr uint32_t kLongChunk = 1024;    // blocks per CTA item of the long path (the table is built once per item: 256 measured 39 us for the tier at C2)

// ---- sources a single warp owns for the whole delete (dg_fused.cuh) ----
// class of a touched source, stored in wl_off[r] (real work-list offsets are < 2^31)
constexpr uint32_t kClsNone = 0xFFFFFFFFu;    // nothing stored (dead / unknown source, empty chain)
constexpr uint32_t kClsSmall = 0xFFFFFFFEu;
constexpr uint32_t kClsMed = 0xFFFFFFFDu;
constexpr uint32_t kClsMin = 0xFFFFFFF0u;     // wl_off values >= this are classes, not offsets
constexpr uint32_t kFusedSmallBlocks = 16;
constexpr uint32_t kFusedSmallTargets = kTinyTargets;   // 8
constexpr uint32_t kFusedMedBlocks = 256;
constexpr uint32_t kFusedMedTargets = kMedTargets;      // 128
constexpr uint32_t kFusedListBlocks = 256;    // blocks a warp keeps (handle + mask) at a time

__host__ __device__ inline uint32_t fused_class(uint32_t k, uint32_t nblk) {
  if (nblk == 0 || k == 0) return kClsNone;
  if (k <= kFusedSmallTargets && nblk <= kFusedSmallBlocks) return kClsSmall;
  if (k <= kFusedMedTargets && nblk <= kFusedMedBlocks) return kClsMed;
  return 0u;   // hub: multi-kernel path
}


// Enumeration plan: work-list segments are disjoint ranges too (alloc_kernel):
//   word a = [63:32] touched sources (counting path only), [31:0] batch entries
//   word b = [63:32] chains a whole warp walks (their big-list slots come out of the scan: one
//            same-address atomic per such source cost more than the rest of the pass),
//            [31:0] blocks of the touched chains
// The match tiers' (run, chunk) items and the long-chain list are filled
// through device counters (order is irrelevant: they only distribute work).
struct EnumLists {
  uint32_t* run_deg;
  uint32_t* wl_off;
  uint2* med_items;    // nullptr on paths without a batch (export, digest)
  uint2* long_items;
  uint32_t* big_list;  // sources whose chain a whole warp walks (enumerate_big_kernel); chains longer than
                       // kHugeWalk blocks are listed from the END of the same array and walked by a whole CTA
  uint32_t big_cap;
  OpState* op;
  uint32_t* run_head;  // fused delete: head block of every warp-owned source (nullptr: no fusion)
  uint4* fmed_rec;     // fused delete: sources of the medium class (a warp per source), two 16-byte words each
                       // {run, vertex, first target, targets} {degree, head, -, -}, filled through op->n_fmed
  uint32_t* zero3;     // delete: run_matched (+ two spare words) of the run start at zero (no memset)
  uint32_t zstride;
  __device__ void write(uint32_t r, uint32_t d, uint32_t nblk, uint32_t k, uint32_t head, uint32_t v, uint32_t es,
                        unsigned long long excl_b, uint32_t med_slot) const {
    run_deg[r] = d;
    if (zero3 != nullptr) {
      zero3[r] = 0u;
      zero3[r + zstride] = 0u;
      zero3[r + 2u * zstride] = 0u;
    }
    if (run_head != nullptr) {   // warp-owned sources take no work-list segment: wl_off carries their class
      const uint32_t cls = fused_class(k, nblk);
      if (cls != 0u) {
        wl_off[r] = cls;
        run_head[r] = head;
        if (cls == kClsMed) {   // (the slot came out of the scan: no same-address atomic per listed source)
          fmed_rec[2u * med_slot] = make_uint4(r, v, es, k);
          fmed_rec[2u * med_slot + 1u] = make_uint4(d, head, 0u, 0u);
        }
        return;
      }
    }
    wl_off[r] = (uint32_t)excl_b;
    if (nblk > kHugeWalk) big_list[big_cap - 1u - atomicAdd(&op->n_huge, 1u)] = r;   // (a few dozen per batch)
    else if (nblk > kLaneWalk) big_list[(uint32_t)(excl_b >> 32)] = r;
    if (med_items != nullptr && nblk > 0) {
      if (k > kMedTargets) {
        const uint32_t n = (nblk + kLongChunk - 1) / kLongChunk;
        const unsigned long long base = atomicAdd(&op->n_items, (unsigned long long)n);
        for (uint32_t c = 0; c < n; ++c) long_items[base + c] = make_uint2(r, c);
      } else if (k > kTinyTargets) {
        const uint32_t n = (nblk + kMedChunk - 1) / kMedChunk;
        const unsigned long long base = atomicAdd(&op->n_med, (unsigned long long)n);
        for (uint32_t c = 0; c < n; ++c) med_items[base + c] = make_uint2(r, c);
      }
    }
  }
};
// word b of the enumeration plan for a chain of nblk blocks
__device__ __forceinline__ unsigned long long enum_word_b(uint32_t nblk) {
  return ((nblk > kLaneWalk && nblk <= kHugeWalk) ? (1ull << 32) : 0ull) | nblk;
}
// fuse: sources a warp owns (fused_class != 0) stay out of the work list
__device__ __forceinline__ unsigned long long enum_word_b(uint32_t nblk, uint32_t k, bool fuse) {
  return (fuse && fused_class(k, nblk) != 0u) ? 0ull : enum_word_b(nblk);
}
// degree of a touched vertex as delete/query see it: dead or unknown sources have
// none (graph.hpp:205, :229).  Predicated, independent loads (see alloc_kernel).
__device__ __forceinline__ uint32_t live_degree(const GraphView& g, uint32_t v, bool wanted, int check_alive) {
  const bool in_range = wanted && v < g.size;
  const uint32_t d = in_range ? g.deg[v] : 0u;
  const uint32_t aw = (in_range && check_alive) ? g.alive[v >> 5] : 0xFFFFFFFFu;
  return ((aw >> (v & 31)) & 1u) ? d : 0u;
}
struct EnumAux {
  uint32_t d, head;
};

// over already-grouped runs (radix path, CSR batches, export: runs = vertices)
struct EnumIn {
  using Aux = EnumAux;
  GraphView g;
  BatchView b;
  int check_alive;
  bool fuse;
  __device__ Sum2 operator()(unsigned long long r64, Aux& x) const {
    const uint32_t r = (uint32_t)r64;
    const uint32_t k = b.run_start != nullptr ? run_len(b, r) : 0u;
    const bool wanted = b.run_start == nullptr || k != 0;  // empty runs: CSR batches
    const uint32_t v = batch_src(b, r);
    x.d = live_degree(g, v, wanted, check_alive);
    x.head = (fuse && wanted && v < g.size) ? g.head[v] : kNull;
    const uint32_t nblk = blocks_for(g, x.d);
    return Sum2{0ull, enum_word_b(nblk, k, fuse), (fuse && fused_class(k, nblk) == kClsMed) ? 1u : 0u};
  }
};
struct EnumOut {
  GraphView g;
  BatchView b;
  EnumLists lists;
  __device__ void operator()(unsigned long long r, unsigned long long, unsigned long long excl_b,
                             Sum2 v, const EnumAux& x) const {
    const uint32_t k = b.run_start != nullptr ? run_len(b, (uint32_t)r) : 0u;
    lists.write((uint32_t)r, x.d, blocks_for(g, x.d), k, x.head, batch_src(b, (uint32_t)r),
                b.run_start != nullptr ? b.run_start[r] : 0u, excl_b, v.c_excl);
  }
};
// fused with the counting group-by: one pass over the batch entries (see GroupPlanIn)
struct GroupEnumIn {
  using Aux = EnumAux;
  GraphView g;
  GroupIndex gi;
  const uint32_t* src;
  const uint32_t* rank;
  const uint32_t* cnt;
  int check_alive;
  bool fuse;
  __device__ Sum2 operator()(unsigned long long i, Aux& x) const {
    const uint32_t s = min(src[i], g.size);  // query batches: unknown sources share one slot
    const bool rep = rank[i] == 0;
    const uint32_t c = rep ? cnt[gi(s)] : 0u;
    x.d = live_degree(g, s, rep, check_alive);
    x.head = (fuse && rep && s < g.size) ? g.head[s] : kNull;
    const uint32_t nblk = blocks_for(g, x.d);
    return Sum2{c ? ((1ull << 32) | c) : 0ull, enum_word_b(nblk, c, fuse), (fuse && fused_class(c, nblk) == kClsMed) ? 1u : 0u};
  }
};
struct GroupEnumOut {
  GraphView g;
  GroupIndex gi;
  const uint32_t* src;
  uint32_t* cnt;
  uint32_t* run_src;
  uint32_t* run_start;
  uint32_t* run_end;
  EnumLists lists;
  __device__ void operator()(unsigned long long i, unsigned long long excl_a, unsigned long long excl_b,
                             Sum2 val, const EnumAux& x) const {
    const uint32_t c = (uint32_t)val.a;
    if (c == 0) return;
    const uint32_t v = min(src[i], g.size);
    const uint32_t r = (uint32_t)(excl_a >> 32);
    const uint32_t es = (uint32_t)excl_a;
    run_src[r] = v;
    run_start[r] = es;
    run_end[r] = es + c;
    cnt[gi(v)] = es;
    lists.write(r, x.d, blocks_for(g, x.d), c, x.head, v, es, excl_b, val.c_excl);
  }
};
struct EnumFin {
  OpState* op;
  unsigned long long wl_cap;
  int set_runs;
  __device__ void operator()(unsigned long long total_a, unsigned long long total_b, unsigned int total_c) const {
    op->n_fmed = total_c;   // sources of the fused medium class (their record slots came out of the scan)
    if (set_runs) op->n_runs = total_a >> 32;
    op->wl_blocks = total_b & 0xFFFFFFFFull;
    op->hole_items = 2ull * (total_b & 0xFFFFFFFFull);
    op->n_big = total_b >> 32;
    if ((total_b & 0xFFFFFFFFull) > wl_cap) {  // cannot happen: wl_cap >= blocks in use (host mirror)
      op->err = 3;
      op->err_detail = kErrScratch;
    }
  }
};

// A warp takes 32 sources; chains of up to kLaneWalk blocks are walked one per
// lane, 32 chains per memory round trip.  Longer chains were listed by the
// scan and go to enumerate_big_kernel.
__global__ void __launch_bounds__(256)
enumerate_walk_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                      const uint32_t* __restrict__ run_deg, uint32_t* __restrict__ wl_handle,
                      uint32_t* __restrict__ wl_run, const OpState* op) {
  if (op->err) return;
  const uint32_t T = (uint32_t)op->n_runs;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < T; r += gridDim.x * blockDim.x) {
    const uint32_t base = wl_off[r];
    const uint32_t nblk = blocks_for(g, run_deg[r]);
    if (nblk == 0 || nblk > kLaneWalk || base >= kClsMin) continue;   // (class words: warp-owned sources)
    uint32_t h = g.head[batch_src(b, r)];
    const uint32_t tag = run_tag(b, r);
    for (uint32_t k = 0; k < nblk; ++k) {
      wl_handle[base + k] = h;
      wl_run[base + k] = tag;
      h = g.next[h];
    }
  }
}

// One warp per long chain.  Each round trip loads next[h .. h+127] and
// confirms the longest prefix with next[h+i] == h+i+1, i.e. a run of
// physically consecutive blocks that really are consecutive in the chain —
// bulk-built hubs advance 128 blocks per memory latency, fragmented chains
// degrade to one block per latency.
__global__ void __launch_bounds__(256)
enumerate_big_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                     const uint32_t* __restrict__ run_deg, const uint32_t* __restrict__ big_list, uint32_t big_cap,
                     uint32_t* __restrict__ wl_handle, uint32_t* __restrict__ wl_run, const OpState* op) {
  if (op->err) return;
  // ---- chains of more than kHugeWalk blocks (the hubs: the critical path of the whole stage): one
  // CTA per chain, every thread checks 4 links, i.e. 1024 blocks per memory round trip
  {
    __shared__ uint32_t s_fail[8];
    __shared__ uint32_t s_next_h;
    const uint32_t nhuge = op->n_huge;
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    for (uint32_t i = blockIdx.x; i < nhuge; i += gridDim.x) {
      const uint32_t r = big_list[big_cap - 1u - i];
      const uint32_t base = wl_off[r];
      const uint32_t nblk = blocks_for(g, run_deg[r]);
      uint32_t h = g.head[batch_src(b, r)];
      const uint32_t tag = run_tag(b, r);
      uint32_t k = 0;
      while (k < nblk) {
        uint32_t nx[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // thread t owns links t + 256 q: coalesced
          const unsigned long long hh = (unsigned long long)h + threadIdx.x + 256u * q;
          nx[q] = (hh < g.ring_cap) ? g.next[hh] : kNull;
        }
        // first link (in chain order) that does not lead to the physically next block
        // (per warp: the smallest failing index among ITS links; chain order interleaves warps per q)
        uint32_t wfail = 1024u;
#pragma unroll
        for (int q = 3; q >= 0; --q) {
          const unsigned long long hh = (unsigned long long)h + threadIdx.x + 256u * q;
          const unsigned m = __ballot_sync(kFull, (unsigned long long)nx[q] != hh + 1);
          if (m) wfail = 256u * q + 32u * warp + (uint32_t)__ffs(m) - 1u;
        }
        if (lane == 0) s_fail[warp] = wfail;
        __syncthreads();
        uint32_t first = 1024u;
#pragma unroll
        for (int w8 = 0; w8 < 8; ++w8) first = min(first, s_fail[w8]);
        // blocks h .. h + len - 1 are consecutive in the chain (the first non-consecutive link still names a valid successor)
        uint32_t len = min(first + 1u, 1024u);
        len = min(len, nblk - k);
        const uint32_t last = len - 1u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t o = threadIdx.x + 256u * q;
          if (o < len) {
            wl_handle[base + k + o] = h + o;
            wl_run[base + k + o] = tag;
          }
          if (o == last) s_next_h = nx[q];
        }
        __syncthreads();
        h = s_next_h;
        k += len;
        __syncthreads();
      }
    }
  }
  const uint32_t nbig = (uint32_t)op->n_big;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nbig; i += nwarps) {
    const uint32_t r = big_list[i];
    const uint32_t base = wl_off[r];
    const uint32_t nblk = blocks_for(g, run_deg[r]);
    uint32_t h = g.head[batch_src(b, r)];
    const uint32_t tag = run_tag(b, r);
    uint32_t k = 0;
    while (k < nblk) {
      uint32_t nx[4];
      unsigned m[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned long long hh = (unsigned long long)h + 32 * q + lane;
        nx[q] = (hh < g.ring_cap) ? g.next[hh] : kNull;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned long long hh = (unsigned long long)h + 32 * q + lane;
        m[q] = __ballot_sync(kFull, (unsigned long long)nx[q] == hh + 1);
      }
      // blocks h .. h+len-1 are consecutive in the chain (block h itself always counts)
      uint32_t len = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (len == 32u * q) len += (m[q] == kFull) ? 32u : (uint32_t)__ffs(~m[q]) - 1u;
      }
      len = min(len + 1, 128u);      // the first non-consecutive link still names a valid successor
      len = min(len, nblk - k);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t o = 32 * q + lane;
        if (o < len) {
          wl_handle[base + k + o] = h + o;
          wl_run[base + k + o] = tag;
        }
      }
      // successor of block h+len-1
      const uint32_t last = len - 1;
      uint32_t nh = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t t = __shfl_sync(kFull, nx[q], last & 31);
        if ((last >> 5) == (uint32_t)q) nh = t;
      }
      h = nh;
      k += len;
    }
  }
}

// ---------------------------------------------------------------------------
// delete: match + tombstone (graph.hpp:376-394) / query: match (graph.hpp:228-241)
//
// The batch is grouped by source only (no order among a source's targets).
//  * match_small_kernel — flat over the worklist, a warp per 32 blocks: each
//    lane resolves one block's metadata, then the warp visits the blocks; the
//    source's targets sit one per lane and are compared by shuffle broadcast
//    (__ballot_sync collects the slot mask).  Sources with more than 32
//    targets on short chains loop over groups of 32 targets.
//  * match_long_kernel — sources with > 32 targets AND a long chain: a CTA per
//    512-block chunk builds an open-addressing table of the targets in shared
//    memory and probes it once per slot.
// Delete records, per block, the bit mask of matched slots (wl_mask) so the
// compaction never re-reads the chains.
// ---------------------------------------------------------------------------
// match_tiny_kernel: sources with at most kTinyTargets targets.
//   B = 32 (one 128-byte line per block): a WARP per 32 consecutive worklist
//   blocks.  Metadata phase: one lane per block (tier tag, handle, source's
//   targets -> the warp's shared-memory strip).  Load phase: the tiny blocks are
//   loaded one slot per lane, all (up to 32) coalesced loads issued before the
//   first compare.  Compare phase: per block, the <= 8 targets are broadcast
//   reads from the strip; __ballot_sync builds the match mask, lane u keeps
//   block u's mask so masks and counters leave coalesced.
//   Other block sizes: the same with 4-byte staging copies and ceil(B / 32) passes of 32 slots
//   (stage_rows32), one mask word per pass.
template <bool kIsDelete, bool kNative>
__global__ void __launch_bounds__(256)
match_tiny_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                  const uint32_t* __restrict__ wl_handle, const uint32_t* __restrict__ wl_run,
                  const uint32_t* __restrict__ run_deg, uint32_t* __restrict__ run_matched,
                  uint32_t* __restrict__ wl_mask, uint8_t* __restrict__ hit, OpState* op) {
  if (op->err) return;
  __shared__ unsigned long long s_warp[8];
  __shared__ __align__(16) uint32_t s_slots[8][32][32];  // [warp][block][slot]
  const uint32_t W = (uint32_t)op->wl_blocks;
  unsigned long long slots = 0;
  {
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = lane_id();
    const uint32_t B = kNative ? 32u : g.B;     // (compile-time constants on the native path)
    const uint32_t mw = kNative ? 1u : g.mw;
    uint32_t(*stg)[32] = s_slots[threadIdx.x >> 5];
    for (uint32_t w0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u; w0 < W; w0 += nwarps * 32u) {
      // ---- metadata: lane = block
      const uint32_t w = w0 + lane;
      uint32_t tag = kTierBit, h = 0;
      if (w < W) {
        tag = wl_run[w];
        h = wl_handle[w];
      }
      const bool tiny = !(tag & kTierBit);
      const unsigned tmask32 = __ballot_sync(kFull, tiny);
      if (tmask32 == 0) continue;
      // ---- stage (first 32 words): every tiny block of the group in flight at once
      if (kNative) stage_blocks32(g, stg, h, tmask32); else stage_rows32(g, stg, h, tmask32, 0);
      uint32_t r = 0, rs = 0, k = 0, cb = 0;
      uint32_t tg[kTinyTargets];
      if (tiny) {
        r = tag;
        rs = b.run_start[r];
        k = b.run_end[r] - rs;
        cb = min(B, run_deg[r] - (w - wl_off[r]) * B);   // live slots of this block
      }
#pragma unroll
      for (int j = 0; j < (int)kTinyTargets; ++j) tg[j] = ((uint32_t)j < k) ? batch_value(b, rs + j) : kTomb;
      slots += cb;
      unsigned long long filt = 0;
#pragma unroll
      for (int j = 0; j < (int)kTinyTargets; ++j)
        if ((uint32_t)j < k) filt |= 1ull << filter_hash(tg[j], 6);
      uint32_t matched = 0;
#pragma unroll 1
      for (uint32_t p = 0; p < mw; ++p) {   // one pass per 32 slots of the block (B = 32: one)
        if (p > 0) stage_rows32(g, stg, h, tmask32, p);
        cp_async_wait_all();
        __syncwarp();
        // ---- compare: lane = block.  Pass 1 tests every slot against a 64-bit filter of the lane's
        // targets (6 instructions per slot); pass 2 compares only the few candidates exactly.
        if (tiny) {
          const uint32_t cnt = cb > 32u * p ? min(32u, cb - 32u * p) : 0u;
          uint32_t cand = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = block_chunk(stg, lane, c);
            cand |= (uint32_t)((filt >> filter_hash(v.x, 6)) & 1ull) << (4 * c);
            cand |= (uint32_t)((filt >> filter_hash(v.y, 6)) & 1ull) << (4 * c + 1);
            cand |= (uint32_t)((filt >> filter_hash(v.z, 6)) & 1ull) << (4 * c + 2);
            cand |= (uint32_t)((filt >> filter_hash(v.w, 6)) & 1ull) << (4 * c + 3);
          }
          cand &= cnt == 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1u);  // slots past deg (and past B) hold stale values
          uint32_t mask = 0;
          while (cand) {
            const uint32_t bit = __ffs(cand) - 1;
            cand &= cand - 1;
            const uint32_t e = block_slot(stg, lane, bit);
#pragma unroll
            for (int j = 0; j < (int)kTinyTargets; ++j) {
              if ((uint32_t)j < k && e == tg[j]) {
                mask |= 1u << bit;
                if (!kIsDelete) hit[rs + j] = 1;
              }
            }
          }
          if (kIsDelete) {
            wl_mask[(unsigned long long)w * mw + p] = mask;
            matched += (uint32_t)__popc(mask);
            while (mask) {
              const uint32_t bit = __ffs(mask) - 1;
              mask &= mask - 1;
              g.slab[(unsigned long long)h * B + 32u * p + bit] = kTomb;
            }
          }
        }
        __syncwarp();   // the rows are restaged by the next pass / group
      }
      if (kIsDelete && matched) atomicAdd(&run_matched[r], matched);
    }
  }
  const unsigned long long t = block_reduce_sum(slots, s_warp);
  if (threadIdx.x == 0 && t) {
    atomicAdd(&op->slots, t);
    atomicAdd(&op->slots_tiny, t);
  }
}

// Open-addressing table of u32 keys in shared memory; kTomb marks an empty slot
// (never a valid destination id).
__device__ __forceinline__ void table_insert(uint32_t* tab, uint32_t tmask, int hshift, uint32_t* bm,
                                             int bm_bits, uint32_t x) {
  const uint32_t hb = filter_hash(x, bm_bits);
  atomicOr(&bm[hb >> 5], 1u << (hb & 31));
  uint32_t pos = (x * 0x9E3779B1u) >> hshift;
#pragma unroll 1
  while (true) {
    const uint32_t old = atomicCAS(&tab[pos], kTomb, x);
    if (old == kTomb || old == x) break;
    pos = (pos + 1) & tmask;
  }
}
// returns the slot holding x, or -1
__device__ __forceinline__ int table_find(const uint32_t* tab, uint32_t tmask, int hshift, uint32_t x) {
  uint32_t pos = (x * 0x9E3779B1u) >> hshift;
  while (true) {
    const uint32_t t = tab[pos];
    if (t == x) return (int)pos;
    if (t == kTomb) return -1;
    pos = (pos + 1) & tmask;
  }
}

// Scans up to 32 blocks of one chain against a shared-memory table.  `hd_lane`
// holds the handle of block u in lane u.  first: this is the first (or only)
// table slice for these blocks, so the mask words are stored rather than OR-ed.
// Returns the number of matches (valid in every lane).
//   ALL blocks of the group are staged in the warp's shared-memory strip `stg` with
//   asynchronous copies (B = 32: one 128-byte line per block, 16-byte copies; other
//   block sizes: 32 words per pass, 4-byte copies, ceil(B / 32) passes), then each
//   lane filters and probes the 32 staged slots of ITS block; lane u keeps block
//   u's mask word so the masks leave coalesced.
template <bool kIsDelete, bool kNative>
__device__ __forceinline__ uint32_t table_scan(const GraphView& g, const uint32_t* tab, uint8_t* flag,
                                               uint32_t tmask, int hshift, const uint32_t* bm, int bm_bits,
                                               uint32_t (*stg)[32],
                                               uint32_t hd_lane, uint32_t ng, uint32_t d,
                                               uint32_t kb_first, uint32_t w_first,
                                               uint32_t* __restrict__ wl_mask, bool first,
                                               unsigned long long& slots) {
  const int lane = lane_id();
  const uint32_t B = kNative ? 32u : g.B;     // (compile-time constants on the native path)
  const uint32_t mw = kNative ? 1u : g.mw;
  const unsigned want = ng >= 32 ? 0xFFFFFFFFu : ((1u << ng) - 1u);
  // live slots of the lane's block: every block but possibly the chain's last one is full
  const uint32_t rem = d - kb_first * B;              // slots from the group's first block to the chain end
  const uint32_t cb = ((uint32_t)lane < ng && rem > B * lane) ? min(B, rem - B * lane) : 0u;
  uint32_t matched = 0;
#pragma unroll 1
  for (uint32_t p = 0; p < mw; ++p) {   // one pass per 32 slots of the blocks (B = 32: one)
    // ALL blocks of the group are staged in the warp's shared-memory strip with asynchronous copies
    // (up to 32 x 128 bytes in flight per warp)
    if (kNative) stage_blocks32(g, stg, hd_lane, want); else stage_rows32(g, stg, hd_lane, want, p);
    cp_async_wait_all();
    __syncwarp();
    // lane = block.  Pass 1 tests the lane's 32 slots against the bitmap filter of the targets;
    // pass 2 probes the table only for the candidates.
    uint32_t mask = 0;
    if ((uint32_t)lane < ng) {
      const uint32_t cnt = cb > 32u * p ? min(32u, cb - 32u * p) : 0u;
      uint32_t cand = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = block_chunk(stg, lane, c);
        const uint32_t evs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t hb = filter_hash(evs[i], bm_bits);
          cand |= ((bm[hb >> 5] >> (hb & 31)) & 1u) << (4 * c + i);
        }
      }
      cand &= cnt == 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1u);  // stale padding
      while (cand) {
        const uint32_t bit = __ffs(cand) - 1;
        cand &= cand - 1;
        const uint32_t ev = block_slot(stg, lane, bit);
        if (ev == kTomb) continue;  // tombstone of an earlier slice
        uint32_t pos = (ev * 0x9E3779B1u) >> hshift;
        uint32_t t = tab[pos];
        while (t != ev && t != kTomb) {
          pos = (pos + 1) & tmask;
          t = tab[pos];
        }
        if (t == ev) {
          mask |= 1u << bit;
          if (!kIsDelete) flag[pos] = 1;
        }
      }
      if (kIsDelete) {
        uint32_t* mword = &wl_mask[(unsigned long long)(w_first + lane) * mw + p];
        if (first) *mword = mask;
        else if (mask) *mword |= mask;  // the same warp owns these blocks in every slice
        uint32_t m2 = mask;
        while (m2) {
          const uint32_t bit = __ffs(m2) - 1;
          m2 &= m2 - 1;
          g.slab[(unsigned long long)hd_lane * B + 32u * p + bit] = kTomb;
        }
      }
    }
    matched += __popc(mask);
    __syncwarp();  // the staging strip is reused by the next pass / the caller's next group
  }
#pragma unroll
  for (int dlt = 16; dlt > 0; dlt >>= 1) matched += __shfl_xor_sync(kFull, matched, dlt);
  if (first) {
    uint32_t gs = cb;
#pragma unroll
    for (int dlt = 16; dlt > 0; dlt >>= 1) gs += __shfl_xor_sync(kFull, gs, dlt);
    if (lane == 0) slots += gs;
  }
  return matched;
}

// match_med_kernel: a WARP per (source, 32-block chunk) item, sources with
// kTinyTargets < k <= kMedTargets targets; the warp keeps the source's targets
// in its own 256-entry shared-memory table.
constexpr uint32_t kMedTable = 512;   // >= 4 x kMedTargets: short probe sequences
// dynamic shared memory: per warp a table, a staging strip and (query) flags
constexpr int kMedFilterBits = 12;     // 4096-bit membership filter per warp: <= 3% false positives
constexpr size_t kMedSmemDelete = 8 * (kMedTable * 4 + 32 * 32 * 4 + (1u << kMedFilterBits) / 8);
constexpr size_t kMedSmemQuery = kMedSmemDelete + 8 * kMedTable;
template <bool kIsDelete, bool kNative>
__global__ void __launch_bounds__(256, 4)
match_med_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                 const uint32_t* __restrict__ wl_handle, const uint2* __restrict__ items,
                 const uint32_t* __restrict__ run_deg, uint32_t* __restrict__ run_matched,
                 uint32_t* __restrict__ wl_mask, uint8_t* __restrict__ hit, OpState* op) {
  if (op->err) return;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ unsigned long long s_warp[8];
  const uint32_t n_items = (uint32_t)op->n_med;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  uint32_t(*stg)[32] = reinterpret_cast<uint32_t(*)[32]>(dyn_smem + (size_t)warp * 32 * 32 * 4);
  uint32_t* tab = reinterpret_cast<uint32_t*>(dyn_smem + 8 * 32 * 32 * 4) + warp * kMedTable;
  uint32_t* bm = reinterpret_cast<uint32_t*>(dyn_smem + 8 * (32 * 32 * 4 + kMedTable * 4)) + warp * ((1u << kMedFilterBits) / 32);
  uint8_t* flag = dyn_smem + kMedSmemDelete + (kIsDelete ? 0 : warp * kMedTable);
  constexpr int hshift = 32 - 9;
  constexpr uint32_t tmask = kMedTable - 1;
  static_assert(kMedTable == 512, "hshift matches the table size");
  unsigned long long slots = 0;
  // items are handed out through a device cursor (they differ 30x in size); the next
  // ticket is requested before the current item is processed
  uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  while (q < n_items) {
    uint32_t q_next = 0;
    if (lane == 0) q_next = nwarps + atomicAdd(&op->med_cursor, 1u);
    const uint2 it = items[q];
    const uint32_t r = it.x, c = it.y;
    const uint32_t rs = b.run_start[r];
    const uint32_t k = b.run_end[r] - rs;
    const uint32_t d = run_deg[r];
    const uint32_t nblk = blocks_for(g, d);
    const uint32_t wbase = wl_off[r];
    const uint32_t kb0 = c * kMedChunk;
    const uint32_t nb = min(kMedChunk, nblk - kb0);
    const uint32_t hd_all = ((uint32_t)lane < nb) ? wl_handle[wbase + kb0 + lane] : 0u;
    for (uint32_t i = lane; i < kMedTable; i += 32) {
      tab[i] = kTomb;
      if (!kIsDelete) flag[i] = 0;
    }
    for (uint32_t i = lane; i < (1u << kMedFilterBits) / 32; i += 32) bm[i] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < k; i += 32)
      table_insert(tab, tmask, hshift, bm, kMedFilterBits, batch_value(b, rs + i));
    __syncwarp();
    const uint32_t matched = table_scan<kIsDelete, kNative>(g, tab, flag, tmask, hshift, bm, kMedFilterBits, stg, hd_all, nb,
                                                   d, kb0, wbase + kb0, wl_mask, true, slots);
    if (kIsDelete) {
      if (lane == 0 && matched) atomicAdd(&run_matched[r], matched);
    } else {
      __syncwarp();
      for (uint32_t i = lane; i < k; i += 32) {
        const int pos = table_find(tab, tmask, hshift, batch_value(b, rs + i));
        if (pos >= 0 && flag[pos]) hit[rs + i] = 1;
      }
    }
    __syncwarp();
    q = __shfl_sync(kFull, q_next, 0);
  }
  const unsigned long long t = block_reduce_sum(slots, s_warp);
  if (threadIdx.x == 0 && t) atomicAdd(&op->slots, t);
}

// match_long_kernel: sources with more than kMedTargets targets.  A CTA per
// kLongChunk-block chunk builds the table of the source's targets in shared
// memory (sized to the target count; kSliceTargets per build) and probes it
// once per slot; warps take groups of four blocks round-robin.
constexpr int kLongThreads = 256;
constexpr uint32_t kTableSize = 8192;      // shared-memory table capacity (u32 keys)
constexpr uint32_t kSliceTargets = 4096;   // targets per table build: load factor <= 0.5
constexpr int kLongFilterBits = 16;    // 64K-bit membership filter per CTA: <= 6% false positives per slice
constexpr size_t kLongSmemDelete = (kLongThreads / 32) * 32 * 32 * 4 + kTableSize * 4 + (1u << kLongFilterBits) / 8;
constexpr size_t kLongSmemQuery = kLongSmemDelete + kTableSize;

template <bool kIsDelete, bool kNative>
__global__ void __launch_bounds__(kLongThreads)
match_long_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                  const uint32_t* __restrict__ wl_handle, const uint2* __restrict__ items,
                  const uint32_t* __restrict__ run_deg, uint32_t* __restrict__ run_matched,
                  uint32_t* __restrict__ wl_mask, uint8_t* __restrict__ hit, OpState* op) {
  if (op->err) return;
  constexpr int kWarps = kLongThreads / 32;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ unsigned long long s_warp[kWarps];
  uint32_t(*stg)[32] = reinterpret_cast<uint32_t(*)[32]>(dyn_smem + (size_t)(threadIdx.x >> 5) * 32 * 32 * 4);
  uint32_t* s_table = reinterpret_cast<uint32_t*>(dyn_smem + kWarps * 32 * 32 * 4);
  uint32_t* s_bm = s_table + kTableSize;
  uint8_t* s_flag = dyn_smem + kLongSmemDelete;
  const uint32_t n_items = (uint32_t)op->n_items;
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  unsigned long long slots = 0;
  __shared__ uint32_t s_next;
  uint32_t q = blockIdx.x;
  while (q < n_items) {
    if (threadIdx.x == 0) s_next = gridDim.x + atomicAdd(&op->long_cursor, 1u);
    const uint2 it = items[q];
    const uint32_t r = it.x, c = it.y;
    const uint32_t rs = b.run_start[r];
    const uint32_t k = b.run_end[r] - rs;
    const uint32_t d = run_deg[r];
    const uint32_t nblk = blocks_for(g, d);
    const uint32_t wbase = wl_off[r];
    const uint32_t kb0 = c * kLongChunk;
    const uint32_t kb1 = min(nblk, kb0 + kLongChunk);
    const uint32_t ngroups = (kb1 - kb0 + 31) / 32;
    unsigned long long matched = 0;
    for (uint32_t t0 = 0; t0 < k; t0 += kSliceTargets) {
      const uint32_t nt = min(kSliceTargets, k - t0);
      // table of 2^tb >= 2 * nt entries (at least 64)
      const int tb = max(6, 32 - __clz(2 * nt - 1));
      const uint32_t tsize = 1u << tb, tmask = tsize - 1u;
      const int hshift = 32 - tb;
      for (uint32_t i = threadIdx.x; i < tsize; i += kLongThreads) {
        s_table[i] = kTomb;
        if (!kIsDelete) s_flag[i] = 0;
      }
      for (uint32_t i = threadIdx.x; i < (1u << kLongFilterBits) / 32; i += kLongThreads) s_bm[i] = 0;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nt; i += kLongThreads)
        table_insert(s_table, tmask, hshift, s_bm, kLongFilterBits, batch_value(b, rs + t0 + i));
      __syncthreads();
      for (uint32_t gi = warp; gi < ngroups; gi += kWarps) {
        const uint32_t kbg = kb0 + 32 * gi;
        const uint32_t ng = min(32u, kb1 - kbg);
        const uint32_t hd_lane = ((uint32_t)lane < ng) ? wl_handle[wbase + kbg + lane] : 0u;
        const uint32_t mm = table_scan<kIsDelete, kNative>(g, s_table, s_flag, tmask, hshift, s_bm, kLongFilterBits, stg,
                                                  hd_lane, ng, d, kbg, wbase + kbg, wl_mask, t0 == 0, slots);
        if (lane == 0) matched += mm;
      }
      __syncthreads();
      if (!kIsDelete) {
        for (uint32_t i = threadIdx.x; i < nt; i += kLongThreads) {
          const int pos = table_find(s_table, tmask, hshift, batch_value(b, rs + t0 + i));
          if (pos >= 0 && s_flag[pos]) hit[rs + t0 + i] = 1;
        }
        __syncthreads();
      }
    }
    if (kIsDelete) {
      const unsigned long long tm = block_reduce_sum(matched, s_warp);
      if (threadIdx.x == 0 && tm) atomicAdd(&run_matched[r], (uint32_t)tm);
    }
    __syncthreads();
    q = s_next;
    __syncthreads();
  }
  const unsigned long long t = block_reduce_sum(slots, s_warp);
  if (threadIdx.x == 0 && t) {
    atomicAdd(&op->slots, t);
    atomicAdd(&op->slots_long, t);
  }
}

// ---------------------------------------------------------------------------
// delete, hub path: compaction of the chains the match tiers tombstoned.
//
// A source with m matches keeps nd = d - m entries: every hole (matched slot) BELOW nd takes a survivor (live slot)
// from AT OR ABOVE nd; holes and survivors are equally many.  Which survivor fills which hole is free, so both are
// simply numbered in chain order: ONE ordered scan over the work list gives every block the number of holes (and of
// survivors) in the blocks before it, survivor j of a source moves into hole j of the source.  The hole list is never
// materialised — a block's holes are the bits of its match mask — so the scratch is two prefix words per work-list
// block, bounded by the blocks in use and known before the op is enqueued (round 1 kept a list of hole addresses
// whose size, up to live edges / 2, was only known after the match: a host-side grow-and-retry in the middle of the op).
// ---------------------------------------------------------------------------
struct NoAux {};
// blocks past each source's new tail go back to the ring: the plan hands every source its range of ring positions,
// so the push needs neither atomics nor barriers (reclaim, block_pool.hpp:192-209)
struct MovesIn {
  using Aux = NoAux;
  GraphView g;
  const uint32_t* run_deg;
  const uint32_t* run_matched;
  __device__ Sum2 operator()(unsigned long long r, Aux&) const {
    const uint32_t m = run_matched[r];
    const uint32_t d = run_deg[r];
    const uint32_t nd = d - m;
    const uint32_t freed = (m != 0 && g.reclaim) ? blocks_for(g, d) - blocks_for(g, nd) : 0u;
    return Sum2{freed, 0ull};
  }
};
struct MovesOut {
  uint32_t* free_off;
  __device__ void operator()(unsigned long long r, unsigned long long excl_a, unsigned long long,
                             Sum2, const NoAux&) const {
    free_off[r] = (uint32_t)excl_a;
  }
};
struct MovesFin {
  GraphView g;
  OpState* op;
  __device__ void operator()(unsigned long long total_a, unsigned long long, unsigned int) const {
    // one cursor bump for the whole batch (atomics: the warp-owned sources push to the same ring from
    // fused_delete_kernel, side by side)
    op->front_old = atomicAdd(&g.st->rear, total_a);   // first ring position of the pushed handles
    atomicAdd(&op->pushed, total_a);
  }
};

// holes below / survivors at or above the new degree in work-list block w
struct BlockHoles {
  uint32_t holes, survivors;
};
__device__ __forceinline__ BlockHoles block_holes(const GraphView& g, const uint32_t* __restrict__ wl_off,
                                                  const uint32_t* __restrict__ wl_run, const uint32_t* __restrict__ run_deg,
                                                  const uint32_t* __restrict__ run_matched, const uint32_t* __restrict__ wl_mask,
                                                  uint32_t w) {
  const uint32_t r = wl_run[w] & kRunMask;
  const uint32_t m = run_matched[r];
  if (m == 0) return BlockHoles{0u, 0u};
  const uint32_t d = run_deg[r];
  const uint32_t nd = d - m;
  const uint32_t base = (w - wl_off[r]) * g.B;
  const uint32_t cnt = min(g.B, d - base);               // live + tombstoned slots of the block
  const uint32_t lo = nd > base ? min(cnt, nd - base) : 0u;   // slots [0, lo) lie below the new degree
  uint32_t below = 0, above = 0;
  for (uint32_t i = 0; i < g.mw && 32u * i < cnt; ++i) {
    const uint32_t bits = wl_mask[(unsigned long long)w * g.mw + i] & low_bits32(cnt - 32u * i);
    const uint32_t lo_bits = lo > 32u * i ? low_bits32(lo - 32u * i) : 0u;
    below += __popc(bits & lo_bits);
    above += __popc(bits & ~lo_bits);
  }
  return BlockHoles{below, (cnt - lo) - above};
}
// ordered scan over 2 W items: [0, W) holes per block, [W, 2 W) survivors per block; prefix[i] = exclusive prefix
struct HoleScanIn {
  GraphView g;
  const uint32_t *wl_off, *wl_run, *run_deg, *run_matched, *wl_mask;
  const OpState* op;
  __device__ unsigned long long operator()(unsigned long long i) const {
    const unsigned long long W = op->wl_blocks;
    const BlockHoles h = block_holes(g, wl_off, wl_run, run_deg, run_matched, wl_mask, (uint32_t)(i < W ? i : i - W));
    return i < W ? h.holes : h.survivors;
  }
};
// (prefixes are kept modulo 2^32: only differences inside one source are ever taken, and a source has < 2^32 slots)
struct HoleScanOut {
  uint32_t* prefix;
  __device__ void operator()(unsigned long long i, unsigned long long excl, unsigned long long) const { prefix[i] = (uint32_t)excl; }
};
struct HoleScanFin {
  uint32_t* prefix;
  const OpState* op;
  __device__ void operator()(unsigned long long total) const { prefix[2ull * op->wl_blocks] = (uint32_t)total; }
};

// delete, step A — a thread per block of the touched chains: returns blocks past the new tail to the ring rear at
// the positions the plan reserved for their source (block_pool.hpp:192-209) and, on a source's first block,
// repairs degree / tail / head (detach_empty_tail, graph.hpp:398-414).  No barriers, no shared cursor.
__global__ void __launch_bounds__(256)
delete_holes_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                    const uint32_t* __restrict__ wl_handle, const uint32_t* __restrict__ wl_run,
                    const uint32_t* __restrict__ run_deg, const uint32_t* __restrict__ run_matched,
                    const uint32_t* __restrict__ free_off, OpState* op) {
  if (op->err) return;
  __shared__ unsigned long long s_warp[8];
  const uint32_t W = (uint32_t)op->wl_blocks;
  const unsigned long long rear_old = op->front_old;
  unsigned long long matched = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x) {
    const uint32_t r = wl_run[w] & kRunMask;
    const uint32_t m = run_matched[r];
    if (m == 0) continue;
    const uint32_t h = wl_handle[w];
    const uint32_t kb = w - wl_off[r];
    const uint32_t d = run_deg[r];
    const uint32_t nd = d - m;
    const uint32_t new_nb = blocks_for(g, nd);
    if (kb >= new_nb && g.reclaim)   // past the new tail: back to the ring, at the source's reserved positions
      g.ring[(rear_old + free_off[r] + (kb - new_nb)) % g.ring_cap] = h;
    if (kb == 0) {
      const uint32_t v = batch_src(b, r);
      g.deg[v] = nd;
      if (nd == 0) {
        g.head[v] = kNull;
        g.tail[v] = kNull;
      } else {
        const uint32_t t = wl_handle[wl_off[r] + new_nb - 1];
        g.tail[v] = t;
        g.next[t] = kNull;
      }
      matched += m;
    }
  }
  const unsigned long long tm = block_reduce_sum(matched, s_warp);
  if (threadIdx.x == 0) {
    if (tm) {
      atomicAdd(&op->matched, tm);
      atomicAdd(&g.st->active_edges, (unsigned long long)(-(long long)tm));  // graph.hpp:211-213
    }
  }
}

// delete, step B — a WARP per block of the touched chains, lane = slot; only blocks reaching past the new degree do
// anything: survivor j of the source (numbered in chain order by the scan) moves into hole j.  One binary search
// over the source's hole prefixes (the same for every lane) finds the block of the block's first hole; each lane
// then steps from there to the block of its own hole — consecutive survivors take consecutive holes.  Every lane's
// chain of dependent loads is a handful long: under the fused kernel's memory load a dependent access costs ~2 us.
__global__ void __launch_bounds__(256)
delete_moves_kernel(GraphView g, const uint32_t* __restrict__ wl_off,
                    const uint32_t* __restrict__ wl_handle, const uint32_t* __restrict__ wl_run,
                    const uint32_t* __restrict__ run_deg, const uint32_t* __restrict__ run_matched,
                    const uint32_t* __restrict__ wl_mask, const uint32_t* __restrict__ prefix,
                    OpState* op) {
  if (op->err) return;
  const uint32_t W = (uint32_t)op->wl_blocks;
  const uint32_t* H = prefix;        // holes in the work-list blocks before w (mod 2^32)
  const uint32_t* S = prefix + W;    // survivors in the work-list blocks before w (+ all holes, mod 2^32)
  const int lane = lane_id();
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t moves = 0;
  const uint32_t warp_id = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (uint32_t it = 0; warp_id + (unsigned long long)nwarps * 32u * it < W; ++it) {
   // 32 work-list blocks per warp and step, one per lane, STRIDED by the warp count: their survivor counts are looked
   // at in one round trip, and neighbouring blocks — the last blocks of a hub, where its survivors sit — belong to
   // different warps, so they are moved in parallel
   const unsigned long long wl = warp_id + (unsigned long long)nwarps * (32u * it + (uint32_t)lane);
   unsigned todo = __ballot_sync(kFull, wl < W && S[wl + 1] != S[wl]);
   while (todo) {
    const uint32_t w = warp_id + nwarps * (32u * it + (uint32_t)(__ffs(todo) - 1));
    todo &= todo - 1;
    const uint32_t r = wl_run[w] & kRunMask;
    const uint32_t w0 = wl_off[r];
    const uint32_t d = run_deg[r];
    const uint32_t nd = d - run_matched[r];
    const uint32_t base = (w - w0) * g.B;
    const uint32_t cnt = min(g.B, d - base);
    const uint32_t lo = nd > base ? min(cnt, nd - base) : 0u;
    const uint32_t j0 = S[w] - S[w0];   // hole rank of this block's first survivor
    const uint32_t Hw0 = H[w0];
    // largest block of [w0, w0 + new_nb) with H - H[w0] <= j0 (an empty block shares its prefix with its successor):
    // a 32-ary search, every lane probes one position per step — three dependent loads for 32 K blocks
    const uint32_t w_hend = w0 + blocks_for(g, nd);
    uint32_t a = w0, z = w_hend;   // answer in [a, z)
    while (z - a > 1) {
      const uint32_t span = z - a;
      const uint32_t stp = (span + 31u) / 32u;
      const uint32_t probe = a + (uint32_t)lane * stp;
      const bool le = probe < z && (uint32_t)(H[probe] - Hw0) <= j0;
      const unsigned mle = __ballot_sync(kFull, le);   // a prefix of the lanes (H is monotone); lane 0 always holds
      const uint32_t last = 31u - (uint32_t)__clz(mle);
      a = a + last * stp;
      z = min(z, a + stp);
    }
    const uint32_t* blk = g.slab + (unsigned long long)wl_handle[w] * g.B;
    uint32_t done = 0;   // survivors of the block's earlier 32-slot rows
    for (uint32_t s0 = 0; s0 < cnt; s0 += 32) {
      const uint32_t s = s0 + lane;
      const uint32_t mword = wl_mask[(unsigned long long)w * g.mw + (s0 >> 5)];
      const bool surv = s >= lo && s < cnt && !((mword >> lane) & 1u);
      const unsigned sm = __ballot_sync(kFull, surv);
      if (surv) {
        const uint32_t e = blk[s];
        const uint32_t j = j0 + done + __popc(sm & ((1u << lane) - 1u));   // this survivor's hole rank in the source
        // the block of THIS survivor's hole: at or after the block of the first one.  A lane-private binary search —
        // holes may be sparse (a small batch in a long chain), so stepping block by block could take hundreds of
        // dependent loads
        uint32_t hb = a, hz = w_hend;
        while (hz - hb > 1) {
          const uint32_t mid = hb + ((hz - hb) >> 1);
          if ((uint32_t)(H[mid] - Hw0) <= j) hb = mid; else hz = mid;
        }
        uint32_t k = j - (uint32_t)(H[hb] - Hw0);
        // the k-th hole of block hb: set bits of its mask below the new degree
        const uint32_t hlim = min(g.B, nd - (hb - w0) * g.B);
        uint32_t slot = 0;
        for (uint32_t i = 0; i < g.mw; ++i) {
          const uint32_t bits = wl_mask[(unsigned long long)hb * g.mw + i] & (hlim > 32u * i ? low_bits32(hlim - 32u * i) : 0u);
          const uint32_t c = __popc(bits);
          if (k < c) {
            slot = 32u * i + __fns(bits, 0, (int)k + 1);
            break;
          }
          k -= c;
        }
        g.slab[(unsigned long long)wl_handle[hb] * g.B + slot] = e;
        ++moves;
      }
      done += __popc(sm);
    }
   }
  }
#pragma unroll
  for (int dl = 16; dl > 0; dl >>= 1) moves += __shfl_xor_sync(kFull, moves, dl);
  if (lane == 0 && moves) atomicAdd(&op->moves, (unsigned long long)moves);
}

// query: scatter sorted hit flags back to the caller's order
__global__ void query_scatter_kernel(const uint8_t* __restrict__ hit,
                                     const uint32_t* __restrict__ index, uint32_t n,
                                     uint8_t* __restrict__ out, OpState* op) {
  __shared__ unsigned long long s_warp[32];
  unsigned long long c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint8_t hv = hit[i];
    out[index[i]] = hv;
    c += hv;
  }
  const unsigned long long t = block_reduce_sum(c, s_warp);
  if (threadIdx.x == 0 && t) atomicAdd(&op->matched, t);
}

// ---------------------------------------------------------------------------
// vertex delete (graph.hpp:252-276): winners were chosen by the host mirror
// of the alive flags; one warp per retired vertex frees its chain.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
retire_vertices_kernel(GraphView g, const uint32_t* __restrict__ ids, uint32_t n, OpState* op) {
  __shared__ unsigned long long s_warp[8];
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  unsigned long long edges = 0, pushed = 0;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const uint32_t v = ids[i];
    const uint32_t d = g.deg[v];
    if (lane == 0) {
      atomicAnd(&g.alive[v >> 5], ~(1u << (v & 31)));  // retire (vertex_dictionary.hpp:75-78)
      edges += d;
    }
    if (g.reclaim && d > 0) {
      const uint32_t nblk = ceil_div(d, g.B);
      uint32_t h = g.head[v];
      uint32_t k = 0;
      while (k < nblk) {
        const unsigned long long hh = (unsigned long long)h + lane;
        const uint32_t nx = (hh < g.ring_cap) ? g.next[hh] : kNull;
        const bool ok = (unsigned long long)nx == hh + 1;
        const unsigned m = __ballot_sync(kFull, ok);
        uint32_t len = (m == kFull) ? 32u : (uint32_t)__ffs(~m);
        len = min(len, nblk - k);
        unsigned long long pos = 0;
        if (lane == 0) pos = atomicAdd(&g.st->rear, (unsigned long long)len);
        pos = __shfl_sync(kFull, pos, 0);
        if ((uint32_t)lane < len) g.ring[(pos + lane) % g.ring_cap] = (uint32_t)hh;
        h = __shfl_sync(kFull, nx, len - 1);
        k += len;
      }
      if (lane == 0) {
        pushed += nblk;
        g.head[v] = kNull;   // s = EdgeSentinel{} (graph.hpp:272)
        g.tail[v] = kNull;
        g.deg[v] = 0;
      }
    }
  }
  const unsigned long long te = block_reduce_sum(edges, s_warp);
  const unsigned long long tp = block_reduce_sum(pushed, s_warp);
  if (threadIdx.x == 0) {
    if (te) atomicAdd(&g.st->active_edges, (unsigned long long)(-(long long)te));  // graph.hpp:263
    if (tp) atomicAdd(&op->pushed, tp);
  }
}

// ---------------------------------------------------------------------------
// export / observables
// ---------------------------------------------------------------------------
struct DegIn {
  const uint32_t* deg;
  __device__ unsigned long long operator()(unsigned long long v) const { return deg[v]; }
};
struct OffsetsOut {
  unsigned long long* offsets;
  __device__ void operator()(unsigned long long v, unsigned long long excl,
                             unsigned long long) const {
    offsets[v] = excl;
  }
};
struct OffsetsFin {
  unsigned long long* offsets;
  unsigned long long n;
  OpState* op;
  __device__ void operator()(unsigned long long total) const {
    offsets[n] = total;
    op->aux0 = total;
  }
};

// active_destinations (graph.hpp:116-129) for every vertex: one warp per block.
// With keys_out != nullptr writes (v<<32|dst) keys for the canonical sort
// instead of plain destinations.
__global__ void __launch_bounds__(256)
export_copy_kernel(GraphView g, const uint32_t* __restrict__ wl_off,
                   const uint32_t* __restrict__ wl_handle, const uint32_t* __restrict__ wl_run,
                   const uint32_t* __restrict__ run_deg,
                   const unsigned long long* __restrict__ offsets, uint32_t* __restrict__ dst_out,
                   unsigned long long* __restrict__ keys_out, const OpState* op) {
  if (op->err) return;
  const uint32_t W = (uint32_t)op->wl_blocks;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < W; w += nwarps) {
    const uint32_t v = wl_run[w] & kRunMask;  // runs are vertices on the export path
    const uint32_t h = wl_handle[w];
    const uint32_t k = w - wl_off[v];
    const uint32_t cnt = min(g.B, run_deg[v] - k * g.B);
    const uint32_t* blk = g.slab + (unsigned long long)h * g.B;
    const unsigned long long o = offsets[v] + (unsigned long long)k * g.B;
    for (uint32_t s = lane; s < cnt; s += 32) {
      const uint32_t e = blk[s];
      if (keys_out) keys_out[o + s] = ((unsigned long long)v << 32) | e;
      else dst_out[o + s] = e;
    }
  }
}

// active_destinations(v) (graph.hpp:116-129) for ONE vertex: one CTA.  Warp 0 walks the chain, confirming up to
// 32 physically consecutive blocks per round trip; the whole CTA then copies that run (chains are compact: the
// live entries are exactly positions [0, degree) in chain order).  op->aux0 = the vertex's degree; at most `cap`
// entries are written.
__global__ void __launch_bounds__(256)
adjacency_copy_kernel(GraphView g, uint32_t v, uint32_t* __restrict__ out, unsigned long long cap, OpState* op) {
  __shared__ uint32_t s_h, s_len;
  const uint32_t d = v < g.size ? g.deg[v] : 0u;
  if (threadIdx.x == 0) op->aux0 = d;
  if (d == 0) return;
  const uint32_t nblk = blocks_for(g, d);
  const unsigned long long lim = cap < d ? cap : (unsigned long long)d;
  uint32_t h = g.head[v];
  uint32_t kb = 0;
  while (kb < nblk) {
    if (threadIdx.x < 32) {
      const unsigned long long hh = (unsigned long long)h + threadIdx.x;
      const uint32_t nx = hh < g.ring_cap ? g.next[hh] : kNull;
      const unsigned okm = __ballot_sync(kFull, (unsigned long long)nx == hh + 1);
      uint32_t len = (okm == kFull) ? 32u : (uint32_t)__ffs(~okm);
      len = min(len, nblk - kb);
      const uint32_t nh = __shfl_sync(kFull, nx, len - 1);
      if (threadIdx.x == 0) {
        s_len = len;
        s_h = nh;
      }
    }
    __syncthreads();
    const uint32_t len = s_len;
    const unsigned long long first = (unsigned long long)kb * g.B;
    const unsigned long long count = (unsigned long long)len * g.B;
    for (unsigned long long i = threadIdx.x; i < count; i += blockDim.x)
      if (first + i < lim) out[first + i] = g.slab[(unsigned long long)h * g.B + i];
    const uint32_t nh = s_h;
    __syncthreads();
    h = nh;
    kb += len;
  }
}

__global__ void keys_low_kernel(const unsigned long long* __restrict__ keys, unsigned long long n,
                                uint32_t* __restrict__ out) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    out[i] = (uint32_t)keys[i];
}

__global__ void degrees_kernel(const uint32_t* __restrict__ deg, uint32_t n,
                               unsigned long long* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = deg[i];
}

// sum over stored copies of mix64(src<<32|dst)
__global__ void __launch_bounds__(256)
digest_kernel(GraphView g, const uint32_t* __restrict__ wl_off,
              const uint32_t* __restrict__ wl_handle, const uint32_t* __restrict__ wl_run,
              const uint32_t* __restrict__ run_deg, OpState* op) {
  __shared__ unsigned long long s_warp[8];
  const uint32_t W = (uint32_t)op->wl_blocks;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  unsigned long long acc = 0, cntacc = 0;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < W; w += nwarps) {
    const uint32_t v = wl_run[w] & kRunMask;
    const uint32_t h = wl_handle[w];
    const uint32_t k = w - wl_off[v];
    const uint32_t cnt = min(g.B, run_deg[v] - k * g.B);
    const uint32_t* blk = g.slab + (unsigned long long)h * g.B;
    for (uint32_t s = lane; s < cnt; s += 32) {
      acc += mix64(((unsigned long long)v << 32) | blk[s]);
      ++cntacc;
    }
  }
  const unsigned long long ta = block_reduce_sum(acc, s_warp);
  const unsigned long long tc = block_reduce_sum(cntacc, s_warp);
  if (threadIdx.x == 0) {
    atomicAdd(&op->aux0, ta);
    atomicAdd(&op->aux1, tc);
  }
}

// stats(): adjacency blocks of alive vertices + max degree
__global__ void stats_kernel(GraphView g, OpState* op) {
  __shared__ unsigned long long s_warp[32];
  unsigned long long blocks = 0;
  uint32_t mx = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.size;
       v += gridDim.x * blockDim.x) {
    if (bit_test(g.alive, v)) {
      const uint32_t d = g.deg[v];
      blocks += ceil_div(d, g.B);
      mx = max(mx, d);
    }
  }
  const unsigned long long t = block_reduce_sum(blocks, s_warp);
  if (threadIdx.x == 0 && t) atomicAdd(&op->aux0, t);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, d));
  if (lane_id() == 0 && mx) atomicMax(&op->aux1, (unsigned long long)mx);
}

// ---------------------------------------------------------------------------
// input-side helpers
// ---------------------------------------------------------------------------
// Counter-based R-MAT: edge i is a pure function of (seed, i).  The host twin
// lives in oracle/rmat.h and paper_2306_08252_b200/rmat.py.
__host__ __device__ inline unsigned long long rmat_mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ inline void rmat_edge(uint32_t scale, unsigned long long seed,
                                          unsigned long long idx, uint32_t ta, uint32_t tab,
                                          uint32_t tabc, uint32_t* src, uint32_t* dst) {
  const unsigned long long base = rmat_mix64(seed ^ (idx * 0xD1342543DE82EF95ull));
  uint32_t s = 0, d = 0;
  for (uint32_t level = 0; level < scale; level += 2) {
    const unsigned long long hsh = rmat_mix64(base + (unsigned long long)(level >> 1) * 0x9E3779B97F4A7C15ull);
    uint32_t r = (uint32_t)hsh;
    for (int half = 0; half < 2 && level + half < scale; ++half) {
      const uint32_t sb = r >= tab ? 1u : 0u;                       // quadrants c, d
      const uint32_t db = (r >= ta && r < tab) || r >= tabc ? 1u : 0u;  // quadrants b, d
      s = (s << 1) | sb;
      d = (d << 1) | db;
      r = (uint32_t)(hsh >> 32);
    }
  }
  *src = s;
  *dst = d;
}

__global__ void rmat_kernel(uint32_t scale, unsigned long long seed, unsigned long long first,
                            unsigned long long n, uint32_t ta, uint32_t tab, uint32_t tabc,
                            uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    rmat_edge(scale, seed, first + i, ta, tab, tabc, &src[i], &dst[i]);
}

// sorted-by-source keys -> CSR offsets over [0, vertex_count]
__global__ void keys_to_offsets_kernel(const unsigned long long* __restrict__ keys, uint32_t n,
                                       unsigned long long vertex_count,
                                       unsigned long long* __restrict__ offsets,
                                       uint32_t* __restrict__ dsts, const OpState* op) {
  if (op->err) return;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
    const unsigned long long cur = (i < n) ? (keys[i] >> 32) : vertex_count;
    const unsigned long long prev = (i == 0) ? 0ull : (keys[i - 1] >> 32) + 1ull;
    // every vertex in [prev, cur] starts at i (prev..cur-1 are empty, cur starts here)
    for (unsigned long long v = prev; v <= cur; ++v) offsets[v] = i;
    if (i < n) dsts[i] = (uint32_t)keys[i];
  }
}

// bijection on [0, 2^bits): owner = perm mod world, local id = perm / world
__host__ __device__ inline uint32_t owner_mask(uint32_t bits) {
  return bits >= 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
}
__host__ __device__ inline uint32_t owner_perm(uint32_t v, uint32_t bits) {
  if (bits == 0) return v;
  const uint32_t mask = owner_mask(bits);
  const uint32_t sh = (bits + 1) / 2;  // 2*sh >= bits: each xorshift is an involution
  uint32_t x = v & mask;
  x = (x * 0x9E3779B1u) & mask;
  x ^= x >> sh;
  x = (x * 0x85EBCA6Bu) & mask;
  x ^= x >> sh;
  return x;
}
__host__ __device__ inline uint32_t mul_inverse_u32(uint32_t a) {  // a odd
  uint32_t x = a;
  for (int i = 0; i < 5; ++i) x *= 2u - a * x;
  return x;
}
__host__ __device__ inline uint32_t owner_perm_inv(uint32_t p, uint32_t bits) {
  if (bits == 0) return p;
  const uint32_t mask = owner_mask(bits);
  const uint32_t sh = (bits + 1) / 2;
  uint32_t x = p & mask;
  x ^= x >> sh;
  x = (x * mul_inverse_u32(0x85EBCA6Bu)) & mask;
  x ^= x >> sh;
  x = (x * mul_inverse_u32(0x9E3779B1u)) & mask;
  return x;
}

// K11 send side: key = owner<<32 | input position (sorted stably by owner afterwards)
__global__ void route_keys_kernel(const uint32_t* __restrict__ src, uint32_t n, uint32_t world,
                                  uint32_t bits, uint32_t vertex_count,
                                  unsigned long long* __restrict__ keys, OpState* op) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t s = src[i];
    if (s >= vertex_count) set_error(op, 2, kErrSrcRange, i);
    const uint32_t owner = owner_perm(s, bits) % world;
    keys[i] = ((unsigned long long)owner << 32) | i;
  }
}

__global__ void route_gather_kernel(const unsigned long long* __restrict__ keys,
                                    const uint32_t* __restrict__ src,
                                    const uint32_t* __restrict__ dst, uint32_t n, uint32_t world,
                                    uint32_t bits, uint32_t* __restrict__ out_src_local,
                                    uint32_t* __restrict__ out_dst, uint32_t* __restrict__ out_index,
                                    unsigned long long* __restrict__ counts, const OpState* op) {
  if (op->err) return;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const unsigned long long k = keys[j];
    const uint32_t i = (uint32_t)k;
    const uint32_t owner = (uint32_t)(k >> 32);
    out_src_local[j] = owner_perm(src[i], bits) / world;
    out_dst[j] = dst[i];
    out_index[j] = i;
    // bucket boundaries: the last element of each owner's run records the run end
    const uint32_t next_owner = (j + 1 < n) ? (uint32_t)(keys[j + 1] >> 32) : world;
    for (uint32_t w = owner; w < next_owner; ++w) counts[w + 1] = j + 1;  // exclusive ends
    if (j == 0) for (uint32_t w = 0; w <= owner; ++w) counts[w] = 0;       // starts up to the first owner
  }
}

// ---------------------------------------------------------------------------
// K11, fused: owner computation + exchange over peer memory.  The receive
// buffers of every rank are mapped into this process (CUDA IPC over NVLink);
// a warp groups its 32 pairs by owner (__match_any_sync), the group leader
// reserves slots with ONE system-scope atomicAdd on the owner's cursor, and
// the lanes store their records straight into the owner's buffers.
// ---------------------------------------------------------------------------
constexpr int kMaxPeers = 16;
// Round words of one rank (first 256 bytes of its exchange allocation).  Two buffer sets alternate between
// rounds: a peer can run at most one round ahead (it cannot finish round e before this rank has ARRIVED in
// round e, which in stream order follows this rank's consumption of round e - 1), so set e & 1 is free again
// when round e + 2 starts.  Counters are only ever ADDED to by peers and reset by their owner.
//   cursor      entries pushed into the set (system-scope atomicAdd by the pushing warps)
//   arrive      [7:0] ranks whose push has landed, [15:8] of them with a data error, [23:16] with an engine error
//   agree       the same encoding, for the validation / plan status of the local op (batch atomicity across
//               ranks, graph.hpp:168-171: nobody mutates unless every rank validated)
//   ans_arrive  ranks whose query answers have landed
struct RoundWords {
  unsigned long long cursor[2];
  unsigned int arrive[2];
  unsigned int agree[2];
  unsigned int ans_arrive[2];
};
struct PeerBuffers {
  RoundWords* words[kMaxPeers];
  uint32_t* src[kMaxPeers][2];
  uint32_t* dst[kMaxPeers][2];
  uint32_t* idx[kMaxPeers][2];
  uint32_t* from[kMaxPeers][2];
  uint8_t* ans[kMaxPeers][2];
  unsigned long long capacity;
  uint32_t world, rank;
};
__device__ __forceinline__ unsigned int status_bits(uint32_t err) {
  return 1u | (err == 2u ? 1u << 8 : 0u) | (err >= 3u ? 1u << 16 : 0u);
}
__device__ __forceinline__ uint32_t status_agreed(unsigned int v) {
  return ((v >> 16) & 0xFFu) ? 3u : (((v >> 8) & 0xFFu) ? 2u : 0u);
}
__device__ __forceinline__ unsigned int ld_acquire_sys_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// spins until every rank has added to *word (or ~4 s have passed); returns the counter, resets it
__device__ __forceinline__ unsigned int wait_all_ranks(unsigned int* word, uint32_t world, bool* timed_out) {
  const long long t0 = clock64();
  unsigned int v = ld_acquire_sys_u32(word);
  *timed_out = false;
  while ((v & 0xFFu) < world) {
    if (clock64() - t0 > 8000000000ll) {
      *timed_out = true;
      break;
    }
    __nanosleep(200);
    v = ld_acquire_sys_u32(word);
  }
  *word = 0u;
  return v;
}

__global__ void __launch_bounds__(256)
exchange_validate_kernel(const uint32_t* __restrict__ src, uint32_t n, uint32_t vertex_count, OpState* op) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (src[i] >= vertex_count) set_error(op, 2, kErrSrcRange, i);
}

__global__ void __launch_bounds__(256)
exchange_push_kernel(PeerBuffers pb, int set, const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                     uint32_t n, uint32_t bits, OpState* op) {
  if (op->err) return;  // a rejected batch pushes nothing
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t npad = (n + 31u) & ~31u;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += gridDim.x * blockDim.x) {
    const bool valid = i < n;
    uint32_t owner = 0xFFFFFFFFu, local = 0, d = 0;
    if (valid) {
      const uint32_t p = owner_perm(src[i], bits);
      owner = p % pb.world;
      local = p / pb.world;
      d = dst[i];
    }
    const unsigned peers = __match_any_sync(kFull, owner);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (valid && lane == leader) base = atomicAdd_system(&pb.words[owner]->cursor[set], (unsigned long long)__popc(peers));
    base = __shfl_sync(kFull, base, leader);
    if (valid) {
      const unsigned long long pos = base + __popc(peers & lt);
      if (pos < pb.capacity) {
        pb.src[owner][set][pos] = local;
        pb.dst[owner][set][pos] = d;
        pb.idx[owner][set][pos] = i;
        pb.from[owner][set][pos] = pb.rank;
      } else {
        set_error(op, 3, kErrScratch, i);  // receive buffer of `owner` is full
      }
    }
  }
}

// After the push (or the answers) of this rank: tell every rank that it has landed.  The fence makes the
// stores of the preceding kernel visible system-wide before the counters move (fences are cumulative).
// which: 0 arrive (carries this rank's routing status), 2 ans_arrive
__global__ void exchange_signal_kernel(PeerBuffers pb, int set, int which, const OpState* op) {
  __threadfence_system();
  const uint32_t p = threadIdx.x;
  if (p < pb.world) {
    unsigned int* w = which == 0 ? &pb.words[p]->arrive[set] : &pb.words[p]->ans_arrive[set];
    atomicAdd_system(w, which == 0 ? status_bits(op->err) : 1u);
  }
}

// Waits until every rank has arrived in this rank's set.  which 0: op->aux0 = agreed routing status,
// op->aux1 = entries received; which 2: answers.
__global__ void exchange_wait_kernel(PeerBuffers pb, int set, int which, OpState* op) {
  if (threadIdx.x != 0) return;
  RoundWords* own = pb.words[pb.rank];
  bool timed_out;
  const unsigned int v = wait_all_ranks(which == 0 ? &own->arrive[set] : &own->ans_arrive[set], pb.world, &timed_out);
  __threadfence_system();
  if (which == 0) {
    op->aux0 = timed_out ? 3u : status_agreed(v);
    op->aux1 = own->cursor[set];
  } else {
    op->aux0 = timed_out ? 3u : 0u;
  }
}

// Batch atomicity across ranks: posts this rank's validation / plan status to every rank, waits for all of
// them, and only an all-clear lets the op's mutating kernels run (they start with `if (op->err) return`).
// An insert's queue front / live-edge count are committed here instead of in the plan's last tile.
__global__ void exchange_agree_kernel(PeerBuffers pb, int set, OpState* op, DeviceState* st, int commit_insert) {
  const uint32_t p = threadIdx.x;
  const uint32_t mine = op->err;
  __threadfence_system();
  if (p < pb.world) atomicAdd_system(&pb.words[p]->agree[set], status_bits(mine));
  if (p != 0) return;
  bool timed_out;
  const unsigned int v = wait_all_ranks(&pb.words[pb.rank]->agree[set], pb.world, &timed_out);
  const uint32_t agreed = timed_out ? 3u : status_agreed(v);
  op->aux0 = agreed;
  if (agreed != 0 && mine == 0) {
    op->err_detail = kErrPeer;
    op->err_index = 0;
    __threadfence();
    op->err = agreed;
  }
  if (agreed == 0 && commit_insert) {
    st->front += op->total_need;          // commit_front (block_pool.hpp:162-166)
    st->active_edges += op->n_edges;      // graph.hpp:186
  }
}

__global__ void __launch_bounds__(256)
exchange_answers_kernel(PeerBuffers pb, int set, const uint8_t* __restrict__ answers, const uint32_t* __restrict__ idx,
                        const uint32_t* __restrict__ from, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    pb.ans[from[i]][set][idx[i]] = answers[i];
}

// dg_digest over GLOBAL source ids for a shard of the source-partitioned store: local id l of rank r is
// vertex perm_inv(l * world + r), so the sum over ranks equals the single-GPU digest of the same multiset.
__global__ void __launch_bounds__(256)
digest_global_kernel(GraphView g, const uint32_t* __restrict__ wl_off, const uint32_t* __restrict__ wl_handle,
                     const uint32_t* __restrict__ wl_run, const uint32_t* __restrict__ run_deg, uint32_t rank, uint32_t world,
                     uint32_t bits, OpState* op) {
  __shared__ unsigned long long s_warp[8];
  const uint32_t W = (uint32_t)op->wl_blocks;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  unsigned long long acc = 0, cntacc = 0;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < W; w += nwarps) {
    const uint32_t v = wl_run[w] & kRunMask;
    const unsigned long long gv = owner_perm_inv(v * world + rank, bits);
    const uint32_t h = wl_handle[w];
    const uint32_t k = w - wl_off[v];
    const uint32_t cnt = min(g.B, run_deg[v] - k * g.B);
    const uint32_t* blk = g.slab + (unsigned long long)h * g.B;
    for (uint32_t s = lane; s < cnt; s += 32) {
      acc += mix64((gv << 32) | blk[s]);
      ++cntacc;
    }
  }
  const unsigned long long ta = block_reduce_sum(acc, s_warp);
  const unsigned long long tc = block_reduce_sum(cntacc, s_warp);
  if (threadIdx.x == 0) {
    atomicAdd(&op->aux0, ta);
    atomicAdd(&op->aux1, tc);
  }
}

}  // namespace dg
