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
  uint32_t B;
  uint32_t size;       // logical size at launch
  uint32_t dst_limit;  // destinations must be < dst_limit (== size single-GPU)
  int reclaim;
  DeviceState* st;
};

struct BatchView {
  const unsigned long long* keys;  // sorted (src<<32|dst), or nullptr on the CSR path
  const uint32_t* dsts;            // CSR path values, or nullptr
  const uint32_t* run_src;         // nullptr => run r is vertex r
  const uint32_t* run_start;       // [T + 1]
};

__device__ __forceinline__ uint32_t batch_value(const BatchView& b, uint32_t i) {
  return b.keys ? (uint32_t)b.keys[i] : b.dsts[i];
}
__device__ __forceinline__ uint32_t batch_src(const BatchView& b, uint32_t r) {
  return b.run_src ? b.run_src[r] : r;
}
__device__ __forceinline__ uint32_t ceil_div(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

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

// ---------------------------------------------------------------------------
// init
// ---------------------------------------------------------------------------
// block_pool.hpp:242-247 pushes one handle per block; here one coalesced store.
__global__ void ring_fill_kernel(uint32_t* __restrict__ ring, unsigned long long nb) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (unsigned long long)gridDim.x * blockDim.x)
    ring[i] = (uint32_t)i;
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
template <int kMode, bool kWithIndex>
__global__ void pack_coo_kernel(GraphView g, const uint32_t* __restrict__ src,
                                const uint32_t* __restrict__ dst, uint32_t n,
                                unsigned long long* __restrict__ keys,
                                uint32_t* __restrict__ index, OpState* op) {
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
    keys[i] = ((unsigned long long)s << 32) | d;
    if (kWithIndex) index[i] = i;
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
// insert: plan (graph.hpp:135-160) as a scan over touched sources
// ---------------------------------------------------------------------------
// Packed scan value: [61:31] append units, [30:0] fresh blocks.
constexpr int kPackShift = 31;
constexpr unsigned long long kPackLoMask = (1ull << kPackShift) - 1ull;

struct PlanIn {
  GraphView g;
  BatchView b;
  uint32_t* run_deg;
  uint32_t* run_tail;
  __device__ unsigned long long operator()(unsigned long long r64) const {
    const uint32_t r = (uint32_t)r64;
    const uint32_t v = batch_src(b, r);
    const uint32_t c = b.run_start[r + 1] - b.run_start[r];
    const uint32_t d = g.deg[v];
    run_deg[r] = d;
    run_tail[r] = g.tail[v];
    if (c == 0) return 0ull;
    // space left in the tail block == block_size - last_insert_offset (graph.hpp:149-150)
    const uint32_t nb = ceil_div(d, g.B);
    const uint32_t space = nb * g.B - d;
    const uint32_t fill = min(c, space);
    const uint32_t need = ceil_div(c - fill, g.B);  // graph.hpp:152-153
    const uint32_t units = need + (fill > 0 ? 1u : 0u);
    return ((unsigned long long)units << kPackShift) | need;
  }
};
struct PlanOut {
  uint32_t* unit_off;
  uint32_t* blk_off;
  __device__ void operator()(unsigned long long r, unsigned long long excl,
                             unsigned long long) const {
    unit_off[r] = (uint32_t)(excl >> kPackShift);
    blk_off[r] = (uint32_t)(excl & kPackLoMask);
  }
};
struct PlanFin {
  GraphView g;
  uint32_t* unit_off;
  OpState* op;
  unsigned long long n_edges;
  __device__ void operator()(unsigned long long total) const {
    const unsigned long long need = total & kPackLoMask;
    const unsigned long long units = total >> kPackShift;
    unit_off[op->n_runs] = (uint32_t)units;
    op->n_units = units;
    op->total_need = need;
    DeviceState* st = g.st;
    // ensure_available (block_pool.hpp:177-189): fail BEFORE any mutation
    if (need > st->rear - st->front) {
      op->err = 3;
      op->err_detail = kErrPoolUnderflow;
      op->err_index = need - (st->rear - st->front);
      return;
    }
    op->front_old = st->front;
    st->front += need;              // commit_front (block_pool.hpp:162-166)
    st->active_edges += n_edges;    // graph.hpp:186
  }
};

// ---------------------------------------------------------------------------
// insert: append (graph.hpp:333-372) — one warp per unit, a unit being either
// the free tail of a source's last block or one fresh block.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
append_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ unit_off,
              const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ run_deg,
              const uint32_t* __restrict__ run_tail, const OpState* op) {
  if (op->err) return;
  const uint32_t T = (uint32_t)op->n_runs;
  const uint32_t U = (uint32_t)op->n_units;
  const unsigned long long front_old = op->front_old;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < U; u += nwarps) {
    const uint32_t r = warp_find_run(unit_off, T, u);
    const uint32_t j = u - unit_off[r];
    const uint32_t v = batch_src(b, r);
    const uint32_t rs = b.run_start[r];
    const uint32_t c = b.run_start[r + 1] - rs;
    const uint32_t d = run_deg[r];
    const uint32_t nb_old = ceil_div(d, g.B);
    const uint32_t space = nb_old * g.B - d;
    const uint32_t fill = min(c, space);
    const uint32_t has_fill = fill > 0 ? 1u : 0u;
    const uint32_t need = ceil_div(c - fill, g.B);
    uint32_t blk, off0, src0, cnt;
    if (has_fill && j == 0) {
      blk = run_tail[r];                 // resume at the last-insert position (graph.hpp:344-349)
      off0 = d - (nb_old - 1) * g.B;
      src0 = rs;
      cnt = fill;
    } else {
      const uint32_t f = j - has_fill;
      const unsigned long long pos = front_old + blk_off[r] + f;  // pop_range (block_pool.hpp:148-158)
      blk = g.ring[pos % g.ring_cap];
      off0 = 0;
      src0 = rs + fill + f * g.B;
      cnt = min(g.B, c - fill - f * g.B);
      if (lane == 0) {
        const uint32_t prev = (f == 0) ? (nb_old > 0 ? run_tail[r] : kNull)
                                       : g.ring[(pos - 1) % g.ring_cap];
        if (prev == kNull) g.head[v] = blk; else g.next[prev] = blk;
        if (f == need - 1) {
          g.next[blk] = kNull;
          g.tail[v] = blk;
        }
      }
    }
    uint32_t* out = g.slab + (unsigned long long)blk * g.B + off0;
    for (uint32_t s = lane; s < cnt; s += 32) out[s] = batch_value(b, src0 + s);
    if (lane == 0 && j == need + has_fill - 1) g.deg[v] = d + c;
  }
}

// ---------------------------------------------------------------------------
// chain enumeration: touched sources -> flat list of their blocks
// ---------------------------------------------------------------------------
struct EnumIn {
  GraphView g;
  BatchView b;
  uint32_t* run_deg;
  int check_alive;  // delete/query skip dead or unknown sources (graph.hpp:205, :229)
  __device__ unsigned long long operator()(unsigned long long r64) const {
    const uint32_t r = (uint32_t)r64;
    const uint32_t v = batch_src(b, r);
    uint32_t d = 0;
    if (v < g.size && (!check_alive || bit_test(g.alive, v))) d = g.deg[v];
    run_deg[r] = d;
    return ceil_div(d, g.B);
  }
};
struct EnumOut {
  uint32_t* wl_off;
  __device__ void operator()(unsigned long long r, unsigned long long excl,
                             unsigned long long) const {
    wl_off[r] = (uint32_t)excl;
  }
};
struct EnumFin {
  uint32_t* wl_off;
  OpState* op;
  unsigned long long wl_cap;
  __device__ void operator()(unsigned long long total) const {
    wl_off[op->n_runs] = (uint32_t)total;
    op->wl_blocks = total;
    if (total > wl_cap) {  // cannot happen: wl_cap >= blocks in use (host mirror)
      op->err = 3;
      op->err_detail = kErrScratch;
    }
  }
};

// One warp per source walks the chain.  Each round trip loads next[h..h+31]
// and confirms the longest prefix with next[h+i] == h+i+1, i.e. a run of
// physically consecutive blocks that really are consecutive in the chain —
// bulk-built hubs advance 32 blocks per memory latency, fragmented chains
// degrade to one block per latency.
__global__ void __launch_bounds__(256)
enumerate_walk_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                      uint32_t* __restrict__ wl_handle, uint32_t* __restrict__ wl_run,
                      const OpState* op) {
  if (op->err) return;
  const uint32_t T = (uint32_t)op->n_runs;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < T; r += nwarps) {
    const uint32_t base = wl_off[r];
    const uint32_t nblk = wl_off[r + 1] - base;
    if (nblk == 0) continue;
    const uint32_t v = batch_src(b, r);
    uint32_t h = g.head[v];
    uint32_t k = 0;
    while (k < nblk) {
      const unsigned long long hh = (unsigned long long)h + lane;
      const uint32_t nx = (hh < g.ring_cap) ? g.next[hh] : kNull;
      const bool ok = (unsigned long long)nx == hh + 1;
      const unsigned m = __ballot_sync(kFull, ok);
      uint32_t len = (m == kFull) ? 32u : (uint32_t)__ffs(~m);
      len = min(len, nblk - k);
      if ((uint32_t)lane < len) {
        wl_handle[base + k + lane] = (uint32_t)hh;
        wl_run[base + k + lane] = r;
      }
      h = __shfl_sync(kFull, nx, len - 1);
      k += len;
    }
  }
}

// ---------------------------------------------------------------------------
// delete: match + tombstone (graph.hpp:376-394) / query: match (graph.hpp:228-241)
// one warp per edge block of a touched chain; the source's targets are a
// dst-sorted slice of the batch, searched by binary search.
// ---------------------------------------------------------------------------
template <bool kIsDelete>
__global__ void __launch_bounds__(256)
match_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
             const uint32_t* __restrict__ wl_handle, const uint32_t* __restrict__ wl_run,
             const uint32_t* __restrict__ run_deg, uint32_t* __restrict__ run_matched,
             uint8_t* __restrict__ hit, OpState* op) {
  if (op->err) return;
  __shared__ unsigned long long s_warp[8];
  const uint32_t W = (uint32_t)op->wl_blocks;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  unsigned long long slots = 0;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < W; w += nwarps) {
    const uint32_t r = wl_run[w];
    const uint32_t h = wl_handle[w];
    const uint32_t k = w - wl_off[r];
    const uint32_t d = run_deg[r];
    const uint32_t rs = b.run_start[r], re = b.run_start[r + 1];
    const uint32_t cnt = min(g.B, d - k * g.B);
    uint32_t* blk = g.slab + (unsigned long long)h * g.B;
    uint32_t matched = 0;
    for (uint32_t s0 = 0; s0 < cnt; s0 += 32) {
      const uint32_t s = s0 + lane;
      const bool valid = s < cnt;
      bool found = false;
      if (valid) {
        const uint32_t e = blk[s];
        const uint32_t lb = lower_bound_lo32(b.keys, rs, re, e);
        found = lb < re && (uint32_t)b.keys[lb] == e;
        if (found) {
          if (kIsDelete) {
            blk[s] = kTomb;
          } else {
            for (uint32_t j = lb; j < re && (uint32_t)b.keys[j] == e; ++j) hit[j] = 1;
          }
        }
      }
      if (kIsDelete) matched += __popc(__ballot_sync(kFull, found));
    }
    if (kIsDelete && lane == 0 && matched) atomicAdd(&run_matched[r], matched);
    if (lane == 0) slots += cnt;
  }
  const unsigned long long t = block_reduce_sum(slots, s_warp);
  if (threadIdx.x == 0 && t) atomicAdd(&op->slots, t);
}

// ---------------------------------------------------------------------------
// delete: compaction plan — per source, moves <= min(matched, new degree)
// ---------------------------------------------------------------------------
struct MovesIn {
  const uint32_t* run_deg;
  const uint32_t* run_matched;
  __device__ unsigned long long operator()(unsigned long long r) const {
    const uint32_t m = run_matched[r];
    const uint32_t nd = run_deg[r] - m;
    return min(m, nd);
  }
};
struct MovesOut {
  uint32_t* mv_off;
  __device__ void operator()(unsigned long long r, unsigned long long excl,
                             unsigned long long) const {
    mv_off[r] = (uint32_t)excl;
  }
};
struct MovesFin {
  uint32_t* mv_off;
  OpState* op;
  unsigned long long mv_cap;
  __device__ void operator()(unsigned long long total) const {
    mv_off[op->n_runs] = (uint32_t)total;
    op->aux0 = total;                      // scratch entries needed
    op->aux1 = total > mv_cap ? 1ull : 0ull;  // host grows the scratch and re-runs the tail
  }
};

// delete: classify — holes below the new degree and survivors at/after it get
// tickets from per-source counters (warp-aggregated); blocks past the new
// tail are pushed to the ring rear (block_pool.hpp:192-209, warp-aggregated
// across the CTA's freed blocks).
__global__ void __launch_bounds__(256)
classify_kernel(GraphView g, const uint32_t* __restrict__ wl_off,
                const uint32_t* __restrict__ wl_handle, const uint32_t* __restrict__ wl_run,
                const uint32_t* __restrict__ run_deg, const uint32_t* __restrict__ run_matched,
                const uint32_t* __restrict__ mv_off, uint32_t* __restrict__ hole_cnt,
                uint32_t* __restrict__ surv_cnt, unsigned long long* __restrict__ hole_addr,
                uint32_t* __restrict__ moved_val, OpState* op) {
  if (op->err || op->aux1) return;
  __shared__ unsigned long long s_warp[8];
  const uint32_t W = (uint32_t)op->wl_blocks;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long pushed = 0;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < W; w += nwarps) {
    const uint32_t r = wl_run[w];
    const uint32_t m = run_matched[r];
    if (m == 0) continue;
    const uint32_t h = wl_handle[w];
    const uint32_t k = w - wl_off[r];
    const uint32_t d = run_deg[r];
    const uint32_t nd = d - m;
    const uint32_t new_nb = ceil_div(nd, g.B);
    const uint32_t cnt = min(g.B, d - k * g.B);
    const uint32_t mo = mv_off[r];
    const uint32_t* blk = g.slab + (unsigned long long)h * g.B;
    for (uint32_t s0 = 0; s0 < cnt; s0 += 32) {
      const uint32_t s = s0 + lane;
      const bool valid = s < cnt;
      const uint32_t e = valid ? blk[s] : 0u;
      const uint32_t p = k * g.B + s;
      const bool is_hole = valid && p < nd && e == kTomb;
      const bool is_surv = valid && p >= nd && e != kTomb;
      const unsigned mh = __ballot_sync(kFull, is_hole);
      const unsigned ms = __ballot_sync(kFull, is_surv);
      if (mh) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&hole_cnt[r], (uint32_t)__popc(mh));
        base = __shfl_sync(kFull, base, 0);
        if (is_hole) hole_addr[mo + base + __popc(mh & lt)] = (unsigned long long)h * g.B + s;
      }
      if (ms) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&surv_cnt[r], (uint32_t)__popc(ms));
        base = __shfl_sync(kFull, base, 0);
        if (is_surv) moved_val[mo + base + __popc(ms & lt)] = e;
      }
    }
    if (k >= new_nb && g.reclaim) {
      if (lane == 0) {
        const unsigned long long pos = atomicAdd(&g.st->rear, 1ull);
        g.ring[pos % g.ring_cap] = h;
        ++pushed;
      }
    }
  }
  const unsigned long long t = block_reduce_sum(pushed, s_warp);
  if (threadIdx.x == 0 && t) atomicAdd(&op->pushed, t);
}

// delete: fill holes with the tail survivors, repair degree / tail / head
// (detach_empty_tail, graph.hpp:398-414).  One warp per touched source.
__global__ void __launch_bounds__(256)
finalize_delete_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ wl_off,
                       const uint32_t* __restrict__ wl_handle,
                       const uint32_t* __restrict__ run_deg,
                       const uint32_t* __restrict__ run_matched,
                       const uint32_t* __restrict__ mv_off, const uint32_t* __restrict__ hole_cnt,
                       const unsigned long long* __restrict__ hole_addr,
                       const uint32_t* __restrict__ moved_val, OpState* op) {
  if (op->err || op->aux1) return;
  __shared__ unsigned long long s_warp[8];
  const uint32_t T = (uint32_t)op->n_runs;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  unsigned long long matched = 0, moves = 0;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < T; r += nwarps) {
    const uint32_t m = run_matched[r];
    if (m == 0) continue;
    const uint32_t v = batch_src(b, r);
    const uint32_t nd = run_deg[r] - m;
    const uint32_t mv = hole_cnt[r];
    const uint32_t mo = mv_off[r];
    for (uint32_t i = lane; i < mv; i += 32) g.slab[hole_addr[mo + i]] = moved_val[mo + i];
    if (lane == 0) {
      g.deg[v] = nd;
      if (nd == 0) {
        g.head[v] = kNull;
        g.tail[v] = kNull;
      } else {
        const uint32_t t = wl_handle[wl_off[r] + ceil_div(nd, g.B) - 1];
        g.tail[v] = t;
        g.next[t] = kNull;
      }
      matched += m;
      moves += mv;
    }
  }
  const unsigned long long tm = block_reduce_sum(matched, s_warp);
  const unsigned long long tv = block_reduce_sum(moves, s_warp);
  if (threadIdx.x == 0) {
    if (tm) {
      atomicAdd(&op->matched, tm);
      atomicAdd(&g.st->active_edges, (unsigned long long)(-(long long)tm));  // graph.hpp:211-213
    }
    if (tv) atomicAdd(&op->moves, tv);
  }
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
    const uint32_t v = wl_run[w];  // runs are vertices on the export path
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
    const uint32_t v = wl_run[w];
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

}  // namespace dg
