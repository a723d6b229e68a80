// dg_device.cuh — device-side building blocks for libdyngraph_b200 (sm_100a).
//
//  * status words shared between kernels of one op (validate-then-mutate
//    without a host round trip: every mutating kernel starts with
//    `if (op->err) return;`),
//  * a single-pass decoupled-look-back prefix scan with pluggable input /
//    output functors (used for run detection, batch planning, work-list
//    offsets, degree -> CSR offsets),
//  * a hand-written Onesweep-style LSD radix sort for 64-bit keys with an
//    optional 32-bit payload (8-bit digits, one histogram pass, one
//    scatter pass per digit with decoupled look-back across tiles).
//
// Nothing here is a port of reference code: the CPU reference has no device
// code at all (kernel inventory).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dg {

constexpr uint32_t kNull = 0xFFFFFFFFu;   // reference: types.hpp:16-17
constexpr uint32_t kTomb = 0xFFFFFFFFu;   // in-slot tombstone; never a valid id
constexpr int kWarp = 32;
constexpr unsigned kFull = 0xFFFFFFFFu;

// ---- error detail codes (op->err_detail) --------------------------------
enum ErrDetail : uint32_t {
  kErrNone = 0,
  kErrSrcRange = 1,       // source id >= logical size
  kErrDstRange = 2,       // csr.hpp:67-72
  kErrDeadSource = 3,     // graph.hpp:322-327
  kErrOffsetsStart = 4,   // csr.hpp:54-56
  kErrOffsetsMonotone = 5,// csr.hpp:57-61
  kErrOffsetsEnd = 6,     // csr.hpp:62-66
  kErrPoolUnderflow = 7,  // block_pool.hpp:177-189
  kErrScratch = 8,        // internal: a work list did not fit its bound (cannot happen: bounds come from the blocks in use)
  kErrPeer = 9,           // sharded store: the batch was rejected on another rank (or a peer never arrived)
  kErrSkipped = 10,       // submitted behind an op that failed: not applied (the failed op reports first, graph.hpp:168-171)
};

// Persistent device-resident scalars of one graph (the queue cursors use the
// reference's unwrapped 64-bit coordinates, block_pool.hpp:31-34).
struct DeviceState {
  unsigned long long front;         // next queue position to serve
  unsigned long long rear;          // one past the last pushed handle
  unsigned long long active_edges;  // graph.hpp:100
  unsigned long long poison;        // != 0: a submitted op failed and has not been reported yet — ops queued behind it do not run
};

// Transient per-op words; zeroed by the host before every op.
struct OpState {
  uint32_t err;            // 0 / DG_ERR_DATA / DG_ERR_ENGINE
  uint32_t err_detail;
  unsigned long long err_index;   // smallest offending index (atomicMin)
  unsigned long long n_runs;      // T
  unsigned long long n_units;     // append work units
  unsigned long long total_need;  // fresh blocks this batch pops
  unsigned long long front_old;   // queue front before the pop
  unsigned long long wl_blocks;   // blocks in touched chains (delete/query/export)
  unsigned long long slots;       // slots in touched chains
  unsigned long long matched;     // delete: entries removed; query: hits
  unsigned long long moves;       // compaction moves (bound, then exact)
  unsigned long long pushed;      // blocks returned to the ring
  unsigned long long aux0;        // op-specific
  unsigned long long aux1;
  unsigned long long n_input;     // device-resident copy of the input length (scan bound)
  unsigned long long n_items;     // CTA work items of the long-chain match path
  unsigned long long n_edges;     // entries an insert commits to active_edges
  unsigned long long slots_long;  // part of `slots` inspected by the long-chain (shared-memory table) path
  unsigned long long n_big;       // chains walked by a whole warp (enumerate_big_kernel)
  unsigned long long n_med;       // warp work items of the medium match tier
  unsigned long long n_aux;       // second device-resident scan bound (vertex count of the counting group-by)
  unsigned int med_cursor;        // dynamic work distribution of the medium / long match tiers
  unsigned int long_cursor;
  unsigned long long slots_tiny;  // part of `slots` inspected by the register-compare tier
  unsigned int n_huge;            // chains walked by a whole CTA (listed from the end of the big list)
  unsigned int committed;         // CSR insert: the append pass ran and published deg/tail/front (rollback needed on error)
  unsigned long long bad_index;   // CSR insert: smallest out-of-range destination index seen by the append pass (~0: none)
  unsigned long long fused_blocks;  // blocks of the warp-owned sources (fused_delete_kernel); wl_blocks counts the rest
  unsigned long long slots_fused;   // part of `slots` inspected by fused_delete_kernel
  unsigned int n_fmed;              // sources of the fused medium class listed by the enumeration plan
  unsigned int scatter_ctas;        // CTAs of group_scatter_kernel that have finished (fused_delete_kernel starts beside it)
  unsigned long long hole_items;    // 2 x wl_blocks: items of the hole / survivor scan of the hub compaction (device-resident bound)
};

__device__ __forceinline__ void set_error(OpState* op, uint32_t code, uint32_t detail,
                                          unsigned long long index) {
  // Smallest index wins so the report is deterministic; the class of the
  // first reporter sticks (all data checks of one op share a class).
  atomicCAS(&op->err, 0u, code);
  atomicCAS(&op->err_detail, 0u, detail);
  atomicMin(&op->err_index, index);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool bit_test(const uint32_t* __restrict__ bits, uint32_t v) {
  return (bits[v >> 5] >> (v & 31)) & 1u;
}

// ===========================================================================
// Decoupled look-back scan
// ===========================================================================
// Tile status word: [63:62] flag, [61:0] value.
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kFlagMask = 3ull << 62;
constexpr unsigned long long kValMask = ~kFlagMask;

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// Scratch layout for one scan launch: [0] ticket counter, [1..] tile status.
__host__ __device__ inline size_t scan_scratch_words(uint64_t n_max) {
  return 2 + (n_max + kScanTile - 1) / kScanTile;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exclusive scan of In(i) over i in [0, *n_ptr).  Out(i, exclusive, value) is
// called for every element, Fin(total) once by the last tile.  Grid must
// cover ceil(n_bound / kScanTile) tiles where n_bound >= *n_ptr; surplus
// tiles exit.  `scratch` must be zeroed before the launch.
template <class In, class Out, class Fin>
__global__ void __launch_bounds__(kScanThreads)
scan_kernel(const unsigned long long* __restrict__ n_ptr, unsigned long long* scratch,
            const OpState* __restrict__ op_guard, In in, Out out, Fin fin) {
  if (op_guard != nullptr && op_guard->err != 0) return;
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  __shared__ unsigned long long s_tile_excl;
  __shared__ unsigned int s_tile;
  const unsigned long long n = *n_ptr;
  const unsigned long long num_tiles = (n + kScanTile - 1) / kScanTile;
  // (the grid is sized from a host-side bound: surplus CTAs leave before they take a ticket, so exactly num_tiles
  // CTAs — the first to be scheduled — draw tiles 0 .. num_tiles - 1 in the order they start)
  if (blockIdx.x >= num_tiles) return;
  if (threadIdx.x == 0) s_tile = atomicAdd(reinterpret_cast<unsigned int*>(scratch), 1u);
  __syncthreads();
  const unsigned int tile = s_tile;
  if (tile >= num_tiles) return;
  unsigned long long* status = scratch + 2;

  // blocked arrangement: thread t owns items [t*ITEMS, t*ITEMS+ITEMS)
  const unsigned long long base = (unsigned long long)tile * kScanTile +
                                  (unsigned long long)threadIdx.x * kScanItems;
  unsigned long long v[kScanItems];
  unsigned long long thread_sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const unsigned long long i = base + j;
    v[j] = (i < n) ? in(i) : 0ull;
    thread_sum += v[j];
  }
  // warp inclusive scan of thread sums
  unsigned long long incl = thread_sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    unsigned long long t = __shfl_up_sync(kFull, incl, d);
    if (lane_id() >= d) incl += t;
  }
  const int warp = threadIdx.x >> 5;
  if (lane_id() == 31) s_warp[warp] = incl;
  __syncthreads();
  unsigned long long warp_excl = 0, tile_sum = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    const unsigned long long s = s_warp[w];
    if (w < warp) warp_excl += s;
    tile_sum += s;
  }
  // publish + look back (thread 0 .. 31 of warp 0 cooperate)
  if (warp == 0) {
    unsigned long long excl = 0;
    if (tile == 0) {
      if (lane_id() == 0) st_volatile_u64(&status[0], kFlagPre | (tile_sum & kValMask));
    } else {
      if (lane_id() == 0) st_volatile_u64(&status[tile], kFlagAgg | (tile_sum & kValMask));
      long long look = (long long)tile - 1;
      while (true) {
        const long long idx = look - lane_id();
        unsigned long long w = (idx >= 0) ? ld_volatile_u64(&status[idx]) : kFlagPre;
        // wait until every polled predecessor published something
        while (__any_sync(kFull, (w & kFlagMask) == 0)) {
          w = (idx >= 0) ? ld_volatile_u64(&status[idx]) : kFlagPre;
        }
        const unsigned pre_mask = __ballot_sync(kFull, (w & kFlagMask) == kFlagPre);
        unsigned long long contrib;
        if (pre_mask) {
          const int first = __ffs(pre_mask) - 1;  // nearest predecessor with a full prefix
          contrib = (lane_id() <= first && idx >= 0) ? (w & kValMask) : 0ull;
        } else {
          contrib = w & kValMask;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) contrib += __shfl_xor_sync(kFull, contrib, d);
        excl += contrib;
        if (pre_mask) break;
        look -= 32;
      }
      if (lane_id() == 0)
        st_volatile_u64(&status[tile], kFlagPre | ((excl + tile_sum) & kValMask));
    }
    if (lane_id() == 0) s_tile_excl = excl;
  }
  __syncthreads();
  unsigned long long run = s_tile_excl + warp_excl + (incl - thread_sum);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const unsigned long long i = base + j;
    if (i < n) out(i, run, v[j]);
    run += v[j];
  }
  if (tile == num_tiles - 1 && threadIdx.x == kScanThreads - 1) fin(run);
}

// ===========================================================================
// Unordered range allocation ("atomic scan")
// ===========================================================================
// Most prefix sums of the batch ops only hand out DISJOINT RANGES (queue
// positions, work-list segments, scratch segments, group slots): order between
// tiles is irrelevant.  alloc_kernel keeps the exclusive scan inside a tile
// and replaces the look-back chain by one atomicAdd per tile and word on a
// global cursor, so tiles never wait for each other.  Two 64-bit words are
// scanned at once (callers pack two 32-bit quantities into each).
//   In(i)                         -> Sum2 (PURE loads; see scan_kernel)
//   Out(i, excl.a, excl.b, value) -> per element
//   Fin(total.a, total.b)         -> once, by the last tile to finish
// scratch: [0] cursor a, [1] cursor b, [2] finished tiles, [3] cursor c; zero at launch, zeroed again by the last tile
// (cursor c is read by nobody here: the op reads it from its own counter, see EnumFin).
struct Sum2 {
  unsigned long long a, b;
  unsigned int c = 0;        // a third, 32-bit quantity (its cursor is scratch[3]); most users leave it at 0
  unsigned int c_excl = 0;   // Out only: the element's exclusive prefix of c (handed over inside the value)
};
constexpr size_t kAllocScratchWords = 4;
constexpr int kAllocThreads = 256;
constexpr int kAllocItemsSmall = 4;    // batches: more tiles, shorter per-tile latency chain
constexpr int kAllocItemsLarge = 4;    // vertex-sized passes (16 items per thread measured 1.8x slower)

// In::Aux is a small per-element payload In fills next to the sums (values it
// already loaded) and Out receives back, so Out never re-loads them.  In must
// use predicated loads (`x = c ? p[i] : 0`), not branches: the kernel issues a
// thread's items back to back and a branch would serialise their latencies.
template <int kAllocItems, class In, class Out, class Fin>
__global__ void __launch_bounds__(kAllocThreads, kAllocItems <= 4 ? 4 : 2)
alloc_kernel(const unsigned long long* __restrict__ n_ptr, unsigned long long* scratch,
             const OpState* __restrict__ op_guard, In in, Out out, Fin fin) {
  if (op_guard != nullptr && op_guard->err != 0) return;
  constexpr int kAllocTile = kAllocThreads * kAllocItems;
  __shared__ Sum2 s_warp[kAllocThreads / 32];
  __shared__ Sum2 s_base;
  const unsigned long long n = *n_ptr;
  const unsigned long long num_tiles = (n + kAllocTile - 1) / kAllocTile;
  const unsigned int tile = blockIdx.x;
  if (tile >= num_tiles) {
    if (n == 0 && tile == 0 && threadIdx.x == 0) fin(0ull, 0ull, 0u);
    return;
  }
  const unsigned long long base = (unsigned long long)tile * kAllocTile +
                                  (unsigned long long)threadIdx.x * kAllocItems;
  Sum2 v[kAllocItems];
  typename In::Aux aux[kAllocItems];
  Sum2 thread_sum{0ull, 0ull};
#pragma unroll
  for (int j = 0; j < kAllocItems; ++j) {
    const unsigned long long i = base + j;
    v[j] = in(i < n ? i : n - 1, aux[j]);   // clamped index keeps the loads unconditional
    if (i >= n) v[j] = Sum2{0ull, 0ull};
    thread_sum.a += v[j].a;
    thread_sum.b += v[j].b;
    thread_sum.c += v[j].c;
  }
  Sum2 incl = thread_sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long ta = __shfl_up_sync(kFull, incl.a, d);
    const unsigned long long tb = __shfl_up_sync(kFull, incl.b, d);
    const unsigned int tc = __shfl_up_sync(kFull, incl.c, d);
    if (lane_id() >= d) {
      incl.a += ta;
      incl.b += tb;
      incl.c += tc;
    }
  }
  const int warp = threadIdx.x >> 5;
  if (lane_id() == 31) s_warp[warp] = incl;
  __syncthreads();
  Sum2 warp_excl{0ull, 0ull}, tile_sum{0ull, 0ull};
#pragma unroll
  for (int w = 0; w < kAllocThreads / 32; ++w) {
    const Sum2 sw = s_warp[w];
    if (w < warp) {
      warp_excl.a += sw.a;
      warp_excl.b += sw.b;
      warp_excl.c += sw.c;
    }
    tile_sum.a += sw.a;
    tile_sum.b += sw.b;
    tile_sum.c += sw.c;
  }
  if (threadIdx.x == 0) {
    Sum2 bs{0ull, 0ull};
    if (tile_sum.a) bs.a = atomicAdd(&scratch[0], tile_sum.a);
    if (tile_sum.b) bs.b = atomicAdd(&scratch[1], tile_sum.b);
    if (tile_sum.c) bs.c = (unsigned int)atomicAdd(&scratch[3], (unsigned long long)tile_sum.c);
    s_base = bs;
  }
  __syncthreads();
  Sum2 run{s_base.a + warp_excl.a + (incl.a - thread_sum.a), s_base.b + warp_excl.b + (incl.b - thread_sum.b),
           s_base.c + warp_excl.c + (incl.c - thread_sum.c)};
#pragma unroll
  for (int j = 0; j < kAllocItems; ++j) {
    const unsigned long long i = base + j;
    v[j].c_excl = run.c;
    if (i < n) out(i, run.a, run.b, v[j], aux[j]);
    run.a += v[j].a;
    run.b += v[j].b;
    run.c += v[j].c;
  }
  // (off the tile's critical path) the last tile to get here sees every tile's
  // contribution to the cursors: thread 0's cursor atomics precede its fence
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(&scratch[2], 1ull);
    if (done == num_tiles - 1) {
      __threadfence();
      const unsigned long long ta = ld_volatile_u64(&scratch[0]), tb = ld_volatile_u64(&scratch[1]);
      const unsigned long long tc = ld_volatile_u64(&scratch[3]);
      scratch[0] = 0ull;   // the cursors are handed back zeroed: the host keeps them in a persistent
      scratch[1] = 0ull;   // buffer and never clears them between ops
      scratch[2] = 0ull;
      scratch[3] = 0ull;
      fin(ta, tb, (unsigned int)tc);
    }
  }
}

// ===========================================================================
// Onesweep radix sort (u64 keys, optional u32 values)
// ===========================================================================
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys
constexpr int kRadix = 256;
constexpr int kMaxPasses = 8;

struct SortPlan {
  int passes;
  int shift[kMaxPasses];
  int bits[kMaxPasses];
};

__host__ __device__ inline size_t sort_tiles(uint64_t n) { return (n + kSortTile - 1) / kSortTile; }

// Accumulates one key into the per-pass shared histograms (layout [pass][256]).
__device__ __forceinline__ void hist_add(unsigned int* s_hist, const SortPlan& plan,
                                         unsigned long long k) {
#pragma unroll
  for (int p = 0; p < kMaxPasses; ++p) {
    if (p < plan.passes) {
      const unsigned d = (unsigned)(k >> plan.shift[p]) & ((1u << plan.bits[p]) - 1u);
      atomicAdd(&s_hist[p * kRadix + d], 1u);
    }
  }
}
__device__ __forceinline__ void hist_clear(unsigned int* s_hist, const SortPlan& plan) {
  for (int i = threadIdx.x; i < plan.passes * kRadix; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
}
__device__ __forceinline__ void hist_flush(const unsigned int* s_hist, const SortPlan& plan,
                                           unsigned int* __restrict__ hist) {
  __syncthreads();
  for (int i = threadIdx.x; i < plan.passes * kRadix; i += blockDim.x) {
    const unsigned c = s_hist[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// Global histogram of every pass in one read of the keys (RAW counts; each
// scatter pass turns its 256 counts into digit bases itself).
// hist layout: [pass][256] u32.  Producers that already stream the keys (the
// COO pack kernels) fold this into their own pass instead.
__global__ void __launch_bounds__(256)
sort_hist_kernel(const unsigned long long* __restrict__ keys, uint64_t n, SortPlan plan,
                 unsigned int* __restrict__ hist, const OpState* __restrict__ op_guard) {
  if (op_guard != nullptr && op_guard->err != 0) return;
  __shared__ unsigned int s_hist[kMaxPasses * kRadix];
  hist_clear(s_hist, plan);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    hist_add(s_hist, plan, keys[i]);
  hist_flush(s_hist, plan, hist);
}

// One scatter pass (Onesweep).  status: [0] ticket, then per tile 256 u64 words; zeroed before the
// launch.  digit_count: this pass's RAW histogram.
//   1. a tile's 4096 keys are loaded warp-striped (coalesced) and ranked inside their warp with
//      __match_any_sync (stable: order = warp, row, lane);
//   2. thread d owns digit d: offsets of the warps inside the digit, the tile's count, the digit's place
//      in the tile's sorted order (CTA scan over the 256 counts);  the count is published at once and the
//      decoupled look-back over the predecessors starts;
//   3. meanwhile the keys are laid out IN SHARED MEMORY in digit order, so that the write-out runs over
//      consecutive shared positions: consecutive threads hold consecutive keys of the same digit and store
//      to consecutive global addresses (full 32-byte sectors instead of one scattered 8-byte store per key).
// Dynamic shared memory: kSortTile keys (+ kSortTile values).
template <bool kHasValues>
__global__ void __launch_bounds__(kSortThreads, 2)
sort_pass_kernel(const unsigned long long* __restrict__ keys_in,
                 unsigned long long* __restrict__ keys_out,
                 const unsigned int* __restrict__ vals_in, unsigned int* __restrict__ vals_out,
                 uint64_t n, int shift, int bits, const unsigned int* __restrict__ digit_count,
                 unsigned long long* status, const OpState* __restrict__ op_guard) {
  if (op_guard != nullptr && op_guard->err != 0) return;
  constexpr int kWarps = kSortThreads / 32;
  static_assert(kSortThreads == kRadix, "thread d owns digit d");
  extern __shared__ __align__(16) unsigned char sort_smem[];
  unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(sort_smem);
  unsigned int* s_vals = reinterpret_cast<unsigned int*>(s_keys + kSortTile);
  __shared__ unsigned int s_cnt[kWarps][kRadix];  // per-warp digit counts -> exclusive offsets inside the digit
  __shared__ unsigned long long s_goff[kRadix];   // global position of the tile's first key of each digit
  __shared__ unsigned int s_loff[kRadix];         // position of the digit in the tile's sorted order
  __shared__ unsigned int s_wsum[kWarps];
  __shared__ unsigned int s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(reinterpret_cast<unsigned int*>(status), 1u);
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kSortThreads) (&s_cnt[0][0])[i] = 0;
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  // exclusive scan of the 256 raw digit counts (thread d -> base of digit d)
  unsigned int digit_base;
  {
    const unsigned c = digit_count[threadIdx.x];
    unsigned incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    unsigned warp_excl = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) warp_excl += (w < warp) ? s_wsum[w] : 0u;
    digit_base = warp_excl + incl - c;
  }
  const unsigned int tile = s_tile;
  unsigned long long* tile_status = status + 2;

  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned dmask = (1u << bits) - 1u;
  const uint64_t tile_base = (uint64_t)tile * kSortTile;
  const uint64_t warp_base = tile_base + (uint64_t)warp * (32 * kSortItems);

  unsigned long long key[kSortItems];
  unsigned int val[kSortItems];
  unsigned short rank[kSortItems];
  // warp-striped load keeps the stable order (warp, row, lane)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint64_t i = warp_base + (uint64_t)j * 32 + lane;
    key[j] = (i < n) ? keys_in[i] : ~0ull;
    if (kHasValues) val[j] = (i < n) ? vals_in[i] : 0u;
  }
  // all sixteen matches are issued before the first is consumed; only the per-warp counter updates are
  // sequential.  (Measured on 67 M keys, us per pass: this 676; one ballot per digit bit instead of
  // MATCH.ANY 734; shared-memory atomicAdd by the group leaders, all rows pipelined, 892.)
  unsigned peers[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint64_t i = warp_base + (uint64_t)j * 32 + lane;
    const unsigned d = (unsigned)(key[j] >> shift) & dmask;
    peers[j] = __match_any_sync(kFull, (i < n) ? d : 0xFFFFFFFFu);
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint64_t i = warp_base + (uint64_t)j * 32 + lane;
    const bool valid = i < n;
    const unsigned d = (unsigned)(key[j] >> shift) & dmask;
    const int leader = __ffs(peers[j]) - 1;
    unsigned before = 0;
    if (valid && lane == leader) {
      before = s_cnt[warp][d];
      s_cnt[warp][d] = before + __popc(peers[j]);
    }
    before = __shfl_sync(kFull, before, leader);
    rank[j] = (unsigned short)(before + __popc(peers[j] & lt_mask));
    __syncwarp();
  }
  __syncthreads();
  // thread d owns digit d: exclusive scan over warps, tile count, publication
  const int d_own = threadIdx.x;
  unsigned tile_cnt;
  {
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const unsigned c = s_cnt[w][d_own];
      s_cnt[w][d_own] = run;
      run += c;
    }
    tile_cnt = run;
  }
  unsigned long long* my = tile_status + (size_t)tile * kRadix + d_own;
  st_volatile_u64(my, (tile == 0 ? kFlagPre : kFlagAgg) | (unsigned long long)tile_cnt);
  // Look back over the predecessors FIRST, kLook status words in flight per thread: the sooner a tile
  // publishes its inclusive prefix, the fewer predecessors its successors have to add up (the look-back
  // reads 2 KB of status per predecessor and tile: with a deep window that traffic dwarfs the keys).
  {
    unsigned long long excl = 0;
    if (tile != 0) {
      constexpr int kLook = 16;
      long long look = (long long)tile - 1;
      bool done = false;
      while (!done) {
        unsigned long long w[kLook];
#pragma unroll
        for (int q = 0; q < kLook; ++q)
          w[q] = (look - q >= 0) ? ld_volatile_u64(tile_status + (size_t)(look - q) * kRadix + d_own) : kFlagPre;
#pragma unroll
        for (int q = 0; q < kLook; ++q) {
          if (done) break;
          while ((w[q] & kFlagMask) == 0)   // predecessor not published yet
            w[q] = ld_volatile_u64(tile_status + (size_t)(look - q) * kRadix + d_own);
          excl += w[q] & kValMask;
          if ((w[q] & kFlagMask) == kFlagPre) done = true;
        }
        look -= kLook;
      }
      st_volatile_u64(my, kFlagPre | (excl + tile_cnt));
    }
    s_goff[d_own] = (unsigned long long)digit_base + excl;
  }
  {
    // the digit's place in the tile: exclusive scan of the tile counts over the digits
    unsigned incl = tile_cnt;
#pragma unroll
    for (int dl = 1; dl < 32; dl <<= 1) {
      const unsigned t = __shfl_up_sync(kFull, incl, dl);
      if (lane >= dl) incl += t;
    }
    __syncthreads();   // (s_wsum is reused)
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    unsigned warp_excl = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) warp_excl += (w < warp) ? s_wsum[w] : 0u;
    s_loff[d_own] = warp_excl + incl - tile_cnt;
  }
  __syncthreads();
  // keys (and values) into shared memory, in digit order
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint64_t i = warp_base + (uint64_t)j * 32 + lane;
    if (i < n) {
      const unsigned d = (unsigned)(key[j] >> shift) & dmask;
      const unsigned p = s_loff[d] + s_cnt[warp][d] + rank[j];
      s_keys[p] = key[j];
      if (kHasValues) s_vals[p] = val[j];
    }
  }
  __syncthreads();
  // write-out over consecutive shared positions
  const unsigned tile_n = (unsigned)((n - tile_base) < (uint64_t)kSortTile ? (n - tile_base) : (uint64_t)kSortTile);
#pragma unroll 4
  for (unsigned i = threadIdx.x; i < tile_n; i += kSortThreads) {
    const unsigned long long k = s_keys[i];
    const unsigned d = (unsigned)(k >> shift) & dmask;
    const unsigned long long pos = s_goff[d] + (i - s_loff[d]);
    keys_out[pos] = k;
    if (kHasValues) vals_out[pos] = s_vals[i];
  }
}
constexpr size_t kSortSmemKeys = (size_t)kSortTile * sizeof(unsigned long long);
constexpr size_t kSortSmemKeysVals = kSortSmemKeys + (size_t)kSortTile * sizeof(unsigned int);

// ---- warp-cooperative 32-ary upper bound -----------------------------------
// Largest r in [0, count) with arr[r] <= x, given arr non-decreasing and
// arr[0] <= x.  All lanes of the warp must call with the same arguments.
template <class T>
__device__ __forceinline__ uint32_t warp_find_run(const T* __restrict__ arr, uint32_t count,
                                                  T x) {
  uint32_t lo = 0, hi = count;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const uint32_t span = hi - lo;
    const uint32_t step = (span + 31) / 32;
    const uint32_t probe = lo + (uint32_t)lane_id() * step;
    const bool le = (probe < hi) && (arr[probe] <= x);
    const unsigned m = __ballot_sync(kFull, le);
    // lanes with le form a prefix (arr is monotone); the last set lane bounds the answer
    const int last = 31 - __clz(m);  // m != 0 because arr[lo] <= x
    const uint32_t nlo = lo + (uint32_t)last * step;
    const uint32_t nhi = min(hi, nlo + step);
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// Scalar lower bound over the low 32 bits of sorted 64-bit keys in [lo, hi).
__device__ __forceinline__ uint32_t lower_bound_lo32(const unsigned long long* __restrict__ keys,
                                                     uint32_t lo, uint32_t hi, uint32_t x) {
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if ((uint32_t)keys[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace dg
