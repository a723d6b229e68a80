// dg_fused.cuh — delete for sources a single warp can own, in ONE kernel (sm_100a, B = 32).
//
// delete_batch (graph.hpp:195-222) per touched source = scan the whole adjacency
// (delete_adjacency, :376-394), drop every copy of every target, repair the
// counters and give emptied tail blocks back to the queue (detach_empty_tail,
// :398-414; reclaim, block_pool.hpp:192-209).  The multi-kernel path (enumerate ->
// match tiers -> compaction plan -> holes -> moves) pays a global round trip of
// work lists and masks between every stage.  Here a warp OWNS its sources for the
// whole op:
//   small  (k <= 8 targets, chain <= 16 blocks): 32 sources per warp, one per lane for
//          the metadata, the chain walk and the compaction; their blocks are pooled
//          into one per-warp list and matched 32 blocks at a time (lane = block).
//   medium (k <= 128 targets, chain <= 256 blocks): a warp per source; the chain is
//          walked 32 links per round trip, the targets sit in a per-warp shared-memory
//          table + membership filter, compaction is warp-parallel.
// Handles and match masks never leave shared memory; no tombstone is ever written
// (a hole below the new degree is overwritten by a survivor from above it, slots
// past the new degree are free).  Everything else (hubs: longer chains or more
// targets) keeps the multi-kernel path and runs beside this kernel.
#pragma once

#include "dg_kernels.cuh"

namespace dg {

// Per-warp shared memory (a CTA is ONE warp: the hardware CTA scheduler is the load balancer, no warp ever
// waits at a CTA barrier for a heavier neighbour).  One byte array, carved per role:
//   small : stg 4096 | hnd 128 x 4 | msk 128 x 4 | own 128 x 2 | targets 32 x 8 x 4 | filters 32 x 8      = 6656 B
//   medium: stg 4096 (compaction: prefix arrays) | hnd 256 x 4 | msk 256 x 4 | table 256 x 4 | filter 512 = 7680 B
constexpr uint32_t kFusedSmallList = 128;   // blocks a warp holds at a time in the small role
constexpr uint32_t kFusedTable = 256;       // >= 2 x kFusedMedTargets
constexpr size_t kFusedSmemBytes = 7680;
// tallies are striped over kTallyStripes x 8 words (one stripe per CTA, round-robin) and folded into
// OpState / DeviceState by fused_tally_kernel: tens of thousands of one-warp CTAs never share a counter line
constexpr uint32_t kTallyStripes = 64;
enum Tally : int { kTalMatched = 0, kTalSlots, kTalBlocks, kTalMoves, kTalPushed, kTalWords = 8 };
static_assert(kFusedMedBlocks <= kFusedListBlocks && kFusedTable >= 2 * kFusedMedTargets, "medium role layout");

__device__ __forceinline__ uint32_t low_bits(uint32_t n) { return n >= 32u ? 0xFFFFFFFFu : ((1u << n) - 1u); }
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, v, d);
    if (lane_id() >= d) v += t;
  }
  return v;
}
__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// The kernel is launched BESIDE the counting group-by's scatter: everything that does not need the grouped
// targets (run records, chain links, the blocks on their way to L2) is issued first, then the warp waits
// until every scatter CTA has finished.  expected == 0: the batch was grouped before the launch.
__device__ __forceinline__ void wait_scatter(const OpState* op, uint32_t expected) {
  if (expected == 0) return;
  if (lane_id() == 0) {
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&op->scatter_ctas) : "memory");
      if (v < expected) __nanosleep(64);
    } while (v < expected);
  }
  __syncwarp();
}

// Pushes `cnt` handles hnd[first .. first + cnt) of every lane to the ring rear: ONE atomicAdd per
// warp (reclaim, block_pool.hpp:192-209).  All lanes must call.
__device__ __forceinline__ uint32_t warp_push_freed(const GraphView& g, const uint32_t* hnd, uint32_t first, uint32_t cnt) {
  const uint32_t incl = warp_incl_scan(cnt);
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  if (total == 0) return 0;
  unsigned long long base = 0;
  if (lane_id() == 0) base = atomicAdd(&g.st->rear, (unsigned long long)total) % g.ring_cap;
  unsigned long long p = __shfl_sync(kFull, base, 0) + (incl - cnt);   // < 2 * ring_cap
#pragma unroll 1
  for (uint32_t j = 0; j < cnt; ++j, ++p) {
    if (p >= g.ring_cap) p -= g.ring_cap;
    g.ring[p] = hnd[first + j];
  }
  return total;
}

__device__ __forceinline__ uint32_t redux_add(uint32_t v) {
  uint32_t r;
  asm volatile("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
// per-lane 32-bit partial sums -> one REDUX per counter, one atomic per counter and warp on the CTA's stripe
__device__ __noinline__ void tally_flush(unsigned long long* tally, uint32_t matched, uint32_t slots, uint32_t blocks,
                                         uint32_t moves, uint32_t pushed) {
  const uint32_t v[5] = {redux_add(matched), redux_add(slots), redux_add(blocks), redux_add(moves), redux_add(pushed)};
  if (lane_id() == 0) {
    unsigned long long* t = tally + (size_t)(blockIdx.x % kTallyStripes) * kTalWords;
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if (v[i]) atomicAdd(&t[i], (unsigned long long)v[i]);
  }
}

// grid: [0, g_med) medium role — CTA c takes med_list[c], med_list[c + g_med], ... (heaviest work first);
//       [g_med, g_med + ceil(T / 32)) small role — 32 consecutive runs per warp, lane = run.
__global__ void __launch_bounds__(32, 28)
fused_delete_kernel(GraphView g, BatchView b, const uint32_t* __restrict__ run_cls, const uint32_t* __restrict__ run_deg,
                    const uint32_t* __restrict__ run_head, const uint4* __restrict__ med_rec, uint32_t g_med,
                    uint32_t runs_bound, GroupIndex gi, uint32_t* __restrict__ cnt, uint32_t scatter_expected,
                    unsigned long long* tally, OpState* op) {
  __shared__ __align__(16) unsigned char smem[kFusedSmemBytes];
  const int lane = lane_id();
  uint32_t(*stg)[32] = reinterpret_cast<uint32_t(*)[32]>(smem);
  // the op words share one line: requested together, tested after the role's own first loads are in flight
  const uint32_t op_err = op->err;
  uint32_t t_matched = 0, t_slots = 0, t_blocks = 0, t_moves = 0, t_pushed = 0;

  if (blockIdx.x >= g_med) {
    // =========================== small sources: lane = source ===========================
    struct SmallSmem {
      uint32_t stg[32][32];
      uint32_t hnd[kFusedSmallList], msk[kFusedSmallList];
      uint16_t own[kFusedSmallList];   // [4:0] owner lane, [10:5] live slots - 1
      uint32_t tg[32 * 8];
      unsigned long long filt[32];
    };
    static_assert(sizeof(SmallSmem) <= kFusedSmemBytes, "small role layout");
    SmallSmem& sw = *reinterpret_cast<SmallSmem*>(smem);
    // every first load is issued before anything is waited for (the run arrays cover the whole grid: entries
    // past the run count hold garbage and are discarded once the count has arrived)
    const uint32_t r = (blockIdx.x - g_med) * 32u + lane;
    const uint32_t rr = min(r, runs_bound - 1u);
    uint32_t cls = run_cls[rr];
    const uint32_t es = b.run_start[rr];
    const uint32_t k = b.run_end[rr] - es;
    const uint32_t d = run_deg[rr];
    const uint32_t h0 = run_head[rr];
    const uint32_t v = batch_src(b, rr);
    const uint32_t T = (uint32_t)op->n_runs;
    if (op_err || r - lane >= T) return;
    if (r >= T) cls = kClsNone;
    // the counting group-by's per-source word goes back to zero (it is never cleared between ops)
    if (cnt != nullptr && r < T) cnt[gi(v)] = 0u;
    uint32_t* s_tg = sw.tg;
    unsigned long long* s_filt = sw.filt;
    const bool small = cls == kClsSmall;
    const uint32_t nb = small ? (d + 31u) >> 5 : 0u;
    unsigned pending = __ballot_sync(kFull, small);
    if (pending == 0) return;
    // the blocks start their way to L2 now: the head is certain, the next three are a guess (chains are
    // physically consecutive unless their blocks were recycled)
    if (small) {
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q)
        if (q < nb && (unsigned long long)h0 + q < g.ring_cap) prefetch_l2(g.slab + ((unsigned long long)h0 + q) * 32u);
    }
    wait_scatter(op, scatter_expected);
#pragma unroll 1
    while (pending) {
      const bool mine_p = (pending >> lane) & 1u;
      const uint32_t incl = warp_incl_scan(mine_p ? nb : 0u);
      const bool mine = mine_p && incl <= kFusedSmallList;   // a prefix of the pending lanes
      const unsigned bmask = __ballot_sync(kFull, mine);
      pending &= ~bmask;
      const uint32_t off = incl - nb;
      const uint32_t N = __shfl_sync(kFull, incl, 31 - __clz(bmask));
      if (mine) {
        // ---- targets + filter of the lane's source
        uint32_t tg[kFusedSmallTargets];
#pragma unroll
        for (int j = 0; j < (int)kFusedSmallTargets; ++j) tg[j] = ((uint32_t)j < k) ? batch_value(b, es + j) : kTomb;
        // ---- chain walk: up to four physically consecutive blocks per round trip
        uint32_t h = h0, j = 0;
#pragma unroll 1
        while (j < nb) {
          uint32_t nx[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const unsigned long long hh = (unsigned long long)h + q;
            nx[q] = hh < g.ring_cap ? g.next[hh] : kNull;
          }
          bool go = true;
          uint32_t succ = kNull;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (go) {
              sw.hnd[off + j] = h + q;
              if (j >= 4) prefetch_l2(g.slab + (unsigned long long)(h + q) * 32u);
              const uint32_t cb = min(32u, d - 32u * j);
              sw.own[off + j] = (uint16_t)(lane | ((cb - 1u) << 5));
              ++j;
              succ = nx[q];
              go = j < nb && succ == h + (uint32_t)q + 1u;
            }
          }
          h = succ;
        }
        unsigned long long filt = 0;
#pragma unroll
        for (int j2 = 0; j2 < (int)kFusedSmallTargets; ++j2) {
          s_tg[lane * 8 + j2] = tg[j2];
          if ((uint32_t)j2 < k) filt |= 1ull << filter_hash(tg[j2], 6);
        }
        s_filt[lane] = filt;
        t_slots += d;
        t_blocks += nb;
      }
      __syncwarp();
      // ---- match: 32 blocks per round, lane = block
#pragma unroll 1
      for (uint32_t base = 0; base < N; base += 32) {
        const uint32_t bi = base + lane;
        const bool valid = bi < N;
        const uint32_t hd = valid ? sw.hnd[bi] : 0u;
        const uint32_t ow = valid ? sw.own[bi] : 0u;
        stage_blocks32(g, stg, hd, low_bits(N - base));
        cp_async_wait_all();
        __syncwarp();
        if (valid) {
          const int o = ow & 31;
          const uint32_t cb = (ow >> 5) + 1u;
          const unsigned long long filt = s_filt[o];
          uint32_t cand = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 x = block_chunk(stg, lane, c);
            cand |= (uint32_t)((filt >> filter_hash(x.x, 6)) & 1ull) << (4 * c);
            cand |= (uint32_t)((filt >> filter_hash(x.y, 6)) & 1ull) << (4 * c + 1);
            cand |= (uint32_t)((filt >> filter_hash(x.z, 6)) & 1ull) << (4 * c + 2);
            cand |= (uint32_t)((filt >> filter_hash(x.w, 6)) & 1ull) << (4 * c + 3);
          }
          cand &= low_bits(cb);   // slots past the degree hold stale values
          uint32_t mask = 0;
          if (cand) {
            const uint4 ta = *reinterpret_cast<const uint4*>(&s_tg[o * 8]);
            const uint4 tb = *reinterpret_cast<const uint4*>(&s_tg[o * 8 + 4]);
#pragma unroll 1
            while (cand) {
              const uint32_t bit = __ffs(cand) - 1;
              cand &= cand - 1;
              const uint32_t e = block_slot(stg, lane, bit);
              if (e == ta.x || e == ta.y || e == ta.z || e == ta.w || e == tb.x || e == tb.y || e == tb.z || e == tb.w)
                mask |= 1u << bit;
            }
          }
          sw.msk[bi] = mask;
        }
        __syncwarp();
      }
      // ---- compaction + repair: lane = source (graph.hpp:398-414 on a compact chain)
      uint32_t nfree = 0, new_nb = nb;
      if (mine) {
        uint32_t m = 0;
#pragma unroll 1
        for (uint32_t j = 0; j < nb; ++j) m += __popc(sw.msk[off + j]);
        if (m) {
          const uint32_t nd = d - m;
          new_nb = (nd + 31u) >> 5;
          uint32_t ps = nd;   // next candidate survivor position (>= nd)
#pragma unroll 1
          for (uint32_t kb = 0; kb * 32u < nd; ++kb) {
            uint32_t bits = sw.msk[off + kb] & low_bits(nd - kb * 32u);
#pragma unroll 1
            while (bits) {
              const uint32_t bit = __ffs(bits) - 1;
              bits &= bits - 1;
#pragma unroll 1
              while ((sw.msk[off + (ps >> 5)] >> (ps & 31u)) & 1u) ++ps;
              const uint32_t val = g.slab[(unsigned long long)sw.hnd[off + (ps >> 5)] * 32u + (ps & 31u)];
              g.slab[(unsigned long long)sw.hnd[off + kb] * 32u + bit] = val;
              ++ps;
              ++t_moves;
            }
          }
          g.deg[v] = nd;
          if (nd == 0) {
            g.head[v] = kNull;
            g.tail[v] = kNull;
          } else {
            const uint32_t t = sw.hnd[off + new_nb - 1];
            g.tail[v] = t;
            g.next[t] = kNull;
          }
          t_matched += m;
          if (g.reclaim) nfree = nb - new_nb;
        }
      }
      {
        const uint32_t pushed = warp_push_freed(g, sw.hnd, off + new_nb, nfree);
        if (lane == 0) t_pushed += pushed;
      }
      __syncwarp();
    }
    tally_flush(tally, t_matched, t_slots, t_blocks, t_moves, t_pushed);
    return;
  }

  // =========================== medium sources: the warp = one source ===========================
  struct MedSmem {
    uint32_t stg[32][32];
    uint32_t hnd[kFusedListBlocks], msk[kFusedListBlocks];
    uint32_t tab[kFusedTable];
    uint32_t bm[(1u << kMedFilterBits) / 32];
  };
  static_assert(sizeof(MedSmem) <= kFusedSmemBytes, "medium role layout");
  MedSmem& sw = *reinterpret_cast<MedSmem*>(smem);
  uint4 rec0 = med_rec[2u * blockIdx.x], rec1 = med_rec[2u * blockIdx.x + 1u];   // (garbage past the count: unused)
  const uint32_t n_med = op->n_fmed;
  if (op_err) return;
#pragma unroll 1
  for (uint32_t qi = blockIdx.x; qi < n_med; qi += g_med) {
    if (qi != blockIdx.x) {
      rec0 = med_rec[2u * qi];
      rec1 = med_rec[2u * qi + 1u];
    }
    const uint32_t mv = rec0.y, mes = rec0.z, mk = rec0.w;
    const uint32_t md = rec1.x, h0 = rec1.y;
    const uint32_t mnb = (md + 31u) >> 5;
    // ---- one round trip: the targets, every link of the chain under the guess that it is physically
    // consecutive (bulk-built and ring-popped chains are), and the first blocks on their way to L2
    uint32_t nx[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const unsigned long long hh = (unsigned long long)h0 + 32u * q + lane;
      nx[q] = (32u * q + lane < mnb && hh < g.ring_cap) ? g.next[hh] : kNull;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const unsigned long long hh = (unsigned long long)h0 + 32u * q + lane;
      if (32u * q + lane < mnb && hh < g.ring_cap) prefetch_l2(g.slab + hh * 32u);
    }
    wait_scatter(op, scatter_expected);
    uint32_t tg[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) tg[q] = (32u * q + lane < mk) ? batch_value(b, mes + 32u * q + lane) : kTomb;
    // ---- table (2^tb >= 2 k entries, at least 32: sized to the source) + 4096-bit membership filter of the targets
    const int tb = max(5, 32 - __clz(2u * mk - 1u));
    const uint32_t tmask = (1u << tb) - 1u;
    const int hshift = 32 - tb;
    constexpr int fb = kMedFilterBits;
#pragma unroll 1
    for (uint32_t i = lane; i <= tmask; i += 32) sw.tab[i] = kTomb;
#pragma unroll
    for (uint32_t i = 0; i < (1u << fb) / 32; i += 32) sw.bm[i + lane] = 0;
    __syncwarp();
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
      const uint32_t t = q == 0 ? tg[0] : q == 1 ? tg[1] : q == 2 ? tg[2] : tg[3];
      if (32u * q + lane < mk) table_insert(sw.tab, tmask, hshift, sw.bm, fb, t);
    }
    // ---- handles: the confirmed consecutive prefix, then a dependent walk for whatever is left
    uint32_t conf = 0;   // blocks h0 .. h0 + conf - 1 are the first conf blocks of the chain
    uint32_t h = h0;
    {
      bool open = true;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (open && 32u * q < mnb) {
          const uint32_t hh = h0 + 32u * q + lane;
          const unsigned okm = __ballot_sync(kFull, nx[q] == hh + 1u);
          uint32_t len = (okm == kFull) ? 32u : (uint32_t)__ffs(~okm);   // links ok for len - 1 blocks; block itself counts
          len = min(len, mnb - 32u * q);
          if ((uint32_t)lane < len) sw.hnd[32u * q + lane] = hh;
          conf = 32u * q + len;
          h = __shfl_sync(kFull, nx[q], len - 1);   // successor of the last confirmed block
          open = len == 32u && okm == kFull;
        }
      }
    }
#pragma unroll 1
    while (conf < mnb) {   // (recycled chains) one round trip per physically consecutive run
      const unsigned long long hh = (unsigned long long)h + lane;
      const uint32_t nxw = hh < g.ring_cap ? g.next[hh] : kNull;
      const unsigned okm = __ballot_sync(kFull, (unsigned long long)nxw == hh + 1);
      uint32_t len = (okm == kFull) ? 32u : (uint32_t)__ffs(~okm);
      len = min(len, mnb - conf);
      if ((uint32_t)lane < len) sw.hnd[conf + lane] = (uint32_t)hh;
      h = __shfl_sync(kFull, nxw, len - 1);
      conf += len;
    }
    __syncwarp();
    // ---- match, 32 blocks per round
    uint32_t matched = 0;
#pragma unroll 1
    for (uint32_t kb = 0; kb < mnb; kb += 32) {
      const uint32_t cnt = min(32u, mnb - kb);
      const uint32_t hd = ((uint32_t)lane < cnt) ? sw.hnd[kb + lane] : 0u;
      if (kb + 64u + lane < mnb) prefetch_l2(g.slab + (unsigned long long)sw.hnd[kb + 64u + lane] * 32u);
      stage_blocks32(g, stg, hd, low_bits(cnt));
      cp_async_wait_all();
      __syncwarp();
      uint32_t mask = 0;
      if ((uint32_t)lane < cnt) {
        const uint32_t cb = min(32u, md - 32u * (kb + lane));
        uint32_t cand = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 x = block_chunk(stg, lane, c);
          const uint32_t evs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t hb = filter_hash(evs[i], fb);
            cand |= ((sw.bm[hb >> 5] >> (hb & 31)) & 1u) << (4 * c + i);
          }
        }
        cand &= low_bits(cb);
#pragma unroll 1
        while (cand) {
          const uint32_t bit = __ffs(cand) - 1;
          cand &= cand - 1;
          const uint32_t ev = block_slot(stg, lane, bit);
          uint32_t pos = (ev * 0x9E3779B1u) >> hshift;
          uint32_t t = sw.tab[pos];
#pragma unroll 1
          while (t != ev && t != kTomb) {
            pos = (pos + 1) & tmask;
            t = sw.tab[pos];
          }
          if (t == ev) mask |= 1u << bit;
        }
        sw.msk[kb + lane] = mask;
      }
      matched += __popc(mask);
      __syncwarp();   // the strip is restaged by the next round
    }
    matched = redux_add(matched);
    if (lane == 0) {
      t_slots += md;
      t_blocks += mnb;
    }
    uint32_t new_nb = mnb, nfree = 0;
    uint32_t moves = 0;
    if (matched) {
      // matches at or above the new degree leave no hole: moves = matches below it (often none: the
      // newest entries of a source sit at the end of its chain)
      const uint32_t nd = md - matched;
      uint32_t m_hi = 0;
#pragma unroll 1
      for (uint32_t bi = (nd >> 5) + lane; bi < mnb; bi += 32) {
        const uint32_t lo = bi * 32u;
        m_hi += __popc(sw.msk[bi] & ~low_bits(nd > lo ? nd - lo : 0u));
      }
      moves = matched - redux_add(m_hi);
    }
    if (matched) {
      const uint32_t nd = md - matched;
      new_nb = (nd + 31u) >> 5;
    }
    if (moves) {
      // ---- warp-parallel compaction: hole j (below the new degree) takes survivor j (above it)
      const uint32_t nd = md - matched;
      uint16_t* hpre = reinterpret_cast<uint16_t*>(&stg[0][0]);   // exclusive hole / survivor counts per block
      uint16_t* spre = hpre + kFusedListBlocks;
      uint32_t carry_h = 0, carry_s = 0;
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < mnb; c0 += 32) {
        const uint32_t bi = c0 + lane;
        uint32_t hc = 0, sc = 0;
        if (bi < mnb) {
          const uint32_t mword = sw.msk[bi];
          const uint32_t lo = bi * 32u;
          const uint32_t below = nd > lo ? min(32u, nd - lo) : 0u;   // slots of this block below the new degree
          const uint32_t live = min(32u, md - lo);
          hc = __popc(mword & low_bits(below));
          sc = __popc(~mword & low_bits(live) & ~low_bits(below));
        }
        const uint32_t hi = warp_incl_scan(hc), si = warp_incl_scan(sc);
        if (bi < mnb) {
          hpre[bi] = (uint16_t)(carry_h + hi - hc);
          spre[bi] = (uint16_t)(carry_s + si - sc);
        }
        carry_h += __shfl_sync(kFull, hi, 31);
        carry_s += __shfl_sync(kFull, si, 31);
      }
      __syncwarp();
      const uint32_t sb0 = nd >> 5;     // first block that can hold a survivor (carry_h == carry_s == moves)
#pragma unroll 1
      for (uint32_t j = lane; j < moves; j += 32) {
        // largest block index with prefix <= j: the block that holds entry j (an empty block shares its
        // prefix with its successor, so it is never the largest)
        uint32_t lo = 0, hi = new_nb;   // holes live in blocks [0, new_nb)
#pragma unroll 1
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (hpre[mid] <= j) lo = mid; else hi = mid;
        }
        const uint32_t hb = lo;
        const uint32_t hbelow = nd > hb * 32u ? min(32u, nd - hb * 32u) : 0u;
        const uint32_t hbits = sw.msk[hb] & low_bits(hbelow);
        const uint32_t hslot = __fns(hbits, 0, (int)(j - hpre[hb]) + 1);
        lo = sb0;
        hi = mnb;
#pragma unroll 1
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (spre[mid] <= j) lo = mid; else hi = mid;
        }
        const uint32_t sb = lo;
        const uint32_t sbelow = nd > sb * 32u ? min(32u, nd - sb * 32u) : 0u;
        const uint32_t sbits = ~sw.msk[sb] & low_bits(min(32u, md - sb * 32u)) & ~low_bits(sbelow);
        const uint32_t sslot = __fns(sbits, 0, (int)(j - spre[sb]) + 1);
        const uint32_t val = g.slab[(unsigned long long)sw.hnd[sb] * 32u + sslot];
        g.slab[(unsigned long long)sw.hnd[hb] * 32u + hslot] = val;
      }
    }
    if (matched) {
      const uint32_t nd = md - matched;
      if (lane == 0) {
        g.deg[mv] = nd;
        if (nd == 0) {
          g.head[mv] = kNull;
          g.tail[mv] = kNull;
        } else {
          const uint32_t t = sw.hnd[new_nb - 1];
          g.tail[mv] = t;
          g.next[t] = kNull;
        }
        t_matched += matched;
        t_moves += moves;
      }
      if (g.reclaim) nfree = mnb - new_nb;
    }
    // freed blocks: contiguous slices per lane
    {
      const uint32_t per = (nfree + 31u) / 32u;
      const uint32_t f0 = min(nfree, per * lane), f1 = min(nfree, per * (lane + 1));
      const uint32_t pushed = warp_push_freed(g, sw.hnd, new_nb + f0, f1 - f0);
      if (lane == 0) t_pushed += pushed;
    }
    __syncwarp();
  }
  tally_flush(tally, t_matched, t_slots, t_blocks, t_moves, t_pushed);
}

// folds the striped tallies into the op words and the live-edge count (graph.hpp:211-213); one warp per
// counter, two stripes per lane, every word handed back zeroed (the buffer is persistent)
__global__ void fused_tally_kernel(GraphView g, unsigned long long* __restrict__ tally, OpState* op) {
  if (op->err) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;   // blockDim = 5 warps
  unsigned long long v = 0;
#pragma unroll
  for (uint32_t s = lane; s < kTallyStripes; s += 32) {
    unsigned long long* p = &tally[(size_t)s * kTalWords + w];
    v += *p;
    *p = 0ull;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  if (lane != 0 || v == 0) return;
  if (w == kTalMatched) {
    atomicAdd(&op->matched, v);
    atomicAdd(&g.st->active_edges, (unsigned long long)(-(long long)v));
  } else if (w == kTalSlots) {
    atomicAdd(&op->slots, v);
    atomicAdd(&op->slots_fused, v);
  } else if (w == kTalBlocks) {
    atomicAdd(&op->fused_blocks, v);
  } else if (w == kTalMoves) {
    atomicAdd(&op->moves, v);
  } else if (w == kTalPushed) {
    atomicAdd(&op->pushed, v);
  }
}

}  // namespace dg
