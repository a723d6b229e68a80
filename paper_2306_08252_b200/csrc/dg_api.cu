// dg_api.cu — host engine + C ABI of libdyngraph_b200.so (see include/dyngraph_b200.h).
//
// Host code is plain C++ over the CUDA runtime; no torch types cross the ABI.
// Every op is a fixed sequence of kernels enqueued on the graph's stream with
// NO host round trip between validation and mutation: validation kernels set
// OpState::err on the device and every later kernel of the op starts with
// `if (op->err) return;` (validate-then-mutate, reference graph.hpp:168-171).
// The op ends with one 256-byte read-back of {DeviceState, OpState}.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <tuple>
#include <new>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/dyngraph_b200.h"
#include "dg_fused.cuh"

using namespace dg;

namespace {

struct DevBlock {  // one contiguous device allocation read back per op
  DeviceState st;
  OpState op;
};

struct Workspace {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
};

constexpr size_t kAlign = 256;
inline size_t aligned(size_t b) { return (b + kAlign - 1) / kAlign * kAlign; }

thread_local std::string g_create_error;

// ---- device memory committed in place (CUDA virtual memory management) -------------------------
// The growing pool arrays (slab, next links) reserve their address range for the largest pool
// once; physical chunks are mapped behind the committed part as the pool grows, so device
// pointers stay valid and nothing is copied.  The driver entry points are looked up at run
// time (cudaGetDriverEntryPoint): the library does not link against libcuda.
struct DrvApi {
  CUresult (*getGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*addressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  bool ok = false;
};
const DrvApi& drv() {
  static DrvApi api = [] {
    DrvApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess && *fn;
    };
    a.ok = get("cuMemGetAllocationGranularity", (void**)&a.getGranularity) && get("cuMemAddressReserve", (void**)&a.addressReserve) &&
           get("cuMemAddressFree", (void**)&a.addressFree) && get("cuMemCreate", (void**)&a.create) &&
           get("cuMemRelease", (void**)&a.release) && get("cuMemMap", (void**)&a.map) && get("cuMemUnmap", (void**)&a.unmap) &&
           get("cuMemSetAccess", (void**)&a.setAccess);
    cudaGetLastError();
    return a;
  }();
  return api;
}
struct VmRange {
  CUdeviceptr base = 0;
  size_t reserved = 0, mapped = 0, gran = 0;
  int device = 0;
  std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> chunks;
  bool reserve(int dev, size_t max_bytes) {
    const DrvApi& d = drv();
    if (!d.ok) return false;
    device = dev;
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev;
    if (d.getGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0) return false;
    reserved = (max_bytes + gran - 1) / gran * gran;
    return d.addressReserve(&base, reserved, 0, 0, 0) == CUDA_SUCCESS;
  }
  // commit at least `bytes` in total
  bool commit(size_t bytes) {
    const DrvApi& d = drv();
    const size_t want = std::min(reserved, (bytes + gran - 1) / gran * gran);
    if (want <= mapped) return bytes <= mapped;
    const size_t add = want - mapped;
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    CUmemGenericAllocationHandle hdl;
    if (d.create(&hdl, add, &prop, 0) != CUDA_SUCCESS) return false;
    if (d.map(base + mapped, add, 0, hdl, 0) != CUDA_SUCCESS) { d.release(hdl); return false; }
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (d.setAccess(base + mapped, add, &acc, 1) != CUDA_SUCCESS) { d.unmap(base + mapped, add); d.release(hdl); return false; }
    chunks.emplace_back(hdl, add);
    mapped = want;
    return bytes <= mapped;
  }
  void destroy() {
    const DrvApi& d = drv();
    if (!base) return;
    size_t off = 0;
    for (auto& c : chunks) { d.unmap(base + off, c.second); d.release(c.first); off += c.second; }
    d.addressFree(base, reserved);
    chunks.clear();
    base = 0; reserved = mapped = 0;
  }
};

}  // namespace

struct dg_graph {
  dg_config cfg{};
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int reclaim = 1;
  int group_mode = 0;  // 0 auto, 1 radix sort, 2 per-vertex counting

  uint32_t B = 0;
  uint64_t size = 0;       // logical size
  uint64_t capacity = 0;   // closest_pow2
  uint64_t alive_count = 0;
  uint64_t dst_limit_override = 0;  // 0 => size
  std::vector<uint64_t> alive_host;  // host mirror of the alive flags

  // vertex dictionary SoA
  uint32_t *head = nullptr, *tail = nullptr, *deg = nullptr, *alive = nullptr;
  // pool
  uint32_t *slab = nullptr, *next = nullptr, *ring = nullptr;
  uint64_t NB = 0;
  // growth (GrowthPolicy, block_pool.hpp:18-29)
  uint64_t nb_max = 0;          // most blocks the pool may hold; <= NB: fixed pool
  double trigger = 0.8, growth = 0.25;
  uint64_t consumed = 0;        // cumulative pops (block_pool.hpp consumed())
  uint64_t total_capacity = 0;  // handles ever made available: created + every re-push of a reclaimed one (block_pool.hpp:42-44)
  bool ws_overflow = false;     // a scratch request did not fit the reserved workspace: the op is rejected
  cudaError_t launch_error = cudaSuccess;   // first kernel launch error of the op (checked at the launch site)
  uint32_t growth_count = 0;
  uint64_t ring_identity = 0;   // ring[p] == p for queue positions below this
  bool pool_vm = false;         // slab / next live in VmRanges
  VmRange vm_slab, vm_next;

  DevBlock* d_blk = nullptr;  // device
  DevBlock* h_blk = nullptr;  // pinned host mirror of the CURRENT op: one slot of h_ring
  DevBlock* h_ring = nullptr; // pinned status slots: every op reads back into its own, so submitted ops need no host wait
  DevBlock* h_ring_dev = nullptr;   // the same slots as the device sees them (mapped host memory; nullptr: memcpy instead)
  uint32_t h_ring_next = 0;
  uint64_t front = 0, rear = 0, active_edges = 0;   // as of the last RETIRED op

  // Submitted (asynchronous) ops, oldest first: enqueued on the stream, status not yet looked at.
  struct Pending {
    uint64_t ticket;
    bool is_insert;
    uint64_t pop_bound;   // most blocks the op can pop (inserts)
    DevBlock* slot;       // where its {DeviceState, OpState} lands
    cudaEvent_t done;     // recorded behind the read-back
    uint64_t launches;
    uint64_t n;
  };
  std::deque<Pending> pending;
  std::vector<cudaEvent_t> done_pool;
  bool submitting = false;        // the op being enqueued ends without a host wait (op_end)
  bool submit_is_insert = false;
  uint64_t submit_pop_bound = 0;
  uint64_t next_ticket = 1;
  uint64_t pending_pop_bound = 0; // sum over `pending`
  uint64_t submitted_applied = 0; // submitted ops retired successfully since the last dg_flush
  // Early count: a submitted counting-path op that follows a submitted counting-path INSERT runs its group_count
  // beside that insert's append pass (it needs the batch and clean counters only — the insert's plan hands the
  // counters back zeroed): own rank buffers, own error words, merged by op_arm_kernel.
  uint32_t* rank_alt[2] = {nullptr, nullptr};
  uint64_t rank_alt_cap = 0, rank_alt_want = 0;
  OpState* d_pre = nullptr;       // two sets of error words
  cudaEvent_t ev_plan_done = nullptr, ev_early = nullptr;
  bool early_possible = false;    // the last enqueued op is such an insert (ev_plan_done is recorded behind its plan)
  cudaEvent_t input_ready = nullptr;   // ingest queue: the copy-done event of the slot being submitted
  uint32_t early_next = 0;
  struct { bool active = false; uint32_t* rank = nullptr; OpState* pre = nullptr; } early;
  int deferred_rc = 0;            // first failure among retired submitted ops, not yet returned to the caller
  uint64_t deferred_ticket = 0;
  std::string deferred_error;

  Workspace ws;

  // independent kernels of one op (chain walks, the match tiers) run side by side on two
  // auxiliary streams between a fork and a join on the op's stream
  cudaStream_t aux[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr}, ev_main = nullptr;
  bool forked = false;
  // Persistent scratch that every op hands back ZEROED (no memset between ops): the per-vertex counters
  // of the counting group-by (their users reset the words they touched), the alloc_kernel cursors (the
  // last tile resets them) and the striped tallies of fused_delete_kernel (fused_tally_kernel resets them).
  // After a failed or non-self-cleaning op the `*_clean` flags are false and the next user clears the buffer.
  uint32_t* cnt_buf = nullptr;
  uint64_t cnt_cap = 0;          // words
  bool cnt_clean = false;
  unsigned long long* zscratch = nullptr;   // [0, 8 x 4) alloc cursors, then kTallyStripes x kTalWords tallies
  bool zscratch_clean = false;
  int zslot = 0;

  struct dg_exchange* agree_x = nullptr;   // sharded store: ops agree their status with the peers before mutating
  std::string last_error;
  uint64_t last_shortfall = 0;  // blocks the last rejected insert was short of (0: it was not a pool underflow)
  dg_op_report report{};
  uint64_t launches = 0;

  // optional per-kernel timing (dg_profile_enable): CUDA events around every launch
  bool profiling = false;
  struct ProfSpan { const char* name; cudaEvent_t a, b; };
  std::vector<ProfSpan> prof_open;
  std::vector<cudaEvent_t> prof_pool;
  std::map<std::string, std::pair<double, uint64_t>> prof_acc;  // name -> (ms, launches)
  std::string prof_text;
  // optional timeline of the last op (DG_TIMELINE=1): events at named points of the op's streams, without
  // serialising them — where the op's time goes when kernels run side by side
  bool timeline = false;
  struct TlMark { const char* name; cudaEvent_t ev; };
  std::vector<TlMark> tl_marks;

  DeviceState* d_state() const { return &d_blk->st; }
  OpState* d_op() const { return &d_blk->op; }
  uint64_t dst_limit() const { return dst_limit_override ? dst_limit_override : size; }
  // (an upper bound while submitted inserts are in flight: sizes work lists, never read as a count)
  uint64_t blocks_in_use() const { return std::min<uint64_t>(NB, NB - (rear - front) + pending_pop_bound); }
  bool alive_h(uint64_t v) const { return v < size && ((alive_host[v >> 6] >> (v & 63)) & 1ull); }
};

struct dg_exchange {
  dg_graph* h = nullptr;
  uint32_t rank = 0, world = 1;
  uint64_t capacity = 0;
  char* base = nullptr;          // this rank's buffers (one cudaMalloc: IPC-exportable)
  size_t bytes = 0;
  void* peer_base[kMaxPeers] = {};  // opened IPC mappings (nullptr for self / not set)
  PeerBuffers pb{};
  uint64_t epoch = 0;            // rounds completed; the current round uses buffer set epoch & 1
  int set() const { return (int)(epoch & 1); }
};

namespace {

int fail(dg_graph* h, int code, const std::string& msg) {
  if (h) h->last_error = msg; else g_create_error = msg;
  return code;
}

#define DG_CUDA(h, expr)                                                              \
  do {                                                                                \
    cudaError_t e__ = (expr);                                                         \
    if (e__ != cudaSuccess)                                                           \
      return fail((h), DG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

cudaEvent_t prof_event(dg_graph* h) {
  if (!h->prof_pool.empty()) {
    cudaEvent_t e = h->prof_pool.back();
    h->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct ProfScope {
  dg_graph* h;
  ProfScope(dg_graph* h_, const char* name) : h(h_) {
    if (!h->profiling) return;
    dg_graph::ProfSpan sp{name, prof_event(h), prof_event(h)};
    cudaEventRecord(sp.a, h->stream);
    h->prof_open.push_back(sp);
  }
  ~ProfScope() {
    if (!h->profiling) return;
    cudaEventRecord(h->prof_open.back().b, h->stream);
  }
};
// call after the stream is synchronised
void prof_collect(dg_graph* h) {
  for (auto& sp : h->prof_open) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess) {
      auto& acc = h->prof_acc[sp.name];
      acc.first += ms;
      acc.second += 1;
    }
    h->prof_pool.push_back(sp.a);
    h->prof_pool.push_back(sp.b);
  }
  h->prof_open.clear();
  cudaGetLastError();
}
void tl_mark(dg_graph* h, const char* name, cudaStream_t s) {
  if (!h->timeline) return;
  cudaEvent_t e = prof_event(h);
  cudaEventRecord(e, s);
  h->tl_marks.push_back({name, e});
}
void tl_report(dg_graph* h) {   // after the op's final synchronise
  if (!h->timeline || h->tl_marks.empty()) return;
  std::string line = "[timeline us]";
  for (size_t i = 1; i < h->tl_marks.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->tl_marks[0].ev, h->tl_marks[i].ev);
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s=%.1f", h->tl_marks[i].name, ms * 1e3);
    line += buf;
  }
  std::fprintf(stderr, "%s\n", line.c_str());
  for (auto& m : h->tl_marks) h->prof_pool.push_back(m.ev);
  h->tl_marks.clear();
  cudaGetLastError();
}
#define DG_LAUNCH(h, name, ...)                                                   \
  do {                                                                            \
    if (!(h)->ws_overflow) {                                                      \
      ProfScope ps__((h), (name));                                                \
      __VA_ARGS__;                                                                \
      const cudaError_t le__ = cudaPeekAtLastError();                             \
      if (le__ != cudaSuccess && (h)->launch_error == cudaSuccess) {              \
        (h)->launch_error = le__;                                                 \
        std::fprintf(stderr, "dyngraph_b200: launch of %s failed: %s\n", (name), cudaGetErrorString(le__)); \
      }                                                                           \
      (h)->launches += 1;                                                         \
    }                                                                             \
  } while (0)

GraphView view(const dg_graph* h) {
  GraphView g;
  g.head = h->head;
  g.tail = h->tail;
  g.deg = h->deg;
  g.alive = h->alive;
  g.slab = h->slab;
  g.next = h->next;
  g.ring = h->ring;
  g.ring_cap = h->NB;
  g.ring_identity = h->ring_identity;
  g.B = h->B;
  g.bsh = (h->B != 0 && (h->B & (h->B - 1)) == 0) ? (int)std::countr_zero(h->B) : -1;
  g.mw = (h->B + 31) / 32;
  g.size = (uint32_t)h->size;
  g.dst_limit = (uint32_t)std::min<uint64_t>(h->dst_limit(), 0xFFFFFFFFull);
  g.reclaim = h->reclaim;
  g.st = h->d_state();
  return g;
}

// ---- workspace ----------------------------------------------------------
int ws_reserve(dg_graph* h, size_t bytes) {
  h->ws.off = 0;
  if (bytes <= h->ws.cap) return DG_OK;
  DG_CUDA(h, cudaStreamSynchronize(h->stream));
  if (h->ws.base) cudaFree(h->ws.base);
  h->ws.base = nullptr;
  h->ws.cap = 0;
  const size_t want = bytes + bytes / 4;
  cudaError_t e = cudaMalloc(&h->ws.base, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    e = cudaMalloc(&h->ws.base, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(h, DG_ERR_ENGINE, "workspace: cannot allocate " + std::to_string(bytes) + " bytes");
    }
    h->ws.cap = bytes;
  } else {
    h->ws.cap = want;
  }
  return DG_OK;
}

template <class T>
T* ws_alloc(dg_graph* h, size_t count) {
  const size_t bytes = aligned(count * sizeof(T));
  T* p = reinterpret_cast<T*>(h->ws.base + h->ws.off);
  h->ws.off += bytes;
  if (h->ws.off > h->ws.cap) {
    // Sizing bug.  Never hand out memory past the reservation: the request aliases the start of the workspace,
    // the op is poisoned on the device (every kernel of an op starts with `if (op->err) return`), launches are
    // skipped from here on and op_end reports an engine error.
    if (!h->ws_overflow) {
      std::fprintf(stderr, "dyngraph_b200: workspace overflow (%zu > %zu): rejecting the op\n", h->ws.off, h->ws.cap);
      cudaMemsetAsync(&h->d_op()->err, 0x03, sizeof(uint32_t), h->stream);
      for (int i = 0; i < 2; ++i)
        if (h->aux[i]) cudaMemsetAsync(&h->d_op()->err, 0x03, sizeof(uint32_t), h->aux[i]);
    }
    h->ws_overflow = true;
    h->ws.off = bytes;
    return reinterpret_cast<T*>(h->ws.base);
  }
  return p;
}

struct WsSizer {
  size_t total = 0;
  template <class T>
  void add(size_t count) { total += aligned(count * sizeof(T)); }
};

// the op's validation / plan status is agreed with the peers before anything mutates (see exchange_agree_kernel)
void enqueue_agree(dg_graph* h, bool commit_insert) {
  dg_exchange* x = h->agree_x;
  if (x == nullptr) return;
  DG_LAUNCH(h, "exchange_agree_kernel", exchange_agree_kernel<<<1, 32, 0, h->stream>>>(x->pb, x->set(), h->d_op(), h->d_state(),
                                                                                      commit_insert ? 1 : 0));
}

inline int grid_for(const dg_graph* h, uint64_t items, int per_block) {
  const uint64_t want = (items + per_block - 1) / per_block;
  const uint64_t cap = (uint64_t)h->sm_count * 8;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, cap));
}

// Grid of a grid-stride kernel: enough CTAs for the work, never more than are RESIDENT at once
// (148 SMs x the kernel's occupancy): a partial second wave only adds a tail.
template <class K>
int resident_ctas_per_sm(K kernel, int block_threads, size_t dyn_smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), block_threads, dyn_smem, dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block_threads, dyn_smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  cache[key] = n;
  return n;
}
template <class K>
int grid_resident(const dg_graph* h, uint64_t items, int per_block, K kernel, int block_threads = 256, size_t dyn_smem = 0) {
  const uint64_t want = (items + per_block - 1) / per_block;
  const uint64_t cap = (uint64_t)h->sm_count * resident_ctas_per_sm(kernel, block_threads, dyn_smem);
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, cap));
}

// ---- fork / join of independent kernels ------------------------------------------
// Between fork() and join() lane(h, i) names stream i of {op stream, aux 0, aux 1}.
// With per-kernel profiling on, everything stays on the op stream so the event
// brackets keep measuring single kernels.
void fork(dg_graph* h) {
  if (h->profiling || h->aux[0] == nullptr) return;
  cudaEventRecord(h->ev_fork, h->stream);
  cudaStreamWaitEvent(h->aux[0], h->ev_fork, 0);
  cudaStreamWaitEvent(h->aux[1], h->ev_fork, 0);
  h->forked = true;
}
inline cudaStream_t lane(const dg_graph* h, int i) { return (h->forked && i > 0) ? h->aux[i - 1] : h->stream; }
void join(dg_graph* h) {
  if (!h->forked) return;
  for (int i = 0; i < 2; ++i) {
    cudaEventRecord(h->ev_join[i], h->aux[i]);
    cudaStreamWaitEvent(h->stream, h->ev_join[i], 0);
  }
  h->forked = false;
}

constexpr size_t kZAllocSlots = 8;
constexpr size_t kZScratchWords = kZAllocSlots * kAllocScratchWords + (size_t)kTallyStripes * kTalWords;
inline unsigned long long* tally_buf(const dg_graph* h) { return h->zscratch + kZAllocSlots * kAllocScratchWords; }

// the counting group-by's counter array: persistent, zero between ops (see dg_graph::cnt_buf)
inline uint64_t cnt_words_for(const dg_graph* h) { return std::bit_ceil(std::max<uint64_t>(h->size, 1)) + 4; }
// (re)allocates for the current vertex count: call before the op's workspace is laid out
int ensure_cnt(dg_graph* h) {
  const uint64_t words = cnt_words_for(h);
  if (words > h->cnt_cap) {
    DG_CUDA(h, cudaStreamSynchronize(h->stream));
    if (h->cnt_buf) cudaFree(h->cnt_buf);
    h->cnt_buf = nullptr;
    h->cnt_cap = 0;
    if (cudaMalloc(&h->cnt_buf, words * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(h, DG_ERR_ENGINE, "group-by counters: device allocation failed");
    }
    h->cnt_cap = words;
    h->cnt_clean = false;
  }
  return DG_OK;
}
// hands out the counters, all zero; `self_cleaning`: the op resets every word it touches (its success keeps the flag)
uint32_t* acquire_cnt(dg_graph* h, bool self_cleaning) {
  if (!h->cnt_clean) cudaMemsetAsync(h->cnt_buf, 0, h->cnt_cap * 4, h->stream);
  h->cnt_clean = self_cleaning;   // (op_end clears the flag when the op is rejected)
  return h->cnt_buf;
}

// ---- op bracket -----------------------------------------------------------
constexpr uint32_t kStatusSlots = 8;   // pinned {DeviceState, OpState} slots: at most kStatusSlots - 1 submitted ops in flight
int retire_oldest(dg_graph* h, bool wait);

int op_begin(dg_graph* h, uint64_t n_input, uint64_t n_runs) {
  // a slot of the pinned status ring nobody is still waiting on
  while (h->pending.size() >= kStatusSlots - 1) {
    const int rc = retire_oldest(h, /*wait=*/true);
    if (rc != DG_OK) return rc;
  }
  h->h_blk = &h->h_ring[h->h_ring_next++ % kStatusSlots];
  OpState& op = h->h_blk->op;
  std::memset(&op, 0, sizeof(op));
  op.err_index = ~0ull;
  op.bad_index = ~0ull;
  op.n_runs = n_runs;
  op.aux1 = 0;
  op.n_input = n_input;  // device-resident copy of the input length for scans
  op.n_aux = h->size + 1;
  tl_mark(h, "begin", h->stream);
  h->early_possible = false;   // (set again by a submitted counting-path insert once its plan is enqueued)
  if (h->submitting) {
    // the op words are installed by a kernel that first looks at what the previous submitted op left behind
    const OpState* pre = nullptr;
    if (h->early.active) {   // this op's group_count already ran on the side stream: its verdict first
      DG_CUDA(h, cudaStreamWaitEvent(h->stream, h->ev_early, 0));
      pre = h->early.pre;
    }
    op_arm_kernel<<<1, 1, 0, h->stream>>>(op, h->d_state(), h->d_op(), h->pending.empty() ? 0 : 1, pre);
    DG_CUDA(h, cudaPeekAtLastError());
  } else {
    // (the same kernel for synchronous ops: the words travel as its argument — no host-to-device copy that would
    // queue behind batch copies on the copy engine; nothing is in flight, so nothing to look at: chain = 0)
    op_arm_kernel<<<1, 1, 0, h->stream>>>(op, h->d_state(), h->d_op(), 0, nullptr);
    DG_CUDA(h, cudaPeekAtLastError());
  }
  h->launches = h->submitting ? (h->early.active ? 3 : 1) : 0;   // (op_arm_kernel; early: + op_pre_arm_kernel, group_count_kernel)
  h->zslot = 0;
  if (!h->zscratch_clean) {
    DG_CUDA(h, cudaMemsetAsync(h->zscratch, 0, kZScratchWords * sizeof(unsigned long long), h->stream));
    h->zscratch_clean = true;
  }
  h->report = dg_op_report{};
  h->report.batch_entries = n_input;
  return DG_OK;
}
inline const unsigned long long* d_n_input(const dg_graph* h) { return &h->d_op()->n_input; }
inline const unsigned long long* d_n_runs(const dg_graph* h) { return &h->d_op()->n_runs; }
inline const unsigned long long* d_n_aux(const dg_graph* h) { return &h->d_op()->n_aux; }

const char* detail_text(uint32_t d) {
  switch (d) {
    case kErrSrcRange: return "source id out of range";
    case kErrDstRange: return "destination out of range";
    case kErrDeadSource: return "insert lists edges for retired vertex";
    case kErrOffsetsStart: return "offsets[0] must be 0";
    case kErrOffsetsMonotone: return "offsets are not monotone";
    case kErrOffsetsEnd: return "destinations length does not match offsets";
    case kErrPoolUnderflow: return "batch needs more blocks than the pool can still provide";
    case kErrScratch: return "internal scratch exhausted";
    case kErrPeer: return "rejected on another rank of the sharded store (nothing was applied on any rank)";
    default: return "unknown";
  }
}

// the host-side conclusion of an op from its status slot: mirrors, report, device-side error
int op_conclude(dg_graph* h, const DevBlock& blk, uint64_t n_input, uint64_t launches) {
  const DeviceState& st = blk.st;
  const OpState& op = blk.op;
  h->report = dg_op_report{};
  h->report.batch_entries = n_input;
  h->report.touched_sources = op.n_runs;
  h->report.blocks_popped = op.total_need;
  h->report.blocks_pushed = op.pushed;
  h->report.slots_scanned = op.slots;
  h->report.blocks_scanned = op.wl_blocks + op.fused_blocks;
  h->report.slots_scanned_fused = op.slots_fused;
  h->report.matched = op.matched;
  h->report.moved = op.moves;
  h->report.kernel_launches = launches;
  h->report.slots_scanned_long = op.slots_long;
  h->report.slots_scanned_tiny = op.slots_tiny;
  h->front = st.front;
  h->rear = st.rear;
  h->active_edges = st.active_edges;
  if (op.err != 0) {
    h->zscratch_clean = false;   // kernels of a rejected op return early: cursors / tallies may be left behind
    h->cnt_clean = false;
    h->report.blocks_popped = 0;
    if (op.err_detail == kErrPoolUnderflow) h->last_shortfall = op.err_index;
    if (op.err_detail == kErrSkipped)
      return fail(h, (int)op.err, "not applied: an op submitted before this one failed");
    return fail(h, (int)op.err,
                std::string(op.err == DG_ERR_DATA ? "csr batch: " : "block pool: ") +
                    detail_text(op.err_detail) + " (index " + std::to_string(op.err_index) + ")");
  }
  h->total_capacity += op.pushed;   // every re-push counts (block_pool.hpp:56-61)
  return DG_OK;
}

// read back {DeviceState, OpState}; translate a device-side error.  A submitted op only enqueues the read-back
// (into its own pinned slot) and an event: its status is looked at when it is retired.
int op_end(dg_graph* h) {
  tl_mark(h, "end", h->stream);
  h->early.active = false;
  static_assert(sizeof(DevBlock) % 8 == 0, "status words");
  if (h->h_ring_dev != nullptr) {   // stores into the mapped slot (see op_publish_kernel)
    unsigned long long* slot_dev = reinterpret_cast<unsigned long long*>(h->h_ring_dev + (h->h_blk - h->h_ring));
    op_publish_kernel<<<1, 32, 0, h->stream>>>(reinterpret_cast<const unsigned long long*>(h->d_blk), slot_dev,
                                               (int)(sizeof(DevBlock) / 8));
    DG_CUDA(h, cudaPeekAtLastError());
  } else {
    DG_CUDA(h, cudaMemcpyAsync(h->h_blk, h->d_blk, sizeof(DevBlock), cudaMemcpyDeviceToHost, h->stream));
  }
  if (h->submitting && h->launch_error == cudaSuccess && !h->ws_overflow) {
    cudaEvent_t ev = nullptr;
    if (!h->done_pool.empty()) {
      ev = h->done_pool.back();
      h->done_pool.pop_back();
    } else {
      DG_CUDA(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    DG_CUDA(h, cudaEventRecord(ev, h->stream));
    h->pending.push_back(dg_graph::Pending{h->next_ticket++, h->submit_is_insert, h->submit_pop_bound, h->h_blk, ev,
                                           h->launches, h->report.batch_entries});
    h->pending_pop_bound += h->submit_pop_bound;
    return DG_OK;
  }
  DG_CUDA(h, cudaStreamSynchronize(h->stream));
  DG_CUDA(h, cudaGetLastError());
  if (h->profiling) prof_collect(h);
  tl_report(h);
  if (h->launch_error != cudaSuccess) {
    const cudaError_t e = h->launch_error;
    h->launch_error = cudaSuccess;
    h->zscratch_clean = h->cnt_clean = false;
    return fail(h, DG_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
  }
  if (h->ws_overflow) {   // (the op was poisoned on the device before anything mutated: see ws_alloc)
    h->ws_overflow = false;
    h->zscratch_clean = h->cnt_clean = false;
    return fail(h, DG_ERR_ENGINE, "internal: per-op workspace was sized too small; the batch was not applied");
  }
  return op_conclude(h, *h->h_blk, h->report.batch_entries, h->launches);
}

// ---- submitted ops: retire / drain ---------------------------------------------------------------
// Looks at the oldest submitted op (waiting for it when `wait`): folds its outcome into the host mirrors, or
// records the pipeline's first failure (returned once, by dg_flush or by the next synchronous call).
// Returns DG_OK when an op was retired or nothing is ready; DG_ERR_CUDA on a runtime error.
int retire_oldest(dg_graph* h, bool wait) {
  if (h->pending.empty()) return DG_OK;
  dg_graph::Pending p = h->pending.front();
  if (wait) {
    DG_CUDA(h, cudaEventSynchronize(p.done));
  } else {
    const cudaError_t q = cudaEventQuery(p.done);
    if (q == cudaErrorNotReady) {
      cudaGetLastError();   // (not an error: keep it out of the launch-error checks)
      return DG_OK;
    }
    DG_CUDA(h, q);
  }
  h->pending.pop_front();
  h->pending_pop_bound -= p.pop_bound;
  h->done_pool.push_back(p.done);
  if (h->deferred_rc != DG_OK) return DG_OK;   // (queued behind the failure: skipped on the device, nothing to fold in)
  const std::string keep = h->last_error;
  const int rc = op_conclude(h, *p.slot, p.n, p.launches);
  if (rc == DG_OK) {
    ++h->submitted_applied;
    if (p.is_insert) h->consumed += h->report.blocks_popped;   // (submit made sure this stays below the growth trigger)
    h->last_error = keep;
  } else {
    h->deferred_rc = rc;
    h->deferred_ticket = p.ticket;
    h->deferred_error = "submitted op #" + std::to_string(p.ticket) + " failed: " + h->last_error +
                        "; ops submitted after it were not applied";
    h->last_error = keep;
  }
  return DG_OK;
}
// waits for every submitted op
int drain(dg_graph* h) {
  while (!h->pending.empty()) {
    const int rc = retire_oldest(h, /*wait=*/true);
    if (rc != DG_OK) return rc;
  }
  return DG_OK;
}
// returns (once) the failure of a submitted op
int take_deferred(dg_graph* h) {
  if (h->deferred_rc == DG_OK) return DG_OK;
  const int rc = h->deferred_rc;
  h->last_error = h->deferred_error;
  h->deferred_rc = DG_OK;
  h->deferred_error.clear();
  return rc;
}
// Every synchronous entry point starts here: nothing submitted is left in flight, and an unreported failure of
// a submitted op is returned INSTEAD of running the call (the caller learns about it before anything else mutates).
int enter(dg_graph* h) {
  cudaSetDevice(h->device);
  if (h->pending.empty() && h->deferred_rc == DG_OK) return DG_OK;
  const int rc = drain(h);
  if (rc != DG_OK) return rc;
  return take_deferred(h);
}
// accessors that cannot return a status: drained state, the failure (if any) stays for the next status call
void enter_quiet(const dg_graph* ch) {
  dg_graph* h = const_cast<dg_graph*>(ch);
  if (h->pending.empty()) return;
  cudaSetDevice(h->device);
  drain(h);
}

// ---- scan / sort launchers -------------------------------------------------
template <class In, class Out, class Fin>
void launch_scan(dg_graph* h, const char* name, uint64_t n_bound, const unsigned long long* n_ptr,
                 In in, Out out, Fin fin, cudaStream_t stream = nullptr) {
  if (stream == nullptr) stream = h->stream;
  const size_t words = scan_scratch_words(n_bound);
  unsigned long long* scratch = ws_alloc<unsigned long long>(h, words);
  cudaMemsetAsync(scratch, 0, words * sizeof(unsigned long long), stream);
  const unsigned tiles = (unsigned)std::max<uint64_t>(1, (n_bound + kScanTile - 1) / kScanTile);
  DG_LAUNCH(h, name, scan_kernel<<<tiles, kScanThreads, 0, stream>>>(n_ptr, scratch, h->d_op(), in, out, fin));
}
// unordered range allocation over [0, *n_ptr): see alloc_kernel
template <class In, class Out, class Fin>
void launch_alloc(dg_graph* h, const char* name, uint64_t n_bound, const unsigned long long* n_ptr,
                  In in, Out out, Fin fin, cudaStream_t stream = nullptr) {
  if (stream == nullptr) stream = h->stream;
  // cursors: a slot of the persistent zeroed scratch (the kernel's last tile hands it back zeroed)
  unsigned long long* scratch = h->zscratch + (size_t)(h->zslot++ % kZAllocSlots) * kAllocScratchWords;
  if (n_bound > (2u << 20)) {
    constexpr int kTile = kAllocThreads * kAllocItemsLarge;
    const unsigned tiles = (unsigned)((n_bound + kTile - 1) / kTile);
    DG_LAUNCH(h, name, alloc_kernel<kAllocItemsLarge><<<tiles, kAllocThreads, 0, stream>>>(n_ptr, scratch, h->d_op(), in, out, fin));
  } else {
    constexpr int kTile = kAllocThreads * kAllocItemsSmall;
    const unsigned tiles = (unsigned)std::max<uint64_t>(1, (n_bound + kTile - 1) / kTile);
    DG_LAUNCH(h, name, alloc_kernel<kAllocItemsSmall><<<tiles, kAllocThreads, 0, stream>>>(n_ptr, scratch, h->d_op(), in, out, fin));
  }
}
inline size_t alloc_ws_bytes() { return aligned(kAllocScratchWords * sizeof(unsigned long long)); }
inline size_t scan_ws_bytes(uint64_t n_bound) {
  return aligned(scan_scratch_words(n_bound) * sizeof(unsigned long long));
}

SortPlan make_sort_plan(int lo_bits, int hi_bits) {
  // digits over key bits [0, lo_bits) then [32, 32 + hi_bits), LSD order
  SortPlan p{};
  p.passes = 0;
  auto add = [&](int base, int nbits) {
    int done = 0;
    while (done < nbits) {
      const int take = std::min(8, nbits - done);
      p.shift[p.passes] = base + done;
      p.bits[p.passes] = take;
      ++p.passes;
      done += take;
    }
  };
  add(0, lo_bits);
  add(32, hi_bits);
  return p;
}

inline size_t sort_ws_bytes(uint64_t n, int passes) {
  return aligned((size_t)kMaxPasses * kRadix * sizeof(unsigned int)) +
         aligned((size_t)std::max(passes, 1) * (2 + sort_tiles(std::max<uint64_t>(n, 1)) * kRadix) * sizeof(unsigned long long));
}

// Sort scratch: per-pass raw digit histograms + per-pass look-back status.
struct SortScratch {
  unsigned int* hist;
  unsigned long long* status;
  size_t per_pass;
};
// Allocates and zeroes the scratch (before the kernel that fills the histograms).
SortScratch sort_prepare(dg_graph* h, uint64_t n, const SortPlan& plan) {
  SortScratch sc{};
  sc.per_pass = 2 + sort_tiles(std::max<uint64_t>(n, 1)) * kRadix;
  sc.hist = ws_alloc<unsigned int>(h, (size_t)kMaxPasses * kRadix);
  sc.status = ws_alloc<unsigned long long>(h, (size_t)std::max(plan.passes, 1) * sc.per_pass);
  cudaMemsetAsync(sc.hist, 0, (size_t)kMaxPasses * kRadix * sizeof(unsigned int), h->stream);
  cudaMemsetAsync(sc.status, 0, (size_t)std::max(plan.passes, 1) * sc.per_pass * sizeof(unsigned long long), h->stream);
  return sc;
}
// Sorts keys (and values) through the passes of `plan`; *keys/*vals end up
// pointing at the buffer holding the sorted data (a or b).  hist_done: the
// producer of the keys already accumulated the histograms into sc.hist.
void sort_keys(dg_graph* h, unsigned long long** keys, unsigned long long** keys_alt,
               uint32_t** vals, uint32_t** vals_alt, uint64_t n, const SortPlan& plan,
               const SortScratch& sc, bool hist_done) {
  if (plan.passes == 0 || n == 0) return;
  if (!hist_done)
    DG_LAUNCH(h, "sort_hist_kernel", sort_hist_kernel<<<grid_for(h, n, 256 * 8), 256, 0, h->stream>>>(*keys, n, plan, sc.hist, h->d_op()));
  const unsigned tiles = (unsigned)sort_tiles(n);
  cudaFuncSetAttribute(sort_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSortSmemKeysVals);
  cudaFuncSetAttribute(sort_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSortSmemKeys);
  for (int p = 0; p < plan.passes; ++p) {
    if (vals && *vals) {
      DG_LAUNCH(h, "sort_pass_kernel<true>", sort_pass_kernel<true><<<tiles, kSortThreads, kSortSmemKeysVals, h->stream>>>(
          *keys, *keys_alt, *vals, *vals_alt, n, plan.shift[p], plan.bits[p], sc.hist + p * kRadix,
          sc.status + (size_t)p * sc.per_pass, h->d_op()));
      std::swap(*vals, *vals_alt);
    } else {
      DG_LAUNCH(h, "sort_pass_kernel<false>", sort_pass_kernel<false><<<tiles, kSortThreads, kSortSmemKeys, h->stream>>>(
          *keys, *keys_alt, nullptr, nullptr, n, plan.shift[p], plan.bits[p], sc.hist + p * kRadix,
          sc.status + (size_t)p * sc.per_pass, h->d_op()));
    }
    std::swap(*keys, *keys_alt);
  }
}

inline int bits_for(uint64_t max_value) { return max_value == 0 ? 0 : (int)std::bit_width(max_value); }
// sort plan of the batch ops: group by source only (no order needed among a source's targets)
inline SortPlan src_sort_plan(const dg_graph* h, uint64_t max_src) { return make_sort_plan(0, bits_for(max_src)); }


// ---- pool ---------------------------------------------------------------------
int create_pool(dg_graph* h, uint32_t B) {
  if (B == 0) return fail(h, DG_ERR_DATA, "block pool: block size must be >= 1");
  const uint64_t per_block = (uint64_t)B * 4 + 8;  // slab + next link + ring slot
  uint64_t nb = h->cfg.pool_blocks ? h->cfg.pool_blocks
                                   : (h->cfg.pool_bytes ? h->cfg.pool_bytes : (1ull << 30)) / per_block;
  if (nb == 0) return fail(h, DG_ERR_ENGINE, "block pool: arena cannot host a single edge block");
  if (nb >= (1ull << 31)) nb = (1ull << 31) - 1;
  h->nb_max = std::min<uint64_t>(h->cfg.pool_max_blocks, (1ull << 31) - 1);
  cudaError_t e = cudaSuccess;
  if (h->nb_max > nb) {
    // growing pool: reserve the address range of the largest pool, commit the initial part
    const bool ok = h->vm_slab.reserve(h->device, h->nb_max * B * sizeof(uint32_t)) && h->vm_slab.commit(nb * B * sizeof(uint32_t)) &&
                    h->vm_next.reserve(h->device, h->nb_max * sizeof(uint32_t)) && h->vm_next.commit(nb * sizeof(uint32_t));
    if (!ok) {
      h->vm_slab.destroy();
      h->vm_next.destroy();
      return fail(h, DG_ERR_ENGINE, "block pool: cannot reserve / commit device memory for a growing pool");
    }
    h->pool_vm = true;
    h->slab = reinterpret_cast<uint32_t*>(h->vm_slab.base);
    h->next = reinterpret_cast<uint32_t*>(h->vm_next.base);
    if ((e = cudaMalloc(&h->ring, nb * sizeof(uint32_t))) != cudaSuccess) {
      cudaGetLastError();
      h->vm_slab.destroy();
      h->vm_next.destroy();
      h->slab = h->next = nullptr;
      h->pool_vm = false;
      return fail(h, DG_ERR_ENGINE, std::string("block pool: device allocation failed: ") + cudaGetErrorString(e));
    }
  } else if ((e = cudaMalloc(&h->slab, nb * B * sizeof(uint32_t))) != cudaSuccess ||
      (e = cudaMalloc(&h->next, nb * sizeof(uint32_t))) != cudaSuccess ||
      (e = cudaMalloc(&h->ring, nb * sizeof(uint32_t))) != cudaSuccess) {
    cudaGetLastError();
    if (h->slab) cudaFree(h->slab);
    if (h->next) cudaFree(h->next);
    h->slab = h->next = h->ring = nullptr;
    return fail(h, DG_ERR_ENGINE, std::string("block pool: device allocation failed: ") + cudaGetErrorString(e));
  }
  h->ring_identity = nb;
  h->B = B;
  h->NB = nb;
  h->total_capacity = nb;
  DG_LAUNCH(h, "ring_fill_kernel", ring_fill_kernel<<<grid_for(h, nb, 256 * 4), 256, 0, h->stream>>>(h->ring, nb));
  DG_CUDA(h, cudaMemsetAsync(h->next, 0xFF, nb * sizeof(uint32_t), h->stream));
  h->h_blk->st.front = 0;
  h->h_blk->st.rear = nb;
  h->h_blk->st.active_edges = h->active_edges;
  h->h_blk->st.poison = 0;
  DG_CUDA(h, cudaMemcpyAsync(h->d_state(), &h->h_blk->st, sizeof(DeviceState), cudaMemcpyHostToDevice, h->stream));
  DG_CUDA(h, cudaStreamSynchronize(h->stream));
  h->front = 0;
  h->rear = nb;
  return DG_OK;
}

// One growth round (try_grow, block_pool.hpp:252-264): growth_fraction of the capacity, clamped to
// what the budget still allows.  Returns false when the pool cannot grow any further.
bool try_grow(dg_graph* h) {
  if (!h->pool_vm || h->NB >= h->nb_max) return false;
  uint64_t want = (uint64_t)((double)h->total_capacity * h->growth);   // block_pool.hpp:253-254
  if (want == 0) want = 1;
  const uint64_t grant = std::min<uint64_t>(want, h->nb_max - h->NB);
  const uint64_t nb_new = h->NB + grant;
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return false;
  if (!h->vm_slab.commit(nb_new * h->B * sizeof(uint32_t)) || !h->vm_next.commit(nb_new * sizeof(uint32_t))) return false;
  uint32_t* ring_new = nullptr;
  if (cudaMalloc(&ring_new, nb_new * sizeof(uint32_t)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  ring_relayout_kernel<<<grid_for(h, (h->rear - h->front) + grant, 256), 256, 0, h->stream>>>(
      h->ring, h->NB, ring_new, nb_new, h->front, h->rear, (uint32_t)h->NB, grant);
  cudaMemsetAsync(h->next + h->NB, 0xFF, grant * sizeof(uint32_t), h->stream);
  if (h->rear == h->ring_identity) h->ring_identity += grant;   // nothing was ever recycled: still a bump allocator
  h->rear += grant;
  h->h_blk->st.front = h->front;
  h->h_blk->st.rear = h->rear;
  h->h_blk->st.active_edges = h->active_edges;
  cudaMemcpyAsync(h->d_state(), &h->h_blk->st, sizeof(DeviceState), cudaMemcpyHostToDevice, h->stream);
  cudaStreamSynchronize(h->stream);
  cudaFree(h->ring);
  h->ring = ring_new;
  h->NB = nb_new;
  h->total_capacity += grant;
  ++h->growth_count;
  return cudaGetLastError() == cudaSuccess;
}

// commit_front's growth rule (block_pool.hpp:162-172): after a batch popped `popped` blocks, grow
// once if cumulative consumption reached trigger_fraction of the capacity.
void after_pop(dg_graph* h, uint64_t popped) {
  h->consumed += popped;   // occupancy() = consumed / total_capacity (block_pool.hpp:168-172)
  if (h->pool_vm && h->total_capacity > 0 && (double)h->consumed / (double)h->total_capacity >= h->trigger) try_grow(h);
}

// ensure_available (block_pool.hpp:177-189) for a batch that was rejected for `shortfall` missing
// blocks: grows until the queue covers it; false (nothing changed) when the budget cannot.
bool grow_for_shortfall(dg_graph* h, uint64_t shortfall) {
  if (!h->pool_vm || h->nb_max - h->NB < shortfall) return false;
  const uint64_t target = (h->rear - h->front) + shortfall;
  while (h->rear - h->front < target)
    if (!try_grow(h)) return false;
  return true;
}

// ensure_available + commit_front around an insert (block_pool.hpp:162-189): a batch rejected for a
// pool underflow left the graph untouched, so when the growth budget covers the shortfall the pool
// grows and the batch runs again; after a successful batch the trigger rule may grow the pool.
template <class F>
int insert_with_growth(dg_graph* h, F&& run) {
  int rc = run();
  if (!h) return rc;
  if (rc == DG_ERR_ENGINE && h->last_shortfall != 0 && grow_for_shortfall(h, h->last_shortfall)) {
    // sharded store: every rank rejected the batch together (device-side agreement) — the pool has grown,
    // the caller repeats the batch on every rank; a lone retry here would wait for peers that never come
    if (h->agree_x == nullptr) rc = run();
  }
  if (rc == DG_OK) after_pop(h, h->report.blocks_popped);
  return rc;
}

// Stage a caller array on the device if it lives on the host.
template <class T>
int stage_in(dg_graph* h, const T* p, uint64_t count, int mem, const T** out) {
  if (mem == DG_MEM_DEVICE || count == 0) {
    *out = p;
    return DG_OK;
  }
  T* d = ws_alloc<T>(h, count);
  DG_CUDA(h, cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, h->stream));
  *out = d;
  return DG_OK;
}

// ---- shared pieces of the batch ops ---------------------------------------------
// upper bound of append units: every non-empty run has at most 1 + ceil(c / B) of them
inline uint64_t units_bound(uint32_t B, uint64_t runs_bound, uint64_t n_edges) {
  return 2 * std::min<uint64_t>(runs_bound, n_edges) + n_edges / std::max<uint32_t>(B, 1) + 1;
}

// per-run outputs of the insert plan
PlanArrays alloc_plan_arrays(dg_graph* h, uint64_t runs_bound, uint64_t n_edges) {
  PlanArrays a{};
  a.run_deg = ws_alloc<uint32_t>(h, runs_bound + 1);
  a.run_tail = ws_alloc<uint32_t>(h, runs_bound + 1);
  a.unit_off = ws_alloc<uint32_t>(h, runs_bound + 1);
  a.blk_off = ws_alloc<uint32_t>(h, runs_bound + 1);
  a.unit_run = ws_alloc<uint32_t>(h, units_bound(h->B, runs_bound, n_edges));
  return a;
}
inline size_t plan_arrays_ws(uint32_t B, uint64_t runs_bound, uint64_t n_edges) {
  return 4 * aligned((runs_bound + 1) * 4) + aligned(units_bound(B, runs_bound, n_edges) * 4) + alloc_ws_bytes();
}

// append over a planned batch.  csr_path: the destination range check rides in
// the append pass and the metadata commit is a separate kernel that only runs
// when nothing failed.
void enqueue_append(dg_graph* h, const BatchView& b, const PlanArrays& a, uint64_t runs_bound,
                    uint64_t n_edges, bool csr_path) {
  GraphView g = view(h);
  const int grid = grid_for(h, units_bound(h->B, runs_bound, n_edges), 8 * 32);
  if (csr_path) {
    DG_LAUNCH(h, "append_kernel<validate>", append_kernel<true, false><<<grid, 256, 0, h->stream>>>(
        g, b, a.unit_off, a.blk_off, a.unit_run, a.run_deg, a.run_tail, h->d_op()));
    DG_LAUNCH(h, "commit_insert_kernel", commit_insert_kernel<<<grid_for(h, runs_bound, 256), 256, 0, h->stream>>>(
        g, b, a.blk_off, a.run_deg, h->d_op()));
  } else {
    DG_LAUNCH(h, "append_kernel<commit>", append_kernel<false, true><<<grid, 256, 0, h->stream>>>(
        g, b, a.unit_off, a.blk_off, a.unit_run, a.run_deg, a.run_tail, h->d_op()));
  }
}

// plan + append over an already grouped batch (radix path: sorted keys + detected runs; CSR: offsets)
void enqueue_plan_append(dg_graph* h, const BatchView& b, uint64_t runs_bound, uint64_t n_edges,
                         bool csr_path) {
  GraphView g = view(h);
  PlanArrays a = alloc_plan_arrays(h, runs_bound, n_edges);
  const bool agree = !csr_path && h->agree_x != nullptr;   // sharded store: the commit waits for every rank's all-clear
  launch_alloc(h, "alloc_kernel<plan>", runs_bound, d_n_runs(h), PlanIn{g, b}, PlanOut{a},
               PlanFin{g, h->d_op(), n_edges, /*set_runs=*/0, (csr_path || agree) ? 0 : 1});
  if (agree) enqueue_agree(h, /*commit_insert=*/true);
  enqueue_append(h, b, a, runs_bound, n_edges, csr_path);
}

inline uint64_t big_bound(const dg_graph* h);

struct Worklist {
  uint32_t* wl_off;
  uint32_t* wl_handle;
  uint32_t* wl_run;
  uint32_t* run_deg;
  uint2* med_items;    // (run, chunk) items of the medium / long match tiers (nullptr without a batch)
  uint2* long_items;
  uint32_t* big_list;  // chains longer than kLaneWalk blocks
  uint32_t* run_head;  // fused delete only: head block of the warp-owned sources (else nullptr)
  uint4* fmed_rec;     // fused delete only: sources of the medium class (two words each)
  uint32_t* zero3;     // delete only: run_matched (+ two spare words per run), zeroed per run by the enumeration plan
  uint32_t zstride;
  EnumLists lists(dg_graph* h) const {
    return EnumLists{run_deg, wl_off, med_items, long_items, big_list, (uint32_t)big_bound(h), h->d_op(), run_head, fmed_rec,
                     zero3, zstride};
  }
};

// items: every run of a tier has at least one, plus one per full chunk of its chain
inline uint64_t med_items_bound(const dg_graph* h, uint64_t n) {
  return n / (kTinyTargets + 1) + h->blocks_in_use() / kMedChunk + 16;
}
inline uint64_t long_items_bound(const dg_graph* h, uint64_t n) {
  return n / (kMedTargets + 1) + h->blocks_in_use() / kLongChunk + 16;
}
inline uint64_t big_bound(const dg_graph* h) { return h->blocks_in_use() / (kLaneWalk + 1) + 16; }

// sources of the fused medium class: more than kFusedSmallBlocks blocks or more than kFusedSmallTargets targets
inline uint64_t fused_med_bound(const dg_graph* h, uint64_t runs_bound, uint64_t n_batch) {
  return std::min<uint64_t>(runs_bound, h->blocks_in_use() / (kFusedSmallBlocks + 1) + n_batch / (kFusedSmallTargets + 1) + 1) + 1;
}
// n_batch: entries of the batch the runs index into; has_batch false: export, digest
Worklist alloc_worklist(dg_graph* h, uint64_t runs_bound, uint64_t n_batch, bool has_batch, bool fuse = false,
                        bool for_delete = false) {
  Worklist w{};
  if (for_delete) {
    w.zero3 = ws_alloc<uint32_t>(h, 3 * (runs_bound + 1));
    w.zstride = (uint32_t)(runs_bound + 1);
  }
  if (fuse) {
    w.run_head = ws_alloc<uint32_t>(h, runs_bound + 1);
    w.fmed_rec = ws_alloc<uint4>(h, 2 * fused_med_bound(h, runs_bound, n_batch));
  }
  const uint64_t wl_cap = h->blocks_in_use();
  w.wl_off = ws_alloc<uint32_t>(h, runs_bound + 1);
  w.run_deg = ws_alloc<uint32_t>(h, runs_bound + 1);
  w.wl_handle = ws_alloc<uint32_t>(h, wl_cap + 1);
  w.wl_run = ws_alloc<uint32_t>(h, wl_cap + 1);
  if (has_batch) {
    w.med_items = ws_alloc<uint2>(h, med_items_bound(h, n_batch));
    w.long_items = ws_alloc<uint2>(h, long_items_bound(h, n_batch));
  }
  w.big_list = ws_alloc<uint32_t>(h, big_bound(h));
  return w;
}
inline size_t worklist_ws(const dg_graph* h, uint64_t runs_bound, uint64_t n_batch) {
  return 3 * aligned((runs_bound + 1) * 4) + aligned(fused_med_bound(h, runs_bound, n_batch) * 32) +
         2 * aligned((h->blocks_in_use() + 1) * 4) +
         aligned(med_items_bound(h, n_batch) * 8) + aligned(long_items_bound(h, n_batch) * 8) +
         aligned(big_bound(h) * 4) + alloc_ws_bytes();
}

// chain walk over a planned worklist
void enqueue_walk(dg_graph* h, const BatchView& b, const Worklist& w, uint64_t runs_bound, cudaStream_t s_big, cudaStream_t s_small) {
  GraphView g = view(h);
  // (the long-chain walk starts first, it is the critical path)
  DG_LAUNCH(h, "enumerate_big_kernel", enumerate_big_kernel<<<grid_resident(h, big_bound(h), 8, enumerate_big_kernel), 256, 0, s_big>>>(
      g, b, w.wl_off, w.run_deg, w.big_list, (uint32_t)big_bound(h), w.wl_handle, w.wl_run, h->d_op()));
  DG_LAUNCH(h, "enumerate_walk_kernel", enumerate_walk_kernel<<<grid_resident(h, runs_bound, 256, enumerate_walk_kernel), 256, 0, s_small>>>(
      g, b, w.wl_off, w.run_deg, w.wl_handle, w.wl_run, h->d_op()));
}
void enqueue_walk(dg_graph* h, const BatchView& b, const Worklist& w, uint64_t runs_bound) {   // inside a fork
  enqueue_walk(h, b, w, runs_bound, lane(h, 1), lane(h, 2));
}

// enumeration over an already grouped batch (radix path, CSR batches) or over every vertex (export)
Worklist enqueue_enumerate(dg_graph* h, const BatchView& b, uint64_t runs_bound, uint64_t n_batch,
                           int check_alive, bool fuse = false, bool walk = true, bool for_delete = false) {
  GraphView g = view(h);
  Worklist w = alloc_worklist(h, runs_bound, n_batch, b.run_start != nullptr, fuse, for_delete);
  launch_alloc(h, "alloc_kernel<enum>", runs_bound, d_n_runs(h), EnumIn{g, b, check_alive, fuse}, EnumOut{g, b, w.lists(h)},
               EnumFin{h->d_op(), h->blocks_in_use(), /*set_runs=*/0});
  if (!walk) return w;
  fork(h);
  enqueue_walk(h, b, w, runs_bound);
  join(h);
  return w;
}

// match over an enumerated worklist: three tiers by the number of targets per source.  kNative: B = 32
// (block size, mask words and the 16-byte staging are compile-time constants); otherwise the same kernels
// with 4-byte staging copies and ceil(B / 32) passes per block.
template <bool kIsDelete, bool kNative>
void enqueue_match_impl(dg_graph* h, const BatchView& b, const Worklist& w, uint64_t n_batch,
                        uint32_t* run_matched, uint32_t* wl_mask, uint8_t* hit, cudaStream_t s_long, cudaStream_t s_med,
                        cudaStream_t s_tiny) {
  GraphView g = view(h);
  const uint64_t wl_bound = std::max<uint64_t>(1, h->blocks_in_use());
  const size_t med_smem = kIsDelete ? kMedSmemDelete : kMedSmemQuery;
  const size_t long_smem = kIsDelete ? kLongSmemDelete : kLongSmemQuery;
  // opt in to > 48 KB of dynamic shared memory: once per device and instantiation (two host API calls per op otherwise)
  {
    static std::mutex mu;
    static std::unordered_set<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert(h->device).second) {
      cudaFuncSetAttribute(match_med_kernel<kIsDelete, kNative>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)med_smem);
      cudaFuncSetAttribute(match_long_kernel<kIsDelete, kNative>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)long_smem);
    }
  }
  // the tiers touch disjoint blocks: side by side, heaviest items first
  const int long_grid = (int)std::min<uint64_t>(long_items_bound(h, n_batch), (uint64_t)h->sm_count * 3);
  DG_LAUNCH(h, kIsDelete ? "match_long_kernel<delete>" : "match_long_kernel<query>",
            match_long_kernel<kIsDelete, kNative><<<long_grid, kLongThreads, long_smem, s_long>>>(
                g, b, w.wl_off, w.wl_handle, w.long_items, w.run_deg, run_matched, wl_mask, hit, h->d_op()));
  const int med_grid = (int)std::min<uint64_t>(grid_for(h, med_items_bound(h, n_batch), 8), (uint64_t)h->sm_count * 4);
  DG_LAUNCH(h, kIsDelete ? "match_med_kernel<delete>" : "match_med_kernel<query>",
            match_med_kernel<kIsDelete, kNative><<<med_grid, 256, med_smem, s_med>>>(
                g, b, w.wl_off, w.wl_handle, w.med_items, w.run_deg, run_matched, wl_mask, hit, h->d_op()));
  DG_LAUNCH(h, kIsDelete ? "match_tiny_kernel<delete>" : "match_tiny_kernel<query>",
            match_tiny_kernel<kIsDelete, kNative><<<grid_resident(h, wl_bound, 256, match_tiny_kernel<kIsDelete, kNative>), 256, 0, s_tiny>>>(
                g, b, w.wl_off, w.wl_handle, w.wl_run, w.run_deg, run_matched, wl_mask, hit, h->d_op()));
}
template <bool kIsDelete>
void enqueue_match(dg_graph* h, const BatchView& b, const Worklist& w, uint64_t n_batch,
                   uint32_t* run_matched, uint32_t* wl_mask, uint8_t* hit) {
  fork(h);
  if (h->B == 32) enqueue_match_impl<kIsDelete, true>(h, b, w, n_batch, run_matched, wl_mask, hit, lane(h, 1), lane(h, 2), lane(h, 0));
  else enqueue_match_impl<kIsDelete, false>(h, b, w, n_batch, run_matched, wl_mask, hit, lane(h, 1), lane(h, 2), lane(h, 0));
  join(h);
}

// ---- grouping a COO batch by source --------------------------------------------------------------
// Two strategies:
//   counting: per-vertex counters (validate + count), ONE alloc pass over the
//             vertices that hands out run slots and group slots TOGETHER WITH the
//             op's own plan (insert: append units + queue positions; delete/query:
//             work-list segments), then a scatter — O(V + n);
//   radix:    pack 64-bit keys, LSD radix sort by source, run detection, then the
//             op's plan as an alloc pass over the runs — O(n).
inline bool use_counting(const dg_graph* h, uint64_t n) {
  if (h->B == 0) return false;  // deferred pool: the plan needs the block size, which needs the run count first
  if (h->group_mode == 1) return false;
  if (h->group_mode == 2) return true;
  return h->size <= std::max<uint64_t>(64 * n, 1ull << 22);  // the counter array is cleared per batch
}

struct Grouped {
  BatchView b{};
  uint64_t runs_bound = 0;
  uint32_t* index = nullptr;  // original position of every grouped entry (queries)
  // counting path, between count and scatter
  GroupIndex gi{};
  uint64_t cnt_words = 0;
  uint32_t* cnt = nullptr;
  uint32_t* rank = nullptr;
  uint32_t* gdst = nullptr;
  uint32_t *run_src = nullptr, *run_start = nullptr, *run_end = nullptr;
};

inline size_t group_ws_bytes(const dg_graph* h, uint64_t n, bool with_index, uint64_t max_src, bool force_radix = false) {
  size_t t = 0;
  if (!force_radix && use_counting(h, n)) {
    t += aligned((std::bit_ceil(std::max<uint64_t>(h->size, 1)) + 4 + 4 * kAllocScratchWords) * 4) + 2 * aligned(n * 4) + (with_index ? aligned(n * 4) : 0);
    t += 3 * aligned((std::min<uint64_t>(n, h->size + 1) + 1) * 4);
  } else {
    t += 2 * aligned(n * 8) + (with_index ? 2 * aligned(n * 4) : 0);
    t += sort_ws_bytes(n, src_sort_plan(h, max_src).passes);
    t += 2 * aligned((n + 1) * 4) + scan_ws_bytes(n);
  }
  return t;
}

// Early count (see dg_graph::rank_alt): call right before op_begin.  On success h->early.active is set and the op must
// use h->early.rank instead of launching group_count_kernel itself.
template <int kMode>
void early_count(dg_graph* h, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n) {
  h->early.active = false;
  static const bool off = std::getenv("DG_NO_EARLY_COUNT") != nullptr;
  if (off || !h->submitting || !h->early_possible || h->pending.empty() || !h->cnt_clean || h->aux[1] == nullptr) return;
  // the side stream is not behind what the caller enqueued on the graph's stream: the batch must be known complete —
  // by contract (DG_FLAG_SUBMIT_INPUTS_READY) or through the ingest slot's copy-done event
  if (h->input_ready == nullptr && !(h->cfg.flags & DG_FLAG_SUBMIT_INPUTS_READY)) return;
  if (n > h->rank_alt_cap) {   // (grown by submit_coo when nothing is in flight)
    h->rank_alt_want = std::max(h->rank_alt_want, n);
    return;
  }
  GraphView g = view(h);
  const uint64_t cap = std::bit_ceil(std::max<uint64_t>(h->size, 1));
  const GroupIndex gi{(uint32_t)(cap - 1), (uint32_t)h->size};
  const uint32_t p = h->early_next++ & 1u;
  cudaStream_t sx = h->aux[1];
  cudaStreamWaitEvent(sx, h->ev_plan_done, 0);
  if (h->input_ready != nullptr) cudaStreamWaitEvent(sx, h->input_ready, 0);
  op_pre_arm_kernel<<<1, 1, 0, sx>>>(h->d_pre + p);
  group_count_kernel<kMode><<<(unsigned)((n + 256 * kGroupItems - 1) / (256 * kGroupItems)), 256, 0, sx>>>(
      g, gi, d_src, d_dst, (uint32_t)n, h->cnt_buf, h->rank_alt[p], h->d_pre + p);
  if (cudaPeekAtLastError() != cudaSuccess || cudaEventRecord(h->ev_early, sx) != cudaSuccess) {
    cudaGetLastError();
    h->cnt_clean = false;   // (whatever ran may have counted: the next user clears the counters)
    return;
  }
  h->early.active = true;
  h->early.rank = h->rank_alt[p];
  h->early.pre = h->d_pre + p;
}

// counting path, step 1: validate + count; allocates the run arrays the op's alloc pass fills
template <int kMode>
Grouped group_count(dg_graph* h, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, bool with_index) {
  GraphView g = view(h);
  Grouped out;
  const uint64_t nv = h->size + 1;  // + 1: the slot unknown query sources are clamped to
  const uint64_t cap = std::bit_ceil(std::max<uint64_t>(h->size, 1));
  out.gi = GroupIndex{(uint32_t)(cap - 1), (uint32_t)h->size};
  out.cnt_words = cap + 1;
  // fused delete (B = 32) resets every counter it touched; query / other block sizes leave them behind
  out.cnt = acquire_cnt(h, kMode == kPackDelete && h->B == 32);
  const bool early = h->early.active;   // (the count already ran beside the previous op: see early_count)
  out.rank = early ? h->early.rank : ws_alloc<uint32_t>(h, n);
  out.gdst = ws_alloc<uint32_t>(h, n);
  if (with_index) out.index = ws_alloc<uint32_t>(h, n);
  out.runs_bound = std::min<uint64_t>(n, nv);
  out.run_start = ws_alloc<uint32_t>(h, out.runs_bound + 1);
  out.run_end = ws_alloc<uint32_t>(h, out.runs_bound + 1);
  out.run_src = ws_alloc<uint32_t>(h, out.runs_bound + 1);
  if (!early) {
    DG_LAUNCH(h, "group_count_kernel", group_count_kernel<kMode><<<(unsigned)((n + 256 * kGroupItems - 1) / (256 * kGroupItems)), 256, 0, h->stream>>>(
        g, out.gi, d_src, d_dst, (uint32_t)n, out.cnt, out.rank, h->d_op()));
  }
  tl_mark(h, "K1", h->stream);
  out.b = BatchView{nullptr, out.gdst, out.run_src, out.run_start, out.run_end};
  return out;
}
// counting path, step 3 (after the op's alloc pass turned cnt into group starts)
inline unsigned scatter_grid(uint64_t n) { return (unsigned)((n + 256 * kGroupItems - 1) / (256 * kGroupItems)); }
template <int kMode>
void group_scatter(dg_graph* h, const Grouped& gr, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n,
                   cudaStream_t stream = nullptr) {
  GraphView g = view(h);
  if (stream == nullptr) stream = h->stream;
  const unsigned grid = scatter_grid(n);
  if (gr.index) {
    DG_LAUNCH(h, "group_scatter_kernel", group_scatter_kernel<kMode, true><<<grid, 256, 0, stream>>>(
        g, gr.gi, d_src, d_dst, (uint32_t)n, gr.cnt, gr.rank, gr.gdst, gr.index, h->d_op()));
  } else {
    DG_LAUNCH(h, "group_scatter_kernel", group_scatter_kernel<kMode, false><<<grid, 256, 0, stream>>>(
        g, gr.gi, d_src, d_dst, (uint32_t)n, gr.cnt, gr.rank, gr.gdst, nullptr, h->d_op()));
  }
}

// radix path: complete grouping (runs laid out in order: run_end == run_start + 1)
template <int kMode>
Grouped group_radix(dg_graph* h, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, bool with_index,
                    uint64_t max_src) {
  GraphView g = view(h);
  Grouped out;
  SortPlan plan = src_sort_plan(h, max_src);
  unsigned long long* keys = ws_alloc<unsigned long long>(h, n);
  unsigned long long* keys_alt = ws_alloc<unsigned long long>(h, n);
  uint32_t *idx = nullptr, *idx_alt = nullptr;
  if (with_index) {
    idx = ws_alloc<uint32_t>(h, n);
    idx_alt = ws_alloc<uint32_t>(h, n);
  }
  SortScratch sc = sort_prepare(h, n, plan);
  if (with_index) {
    DG_LAUNCH(h, "pack_coo_kernel", pack_coo_kernel<kMode, true><<<grid_for(h, n, 256 * 8), 256, 0, h->stream>>>(
        g, d_src, d_dst, (uint32_t)n, keys, idx, plan, sc.hist, h->d_op()));
  } else {
    DG_LAUNCH(h, "pack_coo_kernel", pack_coo_kernel<kMode, false><<<grid_for(h, n, 256 * 8), 256, 0, h->stream>>>(
        g, d_src, d_dst, (uint32_t)n, keys, nullptr, plan, sc.hist, h->d_op()));
  }
  sort_keys(h, &keys, &keys_alt, with_index ? &idx : nullptr, with_index ? &idx_alt : nullptr, n, plan, sc, true);
  out.runs_bound = n;
  uint32_t* run_start = ws_alloc<uint32_t>(h, n + 1);
  uint32_t* run_src = ws_alloc<uint32_t>(h, n + 1);
  launch_scan(h, "scan_kernel<runs>", n, d_n_input(h), RunsIn{keys}, RunsOut{keys, run_start, run_src},
              RunsFin{run_start, h->d_op(), (uint32_t)n});
  out.b = BatchView{keys, nullptr, run_src, run_start, run_start + 1};
  out.index = idx;
  return out;
}

// block size of a deferred pool from the first batch (compute_block_size, csr.hpp:77-88; DG_FLAG_AUTO_BLOCK_NATIVE)
inline uint32_t auto_block_size(const dg_graph* h, uint64_t n_edges, uint64_t n_sources) {
  const uint64_t rounded = std::max<uint64_t>(1, (n_edges + n_sources / 2) / n_sources);
  if ((h->cfg.flags & DG_FLAG_AUTO_BLOCK_NATIVE) && rounded >= 24 && rounded <= 48) return 32u;
  return (uint32_t)std::min<uint64_t>(rounded, 0x7FFFFFFFull);
}

int require_pool(dg_graph* h) {
  if (h->B == 0 || h->slab == nullptr)
    return fail(h, DG_ERR_ENGINE, "graph has no block pool yet (block_size 0 before the first insert)");
  return DG_OK;
}

// group + enumerate a COO batch for a query (either strategy)
template <int kMode>
Grouped group_and_enumerate(dg_graph* h, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n,
                            bool with_index, uint64_t max_src, Worklist* w_out) {
  GraphView g = view(h);
  if (use_counting(h, n)) {
    Grouped gr = group_count<kMode>(h, d_src, d_dst, n, with_index);
    Worklist w = alloc_worklist(h, gr.runs_bound, n, true);
    launch_alloc(h, "alloc_kernel<group+enum>", n, d_n_input(h), GroupEnumIn{g, gr.gi, d_src, gr.rank, gr.cnt, 1, false},
                 GroupEnumOut{g, gr.gi, d_src, gr.cnt, gr.run_src, gr.run_start, gr.run_end, w.lists(h)},
                 EnumFin{h->d_op(), h->blocks_in_use(), /*set_runs=*/1});
    fork(h);   // the scatter and the two chain walks are independent
    group_scatter<kMode>(h, gr, d_src, d_dst, n);
    enqueue_walk(h, gr.b, w, gr.runs_bound);
    join(h);
    *w_out = w;
    return gr;
  }
  Grouped gr = group_radix<kMode>(h, d_src, d_dst, n, with_index, max_src);
  *w_out = enqueue_enumerate(h, gr.b, gr.runs_bound, n, /*check_alive=*/1);
  return gr;
}
inline size_t group_enumerate_ws(const dg_graph* h, uint64_t n, bool with_index, uint64_t max_src) {
  return group_ws_bytes(h, n, with_index, max_src) + worklist_ws(h, std::min<uint64_t>(n, h->size + 1) + 0, n) +
         worklist_ws(h, n, n);  // either strategy's run bound
}

// ---- delete over a grouped batch -----------------------------------------------------------------
// Warp-owned sources (fused_class: short chains, few targets — B = 32 only) are finished by ONE kernel on
// the op stream; the hubs keep the multi-kernel path (walk -> match tiers -> compaction plan -> holes ->
// moves) on the two high-priority side streams, beside it.  Enqueue order on entry: the enumeration plan
// (alloc_kernel<...enum>, which also classifies the sources) is already on the op stream.
//   scatter(): the counting group-by's scatter (needed by both the fused kernel and the hub match).
inline cudaStream_t side(const dg_graph* h, int i) { return h->profiling ? h->stream : h->aux[i]; }

//   scatter(stream): the counting group-by's scatter; scatter_ctas: its grid (0: the batch is already grouped).
//   The fused kernel is launched beside it and waits for its CTAs on the device (wait_scatter).
template <class Scatter>
int delete_run(dg_graph* h, const BatchView& b, const Worklist& w, uint64_t runs_bound, uint64_t n, bool fuse,
               GroupIndex gi, uint32_t* cnt, uint32_t scatter_ctas, Scatter&& scatter) {
  GraphView g = view(h);
  const uint64_t wl_bound = std::max<uint64_t>(1, h->blocks_in_use());
  uint32_t* run_matched = w.zero3;   // (zeroed per run by the enumeration plan)
  uint32_t* free_off = ws_alloc<uint32_t>(h, runs_bound + 1);
  uint32_t* wl_mask = ws_alloc<uint32_t>(h, (wl_bound + 1) * g.mw);
  uint32_t* hole_prefix = ws_alloc<uint32_t>(h, 2 * wl_bound + 2);   // holes / survivors before every work-list block
  unsigned long long* tally = tally_buf(h);   // persistent, zero between ops
  const bool par = !h->profiling;
  cudaStream_t s0 = side(h, 0), s1 = side(h, 1);
  if (par) {
    cudaEventRecord(h->ev_fork, h->stream);
    cudaStreamWaitEvent(s0, h->ev_fork, 0);
    cudaStreamWaitEvent(s1, h->ev_fork, 0);
  }
  tl_mark(h, "K2", h->stream);
  enqueue_walk(h, b, w, runs_bound, s0, s1);   // hub chains only
  tl_mark(h, "walk_big", s0);
  tl_mark(h, "walk_small", s1);
  // (Launching the fused kernel BESIDE the scatter, with a device-side wait for the scatter's CTAs right before
  // the first target load, was measured: the kernel ended 4 us earlier, the scatter itself took up to 50 us
  // longer under the spinning warps.  Stream order it is.)
  scatter(h->stream);
  tl_mark(h, "scatter", h->stream);
  if (par) cudaEventRecord(h->ev_main, h->stream);
  if (fuse) {
    // one-warp CTAs: the medium sources first (heaviest), strided over a bounded grid, then 32 runs per warp
    const uint32_t g_med = (uint32_t)std::clamp<uint64_t>((fused_med_bound(h, runs_bound, n) + 7) / 8, 1, 32768);
    const unsigned grid = g_med + (unsigned)((runs_bound + 31) / 32);
    DG_LAUNCH(h, "fused_delete_kernel", fused_delete_kernel<<<grid, 32, 0, h->stream>>>(
        g, b, w.wl_off, w.run_deg, w.run_head, w.fmed_rec, g_med, (uint32_t)runs_bound, gi, cnt, scatter_ctas, tally, h->d_op()));
    tl_mark(h, "fused", h->stream);
    DG_LAUNCH(h, "fused_tally_kernel", fused_tally_kernel<<<1, 5 * 32, 0, h->stream>>>(g, tally, h->d_op()));
    tl_mark(h, "tally", h->stream);
  }
  if (par) {   // the hub match needs both walks and the scatter
    cudaEventRecord(h->ev_join[0], s0);
    cudaEventRecord(h->ev_join[1], s1);
    cudaStreamWaitEvent(s0, h->ev_join[1], 0);
    cudaStreamWaitEvent(s0, h->ev_main, 0);
    cudaStreamWaitEvent(s1, h->ev_join[0], 0);
    cudaStreamWaitEvent(s1, h->ev_main, 0);
  }
  if (h->B == 32) enqueue_match_impl<true, true>(h, b, w, n, run_matched, wl_mask, nullptr, s0, s1, s1);
  else enqueue_match_impl<true, false>(h, b, w, n, run_matched, wl_mask, nullptr, s0, s1, s1);
  tl_mark(h, "match_long", s0);
  tl_mark(h, "match_med_tiny", s1);
  if (par) {   // both tails need every tier's matches
    cudaEventRecord(h->ev_join[1], s1);
    cudaEventRecord(h->ev_join[0], s0);
    cudaStreamWaitEvent(s0, h->ev_join[1], 0);
    cudaStreamWaitEvent(s1, h->ev_join[0], 0);
  }
  // compaction of the hub chains, two independent halves side by side:
  //   s1: ring positions of the freed blocks -> repair (degree / tail / head) + reclaim;
  //   s0: hole / survivor numbering (one ordered scan over the work list) -> moves.
  // Scratch is bounded by the blocks in use: nothing to size after the match, no retry.
  launch_alloc(h, "alloc_kernel<moves>", runs_bound, d_n_runs(h), MovesIn{g, w.run_deg, run_matched},
               MovesOut{free_off}, MovesFin{g, h->d_op()}, s1);
  DG_LAUNCH(h, "delete_holes_kernel", delete_holes_kernel<<<grid_resident(h, wl_bound, 256, delete_holes_kernel), 256, 0, s1>>>(
      g, b, w.wl_off, w.wl_handle, w.wl_run, w.run_deg, run_matched, free_off, h->d_op()));
  tl_mark(h, "t_repair", s1);
  launch_scan(h, "scan_kernel<holes>", 2 * wl_bound, &h->d_op()->hole_items,
              HoleScanIn{g, w.wl_off, w.wl_run, w.run_deg, run_matched, wl_mask, h->d_op()}, HoleScanOut{hole_prefix},
              HoleScanFin{hole_prefix, h->d_op()}, s0);
  tl_mark(h, "t_scan", s0);
  DG_LAUNCH(h, "delete_moves_kernel", delete_moves_kernel<<<grid_resident(h, wl_bound, 256, delete_moves_kernel), 256, 0, s0>>>(
      g, w.wl_off, w.wl_handle, w.wl_run, w.run_deg, run_matched, wl_mask, hole_prefix, h->d_op()));
  tl_mark(h, "hub_tail", s0);
  if (par) {
    cudaEventRecord(h->ev_join[0], s0);
    cudaEventRecord(h->ev_join[1], s1);
    cudaStreamWaitEvent(h->stream, h->ev_join[0], 0);
    cudaStreamWaitEvent(h->stream, h->ev_join[1], 0);
  }
  return op_end(h);
}
inline size_t delete_matched_ws(const dg_graph* h, uint64_t runs_bound) {
  const uint64_t wl_bound = std::max<uint64_t>(1, h->blocks_in_use());
  return 5 * aligned((runs_bound + 1) * 4) + aligned((wl_bound + 1) * ((h->B + 31) / 32) * 4) + alloc_ws_bytes() +
         aligned((2 * wl_bound + 2) * 4) + scan_ws_bytes(2 * wl_bound);
}

// delete of a COO batch: group (either strategy) + enumeration plan with classification, then delete_run
int delete_coo_run(dg_graph* h, const uint32_t* d_src, const uint32_t* d_dst, uint64_t n, uint64_t max_src) {
  GraphView g = view(h);
  const bool fuse = h->B == 32;
  if (use_counting(h, n)) {
    Grouped gr = group_count<kPackDelete>(h, d_src, d_dst, n, false);
    Worklist w = alloc_worklist(h, gr.runs_bound, n, true, fuse, /*for_delete=*/true);
    launch_alloc(h, "alloc_kernel<group+enum>", n, d_n_input(h), GroupEnumIn{g, gr.gi, d_src, gr.rank, gr.cnt, 1, fuse},
                 GroupEnumOut{g, gr.gi, d_src, gr.cnt, gr.run_src, gr.run_start, gr.run_end, w.lists(h)},
                 EnumFin{h->d_op(), h->blocks_in_use(), /*set_runs=*/1});
    enqueue_agree(h, false);
    return delete_run(h, gr.b, w, gr.runs_bound, n, fuse, gr.gi, fuse ? gr.cnt : nullptr, /*scatter_ctas=*/0,
                      [&](cudaStream_t st) { group_scatter<kPackDelete>(h, gr, d_src, d_dst, n, st); });
  }
  Grouped gr = group_radix<kPackDelete>(h, d_src, d_dst, n, false, max_src);
  Worklist w = enqueue_enumerate(h, gr.b, gr.runs_bound, n, /*check_alive=*/1, fuse, /*walk=*/false, /*for_delete=*/true);
  enqueue_agree(h, false);
  return delete_run(h, gr.b, w, gr.runs_bound, n, fuse, GroupIndex{}, nullptr, 0, [](cudaStream_t) {});
}


}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int dg_abi_version(void) { return DG_ABI_VERSION; }

const char* dg_last_error(const dg_graph* h) {
  return h ? h->last_error.c_str() : g_create_error.c_str();
}

int dg_create(const dg_config* config, uint64_t initial_vertices, uint32_t block_size,
              dg_graph** out) {
  if (!out) return fail(nullptr, DG_ERR_DATA, "dg_create: out is null");
  *out = nullptr;
  dg_config cfg{};
  if (config) cfg = *config;
  if (initial_vertices >= 0xFFFFFFFFull)
    return fail(nullptr, DG_ERR_ENGINE, "dg_create: vertex ids are 32-bit");
  dg_graph* h = new (std::nothrow) dg_graph();
  if (!h) return fail(nullptr, DG_ERR_ENGINE, "dg_create: out of host memory");
  h->cfg = cfg;
  h->device = cfg.device;
  h->reclaim = (cfg.flags & DG_FLAG_NO_RECLAIM) ? 0 : 1;
  h->timeline = std::getenv("DG_TIMELINE") != nullptr;
  h->group_mode = (cfg.flags & DG_FLAG_GROUP_RADIX) ? 1 : ((cfg.flags & DG_FLAG_GROUP_COUNT) ? 2 : 0);
  if (cfg.trigger_fraction > 0.f) h->trigger = cfg.trigger_fraction;
  if (cfg.growth_fraction > 0.f) h->growth = cfg.growth_fraction;
  if (h->trigger > 1.0 || h->growth > 1.0 || cfg.trigger_fraction < 0.f || cfg.growth_fraction < 0.f) {
    delete h;
    return fail(nullptr, DG_ERR_DATA, "growth policy: fractions must be in (0, 1]");   // block_pool.hpp:23-28
  }
  auto bail = [&](int code, const std::string& msg) {
    g_create_error = msg;
    dg_destroy(h);
    return code;
  };
  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) return bail(DG_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device);
  if (cfg.stream) {
    h->stream = (cudaStream_t)cfg.stream;
  } else {
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(DG_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    h->own_stream = true;
  }
  // vertex dictionary: capacity = closest_pow2(max(1, V0)) (vertex_dictionary.hpp:30-31)
  h->size = initial_vertices;
  h->capacity = std::bit_ceil(initial_vertices == 0 ? 1ull : initial_vertices);
  h->alive_count = initial_vertices;
  h->alive_host.assign((h->capacity + 63) / 64, 0ull);
  for (uint64_t v = 0; v < initial_vertices; ++v) h->alive_host[v >> 6] |= 1ull << (v & 63);
  const size_t words = (h->capacity + 31) / 32;
  if (cudaMalloc(&h->head, h->capacity * 4) != cudaSuccess ||
      cudaMalloc(&h->tail, h->capacity * 4) != cudaSuccess ||
      cudaMalloc(&h->deg, h->capacity * 4) != cudaSuccess ||
      cudaMalloc(&h->alive, words * 4) != cudaSuccess ||
      cudaMalloc(&h->d_blk, sizeof(DevBlock)) != cudaSuccess ||
      cudaHostAlloc(&h->h_ring, kStatusSlots * sizeof(DevBlock), cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return bail(DG_ERR_ENGINE, "vertex dictionary: device allocation failed");
  }
  std::memset(h->h_ring, 0, kStatusSlots * sizeof(DevBlock));
  h->h_blk = &h->h_ring[0];
  if (std::getenv("DG_STATUS_MEMCPY") == nullptr) {
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, h->h_ring, 0) == cudaSuccess) h->h_ring_dev = static_cast<DevBlock*>(dp);
    else cudaGetLastError();
  }
  cudaMemsetAsync(h->d_blk, 0, sizeof(DevBlock), h->stream);
  cudaMemsetAsync(h->head, 0xFF, h->capacity * 4, h->stream);
  cudaMemsetAsync(h->tail, 0xFF, h->capacity * 4, h->stream);
  cudaMemsetAsync(h->deg, 0, h->capacity * 4, h->stream);
  cudaMemsetAsync(h->alive, 0, words * 4, h->stream);
  if (initial_vertices > 0) {
    GraphView g = view(h);
    DG_LAUNCH(h, "vertex_init_kernel", vertex_init_kernel<<<grid_for(h, initial_vertices, 256), 256, 0, h->stream>>>(
        g, 0u, (uint32_t)initial_vertices));
  }
  if (block_size > 0) {
    const int rc = create_pool(h, block_size);
    if (rc != DG_OK) return bail(rc, h->last_error);
  }
  if (cudaMalloc(&h->zscratch, kZScratchWords * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    return bail(DG_ERR_ENGINE, "dg_create: device allocation failed");
  }
  // side streams run the (few, latency-critical) hub kernels of an op beside its bulk kernel: highest priority
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  for (int i = 0; i < 2; ++i) {
    if (cudaStreamCreateWithPriority(&h->aux[i], cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_join[i], cudaEventDisableTiming) != cudaSuccess)
      return bail(DG_ERR_CUDA, "dg_create: auxiliary stream");
  }
  if (cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_main, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_plan_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_early, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&h->d_pre, 2 * sizeof(OpState)) != cudaSuccess)
    return bail(DG_ERR_CUDA, "dg_create: auxiliary stream");
  if (cfg.workspace_bytes && ws_reserve(h, cfg.workspace_bytes) != DG_OK) return bail(DG_ERR_ENGINE, h->last_error);
  e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return bail(DG_ERR_CUDA, std::string("dg_create: ") + cudaGetErrorString(e));
  *out = h;
  return DG_OK;
}

void dg_destroy(dg_graph* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->h_ring) drain(h);
  if (h->stream) cudaStreamSynchronize(h->stream);
  cudaFree(h->head);
  cudaFree(h->tail);
  cudaFree(h->deg);
  cudaFree(h->alive);
  if (h->pool_vm) {
    h->vm_slab.destroy();
    h->vm_next.destroy();
  } else {
    cudaFree(h->slab);
    cudaFree(h->next);
  }
  cudaFree(h->ring);
  cudaFree(h->d_blk);
  if (h->h_ring) cudaFreeHost(h->h_ring);
  for (auto& pd : h->pending) cudaEventDestroy(pd.done);
  for (auto e : h->done_pool) cudaEventDestroy(e);
  cudaFree(h->ws.base);
  cudaFree(h->cnt_buf);
  cudaFree(h->zscratch);
  for (int i = 0; i < 2; ++i) {
    if (h->aux[i]) { cudaStreamSynchronize(h->aux[i]); cudaStreamDestroy(h->aux[i]); }
    if (h->ev_join[i]) cudaEventDestroy(h->ev_join[i]);
  }
  if (h->ev_plan_done) cudaEventDestroy(h->ev_plan_done);
  if (h->ev_early) cudaEventDestroy(h->ev_early);
  cudaFree(h->d_pre);
  cudaFree(h->rank_alt[0]);
  cudaFree(h->rank_alt[1]);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_main) cudaEventDestroy(h->ev_main);
  for (auto& sp : h->prof_open) { cudaEventDestroy(sp.a); cudaEventDestroy(sp.b); }
  for (auto e : h->prof_pool) cudaEventDestroy(e);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  cudaGetLastError();
  delete h;
}

// ---- insert -------------------------------------------------------------------
// check_only: validation + plan (every reason the reference would reject the batch for: csr.hpp:49-73,
// graph.hpp:320-328, ensure_available block_pool.hpp:177-189) without any mutation
static int insert_coo_impl(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n,
                           int mem, bool check_only = false) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  h->last_shortfall = 0;
  if (h->submitting) cudaSetDevice(h->device);
  else if (const int erc = enter(h)) return erc;
  if (n == 0) return DG_OK;  // EmptyBatchChangesNothing
  if (n >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  if (h->size == 0) return fail(h, DG_ERR_DATA, "csr batch: source id out of range (graph has no vertices)");
  const bool counting = use_counting(h, n);
  if (counting && ensure_cnt(h) != DG_OK) return DG_ERR_ENGINE;
  WsSizer sz;
  if (mem == DG_MEM_HOST) { sz.add<uint32_t>(n); sz.add<uint32_t>(n); }
  if (counting) {
    const uint64_t cap = std::bit_ceil(std::max<uint64_t>(h->size, 1));
    sz.total += aligned((cap + 4 + 2 * kAllocScratchWords) * 4) + aligned(n * 4) + aligned((cap + 2) * 16) + alloc_ws_bytes();
  } else {
    sz.total += group_ws_bytes(h, n, false, h->size - 1);
    // block size may still be unknown (deferred pool): size the unit list for B = 1
    sz.total += plan_arrays_ws(1, n, n);
  }
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const uint32_t *d_src, *d_dst;
  if ((rc = stage_in(h, src, n, mem, &d_src)) != DG_OK) return rc;
  if ((rc = stage_in(h, dst, n, mem, &d_dst)) != DG_OK) return rc;
  if (counting && !check_only) early_count<kPackInsert>(h, d_src, d_dst, n);
  if ((rc = op_begin(h, n, 0)) != DG_OK) {
    if (h->early.active) h->cnt_clean = false;
    h->early.active = false;
    return rc;
  }
  if (counting) {
    // count -> plan (one alloc pass over the entries) -> entry-parallel append: no grouped copy
    GraphView g = view(h);
    const uint64_t cap = std::bit_ceil(std::max<uint64_t>(h->size, 1));
    GroupIndex gi{(uint32_t)(cap - 1), (uint32_t)h->size};
    uint32_t* cnt = acquire_cnt(h, /*self_cleaning=*/true);   // the plan pass hands every touched counter back zeroed
    const bool early = h->early.active;   // (the count already ran beside the previous insert's append: see early_count)
    uint32_t* rank = early ? h->early.rank : ws_alloc<uint32_t>(h, n);
    uint4* info = ws_alloc<uint4>(h, cap + 2);
    const unsigned grid = (unsigned)((n + 256 * kGroupItems - 1) / (256 * kGroupItems));
    if (!early) {
      DG_LAUNCH(h, "group_count_kernel", group_count_kernel<kPackInsert><<<grid, 256, 0, h->stream>>>(
          g, gi, d_src, d_dst, (uint32_t)n, cnt, rank, h->d_op()));
    }
    launch_alloc(h, "alloc_kernel<group+plan>", n, d_n_input(h), GroupPlanIn{g, gi, d_src, rank, cnt},
                 GroupPlanOut{gi, d_src, info, cnt},
                 PlanFin{g, h->d_op(), n, /*set_runs=*/1, /*commit_globals=*/(h->agree_x || check_only) ? 0 : 1});
    tl_mark(h, "plan", h->stream);
    if (check_only) return op_end(h);
    if (h->submitting && h->ev_plan_done != nullptr && cudaEventRecord(h->ev_plan_done, h->stream) == cudaSuccess)
      h->early_possible = true;   // the next submitted op may count beside this op's append pass
    enqueue_agree(h, /*commit_insert=*/true);
    DG_LAUNCH(h, "append_entries_kernel", append_entries_kernel<<<grid, 256, 0, h->stream>>>(
        g, gi, d_src, d_dst, rank, (uint32_t)n, info, h->d_op()));
    return op_end(h);
  }
  Grouped gr = group_radix<kPackInsert>(h, d_src, d_dst, n, false, h->size - 1);
  if (check_only) {
    if (h->B != 0) {   // (deferred pool: the first batch sizes it, nothing to run out of)
      GraphView g = view(h);
      PlanArrays a = alloc_plan_arrays(h, gr.runs_bound, n);
      launch_alloc(h, "alloc_kernel<plan>", gr.runs_bound, d_n_runs(h), PlanIn{g, gr.b}, PlanOut{a},
                   PlanFin{g, h->d_op(), n, /*set_runs=*/0, /*commit_globals=*/0});
    }
    return op_end(h);
  }
  if (h->B == 0) {
    // deferred pool: compute_block_size (csr.hpp:77-88) from this first batch
    if ((rc = op_end(h)) != DG_OK) return rc;
    const uint64_t T = h->h_blk->op.n_runs;
    if ((rc = create_pool(h, auto_block_size(h, n, T))) != DG_OK) return rc;
    // the run arrays stay valid; re-arm the op words, keeping n_runs
    OpState& op = h->h_blk->op;
    op.err_index = ~0ull;
    DG_CUDA(h, cudaMemcpyAsync(h->d_op(), &op, sizeof(OpState), cudaMemcpyHostToDevice, h->stream));
  }
  enqueue_plan_append(h, gr.b, gr.runs_bound, n, /*csr_path=*/false);
  return op_end(h);
}

int dg_insert_batch_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n,
                        int mem) {
  return insert_with_growth(h, [&] { return insert_coo_impl(h, src, dst, n, mem); });
}

static int insert_csr_impl(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets,
                           const uint32_t* destinations, uint64_t n_edges, int mem,
                           bool require_empty) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  h->last_shortfall = 0;
  if (const int erc = enter(h)) return erc;
  if (n_offsets != h->size + 1)  // csr.hpp:50-53
    return fail(h, DG_ERR_DATA, "csr batch: offsets length " + std::to_string(n_offsets) +
                                    " does not match vertex count " + std::to_string(h->size) + " + 1");
  if (require_empty && h->active_edges != 0)
    return fail(h, DG_ERR_ENGINE, "bulk init: graph is not empty");
  if (n_edges >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  const uint64_t V = h->size;
  WsSizer sz;
  if (mem == DG_MEM_HOST) { sz.add<unsigned long long>(n_offsets); sz.add<uint32_t>(n_edges); }
  if (h->B == 32) {
    sz.add<uint32_t>(V + 1);
    sz.add<CsrItem>(3 * (n_edges / kCsrHeavy) + 16);
    sz.total += alloc_ws_bytes();
  } else {
    sz.add<uint32_t>(V + 2);
    sz.total += plan_arrays_ws(h->B ? h->B : 1, V, n_edges);  // deferred pool: size the unit list for B = 1
  }
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const unsigned long long* d_off;
  const uint32_t* d_dst;
  if ((rc = stage_in(h, reinterpret_cast<const unsigned long long*>(offsets), n_offsets, mem, &d_off)) != DG_OK) return rc;
  if ((rc = stage_in(h, destinations, n_edges, mem, &d_dst)) != DG_OK) return rc;
  if ((rc = op_begin(h, n_edges, V)) != DG_OK) return rc;
  GraphView g = view(h);
  if (h->B == 32 && n_edges > 0 && V > 0) {
    // native block size: plan (offset validation fused) + one TMA-staged append pass that also
    // validates the destinations and publishes deg/tail/front; rollback kernel on a late failure
    const uint64_t items_cap = 3 * (n_edges / kCsrHeavy) + 16;
    uint32_t* blk_off = ws_alloc<uint32_t>(h, V + 1);
    CsrItem* items = ws_alloc<CsrItem>(h, items_cap);
    unsigned long long* plan_scratch = ws_alloc<unsigned long long>(h, kAllocScratchWords);
    cudaMemsetAsync(plan_scratch, 0, kAllocScratchWords * sizeof(unsigned long long), h->stream);
    // a pool nothing was ever popped from: every source is empty and handle == queue position (csr_bulk_kernel)
    const bool fresh = h->active_edges == 0 && h->front == 0 && h->rear == h->NB && h->ring_identity >= h->NB &&
                       std::getenv("DG_NO_BULK_KERNEL") == nullptr;
    const unsigned plan_grid = (unsigned)((V + kCsrPlanTile - 1) / kCsrPlanTile);
    if (fresh) {
      DG_LAUNCH(h, "csr_plan_kernel", csr_plan_kernel<true><<<plan_grid, 256, 0, h->stream>>>(
          g, d_off, (uint32_t)V, n_edges, blk_off, items, items_cap, plan_scratch, h->d_op()));
    } else {
      DG_LAUNCH(h, "csr_plan_kernel", csr_plan_kernel<false><<<plan_grid, 256, 0, h->stream>>>(
          g, d_off, (uint32_t)V, n_edges, blk_off, items, items_cap, plan_scratch, h->d_op()));
    }
    const uint64_t groups = (V + 31) / 32 + items_cap;
    if (fresh) {
      const int ctas_per_sm = resident_ctas_per_sm(csr_bulk_kernel, kBulkWarps * 32, 0);
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((groups + kBulkWarps - 1) / kBulkWarps, (uint64_t)h->sm_count * ctas_per_sm));
      DG_LAUNCH(h, "csr_bulk_kernel", csr_bulk_kernel<<<grid, kBulkWarps * 32, 0, h->stream>>>(
          g, d_off, d_dst, (uint32_t)V, blk_off, items, n_edges, plan_scratch, h->d_op()));
    } else {
      const int csr_ctas_per_sm = resident_ctas_per_sm(csr_append_kernel, kCsrWarps * 32, 0);
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((groups + kCsrWarps - 1) / kCsrWarps, (uint64_t)h->sm_count * csr_ctas_per_sm));
      DG_LAUNCH(h, "csr_append_kernel", csr_append_kernel<<<grid, kCsrWarps * 32, 0, h->stream>>>(
          g, d_off, d_dst, (uint32_t)V, blk_off, items, n_edges, plan_scratch, h->d_op()));
    }
    rc = op_end(h);
    if (rc != DG_OK && h->h_blk->op.committed) {
      const std::string msg = h->last_error;
      csr_rollback_kernel<<<grid_for(h, V, 256), 256, 0, h->stream>>>(g, d_off, (uint32_t)V, h->d_op());
      DG_CUDA(h, cudaMemcpyAsync(&h->h_blk->st, h->d_state(), sizeof(DeviceState), cudaMemcpyDeviceToHost, h->stream));
      DG_CUDA(h, cudaStreamSynchronize(h->stream));
      h->front = h->h_blk->st.front;
      h->rear = h->h_blk->st.rear;
      h->active_edges = h->h_blk->st.active_edges;
      h->last_error = msg;
    }
    return rc;
  }
  uint32_t* run_start = ws_alloc<uint32_t>(h, V + 2);
  DG_LAUNCH(h, "csr_validate_offsets_kernel", csr_validate_offsets_kernel<<<grid_for(h, n_offsets, 256), 256, 0, h->stream>>>(
      g, d_off, (uint32_t)n_offsets, n_edges, /*check_dead_source=*/1, run_start, h->d_op()));
  if (n_edges == 0 || V == 0) return op_end(h);  // validated; nothing to append
  // (the destination range check, csr.hpp:67-72, is fused into the append pass)
  if (h->B == 0) {
    DG_LAUNCH(h, "count_nonzero_runs_kernel", count_nonzero_runs_kernel<<<grid_for(h, V, 256), 256, 0, h->stream>>>(run_start, (uint32_t)V, h->d_op()));
    if ((rc = op_end(h)) != DG_OK) return rc;
    const uint64_t T = h->h_blk->op.aux0;
    if (T == 0) return fail(h, DG_ERR_DATA, "compute_block_size: first batch contains no edges");
    if ((rc = create_pool(h, auto_block_size(h, n_edges, T))) != DG_OK) return rc;
    OpState& op = h->h_blk->op;
    op.err_index = ~0ull;
    op.aux0 = 0;
    DG_CUDA(h, cudaMemcpyAsync(h->d_op(), &op, sizeof(OpState), cudaMemcpyHostToDevice, h->stream));
  }
  BatchView b{nullptr, d_dst, nullptr, run_start, run_start + 1};
  enqueue_plan_append(h, b, V, n_edges, /*csr_path=*/true);
  return op_end(h);
}

int dg_insert_batch_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets,
                        const uint32_t* destinations, uint64_t n_edges, int mem) {
  return insert_with_growth(h, [&] { return insert_csr_impl(h, offsets, n_offsets, destinations, n_edges, mem, false); });
}

int dg_bulk_init_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets,
                     const uint32_t* destinations, uint64_t n_edges, int mem) {
  return insert_with_growth(h, [&] { return insert_csr_impl(h, offsets, n_offsets, destinations, n_edges, mem, true); });
}

// plan_batch (graph.hpp:135-160): validation of an insert batch + the BatchPlan vectors, nothing mutated
int dg_plan_batch_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets, const uint32_t* destinations,
                      uint64_t n_edges, int mem, uint64_t* blocks_required, uint64_t* prefix_sum,
                      uint32_t* space_remaining, uint64_t* total_blocks) {
  if (!h || !blocks_required || !prefix_sum || !space_remaining) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (n_offsets != h->size + 1)  // csr.hpp:50-53
    return fail(h, DG_ERR_DATA, "csr batch: offsets length " + std::to_string(n_offsets) +
                                    " does not match vertex count " + std::to_string(h->size) + " + 1");
  if (n_edges >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  if (int rc = require_pool(h)) return rc;
  const uint64_t V = h->size;
  WsSizer sz;
  sz.add<unsigned long long>(n_offsets); sz.add<uint32_t>(n_edges);
  sz.add<uint32_t>(V + 2);
  sz.add<unsigned long long>(V); sz.add<unsigned long long>(V); sz.add<uint32_t>(V);
  sz.total += scan_ws_bytes(V);
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const unsigned long long* d_off;
  const uint32_t* d_dst;
  if ((rc = stage_in(h, reinterpret_cast<const unsigned long long*>(offsets), n_offsets, mem, &d_off)) != DG_OK) return rc;
  if ((rc = stage_in(h, destinations, n_edges, mem, &d_dst)) != DG_OK) return rc;
  if ((rc = op_begin(h, n_edges, V)) != DG_OK) return rc;
  GraphView g = view(h);
  uint32_t* run_start = ws_alloc<uint32_t>(h, V + 2);
  const bool host_out = mem == DG_MEM_HOST;
  unsigned long long* d_req = host_out ? ws_alloc<unsigned long long>(h, V) : reinterpret_cast<unsigned long long*>(blocks_required);
  unsigned long long* d_pre = host_out ? ws_alloc<unsigned long long>(h, V) : reinterpret_cast<unsigned long long*>(prefix_sum);
  uint32_t* d_space = host_out ? ws_alloc<uint32_t>(h, V) : space_remaining;
  DG_LAUNCH(h, "csr_validate_offsets_kernel", csr_validate_offsets_kernel<<<grid_for(h, n_offsets, 256), 256, 0, h->stream>>>(
      g, d_off, (uint32_t)n_offsets, n_edges, /*check_dead_source=*/1, run_start, h->d_op()));
  if (n_edges > 0) {
    DG_LAUNCH(h, "validate_dsts_kernel", validate_dsts_kernel<<<grid_for(h, n_edges, 256 * 4), 256, 0, h->stream>>>(g, d_dst, (uint32_t)n_edges, h->d_op()));
  }
  if (V > 0) {
    launch_scan(h, "scan_kernel<batch_plan>", V, d_n_runs(h), BatchPlanIn{g, run_start}, BatchPlanOut{g, d_req, d_pre, d_space},
                BatchPlanFin{h->d_op()});
    if (host_out) {
      DG_CUDA(h, cudaMemcpyAsync(blocks_required, d_req, V * 8, cudaMemcpyDeviceToHost, h->stream));
      DG_CUDA(h, cudaMemcpyAsync(prefix_sum, d_pre, V * 8, cudaMemcpyDeviceToHost, h->stream));
      DG_CUDA(h, cudaMemcpyAsync(space_remaining, d_space, V * 4, cudaMemcpyDeviceToHost, h->stream));
    }
  }
  rc = op_end(h);
  h->report.blocks_popped = 0;   // (a plan pops nothing)
  if (rc == DG_OK && total_blocks) *total_blocks = h->h_blk->op.total_need;
  return rc;
}

// ---- delete -------------------------------------------------------------------
static int delete_coo_impl(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, int mem, bool check_only) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (h->submitting) cudaSetDevice(h->device);
  else if (const int erc = enter(h)) return erc;
  if (n == 0) return DG_OK;
  if (n >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  if (h->size == 0) return fail(h, DG_ERR_DATA, "csr batch: source id out of range (graph has no vertices)");
  const bool no_pool = h->B == 0 || check_only;  // no pool yet => no edges: only validation can have an effect
  if (!no_pool && use_counting(h, n) && ensure_cnt(h) != DG_OK) return DG_ERR_ENGINE;
  WsSizer sz;
  if (mem == DG_MEM_HOST) { sz.add<uint32_t>(n); sz.add<uint32_t>(n); }
  if (no_pool) sz.total += group_ws_bytes(h, n, false, h->size - 1, /*force_radix=*/true);
  else sz.total += group_enumerate_ws(h, n, false, h->size - 1) + delete_matched_ws(h, n);
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const uint32_t *d_src, *d_dst;
  if ((rc = stage_in(h, src, n, mem, &d_src)) != DG_OK) return rc;
  if ((rc = stage_in(h, dst, n, mem, &d_dst)) != DG_OK) return rc;
  if (!no_pool && use_counting(h, n)) early_count<kPackDelete>(h, d_src, d_dst, n);
  if ((rc = op_begin(h, n, 0)) != DG_OK) {
    if (h->early.active) h->cnt_clean = false;
    h->early.active = false;
    return rc;
  }
  if (no_pool) {  // validation only (radix path packs + validates; B == 0 never takes the counting path)
    group_radix<kPackDelete>(h, d_src, d_dst, n, false, h->size - 1);
    return op_end(h);
  }
  return delete_coo_run(h, d_src, d_dst, n, h->size - 1);
}
int dg_delete_batch_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, int mem) {
  return delete_coo_impl(h, src, dst, n, mem, false);
}

// ---- submitted (asynchronous) COO updates ----------------------------------------------------------
// The op is enqueued and the call returns without waiting for it: its status lands in a pinned slot and is
// looked at by a later submit / dg_flush / any synchronous call.  Everything the host decides BETWEEN ops in
// the synchronous path is decided here from bounds, before the enqueue; when a bound does not hold the call
// simply runs the op the synchronous way (after waiting for what is in flight), so the outcome never differs:
//   - ensure_available (block_pool.hpp:177-189): the free handles known to the host minus what the inserts
//     in flight can pop at most must cover this insert (an insert pops at most one block per entry);
//   - commit_front's growth rule (block_pool.hpp:162-172): cumulative consumption, counted with the same
//     bounds, must stay below the trigger — the pool never has to grow behind a submitted op;
//   - every scratch array of an op is bounded by the batch and by (an upper bound of) the blocks in use: nothing is
//     sized from what an earlier op of the stream produced.
static int submit_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, bool is_insert, uint64_t* ticket) {
  if (!h) return DG_ERR_DATA;
  if (ticket) *ticket = 0;
  cudaSetDevice(h->device);
  if (h->deferred_rc != DG_OK) {   // an earlier submitted op failed: report it before anything else is queued
    const int rc = drain(h);
    return rc != DG_OK ? rc : take_deferred(h);
  }
  while (!h->pending.empty()) {    // fold in whatever has finished: keeps the bounds tight
    const size_t before = h->pending.size();
    const int rc = retire_oldest(h, /*wait=*/false);
    if (rc != DG_OK) return rc;
    if (h->pending.size() == before) break;
  }
  if (h->deferred_rc != DG_OK) {
    const int rc = drain(h);
    return rc != DG_OK ? rc : take_deferred(h);
  }
  // rank buffers of the early count: sized for the largest submitted batch seen, (re)allocated while nothing is in flight
  h->rank_alt_want = std::max(h->rank_alt_want, n);
  if (h->pending.empty() && h->rank_alt_want > h->rank_alt_cap) {
    cudaStreamSynchronize(h->stream);
    if (h->aux[1]) cudaStreamSynchronize(h->aux[1]);
    uint32_t *a = nullptr, *b = nullptr;
    const uint64_t want = h->rank_alt_want + h->rank_alt_want / 4;
    if (cudaMalloc(&a, want * 4) == cudaSuccess && cudaMalloc(&b, want * 4) == cudaSuccess) {
      cudaFree(h->rank_alt[0]);
      cudaFree(h->rank_alt[1]);
      h->rank_alt[0] = a;
      h->rank_alt[1] = b;
      h->rank_alt_cap = want;
    } else {   // (no early count then: everything still works)
      cudaGetLastError();
      cudaFree(a);
      cudaFree(b);
    }
  }
  bool async_ok = h->B != 0 && h->slab != nullptr && !h->profiling && !h->timeline && h->agree_x == nullptr && n > 0;
  if (async_ok && is_insert) {
    const uint64_t free_known = h->rear - h->front;
    if (free_known < h->pending_pop_bound + n) async_ok = false;
    if (h->pool_vm && h->total_capacity > 0 &&
        (double)(h->consumed + h->pending_pop_bound + n) / (double)h->total_capacity >= h->trigger)
      async_ok = false;
  }
  if (!async_ok) {
    int rc = drain(h);
    if (rc != DG_OK) return rc;
    if ((rc = take_deferred(h)) != DG_OK) return rc;
    rc = is_insert ? dg_insert_batch_coo(h, src, dst, n, DG_MEM_DEVICE) : dg_delete_batch_coo(h, src, dst, n, DG_MEM_DEVICE);
    if (rc == DG_OK) ++h->submitted_applied;
    return rc;
  }
  h->submitting = true;
  h->submit_is_insert = is_insert;
  h->submit_pop_bound = is_insert ? n : 0;
  const size_t before = h->pending.size();
  const uint64_t t = h->next_ticket;
  const int rc = is_insert ? insert_coo_impl(h, src, dst, n, DG_MEM_DEVICE) : delete_coo_impl(h, src, dst, n, DG_MEM_DEVICE, false);
  h->submitting = false;
  if (rc != DG_OK) return rc;            // rejected on the host before anything was enqueued
  if (h->pending.size() == before) {     // (the op ended synchronously after all: launch error path, workspace overflow)
    ++h->submitted_applied;
    return DG_OK;
  }
  if (ticket) *ticket = t;
  return DG_OK;
}

int dg_submit_insert_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t* ticket) {
  return submit_coo(h, src, dst, n, true, ticket);
}
int dg_submit_delete_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t* ticket) {
  return submit_coo(h, src, dst, n, false, ticket);
}
int dg_flush(dg_graph* h, uint64_t* n_applied) {
  if (!h) return DG_ERR_DATA;
  cudaSetDevice(h->device);
  int rc = drain(h);
  if (n_applied) *n_applied = h->submitted_applied;
  h->submitted_applied = 0;
  if (rc != DG_OK) return rc;
  return take_deferred(h);
}
uint64_t dg_pending_ops(const dg_graph* h) { return h ? h->pending.size() : 0; }

int dg_check_batch_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, int is_insert, int mem) {
  if (!h) return DG_ERR_DATA;
  if (!is_insert) return delete_coo_impl(h, src, dst, n, mem, true);
  const int rc = insert_coo_impl(h, src, dst, n, mem, true);
  // (a pool underflow the growth budget covers is not a rejection: the real insert grows the pool first)
  if (rc == DG_ERR_ENGINE && h->last_shortfall != 0 && h->pool_vm && h->nb_max - h->NB >= h->last_shortfall) return DG_OK;
  return rc;
}

int dg_delete_batch_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets,
                        const uint32_t* destinations, uint64_t n_edges, int mem) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (n_offsets != h->size + 1)
    return fail(h, DG_ERR_DATA, "csr batch: offsets length " + std::to_string(n_offsets) +
                                    " does not match vertex count " + std::to_string(h->size) + " + 1");
  if (n_edges >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  const uint64_t V = h->size;
  const uint64_t n = n_edges;
  WsSizer sz;
  if (mem == DG_MEM_HOST) { sz.add<unsigned long long>(n_offsets); sz.add<uint32_t>(n); }
  sz.add<uint32_t>(V + 2);
  if (h->B) sz.total += worklist_ws(h, V, n) + delete_matched_ws(h, V);
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const unsigned long long* d_off;
  const uint32_t* d_dst;
  if ((rc = stage_in(h, reinterpret_cast<const unsigned long long*>(offsets), n_offsets, mem, &d_off)) != DG_OK) return rc;
  if ((rc = stage_in(h, destinations, n, mem, &d_dst)) != DG_OK) return rc;
  if ((rc = op_begin(h, n, V)) != DG_OK) return rc;
  GraphView g = view(h);
  uint32_t* run_start = ws_alloc<uint32_t>(h, V + 2);
  DG_LAUNCH(h, "csr_validate_offsets_kernel", csr_validate_offsets_kernel<<<grid_for(h, n_offsets, 256), 256, 0, h->stream>>>(
      g, d_off, (uint32_t)n_offsets, n, /*check_dead_source=*/0, run_start, h->d_op()));
  if (n > 0) {
    DG_LAUNCH(h, "validate_dsts_kernel", validate_dsts_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(g, d_dst, (uint32_t)n, h->d_op()));
  }
  if (n == 0 || V == 0 || h->B == 0) return op_end(h);
  // a CSR batch is already grouped: run r is vertex r (empty runs are skipped by the enumeration)
  BatchView b{nullptr, d_dst, nullptr, run_start, run_start + 1};
  const bool fuse = h->B == 32;
  Worklist w = enqueue_enumerate(h, b, V, n, /*check_alive=*/1, fuse, /*walk=*/false, /*for_delete=*/true);
  return delete_run(h, b, w, V, n, fuse, GroupIndex{}, nullptr, 0, [](cudaStream_t) {});
}

// ---- query ---------------------------------------------------------------------
int dg_query_edges(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n,
                   uint8_t* out, int mem) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (n == 0) return DG_OK;
  if (n >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  if (h->B == 0 || h->size == 0) {  // no edges stored: every answer is false
    if (mem == DG_MEM_HOST) std::memset(out, 0, n);
    else DG_CUDA(h, cudaMemsetAsync(out, 0, n, h->stream));
    return DG_OK;
  }
  if (use_counting(h, n) && ensure_cnt(h) != DG_OK) return DG_ERR_ENGINE;
  WsSizer sz;
  if (mem == DG_MEM_HOST) { sz.add<uint32_t>(n); sz.add<uint32_t>(n); sz.add<uint8_t>(n); }
  sz.total += group_enumerate_ws(h, n, true, h->size);  // ids are clamped to size (unknown source)
  sz.add<uint8_t>(n);
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const uint32_t *d_src, *d_dst;
  if ((rc = stage_in(h, src, n, mem, &d_src)) != DG_OK) return rc;
  if ((rc = stage_in(h, dst, n, mem, &d_dst)) != DG_OK) return rc;
  uint8_t* d_out = (mem == DG_MEM_HOST) ? ws_alloc<uint8_t>(h, n) : out;
  if ((rc = op_begin(h, n, 0)) != DG_OK) return rc;
  Worklist w;
  Grouped gb = group_and_enumerate<kPackQuery>(h, d_src, d_dst, n, true, h->size, &w);
  uint8_t* hit = ws_alloc<uint8_t>(h, n);
  cudaMemsetAsync(hit, 0, n, h->stream);
  enqueue_match<false>(h, gb.b, w, n, nullptr, nullptr, hit);
  DG_LAUNCH(h, "query_scatter_kernel", query_scatter_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(hit, gb.index, (uint32_t)n, d_out, h->d_op()));
  if (mem == DG_MEM_HOST)
    DG_CUDA(h, cudaMemcpyAsync(out, d_out, n, cudaMemcpyDeviceToHost, h->stream));
  return op_end(h);
}

// ---- export / observables ---------------------------------------------------------
int dg_export_csr(dg_graph* h, uint64_t* offsets, uint32_t* destinations,
                  uint64_t n_dst_capacity, int sorted, int mem) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  const uint64_t V = h->size;
  // phase 1: degrees -> offsets
  WsSizer sz1;
  sz1.add<unsigned long long>(V + 1);
  sz1.total += scan_ws_bytes(std::max<uint64_t>(V, 1));
  int rc = ws_reserve(h, sz1.total);
  if (rc != DG_OK) return rc;
  if ((rc = op_begin(h, V, V)) != DG_OK) return rc;
  unsigned long long* d_off = (mem == DG_MEM_DEVICE) ? reinterpret_cast<unsigned long long*>(offsets)
                                                     : ws_alloc<unsigned long long>(h, V + 1);
  uint64_t total = 0;
  if (V == 0) {
    DG_CUDA(h, cudaMemsetAsync(d_off, 0, sizeof(unsigned long long), h->stream));
    if ((rc = op_end(h)) != DG_OK) return rc;
  } else {
    launch_scan(h, "scan_kernel<offsets>", V, d_n_input(h), DegIn{h->deg}, OffsetsOut{d_off}, OffsetsFin{d_off, V, h->d_op()});
    if ((rc = op_end(h)) != DG_OK) return rc;
    total = h->h_blk->op.aux0;
  }
  if (mem == DG_MEM_HOST)
    DG_CUDA(h, cudaMemcpy(offsets, d_off, (V + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  if (destinations == nullptr || total == 0) return DG_OK;
  if (total > n_dst_capacity)
    return fail(h, DG_ERR_DATA, "export: destinations capacity " + std::to_string(n_dst_capacity) +
                                    " < stored entries " + std::to_string(total));
  if (total >= (1ull << 32)) return fail(h, DG_ERR_ENGINE, "export: more than 2^32 entries");
  // phase 2: enumerate every chain and copy
  SortPlan plan = make_sort_plan(bits_for(h->dst_limit() - 1), bits_for(V - 1));
  WsSizer sz;
  sz.add<unsigned long long>(V + 1);
  sz.total += worklist_ws(h, V, 0);
  if (mem == DG_MEM_HOST) sz.add<uint32_t>(total);
  if (sorted) { sz.add<unsigned long long>(total); sz.add<unsigned long long>(total); sz.total += sort_ws_bytes(total, plan.passes); }
  // (host path: offsets were copied to the caller; re-uploaded after the workspace is re-laid out)
  if ((rc = ws_reserve(h, sz.total)) != DG_OK) return rc;
  unsigned long long* d_off2 = d_off;
  if (mem == DG_MEM_HOST) {
    d_off2 = ws_alloc<unsigned long long>(h, V + 1);
    DG_CUDA(h, cudaMemcpyAsync(d_off2, offsets, (V + 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice, h->stream));
  }
  if ((rc = op_begin(h, V, V)) != DG_OK) return rc;
  GraphView g = view(h);
  BatchView b{nullptr, nullptr, nullptr, nullptr, nullptr};
  Worklist w = enqueue_enumerate(h, b, V, 0, /*check_alive=*/0);
  uint32_t* d_dst = (mem == DG_MEM_HOST) ? ws_alloc<uint32_t>(h, total) : destinations;
  const uint64_t wl_bound = std::max<uint64_t>(1, h->blocks_in_use());
  if (!sorted) {
    DG_LAUNCH(h, "export_copy_kernel", export_copy_kernel<<<grid_for(h, wl_bound, 8), 256, 0, h->stream>>>(
        g, w.wl_off, w.wl_handle, w.wl_run, w.run_deg, d_off2, d_dst, nullptr, h->d_op()));
  } else {
    unsigned long long* keys = ws_alloc<unsigned long long>(h, total);
    unsigned long long* keys_alt = ws_alloc<unsigned long long>(h, total);
    DG_LAUNCH(h, "export_copy_kernel", export_copy_kernel<<<grid_for(h, wl_bound, 8), 256, 0, h->stream>>>(
        g, w.wl_off, w.wl_handle, w.wl_run, w.run_deg, d_off2, nullptr, keys, h->d_op()));
    SortScratch sc = sort_prepare(h, total, plan);
    sort_keys(h, &keys, &keys_alt, nullptr, nullptr, total, plan, sc, false);
    DG_LAUNCH(h, "keys_low_kernel", keys_low_kernel<<<grid_for(h, total, 256 * 4), 256, 0, h->stream>>>(keys, total, d_dst));
  }
  if (mem == DG_MEM_HOST)
    DG_CUDA(h, cudaMemcpyAsync(destinations, d_dst, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  return op_end(h);
}

int dg_active_destinations(dg_graph* h, uint32_t v, uint32_t* out, uint64_t capacity, uint64_t* n_out, int mem) {
  if (!h || !n_out || (capacity && !out)) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  *n_out = 0;
  if (v >= h->size || h->B == 0) return DG_OK;   // graph.hpp:118: unknown vertex -> empty
  int rc = ws_reserve(h, mem == DG_MEM_HOST ? aligned(capacity * 4) : 0);
  if (rc != DG_OK) return rc;
  uint32_t* d_out = (mem == DG_MEM_HOST && capacity) ? ws_alloc<uint32_t>(h, capacity) : out;
  if ((rc = op_begin(h, 1, 0)) != DG_OK) return rc;
  DG_LAUNCH(h, "adjacency_copy_kernel", adjacency_copy_kernel<<<1, 256, 0, h->stream>>>(view(h), v, d_out, capacity, h->d_op()));
  if ((rc = op_end(h)) != DG_OK) return rc;
  const uint64_t d = h->h_blk->op.aux0;
  *n_out = d;
  if (d > capacity)
    return fail(h, DG_ERR_DATA, "active_destinations: capacity " + std::to_string(capacity) + " < degree " + std::to_string(d));
  if (mem == DG_MEM_HOST && d) DG_CUDA(h, cudaMemcpy(out, d_out, d * 4, cudaMemcpyDeviceToHost));
  return DG_OK;
}

int dg_degrees(dg_graph* h, uint64_t* out, int mem) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  const uint64_t V = h->size;
  if (V == 0) return DG_OK;
  int rc = ws_reserve(h, aligned(V * 8));
  if (rc != DG_OK) return rc;
  unsigned long long* d = (mem == DG_MEM_DEVICE) ? reinterpret_cast<unsigned long long*>(out)
                                                 : ws_alloc<unsigned long long>(h, V);
  DG_LAUNCH(h, "degrees_kernel", degrees_kernel<<<grid_for(h, V, 256 * 4), 256, 0, h->stream>>>(h->deg, (uint32_t)V, d));
  if (mem == DG_MEM_HOST)
    DG_CUDA(h, cudaMemcpyAsync(out, d, V * 8, cudaMemcpyDeviceToHost, h->stream));
  DG_CUDA(h, cudaStreamSynchronize(h->stream));
  return DG_OK;
}

int dg_digest(dg_graph* h, uint64_t* out_digest, uint64_t* out_entries) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  const uint64_t V = h->size;
  if (out_digest) *out_digest = 0;
  if (out_entries) *out_entries = 0;
  if (V == 0 || h->B == 0) return DG_OK;
  int rc = ws_reserve(h, worklist_ws(h, V, 0));
  if (rc != DG_OK) return rc;
  if ((rc = op_begin(h, V, V)) != DG_OK) return rc;
  GraphView g = view(h);
  BatchView b{nullptr, nullptr, nullptr, nullptr, nullptr};
  Worklist w = enqueue_enumerate(h, b, V, 0, 0);
  const uint64_t wl_bound = std::max<uint64_t>(1, h->blocks_in_use());
  DG_LAUNCH(h, "digest_kernel", digest_kernel<<<grid_for(h, wl_bound, 8), 256, 0, h->stream>>>(g, w.wl_off, w.wl_handle, w.wl_run,
                                                                 w.run_deg, h->d_op()));
  if ((rc = op_end(h)) != DG_OK) return rc;
  if (out_digest) *out_digest = h->h_blk->op.aux0;
  if (out_entries) *out_entries = h->h_blk->op.aux1;
  return DG_OK;
}

// ---- vertex updates ------------------------------------------------------------------
int dg_insert_vertices(dg_graph* h, uint64_t count) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (count == 0) return DG_OK;  // InsertVertices.ZeroIsANoop
  const uint64_t new_size = h->size + count;
  if (new_size >= 0xFFFFFFFFull || new_size < h->size)
    return fail(h, DG_ERR_ENGINE, "vertex dictionary: vertex ids are 32-bit");
  if (new_size > h->capacity) {
    // doubling migration (vertex_dictionary.hpp:53-71): target = closest_pow2(size + count)
    const uint64_t target = std::bit_ceil(new_size);
    const size_t words_new = (target + 31) / 32, words_old = (h->capacity + 31) / 32;
    uint32_t *nh = nullptr, *nt = nullptr, *nd = nullptr, *na = nullptr;
    if (cudaMalloc(&nh, target * 4) != cudaSuccess || cudaMalloc(&nt, target * 4) != cudaSuccess ||
        cudaMalloc(&nd, target * 4) != cudaSuccess || cudaMalloc(&na, words_new * 4) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(nh); cudaFree(nt); cudaFree(nd); cudaFree(na);
      cudaGetLastError();
      return fail(h, DG_ERR_ENGINE, "vertex dictionary: arena cannot host capacity " + std::to_string(target));
    }
    cudaMemsetAsync(nh, 0xFF, target * 4, h->stream);
    cudaMemsetAsync(nt, 0xFF, target * 4, h->stream);
    cudaMemsetAsync(nd, 0, target * 4, h->stream);
    cudaMemsetAsync(na, 0, words_new * 4, h->stream);
    cudaMemcpyAsync(nh, h->head, h->capacity * 4, cudaMemcpyDeviceToDevice, h->stream);
    cudaMemcpyAsync(nt, h->tail, h->capacity * 4, cudaMemcpyDeviceToDevice, h->stream);
    cudaMemcpyAsync(nd, h->deg, h->capacity * 4, cudaMemcpyDeviceToDevice, h->stream);
    cudaMemcpyAsync(na, h->alive, words_old * 4, cudaMemcpyDeviceToDevice, h->stream);
    DG_CUDA(h, cudaStreamSynchronize(h->stream));
    cudaFree(h->head); cudaFree(h->tail); cudaFree(h->deg); cudaFree(h->alive);
    h->head = nh; h->tail = nt; h->deg = nd; h->alive = na;
    h->capacity = target;
    h->alive_host.resize((target + 63) / 64, 0ull);
  }
  GraphView g = view(h);
  DG_LAUNCH(h, "vertex_init_kernel", vertex_init_kernel<<<grid_for(h, count, 256), 256, 0, h->stream>>>(g, (uint32_t)h->size, (uint32_t)count));
  for (uint64_t v = h->size; v < new_size; ++v) h->alive_host[v >> 6] |= 1ull << (v & 63);
  h->size = new_size;
  h->alive_count += count;
  DG_CUDA(h, cudaStreamSynchronize(h->stream));
  return DG_OK;
}

int dg_delete_vertices(dg_graph* h, const uint32_t* ids, uint64_t n, uint32_t* skipped,
                       uint64_t* n_skipped) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  uint64_t ns = 0;
  std::vector<uint32_t> winners;
  winners.reserve(n);
  // encounter-order semantics of graph.hpp:255-259: dead / unknown / repeated ids are skipped
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t v = ids[i];
    if (!h->alive_h(v)) {
      if (skipped) skipped[ns] = v;
      ++ns;
      continue;
    }
    h->alive_host[v >> 6] &= ~(1ull << (v & 63));   // (in-call duplicates must see it; restored if the op fails)
    winners.push_back(v);
  }
  auto restore_mirror = [&] {
    for (uint32_t v : winners) h->alive_host[v >> 6] |= 1ull << (v & 63);
  };
  if (n_skipped) *n_skipped = ns;
  if (winners.empty()) return DG_OK;
  int rc = ws_reserve(h, aligned(winners.size() * 4));
  if (rc != DG_OK) { restore_mirror(); return rc; }
  uint32_t* d_ids = ws_alloc<uint32_t>(h, winners.size());
  if (cudaMemcpyAsync(d_ids, winners.data(), winners.size() * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) {
    restore_mirror();
    return fail(h, DG_ERR_CUDA, "delete_vertices: copy of the ids failed");
  }
  if ((rc = op_begin(h, winners.size(), 0)) != DG_OK) { restore_mirror(); return rc; }
  GraphView g = view(h);
  if (h->B == 0) g.reclaim = 0;
  DG_LAUNCH(h, "retire_vertices_kernel", retire_vertices_kernel<<<grid_for(h, winners.size(), 8), 256, 0, h->stream>>>(
      g, d_ids, (uint32_t)winners.size(), h->d_op()));
  rc = op_end(h);
  if (rc != DG_OK) { restore_mirror(); return rc; }   // nothing retired on the device: the mirror follows it
  h->alive_count -= winners.size();
  return DG_OK;
}

// ---- observables -----------------------------------------------------------------------
uint32_t dg_block_size(const dg_graph* h) { return h ? h->B : 0; }
uint64_t dg_logical_size(const dg_graph* h) { return h ? h->size : 0; }
uint64_t dg_vertex_capacity(const dg_graph* h) { return h ? h->capacity : 0; }
uint64_t dg_alive_vertices(const dg_graph* h) { return h ? h->alive_count : 0; }
uint64_t dg_active_edges(const dg_graph* h) {
  if (!h) return 0;
  enter_quiet(h);
  return h->active_edges;
}
int dg_vertex_alive(const dg_graph* h, uint32_t v) { return h && h->alive_h(v) ? 1 : 0; }

int dg_stats_get(dg_graph* h, dg_stats* out) {
  if (!h || !out) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  std::memset(out, 0, sizeof(*out));
  int rc;
  if (h->size > 0 && h->B > 0) {
    if ((rc = op_begin(h, h->size, 0)) != DG_OK) return rc;
    DG_LAUNCH(h, "stats_kernel", stats_kernel<<<grid_for(h, h->size, 256), 256, 0, h->stream>>>(view(h), h->d_op()));
    if ((rc = op_end(h)) != DG_OK) return rc;
    out->adjacency_blocks = h->h_blk->op.aux0;
    out->max_degree = h->h_blk->op.aux1;
  }
  out->logical_size = h->size;
  out->capacity = h->capacity;
  out->alive_vertices = h->alive_count;
  out->active_edges = h->active_edges;
  out->occupied_slots = h->active_edges;
  out->hole_slots = 0;
  out->pool_blocks_created = h->NB;
  out->pool_blocks_in_use = h->NB ? h->blocks_in_use() : 0;
  out->pool_queue_size = h->rear - h->front;
  out->queue_front = h->front;
  out->queue_rear = h->rear;
  out->block_size = h->B;
  out->growth_count = h->growth_count;
  return DG_OK;
}

int dg_memory_get(const dg_graph* h, dg_memory* out) {
  if (!h || !out) return DG_ERR_DATA;
  enter_quiet(h);
  out->dictionary_bytes = h->capacity * 4 + (h->capacity + 31) / 32 * 4;
  out->sentinel_bytes = h->capacity * 8;
  out->pool_bytes = h->NB ? h->blocks_in_use() * ((uint64_t)h->B * 4 + 4) : 0;
  out->queue_bytes = h->NB * 4;
  out->pool_reserved_bytes = h->pool_vm ? h->vm_slab.mapped + h->vm_next.mapped : h->NB * ((uint64_t)h->B * 4 + 4);   // committed device memory
  out->workspace_bytes = h->ws.cap;
  return DG_OK;
}

int dg_last_op_report(const dg_graph* h, dg_op_report* out) {
  if (!h || !out) return DG_ERR_DATA;
  enter_quiet(h);
  *out = h->report;
  return DG_OK;
}

int dg_profile_enable(dg_graph* h, int on) {
  if (!h) return DG_ERR_DATA;
  if (const int erc = enter(h)) return erc;
  cudaStreamSynchronize(h->stream);
  prof_collect(h);
  h->profiling = on != 0;
  if (on) h->prof_acc.clear();
  return DG_OK;
}

const char* dg_profile_report(dg_graph* h) {
  if (!h) return "";
  h->prof_text.clear();
  char line[256];
  for (const auto& kv : h->prof_acc) {
    std::snprintf(line, sizeof line, "%s\t%.6f\t%llu\n", kv.first.c_str(), kv.second.first,
                  (unsigned long long)kv.second.second);
    h->prof_text += line;
  }
  return h->prof_text.c_str();
}

void* dg_stream(const dg_graph* h) { return h ? (void*)h->stream : nullptr; }

int dg_synchronize(dg_graph* h) {
  if (!h) return DG_ERR_DATA;
  if (const int erc = enter(h)) return erc;
  DG_CUDA(h, cudaStreamSynchronize(h->stream));
  return DG_OK;
}

// ---- input-side helpers -------------------------------------------------------------------
int dg_compute_block_size_coo(dg_graph* h, const uint32_t* src, uint64_t n, int mem,
                              uint32_t* out_block_size) {
  if (!h || !out_block_size) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (n == 0) return fail(h, DG_ERR_DATA, "compute_block_size: first batch contains no edges");
  if (n >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  SortPlan plan = make_sort_plan(0, 32);
  WsSizer sz;
  if (mem == DG_MEM_HOST) sz.add<uint32_t>(n);
  sz.add<unsigned long long>(n); sz.add<unsigned long long>(n);
  sz.total += sort_ws_bytes(n, plan.passes);
  sz.add<uint32_t>(n + 1); sz.add<uint32_t>(n + 1);
  sz.total += scan_ws_bytes(n);
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const uint32_t* d_src;
  if ((rc = stage_in(h, src, n, mem, &d_src)) != DG_OK) return rc;
  if ((rc = op_begin(h, n, 0)) != DG_OK) return rc;
  GraphView g = view(h);
  g.size = 0xFFFFFFFFu;
  g.dst_limit = 0xFFFFFFFFu;
  unsigned long long* keys = ws_alloc<unsigned long long>(h, n);
  unsigned long long* keys_alt = ws_alloc<unsigned long long>(h, n);
  SortScratch sc = sort_prepare(h, n, plan);
  DG_LAUNCH(h, "pack_coo_kernel<query>", pack_coo_kernel<kPackQuery, false><<<grid_for(h, n, 256 * 8), 256, 0, h->stream>>>(
      g, d_src, d_src, (uint32_t)n, keys, nullptr, plan, sc.hist, h->d_op()));
  sort_keys(h, &keys, &keys_alt, nullptr, nullptr, n, plan, sc, true);
  uint32_t* run_start = ws_alloc<uint32_t>(h, n + 1);
  uint32_t* run_src = ws_alloc<uint32_t>(h, n + 1);
  launch_scan(h, "scan_kernel<runs>", n, d_n_input(h), RunsIn{keys}, RunsOut{keys, run_start, run_src},
              RunsFin{run_start, h->d_op(), (uint32_t)n});
  if ((rc = op_end(h)) != DG_OK) return rc;
  const uint64_t T = h->h_blk->op.n_runs;
  const uint64_t rounded = (n + T / 2) / T;
  *out_block_size = (uint32_t)std::max<uint64_t>(1, rounded);
  return DG_OK;
}

int dg_gen_rmat(dg_graph* h, uint32_t scale, uint64_t seed, uint64_t first_index, uint64_t n,
                uint32_t thr_a, uint32_t thr_ab, uint32_t thr_abc, uint32_t* src_dev,
                uint32_t* dst_dev) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (scale == 0 || scale > 32) return fail(h, DG_ERR_DATA, "rmat: scale must be in [1, 32]");
  if (n == 0) return DG_OK;
  DG_LAUNCH(h, "rmat_kernel", rmat_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(scale, seed, first_index, n, thr_a,
                                                              thr_ab, thr_abc, src_dev, dst_dev));
  DG_CUDA(h, cudaGetLastError());
  return DG_OK;
}

int dg_coo_to_csr(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, int mem,
                  uint64_t vertex_count, uint64_t* offsets_dev, uint32_t* destinations_dev) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (n >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  if (vertex_count == 0 || vertex_count >= 0xFFFFFFFFull)
    return fail(h, DG_ERR_DATA, "coo_to_csr: bad vertex count");
  SortPlan plan = make_sort_plan(0, bits_for(vertex_count - 1));
  WsSizer sz;
  if (mem == DG_MEM_HOST) { sz.add<uint32_t>(n); sz.add<uint32_t>(n); }
  sz.add<unsigned long long>(n + 1); sz.add<unsigned long long>(n + 1);
  sz.total += sort_ws_bytes(std::max<uint64_t>(n, 1), plan.passes);
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  const uint32_t *d_src, *d_dst;
  if ((rc = stage_in(h, src, n, mem, &d_src)) != DG_OK) return rc;
  if ((rc = stage_in(h, dst, n, mem, &d_dst)) != DG_OK) return rc;
  if ((rc = op_begin(h, n, 0)) != DG_OK) return rc;
  GraphView g = view(h);
  g.size = (uint32_t)vertex_count;
  g.dst_limit = 0xFFFFFFFFu;
  unsigned long long* keys = ws_alloc<unsigned long long>(h, n + 1);
  unsigned long long* keys_alt = ws_alloc<unsigned long long>(h, n + 1);
  if (n > 0) {
    SortScratch sc = sort_prepare(h, n, plan);
    DG_LAUNCH(h, "pack_coo_kernel<delete>", pack_coo_kernel<kPackDelete, false><<<grid_for(h, n, 256 * 8), 256, 0, h->stream>>>(
        g, d_src, d_dst, (uint32_t)n, keys, nullptr, plan, sc.hist, h->d_op()));
    sort_keys(h, &keys, &keys_alt, nullptr, nullptr, n, plan, sc, true);
  }
  DG_LAUNCH(h, "keys_to_offsets_kernel", keys_to_offsets_kernel<<<grid_for(h, n + 1, 256), 256, 0, h->stream>>>(
      keys, (uint32_t)n, vertex_count, reinterpret_cast<unsigned long long*>(offsets_dev),
      destinations_dev, h->d_op()));
  return op_end(h);
}

uint32_t dg_owner_perm(uint32_t v, uint32_t bits) { return owner_perm(v, bits); }
uint32_t dg_owner_perm_inv(uint32_t p, uint32_t bits) { return owner_perm_inv(p, bits); }

int dg_set_dst_limit(dg_graph* h, uint64_t limit) {
  if (!h) return DG_ERR_DATA;
  if (limit > 0xFFFFFFFFull) return fail(h, DG_ERR_DATA, "dst limit must fit 32 bits");
  h->dst_limit_override = limit;
  return DG_OK;
}

int dg_route_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t world,
                 uint32_t bits, uint64_t vertex_count, uint32_t* out_src_local, uint32_t* out_dst,
                 uint32_t* out_index, uint64_t* counts_host) {
  if (!h) return DG_ERR_DATA;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (world == 0 || world > 65536) return fail(h, DG_ERR_DATA, "route: world must be in [1, 65536]");
  if (bits > 32 || vertex_count > (bits >= 32 ? (1ull << 32) : (1ull << bits)))
    return fail(h, DG_ERR_DATA, "route: vertex_count exceeds 2^bits");
  if (n >= (1ull << 31)) return fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  for (uint32_t w = 0; w < world; ++w) counts_host[w] = 0;
  if (n == 0) return DG_OK;
  SortPlan plan = make_sort_plan(0, bits_for(world - 1));
  WsSizer sz;
  sz.add<unsigned long long>(n); sz.add<unsigned long long>(n);
  sz.total += sort_ws_bytes(n, std::max(plan.passes, 1));
  sz.add<unsigned long long>(world + 2);
  int rc = ws_reserve(h, sz.total);
  if (rc != DG_OK) return rc;
  if ((rc = op_begin(h, n, 0)) != DG_OK) return rc;
  unsigned long long* keys = ws_alloc<unsigned long long>(h, n);
  unsigned long long* keys_alt = ws_alloc<unsigned long long>(h, n);
  unsigned long long* d_counts = ws_alloc<unsigned long long>(h, world + 2);
  DG_LAUNCH(h, "route_keys_kernel", route_keys_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(
      src, (uint32_t)n, world, bits, (uint32_t)std::min<uint64_t>(vertex_count, 0xFFFFFFFFull), keys, h->d_op()));
  SortScratch sc = sort_prepare(h, n, plan);
  sort_keys(h, &keys, &keys_alt, nullptr, nullptr, n, plan, sc, false);
  DG_LAUNCH(h, "route_gather_kernel", route_gather_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(
      keys, src, dst, (uint32_t)n, world, bits, out_src_local, out_dst, out_index, d_counts, h->d_op()));
  std::vector<unsigned long long> ends(world + 1);
  DG_CUDA(h, cudaMemcpyAsync(ends.data(), d_counts, (world + 1) * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, h->stream));
  if ((rc = op_end(h)) != DG_OK) return rc;
  for (uint32_t w = 0; w < world; ++w) counts_host[w] = ends[w + 1] - ends[w];
  return DG_OK;
}

// ---- fused routing + exchange over peer memory ------------------------------------------------
namespace {
struct ExchangeLayout {
  size_t words, src[2], dst[2], idx[2], from[2], ans[2], total;
};
ExchangeLayout exchange_layout(uint64_t cap) {
  ExchangeLayout l{};
  size_t off = 0;
  l.words = off; off += 256;
  for (int s = 0; s < 2; ++s) {
    l.src[s] = off; off += aligned(cap * 4);
    l.dst[s] = off; off += aligned(cap * 4);
    l.idx[s] = off; off += aligned(cap * 4);
    l.from[s] = off; off += aligned(cap * 4);
    l.ans[s] = off; off += aligned(cap);
  }
  l.total = off;
  return l;
}
static_assert(sizeof(RoundWords) <= 256, "round words fit their slot");
void exchange_bind(dg_exchange* x, uint32_t peer, char* base) {
  const ExchangeLayout l = exchange_layout(x->capacity);
  x->pb.words[peer] = reinterpret_cast<RoundWords*>(base + l.words);
  for (int s = 0; s < 2; ++s) {
    x->pb.src[peer][s] = reinterpret_cast<uint32_t*>(base + l.src[s]);
    x->pb.dst[peer][s] = reinterpret_cast<uint32_t*>(base + l.dst[s]);
    x->pb.idx[peer][s] = reinterpret_cast<uint32_t*>(base + l.idx[s]);
    x->pb.from[peer][s] = reinterpret_cast<uint32_t*>(base + l.from[s]);
    x->pb.ans[peer][s] = reinterpret_cast<uint8_t*>(base + l.ans[s]);
  }
}
int exchange_ready(dg_exchange* x) {
  for (uint32_t p = 0; p < x->world; ++p)
    if (x->pb.words[p] == nullptr) return fail(x->h, DG_ERR_ENGINE, "exchange: peer " + std::to_string(p) + " not set");
  return DG_OK;
}
}  // namespace


int dg_exchange_create(dg_graph* h, uint32_t rank, uint32_t world, uint64_t capacity, dg_exchange** out) {
  if (!h || !out) return DG_ERR_DATA;
  *out = nullptr;
  h->last_error.clear();
  if (const int erc = enter(h)) return erc;
  if (world == 0 || world > (uint32_t)kMaxPeers || rank >= world)
    return fail(h, DG_ERR_DATA, "exchange: world must be in [1, 16] and rank < world");
  if (capacity == 0 || capacity >= (1ull << 31)) return fail(h, DG_ERR_DATA, "exchange: bad capacity");
  dg_exchange* x = new (std::nothrow) dg_exchange();
  if (!x) return fail(h, DG_ERR_ENGINE, "exchange: out of host memory");
  x->h = h;
  x->rank = rank;
  x->world = world;
  x->capacity = capacity;
  x->bytes = exchange_layout(capacity).total;
  if (cudaMalloc(&x->base, x->bytes) != cudaSuccess) {
    cudaGetLastError();
    delete x;
    return fail(h, DG_ERR_ENGINE, "exchange: device allocation failed");
  }
  cudaMemsetAsync(x->base, 0, 256, h->stream);
  x->pb.capacity = capacity;
  x->pb.world = world;
  x->pb.rank = rank;
  exchange_bind(x, rank, x->base);
  DG_CUDA(h, cudaStreamSynchronize(h->stream));
  *out = x;
  return DG_OK;
}

void dg_exchange_destroy(dg_exchange* x) {
  if (!x) return;
  cudaSetDevice(x->h->device);
  cudaStreamSynchronize(x->h->stream);
  if (x->h->agree_x == x) x->h->agree_x = nullptr;
  for (int p = 0; p < kMaxPeers; ++p)
    if (x->peer_base[p]) cudaIpcCloseMemHandle(x->peer_base[p]);
  cudaFree(x->base);
  cudaGetLastError();
  delete x;
}

int dg_exchange_ipc_handle(dg_exchange* x, void* handle_out) {
  if (!x || !handle_out) return DG_ERR_DATA;
  static_assert(sizeof(cudaIpcMemHandle_t) == DG_IPC_HANDLE_BYTES, "IPC handle size");
  cudaSetDevice(x->h->device);
  cudaIpcMemHandle_t hd;
  DG_CUDA(x->h, cudaIpcGetMemHandle(&hd, x->base));
  std::memcpy(handle_out, &hd, sizeof(hd));
  return DG_OK;
}

int dg_exchange_set_peer(dg_exchange* x, uint32_t peer_rank, const void* handle) {
  if (!x || !handle) return DG_ERR_DATA;
  if (peer_rank >= x->world) return fail(x->h, DG_ERR_DATA, "exchange: peer rank out of range");
  if (peer_rank == x->rank) return DG_OK;  // own buffers are bound at creation
  cudaSetDevice(x->h->device);
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  void* p = nullptr;
  DG_CUDA(x->h, cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
  x->peer_base[peer_rank] = p;
  exchange_bind(x, peer_rank, static_cast<char*>(p));
  return DG_OK;
}

int dg_exchange_attach(dg_exchange* x, int on) {
  if (!x) return DG_ERR_DATA;
  x->h->agree_x = on ? x : nullptr;
  return DG_OK;
}

int dg_exchange_push_coo(dg_exchange* x, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t bits,
                         uint64_t vertex_count) {
  if (!x) return DG_ERR_DATA;
  dg_graph* h = x->h;
  h->last_error.clear();
  cudaSetDevice(h->device);
  int rc;
  if ((rc = exchange_ready(x)) != DG_OK) return rc;
  // host-side rejections still ARRIVE (with their status), so that no peer waits for this rank
  int early = DG_OK;
  if (n >= (1ull << 31)) early = fail(h, DG_ERR_ENGINE, "batch too large (n must be < 2^31)");
  else if (n > x->capacity) early = fail(h, DG_ERR_ENGINE, "exchange: batch larger than the exchange capacity");   // origin indices address the answer buffer
  else if (bits > 32 || vertex_count > (bits >= 32 ? (1ull << 32) : (1ull << bits)))
    early = fail(h, DG_ERR_DATA, "exchange: vertex_count exceeds 2^bits");
  const std::string early_msg = h->last_error;
  if ((rc = op_begin(h, n, 0)) != DG_OK) return rc;
  if (early != DG_OK) {
    cudaMemsetAsync(&h->d_op()->err, early == DG_ERR_DATA ? 0x02 : 0x03, 1, h->stream);   // (low byte: the status code)
  } else if (n > 0) {
    DG_LAUNCH(h, "exchange_validate_kernel", exchange_validate_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(
        src, (uint32_t)n, (uint32_t)std::min<uint64_t>(vertex_count, 0xFFFFFFFFull), h->d_op()));
    DG_LAUNCH(h, "exchange_push_kernel", exchange_push_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(
        x->pb, x->set(), src, dst, (uint32_t)n, bits, h->d_op()));
  }
  DG_LAUNCH(h, "exchange_signal_kernel", exchange_signal_kernel<<<1, 32, 0, h->stream>>>(x->pb, x->set(), 0, h->d_op()));
  rc = op_end(h);
  if (early != DG_OK) {
    h->last_error = early_msg;
    return early;
  }
  return rc;
}

int dg_exchange_received(dg_exchange* x, uint64_t* n, uint32_t** src_local, uint32_t** dst,
                         uint32_t** origin_index, uint32_t** origin_rank) {
  if (!x || !n) return DG_ERR_DATA;
  dg_graph* h = x->h;
  cudaSetDevice(h->device);
  *n = 0;
  int rc;
  if ((rc = op_begin(h, 0, 0)) != DG_OK) return rc;
  DG_LAUNCH(h, "exchange_wait_kernel", exchange_wait_kernel<<<1, 32, 0, h->stream>>>(x->pb, x->set(), 0, h->d_op()));
  if ((rc = op_end(h)) != DG_OK) return rc;
  const uint64_t agreed = h->h_blk->op.aux0, c = h->h_blk->op.aux1;
  const int s = x->set();
  if (src_local) *src_local = x->pb.src[x->rank][s];
  if (dst) *dst = x->pb.dst[x->rank][s];
  if (origin_index) *origin_index = x->pb.idx[x->rank][s];
  if (origin_rank) *origin_rank = x->pb.from[x->rank][s];
  if (agreed != 0)
    return fail(h, (int)agreed, agreed == DG_ERR_DATA ? "sharded batch: a rank rejected the batch while routing (source id out of range)"
                                                       : "sharded batch: a rank failed while routing (receive buffer full, or a peer never arrived)");
  if (c > x->capacity) return fail(h, DG_ERR_ENGINE, "exchange: receive buffer overflow");
  *n = c;
  return DG_OK;
}

int dg_exchange_agree(dg_exchange* x, int local_status, int* agreed) {
  if (!x) return DG_ERR_DATA;
  dg_graph* h = x->h;
  cudaSetDevice(h->device);
  int rc;
  if ((rc = exchange_ready(x)) != DG_OK) return rc;
  if ((rc = op_begin(h, 0, 0)) != DG_OK) return rc;
  if (local_status != 0) cudaMemsetAsync(&h->d_op()->err, local_status == DG_ERR_DATA ? 0x02 : 0x03, 1, h->stream);
  DG_LAUNCH(h, "exchange_agree_kernel", exchange_agree_kernel<<<1, 32, 0, h->stream>>>(x->pb, x->set(), h->d_op(), h->d_state(), 0));
  rc = op_end(h);
  const int a = (int)h->h_blk->op.aux0;
  if (agreed) *agreed = a;
  if (rc != DG_OK && local_status == 0 && a != 0)
    return fail(h, a, "sharded batch: rejected on another rank");
  return a != 0 ? a : DG_OK;
}

int dg_exchange_push_answers(dg_exchange* x, const uint8_t* answers, uint64_t n) {
  if (!x) return DG_ERR_DATA;
  dg_graph* h = x->h;
  cudaSetDevice(h->device);
  const int s = x->set();
  if (n > 0) {
    DG_LAUNCH(h, "exchange_answers_kernel", exchange_answers_kernel<<<grid_for(h, n, 256 * 4), 256, 0, h->stream>>>(
        x->pb, s, answers, x->pb.idx[x->rank][s], x->pb.from[x->rank][s], (uint32_t)n));
  }
  DG_LAUNCH(h, "exchange_signal_kernel", exchange_signal_kernel<<<1, 32, 0, h->stream>>>(x->pb, s, 2, h->d_op()));
  DG_CUDA(h, cudaGetLastError());
  return DG_OK;
}

int dg_exchange_answers(dg_exchange* x, uint8_t* out, uint64_t n, int mem) {
  if (!x || (!out && n)) return DG_ERR_DATA;
  dg_graph* h = x->h;
  if (n > x->capacity) return fail(h, DG_ERR_DATA, "exchange: more answers than the buffer holds");
  cudaSetDevice(h->device);
  int rc;
  if ((rc = op_begin(h, 0, 0)) != DG_OK) return rc;
  DG_LAUNCH(h, "exchange_wait_kernel", exchange_wait_kernel<<<1, 32, 0, h->stream>>>(x->pb, x->set(), 2, h->d_op()));
  if (n)
    DG_CUDA(h, cudaMemcpyAsync(out, x->pb.ans[x->rank][x->set()], n,
                               mem == DG_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, h->stream));
  if ((rc = op_end(h)) != DG_OK) return rc;
  if (h->h_blk->op.aux0 != 0) return fail(h, DG_ERR_ENGINE, "sharded query: a peer's answers never arrived");
  return DG_OK;
}

int dg_exchange_end_round(dg_exchange* x) {
  if (!x) return DG_ERR_DATA;
  dg_graph* h = x->h;
  cudaSetDevice(h->device);
  // this round's set is consumed: its cursor goes back to zero (in stream order, after the local op that read it)
  DG_CUDA(h, cudaMemsetAsync(&x->pb.words[x->rank]->cursor[x->set()], 0, sizeof(unsigned long long), h->stream));
  x->epoch += 1;
  return DG_OK;
}

int dg_digest_global(dg_graph* h, uint32_t rank, uint32_t world, uint32_t bits, uint64_t* out_digest, uint64_t* out_entries) {
  if (!h || world == 0 || rank >= world) return DG_ERR_DATA;
  h->last_error.clear();
  cudaSetDevice(h->device);
  const uint64_t V = h->size;
  if (out_digest) *out_digest = 0;
  if (out_entries) *out_entries = 0;
  if (V == 0 || h->B == 0) return DG_OK;
  int rc = ws_reserve(h, worklist_ws(h, V, 0));
  if (rc != DG_OK) return rc;
  if ((rc = op_begin(h, V, V)) != DG_OK) return rc;
  GraphView g = view(h);
  BatchView b{nullptr, nullptr, nullptr, nullptr, nullptr};
  Worklist w = enqueue_enumerate(h, b, V, 0, 0);
  const uint64_t wl_bound = std::max<uint64_t>(1, h->blocks_in_use());
  DG_LAUNCH(h, "digest_global_kernel", digest_global_kernel<<<grid_for(h, wl_bound, 8), 256, 0, h->stream>>>(
      g, w.wl_off, w.wl_handle, w.wl_run, w.run_deg, rank, world, bits, h->d_op()));
  if ((rc = op_end(h)) != DG_OK) return rc;
  if (out_digest) *out_digest = h->h_blk->op.aux0;
  if (out_entries) *out_entries = h->h_blk->op.aux1;
  return DG_OK;
}

// ---- host -> device batch ingest ----------------------------------------------
// The reference harness feeds batches one after the other (io/workload.hpp:141-155).  At ~0.1-0.3 ms
// of device time per 1M-entry batch the 8 MB PCIe copy of a batch costs as much as the op itself,
// so the copy of batch k+1 runs on its own stream while batch k executes: a small ring of device
// slots, one copy-done event per slot the op stream waits on, one slot-free event the copy stream
// waits on before a slot is overwritten.
struct dg_ingest {
  dg_graph* h = nullptr;
  uint64_t capacity = 0;   // entries per slot
  uint32_t depth = 0;
  cudaStream_t copy = nullptr;
  std::vector<uint32_t*> src, dst;
  std::vector<uint64_t> n;
  std::vector<cudaEvent_t> filled, freed;
  std::vector<int> state;  // 0 free, 1 staged
  uint32_t next = 0;
};

int dg_ingest_create(dg_graph* h, uint64_t max_entries, uint32_t depth, dg_ingest** out) {
  if (!h || !out || depth == 0 || max_entries == 0) return fail(h, DG_ERR_DATA, "ingest: bad arguments");
  *out = nullptr;
  cudaSetDevice(h->device);
  dg_ingest* q = new (std::nothrow) dg_ingest();
  if (!q) return fail(h, DG_ERR_ENGINE, "ingest: out of host memory");
  q->h = h;
  q->capacity = max_entries;
  q->depth = depth;
  bool ok = cudaStreamCreateWithFlags(&q->copy, cudaStreamNonBlocking) == cudaSuccess;
  for (uint32_t i = 0; ok && i < depth; ++i) {
    uint32_t *s = nullptr, *d = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    ok = cudaMalloc(&s, max_entries * 4) == cudaSuccess && cudaMalloc(&d, max_entries * 4) == cudaSuccess &&
         cudaEventCreateWithFlags(&a, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&b, cudaEventDisableTiming) == cudaSuccess;
    q->src.push_back(s); q->dst.push_back(d); q->filled.push_back(a); q->freed.push_back(b);
    q->n.push_back(0); q->state.push_back(0);
  }
  if (!ok) {
    cudaGetLastError();
    dg_ingest_destroy(q);
    return fail(h, DG_ERR_ENGINE, "ingest: device allocation failed");
  }
  *out = q;
  return DG_OK;
}

void dg_ingest_destroy(dg_ingest* q) {
  if (!q) return;
  cudaSetDevice(q->h->device);
  drain(q->h);   // submitted ops may still read the slots
  if (q->copy) { cudaStreamSynchronize(q->copy); cudaStreamDestroy(q->copy); }
  for (auto p : q->src) cudaFree(p);
  for (auto p : q->dst) cudaFree(p);
  for (auto e : q->filled) if (e) cudaEventDestroy(e);
  for (auto e : q->freed) if (e) cudaEventDestroy(e);
  cudaGetLastError();
  delete q;
}

int dg_ingest_stage_coo(dg_ingest* q, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t* slot_out) {
  if (!q || !slot_out || (n && (!src || !dst))) return DG_ERR_DATA;
  dg_graph* h = q->h;
  cudaSetDevice(h->device);
  if (n > q->capacity) return fail(h, DG_ERR_DATA, "ingest: batch larger than the slot capacity");
  const uint32_t s = q->next;
  if (q->state[s] != 0) return fail(h, DG_ERR_ENGINE, "ingest: every slot holds a staged batch (run one first)");
  // the op that last read this slot must have finished before the slot is overwritten
  DG_CUDA(h, cudaStreamWaitEvent(q->copy, q->freed[s], 0));
  if (n) {
    DG_CUDA(h, cudaMemcpyAsync(q->src[s], src, n * 4, cudaMemcpyHostToDevice, q->copy));
    DG_CUDA(h, cudaMemcpyAsync(q->dst[s], dst, n * 4, cudaMemcpyHostToDevice, q->copy));
  }
  DG_CUDA(h, cudaEventRecord(q->filled[s], q->copy));
  q->n[s] = n;
  q->state[s] = 1;
  q->next = (s + 1) % q->depth;
  *slot_out = s;
  return DG_OK;
}

static int ingest_run(dg_ingest* q, uint32_t slot, bool is_insert) {
  if (!q || slot >= q->depth) return DG_ERR_DATA;
  dg_graph* h = q->h;
  cudaSetDevice(h->device);
  if (q->state[slot] != 1) return fail(h, DG_ERR_DATA, "ingest: slot holds no staged batch");
  DG_CUDA(h, cudaStreamWaitEvent(h->stream, q->filled[slot], 0));
  const int rc = is_insert ? dg_insert_batch_coo(h, q->src[slot], q->dst[slot], q->n[slot], DG_MEM_DEVICE)
                           : dg_delete_batch_coo(h, q->src[slot], q->dst[slot], q->n[slot], DG_MEM_DEVICE);
  cudaEventRecord(q->freed[slot], h->stream);
  q->state[slot] = 0;
  return rc;
}
int dg_ingest_reset(dg_ingest* q) {
  if (!q) return DG_ERR_DATA;
  dg_graph* h = q->h;
  cudaSetDevice(h->device);
  DG_CUDA(h, cudaStreamSynchronize(q->copy));
  for (auto& st : q->state) st = 0;
  q->next = 0;
  return DG_OK;
}
int dg_ingest_insert(dg_ingest* q, uint32_t slot) { return ingest_run(q, slot, true); }
int dg_ingest_delete(dg_ingest* q, uint32_t slot) { return ingest_run(q, slot, false); }
// the same without the host wait: the op is submitted (dg_submit_*_coo), the slot is handed back by an event
static int ingest_submit(dg_ingest* q, uint32_t slot, bool is_insert, uint64_t* ticket) {
  if (!q || slot >= q->depth) return DG_ERR_DATA;
  dg_graph* h = q->h;
  cudaSetDevice(h->device);
  if (q->state[slot] != 1) return fail(h, DG_ERR_DATA, "ingest: slot holds no staged batch");
  DG_CUDA(h, cudaStreamWaitEvent(h->stream, q->filled[slot], 0));
  h->input_ready = q->filled[slot];   // (an early count on the side stream waits for the slot's copy too)
  const int rc = submit_coo(h, q->src[slot], q->dst[slot], q->n[slot], is_insert, ticket);
  h->input_ready = nullptr;
  cudaEventRecord(q->freed[slot], h->stream);
  q->state[slot] = 0;
  return rc;
}
int dg_ingest_submit_insert(dg_ingest* q, uint32_t slot, uint64_t* ticket) { return ingest_submit(q, slot, true, ticket); }
int dg_ingest_submit_delete(dg_ingest* q, uint32_t slot, uint64_t* ticket) { return ingest_submit(q, slot, false, ticket); }

}  // extern "C"
