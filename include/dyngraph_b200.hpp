// dyngraph_b200.hpp — C++ host-side mirror of the reference's operator API
// over the C ABI of libdyngraph_b200.so (include/dyngraph_b200.h).
//
// `dyngraph_b200::DynamicGraph` has the constructor, method names, argument
// meaning and error behaviour of `dyngraph::DynamicGraph`
// (reference: proj/include/dyngraph/graph.hpp:80-317), so code written against
// the reference — run_workload (io/workload.hpp:132-181), run_one_workload
// (verify.hpp:151-242), oracle_compare (oracle.hpp:113-160) — compiles against
// either by switching the type.  Header-only, C++17, no CUDA headers needed:
// every method is one call into the shared library; failures come back as the
// reference's exception classes (types.hpp:21-32).  There is NO CPU fallback:
// if the library is missing the program does not link.
//
// Not mirrored (physical layout, reported rather than compared — SURVEY.md §8a):
// arena(), dictionary(), pool(), sentinel_of(), adjacency_blocks().
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dyngraph_b200.h"

namespace dyngraph_b200 {

using VertexId = std::uint32_t;                       // types.hpp:11
inline constexpr VertexId kInvalidVertex = 0xFFFFFFFFu;  // types.hpp:16

// types.hpp:21-32
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DataError : public Error {
 public:
  using Error::Error;
};
class EngineError : public Error {
 public:
  using Error::Error;
};

enum class BatchKind { Insert, Delete };  // csr.hpp:12

// csr.hpp:17-25
struct CsrBatch {
  BatchKind kind = BatchKind::Insert;
  std::vector<std::uint64_t> offsets;
  std::vector<VertexId> destinations;
  std::uint64_t vertex_count() const { return offsets.empty() ? 0 : offsets.size() - 1; }
  std::uint64_t edge_count() const { return destinations.size(); }
  std::uint64_t degree(VertexId v) const { return offsets[v + 1] - offsets[v]; }
};

// graph.hpp:33-39
struct BatchPlan {
  std::vector<std::uint64_t> blocks_required;
  std::vector<std::uint64_t> prefix_sum;
  std::vector<std::uint32_t> space_remaining;
  std::uint64_t total_blocks() const { return prefix_sum.empty() ? 0 : prefix_sum.back(); }
};

// csr.hpp:29-45 — stable counting sort of (source, destination) pairs
inline CsrBatch csr_from_pairs(BatchKind kind, std::uint64_t vertex_count,
                               const std::vector<std::pair<VertexId, VertexId>>& edges) {
  CsrBatch b;
  b.kind = kind;
  b.offsets.assign(vertex_count + 1, 0);
  for (const auto& e : edges) {
    if (e.first >= vertex_count) throw DataError("csr batch: source out of range");
    ++b.offsets[e.first + 1];
  }
  for (std::uint64_t v = 0; v < vertex_count; ++v) b.offsets[v + 1] += b.offsets[v];
  b.destinations.resize(edges.size());
  std::vector<std::uint64_t> cursor(b.offsets.begin(), b.offsets.end() - 1);
  for (const auto& e : edges) b.destinations[cursor[e.first]++] = e.second;
  return b;
}

// graph.hpp:23-28; the arena is real device memory here, so the budget is the
// byte size of the edge-block pool (arena_bytes * pool.initial_fraction there).
struct GraphConfig {
  int device = 0;
  std::uint64_t pool_bytes = 0;   // 0 => library default (1 GiB)
  std::uint64_t pool_blocks = 0;  // exact block count; overrides pool_bytes
  bool reclaim_on_delete = true;  // graph.hpp:26
  void* stream = nullptr;         // cudaStream_t; nullptr => library-owned stream
  std::uint64_t workspace_bytes = 0;  // per-op scratch reserved at construction
  // GrowthPolicy (block_pool.hpp:18-29): pool_max_blocks plays the arena's role (0 => fixed pool)
  std::uint64_t pool_max_blocks = 0;
  float trigger_fraction = 0.8f;
  float growth_fraction = 0.25f;
};

struct GraphStats {  // graph.hpp:54-70 (reported, not compared)
  std::uint64_t logical_size = 0, capacity = 0, alive_vertices = 0, active_edges = 0;
  std::uint64_t adjacency_blocks = 0, occupied_slots = 0, hole_slots = 0;
  std::uint64_t pool_blocks_created = 0, pool_blocks_in_use = 0, pool_queue_size = 0;
  std::uint64_t max_degree = 0;
  std::uint32_t block_size = 0;
  std::uint32_t pool_growths = 0;   // graph.hpp:66 (growth rounds)
};

class DynamicGraph {
 public:
  // graph.hpp:84-91
  DynamicGraph(const GraphConfig& config, std::uint64_t initial_vertex_count, std::uint32_t block_size) {
    dg_config c{};
    c.device = config.device;
    c.flags = config.reclaim_on_delete ? 0u : DG_FLAG_NO_RECLAIM;
    c.pool_bytes = config.pool_bytes;
    c.pool_blocks = config.pool_blocks;
    c.stream = config.stream;
    c.workspace_bytes = config.workspace_bytes;
    c.pool_max_blocks = config.pool_max_blocks;
    c.trigger_fraction = config.trigger_fraction;
    c.growth_fraction = config.growth_fraction;
    const int rc = dg_create(&c, initial_vertex_count, block_size, &h_);
    if (rc != DG_OK) raise(rc, dg_last_error(nullptr));
  }
  ~DynamicGraph() { dg_destroy(h_); }
  DynamicGraph(const DynamicGraph&) = delete;             // graph.hpp:93-94
  DynamicGraph& operator=(const DynamicGraph&) = delete;

  // graph.hpp:96-108
  std::uint32_t block_size() const { return dg_block_size(h_); }
  std::uint64_t logical_size() const { return dg_logical_size(h_); }
  std::uint64_t vertex_capacity() const { return dg_vertex_capacity(h_); }
  std::uint64_t alive_vertices() const { return dg_alive_vertices(h_); }
  std::uint64_t active_edges() const { return dg_active_edges(h_); }
  bool vertex_alive(VertexId v) const { return dg_vertex_alive(h_, v) != 0; }

  // graph.hpp:135-160
  BatchPlan plan_batch(const CsrBatch& batch) const {
    if (batch.kind != BatchKind::Insert) throw DataError("plan_batch: expected an insert batch");
    BatchPlan plan;
    const std::uint64_t n = batch.vertex_count();
    plan.blocks_required.resize(n);
    plan.prefix_sum.resize(n);
    plan.space_remaining.resize(n);
    check(dg_plan_batch_csr(h_, batch.offsets.data(), batch.offsets.size(), batch.destinations.data(),
                            batch.destinations.size(), DG_MEM_HOST, plan.blocks_required.data(),
                            plan.prefix_sum.data(), plan.space_remaining.data(), nullptr));
    return plan;
  }
  // graph.hpp:167-188
  void insert_batch(const CsrBatch& batch) {
    if (batch.kind != BatchKind::Insert) throw DataError("plan_batch: expected an insert batch");
    check(dg_insert_batch_csr(h_, batch.offsets.data(), batch.offsets.size(), batch.destinations.data(),
                              batch.destinations.size(), DG_MEM_HOST));
  }
  // graph.hpp:195-222
  void delete_batch(const CsrBatch& batch) {
    if (batch.kind != BatchKind::Delete) throw DataError("delete_batch: expected a delete batch");
    check(dg_delete_batch_csr(h_, batch.offsets.data(), batch.offsets.size(), batch.destinations.data(),
                              batch.destinations.size(), DG_MEM_HOST));
  }
  // O(batch) forms of the same two operators (no V+1 offsets array)
  void insert_pairs(const VertexId* src, const VertexId* dst, std::uint64_t n, int mem = DG_MEM_HOST) {
    check(dg_insert_batch_coo(h_, src, dst, n, mem));
  }
  void delete_pairs(const VertexId* src, const VertexId* dst, std::uint64_t n, int mem = DG_MEM_HOST) {
    check(dg_delete_batch_coo(h_, src, dst, n, mem));
  }

  // the same two operators SUBMITTED: device arrays, no host wait per batch (dg_submit_*_coo); flush() waits for
  // all of them, throws the first failure and returns how many were applied (ops behind a failed one are not)
  std::uint64_t submit_insert_pairs(const VertexId* src_dev, const VertexId* dst_dev, std::uint64_t n) {
    std::uint64_t ticket = 0;
    check(dg_submit_insert_coo(h_, src_dev, dst_dev, n, &ticket));
    return ticket;
  }
  std::uint64_t submit_delete_pairs(const VertexId* src_dev, const VertexId* dst_dev, std::uint64_t n) {
    std::uint64_t ticket = 0;
    check(dg_submit_delete_coo(h_, src_dev, dst_dev, n, &ticket));
    return ticket;
  }
  std::uint64_t flush() {
    std::uint64_t applied = 0;
    check(dg_flush(h_, &applied));
    return applied;
  }

  // graph.hpp:228-241
  bool query_edge(VertexId source, VertexId destination) const {
    std::uint8_t out = 0;
    check(dg_query_edges(h_, &source, &destination, 1, &out, DG_MEM_HOST));
    return out != 0;
  }
  std::vector<std::uint8_t> query_edges(const std::vector<VertexId>& src, const std::vector<VertexId>& dst) const {
    std::vector<std::uint8_t> out(src.size());
    if (!src.empty()) check(dg_query_edges(h_, src.data(), dst.data(), src.size(), out.data(), DG_MEM_HOST));
    return out;
  }

  // graph.hpp:246
  void insert_vertices(std::uint64_t count) { check(dg_insert_vertices(h_, count)); }
  // graph.hpp:252-276 — returns the skipped ids in encounter order
  std::vector<VertexId> delete_vertices(const std::vector<VertexId>& ids) {
    std::vector<VertexId> skipped(ids.size());
    std::uint64_t ns = 0;
    check(dg_delete_vertices(h_, ids.data(), ids.size(), skipped.data(), &ns));
    skipped.resize(ns);
    return skipped;
  }

  // graph.hpp:116-129 (traversal order; sorted = canonical order of oracle_compare)
  std::vector<VertexId> active_destinations(VertexId v, bool sorted = false) const {
    if (v >= logical_size()) return {};
    std::vector<VertexId> out(64);
    std::uint64_t n = 0;
    int rc = dg_active_destinations(h_, v, out.data(), out.size(), &n, DG_MEM_HOST);
    if (rc == DG_ERR_DATA && n > out.size()) {   // the degree came back: once more with room for it
      out.resize(n);
      rc = dg_active_destinations(h_, v, out.data(), out.size(), &n, DG_MEM_HOST);
    }
    check(rc);
    out.resize(n);
    if (sorted) std::sort(out.begin(), out.end());
    return out;
  }
  // every vertex's active_destinations as one CSR
  void export_csr(std::vector<std::uint64_t>& offsets, std::vector<VertexId>& destinations, bool sorted) const {
    offsets.assign(logical_size() + 1, 0);
    check(dg_export_csr(h_, offsets.data(), nullptr, 0, sorted ? 1 : 0, DG_MEM_HOST));
    destinations.assign(offsets.back(), 0);
    if (!destinations.empty())
      check(dg_export_csr(h_, offsets.data(), destinations.data(), destinations.size(), sorted ? 1 : 0, DG_MEM_HOST));
  }
  // sentinel_of(v).active_edge_count for every v (graph.hpp:108)
  std::vector<std::uint64_t> degrees() const {
    std::vector<std::uint64_t> out(logical_size());
    if (!out.empty()) check(dg_degrees(h_, out.data(), DG_MEM_HOST));
    return out;
  }

  // graph.hpp:287-317
  GraphStats stats() const {
    dg_stats s{};
    check(dg_stats_get(h_, &s));
    GraphStats o;
    o.logical_size = s.logical_size; o.capacity = s.capacity; o.alive_vertices = s.alive_vertices;
    o.active_edges = s.active_edges; o.adjacency_blocks = s.adjacency_blocks; o.occupied_slots = s.occupied_slots;
    o.hole_slots = s.hole_slots; o.pool_blocks_created = s.pool_blocks_created;
    o.pool_blocks_in_use = s.pool_blocks_in_use; o.pool_queue_size = s.pool_queue_size;
    o.max_degree = s.max_degree; o.block_size = s.block_size; o.pool_growths = s.growth_count;
    return o;
  }

  dg_graph* handle() const { return h_; }

 private:
  [[noreturn]] static void raise(int rc, const char* msg) {
    const std::string m = msg ? msg : "";
    if (rc == DG_ERR_DATA) throw DataError(m);
    throw EngineError(m);  // resource / contract / CUDA failures
  }
  void check(int rc) const {
    if (rc != DG_OK) raise(rc, dg_last_error(h_));
  }
  dg_graph* h_ = nullptr;
};

// The batch loop of run_workload (io/workload.hpp:141-155) with the host->device copy of the next
// batch overlapped with the running op (dg_ingest_*).  submit() applies batches in order exactly as
// insert_pairs / delete_pairs would; a failing batch throws from the call that executes it.  The
// host arrays must stay valid until their op ran.
class BatchIngest {
 public:
  // synchronous: one host wait per op (dg_ingest_insert / _delete); otherwise ops are SUBMITTED
  // (dg_ingest_submit_*): copies, ops and the host loop overlap, failures surface at a later submit() or flush()
  BatchIngest(DynamicGraph& g, std::uint64_t max_entries, std::uint32_t depth = 2, bool synchronous = false)
      : g_(g), depth_(depth), sync_(synchronous) {
    if (dg_ingest_create(g.handle(), max_entries, depth, &q_) != DG_OK) throw EngineError(dg_last_error(g.handle()));
  }
  ~BatchIngest() { dg_ingest_destroy(q_); }
  BatchIngest(const BatchIngest&) = delete;
  BatchIngest& operator=(const BatchIngest&) = delete;

  void submit(BatchKind kind, const VertexId* src, const VertexId* dst, std::uint64_t n) {
    if (sync_ && pending_.size() == depth_) run_oldest();
    std::uint32_t slot = 0;
    int rc = dg_ingest_stage_coo(q_, src, dst, n, &slot);
    if (rc != DG_OK) raise(rc);
    if (sync_) {
      pending_.emplace_back(kind, slot);
      if (pending_.size() == depth_) run_oldest();
      return;
    }
    rc = kind == BatchKind::Insert ? dg_ingest_submit_insert(q_, slot, nullptr) : dg_ingest_submit_delete(q_, slot, nullptr);
    if (rc != DG_OK) {
      const std::string msg = dg_last_error(g_.handle()) ? dg_last_error(g_.handle()) : "";
      dg_ingest_reset(q_);
      collect();
      if (rc == DG_ERR_DATA) throw DataError(msg);
      throw EngineError(msg);
    }
  }
  // waits for everything submitted; throws the first failure; applied() counts the batches that went in
  void flush() {
    while (!pending_.empty()) run_oldest();
    if (!sync_) {
      const int rc = collect();
      if (rc != DG_OK) raise(rc);
    }
  }
  std::uint64_t applied() const { return applied_; }

 private:
  int collect() {
    std::uint64_t n = 0;
    const int rc = dg_flush(g_.handle(), &n);
    applied_ += n;
    return rc;
  }
  void run_oldest() {
    const auto [kind, slot] = pending_.front();
    pending_.erase(pending_.begin());
    const int rc = kind == BatchKind::Insert ? dg_ingest_insert(q_, slot) : dg_ingest_delete(q_, slot);
    if (rc != DG_OK) {
      pending_.clear();   // later staged batches are dropped, as the reference loop would have stopped here
      const std::string msg = dg_last_error(g_.handle()) ? dg_last_error(g_.handle()) : "";
      dg_ingest_reset(q_);
      if (rc == DG_ERR_DATA) throw DataError(msg);
      throw EngineError(msg);
    }
    ++applied_;
  }
  [[noreturn]] void raise(int rc) const {
    const char* msg = dg_last_error(g_.handle());
    if (rc == DG_ERR_DATA) throw DataError(msg ? msg : "");
    throw EngineError(msg ? msg : "");
  }
  DynamicGraph& g_;
  dg_ingest* q_ = nullptr;
  std::uint32_t depth_;
  bool sync_;
  std::uint64_t applied_ = 0;
  std::vector<std::pair<BatchKind, std::uint32_t>> pending_;
};

}  // namespace dyngraph_b200
