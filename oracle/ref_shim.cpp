// ref_shim.cpp — C driver ABI around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle/dyngraph_oracle.c).  Compiled by
// oracle/Makefile with -I/root/reference/proj/include into
// oracle/_ref/libdyngraph_ref.so; no reference source is copied into this
// repository — this file only calls the reference's public API
// (dyngraph::DynamicGraph, graph.hpp:80-317; csr_from_pairs, csr.hpp:29-45).
// The exported functions mirror oracle/dyngraph_oracle.c's orc_* one for one
// so the same Python driver runs either.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "dyngraph/dyngraph.hpp"

namespace {

struct Ref {
  std::unique_ptr<dyngraph::DynamicGraph> g;
  std::string err;
};

thread_local std::string g_create_err;

template <class Fn>
int guarded(Ref* r, Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const dyngraph::DataError& e) {
    r->err = e.what();
    return 2;
  } catch (const dyngraph::EngineError& e) {
    r->err = e.what();
    return 3;
  } catch (const std::exception& e) {
    r->err = e.what();
    return 3;
  }
}

dyngraph::CsrBatch make_csr(dyngraph::BatchKind kind, const std::uint64_t* off, std::uint64_t n_off,
                            const std::uint32_t* dsts, std::uint64_t n) {
  dyngraph::CsrBatch b;
  b.kind = kind;
  b.offsets.assign(off, off + n_off);
  b.destinations.assign(dsts, dsts + n);
  return b;
}

dyngraph::CsrBatch from_pairs(dyngraph::BatchKind kind, std::uint64_t v, const std::uint32_t* src,
                              const std::uint32_t* dst, std::uint64_t n) {
  for (std::uint64_t i = 0; i < n; ++i)
    if (src[i] >= v) throw dyngraph::DataError("csr batch: source out of range");
  std::vector<std::pair<dyngraph::VertexId, dyngraph::VertexId>> pairs;
  pairs.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i) pairs.emplace_back(src[i], dst[i]);
  return dyngraph::csr_from_pairs(kind, v, pairs);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

void* ref_create(std::uint64_t arena_bytes, double initial_fraction, int reclaim,
                 std::uint32_t workers, std::uint64_t v0, std::uint32_t block_size, int* err) {
  auto* r = new Ref();
  *err = 0;
  try {
    dyngraph::GraphConfig cfg;
    cfg.arena_bytes = arena_bytes;
    cfg.pool.initial_fraction = initial_fraction;
    cfg.reclaim_on_delete = reclaim != 0;
    cfg.workers = workers;
    r->g = std::make_unique<dyngraph::DynamicGraph>(cfg, v0, block_size);
  } catch (const dyngraph::DataError& e) {
    g_create_err = e.what();
    *err = 2;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    *err = 3;
  }
  if (*err) {
    delete r;
    return nullptr;
  }
  return r;
}

void ref_destroy(void* p) { delete static_cast<Ref*>(p); }
const char* ref_last_error(void* p) { return p ? static_cast<Ref*>(p)->err.c_str() : g_create_err.c_str(); }

int ref_insert_csr(void* p, const std::uint64_t* off, std::uint64_t n_off, const std::uint32_t* dsts,
                   std::uint64_t n) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] { r->g->insert_batch(make_csr(dyngraph::BatchKind::Insert, off, n_off, dsts, n)); });
}
int ref_delete_csr(void* p, const std::uint64_t* off, std::uint64_t n_off, const std::uint32_t* dsts,
                   std::uint64_t n) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] { r->g->delete_batch(make_csr(dyngraph::BatchKind::Delete, off, n_off, dsts, n)); });
}
// DynamicGraph::plan_batch (graph.hpp:135-160), copied out of the BatchPlan vectors
int ref_plan_batch(void* p, const std::uint64_t* off, std::uint64_t n_off, const std::uint32_t* dsts, std::uint64_t n,
                   std::uint64_t* blocks_required, std::uint64_t* prefix_sum, std::uint32_t* space_remaining) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] {
    const auto plan = r->g->plan_batch(make_csr(dyngraph::BatchKind::Insert, off, n_off, dsts, n));
    std::copy(plan.blocks_required.begin(), plan.blocks_required.end(), blocks_required);
    std::copy(plan.prefix_sum.begin(), plan.prefix_sum.end(), prefix_sum);
    std::copy(plan.space_remaining.begin(), plan.space_remaining.end(), space_remaining);
  });
}
int ref_insert_coo(void* p, const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t n,
                   double* seconds) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] {
    const auto batch = from_pairs(dyngraph::BatchKind::Insert, r->g->logical_size(), src, dst, n);
    const double t0 = now_s();  // batch construction is outside the timed region
    r->g->insert_batch(batch);
    if (seconds) *seconds = now_s() - t0;
  });
}
int ref_delete_coo(void* p, const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t n,
                   double* seconds) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] {
    const auto batch = from_pairs(dyngraph::BatchKind::Delete, r->g->logical_size(), src, dst, n);
    const double t0 = now_s();
    r->g->delete_batch(batch);
    if (seconds) *seconds = now_s() - t0;
  });
}
int ref_query(void* p, const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t n,
              std::uint8_t* out) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] {
    for (std::uint64_t i = 0; i < n; ++i) out[i] = r->g->query_edge(src[i], dst[i]) ? 1 : 0;
  });
}
int ref_insert_vertices(void* p, std::uint64_t count) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] { r->g->insert_vertices(count); });
}
int ref_delete_vertices(void* p, const std::uint32_t* ids, std::uint64_t n, std::uint32_t* skipped,
                        std::uint64_t* n_skipped) {
  auto* r = static_cast<Ref*>(p);
  return guarded(r, [&] {
    const auto sk = r->g->delete_vertices(std::span<const dyngraph::VertexId>(ids, n));
    if (skipped) std::memcpy(skipped, sk.data(), sk.size() * sizeof(std::uint32_t));
    if (n_skipped) *n_skipped = sk.size();
  });
}

std::uint32_t ref_block_size(void* p) { return static_cast<Ref*>(p)->g->block_size(); }
std::uint64_t ref_logical_size(void* p) { return static_cast<Ref*>(p)->g->logical_size(); }
std::uint64_t ref_vertex_capacity(void* p) { return static_cast<Ref*>(p)->g->vertex_capacity(); }
std::uint64_t ref_alive_vertices(void* p) { return static_cast<Ref*>(p)->g->alive_vertices(); }
std::uint64_t ref_active_edges(void* p) { return static_cast<Ref*>(p)->g->active_edges(); }
int ref_vertex_alive(void* p, std::uint32_t v) { return static_cast<Ref*>(p)->g->vertex_alive(v) ? 1 : 0; }
std::uint64_t ref_queue_size(void* p) { return static_cast<Ref*>(p)->g->pool().queue_size(); }
std::uint64_t ref_blocks_in_use(void* p) { return static_cast<Ref*>(p)->g->pool().blocks_in_use(); }

int ref_degrees(void* p, std::uint64_t* out) {
  auto* r = static_cast<Ref*>(p);
  for (std::uint64_t v = 0; v < r->g->logical_size(); ++v)
    out[v] = r->g->sentinel_of(static_cast<dyngraph::VertexId>(v)).active_edge_count;
  return 0;
}

// Order-independent digest of the stored multiset (sum over live entries of mix64(v << 32 | dst)): the
// device twin is digest_kernel.  Walks active_destinations (graph.hpp:116-129) of every v < logical_size.
static std::uint64_t shim_mix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
int ref_digest(void* p, std::uint64_t* digest, std::uint64_t* entries) {
  auto* r = static_cast<Ref*>(p);
  std::uint64_t acc = 0, cnt = 0;
  const std::uint64_t n = r->g->logical_size();
  for (std::uint64_t v = 0; v < n; ++v) {
    for (std::uint32_t d : r->g->active_destinations(static_cast<dyngraph::VertexId>(v))) {
      acc += shim_mix64((v << 32) | d);
      ++cnt;
    }
  }
  if (digest) *digest = acc;
  if (entries) *entries = cnt;
  return 0;
}

int ref_export_csr(void* p, std::uint64_t* offsets, std::uint32_t* dsts, std::uint64_t cap, int sorted) {
  auto* r = static_cast<Ref*>(p);
  std::uint64_t w = 0;
  const std::uint64_t n = r->g->logical_size();
  for (std::uint64_t v = 0; v < n; ++v) {
    offsets[v] = w;
    auto d = r->g->active_destinations(static_cast<dyngraph::VertexId>(v));
    if (sorted) std::sort(d.begin(), d.end());
    if (dsts) {
      if (w + d.size() > cap) return 2;
      std::memcpy(dsts + w, d.data(), d.size() * sizeof(std::uint32_t));
    }
    w += d.size();
  }
  offsets[n] = w;
  return 0;
}

// compute_block_size (csr.hpp:77-88) over a COO batch, for the bench
int ref_compute_block_size_coo(std::uint64_t v, const std::uint32_t* src, const std::uint32_t* dst,
                               std::uint64_t n, std::uint32_t* out) {
  try {
    std::vector<std::pair<dyngraph::VertexId, dyngraph::VertexId>> pairs;
    pairs.reserve(n);
    for (std::uint64_t i = 0; i < n; ++i) pairs.emplace_back(src[i], dst[i]);
    *out = dyngraph::compute_block_size(dyngraph::csr_from_pairs(dyngraph::BatchKind::Insert, v, pairs));
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

// synth_uniform (io/synthetic.hpp:19-25) as COO in generation order, for golden inputs.  The
// reference's `emplace_back(rng() % V, rng() % V)` leaves the order of the two draws unspecified;
// g++ evaluates right to left, so the first draw is the destination (make_golden.py checks this
// against dyngraph::io::synth_uniform itself).
int ref_synth_uniform_pairs(std::uint64_t v, std::uint64_t e, std::uint64_t seed, std::uint32_t* src,
                            std::uint32_t* dst) {
  std::mt19937_64 rng(seed);
  for (std::uint64_t i = 0; i < e; ++i) {
    dst[i] = static_cast<std::uint32_t>(rng() % v);
    src[i] = static_cast<std::uint32_t>(rng() % v);
  }
  return 0;
}

// ---- io side (io/synthetic.hpp, io/batching.hpp, io/workload.hpp): golden generators for the
// host-side mirror in paper_2306_08252_b200/io.py -------------------------------------------------

// kind 0: synth_uniform (io/synthetic.hpp:16-27), 1: synth_power_law (:32-66); CSR out
int ref_synth_csr(int kind, std::uint64_t v, std::uint64_t e, std::uint64_t seed, std::uint64_t* offsets,
                  std::uint32_t* dsts) {
  try {
    const dyngraph::io::Csr csr = kind == 0 ? dyngraph::io::synth_uniform(v, e, seed) : dyngraph::io::synth_power_law(v, e, seed);
    std::copy(csr.offsets.begin(), csr.offsets.end(), offsets);
    std::copy(csr.destinations.begin(), csr.destinations.end(), dsts);
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

// make_batches (io/batching.hpp:46-66) flattened: every batch's (src, dst) in CSR order, one after
// the other; batch_sizes[i] = edges of batch i; returns the batch count (or -1)
long long ref_make_batches_flat(std::uint64_t v, const std::uint64_t* offsets, const std::uint32_t* dsts, std::uint64_t e,
                                std::uint64_t batch_size, int shuffled, std::uint64_t seed, std::uint32_t* src_out,
                                std::uint32_t* dst_out, std::uint64_t* batch_sizes) {
  try {
    dyngraph::io::Csr csr;
    csr.vertex_count = v;
    csr.offsets.assign(offsets, offsets + v + 1);
    csr.destinations.assign(dsts, dsts + e);
    const auto batches = dyngraph::io::make_batches(csr, batch_size, dyngraph::BatchKind::Insert,
                                                    shuffled ? dyngraph::io::EdgeOrder::Shuffled : dyngraph::io::EdgeOrder::Prefix, seed);
    std::uint64_t k = 0;
    for (std::size_t b = 0; b < batches.size(); ++b) {
      batch_sizes[b] = batches[b].edge_count();
      for (std::uint64_t u = 0; u < v; ++u)
        for (std::uint64_t i = batches[b].offsets[u]; i < batches[b].offsets[u + 1]; ++i) {
          src_out[k] = static_cast<std::uint32_t>(u);
          dst_out[k] = batches[b].destinations[i];
          ++k;
        }
    }
    return static_cast<long long>(batches.size());
  } catch (const std::exception&) {
    return -1;
  }
}

// run_workload (io/workload.hpp:104-190) on a synthetic source with a fake clock (250 us per tick,
// as the reference's io_test.cpp:51-57).  ops: 0 Insert, 1 Delete, 2 InsertThenDelete.
// out[0..7] = edges_inserted, edges_deleted, queries_run, queries_hit, effective_block_size,
//             rows, final active_edges, vertex_count; phases: comma-separated phase names
int ref_run_workload_synth(int kind, std::uint64_t v, std::uint64_t e, std::uint64_t seed, std::uint64_t batch_size, int ops,
                           int shuffled, std::uint32_t block_size, std::uint64_t query_sample, std::uint64_t arena_bytes,
                           std::uint64_t* out, char* phases, std::uint64_t phases_cap) {
  try {
    dyngraph::io::WorkloadSpec spec;
    spec.graph_name = "synth";
    spec.source = kind == 0 ? dyngraph::io::WorkloadSpec::Source::SynthUniform : dyngraph::io::WorkloadSpec::Source::SynthPowerLaw;
    spec.synth_vertices = v;
    spec.synth_edges = e;
    spec.seed = seed;
    spec.batch_size = batch_size;
    spec.ops = ops == 0 ? dyngraph::io::OpsMode::Insert : ops == 1 ? dyngraph::io::OpsMode::Delete : dyngraph::io::OpsMode::InsertThenDelete;
    spec.order = shuffled ? dyngraph::io::EdgeOrder::Shuffled : dyngraph::io::EdgeOrder::Prefix;
    spec.block_size = block_size;
    spec.query_sample = query_sample;
    spec.config.arena_bytes = arena_bytes;
    std::uint64_t t = 0;
    const dyngraph::io::RunReport r = dyngraph::io::run_workload(spec, [&t] { t += 250000; return t; });
    out[0] = r.edges_inserted; out[1] = r.edges_deleted; out[2] = r.queries_run; out[3] = r.queries_hit;
    out[4] = r.effective_block_size; out[5] = r.rows.size(); out[6] = r.final_stats.active_edges; out[7] = r.vertex_count;
    std::string ph;
    for (const auto& row : r.rows) { if (!ph.empty()) ph += ','; ph += row.phase; }
    if (ph.size() + 1 > phases_cap) return 3;
    std::memcpy(phases, ph.c_str(), ph.size() + 1);
    return 0;
  } catch (const dyngraph::DataError&) {
    return 2;
  } catch (const std::exception&) {
    return 3;
  }
}

}  // extern "C"
