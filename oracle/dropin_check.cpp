// dropin_check.cpp — the SAME templated workload driven through the unmodified
// reference class (dyngraph::DynamicGraph, /root/reference/proj/include) and
// through the drop-in mirror (dyngraph_b200::DynamicGraph, include/dyngraph_b200.hpp
// -> C ABI -> CUDA), comparing what oracle_compare compares (oracle.hpp:98-163).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into
// oracle/_ref/dropin_check where the reference headers exist; the binary (not
// the reference source) travels to the GPU box and is run by
// tests/test_gpu_parity.py::test_cpp_dropin_against_reference_class.
// The op mix follows the reference's verify workload (verify.hpp:135-265).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "dyngraph/dyngraph.hpp"
#include "dyngraph_b200.hpp"

namespace {

using Pairs = std::vector<std::pair<std::uint32_t, std::uint32_t>>;

struct Canon {
  std::uint64_t logical_size = 0, capacity = 0, alive = 0, active_edges = 0;
  std::vector<std::uint8_t> alive_flags;
  std::vector<std::vector<std::uint32_t>> adj;  // sorted multiset per vertex
  std::vector<std::string> events;              // status / skipped / answers per op
  bool operator==(const Canon& o) const {
    return logical_size == o.logical_size && capacity == o.capacity && alive == o.alive &&
           active_edges == o.active_edges && alive_flags == o.alive_flags && adj == o.adj && events == o.events;
  }
};

template <class G, class Batch, class Kind, class DataErr, class EngineErr>
struct Driver {
  G& g;
  Canon c;
  Kind ins, del;
  Batch (*from_pairs)(Kind, std::uint64_t, const Pairs&);

  template <class Fn>
  void guarded(const char* what, Fn&& fn) {
    try {
      fn();
      c.events.push_back(std::string(what) + ":ok");
    } catch (const DataErr&) {
      c.events.push_back(std::string(what) + ":data");
    } catch (const EngineErr&) {
      c.events.push_back(std::string(what) + ":engine");
    }
  }
  void insert(const Pairs& p) { guarded("insert", [&] { g.insert_batch(from_pairs(ins, g.logical_size(), p)); }); }
  void erase(const Pairs& p) { guarded("delete", [&] { g.delete_batch(from_pairs(del, g.logical_size(), p)); }); }
  void add_vertices(std::uint64_t n) { guarded("addv", [&] { g.insert_vertices(n); }); }
  void del_vertices(const std::vector<std::uint32_t>& ids) {
    const auto sk = g.delete_vertices(ids);
    std::string s = "delv:";
    for (auto v : sk) s += std::to_string(v) + ",";
    c.events.push_back(s);
  }
  void query(const Pairs& q) {
    std::string s = "q:";
    for (const auto& e : q) s += g.query_edge(e.first, e.second) ? '1' : '0';
    c.events.push_back(s);
  }
  void finish() {
    c.logical_size = g.logical_size();
    c.capacity = g.vertex_capacity();
    c.alive = g.alive_vertices();
    c.active_edges = g.active_edges();
    for (std::uint64_t v = 0; v < c.logical_size; ++v) {
      c.alive_flags.push_back(g.vertex_alive(static_cast<std::uint32_t>(v)) ? 1 : 0);
      auto d = g.active_destinations(static_cast<std::uint32_t>(v));
      std::sort(d.begin(), d.end());
      c.adj.emplace_back(d.begin(), d.end());
    }
  }
};

// one random workload, verify.hpp:135-265 op mix; the script depends only on the seed
template <class D>
void run_script(D& d, std::uint64_t seed, std::uint64_t v0) {
  std::mt19937_64 rng(seed);
  std::uint64_t size = v0;
  std::vector<std::uint32_t> alive;
  for (std::uint64_t v = 0; v < v0; ++v) alive.push_back(static_cast<std::uint32_t>(v));
  std::vector<std::uint32_t> dead;
  Pairs log;
  const int steps = 6 + static_cast<int>(rng() % 18);
  for (int s = 0; s < steps; ++s) {
    const int roll = static_cast<int>(rng() % 100);
    if (roll < 55 && !alive.empty()) {
      Pairs p(1 + rng() % 3000);
      for (auto& e : p) e = {alive[rng() % alive.size()], static_cast<std::uint32_t>(rng() % size)};
      d.insert(p);
      log.insert(log.end(), p.begin(), p.end());
    } else if (roll < 80 && !log.empty()) {
      Pairs p(1 + rng() % 1500);
      for (auto& e : p) {
        if (rng() % 10 < 7) e = log[rng() % log.size()];
        else e = {static_cast<std::uint32_t>(rng() % size), static_cast<std::uint32_t>(rng() % size)};
      }
      d.erase(p);
    } else if (roll < 90) {
      const std::uint64_t n = 1 + rng() % 64;
      d.add_vertices(n);
      for (std::uint64_t i = 0; i < n; ++i) alive.push_back(static_cast<std::uint32_t>(size + i));
      size += n;
    } else if (!alive.empty()) {
      std::vector<std::uint32_t> ids;
      const int n = 1 + static_cast<int>(rng() % 4);
      for (int i = 0; i < n; ++i) ids.push_back(alive[rng() % alive.size()]);
      if (!dead.empty() && rng() % 4 == 0) ids.push_back(dead[0]);
      d.del_vertices(ids);
      for (auto v : ids) {
        auto it = std::find(alive.begin(), alive.end(), v);
        if (it != alive.end()) {
          alive.erase(it);
          dead.push_back(v);
        }
      }
    }
  }
  Pairs q(200);
  for (auto& e : q) {
    if (!log.empty() && rng() % 2) e = log[rng() % log.size()];
    else e = {static_cast<std::uint32_t>(rng() % (size + 3)), static_cast<std::uint32_t>(rng() % (size + 3))};
  }
  d.query(q);
  d.finish();
}

}  // namespace

int main(int argc, char** argv) {
  const int n_workloads = argc > 1 ? std::atoi(argv[1]) : 40;
  int bad = 0;
  for (int w = 0; w < n_workloads; ++w) {
    const std::uint64_t seed = 0x5eed + w;  // acceptance_test.cpp:53-59 base seed
    std::mt19937_64 cfg_rng(seed ^ 0x9e3779b97f4a7c15ull);
    const std::uint64_t v0 = 1 + cfg_rng() % 256;
    const std::uint32_t B = 1 + static_cast<std::uint32_t>(cfg_rng() % 8);
    const bool reclaim = cfg_rng() % 2 == 0;

    dyngraph::GraphConfig rc;
    rc.arena_bytes = 64ull << 20;
    rc.reclaim_on_delete = reclaim;
    rc.workers = 1 + static_cast<std::uint32_t>(cfg_rng() % 3);
    dyngraph::DynamicGraph ref(rc, v0, B);
    Driver<dyngraph::DynamicGraph, dyngraph::CsrBatch, dyngraph::BatchKind, dyngraph::DataError, dyngraph::EngineError>
        dr{ref, {}, dyngraph::BatchKind::Insert, dyngraph::BatchKind::Delete, &dyngraph::csr_from_pairs};
    run_script(dr, seed, v0);

    dyngraph_b200::GraphConfig gc;
    gc.pool_blocks = 1u << 17;
    gc.reclaim_on_delete = reclaim;
    dyngraph_b200::DynamicGraph gpu(gc, v0, B);
    Driver<dyngraph_b200::DynamicGraph, dyngraph_b200::CsrBatch, dyngraph_b200::BatchKind, dyngraph_b200::DataError,
           dyngraph_b200::EngineError>
        dg{gpu, {}, dyngraph_b200::BatchKind::Insert, dyngraph_b200::BatchKind::Delete, &dyngraph_b200::csr_from_pairs};
    run_script(dg, seed, v0);

    if (!(dr.c == dg.c)) {
      ++bad;
      std::printf("workload %d (seed %llu, V0=%llu, B=%u, reclaim=%d): MISMATCH\n", w, (unsigned long long)seed,
                  (unsigned long long)v0, B, (int)reclaim);
    }
  }
  std::printf("dropin_check: %d workloads, %d mismatches\n", n_workloads, bad);
  return bad == 0 ? 0 : 1;
}
