/*
 * rmat.h — host twin of the counter-based R-MAT generator (TEST INFRASTRUCTURE).
 *
 * The reference ships no R-MAT generator; the
 * benchmark shapes in BASELINE.json need one, so edge i is defined as a pure
 * function of (seed, i): splitmix64 of (seed ^ i * K) seeds a splitmix64
 * stream, each 64-bit output decides two levels (low half, then high half)
 * by comparing against 32-bit fixed-point thresholds a, a+b, a+b+c.  The
 * device twin is rmat_edge() in paper_2306_08252_b200/csrc/dg_kernels.cuh and
 * the numpy twin is paper_2306_08252_b200/rmat.py; tests pin all three to the
 * same pairs.
 */
#ifndef ORACLE_RMAT_H
#define ORACLE_RMAT_H
#include <stdint.h>

static inline uint64_t orc_rmat_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline void orc_rmat_edge(uint32_t scale, uint64_t seed, uint64_t idx, uint32_t ta,
                                 uint32_t tab, uint32_t tabc, uint32_t* src, uint32_t* dst) {
  const uint64_t base = orc_rmat_mix64(seed ^ (idx * 0xD1342543DE82EF95ull));
  uint32_t s = 0, d = 0;
  for (uint32_t level = 0; level < scale; level += 2) {
    const uint64_t h = orc_rmat_mix64(base + (uint64_t)(level >> 1) * 0x9E3779B97F4A7C15ull);
    uint32_t r = (uint32_t)h;
    for (int half = 0; half < 2 && level + half < scale; ++half) {
      const uint32_t sb = r >= tab ? 1u : 0u;
      const uint32_t db = ((r >= ta && r < tab) || r >= tabc) ? 1u : 0u;
      s = (s << 1) | sb;
      d = (d << 1) | db;
      r = (uint32_t)(h >> 32);
    }
  }
  *src = s;
  *dst = d;
}
#endif
