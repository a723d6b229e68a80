/*
 * dyngraph_oracle.c — CPU restatement of the reference's dynamic-graph path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_2306_08252_b200/ may link,
 * import or execute this file; it exists so tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg can check the CUDA path.  Parity status:
 * PINNED — tests/test_oracle_cpu.py checks this restatement against (a) the
 * known-answer cases of the reference's own tests
 * (proj/tests/batch_engine_test.cpp, oracle_test.cpp, block_pool_test.cpp),
 * (b) golden vectors in tests/golden/ generated from the reference itself
 * (oracle/_ref, built from /root/reference/proj/include by oracle/Makefile),
 * and (c) oracle/_ref live when it is present.
 *
 * Plain C11, no dependencies.  Each function cites the reference file:line
 * whose behaviour it restates.  The complete-binary-tree adjacency of the
 * reference (cbt.hpp) is held as an implicit heap: a vertex's block at
 * level-order position k is blocks[k-1], children 2k / 2k+1 — the bijection
 * the reference pins in proj/tests/core_test.cpp:151-166.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <time.h>

#define ORC_OK 0
#define ORC_ERR_DATA 2   /* DataError, types.hpp:25-27 */
#define ORC_ERR_ENGINE 3 /* EngineError, types.hpp:30-32 */
#define ORC_NULL 0xFFFFFFFFu

/* ---- arena (arena.hpp:13-49): pure byte accounting ------------------------ */
typedef struct {
  uint64_t capacity, reserved;
  uint32_t reservations;
} Arena;

static uint64_t arena_available(const Arena* a) { return a->capacity - a->reserved; }
static int arena_reserve(Arena* a, uint64_t bytes) { /* arena.hpp:26-34 */
  if (bytes > arena_available(a)) return 0;
  a->reserved += bytes;
  a->reservations++;
  return 1;
}

/* ---- sentinel (edge_block.hpp:34-42) with the implicit-heap block list ----- */
typedef struct {
  uint64_t active_edge_count;
  uint32_t block_count;
  uint32_t* blocks; /* position k -> blocks[k-1] */
  uint32_t blocks_cap;
  uint32_t last_insert_block;
  uint32_t last_insert_offset;
} Sentinel;

typedef struct {
  /* config (graph.hpp:23-28, block_pool.hpp:18-29) */
  double initial_fraction, trigger_fraction, growth_fraction;
  int reclaim_on_delete;
  Arena arena;
  /* vertex dictionary (vertex_dictionary.hpp:26-97) */
  uint64_t size, capacity, alive_count;
  uint8_t* alive;
  Sentinel* sent;
  uint64_t vcap_alloc;
  /* block pool (block_pool.hpp:97-276) */
  uint32_t B;
  uint64_t created, consumed, reserved_bytes;
  uint32_t growths;
  /* lazily materialised storage (block_pool.hpp:214-219) */
  uint64_t materialized;
  uint32_t* dst;
  uint8_t* tomb;
  uint32_t* active;
  uint32_t* occupied;
  /* edge queue (block_pool.hpp:35-84): unwrapped coordinates */
  uint32_t* ring;
  uint64_t ring_cap, front, rear, total_capacity;
  uint64_t active_edges;
  char err[256];
} Oracle;

static uint64_t pow2_ceil(uint64_t n) { /* bits.hpp:11-16 */
  uint64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

static uint64_t bytes_per_block(const Oracle* g) { return (uint64_t)g->B * 8 + 16; } /* block_pool.hpp:124-126 */

static void queue_push(Oracle* g, uint32_t h) { /* block_pool.hpp:54-59 */
  if (g->rear - g->front == g->ring_cap) {
    uint64_t ncap = g->ring_cap ? g->ring_cap * 2 : 16;
    uint32_t* nr = (uint32_t*)malloc(ncap * sizeof(uint32_t));
    for (uint64_t p = g->front; p < g->rear; ++p) nr[p % ncap] = g->ring[p % g->ring_cap];
    free(g->ring);
    g->ring = nr;
    g->ring_cap = ncap;
  }
  g->ring[g->rear % g->ring_cap] = h;
  g->rear++;
  g->total_capacity++;
}

static void push_new_blocks(Oracle* g, uint64_t count) { /* block_pool.hpp:242-247 */
  for (uint64_t i = 0; i < count; ++i) queue_push(g, (uint32_t)(g->created + i));
  g->created += count;
}

static int try_grow(Oracle* g) { /* block_pool.hpp:252-264 */
  uint64_t want = (uint64_t)((double)g->total_capacity * g->growth_fraction);
  if (want == 0) want = 1;
  const uint64_t affordable = arena_available(&g->arena) / bytes_per_block(g);
  const uint64_t grant = want < affordable ? want : affordable;
  if (grant == 0) return 0;
  arena_reserve(&g->arena, grant * bytes_per_block(g));
  g->reserved_bytes += grant * bytes_per_block(g);
  push_new_blocks(g, grant);
  g->growths++;
  return 1;
}

static int ensure_available(Oracle* g, uint64_t blocks) { /* block_pool.hpp:177-189 */
  const uint64_t qsize = g->rear - g->front;
  if (qsize >= blocks) return ORC_OK;
  const uint64_t shortfall = blocks - qsize;
  if (arena_available(&g->arena) / bytes_per_block(g) < shortfall) {
    snprintf(g->err, sizeof g->err, "block pool: batch needs %llu more blocks than the arena can still provide",
             (unsigned long long)shortfall);
    return ORC_ERR_ENGINE;
  }
  while (g->rear - g->front < blocks) {
    if (!try_grow(g)) {
      snprintf(g->err, sizeof g->err, "block pool: growth stalled before satisfying demand");
      return ORC_ERR_ENGINE;
    }
  }
  return ORC_OK;
}

static void materialize(Oracle* g, uint64_t handle_end) { /* block_pool.hpp:214-219 */
  if (handle_end > g->created) handle_end = g->created;
  if (handle_end <= g->materialized) return;
  uint64_t n = g->materialized ? g->materialized : 64;
  while (n < handle_end) n *= 2;
  if (n > g->created) n = g->created;
  g->dst = (uint32_t*)realloc(g->dst, n * g->B * sizeof(uint32_t));
  g->tomb = (uint8_t*)realloc(g->tomb, n * g->B);
  g->active = (uint32_t*)realloc(g->active, n * sizeof(uint32_t));
  g->occupied = (uint32_t*)realloc(g->occupied, n * sizeof(uint32_t));
  memset(g->tomb + g->materialized * g->B, 0, (n - g->materialized) * g->B);
  memset(g->active + g->materialized, 0, (n - g->materialized) * sizeof(uint32_t));
  memset(g->occupied + g->materialized, 0, (n - g->materialized) * sizeof(uint32_t));
  g->materialized = n;
}

static void commit_front(Oracle* g, uint64_t popped) { /* block_pool.hpp:162-166 */
  g->front += popped;
  g->consumed += popped;
  const double occ = g->total_capacity == 0 ? 0.0 : (double)g->consumed / (double)g->total_capacity;
  if (occ >= g->trigger_fraction) try_grow(g);
}

static void reclaim(Oracle* g, const uint32_t* handles, uint64_t n) { /* block_pool.hpp:192-209 */
  for (uint64_t i = 0; i < n; ++i) {
    g->occupied[handles[i]] = 0;
    queue_push(g, handles[i]);
  }
}

static void sentinel_reset(Sentinel* s) {
  s->active_edge_count = 0;
  s->block_count = 0;
  s->last_insert_block = ORC_NULL;
  s->last_insert_offset = 0;
}

static void append_slots(Oracle* g, uint64_t count) { /* vertex_dictionary.hpp:84-91 */
  if (g->size + count > g->vcap_alloc) {
    uint64_t n = g->vcap_alloc ? g->vcap_alloc : 16;
    while (n < g->size + count) n *= 2;
    g->alive = (uint8_t*)realloc(g->alive, n);
    g->sent = (Sentinel*)realloc(g->sent, n * sizeof(Sentinel));
    g->vcap_alloc = n;
  }
  for (uint64_t i = 0; i < count; ++i) {
    g->alive[g->size] = 1;
    memset(&g->sent[g->size], 0, sizeof(Sentinel));
    sentinel_reset(&g->sent[g->size]);
    g->size++;
  }
  g->alive_count += count;
}

/* in-order sequence of level-order positions 1..n (cbt.hpp:58-75) */
static void in_order_positions(uint32_t n, uint32_t* out) {
  uint32_t stack[40];
  int sp = 0;
  uint32_t cur = n >= 1 ? 1 : 0, w = 0;
  while (cur != 0 || sp > 0) {
    while (cur != 0) {
      stack[sp++] = cur;
      cur = (2 * (uint64_t)cur <= n) ? 2 * cur : 0;
    }
    cur = stack[--sp];
    out[w++] = cur;
    cur = (2 * (uint64_t)cur + 1 <= n) ? 2 * cur + 1 : 0;
  }
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y);
}

/* ---- public driver ABI ------------------------------------------------------ */

void orc_destroy(void* p) {
  Oracle* g = (Oracle*)p;
  if (!g) return;
  for (uint64_t v = 0; v < g->size; ++v) free(g->sent[v].blocks);
  free(g->alive); free(g->sent); free(g->dst); free(g->tomb); free(g->active);
  free(g->occupied); free(g->ring); free(g);
}

static char g_create_err[256];
const char* orc_last_error(void* p) { return p ? ((Oracle*)p)->err : g_create_err; }

/* DynamicGraph ctor (graph.hpp:84-91): dictionary (vertex_dictionary.hpp:30-37)
 * then pool (block_pool.hpp:99-116); exactly three reservations. */
void* orc_create(uint64_t arena_bytes, double initial_fraction, int reclaim, uint32_t workers,
                 uint64_t v0, uint32_t block_size, int* err) {
  (void)workers; /* determinism across worker counts: batch_engine_test.cpp:517-540 */
  Oracle* g = (Oracle*)calloc(1, sizeof(Oracle));
  *err = ORC_OK;
  g->initial_fraction = initial_fraction;
  g->trigger_fraction = 0.8;
  g->growth_fraction = 0.25;
  g->reclaim_on_delete = reclaim;
  g->arena.capacity = arena_bytes;
  g->capacity = pow2_ceil(v0 == 0 ? 1 : v0);
  if (!arena_reserve(&g->arena, g->capacity * 12) || !arena_reserve(&g->arena, g->capacity * 24)) {
    snprintf(g_create_err, sizeof g_create_err, "arena: reservation exceeds remaining budget");
    *err = ORC_ERR_ENGINE; orc_destroy(g); return NULL;
  }
  append_slots(g, v0);
  if (!(initial_fraction > 0.0 && initial_fraction <= 1.0)) { /* block_pool.hpp:23-28 */
    snprintf(g_create_err, sizeof g_create_err, "growth policy: all fractions must be in (0, 1]");
    *err = ORC_ERR_DATA; orc_destroy(g); return NULL;
  }
  if (block_size == 0) {
    snprintf(g_create_err, sizeof g_create_err, "block pool: block size must be >= 1");
    *err = ORC_ERR_DATA; orc_destroy(g); return NULL;
  }
  g->B = block_size;
  uint64_t request = (uint64_t)((double)arena_bytes * initial_fraction);
  if (request > arena_available(&g->arena)) request = arena_available(&g->arena);
  if (request / bytes_per_block(g) == 0) {
    snprintf(g_create_err, sizeof g_create_err, "block pool: arena cannot host a single edge block");
    *err = ORC_ERR_ENGINE; orc_destroy(g); return NULL;
  }
  arena_reserve(&g->arena, request);
  g->reserved_bytes = request;
  const uint64_t count = request / bytes_per_block(g);
  g->ring = (uint32_t*)malloc(count * sizeof(uint32_t));
  g->ring_cap = count;
  push_new_blocks(g, count);
  return g;
}

/* validate_batch (csr.hpp:49-73) */
static int validate_batch(Oracle* g, const uint64_t* off, uint64_t n_off, const uint32_t* dsts, uint64_t n) {
  if (n_off != g->size + 1) { snprintf(g->err, sizeof g->err, "csr batch: offsets length mismatch"); return ORC_ERR_DATA; }
  if (off[0] != 0) { snprintf(g->err, sizeof g->err, "csr batch: offsets[0] must be 0"); return ORC_ERR_DATA; }
  for (uint64_t i = 1; i < n_off; ++i)
    if (off[i] < off[i - 1]) { snprintf(g->err, sizeof g->err, "csr batch: offsets are not monotone"); return ORC_ERR_DATA; }
  if (off[n_off - 1] != n) { snprintf(g->err, sizeof g->err, "csr batch: destinations length mismatch"); return ORC_ERR_DATA; }
  for (uint64_t i = 0; i < n; ++i)
    if (dsts[i] >= g->size) { snprintf(g->err, sizeof g->err, "csr batch: destination out of range"); return ORC_ERR_DATA; }
  return ORC_OK;
}

/* plan_batch (graph.hpp:135-160): validate_insert, then per vertex space_remaining (:149-150), blocks_required
 * (:152-153) and their inclusive prefix sum (:154-156).  Nothing is mutated. */
int orc_plan_batch(void* p, const uint64_t* off, uint64_t n_off, const uint32_t* dsts, uint64_t n,
                   uint64_t* blocks_required, uint64_t* prefix_sum, uint32_t* space_remaining) {
  Oracle* g = (Oracle*)p;
  int rc = validate_batch(g, off, n_off, dsts, n);
  if (rc) return rc;
  const uint64_t V = g->size;
  for (uint64_t v = 0; v < V; ++v) /* validate_insert, graph.hpp:320-328 */
    if (off[v + 1] > off[v] && !g->alive[v]) {
      snprintf(g->err, sizeof g->err, "csr batch: insert lists edges for retired vertex %llu", (unsigned long long)v);
      return ORC_ERR_DATA;
    }
  uint64_t running = 0;
  for (uint64_t v = 0; v < V; ++v) {
    const Sentinel* s = &g->sent[v];
    const uint64_t space = s->block_count == 0 ? 0 : g->B - s->last_insert_offset;
    const uint64_t deg = off[v + 1] - off[v];
    const uint64_t overflow = deg > space ? deg - space : 0;
    const uint64_t required = (overflow + g->B - 1) / g->B;
    space_remaining[v] = (uint32_t)space;
    blocks_required[v] = required;
    running += required;
    prefix_sum[v] = running;
  }
  return ORC_OK;
}

/* insert_batch (graph.hpp:167-188) = plan_batch (:135-160) + ensure_available
 * + per-vertex insert_adjacency (:333-372) + commit_front. */
int orc_insert_csr(void* p, const uint64_t* off, uint64_t n_off, const uint32_t* dsts, uint64_t n) {
  Oracle* g = (Oracle*)p;
  int rc = validate_batch(g, off, n_off, dsts, n);
  if (rc) return rc;
  const uint64_t V = g->size;
  for (uint64_t v = 0; v < V; ++v) /* validate_insert, graph.hpp:320-328 */
    if (off[v + 1] > off[v] && !g->alive[v]) {
      snprintf(g->err, sizeof g->err, "csr batch: insert lists edges for retired vertex %llu", (unsigned long long)v);
      return ORC_ERR_DATA;
    }
  /* plan: space_remaining, blocks_required, total */
  uint64_t total = 0;
  for (uint64_t v = 0; v < V; ++v) {
    const Sentinel* s = &g->sent[v];
    const uint64_t space = s->block_count == 0 ? 0 : g->B - s->last_insert_offset;
    const uint64_t deg = off[v + 1] - off[v];
    const uint64_t overflow = deg > space ? deg - space : 0;
    total += (overflow + g->B - 1) / g->B;
  }
  if ((rc = ensure_available(g, total)) != ORC_OK) return rc;
  materialize(g, g->front + total);
  uint64_t pos = g->front;
  for (uint64_t v = 0; v < V; ++v) {
    const uint64_t deg = off[v + 1] - off[v];
    if (deg == 0) continue;
    Sentinel* s = &g->sent[v];
    const uint64_t space = s->block_count == 0 ? 0 : g->B - s->last_insert_offset;
    const uint64_t overflow = deg > space ? deg - space : 0;
    const uint64_t need = (overflow + g->B - 1) / g->B;
    /* attach fresh blocks in level order (cbt_attach, cbt.hpp:35-55) */
    const uint32_t first_fresh = s->block_count;
    if (s->block_count + need > s->blocks_cap) {
      uint32_t nc = s->blocks_cap ? s->blocks_cap : 2;
      while (nc < s->block_count + need) nc *= 2;
      s->blocks = (uint32_t*)realloc(s->blocks, nc * sizeof(uint32_t));
      s->blocks_cap = nc;
    }
    for (uint64_t j = 0; j < need; ++j) {
      const uint32_t h = g->ring[(pos + j) % g->ring_cap]; /* pop_range, block_pool.hpp:148-158 */
      if (h >= g->materialized) materialize(g, (uint64_t)h + 1);
      s->blocks[s->block_count++] = h;
    }
    pos += need;
    uint32_t cur, offset, next_fresh;
    if (space > 0) { cur = s->last_insert_block; offset = s->last_insert_offset; next_fresh = first_fresh; }
    else { cur = s->blocks[first_fresh]; offset = 0; next_fresh = first_fresh + 1; }
    for (uint64_t i = off[v]; i < off[v + 1]; ++i) {
      if (offset == g->B) { cur = s->blocks[next_fresh++]; offset = 0; }
      g->dst[(uint64_t)cur * g->B + offset] = dsts[i];
      g->tomb[(uint64_t)cur * g->B + offset] = 0;
      g->active[cur]++;
      g->occupied[cur]++;
      offset++;
    }
    s->active_edge_count += deg;
    s->last_insert_block = cur;
    s->last_insert_offset = offset;
  }
  g->active_edges += n;
  commit_front(g, total);
  return ORC_OK;
}

/* delete_batch (graph.hpp:195-222) = delete_adjacency (:376-394) +
 * detach_empty_tail (:398-414) + reclaim. */
int orc_delete_csr(void* p, const uint64_t* off, uint64_t n_off, const uint32_t* dsts, uint64_t n) {
  Oracle* g = (Oracle*)p;
  int rc = validate_batch(g, off, n_off, dsts, n);
  if (rc) return rc;
  const uint64_t V = g->size;
  uint32_t* freed = NULL; uint64_t nfreed = 0, cfreed = 0;
  uint32_t* tg = NULL; uint64_t tg_cap = 0;
  uint32_t* order = NULL; uint64_t order_cap = 0;
  for (uint64_t v = 0; v < V; ++v) {
    const uint64_t deg = off[v + 1] - off[v];
    if (deg == 0 || !g->alive[v]) continue; /* graph.hpp:205 */
    Sentinel* s = &g->sent[v];
    if (s->block_count == 0) continue;
    if (deg > tg_cap) { tg_cap = deg * 2; tg = (uint32_t*)realloc(tg, tg_cap * sizeof(uint32_t)); }
    memcpy(tg, dsts + off[v], deg * sizeof(uint32_t));
    qsort(tg, deg, sizeof(uint32_t), cmp_u32); /* membership set, graph.hpp:379 */
    if (s->block_count > order_cap) { order_cap = s->block_count * 2ull; order = (uint32_t*)realloc(order, order_cap * sizeof(uint32_t)); }
    in_order_positions(s->block_count, order);
    uint64_t matched = 0;
    for (uint32_t k = 0; k < s->block_count; ++k) {
      const uint32_t h = s->blocks[order[k] - 1];
      for (uint32_t i = 0; i < g->occupied[h]; ++i) {
        const uint64_t slot = (uint64_t)h * g->B + i;
        if (g->tomb[slot]) continue;
        const uint32_t key = g->dst[slot];
        if (bsearch(&key, tg, deg, sizeof(uint32_t), cmp_u32)) { /* every equal copy, graph.hpp:384-389 */
          g->tomb[slot] = 1;
          g->active[h]--;
          matched++;
        }
      }
    }
    s->active_edge_count -= matched;
    g->active_edges -= matched;
    if (g->reclaim_on_delete && matched > 0) { /* detach_empty_tail, graph.hpp:398-414 */
      int detached = 0;
      while (s->block_count > 0 && g->active[s->blocks[s->block_count - 1]] == 0) {
        if (nfreed == cfreed) { cfreed = cfreed ? cfreed * 2 : 64; freed = (uint32_t*)realloc(freed, cfreed * sizeof(uint32_t)); }
        freed[nfreed++] = s->blocks[--s->block_count];
        detached = 1;
      }
      if (detached) {
        if (s->block_count == 0) sentinel_reset(s);
        else {
          const uint32_t tail = s->blocks[s->block_count - 1];
          s->last_insert_block = tail;
          s->last_insert_offset = g->occupied[tail];
        }
      }
    }
  }
  reclaim(g, freed, nfreed);
  free(freed); free(tg); free(order);
  return ORC_OK;
}

/* csr_from_pairs (csr.hpp:29-45): stable counting sort by source */
static int pairs_to_csr(Oracle* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                        uint64_t** off_out, uint32_t** dst_out) {
  const uint64_t V = g->size;
  for (uint64_t i = 0; i < n; ++i)
    if (src[i] >= V) { snprintf(g->err, sizeof g->err, "csr batch: source out of range"); return ORC_ERR_DATA; }
  uint64_t* off = (uint64_t*)calloc(V + 1, sizeof(uint64_t));
  uint32_t* d = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) off[src[i] + 1]++;
  for (uint64_t v = 0; v < V; ++v) off[v + 1] += off[v];
  uint64_t* cur = (uint64_t*)malloc((V ? V : 1) * sizeof(uint64_t));
  memcpy(cur, off, V * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) d[cur[src[i]]++] = dst[i];
  free(cur);
  *off_out = off; *dst_out = d;
  return ORC_OK;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* *seconds (optional) receives the time of the engine call only: batch
 * construction is outside the reference's timed region. */
int orc_insert_coo(void* p, const uint32_t* src, const uint32_t* dst, uint64_t n, double* seconds) {
  Oracle* g = (Oracle*)p;
  uint64_t* off; uint32_t* d;
  int rc = pairs_to_csr(g, src, dst, n, &off, &d);
  if (rc) return rc;
  const double t0 = now_s();
  rc = orc_insert_csr(g, off, g->size + 1, d, n);
  if (seconds) *seconds = now_s() - t0;
  free(off); free(d);
  return rc;
}

int orc_delete_coo(void* p, const uint32_t* src, const uint32_t* dst, uint64_t n, double* seconds) {
  Oracle* g = (Oracle*)p;
  uint64_t* off; uint32_t* d;
  int rc = pairs_to_csr(g, src, dst, n, &off, &d);
  if (rc) return rc;
  const double t0 = now_s();
  rc = orc_delete_csr(g, off, g->size + 1, d, n);
  if (seconds) *seconds = now_s() - t0;
  free(off); free(d);
  return rc;
}

/* query_edge (graph.hpp:228-241) */
int orc_query(void* p, const uint32_t* src, const uint32_t* dst, uint64_t n, uint8_t* out) {
  Oracle* g = (Oracle*)p;
  for (uint64_t q = 0; q < n; ++q) {
    out[q] = 0;
    const uint32_t v = src[q];
    if (v >= g->size || !g->alive[v]) continue;
    const Sentinel* s = &g->sent[v];
    for (uint32_t k = 0; k < s->block_count && !out[q]; ++k) {
      const uint32_t h = s->blocks[k];
      for (uint32_t i = 0; i < g->occupied[h]; ++i) {
        const uint64_t slot = (uint64_t)h * g->B + i;
        if (!g->tomb[slot] && g->dst[slot] == dst[q]) { out[q] = 1; break; }
      }
    }
  }
  return ORC_OK;
}

/* insert_vertices (graph.hpp:246 -> vertex_dictionary.hpp:53-71) */
int orc_insert_vertices(void* p, uint64_t count) {
  Oracle* g = (Oracle*)p;
  if (count == 0) return ORC_OK;
  const uint64_t target = pow2_ceil(g->size + count);
  if (target > g->capacity) {
    const uint64_t new_bytes = target * (12 + 24);
    if (new_bytes > arena_available(&g->arena)) {
      snprintf(g->err, sizeof g->err, "vertex dictionary: arena cannot host capacity %llu", (unsigned long long)target);
      return ORC_ERR_ENGINE;
    }
    arena_reserve(&g->arena, target * 12);
    arena_reserve(&g->arena, target * 24);
    g->arena.reserved -= g->capacity * 12 + g->capacity * 24;
    g->capacity = target;
  }
  append_slots(g, count);
  return ORC_OK;
}

/* delete_vertices (graph.hpp:252-276) */
int orc_delete_vertices(void* p, const uint32_t* ids, uint64_t n, uint32_t* skipped, uint64_t* n_skipped) {
  Oracle* g = (Oracle*)p;
  uint64_t ns = 0;
  uint32_t* freed = NULL; uint64_t nfreed = 0, cfreed = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t v = ids[i];
    if (v >= g->size || !g->alive[v]) { if (skipped) skipped[ns] = v; ns++; continue; }
    Sentinel* s = &g->sent[v];
    g->active_edges -= s->active_edge_count;
    if (g->reclaim_on_delete && s->block_count > 0) {
      uint32_t* order = (uint32_t*)malloc(s->block_count * sizeof(uint32_t));
      in_order_positions(s->block_count, order);
      for (uint32_t k = 0; k < s->block_count; ++k) {
        const uint32_t h = s->blocks[order[k] - 1];
        g->active[h] = 0;
        if (nfreed == cfreed) { cfreed = cfreed ? cfreed * 2 : 64; freed = (uint32_t*)realloc(freed, cfreed * sizeof(uint32_t)); }
        freed[nfreed++] = h;
      }
      free(order);
      sentinel_reset(s);
    }
    g->alive[v] = 0; /* retire, vertex_dictionary.hpp:75-78 */
    g->alive_count--;
  }
  reclaim(g, freed, nfreed);
  free(freed);
  if (n_skipped) *n_skipped = ns;
  return ORC_OK;
}

uint32_t orc_block_size(void* p) { return ((Oracle*)p)->B; }
uint64_t orc_logical_size(void* p) { return ((Oracle*)p)->size; }
uint64_t orc_vertex_capacity(void* p) { return ((Oracle*)p)->capacity; }
uint64_t orc_alive_vertices(void* p) { return ((Oracle*)p)->alive_count; }
uint64_t orc_active_edges(void* p) { return ((Oracle*)p)->active_edges; }
int orc_vertex_alive(void* p, uint32_t v) { Oracle* g = (Oracle*)p; return v < g->size && g->alive[v]; }
uint64_t orc_queue_size(void* p) { Oracle* g = (Oracle*)p; return g->rear - g->front; }
uint64_t orc_blocks_in_use(void* p) { Oracle* g = (Oracle*)p; return g->created - (g->rear - g->front); }

/* sentinel_of(v).active_edge_count (graph.hpp:108) */
int orc_degrees(void* p, uint64_t* out) {
  Oracle* g = (Oracle*)p;
  for (uint64_t v = 0; v < g->size; ++v) out[v] = g->sent[v].active_edge_count;
  return ORC_OK;
}

/* Order-independent digest of the stored multiset: sum over live entries of mix64(v << 32 | dst)
 * (the device twin is digest_kernel; same coverage as orc_export_csr: active_destinations of every
 * v < logical_size, graph.hpp:116-129). */
static uint64_t orc_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
int orc_digest(void* p, uint64_t* digest, uint64_t* entries) {
  Oracle* g = (Oracle*)p;
  uint64_t acc = 0, cnt = 0;
  for (uint64_t v = 0; v < g->size; ++v) {
    const Sentinel* s = &g->sent[v];
    for (uint32_t k = 0; k < s->block_count; ++k) {
      const uint32_t h = s->blocks[k];
      for (uint32_t i = 0; i < g->occupied[h]; ++i) {
        const uint64_t slot = (uint64_t)h * g->B + i;
        if (g->tomb[slot]) continue;
        acc += orc_mix64((v << 32) | g->dst[slot]);
        cnt++;
      }
    }
  }
  if (digest) *digest = acc;
  if (entries) *entries = cnt;
  return ORC_OK;
}

/* active_destinations (graph.hpp:116-129) for every vertex, optionally sorted */
int orc_export_csr(void* p, uint64_t* offsets, uint32_t* dsts, uint64_t cap, int sorted) {
  Oracle* g = (Oracle*)p;
  uint64_t w = 0;
  uint32_t* order = NULL; uint64_t order_cap = 0;
  for (uint64_t v = 0; v < g->size; ++v) {
    offsets[v] = w;
    const Sentinel* s = &g->sent[v];
    if (s->block_count == 0) continue;
    if (s->block_count > order_cap) { order_cap = s->block_count * 2ull; order = (uint32_t*)realloc(order, order_cap * sizeof(uint32_t)); }
    in_order_positions(s->block_count, order);
    const uint64_t start = w;
    for (uint32_t k = 0; k < s->block_count; ++k) {
      const uint32_t h = s->blocks[order[k] - 1];
      for (uint32_t i = 0; i < g->occupied[h]; ++i) {
        const uint64_t slot = (uint64_t)h * g->B + i;
        if (g->tomb[slot]) continue;
        if (dsts) { if (w >= cap) { free(order); return ORC_ERR_DATA; } dsts[w] = g->dst[slot]; }
        w++;
      }
    }
    if (sorted && dsts) qsort(dsts + start, w - start, sizeof(uint32_t), cmp_u32);
  }
  offsets[g->size] = w;
  free(order);
  return ORC_OK;
}

/* ---- input generators (test inputs, not part of the data structure) ---------- */
#include "rmat.h"

void orc_gen_rmat(uint32_t scale, uint64_t seed, uint64_t first, uint64_t n, uint32_t ta,
                  uint32_t tab, uint32_t tabc, uint32_t* src, uint32_t* dst) {
  for (uint64_t i = 0; i < n; ++i) orc_rmat_edge(scale, seed, first + i, ta, tab, tabc, &src[i], &dst[i]);
}

/* std::mt19937_64 (the engine behind synth_uniform, io/synthetic.hpp:19-25):
 * the published MT19937-64 recurrence, restated so config 1's exact input
 * (synth_uniform(65536, 1000000, 0xbeef), acceptance_test.cpp:241) can be
 * regenerated where the reference is absent.  Pairs are in generation order.
 * NOTE: the reference writes `edges.emplace_back(rng() % V, rng() % V)`; the order of the two
 * draws is unspecified in C++ and g++ (the only toolchain the reference builds with here)
 * evaluates the arguments right to left, so the FIRST draw of a pair is the DESTINATION.
 * Pinned against dyngraph::io::synth_uniform itself (tests/golden/ref_io.npz). */
void orc_synth_uniform_pairs(uint64_t v, uint64_t e, uint64_t seed, uint32_t* src, uint32_t* dst) {
  enum { NN = 312, MM = 156 };
  static const uint64_t MATRIX_A = 0xB5026F5AA96619E9ull, UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  uint64_t mt[NN];
  int mti;
  mt[0] = seed;
  for (mti = 1; mti < NN; mti++) mt[mti] = 6364136223846793005ull * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
  for (uint64_t k = 0; k < 2 * e; ++k) {
    if (mti >= NN) {
      int i;
      for (i = 0; i < NN - MM; i++) { uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM); mt[i] = mt[i + MM] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX_A : 0ull); }
      for (; i < NN - 1; i++) { uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM); mt[i] = mt[i + (MM - NN)] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX_A : 0ull); }
      { uint64_t x = (mt[NN - 1] & UM) | (mt[0] & LM); mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ ((x & 1ull) ? MATRIX_A : 0ull); }
      mti = 0;
    }
    uint64_t x = mt[mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    if ((k & 1) == 0) dst[k >> 1] = (uint32_t)(x % v); else src[k >> 1] = (uint32_t)(x % v);
  }
}
