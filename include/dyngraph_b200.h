/*
 * dyngraph_b200.h — C ABI of libdyngraph_b200.so
 *
 * B200-native (sm_100a) replacement for the operator API of the CPU
 * reference's `class DynamicGraph` (reference: proj/include/dyngraph/graph.hpp:80-317)
 * plus its batch container `CsrBatch` (proj/include/dyngraph/csr.hpp:17-25).
 *
 * Conventions (mirroring SURVEY.md §8b):
 *   - every entry point returns an int status: DG_OK (0), DG_ERR_DATA (2) for
 *     malformed input (reference: DataError, types.hpp:25-27), DG_ERR_ENGINE
 *     (3) for resource exhaustion / contract violations (reference:
 *     EngineError, types.hpp:30-32), DG_ERR_CUDA (4) for a CUDA runtime
 *     failure.  The numeric values 2/3 follow the reference CLI's exit codes
 *     (proj/tools/dyngraph.cpp:17-20).
 *   - no exception crosses the ABI; dg_last_error() returns the message.
 *   - on any non-zero return from a mutating call the graph is unchanged
 *     (validate-then-mutate, reference graph.hpp:168-171).
 *   - the graph owns all device storage; batches are borrowed for the call.
 *   - one caller at a time; batches never overlap.
 *   - every pointer argument carrying bulk data has a `mem` selector saying
 *     whether it points to host memory (DG_MEM_HOST: the library stages it
 *     to the device) or device memory (DG_MEM_DEVICE: used in place, on the
 *     graph's stream).
 *
 * Semantics are the reference's: the store is a MULTISET (inserts never
 * de-duplicate, graph.hpp:355-366), one delete entry removes every equal
 * copy (graph.hpp:379-391), deletes listing a dead source are ignored
 * (graph.hpp:205), inserts listing a dead source reject the whole batch
 * (graph.hpp:322-327), destinations are only range-checked against the
 * logical size (csr.hpp:67-72).
 */
#ifndef DYNGRAPH_B200_H
#define DYNGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_ABI_VERSION 1

/* status codes */
#define DG_OK 0
#define DG_ERR_DATA 2
#define DG_ERR_ENGINE 3
#define DG_ERR_CUDA 4

/* memory-space selector for bulk pointers */
#define DG_MEM_HOST 0
#define DG_MEM_DEVICE 1

/* dg_config.flags */
#define DG_FLAG_NO_RECLAIM 1u /* reclaim_on_delete = false (graph.hpp:26) */
/* How a COO batch is grouped by source (default: chosen per batch from V and n):
 * RADIX = pack keys + LSD radix sort, O(n); COUNT = per-vertex counters + scan, O(V + n). */
#define DG_FLAG_GROUP_RADIX 2u
#define DG_FLAG_GROUP_COUNT 4u
/* block_size = 0 asks for the reference's rule (compute_block_size, csr.hpp:77-88: round-half-up of edges per
 * non-empty source of the first batch).  With this flag a result in [24, 48] becomes 32, the NATIVE block (one
 * 128-byte line: the fused delete, the TMA-staged CSR append and the bulk-init copy are written for it; a 33-slot
 * block is not even 16-byte aligned).  An explicit deviation from the reference's value — block counts, and with
 * them the point where a fixed pool underflows, follow the block size actually used (dg_block_size reports it). */
#define DG_FLAG_AUTO_BLOCK_NATIVE 8u
/* Contract for dg_submit_*_coo: the device arrays handed to a submit call are COMPLETE when the call is made — nothing
 * enqueued on the graph's stream (after the previous submit) produces them.  With this flag the library may start the
 * op's first kernel (the per-source count, which reads only the batch) on a side stream beside the previous
 * submitted op's last kernel, i.e. before the point in the graph's stream where the op itself is enqueued.  Without
 * it every kernel of an op stays behind everything enqueued on the graph's stream before the call.  (The ingest queue
 * needs no flag: it orders the early kernel behind the slot's own copy.) */
#define DG_FLAG_SUBMIT_INPUTS_READY 16u

/* reference: types.hpp:16-17 (kInvalidVertex / kNullBlock) */
#define DG_INVALID_VERTEX 0xFFFFFFFFu
#define DG_NULL_BLOCK 0xFFFFFFFFu

typedef struct dg_graph dg_graph; /* opaque handle */

/*
 * Replaces GraphConfig (graph.hpp:23-28) + GrowthPolicy (block_pool.hpp:18-29).
 * `pool_bytes` plays the role of arena_bytes * initial_fraction: the device
 * bytes given to the edge-block pool (dst slab + next links + free ring).
 * A zero-initialised struct means: device 0, 1 GiB pool, reclaim on, own stream.
 */
typedef struct dg_config {
  int32_t device;            /* CUDA device ordinal */
  uint32_t flags;            /* DG_FLAG_*; 0 => reclaim_on_delete = true (graph.hpp:26) */
  uint64_t pool_bytes;       /* 0 => 1 GiB */
  uint64_t pool_blocks;      /* if non-zero, overrides pool_bytes: exact block count */
  void* stream;              /* cudaStream_t to enqueue on; NULL => library-owned stream */
  uint64_t workspace_bytes;  /* per-op scratch reserved at create (0 => grown on first use) */
  /* Edge-queue growth (GrowthPolicy, block_pool.hpp:18-29; commit_front / ensure_available /
   * try_grow, :162-189, :252-264).  pool_max_blocks plays the arena's role: the most blocks the
   * pool may ever hold.  0 (or <= the initial count) => fixed pool, underflow is an engine error.
   * Otherwise the pool grows by growth_fraction of its capacity whenever cumulative consumption
   * reaches trigger_fraction of it (checked after every insert) and on demand when a batch needs
   * more blocks than are queued; device memory is committed in place (CUDA virtual memory
   * management: the address range is reserved once, physical chunks are mapped as the pool
   * grows, nothing is copied). */
  uint64_t pool_max_blocks;
  float trigger_fraction;    /* 0 => 0.8 */
  float growth_fraction;     /* 0 => 0.25 */
  uint32_t reserved[2];
} dg_config;

/* Replaces GraphStats (graph.hpp:54-70); reported, not compared. */
typedef struct dg_stats {
  uint64_t logical_size;
  uint64_t capacity;
  uint64_t alive_vertices;
  uint64_t active_edges;
  uint64_t adjacency_blocks;   /* blocks held by chains of alive vertices */
  uint64_t occupied_slots;     /* == live entries: chains are kept compact */
  uint64_t hole_slots;         /* always 0 after a delete completes */
  uint64_t pool_blocks_created;
  uint64_t pool_blocks_in_use;
  uint64_t pool_queue_size;
  uint64_t queue_front;        /* unwrapped coordinates, block_pool.hpp:31-34 */
  uint64_t queue_rear;
  uint64_t max_degree;
  uint32_t block_size;
  uint32_t growth_count;       /* growth rounds so far (block_pool.hpp growth_count()) */
} dg_stats;

/* Replaces MemoryBreakdown (graph.hpp:43-52) with real device allocations. */
typedef struct dg_memory {
  uint64_t dictionary_bytes; /* alive bitmap + degree array */
  uint64_t sentinel_bytes;   /* head/tail arrays */
  uint64_t pool_bytes;       /* blocks held by adjacencies * bytes per block */
  uint64_t queue_bytes;      /* free ring */
  uint64_t pool_reserved_bytes; /* whole slab + links */
  uint64_t workspace_bytes;  /* per-batch scratch (sort buffers, work lists) */
} dg_memory;

/* Per-op device timings/counters of the LAST completed op (reported only). */
typedef struct dg_op_report {
  uint64_t batch_entries;   /* n */
  uint64_t touched_sources; /* T: distinct sources in the batch */
  uint64_t blocks_popped;   /* fresh blocks taken from the queue */
  uint64_t blocks_pushed;   /* blocks returned to the queue */
  uint64_t slots_scanned;   /* S: slots of touched chains inspected (delete/query) */
  uint64_t blocks_scanned;
  uint64_t matched;         /* entries removed (delete) / queries answered true */
  uint64_t moved;           /* entries moved by compaction */
  uint64_t kernel_launches; /* kernels enqueued by the op */
  uint64_t slots_scanned_long; /* part of slots_scanned handled by the CTA-table tier (k > 128 targets) */
  uint64_t slots_scanned_tiny; /* part handled by the register-compare tier (k <= 8 targets) */
  uint64_t slots_scanned_fused; /* part handled by fused_delete_kernel (sources a single warp owns) */
} dg_op_report;

/* ---- lifecycle ------------------------------------------------------- */

/* ABI version of the loaded library. */
int dg_abi_version(void);

/* Message of the last failing call on this handle (or on create when h==NULL). */
const char* dg_last_error(const dg_graph* h);

/*
 * Replaces DynamicGraph::DynamicGraph(config, initial_vertex_count, block_size)
 * (graph.hpp:84-91): vertex dictionary as device SoA arrays sized to
 * closest_pow2(initial_vertices) (vertex_dictionary.hpp:30-37, bits.hpp:11-16),
 * the block pool, and the free ring filled with every handle
 * (block_pool.hpp:99-116, :242-247).  block_size == 0 defers the pool until
 * the first insert batch and then applies compute_block_size (csr.hpp:77-88).
 */
int dg_create(const dg_config* config, uint64_t initial_vertices, uint32_t block_size,
              dg_graph** out);
void dg_destroy(dg_graph* h);

/* ---- batch edge updates ---------------------------------------------- */

/*
 * Replaces insert_batch(const CsrBatch&) (graph.hpp:167-188) with the same
 * validation as validate_batch (csr.hpp:49-73) + the dead-source rule
 * (graph.hpp:320-328).  `offsets` has n_offsets = logical_size + 1 entries.
 */
int dg_insert_batch_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets,
                        const uint32_t* destinations, uint64_t n_edges, int mem);
/* Replaces delete_batch(const CsrBatch&) (graph.hpp:195-222). */
int dg_delete_batch_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets,
                        const uint32_t* destinations, uint64_t n_edges, int mem);

/*
 * O(batch) entry points: the same two operators fed with (src,dst) pairs, i.e.
 * insert_batch(csr_from_pairs(Insert, logical_size, pairs)) without the O(V)
 * offsets array (csr.hpp:29-45).  These are the measured entry points.
 */
int dg_insert_batch_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n,
                        int mem);
int dg_delete_batch_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n,
                        int mem);

/*
 * Validation + plan of a COO batch WITHOUT applying it: the status dg_insert_batch_coo / dg_delete_batch_coo
 * would return (validate_batch csr.hpp:49-73, dead-source rule graph.hpp:320-328, ensure_available
 * block_pool.hpp:177-189).  The source-partitioned store calls it on every rank and agrees on the outcome
 * before any rank mutates (NCCL exchange; the peer-memory exchange agrees on the device instead).
 */
int dg_check_batch_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, int is_insert, int mem);

/*
 * Bulk init = the reference's ctor followed by the first insert_batch of the
 * whole graph (io/workload.hpp:113-139).  Requires an empty graph whose
 * logical size is n_offsets - 1; identical to dg_insert_batch_csr otherwise.
 */
int dg_bulk_init_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets,
                     const uint32_t* destinations, uint64_t n_edges, int mem);

/* ---- queries ----------------------------------------------------------- */

/*
 * Batched query_edge (graph.hpp:228-241): out[i] = 1 iff a live entry
 * src[i] -> dst[i] exists; unknown or dead sources answer 0.
 */
int dg_query_edges(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n,
                   uint8_t* out, int mem);

/*
 * active_destinations over every vertex (graph.hpp:116-129) as one CSR:
 * offsets[logical_size + 1] (u64) and destinations[sum of degrees].  With
 * sorted != 0 each vertex's run is ascending (the canonical sorted multiset
 * compared by oracle_compare, oracle.hpp:123-140).  Dead vertices contribute
 * whatever the reference's sentinel would still hold: nothing when
 * reclaim_on_delete, their retained entries otherwise (graph.hpp:264-272).
 * Call with destinations == NULL to obtain only the offsets; n_dst_capacity
 * is the capacity of `destinations` in entries.
 */
int dg_export_csr(dg_graph* h, uint64_t* offsets, uint32_t* destinations,
                  uint64_t n_dst_capacity, int sorted, int mem);

/*
 * active_destinations(v) (graph.hpp:116-129) for ONE vertex: its live destinations in traversal order, at
 * most `capacity` of them, into `out` (host or device per `mem`); *n_out receives the vertex's degree.
 * An unknown vertex yields 0 entries (graph.hpp:118).  DG_ERR_DATA (with *n_out set) when capacity < degree:
 * call again with a larger buffer — dg_degrees / a first call with capacity 0 give the size.
 */
int dg_active_destinations(dg_graph* h, uint32_t v, uint32_t* out, uint64_t capacity, uint64_t* n_out, int mem);

/* sentinel_of(v).active_edge_count for every v < logical_size (graph.hpp:108). */
int dg_degrees(dg_graph* h, uint64_t* out, int mem);

/*
 * Order-independent 64-bit digest of the stored multiset: sum over stored
 * copies of mix64(src, dst) — for scales where a full
 * CSR comparison is too heavy.  Same vertex coverage as dg_export_csr.
 */
int dg_digest(dg_graph* h, uint64_t* out_digest, uint64_t* out_entries);

/* ---- vertex updates ------------------------------------------------------ */

/* insert_vertices (graph.hpp:246 -> vertex_dictionary.hpp:53-71). */
int dg_insert_vertices(dg_graph* h, uint64_t count);
/*
 * delete_vertices (graph.hpp:252-276).  `ids` is a HOST array.  Unknown,
 * already-dead and in-call duplicate ids are written to skipped[] (capacity
 * n) in encounter order; *n_skipped receives their number.
 */
int dg_delete_vertices(dg_graph* h, const uint32_t* ids, uint64_t n, uint32_t* skipped,
                       uint64_t* n_skipped);

/* ---- observables (graph.hpp:96-108) ------------------------------------- */

uint32_t dg_block_size(const dg_graph* h);
uint64_t dg_logical_size(const dg_graph* h);
uint64_t dg_vertex_capacity(const dg_graph* h);
uint64_t dg_alive_vertices(const dg_graph* h);
uint64_t dg_active_edges(const dg_graph* h);
int dg_vertex_alive(const dg_graph* h, uint32_t v);

int dg_stats_get(dg_graph* h, dg_stats* out);          /* stats(), graph.hpp:287-317 */
int dg_memory_get(const dg_graph* h, dg_memory* out);  /* memory(), graph.hpp:278-285 */
int dg_last_op_report(const dg_graph* h, dg_op_report* out);

/*
 * Per-kernel device timing for measurement runs: with profiling on, every
 * kernel launch of this graph is bracketed by CUDA events on the graph's
 * stream.  dg_profile_report returns one "name<TAB>total_ms<TAB>launches" line
 * per kernel accumulated since profiling was last enabled (valid until the
 * next call).  Adds event overhead: never enable it for a throughput number.
 */
int dg_profile_enable(dg_graph* h, int on);
const char* dg_profile_report(dg_graph* h);

/* The CUDA stream (cudaStream_t) every op of this graph is enqueued on. */
void* dg_stream(const dg_graph* h);
/* Block until every enqueued op finished. */
int dg_synchronize(dg_graph* h);

/* ---- helpers that are part of the path's input side ---------------------- */

/*
 * compute_block_size (csr.hpp:77-88) for a COO batch: round-half-up of
 * n / #distinct sources, never below 1.  DG_ERR_DATA when n == 0.
 */
int dg_compute_block_size_coo(dg_graph* h, const uint32_t* src, uint64_t n, int mem,
                              uint32_t* out_block_size);

/*
 * Counter-based R-MAT generator (the reference ships no
 * R-MAT): edge i of (seed) is a pure function of (seed, first_index + i), so
 * host (oracle/rmat.h) and device produce identical pairs.  Probabilities are
 * given as 32-bit fixed-point thresholds a, a+b, a+b+c (out of 2^32).
 * Writes DEVICE arrays src[n], dst[n] on the graph's stream.
 */
int dg_gen_rmat(dg_graph* h, uint32_t scale, uint64_t seed, uint64_t first_index, uint64_t n,
                uint32_t thr_a, uint32_t thr_ab, uint32_t thr_abc, uint32_t* src_dev,
                uint32_t* dst_dev);

/*
 * Stable grouping of a COO batch into CSR on the device (the GPU twin of
 * csr_from_pairs, csr.hpp:29-45): offsets_dev[vertex_count + 1] (u64) and
 * destinations_dev[n], both DEVICE arrays.  Used to prepare bulk-init input.
 */
int dg_coo_to_csr(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, int mem,
                  uint64_t vertex_count, uint64_t* offsets_dev, uint32_t* destinations_dev);

/* ---- multi-GPU routing (nothing in the reference) ---------- */

/*
 * Source-partitioned sharding: owner(v) = perm(v) mod world and local id =
 * perm(v) / world, where perm is a fixed bijection on [0, 2^bits) (a mixing
 * permutation, because R-MAT sources with equal low bits carry ~44% of the
 * edges, SURVEY.md §7 "Hashed ownership").  Each rank owns a dg_graph over
 * its local ids whose destinations stay GLOBAL ids, validated against
 * dg_set_dst_limit().
 */
uint32_t dg_owner_perm(uint32_t v, uint32_t bits);
uint32_t dg_owner_perm_inv(uint32_t p, uint32_t bits);

/* Destinations must be < limit (0 => the logical size, the single-GPU rule csr.hpp:67-72). */
int dg_set_dst_limit(dg_graph* h, uint64_t limit);

/*
 * Owner-bucket partition of a COO batch (the send side of the all-to-all).
 * Validates src < vertex_count (DG_ERR_DATA otherwise, nothing written) and
 * writes, grouped by owner in rank order and stable within an owner,
 * out_src_local[n] (local ids), out_dst[n] (global ids) and out_index[n]
 * (position in the input, for routing query answers back).  counts_host[world]
 * (HOST, u64) receives the per-owner sizes.  All bulk pointers are DEVICE.
 */
int dg_route_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n,
                 uint32_t world, uint32_t bits, uint64_t vertex_count, uint32_t* out_src_local,
                 uint32_t* out_dst, uint32_t* out_index, uint64_t* counts_host);

/*
 * Fused routing + exchange over peer memory (NVLink P2P): instead of
 * partition -> count exchange -> NCCL all-to-all, ONE kernel computes every
 * pair's owner and stores it straight into the owner's receive buffer
 * (peer-mapped through CUDA IPC), reserving slots with a warp-aggregated
 * system-scope atomicAdd on the owner's cursor.  The round protocol runs ON
 * THE DEVICE — no host collective per batch: arrival and status counters live
 * in the peer-mapped buffers (system-scope atomics + a one-warp waiting
 * kernel), two buffer sets alternate between rounds.
 *
 * One round = one batch op; every rank calls the same sequence:
 *     dg_exchange_push_coo      validate + push + "my push has landed" to every rank
 *     dg_exchange_received      wait for every rank's arrival; what this rank received
 *     the local batch op on the received DEVICE arrays (with dg_exchange_attach the op posts its
 *       validation / plan status to every rank and mutates only on an all-clear: a batch is applied
 *       on every rank or on none, graph.hpp:168-171), or dg_exchange_agree when nothing was received
 *     [queries: dg_exchange_push_answers ; dg_exchange_answers]
 *     dg_exchange_end_round
 * A rank that fails to take part makes its peers give up after ~4 s with DG_ERR_ENGINE.
 */
typedef struct dg_exchange dg_exchange;
#define DG_IPC_HANDLE_BYTES 64

/* capacity: most entries this rank can receive (and most answers it can get back) in one round */
int dg_exchange_create(dg_graph* h, uint32_t rank, uint32_t world, uint64_t capacity, dg_exchange** out);
void dg_exchange_destroy(dg_exchange* x);
/* IPC handle of this rank's buffers (64 bytes) — all-gather it, then hand every peer's to set_peer */
int dg_exchange_ipc_handle(dg_exchange* x, void* handle_out);
int dg_exchange_set_peer(dg_exchange* x, uint32_t peer_rank, const void* handle);
/* on != 0: insert / delete COO ops of x's graph agree their status with the peers before mutating */
int dg_exchange_attach(dg_exchange* x, int on);
/* validates src < vertex_count, pushes (local src id, global dst, origin index) of every pair to its owner and
 * signals this rank's arrival (carrying its status) to every rank.  src/dst: DEVICE arrays.  A local
 * DG_ERR_* is returned here; the other ranks learn it in dg_exchange_received. */
int dg_exchange_push_coo(dg_exchange* x, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t bits,
                         uint64_t vertex_count);
/* waits until every rank has arrived; what this rank received (DEVICE arrays owned by the exchange).
 * DG_ERR_DATA / DG_ERR_ENGINE on EVERY rank when any rank's push was rejected (nothing to apply). */
int dg_exchange_received(dg_exchange* x, uint64_t* n, uint32_t** src_local, uint32_t** dst,
                         uint32_t** origin_index, uint32_t** origin_rank);
/* the agreement step for a rank that runs no local op this round; *agreed = max status over the ranks */
int dg_exchange_agree(dg_exchange* x, int local_status, int* agreed);
/* answers[i] (DEVICE, one per received entry) go to answer slot origin_index[i] of rank origin_rank[i] */
int dg_exchange_push_answers(dg_exchange* x, const uint8_t* answers, uint64_t n);
/* waits for every rank's answers; the first n (indexed by the position in this rank's own query batch)
 * are copied to `out` (host or device per `mem`) */
int dg_exchange_answers(dg_exchange* x, uint8_t* out, uint64_t n, int mem);
/* the round is over: its buffer set is handed back, the next round uses the other one */
int dg_exchange_end_round(dg_exchange* x);

/*
 * dg_digest of a shard expressed over GLOBAL source ids (local id l of rank r is vertex
 * perm_inv(l * world + r)): the sum over the ranks equals the single-GPU digest of the same multiset.
 */
int dg_digest_global(dg_graph* h, uint32_t rank, uint32_t world, uint32_t bits, uint64_t* out_digest, uint64_t* out_entries);

/* plan_batch (graph.hpp:135-160) -> BatchPlan (graph.hpp:33-39): validates an INSERT batch exactly as
 * dg_insert_batch_csr does (csr.hpp:49-73, dead-source rule graph.hpp:322-327; DG_ERR_DATA otherwise) and fills, per
 * vertex, the fresh blocks the batch needs (blocks_required), their inclusive prefix sum in vertex order (prefix_sum:
 * the reference's pop schedule) and the free slots of the vertex's last-insert block (space_remaining); *total_blocks
 * (optional) = prefix_sum[V - 1].  Nothing is mutated.  `mem` says where the batch AND the three output arrays
 * (V entries each) live.  space_remaining follows this library's compact chains: equal to the reference's after any
 * insert-only history, smaller or equal after deletes (the reference keeps holes; physical layout is reported, not
 * compared).  DG_ERR_ENGINE while the graph has no pool yet (block_size 0 before the first insert). */
int dg_plan_batch_csr(dg_graph* h, const uint64_t* offsets, uint64_t n_offsets, const uint32_t* destinations,
                      uint64_t n_edges, int mem, uint64_t* blocks_required, uint64_t* prefix_sum,
                      uint32_t* space_remaining, uint64_t* total_blocks);

/* ---- host -> device batch ingest (nothing in the reference) ----------
 *
 * The reference harness hands insert_batch / delete_batch one host batch after the other
 * (io/workload.hpp:141-155).  On the GPU the PCIe copy of a 1M-entry batch (8 MB) costs as much as
 * the op, so an ingest queue keeps `depth` device slots and copies batch k+1 on its own stream
 * while batch k executes:
 *     dg_ingest_stage_coo(q, batch[0]) ;
 *     for k: dg_ingest_stage_coo(q, batch[k+1]) ; dg_ingest_insert(q, slot[k]) ;
 * `src`/`dst` are HOST arrays (pinned memory makes the copy asynchronous) that must stay valid
 * until the slot's op returns.  The ops are dg_insert_batch_coo / dg_delete_batch_coo on the
 * staged device copy: same validation, same status codes, graph unchanged on failure.
 */
typedef struct dg_ingest dg_ingest;
int dg_ingest_create(dg_graph* h, uint64_t max_entries, uint32_t depth, dg_ingest** out);
void dg_ingest_destroy(dg_ingest* q);
/* enqueue the copy of a host COO batch into the next free slot; *slot receives its index */
int dg_ingest_stage_coo(dg_ingest* q, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t* slot);
/* run the op on a staged slot (waits for its copy on the graph's stream); frees the slot */
int dg_ingest_insert(dg_ingest* q, uint32_t slot);
int dg_ingest_delete(dg_ingest* q, uint32_t slot);
/* drop every staged batch (after a failed op: the reference loop would have stopped there) */
int dg_ingest_reset(dg_ingest* q);
/* the same ops SUBMITTED (see below): no host wait, the slot is handed back by an event on the graph's stream;
 * the host arrays must stay valid until a later dg_flush returned (or depth + 8 more batches were submitted) */
int dg_ingest_submit_insert(dg_ingest* q, uint32_t slot, uint64_t* ticket);
int dg_ingest_submit_delete(dg_ingest* q, uint32_t slot, uint64_t* ticket);

/* ---- submitted updates: insert_batch / delete_batch without a host round trip per batch -------
 *
 * The reference's callers apply batches in a loop (io/workload.hpp:141-155): each call validates, mutates
 * and returns or throws before the next one starts (graph.hpp:167-188, :195-222).  The synchronous entry
 * points above keep that shape and pay one host wait per batch, during which the GPU idles.
 * dg_submit_insert_coo / dg_submit_delete_coo enqueue the same op on the graph's stream and return at once;
 * dg_flush waits for everything submitted and returns the FIRST failure (DG_OK when every op applied).
 * The reference's contract is kept on the device: an op submitted behind one that failed does not run (every
 * kernel of it returns at its first line) — a failed batch is reported before anything after it mutates
 * (graph.hpp:168-171).  After a failure dg_flush sets *n_applied to the number of submitted ops that were
 * applied since the previous dg_flush: exactly the ops before the failed one; the caller may fix the batch and
 * submit again from there.  Until the failure has been returned (by dg_flush, or by the next synchronous call
 * of any kind, which returns it INSTEAD of running) further submits are refused with the same status.
 * `src` / `dst` are DEVICE arrays that must stay valid until the op has been flushed.  *ticket (optional)
 * receives the op's sequence number, 0 when the call ran the op synchronously: when the host cannot bound
 * what it would otherwise decide between two ops (pool underflow -> growth, block_pool.hpp:177-189; the growth
 * trigger, :162-172; sharded stores; a graph without a pool yet) the call waits for what is in flight and runs
 * the op the synchronous way — outcomes never differ, only the overlap is lost.  Every other entry point first
 * waits for the submitted ops, so mixing is safe.  At most 7 submitted ops are in flight; one more submit waits
 * for the oldest.
 */
int dg_submit_insert_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t* ticket);
int dg_submit_delete_coo(dg_graph* h, const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t* ticket);
int dg_flush(dg_graph* h, uint64_t* n_applied);
uint64_t dg_pending_ops(const dg_graph* h);

#ifdef __cplusplus
}
#endif
#endif /* DYNGRAPH_B200_H */
