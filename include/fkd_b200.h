/*
 * fkd_b200.h — C ABI of the B200-native stack-free k-d tree query engine.
 *
 * This is the drop-in boundary for the reference's batch query path
 * (flatkd::run_batch, /root/reference/proj/src/batch.cpp:71-134, declared at
 * proj/include/flatkd/batch.hpp:47).  Plain pointers and sizes only; no
 * torch or C++ types.  A C++ shim with the reference's own signatures
 * (flatkd::b200::run_batch / fcp / knn over KdTree, PointSet, BatchOptions,
 * BatchResult) sits on top in include/flatkd_b200/flatkd.hpp.
 *
 * Semantics follow the reference exactly:
 *   - tree: level-order left-balanced complete k-d tree, row-major float[n*dim],
 *     node index = slot, round-robin split dim = depth % dim
 *     (proj/include/flatkd/tree.hpp:12-29, 41-65);
 *   - results: fixed-stride slots, stride = (knn ? k : 1); counts[i] valid hits
 *     ascending by (dist2, node) (hit_order, traverse.hpp:80-83), the rest of
 *     the slot pre-filled with {-1, +inf} (batch.hpp:25-41, batch.cpp:82-86);
 *   - dist2 bit-identical to the reference's left-to-right float
 *     accumulation without FMA (point.hpp:68-75);
 *   - validation order of batch.cpp:72-80, one status per exception type.
 *
 * Every call is re-entrant.  An fkd_tree is immutable after creation and may
 * be shared by any number of concurrent callers.
 */
#ifndef FKD_B200_H
#define FKD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the C++ shim re-throws the reference's exception types. */
typedef enum fkd_status {
    FKD_OK = 0,
    FKD_INVALID_ARGUMENT = 1,  /* std::invalid_argument (e.g. knn k < 1, batch.cpp:72-73) */
    FKD_DATA_ERROR = 2,        /* flatkd::DataError (error.hpp:9-12)                      */
    FKD_INVARIANT_ERROR = 3,   /* flatkd::InvariantError (error.hpp:15-18)                */
    FKD_CUDA_ERROR = 4,        /* device or runtime failure (no CPU fallback exists)      */
    FKD_NO_DEVICE = 5          /* no usable sm_100 device                                  */
} fkd_status;

/* flatkd::QueryKind (batch.hpp:11) */
typedef enum fkd_query_kind { FKD_FCP = 0, FKD_KNN = 1 } fkd_query_kind;

/* flatkd::Engine (batch.hpp:10).  Both engines return identical results; they
 * differ only in how QueryStats count steps (traverse.hpp:250-293). */
typedef enum fkd_engine { FKD_ENGINE_STACK_FREE = 0, FKD_ENGINE_RECURSIVE = 1 } fkd_engine;

/* fkd_batch_options.flags */
#define FKD_FLAG_MORTON     0x1u /* walk queries in Morton order (results land in input order) */
#define FKD_FLAG_UNORDERED  0x2u /* left-first child order instead of close-first */
#define FKD_FLAG_NO_MORTON  0x4u /* force input order even where MORTON is the default        */

/* flatkd::Hit (traverse.hpp:70-76): int32 at offset 0, float at 4, 8 bytes. */
typedef struct fkd_hit {
    int32_t node;
    float dist2;
} fkd_hit;

/* flatkd::QueryStats (traverse.hpp:46-54): three 64-bit counters. */
typedef struct fkd_query_stats {
    int64_t steps;
    int64_t nodes_visited;
    int64_t nodes_processed;
} fkd_query_stats;

/* flatkd::BatchOptions (batch.hpp:16-23) plus B200 flags. */
typedef struct fkd_batch_options {
    int32_t kind;          /* fkd_query_kind                                  */
    int32_t k;             /* knn only                                        */
    float max_radius;      /* inclusive; +inf = unbounded                      */
    int32_t engine;        /* fkd_engine                                      */
    int32_t threads;       /* accepted for signature parity; ignored on GPU   */
    int32_t collect_stats; /* fill *stats with batch totals                    */
    uint32_t flags;        /* FKD_FLAG_*                                       */
} fkd_batch_options;

/* Per-stage device timings of one fkd_run_batch_device call (CUDA events on
 * the launch stream), filled only when the caller passes a non-NULL pointer
 * (adds one stream synchronisation). */
typedef struct fkd_timings {
    float order_ms;   /* Morton keys + radix sort (0 when not sorting)          */
    float walk_ms;    /* traversal kernel(s), overflow pass included             */
    float tail_ms;    /* of walk_ms: the overflow pass for over-budget queries   */
    int32_t launches; /* kernels this library launched for the call             */
    int32_t walk_launches;
    int64_t overflowed; /* queries that left the walk kernel over its step budget
                           (last sub-batch of <= 2^30 queries)                    */
} fkd_timings;

typedef struct fkd_tree fkd_tree;

/* Defaults: kind=fcp, k=1, max_radius=+inf, engine=stack_free, threads=0,
 * collect_stats=0, flags=FKD_FLAG_MORTON (batch.hpp:16-23). */
void fkd_default_options(fkd_batch_options* opt);

/* ---- tree store (replaces flatkd::KdTree::from_level_order, tree.cpp:71-78) ----
 * Copies a level-order host array onto each listed device (ndev >= 1; devices
 * may be NULL meaning {current device}).  The caller keeps ownership of the
 * host array.  Rejects non-finite coordinates with FKD_DATA_ERROR
 * ("tree nodes: non-finite coordinate in point i", point.hpp:59-63). */
fkd_status fkd_tree_create(const float* level_order, int64_t n, int32_t dim,
                           const int32_t* devices, int32_t ndev, fkd_tree** out);

/* Same, from a device-resident level-order array on the current device
 * (e.g. a tensor that arrived by NCCL broadcast).  The array is copied. */
fkd_status fkd_tree_create_device(const float* d_level_order, int64_t n, int32_t dim,
                                  void* stream, fkd_tree** out);

void fkd_tree_destroy(fkd_tree* tree);
int64_t fkd_tree_size(const fkd_tree* tree);
int32_t fkd_tree_dim(const fkd_tree* tree);
/* Devices holding a replica of the tree store, in shard order: writes up to
 * `cap` device ids to `devices` (may be NULL) and returns the replica count.
 * fkd_run_batch_device runs on the first one. */
int32_t fkd_tree_replicas(const fkd_tree* tree, int32_t* devices, int32_t cap);

/* Morton keys of device queries over the tree's bounding box (the key the
 * batch ordering uses, at full resolution: *key_bits = bits per axis x dim,
 * <= 24), for partitioning a batch across GPUs by key range
 * (paper_2210_12859_b200/shard.py).  Rejects non-finite queries. */
fkd_status fkd_morton_keys(const fkd_tree* tree, const float* d_queries, int64_t m, int32_t dim,
                           uint32_t* d_keys, int32_t* key_bits, void* stream);

/* Adds replicas of the tree store on `devices` (appended to the shard
 * order), copied device to device from the existing replicas as a pipelined
 * chain over NVLink / NVSwitch (64 MB pieces; cudaMemcpyPeerAsync staging
 * through the host where a pair has no peer access).  Not thread-safe with
 * concurrent queries on the same tree. */
fkd_status fkd_tree_add_replicas(fkd_tree* tree, const int32_t* devices, int32_t ndev);

/* ---- the batch query path (replaces flatkd::run_batch, batch.cpp:71-134) ----
 * Host buffers: queries[m*dim] row-major; counts[m]; hits[m*stride];
 * stats may be NULL.  Queries are sharded over the tree's devices; H2D, the
 * walk and D2H are pipelined in chunks.  Blocks until the results are in
 * the caller's buffers. */
fkd_status fkd_run_batch(const fkd_tree* tree, const float* queries, int64_t m, int32_t dim,
                         const fkd_batch_options* opt, int32_t* counts, fkd_hit* hits,
                         fkd_query_stats* stats);

/* One host-buffer batch of fkd_run_batches. */
typedef struct fkd_host_batch {
    const float* queries;     /* m x dim, host                               */
    int64_t m;
    int32_t dim;
    fkd_batch_options opt;
    int32_t* counts;          /* [m], host                                   */
    fkd_hit* hits;            /* [m * stride], host                          */
    fkd_query_stats* stats;   /* may be NULL                                 */
    fkd_status status;        /* out: this batch's status                    */
} fkd_host_batch;

/* Several host-buffer batches in one call.  Batches over the same query
 * array (same pointer, m and dim) run as one pipeline: the queries are
 * uploaded, checked and Morton-ordered once per chunk and walked by every
 * batch of the group; other batches run afterwards.  Each batch keeps its own
 * results, counters and status; returns the first non-OK status. */
fkd_status fkd_run_batches(const fkd_tree* tree, fkd_host_batch* batches, int32_t n);

/* Asynchronous fkd_run_batches (a serving loop's submission): starts the
 * batches on a library thread and returns at once with a job handle;
 * fkd_wait joins the job, frees the handle and returns what fkd_run_batches
 * would have (status fields, outputs and counters are valid from then on, and
 * fkd_last_error on the waiting thread explains a failure).  Several jobs may
 * be in flight on one tree: their pipelines share the device, so one job's
 * uploads and walks overlap the previous job's result copies.  The tree, the
 * batch array and every buffer it names must stay valid (the buffers
 * untouched) until fkd_wait returns; every job must be waited for once. */
typedef struct fkd_job fkd_job;
fkd_status fkd_submit_batches(const fkd_tree* tree, fkd_host_batch* batches, int32_t n, fkd_job** job);
fkd_status fkd_wait(fkd_job* job);

/* Device buffers on the tree's first device, launched on `stream` (a
 * cudaStream_t; NULL = legacy default stream).  The kernels are enqueued on
 * `stream`; the call then synchronises that stream once, because the
 * non-finite-query check (batch.cpp:79) must be reported as a status.
 * d_hits must be 8-byte aligned.  per_query (device, may be NULL) receives
 * each query's counters in input order (reference stack-free counting). */
fkd_status fkd_run_batch_device(const fkd_tree* tree, const float* d_queries, int64_t m,
                                int32_t dim, const fkd_batch_options* opt, int32_t* d_counts,
                                fkd_hit* d_hits, fkd_query_stats* stats,
                                fkd_query_stats* d_per_query, void* stream,
                                fkd_timings* timings);

/* One device-resident batch of fkd_run_batches_device. */
typedef struct fkd_device_batch {
    const float* d_queries;      /* m x dim, device                              */
    int64_t m;
    int32_t dim;
    fkd_batch_options opt;
    int32_t* d_counts;           /* [m], device                                  */
    fkd_hit* d_hits;             /* [m * stride], device, 8-byte aligned         */
    fkd_query_stats* stats;      /* host, may be NULL (batch totals)             */
    fkd_query_stats* d_per_query;/* device, may be NULL                          */
    fkd_timings* timings;        /* host, may be NULL                            */
    fkd_status status;           /* out: this batch's status                     */
} fkd_device_batch;

/* Several independent device-resident batches over the same tree in one
 * submission: each runs exactly as fkd_run_batch_device would (own
 * workspace, own result slots, own status), all concurrently on streams
 * forked from `stream`; the most expensive batch gets the highest stream
 * priority so the others fill the SMs its tail passes leave idle.  Joins
 * back into `stream` and synchronises it once.  Returns the first non-OK
 * status (each batch's is in its `status`). */
fkd_status fkd_run_batches_device(const fkd_tree* tree, fkd_device_batch* batches, int32_t n,
                                  void* stream);

/* ---- single-query entry points (traverse.cpp:25-39) ----
 * out_hits holds max(k,1) entries; *out_count receives the number of hits.
 * Validation follows the reference constructors (radius before k). */
fkd_status fkd_fcp(const fkd_tree* tree, const float* query, int32_t dim, float max_radius,
                   fkd_hit* out_hit, int32_t* out_count, fkd_query_stats* stats);
fkd_status fkd_knn(const fkd_tree* tree, const float* query, int32_t dim, int32_t k,
                   float max_radius, fkd_hit* out_hits, int32_t* out_count,
                   fkd_query_stats* stats);

/* ---- device trace (traverse.hpp:56-68) ----
 * Walks m host queries with the literal state machine on the GPU and returns,
 * per query, its hits (stride k, or 1 for fcp), count, QueryStats and the
 * event list the reference's Trace records: node id for "processed", ~node
 * for "bounced" (events[i*cap ...], lens[i] = full length, may exceed cap).
 * A debugging aid: slow by design (no bounce folding, no Morton order). */
fkd_status fkd_trace_batch(const fkd_tree* tree, const float* queries, int32_t m, int32_t dim,
                           int32_t kind, int32_t k, float max_radius, int32_t* counts,
                           fkd_hit* hits, fkd_query_stats* stats, int32_t* events, int64_t cap,
                           int64_t* lens);

/* ---- FKDT / FKDX binary files (io.hpp:10-18, io.cpp:50-99) ----
 * kind 0 = points ("FKDT"), 1 = level-order tree ("FKDX").  Point files may
 * exceed the reference's INT_MAX-floats limit (up to 2^40 points). */
fkd_status fkd_file_info(const char* path, int32_t kind, int64_t* count, int32_t* dim);
/* Streams the payload into device memory d_out (capacity in points) through a
 * pinned double buffer, then checks finiteness on the device. */
fkd_status fkd_read_file_device(const char* path, int32_t kind, float* d_out, int64_t capacity_points,
                                int64_t* count, int32_t* dim, void* stream);
fkd_status fkd_write_file(const char* path, int32_t kind, const float* data, int64_t count, int32_t dim);
/* io::read_tree + KdTree::from_level_order straight onto the device(s). */
fkd_status fkd_tree_load(const char* path, const int32_t* devices, int32_t ndev, fkd_tree** out);

/* ---- host utilities around the path ---- */

/* flatkd::build_tree (tree.cpp:80-89), round-robin policy: the unique
 * left-balanced level-order array.  Multi-threaded host build; output is
 * byte-identical to the reference's. */
fkd_status fkd_build_tree(const float* points, int64_t n, int32_t dim, float* level_order_out);

/* The same build on the GPU: device points in, device
 * level-order array out, byte-identical to flatkd::build_tree.  Rejects
 * non-finite points ("build: non-finite coordinate in point i"). */
fkd_status fkd_build_tree_device(const float* d_points, int64_t n, int32_t dim,
                                 float* d_level_order_out, void* stream);

/* Host points -> GPU build on the first device -> tree store on every listed
 * device (build_tree + KdTree::from_level_order in one call, no host
 * round trip of the level-order array).  level_order_out (host, may be NULL)
 * receives the array. */
fkd_status fkd_tree_build(const float* points, int64_t n, int32_t dim, const int32_t* devices,
                          int32_t ndev, float* level_order_out, fkd_tree** out);

/* BatchResult::result_hash (batch.cpp:30-48). */
uint64_t fkd_result_hash(const int32_t* counts, const fkd_hit* hits, int64_t m, int32_t stride);

/* flatkd::random_points(derive_stream_seed(master, stream), count, dim)
 * (rng.hpp:26-53): mt19937_64, top 24 bits scaled by 2^-24. */
fkd_status fkd_random_points(uint64_t master_seed, uint64_t stream, int64_t count, int32_t dim,
                             float* out);

/* Gaussian-blob generator for the clustered workload (
 * no reference counterpart): `blobs` centres from stream 3, sigma per axis. */
fkd_status fkd_clustered_points(uint64_t master_seed, uint64_t stream, int64_t count, int32_t dim,
                                int32_t blobs, float sigma, float* out);

/* Pinned host memory for zero-staging transfers. */
void* fkd_host_alloc(size_t bytes);
void fkd_host_free(void* p);

/* Profiling builds (-DFKD_BLOCK_TRACE=1) only: every walk / round / CTA-pass
 * block appends {tag, SM id, start ns, end ns} (%globaltimer; tag = list
 * length << 8 | phase) to d_records (device, cap records of 24 bytes; the
 * device counter d_counter must start at 0).  NULL disables.  Other builds
 * return FKD_INVALID_ARGUMENT for a non-NULL buffer. */
fkd_status fkd_debug_block_trace(void* d_records, void* d_counter, int64_t cap);

/* Thread-local message for the last non-OK status. */
const char* fkd_last_error(void);

/* Library version string and the sm arch it was built for. */
const char* fkd_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FKD_B200_H */
