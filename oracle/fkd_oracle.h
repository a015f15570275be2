/*
 * fkd_oracle.h — CPU restatement of the reference (flatkd) query path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it.  The product path (paper_2210_12859_b200/) never links
 * or calls anything here and fails loudly when its CUDA library is missing.
 *
 * Every function restates one reference function; the file:line it follows
 * (relative to the reference tree, proj/...) is cited beside it.  The
 * restatement is pinned against (a) the reference's own known answers
 * (Fig. 1 build, SPEC examples, selfcheck suites) and (b) the reference
 * itself compiled here into oracle/_ref/ (tests/test_oracle.py).
 *
 * Build flags matter: -ffp-contract=off (no FMA contraction), no -ffast-math.
 */
#ifndef FKD_ORACLE_H
#define FKD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- layout-identical result records (traverse.hpp:46-54, 70-76) ---- */
typedef struct fko_hit {
    int32_t node;  /* -1 = empty slot */
    float dist2;   /* +inf for empty slot */
} fko_hit;

typedef struct fko_stats {
    int64_t steps;
    int64_t nodes_visited;
    int64_t nodes_processed;
} fko_stats;

/* status codes, mirroring the reference's exception types */
enum {
    FKO_OK = 0,
    FKO_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    FKO_DATA_ERROR = 2        /* flatkd::DataError */
};

/* ---- RNG (rng.hpp, instancegen.hpp) ---- */
typedef struct fko_mt64 {
    uint64_t mt[312];
    int idx;
} fko_mt64;

uint64_t fko_splitmix64(uint64_t* state);                         /* rng.hpp:11-17 */
uint64_t fko_derive_stream_seed(uint64_t master, uint64_t stream); /* rng.hpp:26-29 */
void fko_mt_seed(fko_mt64* g, uint64_t seed);                     /* std::mt19937_64 */
uint64_t fko_mt_next(fko_mt64* g);
float fko_mt_float01(fko_mt64* g);                                 /* rng.hpp:38, instancegen.hpp:22 */
int fko_mt_next_int(fko_mt64* g, int lo, int hi);                  /* instancegen.cpp:7-10 */
int fko_mt_chance(fko_mt64* g, double p);                          /* instancegen.hpp:23 */
int fko_rng_state_size(void);

/* rng.hpp:46-53 */
void fko_random_points(uint64_t seed, int64_t count, int dim, float* out);
/* instancegen.cpp:12-30 */
void fko_random_point_set(fko_mt64* g, int n, int dim, int grid, double dup_fraction, float* out);
/* instancegen.cpp:32-48 */
void fko_random_query(fko_mt64* g, int dim, const float* points, int n, float* out);

/* ---- tree layout + builder (tree.hpp:16-29, tree.cpp:10-89) ---- */
int fko_left_subtree_size(int n);
int fko_depth_of(int n);
/* Returns 0, or FKO_DATA_ERROR on a non-finite input coordinate. */
int fko_build_tree(const float* points, int n, int dim, float* level_order_out);
/* 1 when every subtree respects its split plane (tree.cpp:128-136). */
int fko_verify_tree(const float* nodes, int n, int dim);

/* ---- single queries (traverse.hpp:198-258, traverse.cpp:25-39) ----
 * kind 0 = fcp, 1 = knn.  out_hits must hold max(k,1) entries.  trace (may
 * be NULL) receives the event list: node for "processed", ~node for
 * "bounced"; *trace_len gets the event count (capped at trace_cap). */
int fko_query(const float* nodes, int n, int dim, const float* q, int kind, int k,
              float max_radius, int recursive, fko_hit* out_hits, int* out_count,
              fko_stats* stats, int32_t* trace, int64_t trace_cap, int64_t* trace_len);

/* ---- batch runner (batch.cpp:71-134) ----
 * counts[m], hits[m*stride] (stride = knn ? k : 1).  stats_total and
 * per_query may be NULL.  threads <= 0 means all OpenMP threads. */
int fko_run_batch(const float* nodes, int n, int tree_dim, const float* queries, int m,
                  int query_dim, int kind, int k, float max_radius, int recursive,
                  int threads, int32_t* counts, fko_hit* hits, fko_stats* stats_total,
                  fko_stats* per_query);

/* ---- brute force ground truth (testing/oracle.cpp:15-43) ---- */
int fko_brute_batch(const float* points, int n, int dim, const float* queries, int m, int kind,
                    int k, float max_radius, int32_t* counts, fko_hit* hits);

/* ---- result hash (batch.cpp:30-48) ---- */
uint64_t fko_result_hash(const int32_t* counts, const fko_hit* hits, int64_t m, int stride);

/* last error message (thread-local) */
const char* fko_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
