/*
 * fkd_oracle.c — CPU restatement of the reference (flatkd) query path.
 *
 * TEST INFRASTRUCTURE ONLY (see fkd_oracle.h).  Written from the reference's
 * behaviour, not copied from it; each function cites the reference lines it
 * restates (paths relative to /root/reference/proj).
 *
 * Must be compiled with -ffp-contract=off and without -ffast-math: the
 * reference's squared_distance (include/flatkd/point.hpp:68-75) is a plain
 * left-to-right float accumulation and any FMA contraction changes dist2
 * bits.
 */
#include "fkd_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* fko_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ RNG */

/* include/flatkd/rng.hpp:11-17 */
uint64_t fko_splitmix64(uint64_t* state) {
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* include/flatkd/rng.hpp:26-29 */
uint64_t fko_derive_stream_seed(uint64_t master, uint64_t stream) {
    uint64_t x = master ^ (stream * 0x9E3779B97F4A7C15ull);
    return fko_splitmix64(&x);
}

/* std::mt19937_64 (the generator behind rng.hpp:34-44 and instancegen.hpp:16-27),
 * restated from its published definition: w=64, n=312, m=156, r=31,
 * a=0xB5026F5AA96619E9, f=6364136223846793005, tempering (u,d,s,b,t,c,l) =
 * (29,0x5555555555555555,17,0x71D67FFFEDA60000,37,0xFFF7EEE000000000,43). */
void fko_mt_seed(fko_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t fko_mt_next(fko_mt64* g) {
    const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* rng.hpp:38 and instancegen.hpp:22: top 24 bits, scaled by 2^-24 */
float fko_mt_float01(fko_mt64* g) { return (float)(fko_mt_next(g) >> 40) * 0x1p-24f; }

/* testing/instancegen.cpp:7-10 */
int fko_mt_next_int(fko_mt64* g, int lo, int hi) {
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    return lo + (int)(fko_mt_next(g) % span);
}

/* instancegen.hpp:23 (float promoted to double for the compare) */
int fko_mt_chance(fko_mt64* g, double p) { return (double)fko_mt_float01(g) < p; }

int fko_rng_state_size(void) { return (int)sizeof(fko_mt64); }

/* rng.hpp:46-53 */
void fko_random_points(uint64_t seed, int64_t count, int dim, float* out) {
    fko_mt64 g;
    fko_mt_seed(&g, seed);
    const int64_t total = count * dim;
    for (int64_t i = 0; i < total; ++i) out[i] = fko_mt_float01(&g);
}

/* testing/instancegen.cpp:12-30.  Note the dup draw happens for every i > 0,
 * even when dup_fraction is 0. */
void fko_random_point_set(fko_mt64* g, int n, int dim, int grid, double dup_fraction, float* out) {
    for (int i = 0; i < n; ++i) {
        float* p = out + (size_t)i * dim;
        if (i > 0 && fko_mt_chance(g, dup_fraction)) {
            const int src = fko_mt_next_int(g, 0, i - 1);
            memcpy(p, out + (size_t)src * dim, sizeof(float) * (size_t)dim);
        } else {
            for (int c = 0; c < dim; ++c) {
                float v = fko_mt_float01(g);
                if (grid > 0) v = roundf(v * (float)grid) / (float)grid;
                p[c] = v;
            }
        }
    }
}

/* testing/instancegen.cpp:32-48 */
void fko_random_query(fko_mt64* g, int dim, const float* points, int n, float* out) {
    for (int c = 0; c < dim; ++c) out[c] = fko_mt_float01(g) * 1.5f - 0.25f;
    if (n > 0) {
        if (fko_mt_chance(g, 0.10)) {
            const int src = fko_mt_next_int(g, 0, n - 1);
            memcpy(out, points + (size_t)src * dim, sizeof(float) * (size_t)dim);
        } else if (fko_mt_chance(g, 0.15)) {
            const int src = fko_mt_next_int(g, 0, n - 1);
            const int d = fko_mt_next_int(g, 0, dim - 1);
            out[d] = points[(size_t)src * dim + d];
        }
    }
}

/* ----------------------------------------------------- tree layout/build */

/* include/flatkd/tree.hpp:20-22: bit_width(n+1) - 1 */
int fko_depth_of(int n) {
    unsigned v = (unsigned)n + 1u;
    int d = -1;
    while (v) {
        ++d;
        v >>= 1;
    }
    return d;
}

/* src/tree.cpp:10-18 */
int fko_left_subtree_size(int n) {
    if (n <= 1) return 0;
    int h = fko_depth_of(n - 1); /* floor(log2 n) */
    const int full = (1 << h) - 1;
    const int last = n - full;
    const int half = 1 << (h - 1);
    return (half - 1) + (last < half ? last : half);
}

static int all_finite(const float* p, int dim) {
    for (int i = 0; i < dim; ++i)
        if (!isfinite(p[i])) return 0;
    return 1;
}

/* RankOrder (src/tree.cpp:40-53): split coordinate, then the whole tuple,
 * then the original index.  Strict total order -> unique build. */
typedef struct {
    const float* pts;
    int dim;
    int d;
} rank_ctx;

static int rank_less(const rank_ctx* c, int a, int b) {
    const float* pa = c->pts + (size_t)a * c->dim;
    const float* pb = c->pts + (size_t)b * c->dim;
    if (pa[c->d] != pb[c->d]) return pa[c->d] < pb[c->d];
    for (int i = 0; i < c->dim; ++i)
        if (pa[i] != pb[i]) return pa[i] < pb[i];
    return a < b;
}

static void swap_int(int* a, int* b) {
    int t = *a;
    *a = *b;
    *b = t;
}

/* Hoare-style quickselect: afterwards ord[kth] is the rank-kth element and
 * the prefix holds exactly the smaller ones (as a set). */
static void select_kth(const rank_ctx* c, int* ord, int n, int kth) {
    int lo = 0, hi = n - 1;
    while (hi > lo) {
        const int mid = lo + (hi - lo) / 2;
        /* median of three into ord[hi] as pivot */
        if (rank_less(c, ord[mid], ord[lo])) swap_int(&ord[mid], &ord[lo]);
        if (rank_less(c, ord[hi], ord[lo])) swap_int(&ord[hi], &ord[lo]);
        if (rank_less(c, ord[mid], ord[hi])) swap_int(&ord[mid], &ord[hi]);
        const int pivot = ord[hi];
        int store = lo;
        for (int i = lo; i < hi; ++i)
            if (rank_less(c, ord[i], pivot)) swap_int(&ord[i], &ord[store++]);
        swap_int(&ord[store], &ord[hi]);
        if (store == kth) return;
        if (store < kth)
            lo = store + 1;
        else
            hi = store - 1;
    }
}

/* src/tree.cpp:55-67 */
static void build_range(const float* pts, int dim, int* ord, int n, int slot, float* out) {
    if (n == 0) return;
    rank_ctx c = {pts, dim, fko_depth_of(slot) % dim};
    const int rank = fko_left_subtree_size(n);
    select_kth(&c, ord, n, rank);
    memcpy(out + (size_t)slot * dim, pts + (size_t)ord[rank] * dim, sizeof(float) * (size_t)dim);
    build_range(pts, dim, ord, rank, 2 * slot + 1, out);
    build_range(pts, dim, ord + rank + 1, n - rank - 1, 2 * slot + 2, out);
}

/* src/tree.cpp:80-89 */
int fko_build_tree(const float* points, int n, int dim, float* level_order_out) {
    for (int i = 0; i < n; ++i)
        if (!all_finite(points + (size_t)i * dim, dim)) {
            snprintf(g_err, sizeof g_err, "build: non-finite coordinate in point %d", i);
            return FKO_DATA_ERROR;
        }
    if (n == 0) return FKO_OK;
    int* ord = (int*)malloc(sizeof(int) * (size_t)(unsigned)n);
    for (int i = 0; i < n; ++i) ord[i] = i;
    build_range(points, dim, ord, n, 0, level_order_out);
    free(ord);
    return FKO_OK;
}

/* src/tree.cpp:128-136: every descendant on the correct side of each plane */
int fko_verify_tree(const float* nodes, int n, int dim) {
    int* stack = (int*)malloc(sizeof(int) * ((size_t)n + 1));
    for (int node = 0; node < n; ++node) {
        const int d = fko_depth_of(node) % dim;
        const float split = nodes[(size_t)node * dim + d];
        for (int side = 0; side < 2; ++side) {
            int top = 0;
            const int child = 2 * node + 1 + side;
            if (child < n) stack[top++] = child;
            while (top) {
                const int i = stack[--top];
                const float c = nodes[(size_t)i * dim + d];
                if (side == 0 ? !(c <= split) : !(c >= split)) {
                    free(stack);
                    return 0;
                }
                if (2 * i + 1 < n) stack[top++] = 2 * i + 1;
                if (2 * i + 2 < n) stack[top++] = 2 * i + 2;
            }
        }
    }
    free(stack);
    return 1;
}

/* ------------------------------------------------------------ candidates */

/* include/flatkd/point.hpp:68-75: left to right from 0.0f, no FMA */
static float squared_distance(const float* a, const float* b, int dim) {
    float acc = 0.0f;
    for (int i = 0; i < dim; ++i) {
        const float d = a[i] - b[i];
        const float sq = d * d;
        acc = acc + sq;
    }
    return acc;
}

/* include/flatkd/traverse.hpp:80-83 */
static int hit_order(fko_hit a, fko_hit b) {
    if (a.dist2 != b.dist2) return a.dist2 < b.dist2;
    return a.node < b.node;
}

/* One sink for both query kinds.  fcp (traverse.hpp:86-108) is the k = 1
 * case with its own admission rule; knn (traverse.hpp:113-175) keeps the k
 * best under hit_order.  Held here as an ascending array rather than the
 * reference's max-heap: the kept set and radius2() are identical. */
typedef struct {
    int kind; /* 0 fcp, 1 knn */
    int k;
    float cap2;
    int count;
    fko_hit* list; /* ascending, count entries */
} sink;

static void sink_consider(sink* s, float d2, int32_t node) {
    if (d2 > s->cap2) return; /* traverse.hpp:92, :122 (inclusive cap) */
    if (s->kind == 0) {
        /* traverse.hpp:93-94 */
        fko_hit* b = &s->list[0];
        if (s->count == 0 || d2 < b->dist2 || (d2 == b->dist2 && node < b->node)) {
            b->node = node;
            b->dist2 = d2;
            s->count = 1;
        }
        return;
    }
    fko_hit h = {node, d2};
    if (s->count == s->k) {
        /* traverse.hpp:128-129: must beat the current worst */
        if (!hit_order(h, s->list[s->k - 1])) return;
        s->count--;
    }
    int pos = s->count;
    while (pos > 0 && hit_order(h, s->list[pos - 1])) {
        s->list[pos] = s->list[pos - 1];
        --pos;
    }
    s->list[pos] = h;
    s->count++;
}

/* traverse.hpp:97 and :135-137 */
static float sink_radius2(const sink* s) {
    if (s->kind == 0) return s->count == 0 ? s->cap2 : s->list[0].dist2;
    return s->count < s->k ? s->cap2 : s->list[s->k - 1].dist2;
}

/* ------------------------------------------------------------- traversal */

typedef struct {
    int32_t* buf;
    int64_t cap;
    int64_t len;
} tracebuf;

static void trace_push(tracebuf* t, int32_t ev) {
    if (!t) return;
    if (t->len < t->cap) t->buf[t->len] = ev;
    t->len++;
}

/* include/flatkd/traverse.hpp:198-248: one transition of the curr/prev
 * state machine.  Returns 0 once the walk has ended. */
static int traverse_step(const float* nodes, int n, int dim, const float* q, int32_t* curr,
                         int32_t* prev, float* radius2, sink* s, fko_stats* st, tracebuf* tr) {
    if (*curr < 0 || n == 0) return 0;
    if (st) st->steps++;
    const int32_t parent = (*curr + 1) / 2 - 1;
    if (*curr >= n) { /* empty child slot: bounce (206-212) */
        trace_push(tr, ~*curr);
        *prev = *curr;
        *curr = parent;
        return 1;
    }
    const int from_parent = *prev < *curr; /* 216 */
    const float* node = nodes + (size_t)*curr * dim;
    if (from_parent) { /* 217-222 */
        if (st) st->nodes_processed++;
        trace_push(tr, *curr);
        sink_consider(s, squared_distance(q, node, dim), *curr);
        *radius2 = sink_radius2(s);
    }
    if (st) st->nodes_visited++;
    const int d = fko_depth_of(*curr) % dim;                  /* 225 */
    const float signed_dist = q[d] - node[d];                 /* 226 */
    const int32_t close_side = signed_dist > 0.0f;            /* 227 */
    const int32_t close_child = 2 * *curr + 1 + close_side;   /* 228 */
    const int32_t far_child = 2 * *curr + 2 - close_side;     /* 229 */
    const float sq = signed_dist * signed_dist;
    const int far_in_range = sq <= *radius2;                  /* 230 */
    int32_t next;
    if (from_parent)
        next = close_child;
    else if (*prev == close_child)
        next = far_in_range ? far_child : parent;
    else
        next = parent;
    if (next == -1) { /* 240-244 */
        *curr = -1;
        return 0;
    }
    *prev = *curr;
    *curr = next;
    return 1;
}

/* traverse.hpp:263-283 */
static void recursive_visit(const float* nodes, int n, int dim, const float* q, sink* s,
                            fko_stats* st, tracebuf* tr, int node) {
    if (st) st->steps++;
    if (node >= n) {
        trace_push(tr, ~node);
        return;
    }
    if (st) {
        st->nodes_visited++;
        st->nodes_processed++;
    }
    trace_push(tr, node);
    const float* p = nodes + (size_t)node * dim;
    sink_consider(s, squared_distance(q, p, dim), node);
    const int d = fko_depth_of(node) % dim;
    const float sd = q[d] - p[d];
    const int close_side = sd > 0.0f;
    recursive_visit(nodes, n, dim, q, s, st, tr, 2 * node + 1 + close_side);
    const float sq = sd * sd;
    if (sq <= sink_radius2(s)) recursive_visit(nodes, n, dim, q, s, st, tr, 2 * node + 2 - close_side);
}

static void run_walk(const float* nodes, int n, int dim, const float* q, sink* s, int recursive,
                     fko_stats* st, tracebuf* tr) {
    if (recursive) {
        if (n == 0) return; /* traverse.hpp:291 */
        recursive_visit(nodes, n, dim, q, s, st, tr, 0);
        return;
    }
    /* traverse.hpp:250-258 */
    int32_t curr = 0, prev = -1;
    float radius2 = sink_radius2(s);
    while (traverse_step(nodes, n, dim, q, &curr, &prev, &radius2, s, st, tr)) {
    }
}

static float radius_cap(float max_radius, int* ok) {
    /* include/flatkd/point.hpp:78-82 */
    *ok = !(isnan(max_radius) || max_radius < 0.0f);
    return max_radius * max_radius;
}

/* traverse.cpp:25-39 with the constructor checks of traverse.hpp:88-89,
 * 115-117 (radius before k: member initialiser order) and validate_query
 * (traverse.hpp:186-192). */
int fko_query(const float* nodes, int n, int dim, const float* q, int kind, int k,
              float max_radius, int recursive, fko_hit* out_hits, int* out_count,
              fko_stats* stats, int32_t* trace, int64_t trace_cap, int64_t* trace_len) {
    int ok;
    const float cap2 = radius_cap(max_radius, &ok);
    if (!ok) return fail(FKO_DATA_ERROR, "max radius must be >= 0 or inf");
    if (kind == 1 && k < 1) return fail(FKO_INVALID_ARGUMENT, "knn: k must be >= 1");
    if (n > 0 && !all_finite(q, dim)) return fail(FKO_DATA_ERROR, "query has a non-finite coordinate");
    const int kk = kind == 1 ? k : 1;
    sink s = {kind, kk, cap2, 0, out_hits};
    for (int j = 0; j < kk; ++j) {
        out_hits[j].node = -1;
        out_hits[j].dist2 = INFINITY;
    }
    tracebuf tb = {trace, trace_cap, 0};
    if (stats) memset(stats, 0, sizeof *stats);
    run_walk(nodes, n, dim, q, &s, recursive, stats, trace ? &tb : NULL);
    *out_count = s.count;
    if (trace_len) *trace_len = tb.len;
    return FKO_OK;
}

/* src/batch.cpp:71-134 */
int fko_run_batch(const float* nodes, int n, int tree_dim, const float* queries, int m,
                  int query_dim, int kind, int k, float max_radius, int recursive,
                  int threads, int32_t* counts, fko_hit* hits, fko_stats* stats_total,
                  fko_stats* per_query) {
    if (kind == 1 && k < 1) return fail(FKO_INVALID_ARGUMENT, "knn: k must be >= 1"); /* 72-73 */
    int ok;
    const float cap2 = radius_cap(max_radius, &ok); /* 74 */
    if (!ok) return fail(FKO_DATA_ERROR, "max radius must be >= 0 or inf");
    if (n > 0 && m > 0) { /* 75-80 */
        if (query_dim != tree_dim) {
            snprintf(g_err, sizeof g_err, "query dimension %d does not match tree dimension %d",
                     query_dim, tree_dim);
            return FKO_DATA_ERROR;
        }
        for (int i = 0; i < m; ++i)
            if (!all_finite(queries + (size_t)i * query_dim, query_dim)) {
                snprintf(g_err, sizeof g_err, "queries: non-finite coordinate in point %d", i);
                return FKO_DATA_ERROR;
            }
    }
    const int stride = kind == 1 ? k : 1;
    long long tot_steps = 0, tot_vis = 0, tot_proc = 0;
#ifdef _OPENMP
    const int nthr = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthr) reduction(+ : tot_steps, tot_vis, tot_proc)
#endif
    for (int i = 0; i < m; ++i) {
        fko_hit* slot = hits + (size_t)i * stride;
        for (int j = 0; j < stride; ++j) {
            slot[j].node = -1;
            slot[j].dist2 = INFINITY;
        }
        sink s = {kind, stride, cap2, 0, slot};
        fko_stats st = {0, 0, 0};
        run_walk(nodes, n, tree_dim, queries + (size_t)i * query_dim, &s, recursive, &st, NULL);
        counts[i] = s.count;
        if (per_query) per_query[i] = st;
        tot_steps += st.steps;
        tot_vis += st.nodes_visited;
        tot_proc += st.nodes_processed;
    }
    (void)threads;
    if (stats_total) {
        stats_total->steps = tot_steps;
        stats_total->nodes_visited = tot_vis;
        stats_total->nodes_processed = tot_proc;
    }
    return FKO_OK;
}

/* testing/oracle.cpp:15-43: exhaustive scan, same admission and tie rule */
int fko_brute_batch(const float* points, int n, int dim, const float* queries, int m, int kind,
                    int k, float max_radius, int32_t* counts, fko_hit* hits) {
    if (kind == 1 && k < 1) return fail(FKO_INVALID_ARGUMENT, "oracle knn: k must be >= 1");
    int ok;
    const float cap2 = radius_cap(max_radius, &ok);
    if (!ok) return fail(FKO_DATA_ERROR, "max radius must be >= 0 or inf");
    const int stride = kind == 1 ? k : 1;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (int i = 0; i < m; ++i) {
        fko_hit* slot = hits + (size_t)i * stride;
        for (int j = 0; j < stride; ++j) {
            slot[j].node = -1;
            slot[j].dist2 = INFINITY;
        }
        sink s = {kind, stride, cap2, 0, slot};
        const float* q = queries + (size_t)i * dim;
        for (int p = 0; p < n; ++p) sink_consider(&s, squared_distance(q, points + (size_t)p * dim, dim), p);
        counts[i] = s.count;
    }
    return FKO_OK;
}

/* src/batch.cpp:30-48: FNV-1a over counts and the valid hits, bytewise LE */
uint64_t fko_result_hash(const int32_t* counts, const fko_hit* hits, int64_t m, int stride) {
    uint64_t h = 0xcbf29ce484222325ull;
#define FKO_MIX(v)                                   \
    do {                                             \
        uint32_t vv = (v);                           \
        for (int b = 0; b < 4; ++b) {                \
            h ^= (vv >> (8 * b)) & 0xffu;            \
            h *= 0x100000001b3ull;                   \
        }                                            \
    } while (0)
    for (int64_t q = 0; q < m; ++q) {
        const int32_t c = counts[q];
        FKO_MIX((uint32_t)c);
        for (int32_t j = 0; j < c; ++j) {
            const fko_hit* hit = &hits[q * stride + j];
            uint32_t bits;
            memcpy(&bits, &hit->dist2, 4);
            FKO_MIX((uint32_t)hit->node);
            FKO_MIX(bits);
        }
    }
#undef FKO_MIX
    return h;
}
