// overflow.cuh — the tail pass: one CTA per query that exceeded the walk
// kernel's step budget.
//
// Why: per-query walk lengths are heavy-tailed.  On the clustered C3
// workload one kNN8 query takes 286k steps (22 ms on its own) while the batch
// average is 378, so a one-thread-per-query grid is as slow as its slowest
// thread.  The walk kernel therefore stops a query after `budget` loop trips,
// leaves its partial candidate list in its own output slot and appends its id
// to an overflow list; this kernel then finishes those queries with a whole
// CTA each:
//
//   1. bound  — r2 starts at the kth distance of the partial list (or the
//      cap): any k admissible points bound the final kth distance from above;
//   2. BFS    — the reachable top of the tree is expanded level by level in
//      shared memory (process the node, push the close child, push the far
//      child iff sd*sd <= r2) until the frontier holds >= 4 x blockDim roots;
//   3. DFS    — threads pull frontier roots from a shared counter and run the
//      same stack-free walk (traverse_step rules) confined to that subtree,
//      each with its own register list, all pruning against min(own kth,
//      shared r2) where the shared r2 is the smallest kth distance any
//      thread has seen (atomicMin on the float bits, valid for d2 >= 0);
//   4. select — the final set lies within the shared bound (any thread's kth
//      distance bounds the final kth from above), so the list entries <= it
//      are compacted into shared memory and, when at most kRankMax survive,
//      each computes its rank among them (distinct keys) and lands in its
//      output slot directly: two barriers instead of 2k.  Otherwise, k rounds
//      of a block-wide min over the threads' list heads.
//
// Exactness: the answer is the k smallest admissible keys under hit_order;
// every pruning bound used is >= the final kth distance and comparisons stay
// inclusive, so no member of the final set is ever skipped, and distances
// come from the same sq_dist (same bits).  Only the order in which nodes are
// visited differs from the reference's walk, which is why STATS mode never
// uses a budget (per-query counters stay exactly the reference's).
#pragma once

#include "walk.cuh"

namespace fkd {

constexpr int kOvfFrontierMax = 4096;
constexpr int kRankMax = 1024;  // rank selection's candidate cap (C^2 / THREADS compares per thread)

template <int KB>
__device__ __forceinline__ uint64_t list_head(const uint64_t (&L)[KB], int dummies) {
    uint64_t h = kEmptyKey;
#pragma unroll
    for (int j = KB - 1; j >= 0; --j) h = (j == dummies) ? L[j] : h;
    return h;
}

template <int KB>
__device__ __forceinline__ void list_pop(uint64_t (&L)[KB], int dummies) {
#pragma unroll
    for (int j = 0; j < KB - 1; ++j)
        if (j >= dummies) L[j] = L[j + 1];
    L[KB - 1] = kEmptyKey;
}

template <int D, int S, int KB, int THREADS>
__global__ void __launch_bounds__(THREADS) overflow_kernel(const WalkArgs a) {
    __shared__ int32_t frontier[2][kOvfFrontierMax];
    __shared__ int fcount[2];
    __shared__ unsigned r2_bits;
    __shared__ unsigned long long slot;
    __shared__ int work_next;
    __shared__ unsigned long long red[THREADS / 32];
    __shared__ unsigned long long winner;
    __shared__ int ccount;

    const int tid = threadIdx.x;
    const int32_t n = a.n;
    const int k = a.k;
    const int dummies = KB - k;
    const float cap2 = a.cap2;

    // many over-budget queries: the resume pass continued them, and this
    // pass takes the ones that outlived it
    const bool resumed = a.resume_min > 0 && *a.ovf_count >= (unsigned long long)a.resume_min;
    const uint32_t* ids = resumed ? a.wave_out : a.ovf_ids;
    const unsigned long long count = resumed ? *a.wave_n_out : *a.ovf_count;
    BlockTrace bt(a);
    bool worked = false;
    while (true) {
        if (tid == 0) slot = atomicAdd(a.ovf_next, 1ull);
        __syncthreads();
        const unsigned long long s = slot;
        if (s >= count) {
            if (worked) bt.end(a, 1);
            return;
        }
        worked = true;
        const int64_t qi = ids[s];

        float q[D];
#pragma unroll
        for (int j = 0; j < D; ++j) q[j] = __ldg(a.queries + qi * D + j);

        uint64_t L[KB];
#pragma unroll
        for (int j = 0; j < KB; ++j) L[j] = j < dummies ? 0ull : kEmptyKey;

        if (tid == 0) {
            // bound from the partial list the walk kernel left in the slot
            float b = cap2;
            // (a full partial list: its last slot holds a hit; the walk does not
            // write the count of a parked query)
            const fkd_hit last = a.hits[qi * k + (k - 1)];
            if (last.node >= 0) b = fminf(b, last.dist2);
            r2_bits = __float_as_uint(b);
            frontier[0][0] = 0;
            fcount[0] = 1;
            fcount[1] = 0;
            work_next = 0;
        }
        __syncthreads();

        auto consider = [&](int32_t node, const float (&p)[D]) {
            const float d2 = sq_dist<D, (D <= 4 && KB <= 8)>(q, p);
            const uint64_t key = make_key(d2, node);
            if (d2 <= cap2 && key < L[KB - 1]) {
                list_insert(L, key);
                const uint64_t kth = L[KB - 1];
                if (kth != kEmptyKey) atomicMin(&r2_bits, __float_as_uint(key_dist(kth)));
            }
        };
        auto bound = [&]() {
            return fminf(__uint_as_float(r2_bits), fminf(cap2, key_dist(L[KB - 1])));
        };

        // ---- 2. BFS over the reachable top of the tree
        int cur = 0, depth = 0;
        while (true) {
            const int fc = fcount[cur];
            if (fc == 0 || fc >= 4 * THREADS || 2 * fc > kOvfFrontierMax) break;
            const int dd = depth % D;
            for (int i = tid; i < fc; i += THREADS) {
                const int32_t node = frontier[cur][i];
                float p[D];
                load_point<D, S>(a.nodes, node, p);
                consider(node, p);
                const float sd = __fsub_rn(pick(q, dd), pick(p, dd));
                const int cs = sd > 0.0f;
                const int32_t close = 2 * node + 1 + cs, far = 2 * node + 2 - cs;
                if (close < n) frontier[cur ^ 1][atomicAdd(&fcount[cur ^ 1], 1)] = close;
                if (far < n && __fmul_rn(sd, sd) <= bound())
                    frontier[cur ^ 1][atomicAdd(&fcount[cur ^ 1], 1)] = far;
            }
            __syncthreads();
            if (tid == 0) fcount[cur] = 0;
            cur ^= 1;
            ++depth;
            __syncthreads();
        }

        // ---- 3. stack-free walks confined to the frontier subtrees
        const int roots = fcount[cur];
        while (true) {
            int ri = 0;
            ri = atomicAdd(&work_next, 1);
            if (ri >= roots) break;
            const int32_t root = frontier[cur][ri];
            const int32_t stop = ((root + 1) >> 1) - 1;  // the root's parent
            int32_t curr = root, prev = stop;
            int d = depth % D;
            while (true) {
                const bool from_parent = prev < curr;
                float p[D];
                load_point<D, S>(a.nodes, curr, p);
                if (from_parent) consider(curr, p);
                const float r2 = bound();
                const float sd = __fsub_rn(pick(q, d), pick(p, d));
                const int cs = sd > 0.0f;
                const bool fir = __fmul_rn(sd, sd) <= r2;
                const int32_t parent = ((curr + 1) >> 1) - 1;
                const int32_t close = 2 * curr + 1 + cs, far = 2 * curr + 2 - cs;
                int32_t next = from_parent ? close : ((prev == close && fir) ? far : parent);
                if (next >= n) {
                    next = (next == close && fir) ? far : parent;
                    if (next >= n) next = parent;
                }
                if (next == stop) break;
                d = next == parent ? dim_down<D>(d) : dim_up<D>(d);
                prev = curr;
                curr = next;
            }
        }
        __syncthreads();

        // ---- 4a. rank selection among the entries within the final bound
        if (tid == 0) ccount = 0;
        __syncthreads();
        // frontier[] is free now; it holds kRankMax 64-bit candidates
        uint64_t* cand = reinterpret_cast<uint64_t*>(&frontier[0][0]);
        static_assert(sizeof(frontier) >= kRankMax * sizeof(uint64_t), "candidate buffer");
        const float fb = __uint_as_float(r2_bits);
#pragma unroll
        for (int j = 0; j < KB; ++j) {
            if (j >= dummies && L[j] != kEmptyKey && key_dist(L[j]) <= fb) {
                const int pos = atomicAdd(&ccount, 1);
                if (pos < kRankMax) cand[pos] = L[j];
            }
        }
        __syncthreads();
        const int C = ccount;
        if (C <= kRankMax) {
            for (int i = tid; i < C; i += THREADS) {
                const uint64_t x = cand[i];
                int rank = 0;
                for (int j = 0; j < C; ++j) rank += key_lt(cand[j], x);
                if (rank < k)
                    reinterpret_cast<int2*>(a.hits + qi * k)[rank] =
                        make_int2(int32_t(uint32_t(x)), int32_t(uint32_t(x >> 32) - kKeyOfs));
            }
            for (int j = C + tid; j < k; j += THREADS)  // fewer than k admissible: Hit{-1, +inf}
                reinterpret_cast<int2*>(a.hits + qi * k)[j] = make_int2(-1, 0x7f800000);
            if (tid == 0) fcount[0] = C < k ? C : k;
            __syncthreads();
        } else {
            // ---- 4b. block-wide k-way merge of the sorted lists
            for (int j = 0; j < k; ++j) {
                uint64_t h = list_head(L, dummies);
                uint64_t m = h;
                for (int off = 16; off > 0; off >>= 1) {
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, m, off);
                    m = o < m ? o : m;
                }
                if ((tid & 31) == 0) red[tid >> 5] = m;
                __syncthreads();
                if (tid < 32) {
                    uint64_t v = tid < THREADS / 32 ? red[tid] : kEmptyKey;
                    for (int off = 16; off > 0; off >>= 1) {
                        const uint64_t o = __shfl_xor_sync(0xffffffffu, v, off);
                        v = o < v ? o : v;
                    }
                    if (tid == 0) winner = v;
                }
                __syncthreads();
                const uint64_t w = winner;
                if (h == w && w != kEmptyKey) list_pop(L, dummies);
                if (tid == 0) {
                    reinterpret_cast<int2*>(a.hits + qi * k)[j] =
                        make_int2(int32_t(uint32_t(w)), int32_t(uint32_t(w >> 32) - kKeyOfs));
                    if (j == 0) fcount[0] = 0;
                    if (w != kEmptyKey) ++fcount[0];  // reuse as the hit counter
                }
                __syncthreads();
            }
        }
        if (tid == 0) a.counts[qi] = fcount[0];
        __syncthreads();
    }
}

}  // namespace fkd
