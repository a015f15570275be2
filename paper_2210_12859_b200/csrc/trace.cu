// trace.cu — device trace of single walks.
//
// The reference threads an optional Trace (processed / bounced events) and
// QueryStats through traverse_step (traverse.hpp:56-68, 198-248).  This
// kernel walks queries with the literal state machine — bounces are real
// loop trips here, not resolved in registers — and records the same event
// list, so a parity failure can be diffed node by node against
// flatkd::fcp/knn's trace.  One thread per query, runtime dim, any k (the
// bounded max-heap lives in the query's output slot, as in walk_heap_kernel).
#include <cstdint>

#include "trace.cuh"
#include "walk.cuh"

namespace fkd {
namespace {

__global__ void trace_kernel(const float* __restrict__ nodes, int32_t n, int dim, int stride,
                             const float* __restrict__ queries, int m, float cap2, int k,
                             int32_t* __restrict__ counts, fkd_hit* __restrict__ hits,
                             fkd_query_stats* __restrict__ stats, int32_t* __restrict__ events,
                             int64_t cap, int64_t* __restrict__ lens) {
    const int qi = int(blockIdx.x) * blockDim.x + threadIdx.x;
    if (qi >= m) return;
    const float* q = queries + int64_t(qi) * dim;
    uint64_t* heap = reinterpret_cast<uint64_t*>(hits + int64_t(qi) * k);
    int32_t* ev = events + int64_t(qi) * cap;
    int64_t len = 0, steps = 0, visited = 0, processed = 0;
    int count = 0;
    float r2 = cap2;
    int32_t curr = 0, prev = -1;
    while (curr >= 0 && n > 0) {                          // traverse.hpp:202
        ++steps;
        const int32_t parent = ((curr + 1) >> 1) - 1;     // 205
        if (curr >= n) {                                  // 206-212: bounce
            if (len < cap) ev[len] = ~curr;
            ++len;
            prev = curr;
            curr = parent;
            continue;
        }
        const float* node = nodes + int64_t(curr) * stride;
        const bool from_parent = prev < curr;             // 216
        if (from_parent) {                                // 217-222
            ++processed;
            if (len < cap) ev[len] = curr;
            ++len;
            float acc = 0.0f;
            for (int j = 0; j < dim; ++j) {
                const float dj = __fsub_rn(q[j], node[j]);
                acc = __fadd_rn(acc, __fmul_rn(dj, dj));
            }
            const uint64_t key = make_key(acc, curr);
            if (acc <= cap2) {
                if (count < k) {
                    int c = count++;
                    while (c > 0 && heap[(c - 1) >> 1] < key) {
                        heap[c] = heap[(c - 1) >> 1];
                        c = (c - 1) >> 1;
                    }
                    heap[c] = key;
                } else if (key < heap[0]) {
                    int c = 0;
                    while (true) {
                        const int l = 2 * c + 1, r = l + 1;
                        if (l >= k) break;
                        int mm = l;
                        if (r < k && heap[r] > heap[l]) mm = r;
                        if (heap[mm] <= key) break;
                        heap[c] = heap[mm];
                        c = mm;
                    }
                    heap[c] = key;
                }
                if (count == k) r2 = key_dist(heap[0]);
            }
        }
        ++visited;
        const int d = depth_of(curr) % dim;               // 225
        const float sd = __fsub_rn(q[d], node[d]);        // 226
        const int cs = sd > 0.0f;                         // 227
        const int32_t close = 2 * curr + 1 + cs;          // 228
        const int32_t far = 2 * curr + 2 - cs;            // 229
        const bool fir = __fmul_rn(sd, sd) <= r2;         // 230
        const int32_t next = from_parent ? close : ((prev == close) ? (fir ? far : parent) : parent);
        prev = curr;
        curr = next;                                      // -1 ends the walk (240-244)
    }
    // ascending order (extract_sorted, traverse.cpp:18-23)
    for (int end = count - 1; end > 0; --end) {
        const uint64_t top = heap[0], x = heap[end];
        heap[end] = top;
        int c = 0;
        while (true) {
            const int l = 2 * c + 1, r = l + 1;
            if (l >= end) break;
            int mm = l;
            if (r < end && heap[r] > heap[l]) mm = r;
            if (heap[mm] <= x) break;
            heap[c] = heap[mm];
            c = mm;
        }
        heap[c] = x;
    }
    int2* out = reinterpret_cast<int2*>(heap);
    for (int j = 0; j < k; ++j) {
        const uint64_t key = j < count ? heap[j] : kEmptyKey;
        out[j] = make_int2(int32_t(uint32_t(key)), int32_t(uint32_t(key >> 32) - kKeyOfs));
    }
    counts[qi] = count;
    stats[qi] = fkd_query_stats{steps, visited, processed};
    lens[qi] = len;
}

}  // namespace

int launch_trace(const float* nodes, int32_t n, int dim, int stride, const float* queries, int m,
                 float cap2, int k, int32_t* counts, fkd_hit* hits, fkd_query_stats* stats,
                 int32_t* events, int64_t cap, int64_t* lens, cudaStream_t st) {
    if (m <= 0) return 0;
    trace_kernel<<<(m + 63) / 64, 64, 0, st>>>(nodes, n, dim, stride, queries, m, cap2, k, counts, hits,
                                                stats, events, cap, lens);
    return 1;
}

}  // namespace fkd
