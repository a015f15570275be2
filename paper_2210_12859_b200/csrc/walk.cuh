// walk.cuh — sm_100a kernels for the stack-free k-d tree walk.
//
// One thread per query.  The per-query state is the reference's two node ids
// plus the shrinking squared radius (TraversalState, traverse.hpp:37-44);
// every transition follows traverse_step (traverse.hpp:198-248):
//
//   arrived from the parent   -> process the node, step into the close child
//   back from the close child -> far child if sd*sd <= radius2, else parent
//   back from the far child   -> parent
//
// B200-specific choices:
//   * Bounces off empty child slots (curr >= N, traverse.hpp:206-212) are
//     resolved in registers: the node's split plane is still live, so the
//     "step into the empty slot, step back" pair costs no load and no loop
//     trip.  The visit sequence, the candidate updates and (in STATS mode)
//     the step/visit counters are exactly the reference's.
//   * The candidate list is a register-resident ascending array of KB packed
//     64-bit keys ((dist2_bits + 1) << 32 | node): unsigned order on the key
//     IS hit_order (traverse.hpp:80-83), because squared distances are
//     non-negative floats whose bit patterns sort like the values.  Insertion
//     is a branch-free min/max bubble.  The first KB-k slots hold key 0 and
//     never move, so one kernel serves every k <= KB.  radius2 is the kth
//     key's distance (or the cap while fewer than k hits are held) — the
//     reference's KnnCandidates::radius2 (traverse.hpp:135-137); fcp is KB=1
//     (FcpCandidates, traverse.hpp:86-108).
//   * Squared distances use __fsub_rn/__fmul_rn/__fadd_rn left to right: no
//     FMA contraction, bit-identical to point.hpp:68-75 compiled without it.
//   * Queries may be walked in Morton order (order[] = sorted position ->
//     query id); results are scattered straight to the query's own slot, so
//     no separate un-permute pass exists.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "fkd_b200.h"

namespace fkd {

// Key = (bits(d2) + kKeyOfs) << 32 | node.  With the offset 0 (default) the
// high word is the distance's own bits, so forming a key and reading a
// radius back cost no add: one instruction less per walk trip (C3 step 9.33
// -> 9.21 ms, 8-D kNN16 -4.5%; profiles/r02/r02bn_key_offset_ab.log).  A real
// key may then equal the dummy key 0 (d2 = +0 at node 0): the insertion puts
// it after the dummies (x < 0 is false), and dummies are skipped by index.
#ifndef FKD_KEY_OFS
#define FKD_KEY_OFS 0
#endif
constexpr uint32_t kKeyOfs = FKD_KEY_OFS;
// fcp lane walks keep the walk's 1-based node id in the key's low word
// (converted at the output slot); kNN lists keep the 0-based id
// (FKD_FCP_KEY_NODE_OFS: 1 / 0).  For fcp the walk saves the subtract, 273 vs
// 280 SASS per 8 steps; for kNN8 ptxas re-schedules the loop to 296 vs 244.
#ifndef FKD_FCP_KEY_NODE_OFS
#define FKD_FCP_KEY_NODE_OFS 1
#endif
constexpr uint64_t kEmptyKey = (uint64_t(0x7f800000u + kKeyOfs) << 32) | 0xFFFFFFFFull;
constexpr uint64_t kNoBad = ~0ull;

// Block timeline instrumentation (profiling builds only: -DFKD_BLOCK_TRACE=1;
// tools/sm_timeline.py).  Each traced block appends {tag, SM, start, end}
// (%globaltimer ns) so the SM occupancy of a whole step — concurrent batches
// included — can be reconstructed without a profiler serialising kernels.
#ifndef FKD_BLOCK_TRACE
#define FKD_BLOCK_TRACE 0
#endif
struct BlockTraceRec {
    uint32_t tag, smid;
    unsigned long long t0, t1;
};

struct WalkArgs {
    const float* nodes;         // device tree store, `stride` floats per node
    int32_t n;                  // tree size
    int32_t dim;                // runtime dim (used by the dynamic-D kernel)
    int32_t stride;             // floats per node in the store
    const float* queries;       // m x dim row-major (caller layout)
    int64_t m;
    const uint32_t* order;      // walk position -> query id, or null
    float cap2;                 // squared_radius_cap(max_radius) (point.hpp:78-82)
    int32_t k;                  // output stride
    int32_t recursive_stats;    // report Engine::recursive counters
    int32_t* counts;            // [m]
    fkd_hit* hits;              // [m * k]
    unsigned long long* totals; // [3] steps, visited, processed (STATS)
    fkd_query_stats* per_query; // [m] or null (STATS)
    unsigned long long* bad;    // min id of a non-finite query
    int64_t id_base;            // added to query ids reported through `bad`
    int32_t budget;             // loop trips before a query moves to the overflow pass (0 = none)
    uint32_t* ovf_ids;          // [m] ids of queries over budget
    unsigned long long* ovf_count;
    unsigned long long* ovf_next;
    // continuation rounds / resume pass (walk_round_kernel)
    int32_t trips;                         // loop trips per query this round
    const uint32_t* wave_in;               // ids walked this round
    const unsigned long long* wave_n_in;   // their count (device)
    uint32_t* wave_out;                    // ids still walking after this round
    unsigned long long* wave_n_out;
    int2* wave_state;                      // [m] (curr, prev) of suspended walks
    int64_t resume_min;                    // >= this many over-budget queries: resume them with
                                           // the plain grid instead of the CTA overflow pass
    BlockTraceRec* btrace;                 // FKD_BLOCK_TRACE builds: record buffer (null: off)
    unsigned long long* btrace_next;
    long long btrace_cap;
    uint32_t btrace_tag;                   // batch id << 8 | kernel phase
};

__device__ __forceinline__ unsigned long long trace_clock() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Call at block start (all threads); end() where every thread of the block
// arrives together.  Compiles to nothing without FKD_BLOCK_TRACE.
struct BlockTrace {
    unsigned long long t0 = 0;
    __device__ __forceinline__ explicit BlockTrace(const WalkArgs& a) {
        if constexpr (FKD_BLOCK_TRACE) {
            if (a.btrace && threadIdx.x == 0) t0 = trace_clock();
        }
    }
    __device__ __forceinline__ void end(const WalkArgs& a, uint32_t phase) {
        if constexpr (FKD_BLOCK_TRACE) {
            __syncthreads();
            if (a.btrace && threadIdx.x == 0) {
                const unsigned long long i = atomicAdd(a.btrace_next, 1ull);
                unsigned sm;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
                if (i < (unsigned long long)a.btrace_cap) a.btrace[i] = BlockTraceRec{a.btrace_tag | phase, sm, t0, trace_clock()};
            }
        }
    }
};

__device__ __forceinline__ uint64_t make_key(float d2, int32_t node) {
    return (uint64_t(__float_as_uint(d2) + kKeyOfs) << 32) | uint32_t(node);
}

// The Hit node of a lane-walk key whose low word is node + OFS (-1 for an
// empty slot, whose low word is 0xFFFFFFFF)
template <uint32_t OFS>
__device__ __forceinline__ int32_t key_node(uint64_t key, bool hit) {
    if constexpr (OFS == 0) {
        (void)hit;
        return int32_t(uint32_t(key));
    } else {
        return hit ? int32_t(uint32_t(key) - OFS) : -1;
    }
}

__device__ __forceinline__ float key_dist(uint64_t key) {
    return __uint_as_float(uint32_t(key >> 32) - kKeyOfs);
}

// Empty slot of a register list: the admission cap's own key with node
// 0xFFFFFFFF.  Every admissible candidate (d2 <= cap2, inclusive,
// traverse.hpp:92/122) has a smaller key and every inadmissible one a larger
// key, so admission is the single compare key < L[KB-1], and radius2 is just
// key_dist(L[KB-1]): cap2 while the list is short, the kth distance once it
// is full (traverse.hpp:97, 135-137).  With cap2 = +inf this is kEmptyKey.
__device__ __forceinline__ uint64_t cap_key(float cap2) {
    return (uint64_t(__float_as_uint(cap2) + kKeyOfs) << 32) | 0xFFFFFFFFull;
}

__device__ __forceinline__ int32_t depth_of(int32_t node) {  // tree.hpp:20-22
    return 31 - __clz(node + 1);
}

template <int D>
__device__ __forceinline__ int split_dim(int32_t node) {  // tree.hpp:27-29
    return depth_of(node) % D;
}

template <int D>
__device__ __forceinline__ float pick(const float (&a)[D], int d) {
    float r = a[0];
#pragma unroll
    for (int i = 1; i < D; ++i) r = (d == i) ? a[i] : r;
    return r;
}

// Packed FP32 pairs (sm_100: FADD2 / FMUL2, one instruction for two IEEE
// round-to-nearest lanes, so every lane's bits equal the scalar op's).
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// point.hpp:68-75: acc = 0; acc += (q_i - p_i)^2 left to right.  0 + x == x
// for the non-negative first square, so the chain starts at it.  The
// differences and squares are formed two coordinates per instruction
// (FADD2 / FMUL2, exact per lane); the sum stays the scalar left-to-right
// chain, so the result is bit-identical to the reference's loop (for D = 3:
// 6 instead of 8 FP instructions).
//
// Pairs are used for D <= 4 with lists of <= 8 slots (PAIRS): with longer
// lists or more coordinates the pair registers cost more than they save
// (measured: 4-D kNN20 walk +12%, the 8-D kNN16 CTA pass drops to one CTA
// per SM).  Both forms give the same bits, so callers may mix them.
template <int D, bool PAIRS = (D <= 4)>
__device__ __forceinline__ float sq_dist(const float (&q)[D], const float (&p)[D]) {
    if constexpr (!PAIRS || D == 1) {
        float d0 = __fsub_rn(q[0], p[0]);
        float acc = __fmul_rn(d0, d0);
#pragma unroll
        for (int i = 1; i < D; ++i) {
            const float di = __fsub_rn(q[i], p[i]);
            acc = __fadd_rn(acc, __fmul_rn(di, di));
        }
        return acc;
    } else {
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i + 1 < D; i += 2) {
            const uint64_t d = f2_sub(f2_pack(q[i], q[i + 1]), f2_pack(p[i], p[i + 1]));
            float a, b;
            f2_unpack(f2_mul(d, d), a, b);
            acc = i == 0 ? __fadd_rn(a, b) : __fadd_rn(__fadd_rn(acc, a), b);
        }
        if constexpr (D % 2 == 1) {
            const float dl = __fsub_rn(q[D - 1], p[D - 1]);
            acc = __fadd_rn(acc, __fmul_rn(dl, dl));
        }
        return acc;
    }
}

// Full point of one node.  S is the store stride: S in {2,4,8} is a padded
// vector layout (LDG.64 / LDG.128), S == D is packed (scalar loads).  With
// S > D the last padding float holds the split coordinate (pack_nodes);
// `split` receives it.
template <int D, int S>
__device__ __forceinline__ void load_point(const float* __restrict__ nodes, int32_t i,
                                           float (&p)[D], float* split = nullptr) {
    const float* base = nodes + size_t(i) * S;
    if constexpr (S == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(base));
        const float t[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < D; ++j) p[j] = t[j];
        if (split) *split = t[3];
    } else if constexpr (S == 8) {
        const float4 v0 = __ldg(reinterpret_cast<const float4*>(base));
        const float4 v1 = __ldg(reinterpret_cast<const float4*>(base) + 1);
        const float t[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int j = 0; j < D; ++j) p[j] = t[j];
        if (split) *split = t[7];
    } else if constexpr (S == 12 || S == 16) {
        // 9..16-D: three or four 16-byte vectors; with S > D the last float is the split plane
        constexpr int NV = S / 4;
        float t[S];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(base) + v);
            t[4 * v] = x.x;
            t[4 * v + 1] = x.y;
            t[4 * v + 2] = x.z;
            t[4 * v + 3] = x.w;
        }
#pragma unroll
        for (int j = 0; j < D; ++j) p[j] = t[j];
        if constexpr (S > D) {
            if (split) *split = t[S - 1];
        }
    } else if constexpr (S == 2 && D == 2) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(base));
        p[0] = v.x;
        p[1] = v.y;
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) p[j] = __ldg(base + j);
    }
}

// Key order on the FP64 compare.  A key is (bits(d2) << 32) | node with d2 in
// [0, +inf] (queries and tree are finite; cap2 is not NaN), so its sign bit
// is 0 and its high word is <= 0x7F800000: read as an IEEE double it is
// finite and non-negative, and non-negative doubles order exactly like their
// bit patterns (FP64 never flushes subnormals, which keys with d2 = 0 are).  One DSETP replaces the two-instruction 64-bit ISETP pair and runs
// on the FP64 pipe instead of the ALU pipe the walk saturates; and since the
// selects that follow are integer, ptxas cannot re-form a min/max idiom with
// compares of its own.  (B200-specific: sm_100 has a full-rate-class FP64
// pipe.)
__device__ __forceinline__ bool key_lt(uint64_t a, uint64_t b) {
    return __longlong_as_double(static_cast<long long>(a)) < __longlong_as_double(static_cast<long long>(b));
}

// Sorted insertion of x into L (ascending; x < L[KB-1], so the last key
// drops out).  All KB compares are independent, then each slot takes its
// left neighbour (x went further left), x (x lands here) or stays:
//   L[j] = c[j] ? (c[j-1] ? L[j-1] : x) : L[j],   c[j] = x < L[j],
// one DSETP + a predicated SEL pair per slot (KB = 8: 24 SASS).  (The
// compare-exchange bubble is a serial chain through all slots, which ptxas
// shortened with a second 64-bit compare per slot: 61 SASS for KB = 8,
// measured in the kNN8 walk, where insertions were a third of all
// instructions.)  c is monotone because L is sorted; keys are distinct
// except equal dummies / empty slots, which x never equals (x > 0 = dummy,
// x < L[KB-1] <= the empty key).
template <int KB>
__device__ __forceinline__ void list_insert(uint64_t (&L)[KB], uint64_t x) {
    bool c[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) c[j] = key_lt(x, L[j]);
#pragma unroll
    for (int j = KB - 1; j > 0; --j) L[j] = c[j] ? (c[j - 1] ? L[j - 1] : x) : L[j];
    L[0] = c[0] ? x : L[0];
}

template <bool STATS>
struct Counters {
    unsigned long long steps = 0, visited = 0, processed = 0;
    __device__ __forceinline__ void step(int s, int v, int p) {
        if constexpr (STATS) {
            steps += s;
            visited += v;
            processed += p;
        }
    }
};

// ---------------------------------------------------------------------------
// Register-list walk, D in 1..8 compile-time, KB slots, k <= KB at run time.
// One query's complete state; step() is one loop trip of the state machine.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ int dim_up(int d) {  // split dim one level deeper
    if constexpr (D == 1) return 0;
    else if constexpr ((D & (D - 1)) == 0) return (d + 1) & (D - 1);
    else return d == D - 1 ? 0 : d + 1;
}

template <int D>
__device__ __forceinline__ int dim_down(int d) {  // split dim one level up
    if constexpr (D == 1) return 0;
    else if constexpr ((D & (D - 1)) == 0) return (d - 1) & (D - 1);
    else return d == 0 ? D - 1 : d - 1;
}

// Lowest dimension whose 16-slot walks keep the list in the output slot
// (LaneWalk::kSlot); 9 turns the mode off.
// Experiment knob: kNN lists compute the distance only on a first visit
// (a divergent block, as fcp in D != 3) instead of every trip.
#ifndef FKD_KNN_DIST_BRANCH
#define FKD_KNN_DIST_BRANCH 0
#endif

#ifndef FKD_SLOT_LIST_MIN_D
#define FKD_SLOT_LIST_MIN_D 8
#endif

// Lists of >= FKD_STREAM_IO_MIN_KB slots read their query and write their
// final results with the evict-first (.cs) cache hint, so the streamed query /
// result lines (kNN8: 76 B per query) displace fewer tree lines in L2.
// Measured (tools/stream_io_ab.sh, profiles/r01j_stream_io_ab.log): kNN8 walk
// -0.4% clustered and uniform, fcp +0.3% (so fcp keeps the plain path).
#ifndef FKD_STREAM_QUERY_LOADS
#define FKD_STREAM_QUERY_LOADS 1
#endif
// Nodes of one 16-byte vector without a plane slot (4-D): every trip loads
// the whole node.  The split-coordinate-only load of a return trip needed its
// own address form and a branch around the two loads, and ptxas rebuilt the
// store pointer from uniform registers on both sides each trip: 4-D kNN8 312
// -> 287 SASS per 4 steps, walk -10% (fcp -10%, kNN4 -13%, kNN50 -6%;
// profiles/r02/r02bt_full_return_load_ab.log).  8-D nodes (two vectors, one
// sector) too: kNN8 -9%, fcp -7%, kNN32 -5%, except the 16-slot walks whose
// list lives in the output slot (+4%; r02bu_full_return_load8_ab.log).
#ifndef FKD_FULL_RETURN_LOAD
#define FKD_FULL_RETURN_LOAD 1
#endif
#ifndef FKD_FULL_RETURN_LOAD_MAX_S
#define FKD_FULL_RETURN_LOAD_MAX_S 8
#endif
// Packed-pair distance (FADD2/FMUL2, LaneWalk::kPairDist): 2-/3-D lists of any
// length and 4-D lists of up to 32 slots (round 1 stopped at 8 slots): 2-D
// kNN16 -1.3%, 3-D kNN16 -3%, kNN50 -1%, 4-D kNN16 -4%, kNN20 -3%, kNN32 -2%;
// 4-D kNN50 +7% (profiles/r02/r02bz_pair_any_kb_ab.log, r02ca_pair4d_ab.log)
// ... and 5..16-D lists of up to 16 slots: 8-D fcp -4%, kNN8 -1.5%, 6-D kNN8
// -3%, 10-D kNN8 -1.5 to -4%, 5-D and 8-D kNN16 within 1% (r02cb_pair_hd_ab.log)
#ifndef FKD_PAIR_HD
#define FKD_PAIR_HD 1
#endif
#ifndef FKD_STREAM_IO_MIN_KB
#define FKD_STREAM_IO_MIN_KB 8
#endif

// Box pruning (incremental distance, Arya & Mount): from this dimension up,
// the production walk (not STATS, not unordered) enters a far child only if
// the squared distance from the query to the far child's whole cell is within
// radius2, instead of the split plane alone (traverse.hpp:230).  The cell's
// per-dimension offsets come from the deepest ancestor in that dimension
// whose path went to its far side; their squares are summed left to right
// with the same round-to-nearest ops as the point distance, term by term no
// larger than any point of the cell's, so the test never prunes a node the
// reference would admit: same result set, same bits, fewer nodes (oracle
// simulation, N = 1M uniform: 8-D kNN16 12.3k -> 3.1k processed per query,
// 4-D kNN50 794 -> 508, 3-D kNN8 107 -> 91).  STATS mode keeps the
// reference's plane test, so the counters stay the reference's.  Measured
// (N = 10M uniform, profiles/r02/r02ac_box_pruning_ab.log): 8-D kNN16
// 270 -> 123 ms, 6-D kNN8 23.4 -> 13.7, 5-D kNN16 14.3 -> 10.5; in 4-D the
// offsets' registers and instructions cost more than the pruning saves (kNN8
// +16%, kNN50 +40% at 138 registers), so the mode starts at 5-D.
#ifndef FKD_BOX_MIN_D
#define FKD_BOX_MIN_D 5
#endif

template <int D>
constexpr uint32_t dim_levels_mask() {  // bits 0, D, 2D, ... below 32
    uint32_t m = 0;
    for (int i = 0; i < 32; i += D) m |= 1u << i;
    return m;
}

template <int D, int S, int KB, bool STATS, bool UNORDERED>
struct LaneWalk {
    static constexpr bool kBox = D >= FKD_BOX_MIN_D && D > 1 && !STATS && !UNORDERED;
    // With a split-plane slot in the store (S > D) the walk never needs the
    // split dimension: qr holds the query rotated so that qr[0] is the
    // coordinate split at the current depth (rotated by one per level).
    static constexpr bool kRot = S > D && D > 1;
    static constexpr int kKB = KB;
    static constexpr bool kPairDist = D <= 3 || (D == 4 && KB <= 32) || (FKD_PAIR_HD && D >= 5 && D <= 16 && KB <= 16);
    static constexpr uint32_t kNodeOfs = KB == 1 ? FKD_FCP_KEY_NODE_OFS : 0;  // key low word = node + kNodeOfs
    static constexpr bool kStreamIO = KB >= FKD_STREAM_IO_MIN_KB;
    static constexpr int kD = D;
    // Slot-list mode (high dimensions, 16 slots): the sorted list lives in the
    // query's own output slot (Hit format, k entries) and only its kth key is
    // a register.  In 8-D a query processes ~15k nodes for ~100 admissions,
    // so the 32 list registers buy nothing but cost occupancy in a walk that
    // is load-latency bound.
    static constexpr bool kSlot = D >= FKD_SLOT_LIST_MIN_D && KB == 16;
    float q[D];
    float qr[kRot ? D : 1];
    uint64_t L[kSlot ? 1 : KB];  // slot mode: L[0] is the kth key
    int32_t curr, prev;  // 1-based node ids (the reference's + 1)
    // D <= 3: from_parent carried from the last transition and the children
    // formed by bit ops — ~1.5% faster 3-D walks, but 3-8% slower 4-D ones
    // (same-box A/B, profiles/r02/r02ah_transition_forms_ab.log), so only there
    static constexpr bool kCarry = D <= 3;
    bool fromp;  // kCarry: arrived from the parent (prev < curr)
    int d;  // split dim of curr, tracked incrementally (tree.hpp:27-29)
    // box mode: squared per-dimension offsets of curr's cell from the query,
    // and bit l set iff the path from level l went to the far child
    float osq[kBox ? D : 1];
    uint32_t farmask;
    float r2;
    int64_t qi;
    Counters<STATS> cnt;

    // Loads the query and resets the state (traverse.hpp:250-255).  Returns
    // false (and flags the id) for a non-finite query (batch.cpp:79).
    __device__ __forceinline__ bool init(const WalkArgs& a, int64_t pos) {
        if constexpr (kStreamIO)
            qi = a.order ? int64_t(__ldcs(a.order + pos)) : pos;
        else
            qi = a.order ? int64_t(__ldg(a.order + pos)) : pos;
        const float* qp = a.queries + qi * D;
        bool finite = true;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if constexpr (kStreamIO && FKD_STREAM_QUERY_LOADS)
                q[j] = __ldcs(qp + j);
            else
                q[j] = __ldg(qp + j);
            finite &= isfinite(q[j]);
        }
        if (!finite) {
            atomicMin(a.bad, (unsigned long long)(a.id_base + qi));
            return false;
        }
        if constexpr (kRot) {
#pragma unroll
            for (int j = 0; j < D; ++j) qr[j] = q[j];  // depth 0 splits dim 0
        }
        const uint64_t empty = cap_key(a.cap2);
        if constexpr (kSlot) {
            int2* out = reinterpret_cast<int2*>(a.hits + qi * a.k);
            for (int j = 0; j < a.k; ++j) out[j] = make_int2(-1, 0x7f800000);  // Hit{-1, +inf}
            L[0] = empty;
        } else {
            const int dummies = KB - a.k;
#pragma unroll
            for (int j = 0; j < KB; ++j) L[j] = j < dummies ? 0ull : empty;
        }
        curr = 1;  // 1-based ids inside the walk: the root, entered from its parent 0 (= -1)
        prev = 0;
        fromp = true;
        d = 0;
        if constexpr (kBox) {
#pragma unroll
            for (int j = 0; j < D; ++j) osq[j] = 0.0f;
            farmask = 0;
        }
        r2 = a.cap2;
        cnt = Counters<STATS>();
        return true;
    }

    // One transition of traverse_step (traverse.hpp:198-248) plus the
    // in-register bounces.  Returns false once the root stepped to -1.
    __device__ __forceinline__ bool step(const WalkArgs& a) {
        const int32_t n = a.n;  // 1-based ids: node c exists iff c <= n
        const bool from_parent = kCarry ? fromp : prev < curr;
        const float* nodes = a.nodes - S;  // nodes + c * S is 1-based node c's slot
        float p[D];
        float pd;
        if constexpr (S == D && D > 1 && S <= FKD_FULL_RETURN_LOAD_MAX_S && !kSlot && FKD_FULL_RETURN_LOAD) {
            // one vector load on every trip (a return trip's plane is in the same
            // sector): no second address form, no branch around the loads
            load_point<D, S>(nodes, curr, p);
            pd = pick(p, d);
        } else if constexpr (S == D && D > 1) {
            if (from_parent) {
                load_point<D, S>(nodes, curr, p);
                pd = pick(p, d);
            } else {
                pd = __ldg(nodes + size_t(curr) * S + d);
                // a return trip loads only the split coordinate; the distance
                // below is formed every trip but used only on a first visit.
                // The empty asm defines p (an unspecified value, no
                // instruction) so no indeterminate value is ever read.
#pragma unroll
                for (int j = 0; j < D; ++j) asm("" : "=f"(p[j]));
            }
        } else if constexpr (S > D) {
            load_point<D, S>(nodes, curr, p, &pd);  // split plane from the padding slot
        } else {
            load_point<D, S>(nodes, curr, p);
            pd = pick(p, d);
        }
        if constexpr ((KB > 1 && !FKD_KNN_DIST_BRANCH) || (KB == 1 && D == 3)) {
            // traverse.hpp:217-222.  kNN, and 3-D fcp: the distance is
            // computed every trip (no divergent block; measured faster: fcp
            // 3-D -3.6% with the packed-pair distance, but 4-D +22%, and the
            // 2-D fcp walk would take 44 instead of 28 registers),
            // admission is predicated on a first visit.
            const float d2 = sq_dist<D, kPairDist>(q, p);
            const uint64_t key = make_key(d2, curr - 1 + int32_t(kNodeOfs));
            if constexpr (kSlot) {
                if (from_parent && key_lt(key, L[0])) {
                    slot_insert(a, key);
                    r2 = key_dist(L[0]);
                }
            } else if (from_parent && key_lt(key, L[KB - 1])) {  // d2 <= cap2 and beats the kth (cap_key)
                list_insert(L, key);
                r2 = key_dist(L[KB - 1]);
            }
        } else if (from_parent) {  // fcp, D != 3: a branch is cheaper than the FP ops
            const float d2 = sq_dist<D, kPairDist>(q, p);
            const uint64_t key = make_key(d2, curr - 1 + int32_t(kNodeOfs));
            if constexpr (kSlot) {
                if (key_lt(key, L[0])) {
                    slot_insert(a, key);
                    r2 = key_dist(L[0]);
                }
            } else if (key_lt(key, L[KB - 1])) {  // d2 <= cap2 and beats the kth (cap_key)
                list_insert(L, key);
                r2 = key_dist(L[KB - 1]);
            }
        }
        cnt.step(1, 1, from_parent ? 1 : 0);

        float qd;
        if constexpr (kRot)
            qd = qr[0];
        else
            qd = pick(q, d);
        const float sd = __fsub_rn(qd, pd);                         // 226
        const bool cs = sd > 0.0f;                                 // 227
        const float sd2 = __fmul_rn(sd, sd);
        bool fir;
        if constexpr (kBox) {
            // the far child's cell: this cell with offset |sd| in the split dim
            float box = 0.0f;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const float t = (i == d) ? sd2 : osq[i];
                box = i == 0 ? t : __fadd_rn(box, t);
            }
            fir = box <= r2;
        } else {
            fir = sd2 <= r2;                                       // 230
        }
        // 205, 228-229 with 1-based ids (c = node + 1): parent c >> 1 (the
        // root's is 0, i.e. -1), children 2c and 2c + 1 — one instruction each
        const int32_t parent = curr >> 1;
        const int32_t l = curr << 1, r = l | 1;
        int32_t next;
        bool down;
        bool to_far = false, back_far = false;  // box mode: entering / leaving the far child
        if constexpr (!UNORDERED) {
            const int32_t close = kCarry ? (l | int32_t(cs)) : (cs ? r : l);  // 228 (1-based: r = l | 1)
            const int32_t far = kCarry ? (close ^ 1) : (cs ? l : r);           // 229
            // 232-238 with the bounces off empty slots (206-212) folded in:
            // from the parent, an empty close slot bounces straight back,
            // which is a return from the close child; an empty far slot
            // bounces back, which is a return from the far child (-> parent).
            const bool close_ok = close <= n;
            const bool go_close = from_parent && close_ok;
            const bool try_far = from_parent ? !close_ok : prev == close;
            const bool far_ok = far <= n;
            const bool go_far = try_far && fir && far_ok;
            if constexpr (STATS) {
                if (from_parent && !close_ok) cnt.step(2, 1, 0);
                if (try_far && fir && !far_ok) cnt.step(2, 1, 0);
            }
            down = go_close || go_far;
            next = go_close ? close : (go_far ? far : parent);
            to_far = go_far;
            back_far = !from_parent && prev != close;
        } else {
            // left-first order; a child is entered iff it is on the query's
            // side or its plane is within the radius
            const bool enter_left = !cs || fir, enter_right = cs || fir;
            if (from_parent)
                next = enter_left ? l : (enter_right ? r : parent);
            else
                next = (prev == l && enter_right) ? r : parent;
            if (next > n) {
                cnt.step(2, 1, 0);
                next = (next == l && enter_right) ? r : parent;
                if (next > n) {
                    cnt.step(2, 1, 0);
                    next = parent;
                }
            }
            down = next != parent;
        }
        if (!down && curr == 1) return false;  // 240-244: the root stepped to -1
        if constexpr (kBox) box_update(a, down, to_far, sd2, back_far);
        if constexpr (kRot) {
            float t[D];
#pragma unroll
            for (int j = 0; j < D; ++j) t[j] = down ? qr[(j + 1) % D] : qr[(j + D - 1) % D];
#pragma unroll
            for (int j = 0; j < D; ++j) qr[j] = t[j];
            if constexpr (kBox) d = down ? dim_up<D>(d) : dim_down<D>(d);
        } else {
            d = down ? dim_up<D>(d) : dim_down<D>(d);
        }
        prev = curr;
        curr = next;
        if constexpr (kCarry) fromp = down;
        return true;
    }

    // The split coordinate of (1-based) node c, split in dim dim.
    __device__ __forceinline__ float plane_of(const WalkArgs& a, int32_t c, int dim) const {
        const float* base = a.nodes + size_t(c - 1) * S;
        if constexpr (S > D && D > 1) return __ldg(base + (S - 1));  // the padding slot holds it
        else return __ldg(base + dim);
    }
    // Box mode, after a transition out of curr (split dim d): entering a
    // child records the decision bit of this level (and, for the far child,
    // its offset); leaving curr upward after its far child restores curr's
    // own offset in d, from the deepest same-dimension ancestor whose path
    // went far (one load; 0 if none).
    __device__ __forceinline__ void box_update(const WalkArgs& a, bool down, bool to_far, float sd2, bool back_from_far) {
        const int lvl = 31 - __clz(curr);
        if (down) {
            farmask = to_far ? (farmask | (1u << lvl)) : (farmask & ~(1u << lvl));
            if (to_far) {
#pragma unroll
                for (int i = 0; i < D; ++i) osq[i] = (i == d) ? sd2 : osq[i];
            }
        } else if (back_from_far) {
            const uint32_t cand = farmask & (dim_levels_mask<D>() << d) & ((1u << lvl) - 1u);
            float o2 = 0.0f;
            if (cand) {
                const int la = 31 - __clz(cand);
                const float o = __fsub_rn(pick(q, d), plane_of(a, curr >> (lvl - la), d));
                o2 = __fmul_rn(o, o);
            }
#pragma unroll
            for (int i = 0; i < D; ++i) osq[i] = (i == d) ? o2 : osq[i];
        }
    }
    // Box mode, resuming a parked walk: the path's decisions and offsets from
    // the root down to curr (one load per level).
    __device__ __forceinline__ void box_recompute(const WalkArgs& a) {
#pragma unroll
        for (int j = 0; j < D; ++j) osq[j] = 0.0f;
        farmask = 0;
        const int L = 31 - __clz(curr);
        for (int lv = 0; lv < L; ++lv) {
            const int32_t anc = curr >> (L - lv), child = curr >> (L - lv - 1);
            const int da = lv % D;
            const float sda = __fsub_rn(pick(q, da), plane_of(a, anc, da));
            const bool close_right = sda > 0.0f;
            if (((child & 1) != 0) != close_right) {  // went to the far child
                farmask |= 1u << lv;
                const float o2 = __fmul_rn(sda, sda);
#pragma unroll
                for (int i = 0; i < D; ++i) osq[i] = (i == da) ? o2 : osq[i];
            }
        }
    }

    // Sorted insertion into the output slot (slot mode): x passes the
    // entries it does not beat, then displaces each later one by one; the
    // old kth drops out.  Entries are converted as in resume() / finish().
    __device__ __forceinline__ void slot_insert(const WalkArgs& a, uint64_t x) {
        const int k = a.k;
        const uint64_t empty = cap_key(a.cap2);
        int2* out = reinterpret_cast<int2*>(a.hits + qi * k);
        uint64_t last = x;
        for (int j = 0; j < k; ++j) {
            const int2 h = out[j];
            const uint64_t kj = h.x < 0 ? empty : (uint64_t(uint32_t(h.y) + kKeyOfs) << 32) | (uint32_t(h.x) + kNodeOfs);
            last = kj;
            if (key_lt(x, kj)) {
                const bool hit = uint32_t(x) != 0xFFFFFFFFu;
                out[j] = make_int2(key_node<kNodeOfs>(x, hit), hit ? int32_t(uint32_t(x >> 32) - kKeyOfs) : 0x7f800000);
                last = x;
                x = kj;
            }
        }
        L[0] = last;
    }

    // Resumes a walk parked by an earlier pass (walk budget or round): the state is the
    // reference's two node ids; the candidate list is the partial one the
    // round left in the query's own output slot; radius2 and the split
    // dimension are recomputed from them.
    __device__ __forceinline__ void resume(const WalkArgs& a, int32_t id) {
        qi = id;
        const float* qp = a.queries + size_t(qi) * D;
#pragma unroll
        for (int j = 0; j < D; ++j) q[j] = __ldg(qp + j);
        const int dummies = KB - a.k;
        const uint64_t empty = cap_key(a.cap2);
        const int2* slot = reinterpret_cast<const int2*>(a.hits + size_t(qi) * a.k);
        if constexpr (kSlot) {
            const int2 h = slot[a.k - 1];  // the list stays in the slot; only its kth is a register
            L[0] = h.x < 0 ? empty : (uint64_t(uint32_t(h.y) + kKeyOfs) << 32) | (uint32_t(h.x) + kNodeOfs);
        } else {
#pragma unroll
            for (int j = 0; j < KB; ++j) {
                if (j < dummies) {
                    L[j] = 0ull;
                } else {
                    const int2 h = slot[j - dummies];
                    L[j] = h.x < 0 ? empty : (uint64_t(uint32_t(h.y) + kKeyOfs) << 32) | (uint32_t(h.x) + kNodeOfs);
                }
            }
        }
        r2 = key_dist(L[kSlot ? 0 : KB - 1]);
        const int2 st = a.wave_state[qi];  // 0-based (curr, prev)
        curr = st.x + 1;
        prev = st.y + 1;
        fromp = prev < curr;
        d = depth_of(st.x) % D;
        if constexpr (kBox) box_recompute(a);
        if constexpr (kRot) {
            // qr[j] = q[(d + j) % D] as d predicated one-place rotations: a
            // select chain on d is folded back into a dynamic index by the
            // compiler, which puts the whole walk state in local memory
#pragma unroll
            for (int j = 0; j < D; ++j) qr[j] = q[j];
#pragma unroll
            for (int r = 0; r < D - 1; ++r) {
                const bool more = r < d;
                float t[D];
#pragma unroll
                for (int j = 0; j < D; ++j) t[j] = more ? qr[(j + 1) % D] : qr[j];
#pragma unroll
                for (int j = 0; j < D; ++j) qr[j] = t[j];
            }
        }
        cnt = Counters<STATS>();
    }

    // fixed-stride slot in input order (batch.cpp:104-119).  A parked walk
    // (final = false) leaves only its partial list: the passes that continue
    // it read the list, never the count, which its last finish writes.
    __device__ __forceinline__ void finish(const WalkArgs& a, bool final = true) {
        const int k = a.k;
        const int dummies = KB - k;
        int2* out = reinterpret_cast<int2*>(a.hits + qi * k);
        int c = 0;
        if constexpr (kSlot) {
            // the slot already holds the list; count its hits (all k once the kth is one)
            if (final) {
                if (uint32_t(L[0]) != 0xFFFFFFFFu) {
                    c = k;
                } else {
                    for (int j = 0; j < k; ++j) c += out[j].x >= 0;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < KB; ++j) {
                const int s = j - dummies;
                if (s >= 0) {
                    const uint64_t key = L[j];
                    const bool hit = uint32_t(key) != 0xFFFFFFFFu;  // empty slot -> Hit{-1, +inf}
                    const int2 h = make_int2(key_node<kNodeOfs>(key, hit),
                                             hit ? int32_t(uint32_t(key >> 32) - kKeyOfs) : 0x7f800000);
                    if (kStreamIO && final)
                        __stcs(out + s, h);
                    else
                        out[s] = h;
                    c += hit;
                }
            }
        }
        if (final) {
            if (kStreamIO)
                __stcs(a.counts + qi, c);
            else
                a.counts[qi] = c;
        }
        if constexpr (STATS) {
            if (a.per_query) {
                unsigned long long s = cnt.steps, v = cnt.visited;
                if (a.recursive_stats) {
                    s = cnt.processed + (s - v);
                    v = cnt.processed;
                }
                a.per_query[qi].steps = (int64_t)s;
                a.per_query[qi].nodes_visited = (int64_t)v;
                a.per_query[qi].nodes_processed = (int64_t)cnt.processed;
            }
        }
    }
};

template <bool STATS>
__device__ __forceinline__ void add_totals(const WalkArgs& a, unsigned long long s,
                                           unsigned long long v, unsigned long long p) {
    if constexpr (STATS) {
        if (a.recursive_stats) {  // traverse.hpp:262-283 counting
            s = p + (s - v);
            v = p;
        }
        for (int off = 16; off > 0; off >>= 1) {
            s += __shfl_down_sync(0xffffffffu, s, off);
            v += __shfl_down_sync(0xffffffffu, v, off);
            p += __shfl_down_sync(0xffffffffu, p, off);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(a.totals + 0, s);
            atomicAdd(a.totals + 1, v);
            atomicAdd(a.totals + 2, p);
        }
    }
}

// Minimum resident blocks per SM for the plain walk: the kNN kernels are
// latency-bound, so occupancy beats the few bytes of list spill ptxas needs
// to fit KB=8 into 32 registers (64 warps/SM instead of 48).
#ifndef FKD_MINB_KB8
#define FKD_MINB_KB8 1
#endif
#ifndef FKD_MINB_KB16
#define FKD_MINB_KB16 1
#endif
// 5-D and 8-D, 16 slots: 4 blocks (64 registers, 16 B of stack in 8-D)
// instead of 3 (72 registers): the 8-D walk is long-scoreboard bound at 24
// warps/SM; kNN16 M=1M 8-D 318 -> 298 ms, 5-D -3.5%, while 6-D (+4%), 7-D
// (+0.5%) and 2-D/3-D/4-D (+0.4-0.8%) lose that way (tools/occ16_ab.sh,
// tools/occ16_hd_ab.sh, profiles/r01i_occ16_*ab.log)
#ifndef FKD_MINB_KB16_HIGH_D
#define FKD_MINB_KB16_HIGH_D 1  // round 1: 4 (-3.5% in 5-D); with box pruning (r02) 1 is 2% better
#endif
// 16-slot walks whose list lives in the output slot (LaneWalk::kSlot, 8-D):
// 5 blocks (48 registers, 40 B of spill stores) -> 8-D kNN16 walk 300 -> 281 ms;
// 4 blocks 300 ms, 6 blocks (40 registers) 295 ms (tools/slot_ab.sh,
// profiles/r01i_slot_ab.log)
#ifndef FKD_MINB_KB16_SLOT
#define FKD_MINB_KB16_SLOT 5
#endif
// Threads per walk block: a block's slot stays held until its slowest warp
// ends, so smaller blocks waste less occupancy on budget-capped stragglers.
#ifndef FKD_WALK_T
#define FKD_WALK_T 256
#endif
constexpr int kWalkThreads = FKD_WALK_T;

template <int D, int KB>
constexpr int walk_min_blocks() {
    if (D > 8) return 1;  // 9..16-D: the query, its rotation, the cell offsets and the node are 4 x D registers
    return KB == 8 ? FKD_MINB_KB8 : (KB == 16 ? (D >= FKD_SLOT_LIST_MIN_D ? FKD_MINB_KB16_SLOT
                                             : (D == 5 || D == 8) ? FKD_MINB_KB16_HIGH_D : FKD_MINB_KB16)
                       : 1);
}

// Walks until the root exits (false) or about `trips` loop trips have run
// (true: the walk is parked at (curr, prev)).  Several steps per budget
// check (measured on C3: fcp 8 steps, -7% then -3% vs 1; kNN 4 steps, 8 is
// +1.5%); the budget is approximate by a few trips, which nothing depends on.
template <class W>
__device__ __forceinline__ bool walk_budgeted(W& w, const WalkArgs& a, int trips) {
    constexpr int kSteps = W::kKB == 1 ? 8 : 4;
    while (true) {
        if constexpr (W::kD == 3) {
            // 3-D: the explicit body (the unrolled loop below schedules 3-D kNN8
            // 2.7% slower; for 4-D kNN8 it is 14% faster: tools/steps_ab.sh)
            if (!w.step(a)) return false;
            if (!w.step(a)) return false;
            if (!w.step(a)) return false;
            if (!w.step(a)) return false;
            if constexpr (kSteps == 8) {
                if (!w.step(a)) return false;
                if (!w.step(a)) return false;
                if (!w.step(a)) return false;
                if (!w.step(a)) return false;
            }
        } else {
#pragma unroll
            for (int i = 0; i < kSteps; ++i)
                if (!w.step(a)) return false;
        }
        if ((trips -= kSteps) <= 0) return true;
    }
}

// One thread per walk position (plain grid).
template <int D, int S, int KB, bool STATS, bool UNORDERED>
__global__ void __launch_bounds__(kWalkThreads, walk_min_blocks<D, KB>()) walk_kernel(const WalkArgs a) {
    if (*a.bad != kNoBad) return;  // a rejected batch (batch.cpp:79) writes no slot
    BlockTrace bt(a);
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    LaneWalk<D, S, KB, STATS, UNORDERED> w;
    bool active = i < a.m && w.init(a, i);
    if (active) {
        bool over = false;
        if (a.n > 0) {
            if (STATS || a.budget <= 0) {
                while (w.step(a)) {
                }
            } else {
                // several steps per budget check (measured on C3: fcp 8 steps,
                // -7% then -3% vs 1; kNN 4 steps, 8 is +1.5%); the budget is
                // approximate by a few trips, which nothing depends on
                over = walk_budgeted(w, a, a.budget);
            }
        }
        w.finish(a, !over);  // over budget: the partial list stays as the overflow pass's bound
        if (over) {
            a.ovf_ids[atomicAdd(a.ovf_count, 1ull)] = uint32_t(w.qi);
            a.wave_state[w.qi] = make_int2(w.curr - 1, w.prev - 1);  // 0-based, for the resume pass
        }
    }
    if (active) add_totals<STATS>(a, w.cnt.steps, w.cnt.visited, w.cnt.processed);
    else add_totals<STATS>(a, 0, 0, 0);
    bt.end(a, 0);
}

// Continuation round (compaction rounds): one thread per id
// of the previous round's parked list, which is dense again, so a warp's 32
// lanes are 32 live walks instead of the few stragglers of a warp of the
// walk kernel.  Each resumes its (curr, prev) + partial list, walks at most
// `trips` more trips, and either finishes or parks again onto the next list
// (warp-aggregated append in lane order, so Morton neighbours stay
// together).  The grid is sized for the largest possible list; blocks past
// the device-side count exit at once.
// The same kernel is the resume pass: with resume_min > 0 it runs only when
// at least that many walks are parked (bulk long walks, e.g. 8-D), else the
// CTA pass takes them all (overflow.cuh reads the same count).
template <int D, int S, int KB, bool UNORDERED>
__global__ void __launch_bounds__(kWalkThreads, walk_min_blocks<D, KB>()) walk_round_kernel(const WalkArgs a) {
    const int64_t items = int64_t(*a.wave_n_in);
    if (a.resume_min > 0 && items < a.resume_min) return;
    const int64_t first = int64_t(blockIdx.x) * blockDim.x;
    if (first >= items) return;
    BlockTrace bt(a);
    const int64_t i = first + threadIdx.x;
    bool park = false;
    uint32_t qid = 0;
    if (i < items) {  // the walk state lives only inside this block (kept in registers)
        LaneWalk<D, S, KB, false, UNORDERED> w;
        qid = a.wave_in[i];
        w.resume(a, int32_t(qid));
        park = walk_budgeted(w, a, a.trips);
        w.finish(a, !park);
        if (park) a.wave_state[qid] = make_int2(w.curr - 1, w.prev - 1);
    }
    const unsigned lane = threadIdx.x & 31u;
    const unsigned mask = __ballot_sync(0xffffffffu, park);
    if (mask) {
        const unsigned leader = __ffs(mask) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(a.wave_n_out, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (park) a.wave_out[base + __popc(mask & ((1u << lane) - 1u))] = qid;
    }
    bt.end(a, 3);
}

// ---------------------------------------------------------------------------
// Generic walk for large k (> register buckets) and/or runtime dim > 8.
// The query's own output slot (k entries) holds a bounded max-heap of keys
// during the walk — the reference's KnnCandidates layout (traverse.hpp:
// 113-175) — and is heap-sorted in place at the end; no scratch memory.
// D == 0 means runtime dim (queries re-read through L1).
// ---------------------------------------------------------------------------
template <int D>
struct QueryRegs {
    float v[D];
};

template <int D, bool STATS, bool UNORDERED>
__global__ void __launch_bounds__(128) walk_heap_kernel(const WalkArgs a) {
    if (*a.bad != kNoBad) return;  // a rejected batch (batch.cpp:79) writes no slot
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool active = i < a.m;
    int64_t qi = 0;
    const int dim = D > 0 ? D : a.dim;
    const float* qp = nullptr;
    if (active) {
        qi = a.order ? int64_t(a.order[i]) : i;
        qp = a.queries + qi * dim;
        bool finite = true;
        for (int j = 0; j < dim; ++j) finite &= isfinite(__ldg(qp + j));
        if (!finite) {
            atomicMin(a.bad, (unsigned long long)(a.id_base + qi));
            active = false;
        }
    }
    Counters<STATS> cnt;
    if (active) {
        const int k = a.k;
        uint64_t* heap = reinterpret_cast<uint64_t*>(a.hits + qi * k);
        int count = 0;
        const float cap2 = a.cap2;
        const int32_t n = a.n;
        float r2 = cap2;
        int32_t curr = 0, prev = -1;
        while (n > 0) {
            const bool from_parent = prev < curr;
            const int d = depth_of(curr) % dim;
            const float* node = a.nodes + size_t(curr) * a.stride;
            if (from_parent) {
                float acc = 0.0f;
                for (int j = 0; j < dim; ++j) {
                    const float dj = __fsub_rn(__ldg(qp + j), __ldg(node + j));
                    acc = __fadd_rn(acc, __fmul_rn(dj, dj));
                }
                const uint64_t key = make_key(acc, curr);
                if (acc <= cap2) {
                    if (count < k) {  // push + sift up (traverse.hpp:123-126)
                        int c = count++;
                        while (c > 0) {
                            const int par = (c - 1) >> 1;
                            const uint64_t pk = heap[par];
                            if (pk >= key) break;
                            heap[c] = pk;
                            c = par;
                        }
                        heap[c] = key;
                    } else if (key < heap[0]) {  // replace top + sift down (128-131)
                        int c = 0;
                        while (true) {
                            const int l = 2 * c + 1, r = l + 1;
                            if (l >= k) break;
                            int m = l;
                            uint64_t mk = heap[l];
                            if (r < k) {
                                const uint64_t rk = heap[r];
                                if (rk > mk) {
                                    m = r;
                                    mk = rk;
                                }
                            }
                            if (mk <= key) break;
                            heap[c] = mk;
                            c = m;
                        }
                        heap[c] = key;
                    }
                    if (count == k) r2 = key_dist(heap[0]);
                }
            }
            cnt.step(1, 1, from_parent ? 1 : 0);
            const float sd = __fsub_rn(__ldg(qp + d), __ldg(node + d));
            const int cs = sd > 0.0f;
            const bool fir = __fmul_rn(sd, sd) <= r2;
            const int32_t parent = ((curr + 1) >> 1) - 1;
            int32_t next;
            if constexpr (!UNORDERED) {
                const int32_t close = 2 * curr + 1 + cs;
                const int32_t far = 2 * curr + 2 - cs;
                next = from_parent ? close : ((prev == close && fir) ? far : parent);
                if (next >= n) {
                    cnt.step(2, 1, 0);
                    next = (next == close && fir) ? far : parent;
                    if (next >= n) {
                        cnt.step(2, 1, 0);
                        next = parent;
                    }
                }
            } else {
                const int32_t left = 2 * curr + 1, right = 2 * curr + 2;
                const bool enter_left = !cs || fir, enter_right = cs || fir;
                if (from_parent)
                    next = enter_left ? left : (enter_right ? right : parent);
                else
                    next = (prev == left && enter_right) ? right : parent;
                if (next >= n) {
                    cnt.step(2, 1, 0);
                    next = (next == left && enter_right) ? right : parent;
                    if (next >= n) {
                        cnt.step(2, 1, 0);
                        next = parent;
                    }
                }
            }
            if (next < 0) break;
            prev = curr;
            curr = next;
        }
        // heap sort ascending in place (extract_sorted, traverse.cpp:18-23)
        for (int end = count - 1; end > 0; --end) {
            const uint64_t top = heap[0];
            const uint64_t x = heap[end];
            heap[end] = top;
            int c = 0;
            while (true) {
                const int l = 2 * c + 1, r = l + 1;
                if (l >= end) break;
                int m = l;
                uint64_t mk = heap[l];
                if (r < end) {
                    const uint64_t rk = heap[r];
                    if (rk > mk) {
                        m = r;
                        mk = rk;
                    }
                }
                if (mk <= x) break;
                heap[c] = mk;
                c = m;
            }
            heap[c] = x;
        }
        int2* out = reinterpret_cast<int2*>(heap);
        for (int j = 0; j < k; ++j) {
            const uint64_t key = j < count ? heap[j] : kEmptyKey;
            out[j] = make_int2(int32_t(uint32_t(key)), int32_t(uint32_t(key >> 32) - kKeyOfs));
        }
        a.counts[qi] = count;
        if constexpr (STATS) {
            if (a.per_query) {
                unsigned long long st = cnt.steps, v = cnt.visited;
                if (a.recursive_stats) {
                    st = cnt.processed + (st - v);
                    v = cnt.processed;
                }
                a.per_query[qi].steps = (int64_t)st;
                a.per_query[qi].nodes_visited = (int64_t)v;
                a.per_query[qi].nodes_processed = (int64_t)cnt.processed;
            }
        }
    }
    if (active) add_totals<STATS>(a, cnt.steps, cnt.visited, cnt.processed);
    else add_totals<STATS>(a, 0, 0, 0);
}

// Host-side dispatch (walk_dispatch.cu).  Returns the number of launches.
// phase 0 launches the walk, phase 1 the overflow pass (0 launches when the
// batch was not budgeted).
int launch_walk(const WalkArgs& a, int dim, int layout_stride, bool stats, bool unordered,
                int phase, cudaStream_t stream);


}  // namespace fkd
