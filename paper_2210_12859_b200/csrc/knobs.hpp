// knobs.hpp — the library's launch/pipeline parameters in one place.
//
// Defaults are the measured best; no value here changes a
// result, only how the work is scheduled.  The parity tests override a few of
// them to force rare paths (tiny step budgets, every resume/round/CTA-pass
// combination, odd chunkings), so those are read from the environment — once
// per API call, here and nowhere else:
//
//   FKD_BUDGET           first walk's loop trips before a query parks (<0 per kind, 0 off)
//   FKD_RROUNDS_FCP      continuation-round trips for fcp, "t1,t2,.." ("0": none)
//   FKD_RROUNDS_KNN      continuation-round trips for every kNN bucket
//   FKD_ROUNDS_MIN_M     batch size from which 8-slot lists take rounds and fcp a third round (2^22)
//   FKD_RESUME_MIN       parked walks that select the plain-grid resume pass (0: SMs x 64)
//   FKD_RESUME_TRIPS     trips the resume pass adds before the CTA pass (0: per kind, <0 unbounded)
//   FKD_CHUNK            host path: uniform chunk size instead of the graduated schedule
//   FKD_CHUNK_DIV        host path: middle chunk = shard / DIV (0: 4 for k = 1, else 8)
//   FKD_STREAMS          host path: slot streams per device (4)
//   FKD_RAMP_HEAD/TAIL   host path: ramp depths of the chunk schedule (2 / 2)
//   FKD_FIRST_BUDGET_DIV host path: first chunk's budget divisor (1)
//   FKD_FULL_STAGING     host path: 0 forces the device-side ring staging
//   FKD_PAGEABLE_STAGING host path: 0 hands pageable caller buffers to cudaMemcpyAsync
//   FKD_HOST_RING        host path: pinned staging slots per direction per device (4)
//   FKD_PIPE_TRACE       host path: 1 prints each job's H2D / walk / D2H end times (stderr)
//
// Experiments that were measured and settled are compile-time constants
// (store layout, node shift, carveout, Morton bits, sort thresholds, CTA-pass
// residency, register-list cap) — see the #defines at their use sites.
#pragma once

#include <cstdint>
#include <vector>

namespace fkd {

struct Knobs {
    // walk schedule
    int budget = -1;
    std::vector<int> rounds_fcp{112, 224, 448};
    std::vector<int> rounds_fcp_small{112, 224};
    std::vector<int> rounds_knn4{256, 512};
    std::vector<int> rounds_knn8{384, 768, 1536};
    bool rounds_fcp_env = false;  // FKD_RROUNDS_FCP given: every batch size
    std::vector<int> rounds_knn_env;
    bool rounds_knn_all = false;  // FKD_RROUNDS_KNN given: every kNN bucket
    int64_t rounds_min_m = int64_t(1) << 22;
    int64_t resume_min = 0;
    int resume_trips = 0;
    // host pipeline
    int64_t chunk = 0;  // 0: graduated schedule
    int chunk_div = 0;  // 0: per kind (chunk_div_for)
    int streams = 4;
    int ramp_head = 2, ramp_tail = 2;
    int first_budget_div = 1;
    bool full_staging = true;
    bool pageable_staging = true;
    int host_ring = 4;
    bool pipe_trace = false;
    // host pipeline: an unbounded-radius batch's counts (min(k, n) for every
    // query) are written on the host and checked on the device instead of
    // copied (FKD_HOST_COUNTS=0 copies them)
    bool host_counts = true;
    // threads of the host copy pool (0: hardware threads, at most 16); read once
    int copy_threads = 0;
    // host copies with streaming stores (FKD_STREAM_COPY=0: memcpy); read once
    bool stream_copy = true;
};

// A snapshot of the environment overrides on top of the defaults.
Knobs read_knobs();

}  // namespace fkd
