// knobs.cpp — environment overrides of the launch/pipeline parameters
// (knobs.hpp lists them).  The only getenv calls in the library.
#include "knobs.hpp"

#include <algorithm>
#include <cstdlib>

namespace fkd {
namespace {

std::vector<int> parse_ints(const char* e) {
    std::vector<int> v;
    for (const char* p = e; *p;) {
        const int x = std::atoi(p);
        if (x > 0) v.push_back(x);
        while (*p && *p != ',') ++p;
        if (*p == ',') ++p;
    }
    return v;
}

}  // namespace

Knobs read_knobs() {
    Knobs k;
    if (const char* e = std::getenv("FKD_BUDGET")) k.budget = std::atoi(e);
    if (const char* e = std::getenv("FKD_ROUNDS_MIN_M")) k.rounds_min_m = std::atoll(e);
    if (const char* e = std::getenv("FKD_RESUME_MIN")) k.resume_min = std::atoll(e);
    if (const char* e = std::getenv("FKD_RESUME_TRIPS")) k.resume_trips = std::atoi(e);
    if (const char* e = std::getenv("FKD_RROUNDS_FCP")) {
        k.rounds_fcp = parse_ints(e);
        k.rounds_fcp_env = true;
    }
    if (const char* e = std::getenv("FKD_RROUNDS_KNN")) {
        k.rounds_knn_env = parse_ints(e);
        k.rounds_knn_all = true;
    }
    if (const char* e = std::getenv("FKD_CHUNK")) k.chunk = std::max<int64_t>(1024, std::atoll(e));
    if (const char* e = std::getenv("FKD_CHUNK_DIV")) k.chunk_div = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("FKD_STREAMS")) k.streams = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("FKD_RAMP_HEAD")) k.ramp_head = std::max(0, std::min(6, std::atoi(e)));
    if (const char* e = std::getenv("FKD_RAMP_TAIL")) k.ramp_tail = std::max(0, std::min(6, std::atoi(e)));
    if (const char* e = std::getenv("FKD_FIRST_BUDGET_DIV")) k.first_budget_div = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("FKD_FULL_STAGING")) k.full_staging = std::atoi(e) != 0;
    if (const char* e = std::getenv("FKD_PAGEABLE_STAGING")) k.pageable_staging = std::atoi(e) != 0;
    if (const char* e = std::getenv("FKD_HOST_RING")) k.host_ring = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("FKD_PIPE_TRACE")) k.pipe_trace = std::atoi(e) != 0;
    if (const char* e = std::getenv("FKD_HOST_COUNTS")) k.host_counts = std::atoi(e) != 0;
    if (const char* e = std::getenv("FKD_COPY_THREADS")) k.copy_threads = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("FKD_STREAM_COPY")) k.stream_copy = std::atoi(e) != 0;
    return k;
}

}  // namespace fkd
