// include/sigsim/metrics.hpp — drop-in fence accounting and checkers
// (proj/include/sigsim/metrics.hpp:13-78), evaluated over DEVICE evidence.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "sigsim/trace.hpp"
#include "sigsim/workload.hpp"

namespace sigsim {

struct FenceAccounting {
    std::int64_t fence_count = 0;
    std::int64_t proxy_stop_episodes = 0;  // always 0 on B200: no proxy
    TimeNs proxy_blocked_total = 0;
    std::vector<TimeNs> per_fence;
    std::int64_t nic_stall_episodes = 0;   // always 0 on B200: no NIC queue pairs
    TimeNs nic_stall_total = 0;
    std::int64_t flagged_signal_count = 0;
};
FenceAccounting fence_accounting(const RunTrace& trace);

struct OrderingViolation {
    std::int64_t tile_id = -1;
    std::uint32_t src_pe = 0;
    std::uint32_t dst_pe = 0;
    TimeNs signal_visible = 0;
    TimeNs put_completion = 0;
};
std::vector<OrderingViolation> verify_ordering(const RunTrace& trace);

struct ConservationReport {
    bool pass = true;
    std::vector<std::string> failures;
    void fail(std::string msg) { pass = false; failures.push_back(std::move(msg)); }
};
ConservationReport conservation_check(const RunTrace& trace, const DispatchWorkload& workload);

struct AlphaBetaFit {
    double alpha_ns = 0.0;
    double beta_ns_per_byte = 0.0;
    double r_squared = 0.0;
};
AlphaBetaFit fit_alpha_beta(const std::vector<std::pair<double, double>>& points);

}  // namespace sigsim
