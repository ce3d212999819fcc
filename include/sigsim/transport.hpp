// include/sigsim/transport.hpp — drop-in subset of proj/include/sigsim/transport.hpp.
//
// Only the LatencyModel (transport.hpp:49-81) crosses the hot-path API: it is an
// argument of run_dispatch (protocols.hpp:62-64).  The reference uses it to time
// a simulated proxy FIFO, NIC queue pairs and NVLink; on B200 the dispatch runs
// in real time over NVLink one-sided stores, so the GPU-backed run_dispatch only
// validates it (same ConfigError rules as transport.cpp:15-24).  The proxy /
// NIC / QP engine itself is out of scope.
#pragma once

#include <cstdint>

#include "sigsim/sim.hpp"

namespace sigsim {

struct LatencyModel {
    TimeNs base_rtt_ns = 400;
    double bandwidth_bytes_per_ns = 25.0;
    double completion_tail_coeff = 1.0;
    TimeNs per_request_nic_service_ns = 100;
    TimeNs proxy_poll_quantum_ns = 500;
    TimeNs issue_cost_ns = 200;
    TimeNs issue_jitter_ns = 0;
    TimeNs gpu_direct_issue_cost_ns = 400;
    TimeNs nvlink_latency_ns = 700;
    std::uint64_t signal_bytes = 8;
    int processors_per_pe = 8;
    double slot_tflops = 200.0;

    void validate() const;
};

}  // namespace sigsim
