// A C++ consumer of the drop-in headers (include/sigsim/*.hpp) linked against
// libperseus.so, as a reference user's code would be: the reference's own
// known answers (test_workload.cpp, test_protocols.cpp, SURVEY §8c golden
// values) through the B200 library's planner.  Exit code 0 = all pass.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "sigsim/metrics.hpp"
#include "sigsim/protocols.hpp"
#include "sigsim/trace.hpp"
#include "sigsim/workload.hpp"

static int failures = 0;
#define EXPECT(cond)                                                   \
    do {                                                               \
        if (!(cond)) {                                                 \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                \
        }                                                              \
    } while (0)

int main() {
    // remote_transfer_count / message_size (test_workload.cpp:9-20)
    EXPECT(sigsim::remote_transfer_count(128, 16, 4) == 96);
    EXPECT(sigsim::remote_transfer_count(128, 8, 1) == 112);
    EXPECT(sigsim::message_size(4096, 8, 128, 2048) == 1048576ull);
    // presets
    auto q = sigsim::model_preset("qwen3-30b");
    EXPECT(q.has_value() && q->hidden_dim == 2048 && q->experts == 128 && q->top_k == 8);
    // Qwen3 P=8 S=4096 per-expert payloads: workload digest (SURVEY §8c golden)
    auto wl = sigsim::build_dispatch(*q, sigsim::ClusterConfig{8, 1, 1}, 4096, 0.0, 0, 1);
    char dig[32];
    std::snprintf(dig, sizeof dig, "%016llx", (unsigned long long)wl.digest());
    EXPECT(std::string(dig) == "fcd7d15946dfc87c");
    EXPECT(wl.remote_transfers.size() == 896);
    // 128-row tiles: 1792 tiles (224 per PE); fences per PE: per tile 224, per destination 7
    auto wl_t = sigsim::build_dispatch(*q, sigsim::ClusterConfig{8, 1, 1}, 4096, 0.0, 128 * 2048 * 2, 1);
    EXPECT(wl_t.remote_transfers.size() == 1792);
    EXPECT(sigsim::expected_fences(sigsim::vanilla_protocol(), wl_t, 0) == 224);
    EXPECT(sigsim::expected_fences(sigsim::combined_protocol(0), wl_t, 0) == 7);
    // assign_groups: a group size that does not divide the PE's transfers is a ConfigError
    std::vector<sigsim::TransferSpec> own;
    for (const auto& t : wl.remote_transfers)
        if (t.src_pe == 0) own.push_back(t);
    bool threw = false;
    try {
        sigsim::assign_groups(own, 5);
    } catch (const sigsim::ConfigError&) {
        threw = true;
    }
    EXPECT(threw);
    EXPECT(sigsim::assign_groups(own, 0).size() == 7);
    // fit_alpha_beta on an exact line
    auto f = sigsim::fit_alpha_beta({{1.0, 12.0}, {2.0, 14.0}, {4.0, 18.0}});
    EXPECT(f.alpha_ns > 9.999 && f.alpha_ns < 10.001 && f.beta_ns_per_byte > 1.999 && f.beta_ns_per_byte < 2.001);
    // the GPU-backed run_dispatch (protocols.hpp:62-64) rejects, before touching a
    // device, what the reference rejects and what the device cannot realise
    auto throws_config = [](auto&& fn) {
        try {
            fn();
        } catch (const sigsim::ConfigError&) {
            return true;
        } catch (...) {
            return false;
        }
        return false;
    };
    sigsim::LatencyModel bad_lat;
    bad_lat.proxy_poll_quantum_ns = 0;  // transport.cpp:15-24
    EXPECT(throws_config([&] { bad_lat.validate(); }));
    EXPECT(throws_config([&] { sigsim::run_dispatch(sigsim::vanilla_protocol(), wl_t, bad_lat, 1); }));
    EXPECT(throws_config([&] { sigsim::run_dispatch(sigsim::decoupled_protocol(5), wl_t, sigsim::LatencyModel{}, 1); }));
    EXPECT(throws_config([&] { sigsim::run_dispatch(sigsim::vanilla_protocol(), wl, sigsim::LatencyModel{}, 1); }));
    // FNV-1a (trace.cpp:53-62)
    EXPECT(sigsim::fnv1a64("", 0) == 0xcbf29ce484222325ULL);
    std::printf("dropin_kats: %s (%d failures)\n", failures ? "FAIL" : "pass", failures);
    return failures ? 1 : 0;
}
