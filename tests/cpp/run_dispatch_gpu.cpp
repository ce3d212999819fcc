// tests/cpp/run_dispatch_gpu.cpp — a C++ caller of the reference's hot-path API,
// linked ONLY against libperseus.so: sigsim::build_dispatch + sigsim::run_dispatch
// (GPU-backed) + the metrics trio, and the perseus::MoELayer RAII wrapper.
// Prints one JSON line per run_dispatch call; the Python test compares them
// with the reference's golden vectors (tests/golden/reference_vectors.json).
#include <cstdio>
#include <string>
#include <vector>

#include "perseus/moe_layer.hpp"
#include "sigsim/metrics.hpp"
#include "sigsim/protocols.hpp"
#include "sigsim/workload.hpp"

static int fails = 0;
#define EXPECT(c)                                                  \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                               \
        }                                                          \
    } while (0)

int main() {
    const auto qwen3 = *sigsim::model_preset("qwen3-30b");
    const std::uint64_t S = 4096, tile = 128 * 2048 * 2;
    for (int P : {2, 4}) {
        const auto wl = sigsim::build_dispatch(qwen3, sigsim::ClusterConfig{P, 1, 1}, S, 0.0, tile, 1);
        for (const auto& pr : {std::make_pair(std::string("vanilla"), sigsim::vanilla_protocol()),
                               std::make_pair(std::string("combined"), sigsim::combined_protocol(0)),
                               std::make_pair(std::string("decoupled8"), sigsim::decoupled_protocol(8))}) {
            const sigsim::RunTrace tr = sigsim::run_dispatch(pr.second, wl, sigsim::LatencyModel{}, 1, 0);
            const auto acc = sigsim::fence_accounting(tr);
            const auto viol = sigsim::verify_ordering(tr);
            const auto cons = sigsim::conservation_check(tr, wl);
            std::printf("{\"P\": %d, \"mode\": \"%s\", \"fence_count\": %lld, \"flagged_signal_count\": %lld, "
                        "\"violations\": %zu, \"conservation\": %d, \"heap_digest\": \"%016llx\", "
                        "\"workload_digest\": \"%016llx\", \"records\": %zu}\n",
                        P, pr.first.c_str(), (long long)acc.fence_count, (long long)acc.flagged_signal_count,
                        viol.size(), cons.pass ? 1 : 0, (unsigned long long)tr.heap_digest,
                        (unsigned long long)tr.workload_digest, tr.records.size());
            EXPECT(viol.empty());
            EXPECT(cons.pass);
        }
        // what the device cannot realise is a ConfigError, as in the reference
        bool threw = false;
        try {
            sigsim::run_dispatch(sigsim::decoupled_protocol(5), wl, sigsim::LatencyModel{}, 1);
        } catch (const sigsim::ConfigError&) {
            threw = true;
        }
        EXPECT(threw);
    }
    {
        bool threw = false;
        const auto wl = sigsim::build_dispatch(qwen3, sigsim::ClusterConfig{2, 1, 1}, S, 0.0, 0, 1);  // per-expert payloads
        try {
            sigsim::run_dispatch(sigsim::vanilla_protocol(), wl, sigsim::LatencyModel{}, 1);
        } catch (const sigsim::ConfigError&) {
            threw = true;
        }
        EXPECT(threw);
        sigsim::LatencyModel bad;
        bad.bandwidth_bytes_per_ns = 0.0;
        threw = false;
        try {
            sigsim::run_dispatch(sigsim::vanilla_protocol(), wl, bad, 1);
        } catch (const sigsim::ConfigError&) {
            threw = true;
        }
        EXPECT(threw);
    }
    // the RAII wrapper: one rank, host API end to end; config errors rethrown
    {
        const sigsim::ModelConfig tiny{"tiny", 256, 512, 8, 2, 0.0};
        perseus::MoELayer layer(tiny, 128);
        std::vector<std::uint16_t> x(128 * 256, 0x3f80);  // bf16 1.0
        const auto y = layer.forward_host(x);
        const auto y2 = layer.forward_host(x);
        EXPECT(y == y2);
        const auto c = layer.counters();
        EXPECT(c.wait_timeouts == 0 && c.errors == 0 && c.epoch == 2);
        bool threw = false;
        try {
            perseus::MoELayer bad(sigsim::ModelConfig{"bad", 300, 512, 8, 2, 0.0}, 128);  // H % 256 != 0
        } catch (const sigsim::ConfigError&) {
            threw = true;
        }
        EXPECT(threw);
    }
    std::printf(fails ? "run_dispatch_gpu: FAIL\n" : "run_dispatch_gpu: pass\n");
    return fails ? 1 : 0;
}
