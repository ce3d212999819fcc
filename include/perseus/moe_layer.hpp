// include/perseus/moe_layer.hpp — header-only C++ face of one expert-parallel
// layer rank over the C ABI (include/perseus.h), for C++ callers of the
// reference's operator API ("moe_layer" with route / dispatch /
// expert FFN / combine / forward / fence accounting behind a thin C ABI).
//
// RAII: the handle owns the device layer (weights, symmetric buffers, peer
// mappings) and destroys it.  Failures come back as the reference's exception
// types (sim.hpp:17-28): status 1 -> sigsim::ConfigError, 3 -> sigsim::ModelError
// (CUDA errors, signal-wait timeouts), 2 -> perseus::VerificationError (a
// verification / ordering failure; the reference CLI's exit code 2,
// tools/main.cpp:6).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "perseus.h"
#include "sigsim/protocols.hpp"
#include "sigsim/workload.hpp"

namespace perseus {

struct VerificationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == PERSEUS_OK) return;
    const std::string msg = perseus_last_error();
    if (rc == PERSEUS_ERR_CONFIG) throw sigsim::ConfigError(msg);
    if (rc == PERSEUS_ERR_VERIFY) throw VerificationError(msg);
    throw sigsim::ModelError(msg);
}

// The device signalling variant a reference protocol selects (protocols.hpp:13-37).
inline int device_signaling(const sigsim::ProtocolConfig& p) {
    if (p.suppress_fences) return PERSEUS_SIGNAL_NONE;
    return p.signaling == sigsim::Signaling::Coupled ? PERSEUS_SIGNAL_COUPLED : PERSEUS_SIGNAL_DECOUPLED;
}

enum class Routing : int { Balanced = PERSEUS_ROUTE_BALANCED, Zipf = PERSEUS_ROUTE_ZIPF, Gate = PERSEUS_ROUTE_GATE };

struct LayerOptions {
    Routing routing = Routing::Balanced;
    double skew = 0.0;                                              // Zipf exponent
    std::uint64_t seed = 1;                                         // workload seed (config.hpp:36)
    sigsim::ProtocolConfig protocol = sigsim::combined_protocol(0);  // Perseus: per-destination groups
    bool synthetic_weights = true;
    int flags = 0;  // extra PERSEUS_F_*
};

class MoELayer {
public:
    MoELayer(const sigsim::ModelConfig& model, std::uint64_t tokens_per_pe, int rank = 0, int world = 1,
             int device = 0, const LayerOptions& opt = LayerOptions()) {
        perseus_layer_config c{};
        c.hidden_dim = model.hidden_dim;
        c.intermediate_dim = model.intermediate_dim;
        c.experts = model.experts;
        c.top_k = model.top_k;
        c.tokens_per_pe = tokens_per_pe;
        c.routing = static_cast<int>(opt.routing);
        c.skew = opt.skew;
        c.seed = opt.seed;
        c.signaling = device_signaling(opt.protocol);
        c.group_size = opt.protocol.group_size;
        c.flags = opt.flags | (opt.synthetic_weights ? PERSEUS_F_SYNTH_WEIGHTS : 0);
        check(perseus_layer_create(&c, rank, world, device, &h_));
        tokens_ = tokens_per_pe;
        hidden_ = model.hidden_dim;
    }
    ~MoELayer() {
        if (h_) perseus_layer_destroy(h_);
    }
    MoELayer(const MoELayer&) = delete;
    MoELayer& operator=(const MoELayer&) = delete;
    MoELayer(MoELayer&& o) noexcept : h_(std::exchange(o.h_, nullptr)), tokens_(o.tokens_), hidden_(o.hidden_) {}
    MoELayer& operator=(MoELayer&& o) noexcept {
        if (this != &o) {
            if (h_) perseus_layer_destroy(h_);
            h_ = std::exchange(o.h_, nullptr);
            tokens_ = o.tokens_;
            hidden_ = o.hidden_;
        }
        return *this;
    }

    perseus_layer* handle() const { return h_; }

    // -- bootstrap: symmetric buffers of every rank (one process per GPU: IPC handles
    //    exchanged by the caller; several ranks in one process: raw pointers) --
    std::vector<std::uint8_t> ipc_handle() const {
        size_t n = 0;
        check(perseus_layer_ipc_export(h_, nullptr, 0, &n));
        std::vector<std::uint8_t> b(n);
        check(perseus_layer_ipc_export(h_, b.data(), b.size(), &n));
        return b;
    }
    void connect(const std::vector<std::vector<std::uint8_t>>& handles_by_rank) {
        std::vector<std::uint8_t> all;
        for (const auto& b : handles_by_rank) all.insert(all.end(), b.begin(), b.end());
        check(perseus_layer_ipc_import(h_, all.data(), handles_by_rank.empty() ? 0 : handles_by_rank[0].size()));
    }
    static void connect_local(const std::vector<MoELayer*>& ranks) {
        std::vector<perseus_layer*> hs;
        for (MoELayer* l : ranks) hs.push_back(l->h_);
        check(perseus_layer_connect_local(hs.data(), int(hs.size())));
    }

    // -- weights / inputs (device pointers, bf16) --
    void set_weights(const void* wg, const void* w1, const void* w2, void* stream = nullptr) {
        check(perseus_layer_set_weights(h_, wg, w1, w2, stream));
    }
    void fill_synthetic_x(void* x, std::uint64_t seed, void* stream = nullptr) {
        check(perseus_fill_synthetic_x(h_, x, seed, stream));
    }

    // -- the hot path: gate/route -> dispatch -> expert FFN -> combine --
    void forward(const void* x, void* out, void* stream = nullptr) { check(perseus_layer_forward(h_, x, out, stream)); }
    // host bf16 bits [S][H] in and out (copies included)
    std::vector<std::uint16_t> forward_host(const std::vector<std::uint16_t>& x_host) {
        std::vector<std::uint16_t> out(x_host.size());
        check(perseus_layer_forward_host(h_, x_host.data(), out.data(), nullptr));
        return out;
    }

    // -- evidence --
    perseus_counters counters() const {
        perseus_counters c{};
        check(perseus_layer_counters(h_, &c));
        return c;
    }
    std::int64_t group_size() const {
        std::int64_t g = 0;
        check(perseus_layer_group_size(h_, &g));
        return g;
    }
    // the remote transfer tiles this rank realised in its last forward (the
    // reference's TransferSpec, workload.hpp:42-49) and the flag ids set here
    std::vector<sigsim::TransferSpec> layout(std::vector<std::int64_t>* flags_seen = nullptr) const {
        size_t n = 0, nf = 0;
        check(perseus_layer_read_layout(h_, nullptr, 0, &n, nullptr, 0, &nf));
        std::vector<perseus_transfer> t(n);
        std::vector<std::int64_t> f(nf);
        check(perseus_layer_read_layout(h_, t.data(), n, &n, f.data(), nf, &nf));
        std::vector<sigsim::TransferSpec> out;
        for (const auto& x : t) out.push_back(sigsim::TransferSpec{x.src_pe, x.dst_pe, x.expert, x.bytes, x.tile_id, x.heap_offset});
        if (flags_seen) *flags_seen = f;
        return out;
    }
    std::uint64_t tokens_per_pe() const { return tokens_; }
    std::int64_t hidden_dim() const { return hidden_; }

private:
    perseus_layer* h_ = nullptr;
    std::uint64_t tokens_ = 0;
    std::int64_t hidden_ = 0;
};

}  // namespace perseus
