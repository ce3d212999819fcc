// planner.cpp — host half of the drop-in sigsim API (include/sigsim/*.hpp)
// and the planner entry points of the C ABI (include/perseus.h).
//
// Everything here is host-side layout/bookkeeping that the reference also does
// on the host: geometry, routing draws for the reference's routing modes, the
// transfer/heap layout, signal groups, digests and the accounting checkers.
// The per-forward work (routing of real tokens, permutation, puts, fences,
// flags, FFN, combine) runs on the device (kernels.cu, gemm.cu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <tuple>

#include "perseus.h"
#include "perseus_internal.h"
#include "sigsim/metrics.hpp"
#include "sigsim/protocols.hpp"
#include "sigsim/trace.hpp"
#include "sigsim/workload.hpp"

namespace sigsim {

// ---------------------------------------------------------------- trace ----
const char* to_string(ReqKind k) {
    static const char* n[] = {"put", "signal", "fence"};
    return unsigned(k) < 3 ? n[unsigned(k)] : "?";
}
const char* to_string(TraceKind k) {
    static const char* n[] = {"submit", "nic_service_start", "completion", "signal_visible",
                              "compute_start", "compute_end", "proxy_block_begin",
                              "proxy_block_end", "nic_block_begin", "nic_block_end"};
    return unsigned(k) < 10 ? n[unsigned(k)] : "?";
}

std::uint64_t fnv1a64(const void* data, std::size_t len, std::uint64_t h) {
    auto* b = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < len; ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
    return h;
}
std::uint64_t fnv1a64(const std::string& s, std::uint64_t h) { return fnv1a64(s.data(), s.size(), h); }

std::string serialize_trace(const RunTrace& t) {
    std::string out;
    char line[256];
    std::snprintf(line, sizeof line,
                  "# trace v1 config=%016llx workload=%016llx seed=%llu heap=%016llx makespan=%lld\n",
                  (unsigned long long)t.config_hash, (unsigned long long)t.workload_digest,
                  (unsigned long long)t.seed, (unsigned long long)t.heap_digest,
                  (long long)t.makespan);
    out += line;
    for (const auto& r : t.records) {
        std::snprintf(line, sizeof line, "%lld %u %s %s %u %u %llu %d %d %lld %lld %llu\n",
                      (long long)r.time, r.pe, to_string(r.kind), to_string(r.req_kind), r.src_pe,
                      r.dst_pe, (unsigned long long)r.size, int(r.fence_flag), r.qp,
                      (long long)r.group_id, (long long)r.tile_id,
                      (unsigned long long)r.submit_seq);
        out += line;
    }
    return out;
}

// ------------------------------------------------------------- workload ----
void ModelConfig::validate() const {
    if (hidden_dim <= 0 || intermediate_dim <= 0 || experts <= 0 || top_k <= 0)
        throw ConfigError("model '" + name + "': all dimensions must be positive");
    if (top_k > experts) throw ConfigError("model '" + name + "': top_k exceeds expert count");
}

// transport.cpp:15-24 — the GPU-backed run_dispatch validates the simulated
// fabric's parameters it is handed, with the reference's messages
void LatencyModel::validate() const {
    if (base_rtt_ns < 0 || per_request_nic_service_ns < 0 || issue_cost_ns < 0 || issue_jitter_ns < 0 ||
        gpu_direct_issue_cost_ns < 0 || nvlink_latency_ns < 0)
        throw ConfigError("latency model: negative time parameter");
    if (bandwidth_bytes_per_ns <= 0.0) throw ConfigError("latency model: bandwidth must be > 0");
    if (completion_tail_coeff < 0.0) throw ConfigError("latency model: tail coefficient must be >= 0");
    if (proxy_poll_quantum_ns <= 0) throw ConfigError("latency model: poll quantum must be > 0");
    if (processors_per_pe < 1) throw ConfigError("latency model: processors_per_pe must be >= 1");
}

void ClusterConfig::validate() const {
    if (nodes < 1 || gpus_per_node < 1)
        throw ConfigError("cluster: nodes and gpus_per_node must be >= 1");
    if (num_qps < 1) throw ConfigError("cluster: num_qps must be >= 1");
}

std::optional<ModelConfig> model_preset(const std::string& name) {
    // published geometries (workload.cpp:25-33)
    static const std::map<std::string, ModelConfig> presets = {
        {"qwen3-30b", {"qwen3-30b", 2048, 768, 128, 8, 4.6}},
        {"gpt-oss-120b", {"gpt-oss-120b", 2880, 2880, 128, 4, 17.3}},
        {"deepseek-v3", {"deepseek-v3", 7168, 2048, 256, 8, 0.0}},
        {"llama4-scout", {"llama4-scout", 5120, 8192, 16, 1, 49.2}},
    };
    auto it = presets.find(name);
    if (it == presets.end()) return std::nullopt;
    return it->second;
}

std::vector<std::string> model_preset_names() {
    return {"qwen3-30b", "gpt-oss-120b", "deepseek-v3", "llama4-scout"};
}

std::int64_t remote_transfer_count(std::int64_t E, std::int64_t P, std::int64_t P_local) {
    if (P <= 0 || E <= 0) throw ConfigError("remote_transfer_count: non-positive config");
    if (E % P)
        throw ConfigError("remote_transfer_count: experts (" + std::to_string(E) +
                          ") not divisible by PEs (" + std::to_string(P) + ")");
    if (P_local > P) throw ConfigError("remote_transfer_count: pes_per_node exceeds pes");
    return (P - P_local) * (E / P);
}

std::uint64_t message_size(std::uint64_t S, std::int64_t k, std::int64_t E, std::int64_t H) {
    if (S == 0) return 0;
    return (S * std::uint64_t(k) / std::uint64_t(E)) * std::uint64_t(H) * 2;
}

std::vector<std::uint64_t> zipf_route_ids(std::uint64_t S, std::int64_t E, double s,
                                          std::int64_t k, std::uint64_t seed,
                                          std::vector<std::int32_t>* ids) {
    if (s < 0.0) throw ConfigError("zipf_route: exponent must be >= 0");
    if (k > E) throw ConfigError("zipf_route: top_k exceeds expert count");
    SeededRng rng(seed);
    // popularity rank -> expert: Fisher-Yates driven by the same stream
    std::vector<std::int64_t> perm(static_cast<std::size_t>(E));
    std::iota(perm.begin(), perm.end(), std::int64_t{0});
    for (std::int64_t n = E; n > 1; --n)
        std::swap(perm[std::size_t(n - 1)], perm[rng.next_below(std::uint64_t(n))]);
    // normalised CDF of r^-s
    std::vector<double> cdf(static_cast<std::size_t>(E));
    double total = 0.0;
    for (std::int64_t r = 0; r < E; ++r) cdf[std::size_t(r)] = (total += std::pow(double(r + 1), -s));
    for (double& c : cdf) c /= total;

    std::vector<std::uint64_t> counts(static_cast<std::size_t>(E), 0);
    if (ids) ids->assign(S * std::uint64_t(k), 0);
    std::vector<std::int64_t> picked;
    picked.reserve(std::size_t(k));
    for (std::uint64_t t = 0; t < S; ++t) {
        picked.clear();
        while (picked.size() < std::size_t(k)) {
            const double u = rng.next_double();
            std::size_t r = std::size_t(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
            const std::int64_t ex = perm[std::min(r, std::size_t(E - 1))];
            if (std::find(picked.begin(), picked.end(), ex) != picked.end()) continue;
            if (ids) (*ids)[t * std::uint64_t(k) + picked.size()] = std::int32_t(ex);
            picked.push_back(ex);
            ++counts[std::size_t(ex)];
        }
    }
    return counts;
}

std::vector<std::uint64_t> zipf_route(std::uint64_t S, std::int64_t E, double s, std::int64_t k,
                                      std::uint64_t seed) {
    return zipf_route_ids(S, E, s, k, seed, nullptr);
}

std::uint64_t DispatchWorkload::total_remote_bytes() const {
    std::uint64_t b = 0;
    for (const auto& t : remote_transfers) b += t.bytes;
    return b;
}

std::uint64_t DispatchWorkload::digest() const {
    std::uint64_t h = 0xcbf29ce484222325ULL;
    auto put = [&](std::uint64_t v) { h = fnv1a64(&v, sizeof v, h); };
    put(std::uint64_t(cluster.nodes));
    put(std::uint64_t(cluster.gpus_per_node));
    put(tokens_per_pe);
    put(std::uint64_t(skew * 1e6));
    put(tile_bytes);
    for (const auto& t : remote_transfers) { put(t.src_pe); put(t.dst_pe); put(std::uint64_t(t.expert)); put(t.bytes); }
    for (const auto& t : local_transfers) { put(t.src_pe); put(t.dst_pe); put(t.bytes); }
    return h;
}

DispatchWorkload build_dispatch_from_counts(const ModelConfig& model, const ClusterConfig& cluster,
                                            std::uint64_t tokens, double skew,
                                            std::uint64_t tile_bytes, std::uint64_t seed,
                                            const std::vector<std::uint64_t>& counts) {
    model.validate();
    cluster.validate();
    const std::int64_t P = cluster.total_pes(), E = model.experts;
    if (E % P)
        throw ConfigError("build_dispatch: experts (" + std::to_string(E) +
                          ") not divisible by PEs (" + std::to_string(P) + ")");
    if (counts.size() != std::size_t(P * E)) throw ConfigError("build_dispatch: count table size");
    DispatchWorkload wl;
    wl.model = model;
    wl.cluster = cluster;
    wl.tokens_per_pe = tokens;
    wl.skew = skew;
    wl.seed = seed;
    wl.tile_bytes = tile_bytes;
    const std::uint64_t row_bytes = std::uint64_t(model.hidden_dim) * 2;
    std::vector<std::uint64_t> cursor(std::size_t(P), 0);  // per-destination heap cursor
    std::int64_t tile = 0;
    const std::uint32_t gpn = std::uint32_t(cluster.gpus_per_node);
    for (std::int64_t s = 0; s < P; ++s) {
        for (std::int64_t e = 0; e < E; ++e) {
            const std::uint32_t d = std::uint32_t(e % P);  // round-robin placement
            const std::uint64_t bytes = counts[std::size_t(s * E + e)] * row_bytes;
            if (std::int64_t(d) == s || bytes == 0) continue;
            auto& list = (d / gpn == std::uint32_t(s) / gpn) ? wl.local_transfers : wl.remote_transfers;
            const std::uint64_t step = tile_bytes ? tile_bytes : bytes;
            for (std::uint64_t off = 0; off < bytes; off += step) {
                TransferSpec t;
                t.src_pe = std::uint32_t(s);
                t.dst_pe = d;
                t.expert = e;
                t.bytes = std::min(step, bytes - off);
                t.tile_id = tile++;
                t.heap_offset = cursor[d];
                cursor[d] += t.bytes;
                list.push_back(t);
            }
        }
    }
    auto key = [](const TransferSpec& t) { return std::make_tuple(t.src_pe, t.dst_pe, t.expert, t.tile_id); };
    auto less = [&](const TransferSpec& a, const TransferSpec& b) { return key(a) < key(b); };
    std::sort(wl.remote_transfers.begin(), wl.remote_transfers.end(), less);
    std::sort(wl.local_transfers.begin(), wl.local_transfers.end(), less);
    return wl;
}

DispatchWorkload build_dispatch(const ModelConfig& model, const ClusterConfig& cluster,
                                std::uint64_t tokens, double skew, std::uint64_t tile_bytes,
                                std::uint64_t seed) {
    model.validate();
    cluster.validate();
    const std::int64_t P = cluster.total_pes(), E = model.experts;
    if (E % P)
        throw ConfigError("build_dispatch: experts (" + std::to_string(E) +
                          ") not divisible by PEs (" + std::to_string(P) + ")");
    if (skew == 0.0 && tokens > 0 && (tokens * std::uint64_t(model.top_k)) % std::uint64_t(E))
        throw ConfigError("build_dispatch: balanced routing needs E | S*k");
    std::vector<std::uint64_t> counts(std::size_t(P * E));
    for (std::int64_t s = 0; s < P; ++s) {
        std::vector<std::uint64_t> c;
        if (skew > 0.0)
            c = zipf_route(tokens, E, skew, model.top_k,
                           seed ^ (0x9E3779B97F4A7C15ULL * std::uint64_t(s + 1)));
        else
            c.assign(std::size_t(E), tokens * std::uint64_t(model.top_k) / std::uint64_t(E));
        std::copy(c.begin(), c.end(), counts.begin() + s * E);
    }
    return build_dispatch_from_counts(model, cluster, tokens, skew, tile_bytes, seed, counts);
}

// ------------------------------------------------------------ protocols ----
const char* to_string(Signaling s) { return s == Signaling::Coupled ? "coupled" : "decoupled"; }

std::string ProtocolConfig::mode_name() const {
    if (transport == TransportPath::GpuDirect)
        return signaling == Signaling::Coupled ? "gpu_direct" : "gpu_direct_decoupled";
    const bool nic = ordering == OrderingMode::NicFence;
    if (signaling == Signaling::Coupled) return nic ? "nic_ordering" : "vanilla";
    return nic ? "combined" : "decoupled";
}

ProtocolConfig vanilla_protocol() { return {}; }
ProtocolConfig decoupled_protocol(std::int64_t gs) {
    ProtocolConfig p;
    p.signaling = Signaling::Decoupled;
    p.group_size = gs;
    return p;
}
ProtocolConfig nic_ordering_protocol() {
    ProtocolConfig p;
    p.ordering = OrderingMode::NicFence;
    return p;
}
ProtocolConfig combined_protocol(std::int64_t gs) {
    ProtocolConfig p = decoupled_protocol(gs);
    p.ordering = OrderingMode::NicFence;
    return p;
}
ProtocolConfig gpu_direct_protocol(Signaling s) {
    ProtocolConfig p;
    p.signaling = s;
    p.transport = TransportPath::GpuDirect;
    return p;
}

std::vector<SignalGroup> assign_groups(const std::vector<TransferSpec>& v, std::int64_t gs) {
    std::vector<std::size_t> ord(v.size());
    std::iota(ord.begin(), ord.end(), std::size_t{0});
    std::sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) {
        return std::make_tuple(v[a].dst_pe, v[a].expert, v[a].tile_id) <
               std::make_tuple(v[b].dst_pe, v[b].expert, v[b].tile_id);
    });
    std::vector<SignalGroup> out;
    if (gs == 0) {
        for (std::size_t idx : ord) {
            if (out.empty() || v[out.back().members.front()].dst_pe != v[idx].dst_pe) {
                out.emplace_back();
                out.back().group_id = std::int64_t(out.size() - 1);
            }
            out.back().members.push_back(idx);
        }
    } else {
        if (gs < 0 || v.size() % std::size_t(gs))
            throw ConfigError("assign_groups: group size " + std::to_string(gs) +
                              " does not divide transfer count " + std::to_string(v.size()));
        out.resize(v.size() / std::size_t(gs));
        for (std::size_t p = 0; p < ord.size(); ++p) out[p / std::size_t(gs)].members.push_back(ord[p]);
        for (std::size_t g = 0; g < out.size(); ++g) out[g].group_id = std::int64_t(g);
    }
    for (auto& g : out) {
        g.leader = g.members.front();
        g.target = std::int64_t(g.members.size());
    }
    return out;
}

std::int64_t expected_fences(const ProtocolConfig& p, const DispatchWorkload& wl, std::uint32_t src) {
    if (p.transport == TransportPath::GpuDirect || p.suppress_fences) return 0;
    std::vector<TransferSpec> own;
    for (const auto& t : wl.remote_transfers)
        if (t.src_pe == src) own.push_back(t);
    if (p.signaling == Signaling::Coupled) return std::int64_t(own.size());
    return own.empty() ? 0 : std::int64_t(assign_groups(own, p.group_size).size());
}

// -------------------------------------------------------------- metrics ----
FenceAccounting fence_accounting(const RunTrace& trace) {
    FenceAccounting acc;
    std::map<std::uint32_t, TimeNs> proxy_open;
    std::map<std::tuple<std::uint32_t, std::uint32_t, int>, TimeNs> nic_open;
    for (const auto& r : trace.records) {
        if (r.kind == TraceKind::Submit && r.req_kind == ReqKind::FenceMarker) ++acc.fence_count;
        if (r.kind == TraceKind::NicServiceStart && r.req_kind == ReqKind::Signal && r.fence_flag)
            ++acc.flagged_signal_count;
        if (r.kind == TraceKind::ProxyBlockBegin) {
            if (!proxy_open.emplace(r.pe, r.time).second) throw TraceError("nested proxy_block_begin");
            ++acc.proxy_stop_episodes;
        } else if (r.kind == TraceKind::ProxyBlockEnd) {
            auto it = proxy_open.find(r.pe);
            if (it == proxy_open.end()) throw TraceError("proxy_block_end without begin");
            acc.per_fence.push_back(r.time - it->second);
            acc.proxy_blocked_total += r.time - it->second;
            proxy_open.erase(it);
        } else if (r.kind == TraceKind::NicBlockBegin) {
            if (!nic_open.emplace(std::make_tuple(r.pe, r.dst_pe, int(r.qp)), r.time).second)
                throw TraceError("nested nic_block_begin");
            ++acc.nic_stall_episodes;
        } else if (r.kind == TraceKind::NicBlockEnd) {
            auto it = nic_open.find(std::make_tuple(r.pe, r.dst_pe, int(r.qp)));
            if (it == nic_open.end()) throw TraceError("nic_block_end without begin");
            acc.nic_stall_total += r.time - it->second;
            nic_open.erase(it);
        }
    }
    if (!proxy_open.empty() || !nic_open.empty()) throw TraceError("unmatched block_begin at end of trace");
    return acc;
}

std::vector<OrderingViolation> verify_ordering(const RunTrace& trace) {
    std::map<std::int64_t, TimeNs> landed;
    for (const auto& r : trace.records)
        if (r.kind == TraceKind::Completion && r.req_kind == ReqKind::Put && r.tile_id >= 0) {
            auto& t = landed[r.tile_id];
            t = std::max(t, r.time);
        }
    std::vector<OrderingViolation> bad;
    for (const auto& r : trace.records) {
        if (r.kind != TraceKind::SignalVisible || r.tile_id < 0) continue;
        auto it = landed.find(r.tile_id);
        if (it != landed.end() && r.time < it->second)
            bad.push_back({r.tile_id, r.src_pe, r.dst_pe, r.time, it->second});
    }
    return bad;
}

ConservationReport conservation_check(const RunTrace& trace, const DispatchWorkload& wl) {
    ConservationReport rep;
    std::uint64_t want = wl.total_remote_bytes();
    for (const auto& t : wl.local_transfers) want += t.bytes;
    std::map<std::int64_t, int> submitted, completed, signaled;
    std::uint64_t delivered = 0;
    for (const auto& r : trace.records) {
        if (r.req_kind == ReqKind::Put && r.kind == TraceKind::Submit) submitted[r.tile_id] = 1;
        if (r.req_kind == ReqKind::Put && r.kind == TraceKind::Completion) {
            ++completed[r.tile_id];
            delivered += r.size;
        }
        if (r.kind == TraceKind::SignalVisible) ++signaled[r.tile_id];
    }
    if (trace.total_put_bytes_submitted != want)
        rep.fail("submitted bytes " + std::to_string(trace.total_put_bytes_submitted) +
                 " != workload bytes " + std::to_string(want));
    if (delivered != trace.total_put_bytes_submitted)
        rep.fail("delivered bytes " + std::to_string(delivered) + " != submitted bytes " +
                 std::to_string(trace.total_put_bytes_submitted));
    // the reference's failure messages, in its order (metrics.cpp:166-188):
    // every put's completion count first, then every transfer's signal count
    auto times = [](const std::map<std::int64_t, int>& m, std::int64_t tile) {
        auto it = m.find(tile);
        return it == m.end() ? 0 : it->second;
    };
    for (const auto& kv : submitted) {
        const int c = times(completed, kv.first);
        if (c == 0) rep.fail("put tile " + std::to_string(kv.first) + " has no completion");
        else if (c != 1) rep.fail("put tile " + std::to_string(kv.first) + " completed " + std::to_string(c) + " times");
    }
    if (!wl.put_only)
        for (const auto& kv : submitted) {
            const int c = times(signaled, kv.first);
            if (c == 0) rep.fail("transfer tile " + std::to_string(kv.first) + " was never signaled");
            else if (c != 1) rep.fail("tile " + std::to_string(kv.first) + " signaled " + std::to_string(c) + " times");
        }
    return rep;
}

AlphaBetaFit fit_alpha_beta(const std::vector<std::pair<double, double>>& pts) {
    if (pts.size() < 2) throw ConfigError("fit_alpha_beta: need at least 2 points");
    double mx = 0, my = 0;
    for (auto [x, y] : pts) { mx += x; my += y; }
    mx /= double(pts.size());
    my /= double(pts.size());
    double sxx = 0, sxy = 0, syy = 0;
    for (auto [x, y] : pts) {
        sxx += (x - mx) * (x - mx);
        sxy += (x - mx) * (y - my);
        syy += (y - my) * (y - my);
    }
    if (sxx == 0.0) throw ConfigError("fit_alpha_beta: degenerate fit, all message sizes equal");
    AlphaBetaFit f;
    f.beta_ns_per_byte = sxy / sxx;
    f.alpha_ns = my - f.beta_ns_per_byte * mx;
    double res = 0;
    for (auto [x, y] : pts) res += (y - f.alpha_ns - f.beta_ns_per_byte * x) * (y - f.alpha_ns - f.beta_ns_per_byte * x);
    f.r_squared = syy == 0.0 ? 1.0 : 1.0 - res / syy;
    return f;
}

}  // namespace sigsim

// ============================================================= C ABI ======
using perseus::guarded;

namespace {
perseus_transfer to_c(const sigsim::TransferSpec& t) {
    return perseus_transfer{t.src_pe, t.dst_pe, t.expert, t.bytes, t.tile_id, t.heap_offset};
}
sigsim::TransferSpec from_c(const perseus_transfer& t) {
    sigsim::TransferSpec s;
    s.src_pe = t.src_pe;
    s.dst_pe = t.dst_pe;
    s.expert = t.expert;
    s.bytes = t.bytes;
    s.tile_id = t.tile_id;
    s.heap_offset = t.heap_offset;
    return s;
}
}  // namespace

extern "C" {

int perseus_abi_version(void) { return PERSEUS_ABI_VERSION; }

int perseus_remote_transfer_count(int64_t E, int64_t P, int64_t P_local, int64_t* out) {
    return guarded([&] { *out = sigsim::remote_transfer_count(E, P, P_local); });
}

uint64_t perseus_message_size(uint64_t S, int64_t k, int64_t E, int64_t H) {
    return sigsim::message_size(S, k, E, H);
}

int perseus_zipf_route(uint64_t S, int64_t E, double s, int64_t k, uint64_t seed,
                       uint64_t* counts, int32_t* ids) {
    return guarded([&] {
        std::vector<int32_t> v;
        auto c = sigsim::zipf_route_ids(S, E, s, k, seed, ids ? &v : nullptr);
        std::copy(c.begin(), c.end(), counts);
        if (ids) std::copy(v.begin(), v.end(), ids);
    });
}

int perseus_build_dispatch(int64_t H, int64_t I, int64_t E, int64_t k, int nodes, int gpn,
                           int nqps, uint64_t S, double skew, uint64_t tile_bytes, uint64_t seed,
                           perseus_transfer* remote, size_t remote_cap, size_t* n_remote,
                           perseus_transfer* local, size_t local_cap, size_t* n_local,
                           uint64_t* digest) {
    return guarded([&] {
        sigsim::ModelConfig m{"custom", H, I, E, k, 0.0};
        auto wl = sigsim::build_dispatch(m, sigsim::ClusterConfig{nodes, gpn, nqps}, S, skew,
                                         tile_bytes, seed);
        *n_remote = wl.remote_transfers.size();
        *n_local = wl.local_transfers.size();
        if (remote)
            for (size_t i = 0; i < wl.remote_transfers.size() && i < remote_cap; ++i)
                remote[i] = to_c(wl.remote_transfers[i]);
        if (local)
            for (size_t i = 0; i < wl.local_transfers.size() && i < local_cap; ++i)
                local[i] = to_c(wl.local_transfers[i]);
        if (digest) *digest = wl.digest();
    });
}

int perseus_assign_groups(const perseus_transfer* t, size_t n, int64_t gs, int64_t* group_of,
                          int64_t* leaders, size_t* n_groups) {
    return guarded([&] {
        std::vector<sigsim::TransferSpec> v(n);
        for (size_t i = 0; i < n; ++i) v[i] = from_c(t[i]);
        auto groups = sigsim::assign_groups(v, gs);
        *n_groups = groups.size();
        for (size_t g = 0; g < groups.size(); ++g) {
            if (leaders) leaders[g] = int64_t(groups[g].leader);
            for (size_t m : groups[g].members) group_of[m] = int64_t(g);
        }
    });
}

uint64_t perseus_heap_digest(const uint64_t* ext, size_t n_ext, const uint64_t* flags,
                             size_t n_flags) {
    std::vector<std::tuple<uint64_t, uint64_t, uint64_t>> e(n_ext);
    for (size_t i = 0; i < n_ext; ++i) e[i] = {ext[3 * i], ext[3 * i + 1], ext[3 * i + 2]};
    std::sort(e.begin(), e.end());
    std::vector<uint64_t> f(flags, flags + n_flags);
    std::sort(f.begin(), f.end());
    f.erase(std::unique(f.begin(), f.end()), f.end());
    uint64_t h = 0xcbf29ce484222325ULL;
    for (auto& [pe, off, len] : e) {
        uint64_t v[3] = {pe, off, len};
        h = sigsim::fnv1a64(v, sizeof v, h);
    }
    for (uint64_t x : f) h = sigsim::fnv1a64(&x, sizeof x, h);
    return h;
}

}  // extern "C"

namespace perseus {
// One direction's device events (all PEs) as a sigsim::RunTrace (see perseus.h):
// puts -> Submit/Put; group fences -> Submit/FenceMarker (both orderings), plus the
// flag on the group's first signal (NicFence); flag writes -> NicServiceStart/Signal;
// receiver observations -> SignalVisible + Completion/Put at the time the tile's
// content was first complete.
// ordering: 0 ProxyFence (fences -> FenceMarker records), 1 NicFence (the group's first
// flag carries the fence), 2 GPU-direct (the reference records neither, protocols.cpp:244-246)
sigsim::RunTrace device_run_trace(const perseus_trace_event* ev, size_t n, int dir, int ordering,
                                  int64_t* late_tiles) {
    const int base = dir == 0 ? PERSEUS_EV_DISPATCH_PUT : PERSEUS_EV_COMBINE_PUT;
    sigsim::RunTrace tr;
    // each PE stamps its own globaltimer: times are made relative to the PE's first
    // event of the forward (ordering checks compare times recorded on one PE only)
    std::map<int32_t, uint64_t> t0;
    for (size_t i = 0; i < n; ++i) {
        auto it = t0.find(ev[i].pe);
        if (it == t0.end() || ev[i].t < it->second) t0[ev[i].pe] = ev[i].t;
    }
    std::map<int64_t, uint64_t> put_bytes;  // tile -> bytes
    for (size_t i = 0; i < n; ++i)
        if (ev[i].kind == base) put_bytes[ev[i].tile] = ev[i].bytes;
    for (size_t i = 0; i < n; ++i) {
        const perseus_trace_event& e = ev[i];
        const int k = e.kind - base;
        if (k < 0 || k > 3) continue;
        sigsim::TraceRecord r;
        r.time = sigsim::TimeNs(e.t - t0[e.pe]);
        r.pe = uint32_t(e.pe);
        r.tile_id = e.tile;
        r.group_id = e.group;
        if (k == 0) {
            r.kind = sigsim::TraceKind::Submit;
            r.req_kind = sigsim::ReqKind::Put;
            r.src_pe = uint32_t(e.pe);
            r.dst_pe = uint32_t(e.peer);
            r.size = e.bytes;
            tr.total_put_bytes_submitted += e.bytes;
            tr.add(r);
        } else if (k == 1) {
            // ProxyFence and NicFence both submit a FenceMarker per group (under
            // NicFence it arms the flag of the next signal, transport.cpp:149-166);
            // GPU-direct records none (protocols.cpp:244-246,285-287)
            if (ordering == 2) continue;
            r.kind = sigsim::TraceKind::Submit;
            r.req_kind = sigsim::ReqKind::FenceMarker;
            r.src_pe = uint32_t(e.pe);
            r.dst_pe = uint32_t(e.peer);
            tr.add(r);
        } else if (k == 2) {
            r.kind = sigsim::TraceKind::NicServiceStart;
            r.req_kind = sigsim::ReqKind::Signal;
            r.src_pe = uint32_t(e.pe);
            r.dst_pe = uint32_t(e.peer);
            r.fence_flag = ordering == 1 && e.aux != 0;
            tr.add(r);
        } else {
            r.kind = sigsim::TraceKind::SignalVisible;
            r.req_kind = sigsim::ReqKind::Signal;
            r.src_pe = uint32_t(e.peer);
            r.dst_pe = uint32_t(e.pe);
            tr.add(r);
            sigsim::TraceRecord c = r;
            c.kind = sigsim::TraceKind::Completion;
            c.req_kind = sigsim::ReqKind::Put;
            c.time = sigsim::TimeNs(e.t - t0[e.pe] + (e.aux ? 0 : e.bytes));
            auto it = put_bytes.find(e.tile);
            c.size = it == put_bytes.end() ? 0 : it->second;
            tr.total_put_bytes_delivered += c.size;
            tr.add(c);
            if (!e.aux && late_tiles) ++*late_tiles;
        }
    }
    std::stable_sort(tr.records.begin(), tr.records.end(),
                     [](const sigsim::TraceRecord& a, const sigsim::TraceRecord& b) { return a.time < b.time; });
    if (!tr.records.empty()) tr.makespan = tr.records.back().time - tr.records.front().time;
    return tr;
}

}  // namespace perseus

namespace {
using perseus::device_run_trace;

sigsim::DispatchWorkload realised_workload(const perseus_transfer* transfers, size_t n, int dir) {
    sigsim::DispatchWorkload wl;
    for (size_t i = 0; i < n; ++i) {
        sigsim::TransferSpec t = from_c(transfers[i]);
        if (dir == 1) std::swap(t.src_pe, t.dst_pe);  // combine: the same tiles travelling back
        wl.remote_transfers.push_back(t);
    }
    return wl;
}
}  // namespace

extern "C" {

int perseus_trace_analyze(const perseus_trace_event* ev, size_t n, int nic_ordering,
                          const perseus_transfer* transfers, size_t n_transfers, perseus_trace_report* out) {
    return guarded([&] {
        *out = perseus_trace_report{};
        for (int dir = 0; dir < 2; ++dir) {
            const sigsim::RunTrace tr = device_run_trace(ev, n, dir, nic_ordering, &out->late_tiles[dir]);
            const auto acc = sigsim::fence_accounting(tr);
            out->records += int64_t(tr.records.size());
            out->fence_count[dir] = acc.fence_count;
            out->flagged_signal_count[dir] = acc.flagged_signal_count;
            out->ordering_violations[dir] = int64_t(sigsim::verify_ordering(tr).size());
            out->put_bytes[dir] = int64_t(tr.total_put_bytes_submitted);
            const auto rep = sigsim::conservation_check(tr, realised_workload(transfers, n_transfers, dir));
            out->conservation_ok[dir] = rep.pass ? 1 : 0;
            if (!rep.pass && !out->conservation_error[0] && !rep.failures.empty())
                std::snprintf(out->conservation_error, sizeof out->conservation_error, "%s: %s",
                              dir == 0 ? "dispatch" : "combine", rep.failures.front().c_str());
        }
    });
}

int perseus_trace_records(const perseus_trace_event* ev, size_t n, int nic_ordering, int direction,
                          perseus_trace_record* out, size_t cap, size_t* len, uint64_t* submitted_bytes,
                          uint64_t* delivered_bytes) {
    return guarded([&] {
        if (direction != 0 && direction != 1) throw sigsim::ConfigError("direction must be 0 (dispatch) or 1 (combine)");
        const sigsim::RunTrace tr = device_run_trace(ev, n, direction, nic_ordering, nullptr);
        *len = tr.records.size();
        if (submitted_bytes) *submitted_bytes = tr.total_put_bytes_submitted;
        if (delivered_bytes) *delivered_bytes = tr.total_put_bytes_delivered;
        if (!out) return;
        for (size_t i = 0; i < tr.records.size() && i < cap; ++i) {
            const sigsim::TraceRecord& r = tr.records[i];
            out[i] = perseus_trace_record{r.time, r.pe, int32_t(r.kind), int32_t(r.req_kind), r.src_pe, r.dst_pe,
                                          r.fence_flag ? 1 : 0, r.size, r.qp, 0, r.group_id, r.tile_id, r.submit_seq};
        }
    });
}

int perseus_trace_serialize(const perseus_trace_event* ev, size_t n, int nic_ordering, int direction,
                            char* buf, size_t cap, size_t* len) {
    return guarded([&] {
        if (direction != 0 && direction != 1) throw sigsim::ConfigError("direction must be 0 (dispatch) or 1 (combine)");
        const std::string text = sigsim::serialize_trace(device_run_trace(ev, n, direction, nic_ordering, nullptr));
        *len = text.size();
        if (buf && cap) {
            const size_t m = std::min(cap - 1, text.size());
            std::memcpy(buf, text.data(), m);
            buf[m] = 0;
        }
    });
}

int perseus_fit_alpha_beta(const double* bytes, const double* ns, size_t n, double* alpha_ns,
                           double* beta_ns_per_byte, double* r_squared) {
    return guarded([&] {
        std::vector<std::pair<double, double>> pts(n);
        for (size_t i = 0; i < n; ++i) pts[i] = {bytes[i], ns[i]};
        const auto f = sigsim::fit_alpha_beta(pts);
        *alpha_ns = f.alpha_ns;
        *beta_ns_per_byte = f.beta_ns_per_byte;
        *r_squared = f.r_squared;
    });
}

uint64_t perseus_fnv1a64(const void* data, size_t len, uint64_t h) {
    return sigsim::fnv1a64(data, len, h);
}

}  // extern "C"
