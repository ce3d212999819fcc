// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A flat extern "C" face over the UNMODIFIED reference library `sigsim`, compiled
// from the reference's own sources under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libsigsim_ref.so.  Nothing here re-implements
// reference logic: every function forwards to the reference symbol named in its
// comment.  Only tests/, __graft_entry__.smoke() and bench.py's reference /
// cpu_baseline legs load this library.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sigsim/metrics.hpp"
#include "sigsim/protocols.hpp"
#include "sigsim/trace.hpp"
#include "sigsim/workload.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

#define REF_TRY(body)                                                   \
    try {                                                               \
        body;                                                           \
        return 0;                                                       \
    } catch (const sigsim::ConfigError& e) { return fail(e, 1); }      \
    catch (const sigsim::ModelError& e) { return fail(e, 3); }         \
    catch (const sigsim::TraceError& e) { return fail(e, 3); }         \
    catch (const std::exception& e) { return fail(e, 3); }

// flat transfer record, same field order as include/perseus.h:perseus_transfer
struct FlatTransfer {
    uint32_t src_pe, dst_pe;
    int64_t expert;
    uint64_t bytes;
    int64_t tile_id;
    uint64_t heap_offset;
};

sigsim::ProtocolConfig protocol_for(int mode, int64_t group_size) {
    switch (mode) {
        case 0: return sigsim::vanilla_protocol();
        case 1: return sigsim::decoupled_protocol(group_size);
        case 2: return sigsim::nic_ordering_protocol();
        case 3: return sigsim::combined_protocol(group_size);
        case 4: return sigsim::gpu_direct_protocol(sigsim::Signaling::Coupled);
        default: return sigsim::gpu_direct_protocol(sigsim::Signaling::Decoupled);
    }
}

sigsim::DispatchWorkload make_wl(int64_t H, int64_t I, int64_t E, int64_t k, int nodes, int gpn,
                                 int nqps, uint64_t S, double skew, uint64_t tile_bytes,
                                 uint64_t seed) {
    sigsim::ModelConfig m{"custom", H, I, E, k, 0.0};
    sigsim::ClusterConfig c{nodes, gpn, nqps};
    return sigsim::build_dispatch(m, c, S, skew, tile_bytes, seed);
}

void flatten(const std::vector<sigsim::TransferSpec>& v, FlatTransfer* out, size_t cap) {
    for (size_t i = 0; i < v.size() && i < cap; ++i) {
        out[i] = FlatTransfer{v[i].src_pe, v[i].dst_pe, v[i].expert, v[i].bytes, v[i].tile_id,
                              v[i].heap_offset};
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// sigsim::remote_transfer_count (workload.cpp:39-47)
int ref_remote_transfer_count(int64_t E, int64_t P, int64_t P_local, int64_t* out) {
    REF_TRY(*out = sigsim::remote_transfer_count(E, P, P_local));
}

// sigsim::message_size (workload.cpp:49-55)
uint64_t ref_message_size(uint64_t S, int64_t k, int64_t E, int64_t H) {
    return sigsim::message_size(S, k, E, H);
}

// sigsim::zipf_route (workload.cpp:57-97)
int ref_zipf_route(uint64_t S, int64_t E, double s, int64_t k, uint64_t seed, uint64_t* counts) {
    REF_TRY({
        auto c = sigsim::zipf_route(S, E, s, k, seed);
        std::memcpy(counts, c.data(), c.size() * sizeof(uint64_t));
    });
}

// sigsim::build_dispatch (workload.cpp:155-213) + DispatchWorkload::digest (:105-126)
int ref_build_dispatch(int64_t H, int64_t I, int64_t E, int64_t k, int nodes, int gpn, int nqps,
                       uint64_t S, double skew, uint64_t tile_bytes, uint64_t seed,
                       FlatTransfer* remote, size_t remote_cap, size_t* n_remote,
                       FlatTransfer* local, size_t local_cap, size_t* n_local, uint64_t* digest) {
    REF_TRY({
        auto wl = make_wl(H, I, E, k, nodes, gpn, nqps, S, skew, tile_bytes, seed);
        *n_remote = wl.remote_transfers.size();
        *n_local = wl.local_transfers.size();
        if (remote) flatten(wl.remote_transfers, remote, remote_cap);
        if (local) flatten(wl.local_transfers, local, local_cap);
        *digest = wl.digest();
    });
}

// sigsim::assign_groups (protocols.cpp:52-94). group_of[i] = group of transfer i;
// leaders[g] = leader index of group g.
int ref_assign_groups(const FlatTransfer* t, size_t n, int64_t group_size, int64_t* group_of,
                      int64_t* leaders, size_t* n_groups) {
    REF_TRY({
        std::vector<sigsim::TransferSpec> v(n);
        for (size_t i = 0; i < n; ++i) {
            v[i].src_pe = t[i].src_pe;
            v[i].dst_pe = t[i].dst_pe;
            v[i].expert = t[i].expert;
            v[i].bytes = t[i].bytes;
            v[i].tile_id = t[i].tile_id;
            v[i].heap_offset = t[i].heap_offset;
        }
        auto groups = sigsim::assign_groups(v, group_size);
        *n_groups = groups.size();
        for (size_t g = 0; g < groups.size(); ++g) {
            if (leaders) leaders[g] = static_cast<int64_t>(groups[g].leader);
            for (size_t m : groups[g].members) group_of[m] = static_cast<int64_t>(g);
        }
    });
}

// Result of one reference dispatch run: run_dispatch (protocols.cpp:346-362)
// followed by fence_accounting / verify_ordering / conservation_check
// (metrics.cpp:10-59,118-190).
struct RefRunResult {
    uint64_t workload_digest;
    uint64_t heap_digest;
    int64_t fence_count;
    int64_t flagged_signal_count;
    int64_t proxy_stop_episodes;
    int64_t nic_stall_episodes;
    int64_t proxy_blocked_total_ns;
    int64_t makespan_ns;
    int64_t n_records;
    int64_t n_violations;
    int64_t conservation_pass;
    uint64_t total_put_bytes;
    int64_t n_signals_visible;
};

int ref_run_dispatch(int mode, int64_t group_size, int64_t H, int64_t I, int64_t E, int64_t k,
                     int nodes, int gpn, int nqps, uint64_t S, double skew, uint64_t tile_bytes,
                     uint64_t wl_seed, uint64_t run_seed, int64_t* fences_per_pe,
                     RefRunResult* out) {
    REF_TRY({
        auto wl = make_wl(H, I, E, k, nodes, gpn, nqps, S, skew, tile_bytes, wl_seed);
        sigsim::LatencyModel lat;
        auto trace = sigsim::run_dispatch(protocol_for(mode, group_size), wl, lat, run_seed);
        auto acc = sigsim::fence_accounting(trace);
        auto viol = sigsim::verify_ordering(trace);
        auto cons = sigsim::conservation_check(trace, wl);
        out->workload_digest = trace.workload_digest;
        out->heap_digest = trace.heap_digest;
        out->fence_count = acc.fence_count;
        out->flagged_signal_count = acc.flagged_signal_count;
        out->proxy_stop_episodes = acc.proxy_stop_episodes;
        out->nic_stall_episodes = acc.nic_stall_episodes;
        out->proxy_blocked_total_ns = acc.proxy_blocked_total;
        out->makespan_ns = trace.makespan;
        out->n_records = static_cast<int64_t>(trace.records.size());
        out->n_violations = static_cast<int64_t>(viol.size());
        out->conservation_pass = cons.pass ? 1 : 0;
        out->total_put_bytes = trace.total_put_bytes_submitted;
        int64_t sv = 0;
        const int P = nodes * gpn;
        if (fences_per_pe) std::memset(fences_per_pe, 0, sizeof(int64_t) * P);
        for (const auto& r : trace.records) {
            if (r.kind == sigsim::TraceKind::SignalVisible) ++sv;
            if (fences_per_pe && r.kind == sigsim::TraceKind::Submit &&
                r.req_kind == sigsim::ReqKind::FenceMarker && r.src_pe < (uint32_t)P)
                fences_per_pe[r.src_pe] += 1;
        }
        out->n_signals_visible = sv;
    });
}

#define COMMA ,
// sigsim::fit_alpha_beta (metrics.cpp:69-95); out = {alpha_ns, beta_ns_per_byte, r_squared}
int ref_fit_alpha_beta(const double* x, const double* y, size_t n, double* out) {
    REF_TRY({
        std::vector<std::pair<double COMMA double>> pts(n);
        for (size_t i = 0; i < n; ++i) pts[i] = std::make_pair(x[i] COMMA y[i]);
        auto f = sigsim::fit_alpha_beta(pts);
        out[0] = f.alpha_ns;
        out[1] = f.beta_ns_per_byte;
        out[2] = f.r_squared;
    });
}

// flat sigsim::TraceRecord, same layout as include/perseus.h:perseus_trace_record
struct FlatRecord {
    int64_t time;
    uint32_t pe;
    int32_t kind, req_kind;
    uint32_t src_pe, dst_pe;
    int32_t fence_flag;
    uint64_t size;
    int32_t qp, pad;
    int64_t group_id, tile_id;
    uint64_t submit_seq;
};

struct RefCheckReport {
    int64_t fence_count, flagged_signal_count, proxy_stop_episodes, nic_stall_episodes;
    int64_t proxy_blocked_total_ns, nic_stall_total_ns;
    int64_t n_violations;
    int64_t conservation_pass;
    int64_t n_failures;
};

// The reference's own checkers — sigsim::fence_accounting (metrics.cpp:10-59),
// verify_ordering (:118-138), conservation_check (:140-190) — run unmodified on
// a RunTrace built from flat records (e.g. a device RunTrace handed out by
// perseus_trace_records).  `transfers` = the workload's remote transfers; with
// `swap` their src/dst are exchanged (the combine direction's mirror).
// failures: the conservation failure messages, '\n'-joined, into msg[cap].
int ref_analyze_records(const FlatRecord* recs, size_t n, uint64_t submitted, uint64_t delivered,
                        const FlatTransfer* t, size_t nt, int swap, RefCheckReport* out, char* msg,
                        size_t cap) {
    REF_TRY({
        sigsim::RunTrace tr;
        for (size_t i = 0; i < n; ++i) {
            sigsim::TraceRecord r;
            r.time = recs[i].time;
            r.pe = recs[i].pe;
            r.kind = static_cast<sigsim::TraceKind>(recs[i].kind);
            r.req_kind = static_cast<sigsim::ReqKind>(recs[i].req_kind);
            r.src_pe = recs[i].src_pe;
            r.dst_pe = recs[i].dst_pe;
            r.size = recs[i].size;
            r.fence_flag = recs[i].fence_flag != 0;
            r.qp = recs[i].qp;
            r.group_id = recs[i].group_id;
            r.tile_id = recs[i].tile_id;
            r.submit_seq = recs[i].submit_seq;
            tr.add(r);
        }
        tr.total_put_bytes_submitted = submitted;
        tr.total_put_bytes_delivered = delivered;
        sigsim::DispatchWorkload wl;
        for (size_t i = 0; i < nt; ++i) {
            sigsim::TransferSpec x;
            x.src_pe = swap ? t[i].dst_pe : t[i].src_pe;
            x.dst_pe = swap ? t[i].src_pe : t[i].dst_pe;
            x.expert = t[i].expert;
            x.bytes = t[i].bytes;
            x.tile_id = t[i].tile_id;
            x.heap_offset = t[i].heap_offset;
            wl.remote_transfers.push_back(x);
        }
        const auto acc = sigsim::fence_accounting(tr);
        const auto viol = sigsim::verify_ordering(tr);
        const auto cons = sigsim::conservation_check(tr, wl);
        out->fence_count = acc.fence_count;
        out->flagged_signal_count = acc.flagged_signal_count;
        out->proxy_stop_episodes = acc.proxy_stop_episodes;
        out->nic_stall_episodes = acc.nic_stall_episodes;
        out->proxy_blocked_total_ns = acc.proxy_blocked_total;
        out->nic_stall_total_ns = acc.nic_stall_total;
        out->n_violations = static_cast<int64_t>(viol.size());
        out->conservation_pass = cons.pass ? 1 : 0;
        out->n_failures = static_cast<int64_t>(cons.failures.size());
        std::string all;
        for (const auto& f : cons.failures) all += f + "\n";
        if (msg && cap) {
            const size_t m = all.size() < cap - 1 ? all.size() : cap - 1;
            std::memcpy(msg, all.data(), m);
            msg[m] = 0;
        }
    });
}

// fnv1a64 (trace.cpp:53-62)
uint64_t ref_fnv1a64(const void* data, size_t len, uint64_t h) {
    return sigsim::fnv1a64(data, len, h);
}

}  // extern "C"
