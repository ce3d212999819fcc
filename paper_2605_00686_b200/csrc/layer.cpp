// layer.cpp — host runtime of one layer rank (the C ABI of include/perseus.h).
//
// Owns: weights, the symmetric region (count table, receive heap, combine
// buffer, flag words — double-buffered by forward parity), the peer mappings
// (cudaIpc), the device plan buffers, TMA descriptors and the launch sequence.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <tuple>
#include <vector>

#include "layer_dev.h"
#include "perseus.h"
#include "perseus_internal.h"
#include "sigsim/protocols.hpp"
#include "sigsim/workload.hpp"

namespace perseus {

// kernels.cu / gemm.cu
void launch_synth_fill(bf16* out, uint64_t base, uint64_t first, uint64_t n, float scale, cudaStream_t st);
void launch_gate_exact(const DevCtx& c, cudaStream_t st);
void launch_gate_tc(const CUtensorMap& tx, const CUtensorMap& twg, const DevCtx& c, int grid, cudaStream_t st);
void launch_route(const DevCtx& c, bool with_plan, cudaStream_t st);
void launch_plan(const DevCtx& c, cudaStream_t st);
void launch_dispatch(const DevCtx& c, cudaStream_t st);
cudaError_t configure_moe();
cudaError_t configure_moe2();
cudaError_t launch_moe2(const CUtensorMap& a1, const CUtensorMap& b1, const CUtensorMap& a2, const CUtensorMap& b2,
                        const CUtensorMap* smaps,
                        const DevCtx& c, int64_t a1_row_base, int grid, cudaStream_t st);
cudaError_t launch_moe(const CUtensorMap& a1, const CUtensorMap& b1, const CUtensorMap& a2, const CUtensorMap& b2,
                       const DevCtx& c, int64_t a1_row_base, int grid, cudaStream_t st);
void launch_combine(const DevCtx& c, int num_sms, cudaStream_t st);
cudaError_t configure_kernels(const DevCtx& c);
size_t gemm_smem_bytes();
cudaError_t configure_gemm();
void launch_gemm(int mode, const CUtensorMap& ta, const CUtensorMap& tb,
                 const DevCtx& c, int n_nb, int num_kb, int64_t a_row_base, int grid, cudaStream_t st);

namespace {
thread_local std::string g_err;

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

uint64_t splitmix64(uint64_t z) { return sigsim::SeededRng::mix(z); }
uint64_t tensor_base(uint64_t seed, uint32_t tensor) {
    return splitmix64(seed ^ (uint64_t(tensor) * 0xD1B54A32D192ED03ULL));
}
enum : uint32_t { kTX = 1, kTWG = 2, kTW1 = 3, kTW2 = 4 };

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
    static EncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
           "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiled>(p);
    }
    return fn;
}

// bf16 row-major [rows][cols] viewed as a 2D tensor, box 64 (K) x box_rows, SW128
// (box_rows = 1 for tile::gather4 maps)
CUtensorMap make_tmap(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows = 128) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
}  // namespace

void set_last_error(const std::string& msg) { g_err = msg; }

}  // namespace perseus

using namespace perseus;

struct perseus_layer {
    perseus_layer_config cfg{};
    int rank = 0, world = 1, device = 0;
    int H = 0, I = 0, E = 0, k = 0, S = 0, El = 0;
    int64_t R_max = 0, T_max = 0, Y_rows = 0;
    int max_send = 0, max_recv = 0;
    int gate_splits = 1, hist_blocks = 1;
    int num_sms = 148;
    int64_t gs = 0;  // resolved DECOUPLED group size (resolve_group_size)
    uint32_t epoch = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;                      // router GEMM side stream
    cudaEvent_t ev_x = nullptr, ev_gate = nullptr;

    // local
    bf16 *x_stage = nullptr, *out_stage = nullptr;
    // pipelined host API (perseus_layer_forward_host_async): 2 staging slots,
    // upload / download streams and per-slot events
    static constexpr int kHostSlots = 3;  // pipelined host batches in flight (forward_host_async)
    bf16 *xs2[kHostSlots] = {}, *os2[kHostSlots] = {};
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t ev_up[kHostSlots] = {}, ev_fwd[kHostSlots] = {}, ev_down[kHostSlots] = {};
    int host_slots = 2;  // in use (PERSEUS_HOST_SLOTS, 2..kHostSlots)
    uint64_t host_calls = 0;
    bf16 *wg = nullptr, *w1 = nullptr, *w2 = nullptr, *hbuf = nullptr;
    float *logits = nullptr, *weights = nullptr;
    int32_t *ids = nullptr, *counts = nullptr, *offsets = nullptr, *rows = nullptr, *pos = nullptr,
            *zipf_ids = nullptr, *hist = nullptr;
    PlanHeader* hdr = nullptr;
    SendTile* send = nullptr;
    Group *groups = nullptr, *cgroups = nullptr;
    RecvTile* recv = nullptr;
    uint32_t *group_ctr = nullptr, *cgroup_ctr = nullptr, *tile_ctr = nullptr;
    int32_t *sorder = nullptr, *rorder = nullptr;
    uint32_t *send_done = nullptr, *g1_done = nullptr, *self_ready = nullptr, *sched = nullptr;
    unsigned long long* fwd_t = nullptr;
    unsigned long long* tl = nullptr;  // kernel timeline (perseus_layer_set_timeline)
    TraceEv* trace = nullptr;          // device event log (perseus_layer_set_trace)
    uint32_t *trace_n = nullptr, *trace_seen_ep = nullptr;
    uint32_t trace_cap = 0;
    int32_t* send_first = nullptr;
    bool fused = true;  // forward() uses the fused persistent kernel
    bool stage_timing = false, timed_last = false;  // per-stage CUDA events (perseus_layer_set_stage_timing)
    bool pair = true;   // ... on CTA pairs (cta_group::2)
    int32_t* pairs = nullptr;
    unsigned long long* stats = nullptr;
    int32_t* tok_ready = nullptr;             // dataflow combine (one PE): per-token rows written
    unsigned long long* ready_q = nullptr;    // ... tokens in readiness order
    bool df_combine = false;

    // symmetric region
    uint8_t* sym = nullptr;
    size_t sym_bytes = 0;
    size_t off_ctab = 0, off_cflag_cnt = 0, off_dflag = 0, off_cflag = 0, off_heap = 0, off_ybuf = 0;
    size_t off_dd = 0, off_didx = 0, off_ddflag = 0;  // token dedup (PERSEUS_F_DEDUP)
    bool dedup = false;
    int32_t *dhist = nullptr, *uidx = nullptr, *dtot = nullptr, *drows = nullptr;
    uint32_t *dsent = nullptr, *ex_done = nullptr;
    uint32_t* route_ctr = nullptr;  // k_route CTAs done (reset by the last)
    uint8_t* peer[kMaxPes] = {};
    bool ipc_mapped[kMaxPes] = {};
    bool connected = false;

    CUtensorMap tm_a1{}, tm_b1{}, tm_a2{}, tm_b2{}, tm_wg{}, tm_x{}, tm_xg{};
    CUtensorMap* smaps = nullptr;  // device copy of the epilogue's TMA store maps (store_maps())
    const void* tm_x_ptr = nullptr;
    static constexpr int kTmCache = 4;  // second-level cache: the pipelined staging slots (+ the caller's x)
    CUtensorMap tm_x_c[kTmCache]{}, tm_xg_c[kTmCache]{};
    const void* tm_x_cptr[kTmCache] = {};
    int tm_x_next = 0;  // round-robin replacement
    cudaEvent_t ev[6] = {};
    const void* last_x = nullptr;

    DevCtx ctx(const void* x, void* out) const {
        DevCtx c{};
        c.H = H; c.I = I; c.E = E; c.k = k; c.P = world; c.rank = rank; c.E_loc = El; c.S = S;
        c.routing = cfg.routing;
        c.signaling = cfg.signaling;
        c.group_size = cfg.signaling == PERSEUS_SIGNAL_DECOUPLED ? int32_t(gs) : 1;
        c.epoch = epoch;
        c.par = int32_t(epoch & 1u);
        c.x = static_cast<const bf16*>(x);
        c.out = static_cast<bf16*>(out);
        c.wg = wg; c.logits = logits; c.ids = ids; c.weights = weights; c.counts = counts;
        c.offsets = offsets; c.rows = rows; c.pos = pos; c.zipf_ids = zipf_ids; c.hbuf = hbuf;
        c.hist = hist;
        c.hist_blocks = hist_blocks;
        c.gate_splits = gate_splits;
        for (int p = 0; p < world; ++p) {
            uint8_t* b = peer[p];
            c.count_table[p] = reinterpret_cast<int32_t*>(b + off_ctab);
            c.count_flag[p] = reinterpret_cast<uint32_t*>(b + off_cflag_cnt);
            // compute-only twins (diagnostics): a direction's peer stores and flags
            // go to this rank's own buffers instead (the receivers skip those waits)
            uint8_t* bd = (cfg.flags & PERSEUS_F_LOCAL_DISPATCH) ? peer[rank] : b;
            uint8_t* bc = (cfg.flags & PERSEUS_F_LOCAL_COMBINE) ? peer[rank] : b;
            c.heap[p] = reinterpret_cast<bf16*>(bd + off_heap);
            c.dflag[p] = reinterpret_cast<uint32_t*>(bd + off_dflag);
            c.ybuf[p] = reinterpret_cast<bf16*>(bc + off_ybuf);
            c.cflag[p] = reinterpret_cast<uint32_t*>(bc + off_cflag);
            if (dedup) {
                c.dd[p] = reinterpret_cast<bf16*>(b + off_dd);
                c.didx[p] = reinterpret_cast<int32_t*>(b + off_didx);
                c.ddflag[p] = reinterpret_cast<uint32_t*>(b + off_ddflag);
            }
        }
        c.dedup = dedup ? 1 : 0;
        c.route_ctr = route_ctr;
        c.dhist = dhist; c.uidx = uidx; c.dtot = dtot; c.drows = drows; c.dsent = dsent; c.ex_done = ex_done;
        c.local_dispatch = (cfg.flags & PERSEUS_F_LOCAL_DISPATCH) ? 1 : 0;
        c.local_combine = (cfg.flags & PERSEUS_F_LOCAL_COMBINE) ? 1 : 0;
        c.R_max = R_max; c.T_max = T_max; c.Y_rows = Y_rows;
        c.hdr = hdr; c.send = send; c.groups = groups; c.recv = recv; c.cgroups = cgroups;
        c.group_ctr = group_ctr; c.cgroup_ctr = cgroup_ctr; c.tile_ctr = tile_ctr;
        c.max_send = max_send; c.max_recv = max_recv;
        c.sorder = sorder; c.rorder = rorder; c.send_done = send_done; c.g1_done = g1_done;
        c.self_ready = self_ready; c.sched = sched; c.fwd_t = fwd_t; c.tl = tl;
        c.trace = trace; c.trace_n = trace_n; c.trace_cap = trace_cap; c.trace_seen_ep = trace_seen_ep; c.send_first = send_first; c.pairs = pairs;
        c.stats = stats;
        c.pdl = (cfg.flags & PERSEUS_F_NO_PDL) ? 0 : 1;
        {
            // measured at EP=4 (same box, alternating, 3 x 2 runs): K-step 433.4 -> 431.3 us
            static const int sn = [] { const char* e = getenv("PERSEUS_SNAKE"); return e ? atoi(e) : 1; }();
            c.snake = sn;
        }
        c.df_combine = df_combine ? 1 : 0;
        c.tok_ready = df_combine ? tok_ready : nullptr;
        c.ready_q = ready_q;
        return c;
    }
};

namespace {

void validate(const perseus_layer_config& c, int rank, int world) {
    sigsim::ModelConfig m{"layer", c.hidden_dim, c.intermediate_dim, c.experts, c.top_k, 0.0};
    m.validate();
    if (world < 1 || world > kMaxPes) throw sigsim::ConfigError("world size must be in [1, 8]");
    if (rank < 0 || rank >= world) throw sigsim::ConfigError("rank out of range");
    if (c.experts % world) throw sigsim::ConfigError("experts not divisible by PEs");
    if (c.hidden_dim % 256) throw sigsim::ConfigError("hidden_dim must be a multiple of 256");
    if (c.hidden_dim > 8192) throw sigsim::ConfigError("hidden_dim must be <= 8192");
    if (c.intermediate_dim % 128) throw sigsim::ConfigError("intermediate_dim must be a multiple of 128");
    if (c.experts > 256) throw sigsim::ConfigError("experts must be <= 256");
    if (c.top_k > 16) throw sigsim::ConfigError("top_k must be <= 16");
    if (int64_t(world) * c.experts > 4096) throw sigsim::ConfigError("P*E must be <= 4096");
    if (c.tokens_per_pe == 0) throw sigsim::ConfigError("tokens_per_pe must be > 0");
    if (c.routing == PERSEUS_ROUTE_BALANCED && (c.tokens_per_pe * uint64_t(c.top_k)) % uint64_t(c.experts))
        throw sigsim::ConfigError("build_dispatch: balanced routing needs E | S*k");
    if (c.routing < 0 || c.routing > 2) throw sigsim::ConfigError("unknown routing mode");
    if (c.routing == PERSEUS_ROUTE_ZIPF && c.skew < 0.0) throw sigsim::ConfigError("zipf_route: exponent must be >= 0");
    if (c.signaling < 0 || c.signaling > 3) throw sigsim::ConfigError("unknown signaling mode");
    if (c.group_size < 0 && c.group_size != PERSEUS_GROUP_AUTO)
        throw sigsim::ConfigError("group size must be >= 0 (or PERSEUS_GROUP_AUTO)");
}

int64_t gcd64(int64_t a, int64_t b) {
    while (b) {
        const int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Resolve the signal-group size of the DECOUPLED protocol on the host, where the
// per-(src, expert) counts of the reference routing modes are known for every
// PE (balanced: exact capacity, workload.cpp:180-195; Zipf: the same seeded
// draws every rank makes, workload.cpp:186-189).  group_size > 0 must divide
// every PE's remote tile count in both directions — the reference's own
// precheck (protocols.cpp:348-359) and assign_groups (:77-88) throw
// ConfigError otherwise; the device would only flag the plan as bad.
// PERSEUS_GROUP_AUTO picks the largest common divisor g of those counts with
// 8 <= g <= (tiles per destination) / 4: at least 8x fewer fences than per tile,
// and every destination's tiles land in >= 4 groups (an early first group);
// none exists -> one group per destination.  Learned-gate counts exist only on
// the device, so fixed / auto sizes need reference routing.
int64_t resolve_group_size(const perseus_layer_config& c, int world) {
    if (c.signaling != PERSEUS_SIGNAL_DECOUPLED || c.group_size == 0 || world == 1)
        return c.group_size == PERSEUS_GROUP_AUTO ? 0 : c.group_size;
    if (c.routing == PERSEUS_ROUTE_GATE)
        throw sigsim::ConfigError("group_size != 0 needs reference routing (balanced or zipf): learned-gate "
                                  "tile counts exist only on the device");
    const int P = world;
    const int64_t E = c.experts, S = int64_t(c.tokens_per_pe), k = c.top_k;
    std::vector<std::vector<int64_t>> cnt(P, std::vector<int64_t>(E, S * k / E));
    if (c.routing == PERSEUS_ROUTE_ZIPF)
        for (int s = 0; s < P; ++s) {
            const auto v = sigsim::zipf_route(uint64_t(S), E, c.skew, k,
                                              c.seed ^ (0x9E3779B97F4A7C15ULL * uint64_t(s + 1)));
            for (int64_t e = 0; e < E; ++e) cnt[s][e] = int64_t(v[e]);
        }
    // tiles[s][d]: 128-row transfer tiles PE s sends to PE d (workload.cpp:132-151)
    std::vector<std::vector<int64_t>> tiles(P, std::vector<int64_t>(P, 0));
    for (int s = 0; s < P; ++s)
        for (int64_t e = 0; e < E; ++e) tiles[s][e % P] += (cnt[s][e] + kTileRows - 1) / kTileRows;
    std::vector<int64_t> totals;  // per-PE remote tile counts: dispatch (send) and combine (receive)
    int64_t min_per_dst = INT64_MAX;
    for (int s = 0; s < P; ++s) {
        int64_t snd = 0, rcv = 0;
        for (int d = 0; d < P; ++d) {
            if (d == s) continue;
            snd += tiles[s][d];
            rcv += tiles[d][s];
            if (tiles[s][d] > 0) min_per_dst = std::min(min_per_dst, tiles[s][d]);
        }
        totals.push_back(snd);
        totals.push_back(rcv);
    }
    if (c.group_size > 0) {
        for (int64_t n : totals)
            if (n % c.group_size)
                throw sigsim::ConfigError("run_dispatch: group size does not divide remote transfer count");
        return c.group_size;
    }
    int64_t g = 0;
    for (int64_t n : totals) g = gcd64(g, n);
    const int64_t hi = min_per_dst == INT64_MAX ? 0 : std::max<int64_t>(8, min_per_dst / 4);
    for (int64_t d = std::min(g, hi); d >= 8; --d)
        if (g % d == 0) return d;
    return 0;
}

template <class T>
T* dalloc(size_t n) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
    ck(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)), "cudaMemset");
    return static_cast<T*>(p);
}

void free_layer(perseus_layer* L) {
    if (!L) return;
    cudaSetDevice(L->device);
    cudaDeviceSynchronize();
    for (int p = 0; p < kMaxPes; ++p)
        if (L->ipc_mapped[p]) cudaIpcCloseMemHandle(L->peer[p]);
    void* ptrs[] = {L->x_stage, L->out_stage, L->wg, L->w1, L->w2, L->hbuf, L->logits, L->weights, L->ids,
                    L->counts, L->offsets, L->rows, L->pos, L->zipf_ids, L->hist, L->hdr, L->send, L->groups,
                    L->cgroups, L->recv, L->group_ctr, L->cgroup_ctr, L->tile_ctr, L->stats, L->sym,
                    L->sorder, L->rorder, L->send_done, L->g1_done, L->self_ready, L->sched, L->fwd_t, L->tl, L->smaps, L->trace, L->trace_n, L->trace_seen_ep,
                    L->send_first, L->pairs, L->tok_ready, L->ready_q,
                    L->dhist, L->uidx, L->dtot, L->drows, L->dsent, L->ex_done, L->route_ctr};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (auto& e : L->ev)
        if (e) cudaEventDestroy(e);
    if (L->stream) cudaStreamDestroy(L->stream);
    if (L->stream2) cudaStreamDestroy(L->stream2);
    for (int i = 0; i < perseus_layer::kHostSlots; ++i) {
        if (L->xs2[i]) cudaFree(L->xs2[i]);
        if (L->os2[i]) cudaFree(L->os2[i]);
        for (cudaEvent_t e : {L->ev_up[i], L->ev_fwd[i], L->ev_down[i]})
            if (e) cudaEventDestroy(e);
    }
    if (L->up) cudaStreamDestroy(L->up);
    if (L->down) cudaStreamDestroy(L->down);
    if (L->ev_x) cudaEventDestroy(L->ev_x);
    if (L->ev_gate) cudaEventDestroy(L->ev_gate);
    delete L;
}

// TMA store maps of the pair kernel's epilogue (box 64 x 32, SW128), built once
// the peers are mapped: [0] hbuf, [1 + p] PE p's combine buffer (both halves)
const CUtensorMap* store_maps(perseus_layer* L) {
    if (!L->smaps) {
        std::vector<CUtensorMap> m(1 + kMaxPes);
        m[0] = make_tmap(L->hbuf, uint64_t(L->R_max), uint64_t(L->I), 32);
        const bool local_c = (L->cfg.flags & PERSEUS_F_LOCAL_COMBINE) != 0;
        for (int p = 0; p < L->world; ++p)
            m[1 + p] = make_tmap((local_c ? L->peer[L->rank] : L->peer[p]) + L->off_ybuf, 2 * uint64_t(L->Y_rows),
                                 uint64_t(L->H), 32);
        void* d = nullptr;
        ck(cudaMalloc(&d, m.size() * sizeof(CUtensorMap)), "cudaMalloc store maps");
        ck(cudaMemcpy(d, m.data(), m.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice), "memcpy store maps");
        L->smaps = static_cast<CUtensorMap*>(d);
    }
    return L->smaps;
}

void run_phase(perseus_layer* L, int phase, const void* x, void* out, cudaStream_t st) {
    if (!L->connected) throw sigsim::ModelError("layer not connected (ipc_import / connect_local)");
    ck(cudaSetDevice(L->device), "cudaSetDevice");
    if (phase == PERSEUS_PHASE_ROUTE || phase == PERSEUS_PHASE_ALL) ++L->epoch;
    if (x) L->last_x = x;
    DevCtx c = L->ctx(x ? x : L->last_x, out);
    if (c.x != L->tm_x_ptr) {  // TMA maps over the caller's token buffer (router tiles + row gathers)
        int hit = -1;
        for (int i = 0; i < perseus_layer::kTmCache; ++i)
            if (L->tm_x_cptr[i] == c.x) hit = i;
        if (hit < 0) {
            hit = L->tm_x_next;
            L->tm_x_next = (L->tm_x_next + 1) % perseus_layer::kTmCache;
            L->tm_x_c[hit] = make_tmap(c.x, uint64_t(L->S), uint64_t(L->H));
            L->tm_xg_c[hit] = make_tmap(c.x, uint64_t(L->S), uint64_t(L->H), 1);
            L->tm_x_cptr[hit] = c.x;
        }
        L->tm_x = L->tm_x_c[hit];
        L->tm_xg = L->tm_xg_c[hit];
        L->tm_x_ptr = c.x;
    }
    const bool all = phase == PERSEUS_PHASE_ALL;
    // stage events only when asked for (each record costs ~1-3 us of stream time)
    const bool tev = all && L->stage_timing;
    if (all) L->timed_last = tev;
    if (tev) ck(cudaEventRecord(L->ev[0], st), "event");
    static const bool tl_keep = [] { const char* e = getenv("PERSEUS_TL_KEEP"); return e && atoi(e) != 0; }();
    if (all && L->tl && !tl_keep) ck(cudaMemsetAsync(L->tl, 0, 2 * kTlCount * sizeof(unsigned long long), st), "memset");
    if (L->trace && (all || phase == PERSEUS_PHASE_ROUTE)) {
        // trace mode: empty event log, and this forward's receive buffers
        // poisoned (bf16 0xFFFF) so a tile seen before its data shows up
        ck(cudaMemsetAsync(L->trace_n, 0, sizeof(uint32_t), st), "memset");
        ck(cudaMemsetAsync(L->sym + L->off_heap + size_t(c.par) * L->R_max * L->H * 2, 0xff,
                           size_t(L->R_max) * L->H * 2, st), "poison heap");
        ck(cudaMemsetAsync(L->sym + L->off_ybuf + size_t(c.par) * L->Y_rows * L->H * 2, 0xff,
                           size_t(L->Y_rows) * L->H * 2, st), "poison ybuf");
    }
    // Reference routing modes: the expert ids do not depend on the logits, so the
    // router GEMM runs beside route/permute/plan and only the routing weights
    // (written by the fused kernel's copy warps) wait for it.  With PDL the
    // router is launched in the stream AFTER the permute/plan kernel and
    // triggers its dependents at once: it starts while the plan is built, and
    // the fused kernel launches early behind it (its pdl_wait covers router and
    // plan) — no cross-stream event, which would serialise the fused kernel's
    // launch (measured ~10 us from plan end to fused start with the event).
    // Without PDL: the router on a side stream, joined by an event before the
    // fused kernel.  PERSEUS_SIDE_GATE=0 / 1 / 2 forces serial / side stream / inline.
    static const int side_env = [] { const char* e = getenv("PERSEUS_SIDE_GATE"); return e ? atoi(e) : -1; }();
    const int side_mode = side_env >= 0 ? side_env : (c.pdl ? 2 : 1);
    const bool late_ok = all && L->fused && L->cfg.routing != PERSEUS_ROUTE_GATE;
    const bool side_gate = late_ok && side_mode == 1;
    c.gate_inline = late_ok && side_mode == 2 ? 1 : 0;
    c.weights_late = side_gate || c.gate_inline;
    // pair order: at least one wave of GEMM1 items on self pairs before the
    // remote pairs (the lag of launch_moe2's item interleave)
    c.self_head = std::max(1, (L->num_sms / 2 + L->I / 128 - 1) / (L->I / 128));
    {
        const double t_tile = 128.0 * L->H * 2 / 600e9;                   // NVLink store rate per sender
        const double t_pair = 2.0 * 128 * 6.0 * L->H * L->I / 1.0e15;      // GPU-wide: pairs complete at ~1 PFLOP/s
        static const double scale = [] { const char* e = getenv("PERSEUS_HEAD_SCALE"); return e ? atof(e) : 1.0; }();
        c.head_ratio = float(scale * t_tile / t_pair);
    }
    if (all || phase == PERSEUS_PHASE_ROUTE) {
        if (L->cfg.routing == PERSEUS_ROUTE_GATE) {
            launch_gate_exact(c, st);  // bit-exact fp32 order: learned top-k ids must match the oracle
        } else if (side_gate) {
            ck(cudaEventRecord(L->ev_x, st), "event");
            ck(cudaStreamWaitEvent(L->stream2, L->ev_x, 0), "wait");
            launch_gate_tc(L->tm_x, L->tm_wg, c, L->num_sms, L->stream2);
            ck(cudaEventRecord(L->ev_gate, L->stream2), "event");
        } else if (!c.gate_inline) {
            launch_gate_tc(L->tm_x, L->tm_wg, c, L->num_sms, st);  // serial
        }
        launch_route(c, /*with_plan=*/all, st);
        if (c.gate_inline) launch_gate_tc(L->tm_x, L->tm_wg, c, L->num_sms, st);  // after the plan, early (PDL)
    }
    if (tev) ck(cudaEventRecord(L->ev[1], st), "event");
    if (all && L->fused) {
        // one persistent kernel: dispatch puts + GEMM1 + GEMM2/combine puts,
        // overlapped tile by tile (gemm.cu:k_moe)
        if (side_gate) ck(cudaStreamWaitEvent(st, L->ev_gate, 0), "wait");  // router done before the persistent kernel
        if (tev) ck(cudaEventRecord(L->ev[2], st), "event");
        if (L->pair)
            ck(launch_moe2(L->tm_a1, L->tm_b1, L->tm_a2, L->tm_b2, store_maps(L), c, int64_t(c.par) * L->R_max,
                           L->num_sms, st),
               "launch k_moe2");
        else
            ck(launch_moe(L->tm_a1, L->tm_b1, L->tm_a2, L->tm_b2, c, int64_t(c.par) * L->R_max, L->num_sms, st),
               "launch k_moe");
        if (tev) ck(cudaEventRecord(L->ev[3], st), "event");
        if (tev) ck(cudaEventRecord(L->ev[4], st), "event");
        if (!c.df_combine) launch_combine(c, L->num_sms, st);  // else the fused kernel combined every token
        if (tev) ck(cudaEventRecord(L->ev[5], st), "event");
        ck(cudaGetLastError(), "kernel launch");
        return;
    }
    if (phase == PERSEUS_PHASE_DISPATCH) launch_plan(c, st);  // all: built by k_perm's plan CTA
    if (all || phase == PERSEUS_PHASE_DISPATCH) launch_dispatch(c, st);
    if (tev) ck(cudaEventRecord(L->ev[2], st), "event");
    if (all || phase == PERSEUS_PHASE_EXPERT) {
        launch_gemm(1, L->tm_a1, L->tm_b1, c, L->I / 128, L->H / 64, int64_t(c.par) * L->R_max, L->num_sms, st);
        if (tev) ck(cudaEventRecord(L->ev[3], st), "event");
        launch_gemm(2, L->tm_a2, L->tm_b2, c, L->H / 256, L->I / 64, 0, L->num_sms, st);
    }
    if (tev) ck(cudaEventRecord(L->ev[4], st), "event");
    if (all || phase == PERSEUS_PHASE_COMBINE) launch_combine(c, L->num_sms, st);
    if (tev) ck(cudaEventRecord(L->ev[5], st), "event");
    ck(cudaGetLastError(), "kernel launch");
}

}  // namespace

extern "C" {

const char* perseus_last_error(void) { return perseus::g_err.c_str(); }

int perseus_layer_create(const perseus_layer_config* cfg, int rank, int world, int device,
                         perseus_layer** out) {
    return guarded([&] {
        *out = nullptr;
        validate(*cfg, rank, world);
        const int64_t gs = resolve_group_size(*cfg, world);
        auto* L = new perseus_layer;
        try {
            L->cfg = *cfg;
            L->gs = gs;
            L->fused = !(cfg->flags & PERSEUS_F_UNFUSED);
            // CTA pairs share one expert's weights across two 128-row tiles; when a
            // local expert receives at most one tile per forward on average
            // (DeepSeek-V3 at EP=1: 128 rows) the second CTA of every pair would
            // idle, so the 1-CTA fused kernel is used instead
            L->pair = !(cfg->flags & PERSEUS_F_NO_PAIR) &&
                      ((cfg->flags & PERSEUS_F_FORCE_PAIR) ||
                       int64_t(world) * int64_t(cfg->tokens_per_pe) * cfg->top_k > int64_t(kTileRows) * cfg->experts);
            L->dedup = (cfg->flags & PERSEUS_F_DEDUP) && world > 1;
            if (L->dedup && (!L->fused || !L->pair))
                throw sigsim::ConfigError("token dedup (PERSEUS_F_DEDUP) needs the fused CTA-pair kernel");
            if (L->dedup && (cfg->flags & (PERSEUS_F_LOCAL_DISPATCH | PERSEUS_F_DF_COMBINE)))
                throw sigsim::ConfigError("token dedup (PERSEUS_F_DEDUP) excludes LOCAL_DISPATCH and DF_COMBINE");
            if (L->dedup && cfg->signaling >= PERSEUS_SIGNAL_NONE)
                throw sigsim::ConfigError("token dedup (PERSEUS_F_DEDUP) always fences and signals per destination");
            L->rank = rank;
            L->world = world;
            L->device = device;
            L->H = int(cfg->hidden_dim);
            L->I = int(cfg->intermediate_dim);
            L->E = int(cfg->experts);
            L->k = int(cfg->top_k);
            L->S = int(cfg->tokens_per_pe);
            L->El = L->E / world;
            const int64_t Sk = int64_t(L->S) * L->k;
            L->R_max = int64_t(world) * L->S * std::min(L->k, L->El) + 2 * kTileRows;
            L->T_max = int64_t(world) * (Sk / kTileRows + L->E + 1) + 16;
            L->Y_rows = Sk + kTileRows;
            L->max_send = int(Sk / kTileRows + L->E + 1);
            L->max_recv = int(int64_t(world) * (int64_t(L->S) * std::min(L->k, L->El) / kTileRows + L->El + 1));
            ck(cudaSetDevice(device), "cudaSetDevice");
            ck(cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
            // PERSEUS_NUM_SMS: cap the persistent grids (several ranks sharing one GPU in
            // oversubscribed multi-rank tests; each rank's fused kernel then fits beside the others)
            if (const char* e = getenv("PERSEUS_NUM_SMS")) L->num_sms = std::max(2, std::min(L->num_sms, atoi(e)) & ~1);
            ck(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&L->stream2, cudaStreamNonBlocking), "stream2");
            ck(cudaEventCreateWithFlags(&L->ev_x, cudaEventDisableTiming), "event");
            ck(cudaEventCreateWithFlags(&L->ev_gate, cudaEventDisableTiming), "event");
            for (auto& e : L->ev) ck(cudaEventCreate(&e), "event");

            const size_t H = L->H, I = L->I, E = L->E, El = L->El, S = L->S, P = world;
            L->x_stage = dalloc<bf16>(S * H);
            L->out_stage = dalloc<bf16>(S * H);
            L->wg = dalloc<bf16>(E * H);
            L->w1 = dalloc<bf16>(El * 2 * I * H);
            L->w2 = dalloc<bf16>(El * H * I);
            L->hbuf = dalloc<bf16>(size_t(L->R_max) * I);
            L->hist_blocks = int((S + 255) / 256);
            {
                // router split-K (partial logits summed by the weights' readers); PERSEUS_GATE_SPLITS overrides
                static const int gs_env = [] { const char* e = getenv("PERSEUS_GATE_SPLITS"); return e ? atoi(e) : 0; }();
                const int want = gs_env > 0 ? gs_env : 4;
                L->gate_splits = (H / 64) % want == 0 ? want : 1;
            }
            L->logits = dalloc<float>(size_t(L->gate_splits) * S * E);
            L->weights = dalloc<float>(Sk);
            L->ids = dalloc<int32_t>(Sk);
            L->counts = dalloc<int32_t>(E);
            L->offsets = dalloc<int32_t>(E + 1);
            L->rows = dalloc<int32_t>(Sk);
            L->pos = dalloc<int32_t>(Sk);
            L->zipf_ids = dalloc<int32_t>(Sk);
            L->hist = dalloc<int32_t>(2 * size_t(L->hist_blocks) * E);
            L->hdr = dalloc<PlanHeader>(1);
            L->send = dalloc<SendTile>(L->max_send);
            L->groups = dalloc<Group>(L->max_send);
            L->recv = dalloc<RecvTile>(L->max_recv);
            L->cgroups = dalloc<Group>(L->max_recv);
            L->group_ctr = dalloc<uint32_t>(L->max_send);
            L->cgroup_ctr = dalloc<uint32_t>(L->max_recv);
            L->tile_ctr = dalloc<uint32_t>(L->max_recv);
            L->sorder = dalloc<int32_t>(L->max_send);
            L->rorder = dalloc<int32_t>(L->max_recv);
            L->send_done = dalloc<uint32_t>(L->max_send);
            L->g1_done = dalloc<uint32_t>(L->max_recv);
            L->self_ready = dalloc<uint32_t>(L->max_recv);
            L->sched = dalloc<uint32_t>(8);
            L->fwd_t = dalloc<unsigned long long>(kFwdSlots);
            L->send_first = dalloc<int32_t>(E);
            L->pairs = dalloc<int32_t>(2 * size_t(L->max_recv) + 4);
            L->stats = dalloc<unsigned long long>(kStatCount);
            if (L->dedup) {
                L->dhist = dalloc<int32_t>(2 * size_t(L->hist_blocks) * kMaxPes);
                L->uidx = dalloc<int32_t>(Sk);
                L->dtot = dalloc<int32_t>(kMaxPes);
                L->drows = dalloc<int32_t>(kMaxPes);
                L->dsent = dalloc<uint32_t>(kMaxPes);
                L->ex_done = dalloc<uint32_t>(L->max_recv);
            }
            L->route_ctr = dalloc<uint32_t>(1);
            L->tok_ready = dalloc<int32_t>(S);
            L->ready_q = dalloc<unsigned long long>(S);

            // symmetric region: identical layout on every rank
            size_t o = 0;
            L->off_ctab = o; o = align_up(o + 2 * P * E * 4, 256);
            L->off_cflag_cnt = o; o = align_up(o + kMaxPes * 4, 256);
            L->off_dflag = o; o = align_up(o + 2 * size_t(L->T_max) * 4, 256);
            L->off_cflag = o; o = align_up(o + 2 * size_t(L->T_max) * 4, 1024);
            L->off_heap = o; o = align_up(o + 2 * size_t(L->R_max) * H * 2, 1024);
            L->off_ybuf = o; o = align_up(o + 2 * size_t(L->Y_rows) * H * 2, 1024);
            if (L->dedup) {
                L->off_dd = o; o = align_up(o + 2 * size_t(P) * S * H * 2, 1024);
                L->off_didx = o; o = align_up(o + 2 * size_t(L->R_max) * 4, 256);
                L->off_ddflag = o; o = align_up(o + 2 * kMaxPes * 4, 256);
            }
            L->sym_bytes = o;
            L->sym = dalloc<uint8_t>(o);

            if (cfg->routing == PERSEUS_ROUTE_ZIPF) {
                std::vector<int32_t> z;
                sigsim::zipf_route_ids(S, L->E, cfg->skew, L->k,
                                       cfg->seed ^ (0x9E3779B97F4A7C15ULL * uint64_t(rank + 1)), &z);
                ck(cudaMemcpy(L->zipf_ids, z.data(), z.size() * 4, cudaMemcpyHostToDevice), "memcpy");
                // EP=1 under skewed routing: experts with an odd tile count make pairs
                // whose second CTA recomputes the first's rows.  When the pairs'
                // useful fraction (tiles / 2·pairs) is below 0.85 the 1-CTA kernel is
                // faster (measured EP=1 Zipf s=1.0 / 1.5: 0.78 / 0.76 useful, 6–14%
                // faster single; s=0.5: 0.91, pairs 4% faster).  With P > 1 the pair
                // kernel stayed faster under the same skew (EP=4: 5–7%).
                if (world == 1 && !(cfg->flags & (PERSEUS_F_NO_PAIR | PERSEUS_F_FORCE_PAIR))) {
                    std::vector<int64_t> cnt(L->E, 0);
                    for (int32_t e : z) ++cnt[e];
                    int64_t tiles = 0, pairs = 0;
                    for (int64_t n : cnt) {
                        const int64_t t = (n + kTileRows - 1) / kTileRows;
                        tiles += t;
                        pairs += (t + 1) / 2;
                    }
                    if (pairs > 0 && double(tiles) < 0.85 * 2.0 * double(pairs)) L->pair = false;
                }
            }
            // PERSEUS_F_DF_COMBINE (one PE, CTA pairs): the fused kernel combines
            // tokens as their rows complete instead of a combine kernel after it.
            // Off by default: measured slower (Qwen3 EP=1: the fused kernel grows
            // by ~75 us vs a 30 us combine kernel; the last pairs' GEMM2 — a third
            // of the tokens' last rows — comes at the end of the schedule anyway)
            L->df_combine = (cfg->flags & PERSEUS_F_DF_COMBINE) && world == 1 && L->fused && L->pair;
            L->tm_a1 = make_tmap(L->sym + L->off_heap, 2 * uint64_t(L->R_max), H);
            L->tm_b1 = make_tmap(L->w1, El * 2 * I, H);
            L->tm_a2 = make_tmap(L->hbuf, uint64_t(L->R_max), I);
            L->tm_b2 = make_tmap(L->w2, El * H, I);
            L->tm_wg = make_tmap(L->wg, E, H);
            ck(configure_gemm(), "configure_gemm");
            ck(configure_moe(), "configure_moe");
            ck(configure_moe2(), "configure_moe2");
            ck(configure_kernels(L->ctx(nullptr, nullptr)), "configure_kernels");
            if (world == 1) {
                L->peer[0] = L->sym;
                L->connected = true;
                store_maps(L);
            }
            if (cfg->flags & PERSEUS_F_SYNTH_WEIGHTS) {
                if (perseus_layer_init_synthetic(L, cfg->seed, nullptr)) throw CudaError(perseus::g_err);
            }
            ck(cudaDeviceSynchronize(), "create sync");
        } catch (...) {
            free_layer(L);
            throw;
        }
        *out = L;
    });
}

int perseus_layer_destroy(perseus_layer* L) {
    return guarded([&] { free_layer(L); });
}

int perseus_layer_ipc_export(perseus_layer* L, void* blob, size_t cap, size_t* len) {
    return guarded([&] {
        *len = sizeof(cudaIpcMemHandle_t);
        if (!blob) return;
        if (cap < sizeof(cudaIpcMemHandle_t)) throw sigsim::ConfigError("ipc blob buffer too small");
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, L->sym), "cudaIpcGetMemHandle");
        std::memcpy(blob, &h, sizeof h);
    });
}

int perseus_layer_ipc_import(perseus_layer* L, const void* blobs, size_t len_each) {
    return guarded([&] {
        if (len_each != sizeof(cudaIpcMemHandle_t)) throw sigsim::ConfigError("bad ipc blob size");
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        for (int p = 0; p < L->world; ++p) {
            if (p == L->rank) {
                L->peer[p] = L->sym;
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const uint8_t*>(blobs) + p * len_each, sizeof h);
            void* ptr = nullptr;
            ck(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            L->peer[p] = static_cast<uint8_t*>(ptr);
            L->ipc_mapped[p] = true;
        }
        L->connected = true;
        store_maps(L);  // now, not in the first forward: cudaMalloc may synchronise the device
    });
}

int perseus_layer_connect_local(perseus_layer* const* ranks, int world) {
    return guarded([&] {
        for (int r = 0; r < world; ++r) {
            if (ranks[r]->world != world || ranks[r]->rank != r) throw sigsim::ConfigError("rank list mismatch");
            for (int p = 0; p < world; ++p) ranks[r]->peer[p] = ranks[p]->sym;
            ranks[r]->connected = true;
            ck(cudaSetDevice(ranks[r]->device), "cudaSetDevice");
            // built here, not in the first forward: ranks sharing one device in this
            // process are launched back to back, and cudaMalloc may synchronise the
            // device while an earlier rank's kernels wait for this rank's counts
            store_maps(ranks[r]);
        }
    });
}

int perseus_layer_set_weights(perseus_layer* L, const void* wg, const void* w1, const void* w2, void* stream) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        auto st = static_cast<cudaStream_t>(stream);
        const size_t H = L->H, I = L->I, E = L->E, El = L->El;
        if (wg) ck(cudaMemcpyAsync(L->wg, wg, E * H * 2, cudaMemcpyDeviceToDevice, st), "memcpy wg");
        if (w1) ck(cudaMemcpyAsync(L->w1, w1, El * 2 * I * H * 2, cudaMemcpyDeviceToDevice, st), "memcpy w1");
        if (w2) ck(cudaMemcpyAsync(L->w2, w2, El * H * I * 2, cudaMemcpyDeviceToDevice, st), "memcpy w2");
    });
}

int perseus_layer_init_synthetic(perseus_layer* L, uint64_t seed, void* stream) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        auto st = static_cast<cudaStream_t>(stream);
        const uint64_t H = L->H, I = L->I, E = L->E;
        const float s_h = float(std::sqrt(3.0 / double(H))), s_i = float(std::sqrt(3.0 / double(I)));
        launch_synth_fill(L->wg, tensor_base(seed, kTWG), 0, E * H, s_h, st);
        for (int j = 0; j < L->El; ++j) {
            const uint64_t e = uint64_t(L->rank) + uint64_t(L->world) * j;
            launch_synth_fill(L->w1 + j * 2 * I * H, tensor_base(seed, kTW1), e * 2 * I * H, 2 * I * H, s_h, st);
            launch_synth_fill(L->w2 + j * H * I, tensor_base(seed, kTW2), e * H * I, H * I, s_i, st);
        }
        ck(cudaGetLastError(), "synth fill");
    });
}

int perseus_fill_synthetic_x(perseus_layer* L, void* x, uint64_t seed, void* stream) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        const uint64_t n = uint64_t(L->S) * L->H;
        launch_synth_fill(static_cast<bf16*>(x), tensor_base(seed, kTX), uint64_t(L->rank) * n, n,
                          float(std::sqrt(3.0)), static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "synth fill x");
    });
}

int perseus_layer_forward(perseus_layer* L, const void* x, void* out, void* stream) {
    return guarded([&] { run_phase(L, PERSEUS_PHASE_ALL, x, out, static_cast<cudaStream_t>(stream)); });
}

int perseus_layer_forward_phase(perseus_layer* L, int phase, const void* x, void* out, void* stream) {
    return guarded([&] {
        if (phase < 0 || (phase > 3 && phase != PERSEUS_PHASE_ALL)) throw sigsim::ConfigError("bad phase");
        if (L->dedup && phase != PERSEUS_PHASE_ALL)
            throw sigsim::ConfigError("token dedup (PERSEUS_F_DEDUP) runs whole forwards only");
        run_phase(L, phase, x, out, static_cast<cudaStream_t>(stream));
    });
}

int perseus_layer_forward_host(perseus_layer* L, const void* x_host, void* out_host, void* stream) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        auto st = stream ? static_cast<cudaStream_t>(stream) : L->stream;
        const size_t bytes = size_t(L->S) * L->H * 2;
        ck(cudaMemcpyAsync(L->x_stage, x_host, bytes, cudaMemcpyHostToDevice, st), "H2D x");
        run_phase(L, PERSEUS_PHASE_ALL, L->x_stage, L->out_stage, st);
        ck(cudaMemcpyAsync(out_host, L->out_stage, bytes, cudaMemcpyDeviceToHost, st), "D2H out");
        ck(cudaStreamSynchronize(st), "forward_host sync");
    });
}

int perseus_layer_forward_host_async(perseus_layer* L, const void* x_host, void* out_host) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        const size_t bytes = size_t(L->S) * L->H * 2;
        if (!L->up) {
            ck(cudaStreamCreateWithFlags(&L->up, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&L->down, cudaStreamNonBlocking), "stream");
            static const int slots_env = [] { const char* e = getenv("PERSEUS_HOST_SLOTS"); return e ? atoi(e) : 0; }();
            L->host_slots = slots_env >= 2 ? std::min(slots_env, int(perseus_layer::kHostSlots)) : 3;
            for (int i = 0; i < L->host_slots; ++i) {
                ck(cudaMalloc(&L->xs2[i], bytes), "cudaMalloc");
                ck(cudaMalloc(&L->os2[i], bytes), "cudaMalloc");
                for (cudaEvent_t* e : {&L->ev_up[i], &L->ev_fwd[i], &L->ev_down[i]}) {
                    ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
                    ck(cudaEventRecord(*e, L->stream), "event");
                }
            }
        }
        const int s = int(L->host_calls++ % uint64_t(L->host_slots));
        // upload: after the forward that last read this slot
        ck(cudaStreamWaitEvent(L->up, L->ev_fwd[s], 0), "wait");
        ck(cudaMemcpyAsync(L->xs2[s], x_host, bytes, cudaMemcpyHostToDevice, L->up), "H2D x");
        ck(cudaEventRecord(L->ev_up[s], L->up), "event");
        // forward: after the upload and after the download that last read this slot's output
        ck(cudaStreamWaitEvent(L->stream, L->ev_up[s], 0), "wait");
        ck(cudaStreamWaitEvent(L->stream, L->ev_down[s], 0), "wait");
        run_phase(L, PERSEUS_PHASE_ALL, L->xs2[s], L->os2[s], L->stream);
        ck(cudaEventRecord(L->ev_fwd[s], L->stream), "event");
        // download
        ck(cudaStreamWaitEvent(L->down, L->ev_fwd[s], 0), "wait");
        ck(cudaMemcpyAsync(out_host, L->os2[s], bytes, cudaMemcpyDeviceToHost, L->down), "D2H out");
        ck(cudaEventRecord(L->ev_down[s], L->down), "event");
    });
}

int perseus_layer_host_wait(perseus_layer* L) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        if (L->down) ck(cudaStreamSynchronize(L->down), "host_wait");
        ck(cudaStreamSynchronize(L->stream), "host_wait");
    });
}

int perseus_layer_counters(perseus_layer* L, perseus_counters* out) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        unsigned long long s[kStatCount];
        ck(cudaMemcpy(s, L->stats, sizeof s, cudaMemcpyDeviceToHost), "memcpy stats");
        out->epoch = L->epoch;
        out->dispatch_fences = int64_t(s[kStatDispatchFences]);
        out->dispatch_signals = int64_t(s[kStatDispatchSignals]);
        out->dispatch_puts = int64_t(s[kStatDispatchPuts]);
        out->dispatch_put_bytes = int64_t(s[kStatDispatchBytes]);
        out->combine_fences = int64_t(s[kStatCombineFences]);
        out->combine_signals = int64_t(s[kStatCombineSignals]);
        out->combine_puts = int64_t(s[kStatCombinePuts]);
        out->combine_put_bytes = int64_t(s[kStatCombineBytes]);
        out->recv_tiles = int64_t(s[kStatRecvTiles]);
        out->wait_timeouts = int64_t(s[kStatTimeouts]);
        out->errors = int64_t(s[kStatErrors]);
        out->wait_dispatch_ns = int64_t(s[kStatWaitDispatchNs]);
        out->wait_g1_ns = int64_t(s[kStatWaitG1Ns]);
        out->copy_ns = int64_t(s[kStatCopyNs]);
        out->cta_ns = int64_t(s[kStatCtaNs]);
        out->wait_remote_ns = int64_t(s[kStatWaitRemoteNs]);
        out->dispatch_span_ns = int64_t(s[kStatDispatchSpanNs]);
        out->combine_span_ns = int64_t(s[kStatCombineSpanNs]);
        out->combine_wait_ns = int64_t(s[kStatCombineWaitNs]);
        out->mma_cycles = int64_t(s[kStatMmaCycles]);
        out->mma_ring_wait = int64_t(s[kStatMmaRingWait]);
        out->mma_acc_wait = int64_t(s[kStatMmaAccWait]);
        out->mma_data_wait = int64_t(s[kStatMmaDataWait]);
    });
}

int perseus_layer_read_routing(perseus_layer* L, int32_t* ids, float* weights, int32_t* counts, int32_t* pos) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        const size_t Sk = size_t(L->S) * L->k;
        if (ids) ck(cudaMemcpy(ids, L->ids, Sk * 4, cudaMemcpyDeviceToHost), "memcpy");
        if (weights) ck(cudaMemcpy(weights, L->weights, Sk * 4, cudaMemcpyDeviceToHost), "memcpy");
        if (counts) ck(cudaMemcpy(counts, L->counts, size_t(L->E) * 4, cudaMemcpyDeviceToHost), "memcpy");
        if (pos) ck(cudaMemcpy(pos, L->pos, Sk * 4, cudaMemcpyDeviceToHost), "memcpy");
    });
}

int perseus_layer_read_layout(perseus_layer* L, perseus_transfer* sent, size_t cap, size_t* n_sent,
                              int64_t* flags_seen, size_t flags_cap, size_t* n_flags_seen) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        PlanHeader h;
        ck(cudaMemcpy(&h, L->hdr, sizeof h, cudaMemcpyDeviceToHost), "memcpy hdr");
        if (h.error) throw VerifyError("device plan error " + std::to_string(h.error));
        std::vector<SendTile> st(size_t(std::max(h.n_send_remote, 0)));
        if (!st.empty())
            ck(cudaMemcpy(st.data(), L->send, st.size() * sizeof(SendTile), cudaMemcpyDeviceToHost), "memcpy send");
        *n_sent = st.size();
        if (sent)
            for (size_t i = 0; i < st.size() && i < cap; ++i)
                sent[i] = perseus_transfer{uint32_t(L->rank), uint32_t(st[i].dst), st[i].expert,
                                           uint64_t(st[i].rows) * L->H * 2, st[i].tile_id,
                                           uint64_t(st[i].heap_row) * L->H * 2};
        const int par = int(L->epoch & 1u);
        std::vector<uint32_t> fl(size_t(L->T_max));
        ck(cudaMemcpy(fl.data(), L->sym + L->off_dflag + size_t(par) * L->T_max * 4, fl.size() * 4,
                      cudaMemcpyDeviceToHost),
           "memcpy flags");
        size_t n = 0;
        for (size_t t = 0; t < fl.size(); ++t)
            if (fl[t] == L->epoch) {
                if (flags_seen && n < flags_cap) flags_seen[n] = int64_t(t);
                ++n;
            }
        *n_flags_seen = n;
    });
}

int perseus_layer_read_count_table(perseus_layer* L, int32_t* table) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        const int par = int(L->epoch & 1u);
        const size_t n = size_t(L->world) * L->E;
        ck(cudaMemcpy(table, L->sym + L->off_ctab + size_t(par) * n * 4, n * 4, cudaMemcpyDeviceToHost), "memcpy");
    });
}

int perseus_layer_set_timeline(perseus_layer* L, int on) {
    return guarded([&] {
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        if (on && !L->tl) {
            ck(cudaMalloc(&L->tl, 2 * kTlCount * sizeof(unsigned long long)), "cudaMalloc");
            ck(cudaMemset(L->tl, 0, 2 * kTlCount * sizeof(unsigned long long)), "memset");
        } else if (!on && L->tl) {
            ck(cudaDeviceSynchronize(), "sync");
            ck(cudaFree(L->tl), "cudaFree");
            L->tl = nullptr;
        }
    });
}

int perseus_layer_read_timeline(perseus_layer* L, uint64_t* start_end, int n) {
    return guarded([&] {
        if (!L->tl) throw sigsim::ConfigError("timeline is off");
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");  // the forward ran on non-blocking streams
        std::vector<unsigned long long> h(2 * kTlCount);
        ck(cudaMemcpy(h.data(), L->tl, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "memcpy");
        for (int i = 0; i < n && i < kTlCount; ++i) {
            start_end[2 * i] = h[2 * i] ? ~h[2 * i] : 0;
            start_end[2 * i + 1] = h[2 * i + 1];
        }
    });
}

int perseus_layer_info(perseus_layer* L, int* fused, int* cta_pairs) {
    return guarded([&] {
        if (fused) *fused = L->fused ? 1 : 0;
        if (cta_pairs) *cta_pairs = (L->fused && L->pair) ? 1 : 0;
    });
}

int perseus_resolve_group_size(const perseus_layer_config* cfg, int world, int64_t* group_size) {
    return guarded([&] {
        validate(*cfg, 0, world);
        *group_size = resolve_group_size(*cfg, world);
    });
}

int perseus_layer_group_size(perseus_layer* L, int64_t* group_size) {
    return guarded([&] { *group_size = L->cfg.signaling == PERSEUS_SIGNAL_DECOUPLED ? L->gs : 1; });
}

int perseus_layer_set_trace(perseus_layer* L, int on) {
    return guarded([&] {
        if (on && L->dedup)
            throw sigsim::ConfigError("token dedup (PERSEUS_F_DEDUP) has no reference event trace");
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        if (on && !L->trace) {
            // per tile: put / signal / fence / observe events, plus the fused kernel's
            // diagnostic GEMM1-item waits (one per n-block per CTA: I/128 per tile)
            L->trace_cap = uint32_t((8 + int64_t(L->I) / 128) * (int64_t(L->max_send) + L->max_recv) + 1024);
            ck(cudaMalloc(&L->trace, size_t(L->trace_cap) * sizeof(TraceEv)), "cudaMalloc trace");
            ck(cudaMalloc(&L->trace_n, sizeof(uint32_t)), "cudaMalloc");
            ck(cudaMemset(L->trace_n, 0, sizeof(uint32_t)), "memset");
            ck(cudaMalloc(&L->trace_seen_ep, size_t(L->T_max) * sizeof(uint32_t)), "cudaMalloc");
            ck(cudaMemset(L->trace_seen_ep, 0, size_t(L->T_max) * sizeof(uint32_t)), "memset");
        } else if (!on && L->trace) {
            cudaFree(L->trace);
            cudaFree(L->trace_n);
            cudaFree(L->trace_seen_ep);
            L->trace = nullptr;
            L->trace_n = L->trace_seen_ep = nullptr;
            L->trace_cap = 0;
        }
    });
}

int perseus_layer_read_trace(perseus_layer* L, perseus_trace_event* events, size_t cap, size_t* n) {
    static_assert(sizeof(perseus_trace_event) == sizeof(TraceEv), "trace event layout");
    return guarded([&] {
        if (!L->trace) throw sigsim::ConfigError("trace mode is off");
        ck(cudaSetDevice(L->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        uint32_t cnt = 0;
        ck(cudaMemcpy(&cnt, L->trace_n, sizeof cnt, cudaMemcpyDeviceToHost), "memcpy");
        if (cnt > L->trace_cap) throw sigsim::ModelError("device event log overflowed");
        *n = cnt;
        if (events && cap)
            ck(cudaMemcpy(events, L->trace, std::min<size_t>(cap, cnt) * sizeof(TraceEv), cudaMemcpyDeviceToHost),
               "memcpy trace");
    });
}

int perseus_layer_set_stage_timing(perseus_layer* L, int on) {
    return guarded([&] { L->stage_timing = on != 0; });
}

int perseus_layer_read_timing(perseus_layer* L, float* ms, int n) {
    return guarded([&] {
        if (!L->timed_last) throw sigsim::ConfigError("stage timing was off for the last forward");
        ck(cudaEventSynchronize(L->ev[5]), "event sync");
        for (int i = 0; i < n && i < 5; ++i) ck(cudaEventElapsedTime(&ms[i], L->ev[i], L->ev[i + 1]), "elapsed");
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// sigsim::run_dispatch backed by the GPU (include/sigsim/protocols.hpp).
// Replaces the reference's simulated hot path (protocols.cpp:346-362): the
// workload's PEs run as layer ranks on the current device, concurrently.
// ---------------------------------------------------------------------------
namespace {

void rethrow(int rc) {
    if (rc == PERSEUS_OK) return;
    const std::string msg = perseus::g_err;
    if (rc == PERSEUS_ERR_CONFIG) throw sigsim::ConfigError(msg);
    throw sigsim::ModelError(msg);
}

struct RankSet {  // RAII: layers, their token / output buffers and streams
    std::vector<perseus_layer*> layers;
    std::vector<void*> bufs;
    std::vector<cudaStream_t> streams;
    ~RankSet() {
        for (perseus_layer* l : layers) perseus_layer_destroy(l);
        for (void* b : bufs) cudaFree(b);
        for (cudaStream_t s : streams) cudaStreamDestroy(s);
    }
};

}  // namespace

namespace sigsim {

RunTrace run_dispatch(const ProtocolConfig& protocol, const DispatchWorkload& wl, const LatencyModel& latency,
                      std::uint64_t seed, std::uint64_t config_hash) {
    latency.validate();
    const int P = wl.cluster.total_pes();
    if (protocol.signaling == Signaling::Decoupled && protocol.group_size > 0)
        for (int pe = 0; pe < P; ++pe) {  // the reference's precheck (protocols.cpp:348-359)
            std::size_t count = 0;
            for (const auto& t : wl.remote_transfers) count += t.src_pe == uint32_t(pe) ? 1 : 0;
            if (count % std::size_t(protocol.group_size))
                throw ConfigError("run_dispatch: group size does not divide remote transfer count");
        }
    if (wl.cluster.gpus_per_node != 1)
        throw ConfigError("GPU run_dispatch: one GPU rank per PE (ClusterConfig{P,1,1}); same-node PEs would "
                          "need no fences in the reference (transport.cpp:303-320) but NVLink stores do");
    if (P < 1 || P > kMaxPes) throw ConfigError("GPU run_dispatch: 1..8 PEs");
    const uint64_t tile_bytes = uint64_t(kTileRows) * uint64_t(wl.model.hidden_dim) * 2;
    if (wl.tile_bytes != tile_bytes)
        throw ConfigError("GPU run_dispatch realises 128-row tiles: tile_bytes must be 128 * hidden_dim * 2 = " +
                          std::to_string(tile_bytes));
    if (wl.put_only || wl.microbench) throw ConfigError("GPU run_dispatch: MoE dispatch workloads only");

    perseus_layer_config cfg{};
    cfg.hidden_dim = wl.model.hidden_dim;
    cfg.intermediate_dim = wl.model.intermediate_dim;
    cfg.experts = wl.model.experts;
    cfg.top_k = wl.model.top_k;
    cfg.tokens_per_pe = wl.tokens_per_pe;
    cfg.routing = wl.skew > 0.0 ? PERSEUS_ROUTE_ZIPF : PERSEUS_ROUTE_BALANCED;
    cfg.skew = wl.skew;
    cfg.seed = wl.seed;
    cfg.signaling = protocol.suppress_fences ? PERSEUS_SIGNAL_NONE
                    : protocol.signaling == Signaling::Coupled ? PERSEUS_SIGNAL_COUPLED : PERSEUS_SIGNAL_DECOUPLED;
    cfg.group_size = protocol.group_size;
    // several ranks on one device: no PDL, each rank's persistent grid capped to 1/P of the SMs
    cfg.flags = PERSEUS_F_SYNTH_WEIGHTS | PERSEUS_F_NO_PDL | PERSEUS_F_FORCE_PAIR;
    int dev = 0, n_sms = 148;
    perseus::ck(cudaGetDevice(&dev), "cudaGetDevice");
    perseus::ck(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    RankSet rs;
    for (int r = 0; r < P; ++r) {
        perseus_layer* L = nullptr;
        rethrow(perseus_layer_create(&cfg, r, P, dev, &L));
        rs.layers.push_back(L);
        L->num_sms = std::max(2, (n_sms / P) & ~1);
    }
    rethrow(perseus_layer_connect_local(rs.layers.data(), P));
    const size_t xbytes = size_t(wl.tokens_per_pe) * size_t(wl.model.hidden_dim) * 2;
    for (int r = 0; r < P; ++r) {
        void *x = nullptr, *out = nullptr;
        cudaStream_t st = nullptr;
        perseus::ck(cudaMalloc(&x, xbytes), "cudaMalloc");
        rs.bufs.push_back(x);
        perseus::ck(cudaMalloc(&out, xbytes), "cudaMalloc");
        rs.bufs.push_back(out);
        perseus::ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        rs.streams.push_back(st);
        rethrow(perseus_fill_synthetic_x(rs.layers[r], x, wl.seed, st));
        rethrow(perseus_layer_set_trace(rs.layers[r], 1));
    }
    perseus::ck(cudaDeviceSynchronize(), "sync");
    for (int r = 0; r < P; ++r) rethrow(perseus_layer_forward(rs.layers[r], rs.bufs[2 * r], rs.bufs[2 * r + 1], rs.streams[r]));
    perseus::ck(cudaDeviceSynchronize(), "run_dispatch forward");

    std::vector<perseus_trace_event> ev;
    std::vector<perseus_transfer> got;
    std::vector<uint64_t> flags;
    for (int r = 0; r < P; ++r) {
        perseus_counters c{};
        rethrow(perseus_layer_counters(rs.layers[r], &c));
        if (c.wait_timeouts || c.errors)
            throw ModelError("GPU run_dispatch: rank " + std::to_string(r) + " saw " + std::to_string(c.wait_timeouts) +
                             " signal-wait timeouts / " + std::to_string(c.errors) + " device errors");
        size_t n = 0;
        rethrow(perseus_layer_read_trace(rs.layers[r], nullptr, 0, &n));
        std::vector<perseus_trace_event> e(n);
        rethrow(perseus_layer_read_trace(rs.layers[r], e.data(), n, &n));
        ev.insert(ev.end(), e.begin(), e.end());
        size_t ns = 0, nf = 0;
        rethrow(perseus_layer_read_layout(rs.layers[r], nullptr, 0, &ns, nullptr, 0, &nf));
        std::vector<perseus_transfer> t(ns);
        std::vector<int64_t> f(nf);
        rethrow(perseus_layer_read_layout(rs.layers[r], t.data(), ns, &ns, f.data(), nf, &nf));
        got.insert(got.end(), t.begin(), t.end());
        for (int64_t x : f) flags.push_back(uint64_t(x));
    }
    // the realised layout must be the workload's (build_dispatch, workload.cpp:132-213)
    auto key = [](const perseus_transfer& t) { return std::make_tuple(t.src_pe, t.dst_pe, t.expert, t.tile_id); };
    std::sort(got.begin(), got.end(), [&](const perseus_transfer& a, const perseus_transfer& b) { return key(a) < key(b); });
    std::vector<TransferSpec> want = wl.remote_transfers;
    std::sort(want.begin(), want.end(), [](const TransferSpec& a, const TransferSpec& b) {
        return std::make_tuple(a.src_pe, a.dst_pe, a.expert, a.tile_id) < std::make_tuple(b.src_pe, b.dst_pe, b.expert, b.tile_id);
    });
    bool same = got.size() == want.size();
    for (size_t i = 0; same && i < got.size(); ++i)
        same = got[i].src_pe == want[i].src_pe && got[i].dst_pe == want[i].dst_pe && got[i].expert == want[i].expert &&
               got[i].bytes == want[i].bytes && got[i].tile_id == want[i].tile_id &&
               got[i].heap_offset == want[i].heap_offset;
    if (!same) throw ModelError("GPU run_dispatch: the device's realised dispatch layout differs from the workload");

    const int ordering = protocol.transport == TransportPath::GpuDirect ? 2
                         : protocol.ordering == OrderingMode::NicFence ? 1 : 0;
    RunTrace tr = perseus::device_run_trace(ev.data(), ev.size(), 0, ordering, nullptr);
    tr.config_hash = config_hash;
    tr.workload_digest = wl.digest();
    tr.seed = seed;
    std::vector<uint64_t> ext;
    for (const auto& t : got) {
        ext.push_back(t.dst_pe);
        ext.push_back(t.heap_offset);
        ext.push_back(t.bytes);
    }
    tr.heap_digest = perseus_heap_digest(ext.data(), got.size(), flags.data(), flags.size());
    return tr;
}

}  // namespace sigsim
