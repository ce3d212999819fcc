// layer_dev.h — the by-value kernel context of one layer rank.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <utility>

#include "perseus_internal.h"

namespace perseus {

using bf16 = __nv_bfloat16;

struct DevCtx {
    // geometry
    int32_t H, I, E, k, P, rank, E_loc;
    int32_t S;
    int32_t routing;     // PERSEUS_ROUTE_*
    int32_t signaling;   // PERSEUS_SIGNAL_*
    int32_t group_size;  // effective: 1 = per tile, 0 = per destination, >1 fixed
    uint32_t epoch;      // forward counter, value of every flag written this forward
    int32_t par;         // epoch & 1: which half of every symmetric double buffer

    // local buffers
    const bf16* x;
    bf16* out;
    const bf16* wg;      // [E][H]
    float* logits;       // [S][E]
    int32_t* ids;        // [S][k]
    float* weights;      // [S][k]
    int32_t* counts;     // [E]
    int32_t* offsets;    // [E+1]: sorted segment starts of this rank's (token, j) pairs
    int32_t* rows;       // [S*k]: token of each sorted slot
    int32_t* pos;        // [S*k]: sorted slot of each (token, j)
    int32_t* hist;       // [2][hist_blocks][E]: per-256-token-block expert histogram (parity halves)
    int32_t hist_blocks; // ceil(S/256)
    int32_t gate_splits; // tensor-core router: K splits, logits = sum of [gate_splits][S][E] partials
    int32_t weights_late; // 1: the router ran beside route/permute/plan; the fused kernel's copy warps write weights
    int32_t gate_inline;  // 1: the router runs in the stream after the plan kernel, launched early (PDL)
    const int32_t* zipf_ids;  // [S*k]: reference Zipf draws (routing == ZIPF)
    bf16* hbuf;          // [R_max][I]

    // symmetric buffers, one base pointer per PE (peer-mapped; [rank] = local)
    int32_t* count_table[kMaxPes];  // [2][P][E]
    uint32_t* count_flag[kMaxPes];  // [P]
    uint32_t* route_ctr;            // CTAs of k_route done (the last one publishes the counts)
    bf16* heap[kMaxPes];            // [2][R_max][H]
    uint32_t* dflag[kMaxPes];       // [2][T_max]
    bf16* ybuf[kMaxPes];            // [2][Y_rows][H]
    uint32_t* cflag[kMaxPes];       // [2][T_max]
    int64_t R_max, T_max, Y_rows;

    // plan (local)
    PlanHeader* hdr;
    SendTile* send;
    Group* groups;
    RecvTile* recv;
    Group* cgroups;
    uint32_t* group_ctr;
    uint32_t* cgroup_ctr;
    uint32_t* tile_ctr;
    int32_t max_send, max_recv;
    // fused-kernel scheduling (rebuilt by the plan every forward)
    int32_t* sorder;      // [max_send]: remote send positions in copy order (rotated destinations)
    int32_t* rorder;      // [max_recv]: recv positions in processing order (self, then by arrival)
    uint32_t* send_done;  // [max_send]: rows copied per send tile
    uint32_t* g1_done;    // [max_recv]: GEMM1 n-blocks finished per M-tile
    uint32_t* self_ready; // [max_recv]: epoch when a self tile's rows are in the heap
    uint32_t* sched;      // [4]: work-item / copy-unit counters
    int32_t* send_first;  // [E]: first send position of each expert's tiles
    int32_t* pairs;       // [max_recv][2]: M-tile pairs (recv positions, -1 = none) in processing order
    int32_t with_plan;    // k_perm: one extra CTA builds the plan
    int32_t self_head;    // minimum self pairs processed before the remote ones
    float head_ratio;     // est. link time of one tile / compute time of one M-tile pair

    unsigned long long* stats;  // [kStatCount]
    unsigned long long* fwd_t;  // [kFwdSlots]: this forward's communication timestamps (P > 1)
    TraceEv* trace;             // device event log (trace mode) or null
    uint32_t* trace_n;          // events recorded this forward
    uint32_t trace_cap;
    uint32_t* trace_seen_ep;    // [T_max] combine tiles already observed this forward (epoch-valued)
    unsigned long long* tl;     // [2 * kTlCount] kernel timeline of the last forward (~start, end) or null
    // dataflow combine (one PE, CTA-pair kernel): the fused kernel combines every
    // token as soon as its k expert rows exist, instead of a combine kernel after it
    int32_t df_combine;
    int32_t* tok_ready;             // [S] expert rows of the token written this forward
    unsigned long long* ready_q;    // [S] (epoch << 32 | token), in readiness order
    // per-destination token dedup of the dispatch (PERSEUS_F_DEDUP; P > 1)
    int32_t dedup;
    int32_t* dhist;                 // [2][hist_blocks][kMaxPes]: per-256-token-block tokens per destination
    int32_t* uidx;                  // [S*k] sorted slot -> the token's row in its destination's token buffer (-1: self)
    int32_t* dtot;                  // [kMaxPes]: unique tokens this rank sends to each destination
    int32_t* drows;                 // [kMaxPes]: rows of the reference layout this rank sends to each destination
    uint32_t* dsent;                // [kMaxPes]: token rows + index entries written to each destination
    uint32_t* ex_done;              // [max_recv]: rows expanded per received remote tile
    bf16* dd[kMaxPes];              // symmetric [2][P][S][H]: token buffer per (parity, source)
    int32_t* didx[kMaxPes];         // symmetric [2][R_max]: token-buffer row of every receive-heap row
    uint32_t* ddflag[kMaxPes];      // symmetric [2][P]: per source, its token buffer + index complete (epoch)
    int32_t local_dispatch;     // compute-only twin: dispatch puts / flags stay local, remote tiles not awaited
    int32_t local_combine;      // compute-only twin: combine puts / flags stay local, combine flags not awaited
    int32_t pdl;                // launch with programmatic dependent launch (PERSEUS_F_NO_PDL clears it)
    int32_t snake;              // plan: odd remote classes' pairs in descending expert order (L2 reuse)
};

// kernel ids of the diagnostic timeline (DevCtx::tl)
enum TlKernel : int { kTlGate = 0, kTlRoute, kTlPerm, kTlPlan, kTlFused, kTlCombine, kTlDispatch, kTlGemm1, kTlGemm2,
                      kTlMmaOut, kTlCopyEnd, kTlEpiEnd, kTlCounts, kTlPlanReady, kTlFusedEnter, kTlPlanB, kTlPlanC,
                      kTlPermBlkStart, kTlPermBlkEnd, kTlPermHist, kTlPermScan, kTlPermBits, kTlCount };

#ifdef __CUDACC__
// Launch with programmatic stream serialization (the kernel calls pdl_wait()
// before touching anything an earlier kernel wrote) unless the layer runs
// without PDL (c.pdl == 0: several ranks sharing one device — a grid waiting
// for its PDL primary's trigger holds up the work distributor, and with it the
// grids of the other ranks that the primary waits for).
template <typename K>
inline cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const DevCtx& c) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = c.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, c);
}

__device__ __forceinline__ uint64_t fwd_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Kernel timeline (diagnostics, perseus_layer_set_timeline): the first CTAs
// record ~start (max of ~t = min of t), the last CTAs their end (globaltimer).
__device__ __forceinline__ void tl_start(const DevCtx& c, int id) {
    if (c.tl && threadIdx.x == 0 && blockIdx.x < 4) atomicMax(c.tl + 2 * id, ~fwd_now());
}
__device__ __forceinline__ void tl_end(const DevCtx& c, int id, bool me) {
    if (c.tl && me && blockIdx.x + 4 >= gridDim.x) atomicMax(c.tl + 2 * id + 1, fwd_now());
}
// a point event (first and last time any caller reached it)
__device__ __forceinline__ void tl_mark(const DevCtx& c, int id) {
    if (!c.tl) return;
    const uint64_t t = fwd_now();
    atomicMax(c.tl + 2 * id, ~t);
    atomicMax(c.tl + 2 * id + 1, t);
}
// ... recorded later (a time taken with tl_now): the atomics stay off the
// critical path of latency-bound code that synchronises right after the point
__device__ __forceinline__ uint64_t tl_now(const DevCtx& c) { return c.tl ? fwd_now() : 0; }
__device__ __forceinline__ void tl_at(const DevCtx& c, int id, uint64_t t) {
    if (!c.tl || !t) return;
    atomicMax(c.tl + 2 * id, ~t);
    atomicMax(c.tl + 2 * id + 1, t);
}

// Append one event to the device event log (trace mode only).
__device__ __forceinline__ void trace_ev(const DevCtx& c, int kind, int peer, int tile, int group, uint32_t bytes,
                                         uint32_t aux, uint64_t t) {
    if (!c.trace) return;
    const uint32_t i = atomicAdd(c.trace_n, 1u);
    if (i >= c.trace_cap) return;
    TraceEv e;
    e.t = t;
    e.kind = kind;
    e.pe = c.rank;
    e.peer = peer;
    e.tile = tile;
    e.group = group;
    e.bytes = bytes;
    e.aux = aux;
    e.pad = 0;
    c.trace[i] = e;
}

// Receiver side, trace mode: a remote tile's flag has just been seen; check
// its rows (first and last 16 bytes of each) for the poison the receive
// buffers were filled with before the forward.  Incomplete content = the
// signal became visible before the data: wait for it, record both times.
__device__ __forceinline__ void trace_seen(const DevCtx& c, int kind, int src, int tile, const bf16* rows0, int rows) {
    const uint64_t t_seen = fwd_now();
    auto complete = [&]() {
        for (int r = 0; r < rows; ++r) {
            const uint4* p = reinterpret_cast<const uint4*>(rows0 + size_t(r) * c.H);
            const uint4 a = __ldcv(p), b = __ldcv(p + c.H / 8 - 1);
            if ((a.x & a.y & a.z & a.w) == 0xffffffffu || (b.x & b.y & b.z & b.w) == 0xffffffffu) return false;
        }
        return true;
    };
    const bool ok = complete();
    uint64_t t_land = t_seen;
    if (!ok) {
        while (!complete() && fwd_now() - t_seen < 1000000000ull) {
        }
        t_land = fwd_now();
    }
    trace_ev(c, kind, src, tile, -1, uint32_t(t_land - t_seen > 0xffffffffull ? 0xffffffffull : t_land - t_seen), ok ? 1u : 0u,
             t_seen);
}

// Routing weights of token t by one warp: lane j < k holds the logit of its
// j-th expert (the router's split-K partials summed in fixed order); every lane
// then forms the max and the sum of exponentials SEQUENTIALLY in j (values
// broadcast one by one), as orc_route_weights does, so all lanes — and every
// kernel using this (k_route, the fused kernel's dataflow combine) — get the
// same bits.  Returns lane j's weight (0 for lanes >= k).
__device__ __forceinline__ float route_weight_lane(const DevCtx& c, int t, int lane) {
    float l = -INFINITY;
    if (lane < c.k) {
        const int e = c.ids[size_t(t) * c.k + lane];
        l = 0.f;
        for (int q = 0; q < c.gate_splits; ++q) l += c.logits[(size_t(q) * c.S + t) * c.E + e];
    }
    float m = -INFINITY;
    for (int j = 0; j < c.k; ++j) m = fmaxf(m, __shfl_sync(0xffffffffu, l, j));
    float s = 0.f;
    for (int j = 0; j < c.k; ++j) s += expf(__shfl_sync(0xffffffffu, l, j) - m);
    return lane < c.k ? expf(l - m) / s : 0.f;
}

// ... and stores it: weights[t][j] = lane j's weight
__device__ __forceinline__ void route_weights_warp(const DevCtx& c, int t, int lane) {
    const float w = route_weight_lane(c, t, lane);
    if (lane < c.k) c.weights[size_t(t) * c.k + lane] = w;
}
#endif

}  // namespace perseus
