// kernels.cu — the CUDA-core stages of the layer forward (sm_100a):
//   synthetic tensors, gate logits (pinned fp32 order), route (top-k / reference
//   routing + combine weights), permutation (stable counting sort), count
//   exchange, the per-forward device plan, dispatch puts + signals, combine.
// The grouped expert FFN (tcgen05) is in gemm.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "layer_dev.h"
#include "perseus.h"
#include "ptx.cuh"
#include "signal.cuh"
#include "plan.cuh"

namespace perseus {

using namespace ptx;

size_t perm_smem_bytes(const DevCtx& c);


// ------------------------------------------------------------ synthetic ----
// Same counter hash as oracle/oracle.c:orc_fill_bf16 (bit-identical bf16).
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_synth_fill(bf16* __restrict__ out, uint64_t base, uint64_t first, uint64_t n,
                             float scale) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t h = splitmix64(base + first + i);
        const float f = __fsub_rn(__fmul_rn(float(uint32_t(h >> 40)), 0x1.0p-23f), 1.0f);
        out[i] = __float2bfloat16_rn(__fmul_rn(f, scale));
    }
}

void launch_synth_fill(bf16* out, uint64_t base, uint64_t first, uint64_t n, float scale,
                       cudaStream_t st) {
    if (!n) return;
    k_synth_fill<<<148 * 8, 256, 0, st>>>(out, base, first, n, scale);
}

// ------------------------------------------------------------------ gate ----
// logits[t][e] = sum_h x[t][h] * wg[e][h]: ONE fmaf per h, h ascending — the
// contract oracle.c:orc_gate_logits restates, so logits (and learned top-k ids)
// are bit-exact.  CTA tile: 64 tokens x 64 experts; thread: 8 tokens x 2 experts
// (16 independent chains).  128-deep h steps staged through shared memory (fp32,
// h-major), the next step's tiles loaded into registers while the current one
// is consumed, so the global load latency hides under 2048 FMAs per thread.
constexpr int kGateE = 64, kGateH = 128;
template <int TT>  // tokens per thread (the CTA tile is 8 * TT tokens x 64 experts)
constexpr size_t gate_smem() { return sizeof(float) * kGateH * (8 * TT + kGateE); }

template <int TT>
__global__ void __launch_bounds__(256) k_gate(const bf16* __restrict__ x, const bf16* __restrict__ wg,
                                              float* __restrict__ logits, int S, int H, int E) {
    constexpr int kT = 8 * TT;            // tokens per CTA: warp w has tokens w * TT + [0, TT)
    extern __shared__ __align__(16) float gsm[];
    float* xs = gsm;                      // [kGateH][kT]
    float* ws = gsm + kGateH * kT;        // [kGateH][kGateE]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t0 = blockIdx.x * kT, e0 = blockIdx.y * kGateE;
    float acc[TT][2];
#pragma unroll
    for (int q = 0; q < TT; ++q) acc[q][0] = acc[q][1] = 0.f;

    // loader: x rows tid % kT with 8-wide h chunks (tid / kT) + (256 / kT) i; w rows
    // tid % 64 with chunks (tid / 64) + 4 i — a warp stores 32 consecutive rows of
    // one h (conflict-free h-major staging)
    constexpr int kXC = 256 / kT, kXN = 16 / kXC;  // x: chunk stride, chunks per thread
    const int xr = tid % kT, xc = tid / kT, wr = tid & 63, wc = tid >> 6;
    const bool xok = t0 + xr < S, wok = e0 + wr < E;
    uint4 px[kXN], pw[4];
    auto fetch = [&](int h0) {
#pragma unroll
        for (int i = 0; i < kXN; ++i) {
            const int h = h0 + (xc + kXC * i) * 8;
            px[i] = xok && h < H ? *reinterpret_cast<const uint4*>(x + size_t(t0 + xr) * H + h) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int h = h0 + (wc + 4 * i) * 8;
            pw[i] = wok && h < H ? *reinterpret_cast<const uint4*>(wg + size_t(e0 + wr) * H + h) : make_uint4(0, 0, 0, 0);
        }
    };
    auto stage = [&]() {
#pragma unroll
        for (int i = 0; i < kXN; ++i) {
            const int hh = (xc + kXC * i) * 8;
            const bf16* b = reinterpret_cast<const bf16*>(&px[i]);
#pragma unroll
            for (int q = 0; q < 8; ++q) xs[(hh + q) * kT + xr] = __bfloat162float(b[q]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int hh = (wc + 4 * i) * 8;
            const bf16* c = reinterpret_cast<const bf16*>(&pw[i]);
#pragma unroll
            for (int q = 0; q < 8; ++q) ws[(hh + q) * kGateE + wr] = __bfloat162float(c[q]);
        }
    };
    fetch(0);
    for (int h0 = 0; h0 < H; h0 += kGateH) {
        stage();
        __syncthreads();
        if (h0 + kGateH < H) fetch(h0 + kGateH);  // in flight under this step's FMAs
        const int hn = min(kGateH, H - h0);
#pragma unroll 8
        for (int h = 0; h < hn; ++h) {
            float xv[TT];
#pragma unroll
            for (int q = 0; q < TT; q += 4) {
                const float4 xa = *reinterpret_cast<const float4*>(&xs[h * kT + warp * TT + q]);
                xv[q] = xa.x; xv[q + 1] = xa.y; xv[q + 2] = xa.z; xv[q + 3] = xa.w;
            }
            const float2 wv = *reinterpret_cast<const float2*>(&ws[h * kGateE + lane * 2]);
#pragma unroll
            for (int q = 0; q < TT; ++q) {
                acc[q][0] = __fmaf_rn(xv[q], wv.x, acc[q][0]);
                acc[q][1] = __fmaf_rn(xv[q], wv.y, acc[q][1]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < TT; ++q) {
        const int t = t0 + warp * TT + q;
        if (t >= S) continue;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int e = e0 + lane * 2 + i;
            if (e < E) logits[size_t(t) * E + e] = acc[q][i];
        }
    }
}

// ----------------------------------------------------------------- route ----
// Top-k of one token's E logits by one warp (lane j < k returns the j-th choice):
// descending logit, ties to the lower expert index (orc_topk).  Each lane holds
// PER >= ceil(E / 32) candidates (expert lane + 32 i) in registers.
template <int PER>
__device__ __forceinline__ int topk_warp(const float* l, int E, int k, int lane) {
    float v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) v[i] = lane + 32 * i < E ? l[lane + 32 * i] : -INFINITY;
    unsigned taken = 0;  // bit i: slot i already chosen
    int my_id = -1;
    for (int j = 0; j < k; ++j) {
        float bv = -INFINITY;
        int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = lane + 32 * i;
            if (e < E && !(taken >> i & 1u) && (v[i] > bv || (v[i] == bv && e < bi))) {
                bv = v[i];
                bi = e;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        if (lane == j) my_id = bi;
    }
    return my_id;
}

// One warp per token: choose k experts, then softmax over their logits.
//   GATE     : top-k by descending logit, ties to the lower index (orc_topk)
//   BALANCED : id[t*k+j] = (t*k+j) mod E (exact capacity, workload.cpp:180-195)
//   ZIPF     : the reference's Zipf draws (workload.cpp:57-97), host-expanded
// One token of k_route (one warp).
__device__ __forceinline__ void route_token(const DevCtx& c, int t, int lane) {
    const float* l = c.logits + size_t(t) * c.E;
    int my_id = -1;  // lane j < k holds the j-th chosen expert
    if (c.routing == PERSEUS_ROUTE_GATE) {
        const int per = (c.E + 31) / 32;
        my_id = per <= 4 ? topk_warp<4>(l, c.E, c.k, lane) : per <= 8 ? topk_warp<8>(l, c.E, c.k, lane)
                                                                     : topk_warp<32>(l, c.E, c.k, lane);
    } else if (lane < c.k) {
        const int64_t flat = int64_t(t) * c.k + lane;
        my_id = c.routing == PERSEUS_ROUTE_BALANCED ? int(flat % c.E) : c.zipf_ids[flat];
    }
    if (lane == 0 && c.tok_ready) c.tok_ready[t] = 0;  // dataflow combine: this forward's row count
    if (lane < c.k) {
        c.ids[size_t(t) * c.k + lane] = my_id;
        // per-256-token-block expert histogram (this forward's parity half)
        atomicAdd(&c.hist[(size_t(c.par) * c.hist_blocks + t / 256) * c.E + my_id], 1);
    }
    if (c.dedup) {
        // token dedup: per-256-token-block count of tokens per remote destination
        unsigned dm = lane < c.k && my_id % c.P != c.rank ? 1u << (my_id % c.P) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) dm |= __shfl_xor_sync(0xffffffffu, dm, o);
        if (lane < c.P && (dm >> lane & 1u))
            atomicAdd(&c.dhist[(size_t(c.par) * c.hist_blocks + t / 256) * kMaxPes + lane], 1);
    }
    // The routing weights.  Learned gate: from the exact logits.  Reference
    // routing modes: the ids do not depend on the logits; when the router GEMM
    // ran on a side stream (fused path) the fused kernel's copy warps write the
    // weights, otherwise the split-K partials are already summable here.
    if (c.routing == PERSEUS_ROUTE_GATE) {
        const float mine = lane < c.k ? l[my_id] : -INFINITY;
        float m = mine;
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const float ex = lane < c.k ? expf(mine - m) : 0.f;
        float s = ex;
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane < c.k) c.weights[size_t(t) * c.k + lane] = ex / s;
    } else if (!c.weights_late) {
        __syncwarp();
        route_weights_warp(c, t, lane);
    }
}

// Count exchange, by the last CTA of k_route to finish its histogram atomics:
// this rank's per-expert counts (the block histograms summed) into its row of
// every PE's [P][E] count table, one fence, then the per-source ready flag at
// every PE.  Published here rather than by the permutation kernel so the plans
// (this rank's and the peers') get the counts a kernel launch earlier.
__device__ __forceinline__ void publish_counts(const DevCtx& c) {
    __shared__ int s_last;
    __shared__ int32_t part[256];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this CTA's histogram atomics before its arrival
        s_last = atomicAdd(c.route_ctr, 1u) == gridDim.x - 1;
        if (s_last) *c.route_ctr = 0;  // every CTA of this launch has arrived
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int E = c.E, tid = threadIdx.x, nb = c.hist_blocks;
    const int32_t* hist = c.hist + size_t(c.par) * c.hist_blocks * E;
    const int G = max(1, int(blockDim.x) / E);  // threads per expert (E <= 256)
    if (tid < G * E) {
        const int e = tid % E, h = tid / E;
        int32_t sum = 0;
        int q = h;
        for (; q + 7 * G < nb; q += 8 * G) {
            int32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(hist + size_t(q + u * G) * E + e);
#pragma unroll
            for (int u = 0; u < 8; ++u) sum += v[u];
        }
        for (; q < nb; q += G) sum += __ldcg(hist + size_t(q) * E + e);
        part[tid] = sum;
    }
    __syncthreads();
    for (int e = tid; e < E; e += blockDim.x) {
        int32_t cnt = 0;
        for (int h = 0; h < G; ++h) cnt += part[h * E + e];
        c.counts[e] = cnt;
        for (int p = 0; p < c.P; ++p) c.count_table[p][(size_t(c.par) * c.P + c.rank) * E + e] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
        // one fence (cumulative over the CTA barrier: every thread's table
        // stores), then the flags; the plans acquire them
        if (c.P > 1) fence_acq_rel_sys();
        else fence_acq_rel_gpu();
        for (int p = 0; p < c.P; ++p) st_relaxed_sys(c.count_flag[p] + c.rank, c.epoch);
        tl_mark(c, kTlCounts);
    }
}

__global__ void __launch_bounds__(256) k_route(DevCtx c) {
    pdl_wait();
    pdl_launch_dependents();
    tl_start(c, kTlRoute);
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (t < c.S) route_token(c, t, lane);
    publish_counts(c);
    tl_end(c, kTlRoute, threadIdx.x == 0);
}

// ----------------------------------------------------------- permutation ----
// Stable counting sort of the (token, j) pairs by expert (orc_permute): tokens
// ascending inside each expert segment, over 256-token blocks:
//   k_route: per-block expert histogram hist[b][e] (global atomics)
//   k_perm : segment offsets (scan of the block histograms), then stable
//            in-block ranks from a per-expert token bitmask (popcount of the
//            lower lanes).
constexpr int kPermT = 256;

__device__ int32_t block_exclusive_scan(int32_t* a, int n, int32_t* scratch /*33*/);

// K: the top-k (8, or 0 = any k <= 16); DEDUP: the token-dedup buffer rows.
// Specialised so the common kernel carries no code it does not run — the
// kernel is instruction-fetch bound (half its stall samples, ncu).
template <int K, bool DEDUP>
__global__ void __launch_bounds__(kPermT) k_perm(DevCtx c) {
    constexpr int KM = K > 0 ? K : 16;
    // Trigger before waiting: the next kernel (the router GEMM, which reads only
    // x and the router weights) may then run beside k_route as well.  Every CTA
    // of this grid is resident once all have triggered, so nothing behind it can
    // take their SMs.
    pdl_launch_dependents();
    pdl_wait();
    extern __shared__ int32_t sm[];
    const int E = c.E, b = blockIdx.x, nb = int(gridDim.x) - c.with_plan, tid = threadIdx.x;
    if (b == nb) {
        // the plan CTA: waits for every PE's counts (this rank's from CTA 0 below)
        // and builds the plan while the other CTAs rank their tokens
        static_assert(kPermT == kPlanThreads, "the plan CTA runs plan_body with all its threads");
        if (tid == 0 && c.tl) atomicMax(c.tl + 2 * kTlPlan, ~fwd_now());
        plan_body(c, sm);
        if (tid == 0 && c.tl) atomicMax(c.tl + 2 * kTlPlan + 1, fwd_now());
        return;
    }
    tl_start(c, kTlPerm);
    const uint64_t t_blk = tl_now(c);
    // Per-expert shared arrays are stored at a swizzled expert slot: with the
    // balanced routing a warp's lanes hit experts 8 apart, which all fall in one
    // bank at a stride of 8 words (16-way conflicts); the XOR spreads them over
    // all 32 banks.  A bijection on [0, E) when E is a multiple of 32.
    const bool swz = (E & 31) == 0;
    auto sw = [swz](int e) { return swz ? e ^ ((e >> 3) & 31) : e; };
    uint32_t* bits = reinterpret_cast<uint32_t*>(sm);  // [kPermT / 32][E] (swizzled expert slot)
    int32_t* base = sm + E * (kPermT / 32);             // [E] (swizzled)
    int32_t* tot = base + E;                            // [E]
    int32_t* scratch = tot + E;                         // [33]
    int32_t* pre = scratch + 40;                        // [kPermT / 32][E] (swizzled)
    int32_t* part = pre + E * (kPermT / 32);            // [kPermT][2] histogram partial sums
    for (int i = tid; i < E * (kPermT / 32); i += kPermT) bits[i] = 0;
    const int32_t* hist = c.hist + size_t(c.par) * c.hist_blocks * E;
    int32_t* hist_next = c.hist + size_t(c.par ^ 1) * c.hist_blocks * E;  // zeroed for the next forward
    // the block histograms: G = kPermT / E threads per expert (E <= 256), each
    // summing every G-th block with up to 16 loads in flight (latency-bound)
    {
        const int G = kPermT / E;
        if (tid < G * E) {
            const int e = tid % E, h = tid / E;
            int32_t before = 0, after = 0;
            int q = h;
            for (; q + 15 * G < nb; q += 16 * G) {
                int32_t v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = hist[size_t(q + u * G) * E + e];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    if (q + u * G < b) before += v[u]; else after += v[u];
                }
            }
            for (; q < nb; q += G) {
                const int32_t v = hist[size_t(q) * E + e];
                if (q < b) before += v; else after += v;
            }
            part[2 * tid] = before;
            part[2 * tid + 1] = after;
        }
        __syncthreads();
    }
    for (int e = tid; e < E; e += kPermT) {
        int32_t before = 0, after = 0;
        for (int h = 0; h < kPermT / E; ++h) {
            before += part[2 * (h * E + e)];
            after += part[2 * (h * E + e) + 1];
        }
        base[sw(e)] = before;
        tot[e] = before + after;
        hist_next[size_t(b) * E + e] = 0;
    }
    __syncthreads();
    const uint64_t t_hist = tl_now(c);  // (the counts were published by k_route's last CTA)
    if (DEDUP && b == 0 && tid < c.P) {  // rows of the reference layout this rank sends to each PE
        int32_t r = 0;
        for (int e = tid; e < E; e += c.P) r += tot[e];
        c.drows[tid] = r;
    }
    const int32_t total = block_exclusive_scan(tot, E, scratch);
    for (int e = tid; e < E; e += kPermT) {
        base[sw(e)] += tot[e];
        if (b == 0) c.offsets[e] = tot[e];
    }
    if (b == 0 && tid == 0) c.offsets[E] = total;
    const uint64_t t_scan = tl_now(c);
    const int t = b * kPermT + tid;
    const int k = K > 0 ? K : c.k;
    int32_t my[KM];
    if (t < c.S) {
#pragma unroll
        for (int j = 0; j < KM; ++j)
            if (j < k) my[j] = c.ids[size_t(t) * k + j];
#pragma unroll
        for (int j = 0; j < KM; ++j)
            if (j < k) atomicOr(&bits[(tid >> 5) * E + sw(my[j])], 1u << (tid & 31));
    }
    __syncthreads();
    // per expert, the tokens of the earlier warps of this block (one pass, so a
    // token's rank is two shared loads instead of a popcount over every earlier warp)
    for (int e = tid; e < E; e += kPermT) {
        int32_t acc = 0;
#pragma unroll
        for (int q = 0; q < kPermT / 32; ++q) {
            pre[q * E + sw(e)] = acc;
            acc += __popc(bits[q * E + sw(e)]);
        }
    }
    __syncthreads();
    const uint64_t t_bits = tl_now(c);
    const int w = tid >> 5;
    const uint32_t below = (1u << (tid & 31)) - 1u;
    if (t < c.S) {
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            if (j >= k) break;
            const int se = sw(my[j]), i = w * E + se;
            const int32_t p = base[se] + pre[i] + __popc(bits[i] & below);
            c.rows[p] = t;
            c.pos[size_t(t) * k + j] = p;
        }
    }
    if constexpr (DEDUP) {
        // token dedup: this token's row in each remote destination's token buffer
        // (tokens in ascending order per destination: earlier blocks, earlier
        // warps, earlier lanes), stored per (expert, row) slot
        __shared__ int32_t dwarp[kPermT / 32][kMaxPes], dbase[kMaxPes];
        int32_t u_of[kMaxPes];
        unsigned dm = 0;
        if (t < c.S) {
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < k && my[j] % c.P != c.rank) dm |= 1u << (my[j] % c.P);
        }
#pragma unroll
        for (int d = 0; d < kMaxPes; ++d) {
            const unsigned bal = __ballot_sync(0xffffffffu, d < c.P && (dm >> d & 1u));
            if ((tid & 31) == 0) dwarp[w][d] = __popc(bal);
            u_of[d] = __popc(bal & below);
        }
        if (tid < c.P) {
            const int32_t* dh = c.dhist + size_t(c.par) * c.hist_blocks * kMaxPes;
            int32_t before = 0, all = 0;
            for (int q = 0; q < nb; ++q) {
                const int32_t v = dh[size_t(q) * kMaxPes + tid];
                before += q < b ? v : 0;
                all += v;
            }
            dbase[tid] = before;
            if (b == 0) c.dtot[tid] = all;
            c.dhist[(size_t(c.par ^ 1) * c.hist_blocks + b) * kMaxPes + tid] = 0;  // next forward's half
        }
        __syncthreads();
#pragma unroll
        for (int d = 0; d < kMaxPes; ++d) {
            int32_t off = d < c.P ? dbase[d] : 0;
            for (int q = 0; q < w; ++q) off += d < c.P ? dwarp[q][d] : 0;
            u_of[d] += off;
        }
        if (t < c.S) {
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                if (j >= k) break;
                const int d = my[j] % c.P;
                int32_t u = -1;
#pragma unroll
                for (int q = 0; q < kMaxPes; ++q) u = (q == d && d != c.rank) ? u_of[q] : u;
                const int se = sw(my[j]), i = w * E + se;
                c.uidx[base[se] + pre[i] + __popc(bits[i] & below)] = u;
            }
        }
    }
    tl_end(c, kTlPerm, tid == 0);
    if (tid == 0) {
        tl_at(c, kTlPermBlkStart, t_blk);
        tl_at(c, kTlPermHist, t_hist);
        tl_at(c, kTlPermScan, t_scan);
        tl_at(c, kTlPermBits, t_bits);
        tl_mark(c, kTlPermBlkEnd);
    }
}

// ------------------------------------------------------------------ plan ----
// Block-wide exclusive scan of n ints in shared memory (any blockDim that is a
// multiple of 32); returns the total.  Must be called by every thread.
__device__ int32_t block_exclusive_scan(int32_t* a, int n, int32_t* scratch /*33*/) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = tid * per;
    int32_t local = 0;
    for (int i = 0; i < per; ++i)
        if (b + i < n) local += a[b + i];
    int32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) scratch[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int32_t v = lane < nwarps ? scratch[lane] : 0;
        int32_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += u;
        }
        scratch[lane] = wi - v;
        if (lane == 31) scratch[32] = wi;
    }
    __syncthreads();
    int32_t run = scratch[warp] + incl - local;
    for (int i = 0; i < per; ++i)
        if (b + i < n) {
            const int32_t v = a[b + i];
            a[b + i] = run;
            run += v;
        }
    const int32_t total = scratch[32];
    __syncthreads();
    return total;
}

__device__ __forceinline__ int32_t ceil_tiles(int32_t rows) { return (rows + kTileRows - 1) / kTileRows; }

// (The per-forward plan is in plan.cuh, run by k_perm's extra CTA.)

// -------------------------------------------------------------- dispatch ----
// One CTA per send tile: gather the tile's token rows (sorted order) and store
// them into the destination's receive heap — a one-sided NVLink store for a
// peer, a local copy for the self segment — then signal (Phase 1: counter;
// the completing producer runs Phase 2).
__global__ void __launch_bounds__(256) k_dispatch(DevCtx c) {
    tl_start(c, kTlDispatch);
    const PlanHeader hdr = *c.hdr;
    const int i = blockIdx.x;
    if (i >= hdr.n_send || hdr.error) return;
    const SendTile st = c.send[i];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t abs0 = c.offsets[st.expert] + st.row0;
    bf16* dbase = c.heap[st.dst] + (size_t(c.par) * c.R_max + st.heap_row) * c.H;
    const int nvec = c.H / 8;  // 16-byte vectors per row
    for (int rr = warp; rr < st.rows; rr += 8) {
        const int32_t tok = c.rows[abs0 + rr];
        const uint4* src = reinterpret_cast<const uint4*>(c.x + size_t(tok) * c.H);
        uint4* dst = reinterpret_cast<uint4*>(dbase + size_t(rr) * c.H);
        int v = lane;
        for (; v + 96 < nvec; v += 128) {
            const uint4 a = __ldg(src + v), b = __ldg(src + v + 32), d = __ldg(src + v + 64),
                        e = __ldg(src + v + 96);
            dst[v] = a;
            dst[v + 32] = b;
            dst[v + 64] = d;
            dst[v + 96] = e;
        }
        for (; v < nvec; v += 32) dst[v] = __ldg(src + v);
    }
    if (c.tl && threadIdx.x == 0 && i + 4 >= hdr.n_send) atomicMax(c.tl + 2 * kTlDispatch + 1, fwd_now());
    if (st.dst == c.rank) return;  // self segment: ordered by the stream, no signal
    __syncthreads();
    if (warp != 0) return;
    if (lane == 0) {
        atomicAdd(&c.stats[kStatDispatchPuts], 1ull);
        atomicAdd(&c.stats[kStatDispatchBytes], (unsigned long long)st.rows * c.H * 2);
        if (c.trace) trace_ev(c, PERSEUS_EV_DISPATCH_PUT, st.dst, st.tile_id, st.group, uint32_t(st.rows) * c.H * 2, 0, fwd_now());
    }
    const Group g = c.groups[st.group];
    auto flag_of = [&](int m) {
        const SendTile& t = c.send[m];
        return c.dflag[t.dst] + size_t(c.par) * c.T_max + t.tile_id;
    };
    publish_member_warp(c, g, c.group_ctr + st.group, flag_of, c.signaling >= PERSEUS_SIGNAL_NONE,
                        kStatDispatchFences, kStatDispatchSignals);
}

// --------------------------------------------------------------- combine ----
// Wait for every combine tile this rank dispatched to come back, then
// out[t] = sum_j w[t][j] * y[pos(t, j)] in fixed j order (fp32) -> bf16.
// One CTA per token, one thread per 16-byte column chunk.  Only the (at most
// k) combine tiles that carry this token's rows are waited on — the tile of
// sorted slot p is send tile send_first[e] + (p - offsets[e]) / 128.
template <int K, int CPT, bool CS>
__global__ void __launch_bounds__(1024) k_combine(DevCtx c) {
    // TPC tokens per CTA step, TT = H / (8 * CPT) threads per token, CPT 16-byte
    // column chunks per thread (all CPT * k loads in flight).  Grid-stride over
    // token blocks: the launch sizes the grid to the resident CTAs (no partial
    // last wave) or to one block per CTA.
    pdl_wait();
    tl_start(c, kTlCombine);
    const int TT = c.H / (8 * CPT);
    const int tpc = blockDim.x / TT;
    const int tl = threadIdx.x / TT, v = threadIdx.x - tl * TT;
    const int k = K > 0 ? K : c.k;
    const int nblk = (c.S + tpc - 1) / tpc;
    const bf16* y = c.ybuf[c.rank] + size_t(c.par) * c.Y_rows * c.H;
    constexpr int KM = K > 0 ? K : 16;
    unsigned long long waited_max = 0;
    for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int t = blk * tpc + tl;
        const bool live = t < c.S;
        uint64_t t_start = 0;
        if (c.P > 1 && threadIdx.x == 0) t_start = fwd_now();
        if (c.P > 1 && live && v < k && !c.local_combine) {
            const int e = c.ids[size_t(t) * k + v];
            if (e % c.P != c.rank) {
                const int32_t rel = c.pos[size_t(t) * k + v] - c.offsets[e];
                const int sp = c.send_first[e] + rel / kTileRows;
                const int tile = c.send[sp].tile_id;
                if (!wait_flag_geq(c.cflag[c.rank] + size_t(c.par) * c.T_max + tile, c.epoch, kWaitTimeoutNs))
                    atomicAdd(&c.stats[kStatTimeouts], 1ull);
                if (c.trace && atomicExch(c.trace_seen_ep + tile, c.epoch) != c.epoch) {
                    const SendTile st = c.send[sp];  // the tile's rows came back into our sorted slots
                    trace_seen(c, PERSEUS_EV_COMBINE_SEEN, st.dst, tile,
                               c.ybuf[c.rank] + (size_t(c.par) * c.Y_rows + c.offsets[e] + st.row0) * c.H, st.rows);
                }
            }
        }
        __syncthreads();
        if (c.P > 1 && threadIdx.x == 0) waited_max = max(waited_max, (unsigned long long)(fwd_now() - t_start));
        if (!live) continue;
        uint4 u[CPT][KM];
        float w[KM];
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            if (j < k) {
                const int32_t p = c.pos[size_t(t) * k + j];
                w[j] = c.weights[size_t(t) * k + j];
#pragma unroll
                for (int q = 0; q < CPT; ++q)
                {
                    const uint4* src = reinterpret_cast<const uint4*>(y + size_t(p) * c.H + (v + q * TT) * 8);
                    u[q][j] = CS ? __ldcs(src) : *src;  // CS: every y row is read exactly once
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                if (j < k) {
                    const bf16* b = reinterpret_cast<const bf16*>(&u[q][j]);
#pragma unroll
                    for (int z = 0; z < 8; ++z) acc[z] = __fmaf_rn(w[j], __bfloat162float(b[z]), acc[z]);
                }
            }
            uint4 o;
            o.x = pack_bf16(acc[0], acc[1]);
            o.y = pack_bf16(acc[2], acc[3]);
            o.z = pack_bf16(acc[4], acc[5]);
            o.w = pack_bf16(acc[6], acc[7]);
            uint4* dst = reinterpret_cast<uint4*>(c.out + size_t(t) * c.H + (v + q * TT) * 8);
            if (CS) __stcs(dst, o);
            else *dst = o;
        }
    }
    if (c.P > 1 && threadIdx.x == 0) {
        // exposed-communication accounting: the longest any CTA waited for its
        // combine flags; the last CTA folds this forward's timestamps into the stats
        if (waited_max > *reinterpret_cast<volatile unsigned long long*>(c.fwd_t + kFwdWaitMax))
            atomicMax(c.fwd_t + kFwdWaitMax, waited_max);
        __threadfence();
        if (atomicAdd(c.fwd_t + kFwdDoneCtas, 1ull) == gridDim.x - 1) {
            __threadfence();
            volatile unsigned long long* ft = c.fwd_t;
            auto span = [&](int a, int b) { return ft[b] > ft[a] && ft[a] != ~0ull ? ft[b] - ft[a] : 0ull; };
            atomicAdd(&c.stats[kStatDispatchSpanNs], span(kFwdDispFirst, kFwdDispLast));
            atomicAdd(&c.stats[kStatCombineSpanNs], span(kFwdCombFirst, kFwdCombLast));
            atomicAdd(&c.stats[kStatCombineWaitNs], ft[kFwdWaitMax]);
        }
    }
    tl_end(c, kTlCombine, threadIdx.x == 0);
}

// ------------------------------------------------------------- launchers ----
// bit-exact CUDA-core gate (learned-gate routing)
// (8 tokens per thread; 4 per thread — 32-token tiles, twice the warps per SM —
// was bit-identical but 117 vs 95 us)
void launch_gate_exact(const DevCtx& c, cudaStream_t st) {
    dim3 g((c.S + 63) / 64, (c.E + kGateE - 1) / kGateE);
    k_gate<8><<<g, 256, gate_smem<8>(), st>>>(c.x, c.wg, c.logits, c.S, c.H, c.E);
}

// the per-forward plan (plan.cuh), one CTA of 8 warps
__global__ void __launch_bounds__(kPlanThreads) k_plan4(DevCtx c) {
    pdl_wait();
    pdl_launch_dependents();
    if (c.tl && threadIdx.x == 0) atomicMax(c.tl + 2 * kTlPlan, ~fwd_now());
    extern __shared__ int32_t sm[];
    plan_body(c, sm);
    if (c.tl && threadIdx.x == 0) atomicMax(c.tl + 2 * kTlPlan + 1, fwd_now());
}

// route + permutation + count publish (after the gate logits exist)
// route + permutation + count publish (+ the plan, by one extra CTA of k_perm)
void launch_route(const DevCtx& c, bool with_plan, cudaStream_t st) {
    launch_pdl(k_route, dim3((c.S + 7) / 8), dim3(256), 0, st, c);  // + block histograms
    const int nb = (c.S + kPermT - 1) / kPermT;
    DevCtx cc = c;
    cc.with_plan = with_plan ? 1 : 0;
    const dim3 grid(nb + cc.with_plan);
    const size_t smem = std::max(perm_smem_bytes(c), plan_smem_bytes(c));
    if (c.k == 8)
        launch_pdl(c.dedup ? k_perm<8, true> : k_perm<8, false>, grid, dim3(kPermT), smem, st, cc);  // + count publish
    else
        launch_pdl(c.dedup ? k_perm<0, true> : k_perm<0, false>, grid, dim3(kPermT), smem, st, cc);
}

size_t perm_smem_bytes(const DevCtx& c) {
    // At least 32 KB: the router GEMM (211 KB of shared memory per CTA) runs
    // beside this grid, and a router CTA sharing an SM with the plan CTA
    // doubled the plan's critical path (measured: plan end 22.1 -> 17.0 us into
    // the forward with the reservation).  PERSEUS_PERM_SMEM_KB overrides.
    static const size_t floor_b = [] {
        const char* e = getenv("PERSEUS_PERM_SMEM_KB");
        return e ? size_t(atoi(e)) * 1024 : size_t(32) * 1024;
    }();
    return std::max(floor_b, sizeof(int32_t) * (2 * size_t(c.E) * (kPermT / 32) + 2 * size_t(c.E) + 40 + 2 * kPermT));
}

void launch_plan(const DevCtx& c, cudaStream_t st) {
    launch_pdl(k_plan4, dim3(1), dim3(kPlanThreads), plan_smem_bytes(c), st, c);
}

void launch_dispatch(const DevCtx& c, cudaStream_t st) { k_dispatch<<<c.max_send, 256, 0, st>>>(c); }

// combine variant: chunks per thread (1: one token per CTA; 2: two tokens per
// 256-thread CTA at H = 2048), PERSEUS_COMBINE_CPT overrides (experiments)
static int combine_cpt(const DevCtx& c) {
    static const int env = [] { const char* e = getenv("PERSEUS_COMBINE_CPT"); return e ? atoi(e) : 0; }();
    const int cpt = env > 0 ? env : 2;
    return (c.H % (8 * cpt) == 0 && c.H / (8 * cpt) <= 1024) ? cpt : 1;
}

// Grid of the combine: one token block per CTA (default), or with
// PERSEUS_COMBINE_PERSIST=1 the CTAs that fit at once on the device (occupancy x
// SMs, grid-stride over the token blocks, no partial last wave).  Measured at
// EP=1 (same box, alternating): K-step 351.6 vs 353.0 us, ncu 30.1 vs 30.7 us —
// no gain, so the plain grid stays.
template <typename Kern>
static dim3 combine_grid(Kern kern, int nblk, int block, int num_sms) {
    static const bool persist = [] { const char* e = getenv("PERSEUS_COMBINE_PERSIST"); return e && atoi(e) != 0; }();
    if (!persist) return dim3(nblk);
    // resident CTAs per SM of this kernel at this block size (cached per thread)
    thread_local const void* last_k = nullptr;
    thread_local int last_block = 0, last_per_sm = 0;
    if (last_k != reinterpret_cast<const void*>(kern) || last_block != block) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, 0) != cudaSuccess) {
            (void)cudaGetLastError();
            per_sm = 0;
        }
        last_k = reinterpret_cast<const void*>(kern);
        last_block = block;
        last_per_sm = per_sm;
    }
    if (last_per_sm < 1) return dim3(nblk);
    return dim3(std::min(nblk, last_per_sm * num_sms));
}

template <int CPT, bool CS>
static void launch_combine_cpt(const DevCtx& c, int num_sms, cudaStream_t st) {
    const int tt = c.H / (8 * CPT);                 // threads per token
    const int tpc = std::max(1, 256 / tt);          // tokens per CTA
    const int nblk = (c.S + tpc - 1) / tpc;
    const dim3 block(tt * tpc);
    auto go = [&](auto kern) { launch_pdl(kern, combine_grid(kern, nblk, int(block.x), num_sms), block, 0, st, c); };
    switch (c.k) {
        case 1: go(k_combine<1, CPT, CS>); break;
        case 2: go(k_combine<2, CPT, CS>); break;
        case 4: go(k_combine<4, CPT, CS>); break;
        case 8: go(k_combine<8, CPT, CS>); break;
        default: go(k_combine<0, CPT, CS>); break;
    }
}

// streaming (evict-first) loads of y and stores of out: y rows and out rows are
// touched once, so they should not displace the next forward's x / weights in L2.
// Same-box A/B at EP=1 (tools/ab_combine_cs.sh): combine 40.0 -> 36.8 us.
// PERSEUS_COMBINE_CS=0 restores plain loads/stores (experiments).
static bool combine_cs() {
    static const bool cs = [] { const char* e = getenv("PERSEUS_COMBINE_CS"); return e ? atoi(e) != 0 : true; }();
    return cs;
}

void launch_combine(const DevCtx& c, int num_sms, cudaStream_t st) {
    const bool cs = combine_cs();
    if (combine_cpt(c) == 2) cs ? launch_combine_cpt<2, true>(c, num_sms, st) : launch_combine_cpt<2, false>(c, num_sms, st);
    else cs ? launch_combine_cpt<1, true>(c, num_sms, st) : launch_combine_cpt<1, false>(c, num_sms, st);
}

// Every kernel of the forward asks for the maximum shared-memory carveout, so
// consecutive kernels never wait for an SM to drain and re-split L1/smem (the
// fused and GEMM kernels need it anyway).
template <typename K>
static cudaError_t max_carveout(K* kernel) {
    return cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel), cudaFuncAttributePreferredSharedMemoryCarveout,
                                int(cudaSharedmemCarveoutMaxShared));
}

template <int CPT, bool CS>
static cudaError_t combine_carveouts() {
    const cudaError_t es[] = {max_carveout(k_combine<0, CPT, CS>), max_carveout(k_combine<1, CPT, CS>),
                              max_carveout(k_combine<2, CPT, CS>), max_carveout(k_combine<4, CPT, CS>),
                              max_carveout(k_combine<8, CPT, CS>)};
    for (cudaError_t x : es)
        if (x != cudaSuccess) return x;
    return cudaSuccess;
}

cudaError_t configure_kernels(const DevCtx& c) {
    cudaError_t e = cudaFuncSetAttribute(k_plan4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan_smem_bytes(c)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gate<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gate_smem<8>()));
    if (e != cudaSuccess) return e;
    for (auto f : {k_perm<8, false>, k_perm<8, true>, k_perm<0, false>, k_perm<0, true>}) {
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(std::max(perm_smem_bytes(c), plan_smem_bytes(c))));
        if (e != cudaSuccess) return e;
        e = max_carveout(f);
        if (e != cudaSuccess) return e;
    }
    const cudaError_t es[] = {max_carveout(k_route), max_carveout(k_plan4), max_carveout(k_dispatch),
                              max_carveout(k_gate<8>), max_carveout(k_synth_fill), combine_carveouts<1, false>(),
                              combine_carveouts<2, false>(), combine_carveouts<1, true>(), combine_carveouts<2, true>()};
    for (cudaError_t x : es)
        if (x != cudaSuccess) return x;
    return cudaSuccess;
}

}  // namespace perseus
