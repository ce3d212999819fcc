// gemm.cu — grouped expert-FFN GEMMs on the 5th-gen tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel per GEMM of the SwiGLU FFN over the
// ragged list of M-tiles (RecvTile) the plan produced (plus the router GEMM):
//   GATE : logits = x * Wg^T (fp32 out; reference routing modes only — the
//          learned-gate mode uses the bit-exact CUDA-core kernel)
//   GEMM1: [gate|up] = A * W1_e^T   (A = received token rows, K = H)
//          epilogue: h = silu(gate) * up  -> bf16 h rows
//   GEMM2: y = h * W2_e^T           (K = I)
//          epilogue: bf16 y rows pushed straight into the token owner's
//          combine buffer (TMA bulk stores — over NVLink for a peer) + per-tile
//          / per-group release signalling: the compute->collective fusion.
//
// Roles (256 threads, 1 CTA/SM): warp0 = TMA producer, warp1 = MMA issuer
// (one thread issues tcgen05.mma), warp2 = TMEM allocator, warps4-7 =
// epilogue (TMEM -> registers -> global).  A 4-stage smem ring of 48 KB
// (A 128x64 + B 256x64 bf16, 128B-swizzled, TMA-fed) and a double-buffered
// 2 x 256-column fp32 accumulator in TMEM let the epilogue of tile i overlap
// the MMAs of tile i+1.  UMMA shape M=128, N=256, K=16 (kind::f16).
//
// (Self-tile rows gathered straight from x instead of the dispatched heap —
// TMA tile::gather4, or 16-byte cp.async from the producer warp — measured
// 2.5x slower: 512 B per TMA request caps the gather at ~6 B/cycle/SM.)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "layer_dev.h"
#include "perseus.h"
#include "ptx.cuh"
#include "signal.cuh"

namespace perseus {

using namespace ptx;

constexpr int kStages = 4;
constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr int kABytes = kBM * kBK * 2;      // 16 KB
constexpr int kBBytes = kBN * kBK * 2;      // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kTmemCols = 512;              // 2 accumulators x 256 fp32 columns
constexpr int kStgRow = 128 + 16;           // GEMM2 staging row: 64 bf16 + pad (conflict-free)
constexpr int kStgBytes = 128 * kStgRow;    // 4 epilogue warps x 32 rows
constexpr size_t kGemmSmem = 1024 + size_t(kStages) * kStageBytes + kStgBytes + 256;

struct GemmArgs {
    int32_t n_nb;        // N blocks per M-tile
    int32_t num_kb;      // K blocks of 64
    int64_t a_row_base;  // row offset of this forward's A buffer in the A tensor map
    int32_t nbox;        // B boxes of 128 rows per stage (UMMA N = 128 * nbox)
    int32_t n_tiles;     // GATE: token tiles x K splits (work items)
    int32_t ksplit;      // GATE: K splits (partial logits summed by k_route)
};

// What one work item loads and where its rows go.
struct Job {
    int32_t ti, nb, rows;
    int32_t a_row, b0, b1;
};

template <int kMode>
__device__ __forceinline__ Job job_of(int w, const DevCtx& c, const GemmArgs& g, RecvTile& rt) {
    Job j;
    if (kMode == 0) {
        j.ti = w / g.ksplit;
        j.nb = w % g.ksplit;  // K split index
        j.rows = min(kBM, c.S - j.ti * kBM);
        j.a_row = j.ti * kBM;
        j.b0 = 0;
        j.b1 = 128;
        return j;
    }
    j.ti = w / g.n_nb;
    j.nb = w % g.n_nb;
    rt = c.recv[j.ti];
    j.rows = rt.rows;
    j.a_row = int32_t(g.a_row_base + rt.heap_row);
    if (kMode == 1) {
        j.b0 = rt.e_local * 2 * c.I + j.nb * 128;
        j.b1 = j.b0 + c.I;
    } else {
        j.b0 = rt.e_local * c.H + j.nb * 256;
        j.b1 = j.b0 + 128;
    }
    return j;
}

__device__ __forceinline__ float silu_mul(float g, float u) {
    return __fdividef(g, 1.0f + __expf(-g)) * u;
}

// GEMM2 tile completion, run by the 4 epilogue warps after the tile's bulk
// stores have COMPLETED: the n-block that finishes a remote M-tile publishes
// it (Phase 1 counter) and the group's completing warp runs Phase 2.
__device__ __forceinline__ void finish_tile(const DevCtx& c, const GemmArgs& g, int ti, int nb) {
    named_bar_sync(1, 128);
    if ((threadIdx.x >> 5) != 4) return;
    const int lane = threadIdx.x & 31;
    const RecvTile rt = c.recv[ti];
    if (lane == 0 && nb == 0) atomicAdd(&c.stats[kStatRecvTiles], 1ull);
    if (rt.cgroup < 0) return;
    uint32_t done = 0;
    if (lane == 0) done = atom_add_acq_rel_gpu(c.tile_ctr + ti, 1u) + 1 == uint32_t(g.n_nb);
    if (!__shfl_sync(0xffffffffu, done, 0)) return;
    if (lane == 0) {
        atomicAdd(&c.stats[kStatCombinePuts], 1ull);
        atomicAdd(&c.stats[kStatCombineBytes], (unsigned long long)rt.rows * c.H * 2);
        if (c.trace) trace_ev(c, PERSEUS_EV_COMBINE_PUT, rt.src, rt.tile_id, rt.cgroup, uint32_t(rt.rows) * c.H * 2, 0, fwd_now());
    }
    const Group grp = c.cgroups[rt.cgroup];
    auto flag_of = [&](int m) {
        const RecvTile& mt = c.recv[m];
        return c.cflag[mt.src] + size_t(c.par) * c.T_max + mt.tile_id;
    };
    publish_member_warp(c, grp, c.cgroup_ctr + rt.cgroup, flag_of, c.signaling >= PERSEUS_SIGNAL_NONE,
                        kStatCombineFences, kStatCombineSignals);
}

template <int kMode>
__global__ void __launch_bounds__(256, 1)
    k_gemm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
           DevCtx c, GemmArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_out = smem + kStages * kStageBytes;  // GEMM2 epilogue staging
    uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + kStgBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    constexpr int kTlId = kMode == 0 ? kTlGate : (kMode == 1 ? kTlGemm1 : kTlGemm2);
    // router between the plan and the fused kernel (gate_inline): it reads only
    // x and the router weights, so it neither waits for the plan nor holds the
    // fused kernel's launch (which waits for this grid — and, transitively,
    // the plan — at its pdl_wait)
    if (kMode == 0 && c.gate_inline) pdl_launch_dependents();
    tl_start(c, kTlId);
    int total;
    if (kMode == 0) {
        total = g.n_tiles;
    } else {
        const PlanHeader hdr = *c.hdr;
        if (hdr.error) return;
        total = hdr.n_recv * g.n_nb;
    }
    const int warp = warp_id(), lane = lane_id();
    const uint32_t stage_tx = kABytes + uint32_t(g.nbox) * (kBBytes / 2);
    const uint32_t idesc = idesc_bf16_f32(kBM, 128 * g.nbox);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tma_a);
        tma_prefetch_desc(&tma_b);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        tmem_alloc(tmem_holder, kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (one thread) ----------------
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t* dflags = c.dflag[c.rank] + size_t(c.par) * c.T_max;
            for (int w = blockIdx.x; w < total; w += gridDim.x) {
                RecvTile rt;
                const Job j = job_of<kMode>(w, c, g, rt);
                if (kMode == 1 && rt.tile_id >= 0) {
                    // the tile's dispatch signal: its rows are in our heap
                    if (!wait_flag_geq(dflags + rt.tile_id, c.epoch, kWaitTimeoutNs))
                        atomicAdd(&c.stats[kStatTimeouts], 1ull);
                    if (c.trace && j.nb == 0)
                        trace_seen(c, PERSEUS_EV_DISPATCH_SEEN, rt.src, rt.tile_id,
                                   c.heap[c.rank] + (size_t(c.par) * c.R_max + rt.heap_row) * c.H, rt.rows);
                    fence_proxy_async();
                }
                for (int kb = 0; kb < g.num_kb; ++kb) {
                    uint8_t* sa = smem + stage * kStageBytes;
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], stage_tx);
                    const int kc = (kMode == 0 ? j.nb * g.num_kb + kb : kb) * kBK;
                    tma_load_2d(sa, &tma_a, &full[stage], kc, j.a_row);
                    tma_load_2d(sa + kABytes, &tma_b, &full[stage], kc, j.b0);
                    if (g.nbox == 2) tma_load_2d(sa + kABytes + kBBytes / 2, &tma_b, &full[stage], kc, j.b1);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread) ----------------
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int w = blockIdx.x; w < total; w += gridDim.x) {
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * kBN);
                for (int kb = 0; kb < g.num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    uint8_t* sa = smem + stage * kStageBytes;
                    const uint64_t adesc = smem_desc_sw128(sa);
                    const uint64_t bdesc = smem_desc_sw128(sa + kABytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)  // +32 B along K inside the swizzle atom
                        umma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
                    umma_commit(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                umma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (4 warps = 4 TMEM lane quadrants) ----------------
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int acc = 0;
        uint32_t aphase = 0;
        int pend_ti = -1, pend_nb = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            RecvTile rt;
            const Job j = job_of<kMode>(w, c, g, rt);
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            const bool valid = row < j.rows;
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kBN);
            if (kMode == 0) {
                // router logits, fp32 [S][E]
                float* dst = c.logits + (size_t(j.nb) * c.S + j.a_row + row) * c.E;
#pragma unroll 1
                for (int cc = 0; cc < c.E; cc += 32) {
                    uint32_t v32[32];
                    tmem_ld_32x32b_x32(taddr + cc, v32);
                    tmem_ld_wait();
                    if (valid) {
                        if (cc + 32 <= c.E && (c.E & 3) == 0) {
#pragma unroll
                            for (int v = 0; v < 8; ++v)
                                st_global_v4(dst + cc + 4 * v, v32[4 * v], v32[4 * v + 1], v32[4 * v + 2], v32[4 * v + 3]);
                        } else {
                            for (int i = 0; i < 32 && cc + i < c.E; ++i) dst[cc + i] = __uint_as_float(v32[i]);
                        }
                    }
                }
            } else if (kMode == 1) {
                bf16* dst = c.hbuf + size_t(rt.heap_row + row) * c.I + j.nb * 128;
#pragma unroll 1
                for (int cc = 0; cc < 128; cc += 32) {
                    uint32_t gv[32], uv[32];
                    tmem_ld_32x32b_x32(taddr + cc, gv);
                    tmem_ld_32x32b_x32(taddr + 128 + cc, uv);
                    tmem_ld_wait();
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        pk[i] = pack_bf16(silu_mul(__uint_as_float(gv[2 * i]), __uint_as_float(uv[2 * i])),
                                          silu_mul(__uint_as_float(gv[2 * i + 1]), __uint_as_float(uv[2 * i + 1])));
                    if (valid) {
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            st_global_v4(dst + cc + v * 8, pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                    }
                }
            } else {
                // y rows go to the token owner's combine buffer — over NVLink
                // for a peer.  Each warp stages its 32 rows x 64 columns in
                // shared memory and every lane pushes its row segment (128 B)
                // with one TMA bulk copy: whole-row writes instead of 16 B
                // scattered stores.
                bf16* dst = c.ybuf[rt.src] +
                            (size_t(c.par) * c.Y_rows + size_t(rt.ybuf_row + row)) * c.H + j.nb * 256;
                if (rt.src == c.rank) {
                    // local owner: plain 16 B stores (L2 write-combines them)
#pragma unroll 1
                    for (int cc = 0; cc < 256; cc += 32) {
                        uint32_t v32[32];
                        tmem_ld_32x32b_x32(taddr + cc, v32);
                        tmem_ld_wait();
                        if (valid) {
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                st_global_v4(dst + cc + v * 8,
                                             pack_bf16(__uint_as_float(v32[8 * v]), __uint_as_float(v32[8 * v + 1])),
                                             pack_bf16(__uint_as_float(v32[8 * v + 2]), __uint_as_float(v32[8 * v + 3])),
                                             pack_bf16(__uint_as_float(v32[8 * v + 4]), __uint_as_float(v32[8 * v + 5])),
                                             pack_bf16(__uint_as_float(v32[8 * v + 6]), __uint_as_float(v32[8 * v + 7])));
                        }
                    }
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) bulk_commit();  // keep 4 groups per tile on every lane
                } else {
                uint8_t* srow_p = stage_out + (q * 32 + lane) * kStgRow;
                const uint32_t srow = smem_u32(srow_p);
#pragma unroll 1
                for (int cc = 0; cc < 256; cc += 64) {
                    uint32_t v0[32], v1[32];
                    tmem_ld_32x32b_x32(taddr + cc, v0);
                    tmem_ld_32x32b_x32(taddr + cc + 32, v1);
                    tmem_ld_wait();
                    bulk_wait_read0();  // this lane's previous segment has left smem
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        st_shared_v4(srow + v * 16, pack_bf16(__uint_as_float(v0[8 * v]), __uint_as_float(v0[8 * v + 1])),
                                     pack_bf16(__uint_as_float(v0[8 * v + 2]), __uint_as_float(v0[8 * v + 3])),
                                     pack_bf16(__uint_as_float(v0[8 * v + 4]), __uint_as_float(v0[8 * v + 5])),
                                     pack_bf16(__uint_as_float(v0[8 * v + 6]), __uint_as_float(v0[8 * v + 7])));
                        st_shared_v4(srow + 64 + v * 16, pack_bf16(__uint_as_float(v1[8 * v]), __uint_as_float(v1[8 * v + 1])),
                                     pack_bf16(__uint_as_float(v1[8 * v + 2]), __uint_as_float(v1[8 * v + 3])),
                                     pack_bf16(__uint_as_float(v1[8 * v + 4]), __uint_as_float(v1[8 * v + 5])),
                                     pack_bf16(__uint_as_float(v1[8 * v + 6]), __uint_as_float(v1[8 * v + 7])));
                    }
                    fence_proxy_async_smem();
                    if (valid) bulk_store(dst + cc, srow_p, 128);
                    bulk_commit();  // one group per chunk on every lane (uniform counts)
                }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (kMode == 2) {
                // Signal the PREVIOUS tile of this CTA once its 4 bulk groups
                // completed (this tile's 4 stay in flight): the epilogue never
                // idles on NVLink write acknowledgements.
                if (pend_ti >= 0) {
                    bulk_wait<4>();
                    fence_proxy_async();  // async-proxy writes -> generic release
                    finish_tile(c, g, pend_ti, pend_nb);
                }
                pend_ti = j.ti;
                pend_nb = j.nb;
            }
            if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
        if (kMode == 2 && pend_ti >= 0) {
            bulk_wait0();
            fence_proxy_async();
            finish_tile(c, g, pend_ti, pend_nb);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    tl_end(c, kTlId, threadIdx.x == 0);
    if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

// ======================================================= fused forward ====
// k_moe: ONE persistent kernel (1 CTA per SM, cooperative launch) that runs
// the dispatch puts, GEMM1+SwiGLU and GEMM2+combine-put of a forward with
// tile-granular dependencies instead of kernel boundaries:
//   warps 2-3 (copy warps): stream 16-row units of the send tiles, in the
//     rotated destination order, into the destination heaps (NVLink stores
//     for peers); the warp completing a tile runs Perseus Phase 1/2, or marks
//     a self tile ready (gpu-scope release).
//   warp 0 (scheduler + TMA producer): grabs work items from a global atomic
//     counter — GEMM1 items of the M-tiles in arrival order, GEMM2 items of the
//     same tiles `lag` tiles behind — pushes them through an smem ring to the
//     MMA and epilogue warps, waits each item's dependency (dispatch flag /
//     self-ready flag / all GEMM1 n-blocks of the tile done), then streams
//     its A/B k-blocks with TMA.
//   warp 1: tcgen05.mma issuer; warps 4-7: epilogues (h rows; y rows pushed
//     to the owner + combine-direction signalling).
// Every item depends only on items with a smaller index, on copy units (which
// never wait) and on other GPUs' copy units, so co-residency makes it
// deadlock-free.
struct FusedArgs {
    int32_t n1, n2;     // N blocks of GEMM1 (I/128) and GEMM2 (H/256)
    int32_t kb1, kb2;   // K blocks of GEMM1 (H/64) and GEMM2 (I/64)
    int32_t lag;        // GEMM2 items trail GEMM1 items by this many M-tiles
    int32_t pad;
    int64_t a1_row_base;
};

struct Item {
    int32_t kind, t, nb;  // kind 1 = GEMM1, 2 = GEMM2, 0 = none
};

__device__ __forceinline__ Item item_of(int w, int T, const FusedArgs& f) {
    const int L = min(f.lag, T), n1 = f.n1, n2 = f.n2;
    if (w < L * n1) return {1, w / n1, w % n1};
    w -= L * n1;
    const int steady = (T - L) * (n1 + n2);
    if (w < steady) {
        const int st = w / (n1 + n2), r = w % (n1 + n2);
        return r < n1 ? Item{1, L + st, r} : Item{2, st, r - n1};
    }
    w -= steady;
    if (w < L * n2) return {2, T - L + w / n2, w % n2};
    return {0, 0, 0};
}

constexpr int kRing = 8;
constexpr int kUnitRows = 2;
constexpr int kUnitsPerTile = kTileRows / kUnitRows;

__device__ __forceinline__ void copy_unit_warp(const DevCtx& c, const SendTile& st, int r0, int nrows, int lane) {
    const int32_t abs0 = c.offsets[st.expert] + st.row0 + r0;
    bf16* dbase = c.heap[st.dst] + (size_t(c.par) * c.R_max + st.heap_row + r0) * c.H;
    const int nvec = c.H / 8;
    for (int rr = 0; rr < nrows; ++rr) {
        const int32_t tok = c.rows[abs0 + rr];
        const uint4* src = reinterpret_cast<const uint4*>(c.x + size_t(tok) * c.H);
        uint4* dst = reinterpret_cast<uint4*>(dbase + size_t(rr) * c.H);
        int v = lane;
        for (; v + 224 < nvec; v += 256) {
            uint4 a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __ldg(src + v + 32 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) dst[v + 32 * u] = a[u];
        }
        for (; v < nvec; v += 32) dst[v] = __ldg(src + v);
    }
}

__global__ void __launch_bounds__(256, 1)
    k_moe(const __grid_constant__ CUtensorMap tm_a1, const __grid_constant__ CUtensorMap tm_b1,
          const __grid_constant__ CUtensorMap tm_a2, const __grid_constant__ CUtensorMap tm_b2, DevCtx c,
          FusedArgs f) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_out = smem + kStages * kStageBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + kStgBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* rfull = tempty + 2;
    uint64_t* rempty = rfull + kRing;
    int32_t* ring = reinterpret_cast<int32_t*>(rempty + kRing);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ring + kRing);

    const PlanHeader hdr = *c.hdr;
    if (hdr.error) return;
    const int T = hdr.n_recv;
    const int total = T * (f.n1 + f.n2);
    const int warp = warp_id(), lane = lane_id();
    const uint32_t idesc = idesc_bf16_f32(kBM, kBN);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_a1);
        tma_prefetch_desc(&tm_b1);
        tma_prefetch_desc(&tm_a2);
        tma_prefetch_desc(&tm_b2);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&rfull[s], 1);
            mbar_init(&rempty[s], 5);  // MMA thread + 4 epilogue warps
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        tmem_alloc(tmem_holder, kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- scheduler + TMA producer ----------------
            int stage = 0, slot = 0;
            uint32_t phase = 0, rphase = 0;
            const uint32_t* dflags = c.dflag[c.rank] + size_t(c.par) * c.T_max;
            while (true) {
                const int w = int(atomicAdd(&c.sched[0], 1u));
                const Item it = w < total ? item_of(w, T, f) : Item{0, 0, 0};
                mbar_wait(&rempty[slot], rphase ^ 1);
                ring[slot] = it.kind ? w : -1;
                mbar_arrive(&rfull[slot]);
                if (++slot == kRing) { slot = 0; rphase ^= 1; }
                if (!it.kind) break;
                const int p = c.rorder[it.t];
                const RecvTile rt = c.recv[p];
                int32_t a_row, b0, b1, nkb;
                const CUtensorMap* ta;
                const CUtensorMap* tb;
                if (it.kind == 1) {
                    const bool ok = rt.tile_id >= 0 ? (c.local_dispatch || wait_flag_geq(dflags + rt.tile_id, c.epoch, kWaitTimeoutNs))
                                                    : wait_flag_geq(c.self_ready + p, c.epoch, kWaitTimeoutNs);
                    if (!ok) atomicAdd(&c.stats[kStatTimeouts], 1ull);
                    a_row = int32_t(f.a1_row_base + rt.heap_row);
                    b0 = rt.e_local * 2 * c.I + it.nb * 128;
                    b1 = b0 + c.I;
                    nkb = f.kb1;
                    ta = &tm_a1;
                    tb = &tm_b1;
                } else {
                    if (!wait_flag_geq(c.g1_done + p, uint32_t(f.n1), kWaitTimeoutNs))
                        atomicAdd(&c.stats[kStatTimeouts], 1ull);
                    a_row = int32_t(rt.heap_row);
                    b0 = rt.e_local * c.H + it.nb * 256;
                    b1 = b0 + 128;
                    nkb = f.kb2;
                    ta = &tm_a2;
                    tb = &tm_b2;
                }
                fence_proxy_async();  // generic writes observed above -> TMA reads
                for (int kb = 0; kb < nkb; ++kb) {
                    uint8_t* sa = smem + stage * kStageBytes;
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], kStageBytes);
                    tma_load_2d(sa, ta, &full[stage], kb * kBK, a_row);
                    tma_load_2d(sa + kABytes, tb, &full[stage], kb * kBK, b0);
                    tma_load_2d(sa + kABytes + kBBytes / 2, tb, &full[stage], kb * kBK, b1);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            int stage = 0, slot = 0, acc = 0;
            uint32_t phase = 0, rphase = 0, aphase = 0;
            while (true) {
                mbar_wait(&rfull[slot], rphase);
                const int w = ring[slot];
                mbar_arrive(&rempty[slot]);
                if (++slot == kRing) { slot = 0; rphase ^= 1; }
                if (w < 0) break;
                const Item it = item_of(w, T, f);
                const int nkb = it.kind == 1 ? f.kb1 : f.kb2;
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * kBN);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    uint8_t* sa = smem + stage * kStageBytes;
                    const uint64_t adesc = smem_desc_sw128(sa);
                    const uint64_t bdesc = smem_desc_sw128(sa + kABytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        umma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
                    umma_commit(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                umma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else if (warp < 4) {
        // ---------------- copy warps: dispatch puts ----------------
        // self queue (warp 2 first) and remote queue (warp 3 first), as in k_moe2
        const int remote_units = hdr.n_send_remote * kUnitsPerTile;
        const int self_units = (hdr.n_send - hdr.n_send_remote) * kUnitsPerTile;
        bool remote_q = warp == 3, other_done = false;
        while (true) {
            int u = 0;
            if (lane == 0) u = int(atomicAdd(&c.sched[remote_q ? 1 : 2], 1u));
            u = __shfl_sync(0xffffffffu, u, 0);
            if (u >= (remote_q ? remote_units : self_units)) {
                if (other_done) break;
                other_done = true;
                remote_q = !remote_q;
                continue;
            }
            const int sp = remote_q ? c.sorder[u / kUnitsPerTile] : hdr.n_send_remote + u / kUnitsPerTile;
            const SendTile st = c.send[sp];
            const int r0 = (u % kUnitsPerTile) * kUnitRows;
            if (r0 >= st.rows) continue;
            const int nrows = min(kUnitRows, st.rows - r0);
            copy_unit_warp(c, st, r0, nrows, lane);
            __syncwarp();
            uint32_t done = 0;
            if (lane == 0) done = atom_add_acq_rel_gpu(c.send_done + sp, uint32_t(nrows)) + nrows == uint32_t(st.rows);
            if (!__shfl_sync(0xffffffffu, done, 0)) continue;
            if (st.dst == c.rank) {
                if (lane == 0) st_release_gpu(c.self_ready + st.recv_pos, c.epoch);
                continue;
            }
            if (lane == 0) {
                atomicAdd(&c.stats[kStatDispatchPuts], 1ull);
                atomicAdd(&c.stats[kStatDispatchBytes], (unsigned long long)st.rows * c.H * 2);
            }
            const Group g = c.groups[st.group];
            auto flag_of = [&](int m) {
                const SendTile& t = c.send[m];
                return c.dflag[t.dst] + size_t(c.par) * c.T_max + t.tile_id;
            };
            publish_member_warp(c, g, c.group_ctr + st.group, flag_of, c.signaling >= PERSEUS_SIGNAL_NONE,
                                kStatDispatchFences, kStatDispatchSignals);
        }
        // the routing weights (router GEMM ran on a side stream), after the puts
        if (c.weights_late)
            for (int t = blockIdx.x * 2 + (warp - 2); t < c.S; t += gridDim.x * 2) route_weights_warp(c, t, lane);
    } else {
        // ---------------- epilogue (4 warps = 4 TMEM lane quadrants) ----------------
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int acc = 0, slot = 0;
        uint32_t aphase = 0, rphase = 0;
        int pend_ti = -1, pend_nb = 0;
        GemmArgs g2{f.n2, f.kb2, 0, 2, 0, 1};
        while (true) {
            mbar_wait(&rfull[slot], rphase);
            const int w = ring[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&rempty[slot]);
            if (++slot == kRing) { slot = 0; rphase ^= 1; }
            if (w < 0) break;
            const Item it = item_of(w, T, f);
            const int p = c.rorder[it.t];
            const RecvTile rt = c.recv[p];
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            const bool valid = row < rt.rows;
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kBN);
            if (it.kind == 1) {
                bf16* dst = c.hbuf + size_t(rt.heap_row + row) * c.I + it.nb * 128;
#pragma unroll 1
                for (int cc = 0; cc < 128; cc += 32) {
                    uint32_t gv[32], uv[32];
                    tmem_ld_32x32b_x32(taddr + cc, gv);
                    tmem_ld_32x32b_x32(taddr + 128 + cc, uv);
                    tmem_ld_wait();
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        pk[i] = pack_bf16(silu_mul(__uint_as_float(gv[2 * i]), __uint_as_float(uv[2 * i])),
                                          silu_mul(__uint_as_float(gv[2 * i + 1]), __uint_as_float(uv[2 * i + 1])));
                    if (valid) {
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            st_global_v4(dst + cc + v * 8, pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                // publish the h n-block: GEMM2 items of this tile wait for all n1
                named_bar_sync(2, 128);
                if (threadIdx.x == 128) atom_add_acq_rel_gpu(c.g1_done + p, 1u);
            } else {
                bf16* dst = c.ybuf[rt.src] +
                            (size_t(c.par) * c.Y_rows + size_t(rt.ybuf_row + row)) * c.H + it.nb * 256;
                if (rt.src == c.rank) {
#pragma unroll 1
                    for (int cc = 0; cc < 256; cc += 32) {
                        uint32_t v32[32];
                        tmem_ld_32x32b_x32(taddr + cc, v32);
                        tmem_ld_wait();
                        if (valid) {
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                st_global_v4(dst + cc + v * 8,
                                             pack_bf16(__uint_as_float(v32[8 * v]), __uint_as_float(v32[8 * v + 1])),
                                             pack_bf16(__uint_as_float(v32[8 * v + 2]), __uint_as_float(v32[8 * v + 3])),
                                             pack_bf16(__uint_as_float(v32[8 * v + 4]), __uint_as_float(v32[8 * v + 5])),
                                             pack_bf16(__uint_as_float(v32[8 * v + 6]), __uint_as_float(v32[8 * v + 7])));
                        }
                    }
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) bulk_commit();
                } else {
                    uint8_t* srow_p = stage_out + (q * 32 + lane) * kStgRow;
                    const uint32_t srow = smem_u32(srow_p);
#pragma unroll 1
                    for (int cc = 0; cc < 256; cc += 64) {
                        uint32_t v0[32], v1[32];
                        tmem_ld_32x32b_x32(taddr + cc, v0);
                        tmem_ld_32x32b_x32(taddr + cc + 32, v1);
                        tmem_ld_wait();
                        bulk_wait_read0();
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            st_shared_v4(srow + v * 16, pack_bf16(__uint_as_float(v0[8 * v]), __uint_as_float(v0[8 * v + 1])),
                                         pack_bf16(__uint_as_float(v0[8 * v + 2]), __uint_as_float(v0[8 * v + 3])),
                                         pack_bf16(__uint_as_float(v0[8 * v + 4]), __uint_as_float(v0[8 * v + 5])),
                                         pack_bf16(__uint_as_float(v0[8 * v + 6]), __uint_as_float(v0[8 * v + 7])));
                            st_shared_v4(srow + 64 + v * 16, pack_bf16(__uint_as_float(v1[8 * v]), __uint_as_float(v1[8 * v + 1])),
                                         pack_bf16(__uint_as_float(v1[8 * v + 2]), __uint_as_float(v1[8 * v + 3])),
                                         pack_bf16(__uint_as_float(v1[8 * v + 4]), __uint_as_float(v1[8 * v + 5])),
                                         pack_bf16(__uint_as_float(v1[8 * v + 6]), __uint_as_float(v1[8 * v + 7])));
                        }
                        fence_proxy_async_smem();
                        if (valid) bulk_store(dst + cc, srow_p, 128);
                        bulk_commit();
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                if (pend_ti >= 0) {
                    bulk_wait<4>();
                    fence_proxy_async();
                    finish_tile(c, g2, pend_ti, pend_nb);
                }
                pend_ti = p;
                pend_nb = it.nb;
            }
            if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
        if (pend_ti >= 0) {
            bulk_wait0();
            fence_proxy_async();
            finish_tile(c, g2, pend_ti, pend_nb);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

constexpr size_t kMoeSmem = kGemmSmem + 256;

// ----------------------------------------------------------------- host ----
size_t gemm_smem_bytes() { return kGemmSmem; }

cudaError_t configure_moe() {
    return cudaFuncSetAttribute(k_moe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMoeSmem));
}

cudaError_t launch_moe(const CUtensorMap& a1, const CUtensorMap& b1, const CUtensorMap& a2, const CUtensorMap& b2,
                       const DevCtx& c, int64_t a1_row_base, int grid, cudaStream_t st) {
    FusedArgs f;
    f.n1 = c.I / 128;
    f.n2 = c.H / 256;
    f.kb1 = c.H / kBK;
    f.kb2 = c.I / kBK;
    f.lag = std::max(1, (2 * grid + f.n1 - 1) / f.n1);
    f.pad = 0;
    f.a1_row_base = a1_row_base;
    DevCtx cc = c;
    void* args[] = {const_cast<CUtensorMap*>(&a1), const_cast<CUtensorMap*>(&b1), const_cast<CUtensorMap*>(&a2),
                    const_cast<CUtensorMap*>(&b2), &cc, &f};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = kMoeSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: tile dependencies cross CTAs
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k_moe), args);
}

cudaError_t configure_gemm() {
    cudaError_t e = cudaFuncSetAttribute(k_gemm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_gemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
}

void launch_gemm(int mode, const CUtensorMap& ta, const CUtensorMap& tb, const DevCtx& c, int n_nb,
                 int num_kb, int64_t a_row_base, int grid, cudaStream_t st) {
    GemmArgs g{n_nb, num_kb, a_row_base, 2, 0, 1};
    if (mode == 1)
        k_gemm<1><<<grid, 256, kGemmSmem, st>>>(ta, tb, c, g);
    else
        k_gemm<2><<<grid, 256, kGemmSmem, st>>>(ta, tb, c, g);
}

// Router logits on the tensor cores: one 128-token M-tile per work item,
// N = 128 (E <= 128) or 256 (E <= 256) expert columns, K = H.
void launch_gate_tc(const CUtensorMap& tx, const CUtensorMap& twg, const DevCtx& c, int grid, cudaStream_t st) {
    const int tiles = (c.S + kBM - 1) / kBM;
    const int ks = c.gate_splits;
    GemmArgs g{1, c.H / kBK / ks, 0, c.E > 128 ? 2 : 1, tiles * ks, ks};
    if (c.gate_inline && c.pdl) {
        // behind the permute/plan kernel, launched early (it reads only x and
        // the router weights; see run_phase)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(std::min(grid, tiles * ks));
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = kGemmSmem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        (void)cudaLaunchKernelEx(&cfg, k_gemm<0>, tx, twg, c, g);
        return;
    }
    k_gemm<0><<<std::min(grid, tiles * ks), 256, kGemmSmem, st>>>(tx, twg, c, g);
}

}  // namespace perseus
