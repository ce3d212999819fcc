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
    int32_t n_tiles;     // GATE: token tiles
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
        j.ti = w;
        j.nb = 0;
        j.rows = min(kBM, c.S - w * kBM);
        j.a_row = w * kBM;
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
    }
    const Group grp = c.cgroups[rt.cgroup];
    auto flag_of = [&](int m) {
        const RecvTile& mt = c.recv[m];
        return c.cflag[mt.src] + size_t(c.par) * c.T_max + mt.tile_id;
    };
    publish_member_warp(c, grp, c.cgroup_ctr + rt.cgroup, flag_of, c.signaling == PERSEUS_SIGNAL_NONE,
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
                    fence_proxy_async();
                }
                for (int kb = 0; kb < g.num_kb; ++kb) {
                    uint8_t* sa = smem + stage * kStageBytes;
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], stage_tx);
                    tma_load_2d(sa, &tma_a, &full[stage], kb * kBK, j.a_row);
                    tma_load_2d(sa + kABytes, &tma_b, &full[stage], kb * kBK, j.b0);
                    if (g.nbox == 2) tma_load_2d(sa + kABytes + kBBytes / 2, &tma_b, &full[stage], kb * kBK, j.b1);
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
                float* dst = c.logits + size_t(j.a_row + row) * c.E;
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
    if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

// ----------------------------------------------------------------- host ----
size_t gemm_smem_bytes() { return kGemmSmem; }

cudaError_t configure_gemm() {
    cudaError_t e = cudaFuncSetAttribute(k_gemm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_gemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
}

void launch_gemm(int mode, const CUtensorMap& ta, const CUtensorMap& tb, const DevCtx& c, int n_nb,
                 int num_kb, int64_t a_row_base, int grid, cudaStream_t st) {
    GemmArgs g{n_nb, num_kb, a_row_base, 2, 0};
    if (mode == 1)
        k_gemm<1><<<grid, 256, kGemmSmem, st>>>(ta, tb, c, g);
    else
        k_gemm<2><<<grid, 256, kGemmSmem, st>>>(ta, tb, c, g);
}

// Router logits on the tensor cores: one 128-token M-tile per work item,
// N = 128 (E <= 128) or 256 (E <= 256) expert columns, K = H.
void launch_gate_tc(const CUtensorMap& tx, const CUtensorMap& twg, const DevCtx& c, int grid, cudaStream_t st) {
    const int tiles = (c.S + kBM - 1) / kBM;
    GemmArgs g{1, c.H / kBK, 0, c.E > 128 ? 2 : 1, tiles};
    k_gemm<0><<<std::min(grid, tiles), 256, kGemmSmem, st>>>(tx, twg, c, g);
}

}  // namespace perseus
