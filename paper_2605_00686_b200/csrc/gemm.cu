// gemm.cu — grouped expert-FFN GEMMs on the 5th-gen tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel per GEMM of the SwiGLU FFN over the
// ragged list of M-tiles (RecvTile) the plan produced:
//   GEMM1: [gate|up] = A * W1_e^T   (A = received token rows, K = H)
//          epilogue: h = silu(gate) * up  -> bf16 h rows
//   GEMM2: y = h * W2_e^T           (K = I)
//          epilogue: bf16 y rows stored straight into the token owner's
//          combine buffer (a one-sided NVLink store for a peer) + per-tile /
//          per-group release signalling — the compute->collective fusion.
//
// Roles (256 threads, 1 CTA/SM): warp0 = TMA producer, warp1 = MMA issuer
// (one thread issues tcgen05.mma), warp2 = TMEM allocator, warps4-7 =
// epilogue (TMEM -> registers -> global).  A 4-stage smem ring of 48 KB
// (A 128x64 + B 256x64 bf16, 128B-swizzled, TMA-fed) and a double-buffered
// 2 x 256-column fp32 accumulator in TMEM let the epilogue of tile i overlap
// the MMAs of tile i+1.  UMMA shape M=128, N=256, K=16 (kind::f16).
#include <cuda.h>
#include <cuda_runtime.h>

#include "layer_dev.h"
#include "perseus.h"
#include "ptx.cuh"

namespace perseus {

using namespace ptx;

constexpr int kStages = 4;
constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr int kABytes = kBM * kBK * 2;      // 16 KB
constexpr int kBBytes = kBN * kBK * 2;      // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kTmemCols = 512;              // 2 accumulators x 256 fp32 columns
constexpr uint32_t kIdesc = idesc_bf16_f32(kBM, kBN);
constexpr size_t kGemmSmem = 1024 + size_t(kStages) * kStageBytes + 256;

struct GemmArgs {
    int32_t n_nb;        // N blocks per M-tile
    int32_t num_kb;      // K blocks of 64
    int64_t a_row_base;  // row offset of this forward's A buffer in the A tensor map
};

__device__ __forceinline__ float silu_mul(float g, float u) {
    return __fdividef(g, 1.0f + __expf(-g)) * u;
}

template <int kMode>
__global__ void __launch_bounds__(256, 1)
    k_gemm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
           DevCtx c, GemmArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const PlanHeader hdr = *c.hdr;
    if (hdr.error) return;
    const int warp = warp_id(), lane = lane_id();
    const int total = hdr.n_recv * g.n_nb;

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
            // ---------------- TMA producer ----------------
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t* dflags = c.dflag[c.rank] + size_t(c.par) * c.T_max;
            for (int w = blockIdx.x; w < total; w += gridDim.x) {
                const RecvTile rt = c.recv[w / g.n_nb];
                const int nb = w % g.n_nb;
                if (kMode == 1 && rt.tile_id >= 0) {
                    // the tile's dispatch signal: its rows are in our heap
                    if (!wait_flag_geq(dflags + rt.tile_id, c.epoch, kWaitTimeoutNs))
                        atomicAdd(&c.stats[kStatTimeouts], 1ull);
                    fence_proxy_async();
                }
                const int32_t a_row = int32_t(g.a_row_base + rt.heap_row);
                int32_t b0, b1;
                if (kMode == 1) {
                    b0 = rt.e_local * 2 * c.I + nb * 128;
                    b1 = b0 + c.I;
                } else {
                    b0 = rt.e_local * c.H + nb * 256;
                    b1 = b0 + 128;
                }
                for (int kb = 0; kb < g.num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * kStageBytes;
                    mbar_arrive_expect_tx(&full[stage], kStageBytes);
                    tma_load_2d(sa, &tma_a, &full[stage], kb * kBK, a_row);
                    tma_load_2d(sa + kABytes, &tma_b, &full[stage], kb * kBK, b0);
                    tma_load_2d(sa + kABytes + kBBytes / 2, &tma_b, &full[stage], kb * kBK, b1);
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
                        umma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, kIdesc, (kb | kk) != 0);
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
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            const int ti = w / g.n_nb;
            const RecvTile rt = c.recv[ti];
            const int nb = w % g.n_nb;
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            const bool valid = row < rt.rows;
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kBN);
            if (kMode == 1) {
                bf16* dst = c.hbuf + size_t(rt.heap_row + row) * c.I + nb * 128;
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
                bf16* dst = c.ybuf[rt.src] +
                            (size_t(c.par) * c.Y_rows + size_t(rt.ybuf_row + row)) * c.H + nb * 256;
#pragma unroll 1
                for (int cc = 0; cc < 256; cc += 32) {
                    uint32_t v32[32];
                    tmem_ld_32x32b_x32(taddr + cc, v32);
                    tmem_ld_wait();
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        pk[i] = pack_bf16(__uint_as_float(v32[2 * i]), __uint_as_float(v32[2 * i + 1]));
                    if (valid) {
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            st_global_v4(dst + cc + v * 8, pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (kMode == 2) {
                // tile completion: the n-block that finishes a remote tile runs
                // the combine-direction signalling for it.
                named_bar_sync(1, 128);
                if (threadIdx.x == 128) {
                    if (nb == 0) atomicAdd(&c.stats[kStatRecvTiles], 1ull);
                    if (rt.cgroup >= 0) {
                        const uint32_t done = atom_add_acq_rel_gpu(c.tile_ctr + ti, 1u);
                        if (done + 1 == uint32_t(g.n_nb)) {
                            atomicAdd(&c.stats[kStatCombinePuts], 1ull);
                            atomicAdd(&c.stats[kStatCombineBytes], (unsigned long long)rt.rows * c.H * 2);
                            const Group grp = c.cgroups[rt.cgroup];
                            const bool suppress = c.signaling == PERSEUS_SIGNAL_NONE;
                            bool run = grp.count == 1;
                            if (!run) run = atom_add_acq_rel_gpu(c.cgroup_ctr + rt.cgroup, 1u) + 1 == uint32_t(grp.count);
                            if (run) {
                                if (!suppress) {
                                    fence_acq_rel_sys();
                                    atomicAdd(&c.stats[kStatCombineFences], 1ull);
                                }
                                for (int m = 0; m < grp.count; ++m) {
                                    const RecvTile mt = c.recv[grp.first + m];
                                    st_relaxed_sys(c.cflag[mt.src] + size_t(c.par) * c.T_max + mt.tile_id, c.epoch);
                                }
                                atomicAdd(&c.stats[kStatCombineSignals], (unsigned long long)grp.count);
                            }
                        }
                    }
                }
            }
            if (++acc == 2) { acc = 0; aphase ^= 1; }
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
    cudaError_t e = cudaFuncSetAttribute(k_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_gemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGemmSmem));
}

void launch_gemm(int mode, const CUtensorMap& ta, const CUtensorMap& tb, const DevCtx& c,
                 int n_nb, int num_kb, int64_t a_row_base, int grid, cudaStream_t st) {
    GemmArgs g{n_nb, num_kb, a_row_base};
    if (mode == 1)
        k_gemm<1><<<grid, 256, kGemmSmem, st>>>(ta, tb, c, g);
    else
        k_gemm<2><<<grid, 256, kGemmSmem, st>>>(ta, tb, c, g);
}

}  // namespace perseus
