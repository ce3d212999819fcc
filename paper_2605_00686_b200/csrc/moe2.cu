// moe2.cu — the fused forward on CTA PAIRS (tcgen05 cta_group::2).
//
// Same structure as k_moe (gemm.cu): copy warps stream dispatch units, a
// scheduler + TMA producer, one MMA thread, four epilogue warps — but each
// work item is a PAIR of M-tiles of the same expert (consecutive chunks of a
// (src, expert) segment) computed as ONE 256 x 256 UMMA tile by two CTAs of a
// cluster:
//   * each CTA loads its own 128 A rows and HALF of the B tile (GEMM1: CTA0
//     the gate rows, CTA1 the up rows; GEMM2: the two 128-row halves of W2's
//     256-row n-block), so every weight byte crosses L2->SM once per pair
//     instead of once per M-tile: 32 KB/stage/CTA instead of 48 KB.  At EP=1
//     the L2->SM bandwidth (not HBM, not the tensor pipe) caps the 1-CTA
//     kernel near 45% tensor utilisation; this removes a third of that traffic;
//   * the leader CTA (cluster rank 0) grabs work items, mirrors them into its
//     peer's ring through DSMEM, and issues tcgen05.mma.cta_group::2; the
//     peer's TMA bytes complete on the leader's full barrier; MMA completion
//     is committed to both CTAs' barriers (multicast); both CTAs' epilogues
//     release the leader's TMEM-empty barrier.
// An odd last chunk is paired with nothing: the peer recomputes its partner's
// rows and discards them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstring>

#include <algorithm>

#include "layer_dev.h"
#include "perseus.h"
#include "ptx.cuh"
#include "signal.cuh"

namespace perseus {
namespace {

using namespace ptx;

constexpr int kStages = 6;
constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr int kA = kBM * kBK * 2;         // 16 KB: this CTA's A rows
constexpr int kBh = 128 * kBK * 2;        // 16 KB: this CTA's half of B
constexpr int kStage = kA + kBh;          // 32 KB
constexpr int kTmemCols = 512;
constexpr int kStgRow = 128 + 16;              // partial-tile fallback: padded 128-byte rows
constexpr int kStgWarp = 2 * 32 * 128;          // per epilogue warp: 2 x (32 rows x 64 cols bf16), SW128
constexpr int kStgBytes = 4 * kStgWarp;         // (>= 128 * kStgRow)
static_assert(kStgBytes >= 128 * kStgRow, "staging");
constexpr int kRing = 8;
constexpr int kUnitRows = 2;  // fine units: few tiles in flight, so tiles land one after another at link rate
constexpr int kUnitsPerTile = kTileRows / kUnitRows;
constexpr size_t kSmem = 1024 + size_t(kStages) * kStage + kStgBytes + 512;

struct Args {
    int32_t n1, n2, kb1, kb2, lag;
    int32_t lag_end;  // lag over the last pairs (>= lag; see launch_moe2)
    int32_t self_window;  // self tiles copied ahead of the tiles the scheduler handed out
    int32_t discard;      // bit 0: heap rows after GEMM1, bit 1: h rows after GEMM2 (discard.global.L2)
    int32_t remote_warps; // copy warps (of 6) that take remote dispatch units
    int32_t ahead;        // producer: k-blocks before an item's end to take the next item and poll its flag
    const CUtensorMap* smaps;  // store maps, box 64 x 32, SW128: [0] hbuf, [1 + p] ybuf of PE p
    int64_t a1_row_base;
};
struct Item {
    int32_t kind, t, nb;
};

__device__ __forceinline__ Item item_of(int w, int T, const Args& f) {
    const int L = min(f.lag, T), L2 = max(L, min(f.lag_end, T)), n1 = f.n1, n2 = f.n2;
    // A: GEMM1 of pairs [0, L)
    if (w < L * n1) return {1, w / n1, w % n1};
    w -= L * n1;
    // B: steady state, GEMM1 of pair L + st with GEMM2 of pair st, st in [0, T - L2)
    const int steady = (T - L2) * (n1 + n2);
    if (w < steady) {
        const int st = w / (n1 + n2), r = w % (n1 + n2);
        return r < n1 ? Item{1, L + st, r} : Item{2, st, r - n1};
    }
    w -= steady;
    // C: GEMM1 of pairs [T - L2 + L, T): the lag grows to L2 for the end
    const int c1 = (L2 - L) * n1;
    if (w < c1) return {1, T - L2 + L + w / n1, w % n1};
    w -= c1;
    // D: GEMM2 of pairs [T - L2, T)
    if (w < L2 * n2) return {2, T - L2 + w / n2, w % n2};
    return {0, 0, 0};
}

__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

__device__ __forceinline__ void copy_unit(const DevCtx& c, const SendTile& st, int r0, int nrows, int lane) {
    // both rows' loads in flight before any store: one memory latency per unit
    const int32_t abs0 = c.offsets[st.expert] + st.row0 + r0;
    bf16* dbase = c.heap[st.dst] + (size_t(c.par) * c.R_max + st.heap_row + r0) * c.H;
    const int nvec = c.H / 8;
    const int32_t tok0 = c.rows[abs0];
    const int32_t tok1 = nrows > 1 ? c.rows[abs0 + 1] : tok0;
    const uint4* s0 = reinterpret_cast<const uint4*>(c.x + size_t(tok0) * c.H);
    const uint4* s1 = reinterpret_cast<const uint4*>(c.x + size_t(tok1) * c.H);
    uint4* d0 = reinterpret_cast<uint4*>(dbase);
    uint4* d1 = reinterpret_cast<uint4*>(dbase + c.H);
    int v = lane;
    for (; v + 224 < nvec; v += 256) {
        uint4 a[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = __ldg(s0 + v + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) b[u] = __ldg(s1 + v + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) d0[v + 32 * u] = a[u];
        if (nrows > 1) {
#pragma unroll
            for (int u = 0; u < 8; ++u) d1[v + 32 * u] = b[u];
        }
    }
    for (; v < nvec; v += 32) {
        const uint4 a = __ldg(s0 + v), b = __ldg(s1 + v);
        d0[v] = a;
        if (nrows > 1) d1[v] = b;
    }
}

// One 32-row x 64-column bf16 chunk of an epilogue warp through its
// double-buffered, 128B-swizzled staging slot into a TMA tensor store (lane 0
// issues; one bulk group per chunk).  w[0..31] = 64 bf16 packed in pairs.
__device__ __forceinline__ void store_chunk(uint8_t* stg_warp, int& buf, const uint32_t* w, int lane,
                                            const CUtensorMap* map, int32_t col, int32_t row) {
    uint8_t* b = stg_warp + buf * (32 * 128);
    if (lane == 0) bulk_wait_read<1>();  // the store that last used this buffer has read it
    __syncwarp();
    const uint32_t base = smem_u32(b) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        st_shared_v4(base + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
        tma_store_2d(map, b, col, row);
        bulk_commit();
    }
    buf ^= 1;
}

// Rows [row0, row0 + rows) of a bf16 [*][cols] buffer are dead: drop their L2
// lines without write-back (one warp).
__device__ __forceinline__ void discard_rows(const bf16* base, int64_t row0, int rows, int cols, int lane) {
    const char* p = reinterpret_cast<const char*>(base + size_t(row0) * cols);
    const int lines = rows * cols * 2 / 128;
    for (int i = lane; i < lines; i += 32) discard_l2(p + size_t(i) * 128);
}

// One token's combine by one warp (dataflow combine): routing weights (when the
// router ran on a side stream; lane j holds w[j]), then out[t] = sum_j w[j] *
// y[pos(t, j)] in j order with fmaf in fp32 -> bf16 — k_combine's arithmetic —
// one 16-byte chunk per lane per step with the token's k rows in flight.  KM >= k.
template <int KM>
__device__ __forceinline__ void combine_token_warp(const DevCtx& c, int t, int lane) {
    const int k = c.k;
    float wl;
    if (c.weights_late) {
        wl = route_weight_lane(c, t, lane);
        if (lane < k) c.weights[size_t(t) * k + lane] = wl;
    } else {
        wl = lane < k ? c.weights[size_t(t) * k + lane] : 0.f;
    }
    const int32_t pl = lane < k ? c.pos[size_t(t) * k + lane] : 0;
    const bf16* y = c.ybuf[c.rank] + size_t(c.par) * c.Y_rows * c.H;
    const int nvec = c.H / 8;
    for (int v0 = lane; v0 < nvec; v0 += 32) {
        uint4 a[KM];
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const int32_t pj = __shfl_sync(0xffffffffu, pl, j);
            if (j < k) a[j] = __ldcs(reinterpret_cast<const uint4*>(y + size_t(pj) * c.H) + v0);
        }
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const float wj = __shfl_sync(0xffffffffu, wl, j);
            if (j < k) {
                const bf16* x = reinterpret_cast<const bf16*>(&a[j]);
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[q] = __fmaf_rn(wj, __bfloat162float(x[q]), acc[q]);
            }
        }
        __stcs(reinterpret_cast<uint4*>(c.out + size_t(t) * c.H) + v0,
               make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]), pack_bf16(acc[4], acc[5]),
                          pack_bf16(acc[6], acc[7])));
    }
}

// combine-direction completion of one n-block of a remote M-tile (4 epilogue warps)
__device__ __forceinline__ void finish_tile(const DevCtx& c, int n_nb, int ti, int nb, bool discard_h) {
    named_bar_sync(1, 128);
    if ((threadIdx.x >> 5) != 4) return;
    const int lane = threadIdx.x & 31;
    const RecvTile rt = c.recv[ti];
    if (lane == 0 && nb == 0) atomicAdd(&c.stats[kStatRecvTiles], 1ull);
    if (rt.cgroup < 0 && !discard_h && !c.df_combine) return;
    uint32_t done = 0;
    if (lane == 0) done = atom_add_acq_rel_gpu(c.tile_ctr + ti, 1u) + 1 == uint32_t(n_nb);
    if (!__shfl_sync(0xffffffffu, done, 0)) return;
    // every GEMM2 n-block of this tile has run (its TMA loads of h are complete;
    // its y rows are written: each n-block's stores completed + proxy fence before
    // its release on tile_ctr, which the acquire above observed)
    if (discard_h) discard_rows(c.hbuf, rt.heap_row, rt.rows, c.I, lane);
    if (c.df_combine) {
        // dataflow combine: one more expert row of each of the tile's tokens; a token
        // whose k rows all exist goes on the ready queue (release -> the combiner's acquire)
        for (int r = lane; r < rt.rows; r += 32) {
            const int32_t t = c.rows[rt.ybuf_row + r];
            if (int(atom_add_acq_rel_gpu(reinterpret_cast<uint32_t*>(c.tok_ready) + t, 1u)) + 1 == c.k) {
                const uint32_t slot = atomicAdd(&c.sched[4], 1u);
                st_release_gpu_u64(c.ready_q + slot, (static_cast<unsigned long long>(c.epoch) << 32) | uint32_t(t));
            }
        }
    }
    if (rt.cgroup < 0) return;
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
    if (lane == 0) atomicMax(c.fwd_t + kFwdCombLast, fwd_now());
}

__device__ __forceinline__ uint32_t pk(const uint32_t* v, int i) {
    return pack_bf16(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
}

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_moe2(const __grid_constant__ CUtensorMap tm_a1, const __grid_constant__ CUtensorMap tm_b1,
           const __grid_constant__ CUtensorMap tm_a2, const __grid_constant__ CUtensorMap tm_b2, DevCtx c,
           Args f) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_out = smem + kStages * kStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + kStgBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* rfull = tempty + 2;
    uint64_t* rempty = rfull + kRing;
    int32_t* ring = reinterpret_cast<int32_t*>(rempty + kRing);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ring + kRing);

    const int warp = warp_id(), lane = lane_id();
    const uint32_t crank = cluster_ctarank();
    const bool lead = crank == 0;

    if (warp == 0 && lane == 0) {
        tl_mark(c, kTlFusedEnter);
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
            mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the live one)
        }
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&rfull[s], 1);
            mbar_init(&rempty[s], 10);  // leader: MMA + 4 epi; peer: producer + 4 epi
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        tmem_alloc_pair(tmem_holder, kTmemCols);
        tmem_relinquish_pair();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // everything above overlapped the previous kernel's tail (PDL); from here
    // on the plan, heap and flags of this forward are read
    pdl_wait();
    tl_start(c, kTlFused);
    PlanHeader hdr = *c.hdr;  // identical in both CTAs
    if (hdr.error) hdr.n_pairs = hdr.n_send = hdr.n_send_remote = 0;  // no work; both CTAs fall through
    const int T = hdr.n_pairs;
    const int total = T * (f.n1 + f.n2);
    const uint64_t t_cta0 = globaltimer();

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- scheduler (leader) + TMA producer (both) ----------------
            // One item of lookahead: the next item is taken a few k-blocks before
            // the current one ends.
            unsigned long long wait_d = 0, wait_g = 0, wait_r = 0;
            int stage = 0, slot = 0;
            uint32_t phase = 0, rphase = 0;
            const uint32_t* dflags = c.dflag[c.rank] + size_t(c.par) * c.T_max;
            auto grab = [&]() {
                int w;
                if (lead) {
                    w = int(atomicAdd(&c.sched[0], 1u));
                    if (w >= total) w = -1;
                    mbar_wait(&rempty[slot], rphase ^ 1);
                    ring[slot] = w;
                    mbar_arrive(&rfull[slot]);
                    st_cluster_u32(mapa(smem_u32(&ring[slot]), 1), uint32_t(w));
                    mbar_arrive_cluster(mapa(smem_u32(&rfull[slot]), 1));
                } else {
                    mbar_wait(&rfull[slot], rphase);
                    w = ring[slot];
                    mbar_arrive_cluster(mapa(smem_u32(&rempty[slot]), 0));
                }
                if (++slot == kRing) { slot = 0; rphase ^= 1; }
                return w;
            };
            struct Op {
                const CUtensorMap* ta;
                const CUtensorMap* tb;
                int32_t a_row, b_row, nkb, kind, mine, dup, nb;
            };
            auto op_of = [&](int w) {
                const Item it = item_of(w, T, f);
                const int t0 = c.pairs[2 * it.t], t1 = c.pairs[2 * it.t + 1];
                Op o;
                o.mine = (crank == 0 || t1 < 0) ? t0 : t1;
                o.dup = crank != 0 && t1 < 0;  // odd pair: the peer CTA recomputes t0's rows
                o.nb = it.nb;
                const RecvTile rt = c.recv[o.mine];
                o.kind = it.kind;
                if (it.kind == 1) {
                    o.a_row = int32_t(f.a1_row_base + rt.heap_row);
                    o.b_row = rt.e_local * 2 * c.I + it.nb * 128 + (crank ? c.I : 0);  // gate | up
                    o.nkb = f.kb1;
                    o.ta = &tm_a1;
                    o.tb = &tm_b1;
                } else {
                    o.a_row = int32_t(rt.heap_row);
                    o.b_row = rt.e_local * c.H + it.nb * 256 + int(crank) * 128;
                    o.nkb = f.kb2;
                    o.ta = &tm_a2;
                    o.tb = &tm_b2;
                }
                return o;
            };
            // the dependency flag of an item (remote dispatch flag: sys scope; this
            // GPU's self-ready / GEMM1 counts: gpu scope) and the value it must reach
            auto dep_of = [&](const Op& o, uint32_t& want, bool& sys) -> const uint32_t* {
                sys = false;
                if (o.kind == 1) {
                    const int tile_id = c.recv[o.mine].tile_id;
                    want = c.epoch;
                    if (tile_id >= 0) {
                        sys = true;
                        return c.local_dispatch ? nullptr : dflags + tile_id;
                    }
                    return c.self_ready + o.mine;
                }
                want = uint32_t(f.n1);
                return c.g1_done + o.mine;
            };
            int w = grab();
            Op cur{};
            if (w >= 0) cur = op_of(w);
            bool cur_ready = false;  // the current item's dependency was already seen satisfied
            while (w >= 0) {
                // dependencies of the current item
                const uint64_t tw0 = globaltimer();
                if (cur_ready) {
                    // observed by the early poll during the previous item: no round trip here
                } else if (cur.kind == 1) {
                    const int tile_id = c.recv[cur.mine].tile_id;
                    const bool ok = tile_id >= 0 ? (c.local_dispatch || wait_flag_geq(dflags + tile_id, c.epoch, kWaitTimeoutNs))
                                                 : wait_flag_geq(c.self_ready + cur.mine, c.epoch, kWaitTimeoutNs);
                    if (!ok) atomicAdd(&c.stats[kStatTimeouts], 1ull);
                    const uint64_t dw = globaltimer() - tw0;
                    wait_d += dw;
                    if (tile_id >= 0) wait_r += dw;
                    if (c.trace) trace_ev(c, kEvDiagItemWait, tile_id >= 0 ? c.recv[cur.mine].src : c.rank, cur.mine,
                                          cur.nb, uint32_t(dw), uint32_t(w), tw0);
                    if (c.trace && tile_id >= 0 && !cur.dup && cur.nb == 0) {  // first n-block's observation
                        const RecvTile rt = c.recv[cur.mine];
                        trace_seen(c, PERSEUS_EV_DISPATCH_SEEN, rt.src, tile_id,
                                   c.heap[c.rank] + (size_t(c.par) * c.R_max + rt.heap_row) * c.H, rt.rows);
                    }
                } else {
                    if (!wait_flag_geq(c.g1_done + cur.mine, uint32_t(f.n1), kWaitTimeoutNs))
                        atomicAdd(&c.stats[kStatTimeouts], 1ull);
                    wait_g += globaltimer() - tw0;
                }
                fence_proxy_async();
                int wn = -2;  // not taken yet
                Op nxt{};
                // take the next item f.ahead k-blocks before the end and issue its
                // dependency poll then (used only after this item's loads are issued,
                // so the flag's round trip overlaps them); trace mode records the
                // first observation itself, so it always waits at the top
                const int take_at = max(0, cur.nkb - f.ahead);
                const uint32_t* pre_flag = nullptr;
                uint32_t pre_want = 0, pre_val = 0;
                bool pre_none = false;
                for (int kb = 0; kb < cur.nkb; ++kb) {
                    if (kb == take_at) {
                        wn = grab();
                        if (wn >= 0) {
                            nxt = op_of(wn);
                            if (f.ahead > 1 && !c.trace) {
                                bool sys;
                                pre_flag = dep_of(nxt, pre_want, sys);
                                if (!pre_flag) pre_none = true;
                                else pre_val = sys ? ld_acquire_sys(pre_flag) : ld_acquire_gpu(pre_flag);
                            }
                        }
                    }
                    uint8_t* sa = smem + stage * kStage;
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (lead) mbar_arrive_expect_tx(&full[stage], 2 * kStage);
                    const uint32_t fb = mapa(smem_u32(&full[stage]), 0);
                    tma_load_2d_pair(sa, cur.ta, fb, kb * kBK, cur.a_row);
                    tma_load_2d_pair(sa + kA, cur.tb, fb, kb * kBK, cur.b_row);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                if (wn == -2) {
                    wn = grab();
                    if (wn >= 0) nxt = op_of(wn);
                }
                w = wn;
                cur = nxt;
                cur_ready = pre_none || (pre_flag && int32_t(pre_val - pre_want) >= 0);
            }
            atomicAdd(&c.stats[kStatWaitDispatchNs], wait_d);
            atomicAdd(&c.stats[kStatWaitG1Ns], wait_g);
            atomicAdd(&c.stats[kStatWaitRemoteNs], wait_r);
        }
    } else if (warp == 1) {
        if (lane == 0 && lead) {
            // ---------------- MMA issuer (leader CTA) ----------------
            const uint32_t idesc = idesc_bf16_f32(2 * kBM, kBN);
            int stage = 0, slot = 0, acc = 0;
            uint32_t phase = 0, rphase = 0, aphase = 0;
            // issue-side stall accounting (SM cycles): waiting for the next item,
            // for a free accumulator (epilogue back-pressure), for operand stages
            long long cy_ring = 0, cy_acc = 0, cy_data = 0;
            const long long cy0 = clock64();
            while (true) {
                long long t = clock64();
                mbar_wait(&rfull[slot], rphase);
                cy_ring += clock64() - t;
                const int w = ring[slot];
                mbar_arrive(&rempty[slot]);
                if (++slot == kRing) { slot = 0; rphase ^= 1; }
                if (w < 0) break;
                const Item it = item_of(w, T, f);
                const int nkb = it.kind == 1 ? f.kb1 : f.kb2;
                t = clock64();
                mbar_wait(&tempty[acc], aphase ^ 1);
                cy_acc += clock64() - t;
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * kBN);
                for (int kb = 0; kb < nkb; ++kb) {
                    t = clock64();
                    mbar_wait(&full[stage], phase);
                    cy_data += clock64() - t;
                    tc_fence_after();
                    uint8_t* sa = smem + stage * kStage;
                    const uint64_t adesc = smem_desc_sw128(sa);
                    const uint64_t bdesc = smem_desc_sw128(sa + kA);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        umma_bf16_pair(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
                    umma_commit_pair(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                umma_commit_pair(&tfull[acc]);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
            atomicAdd(&c.stats[kStatMmaCycles], (unsigned long long)(clock64() - cy0));
            if (c.tl) {  // when the first / last MMA issuer ran out of work items
                atomicMax(c.tl + 2 * kTlMmaOut, ~fwd_now());
                atomicMax(c.tl + 2 * kTlMmaOut + 1, fwd_now());
            }
            atomicAdd(&c.stats[kStatMmaRingWait], (unsigned long long)cy_ring);
            atomicAdd(&c.stats[kStatMmaAccWait], (unsigned long long)cy_acc);
            atomicAdd(&c.stats[kStatMmaDataWait], (unsigned long long)cy_data);
        }
    } else if (warp < 4 || warp >= 8) {
        // ---------------- copy warps: dispatch puts ----------------
        // Copy warps first copy the self tiles of the head pairs (the GEMMs start
        // on them), then stream the remote tiles (NVLink, rotated destination
        // order), then the rest of the self tiles.
        const int remote_units = hdr.n_send_remote * kUnitsPerTile;
        const int self_units = (hdr.n_send - hdr.n_send_remote) * kUnitsPerTile;
        const int head_units = min(self_units, 2 * hdr.self_head * kUnitsPerTile);
        const uint64_t tc0 = globaltimer();
        // warps 10-11 open the remote stream at once (the first destination's
        // group must land while the head computes)
        // f.remote_warps of the 6 copy warps (warps 11, 10, 9, ... first) take remote units
        const bool remote_ok = (warp < 4 ? warp - 2 : warp - 6) >= 6 - f.remote_warps;
        int state = (head_units > 0 && warp < 10) ? 0 : (remote_ok ? 1 : 2);  // 0: self head, 1: remote, 2: self rest
        bool first_remote = true;
        if (c.signaling == PERSEUS_SIGNAL_FAULT_EARLY) {
            // fault injection: every remote tile's flag is written as its put is
            // issued — here, before any row is copied — with no fence: the
            // "signal before data" bug verify_ordering must catch
            const int cw = warp < 4 ? warp - 2 : warp - 6;  // 0..5
            for (int i = (blockIdx.x * 6 + cw) * 32 + lane; i < hdr.n_send_remote; i += gridDim.x * 6 * 32) {
                const SendTile st = c.send[i];
                st_relaxed_sys(c.dflag[st.dst] + size_t(c.par) * c.T_max + st.tile_id, c.epoch);
                atomicAdd(&c.stats[kStatDispatchSignals], 1ull);
                if (c.trace) trace_ev(c, PERSEUS_EV_DISPATCH_SIGNAL, st.dst, st.tile_id, st.group, 0, 0, fwd_now());
            }
        }
        // (fault) ... and the remote puts are slow to land (a congested link): they
        // start 200 us after their signals — later than the receivers reach their
        // first remote tiles — so receivers that trust the flags read rows not there yet
        const uint64_t t_fault = globaltimer() + 200000;
        // token dedup: the remote queue is this rank's tokens (each sent once per
        // destination), then an expansion queue over the received remote tiles
        const int remote_n = c.dedup ? c.S : remote_units;
        const int expand_units = c.dedup ? hdr.n_recv_remote * kUnitsPerTile : 0;
        bool expanded = false;  // this warp found the expansion queue empty
        while (true) {
            const bool remote_q = state == 1;
            if (state == 3) {
                // token dedup, receiver: expand the sources' token buffers into the
                // receive heap, tile by tile in arrival order, and release each
                // tile to the GEMMs (the flag the producer waits on, set locally)
                int u = 0;
                if (lane == 0) u = int(atomicAdd(&c.sched[6], 1u));
                u = __shfl_sync(0xffffffffu, u, 0);
                if (u >= expand_units) {
                    state = expanded ? 4 : 2;  // 4: done (came here from the self rest)
                    expanded = true;
                    if (state == 4) break;
                    continue;
                }
                const int ti = c.rorder[hdr.n_recv - hdr.n_recv_remote + u / kUnitsPerTile];
                const RecvTile rt = c.recv[ti];
                const int r0 = (u % kUnitsPerTile) * kUnitRows;
                if (r0 >= rt.rows) continue;
                const int nrows = min(kUnitRows, rt.rows - r0);
                if (lane == 0 &&
                    !wait_flag_geq(c.ddflag[c.rank] + size_t(c.par) * kMaxPes + rt.src, c.epoch, kWaitTimeoutNs))
                    atomicAdd(&c.stats[kStatTimeouts], 1ull);
                __syncwarp();
                const bf16* buf = c.dd[c.rank] + (size_t(c.par) * c.P + rt.src) * size_t(c.S) * c.H;
                bf16* heap = c.heap[c.rank] + (size_t(c.par) * c.R_max + rt.heap_row) * c.H;
                for (int r = 0; r < nrows; ++r) {
                    const int32_t row = ld_relaxed_sys(reinterpret_cast<const uint32_t*>(
                        c.didx[c.rank] + size_t(c.par) * c.R_max + rt.heap_row + r0 + r));
                    const uint4* src = reinterpret_cast<const uint4*>(buf + size_t(row) * c.H);
                    uint4* dst = reinterpret_cast<uint4*>(heap + size_t(r0 + r) * c.H);
                    for (int v = lane; v < c.H / 8; v += 32) dst[v] = __ldcg(src + v);
                }
                __syncwarp();
                if (lane == 0 && atom_add_acq_rel_gpu(c.ex_done + ti, uint32_t(nrows)) + nrows == uint32_t(rt.rows))
                    st_release_gpu(c.dflag[c.rank] + size_t(c.par) * c.T_max + rt.tile_id, c.epoch);
                continue;
            }
            if (remote_q && c.dedup) {
                // token dedup, sender: one token per claim; its row crosses to each
                // remote destination of its experts once, with the token-buffer row of
                // each of its (expert, row) slots in the destination's heap layout
                int t = 0;
                if (lane == 0) t = int(atomicAdd(&c.sched[1], 1u));
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= remote_n) {
                    state = expand_units > 0 ? 3 : 2;
                    continue;
                }
                if (first_remote) {
                    if (lane == 0) atomicMin(c.fwd_t + kFwdDispFirst, fwd_now());
                    first_remote = false;
                }
                const int e_l = lane < c.k ? c.ids[size_t(t) * c.k + lane] : 0;
                const int p_l = lane < c.k ? c.pos[size_t(t) * c.k + lane] : 0;
                const int d_l = lane < c.k ? e_l % c.P : c.rank;
                // index entries: lane j < k writes its slot's token-buffer row at the destination
                if (d_l != c.rank) {
                    const int32_t rel = p_l - c.offsets[e_l];
                    const SendTile st = c.send[c.send_first[e_l] + rel / kTileRows];
                    c.didx[d_l][size_t(c.par) * c.R_max + st.heap_row + rel % kTileRows] = c.uidx[p_l];
                }
                const uint4* srow = reinterpret_cast<const uint4*>(c.x + size_t(t) * c.H);
                for (int d = 0; d < c.P; ++d) {
                    const unsigned on = __ballot_sync(0xffffffffu, lane < c.k && d_l == d && d != c.rank);
                    if (!on) continue;
                    const int32_t urow = __shfl_sync(0xffffffffu, c.uidx[p_l], __ffs(on) - 1);
                    uint4* drow = reinterpret_cast<uint4*>(c.dd[d] + ((size_t(c.par) * c.P + c.rank) * size_t(c.S) + urow) * c.H);
                    for (int v = lane; v < c.H / 8; v += 32) drow[v] = __ldg(srow + v);
                    __syncwarp();
                    if (lane == 0) {
                        atomicAdd(&c.stats[kStatDispatchPuts], 1ull);
                        atomicAdd(&c.stats[kStatDispatchBytes], (unsigned long long)c.H * 2 + 4ull * __popc(on));
                        const uint32_t n = 1u + __popc(on);
                        if (atom_add_acq_rel_gpu(c.dsent + d, n) + n == uint32_t(c.dtot[d] + c.drows[d])) {
                            // this destination's token buffer and index are complete:
                            // one fence, one flag (Perseus per-destination signalling)
                            fence_acq_rel_sys();
                            st_relaxed_sys(c.ddflag[d] + size_t(c.par) * kMaxPes + c.rank, c.epoch);
                            atomicAdd(&c.stats[kStatDispatchFences], 1ull);
                            atomicAdd(&c.stats[kStatDispatchSignals], 1ull);
                            atomicMax(c.fwd_t + kFwdDispLast, fwd_now());
                        }
                    }
                }
                continue;
            }
            int u = 0;
            if (lane == 0) u = int(atomicAdd(&c.sched[remote_q ? 1 : 2], 1u));
            u = __shfl_sync(0xffffffffu, u, 0);
            if (u >= (remote_q ? remote_units : self_units)) {
                if (state == 2 && expand_units > 0 && !expanded) {
                    // token dedup: warps done with the self rows help expand
                    expanded = true;
                    state = 3;
                    continue;
                }
                if (state == 2) break;
                state = (state == 0 && remote_ok) ? 1 : 2;
                continue;
            }
            if (state == 0 && u >= head_units) state = remote_ok ? 1 : 2;  // head claimed: this unit, then the remote queue
            if (!remote_q) {
                // Pace the self copies: stay at most f.self_window tiles ahead of the
                // tiles the scheduler has handed out, so heap rows are still in L2
                // when GEMM1 reads them (self tiles are consumed first, in this
                // order).  The items of every grabbed tile are always allowed.
                const int need = u / kUnitsPerTile;
                if (lane == 0) {
                    while (true) {
                        const int w = int(*reinterpret_cast<volatile uint32_t*>(c.sched));
                        const int L = min(f.lag, T);
                        const int started = w < L * f.n1 ? w / f.n1 : L + (w - L * f.n1) / (f.n1 + f.n2);
                        if (need < 2 * started + f.self_window) break;
                        __nanosleep(256);
                    }
                }
                __syncwarp();
            }
            const int sp = remote_q ? c.sorder[u / kUnitsPerTile] : hdr.n_send_remote + u / kUnitsPerTile;
            const SendTile st = c.send[sp];
            const int r0 = (u % kUnitsPerTile) * kUnitRows;
            if (r0 >= st.rows) continue;
            const int nrows = min(kUnitRows, st.rows - r0);
            if (remote_q && first_remote) {
                if (c.signaling == PERSEUS_SIGNAL_FAULT_EARLY)
                    while (globaltimer() < t_fault) __nanosleep(1000);
                if (lane == 0) atomicMin(c.fwd_t + kFwdDispFirst, fwd_now());
                first_remote = false;
            }
            const bool fault_early = c.signaling == PERSEUS_SIGNAL_FAULT_EARLY;  // flags already written
            copy_unit(c, st, r0, nrows, lane);
            __syncwarp();
            uint32_t done = 0;
            if (lane == 0) done = atom_add_acq_rel_gpu(c.send_done + sp, uint32_t(nrows)) + nrows == uint32_t(st.rows);
            if (!__shfl_sync(0xffffffffu, done, 0)) continue;
            if (st.dst == c.rank) {
                if (lane == 0) {
                    st_release_gpu(c.self_ready + st.recv_pos, c.epoch);
                    if (c.trace) trace_ev(c, kEvDiagSelfReady, c.rank, st.recv_pos, -1, 0, 0, fwd_now());
                }
                continue;
            }
            if (lane == 0) {
                atomicAdd(&c.stats[kStatDispatchPuts], 1ull);
                atomicAdd(&c.stats[kStatDispatchBytes], (unsigned long long)st.rows * c.H * 2);
                if (c.trace) trace_ev(c, PERSEUS_EV_DISPATCH_PUT, st.dst, st.tile_id, st.group, uint32_t(st.rows) * c.H * 2, 0, fwd_now());
            }
            if (!fault_early) {
                const Group g = c.groups[st.group];
                auto flag_of = [&](int m) {
                    const SendTile& t = c.send[m];
                    return c.dflag[t.dst] + size_t(c.par) * c.T_max + t.tile_id;
                };
                publish_member_warp(c, g, c.group_ctr + st.group, flag_of, c.signaling >= PERSEUS_SIGNAL_NONE,
                                    kStatDispatchFences, kStatDispatchSignals);
            }
            if (lane == 0) atomicMax(c.fwd_t + kFwdDispLast, fwd_now());
        }
        if (lane == 0) atomicAdd(&c.stats[kStatCopyNs], (unsigned long long)(globaltimer() - tc0));
        if (c.tl && lane == 0) {
            atomicMax(c.tl + 2 * kTlCopyEnd, ~fwd_now());
            atomicMax(c.tl + 2 * kTlCopyEnd + 1, fwd_now());
        }
        if (c.df_combine) {
            // dataflow combine: take tokens in the order their k expert rows were
            // completed; out[t] = sum_j w[t][j] * y[pos(t, j)] in fixed j order (fmaf),
            // exactly k_combine's arithmetic
            while (true) {
                uint32_t i = 0;
                if (lane == 0) i = atomicAdd(&c.sched[5], 1u);
                i = __shfl_sync(0xffffffffu, i, 0);
                if (i >= uint32_t(c.S)) break;
                unsigned long long v = 0;
                if (lane == 0) {
                    const uint64_t t0 = globaltimer();
                    while (uint32_t((v = ld_acquire_gpu_u64(c.ready_q + i)) >> 32) != c.epoch) {
                        if (globaltimer() - t0 > kWaitTimeoutNs) {
                            atomicAdd(&c.stats[kStatTimeouts], 1ull);
                            break;
                        }
                        __nanosleep(128);
                    }
                }
                v = __shfl_sync(0xffffffffu, v, 0);
                if (uint32_t(v >> 32) != c.epoch) continue;
                if (c.k <= 8) combine_token_warp<8>(c, int(uint32_t(v)), lane);
                else combine_token_warp<16>(c, int(uint32_t(v)), lane);
            }
        } else if (c.weights_late) {
            // the routing weights (router GEMM ran beside route/permute/plan), after the puts
            const int cw = warp < 4 ? warp - 2 : warp - 6;  // 0..5
            for (int t = blockIdx.x * 6 + cw; t < c.S; t += gridDim.x * 6) route_weights_warp(c, t, lane);
        }
    } else {
        // ---------------- epilogue (4 warps, this CTA's 128 accumulator rows) ----------------
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int acc = 0, slot = 0;
        uint32_t aphase = 0, rphase = 0;
        int pend_ti = -1, pend_nb = 0;
        bool first_put = true;
        uint8_t* stg_warp = stage_out + q * kStgWarp;
        int sbuf = 0;
        const uint32_t tempty_lead = mapa(smem_u32(&tempty[0]), 0);
        const uint32_t rempty_lead = mapa(smem_u32(&rempty[0]), 0);
        while (true) {
            mbar_wait(&rfull[slot], rphase);
            const int w = ring[slot];
            __syncwarp();
            if (lane == 0) {
                if (lead) mbar_arrive(&rempty[slot]);
                else mbar_arrive_cluster(rempty_lead + 8u * slot);
            }
            if (++slot == kRing) { slot = 0; rphase ^= 1; }
            if (w < 0) break;
            const Item it = item_of(w, T, f);
            const int t0 = c.pairs[2 * it.t], t1 = c.pairs[2 * it.t + 1];
            const int mine = crank == 0 ? t0 : t1;  // -1: padding half of an odd pair
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kBN);
            RecvTile rt;
            if (mine >= 0) rt = c.recv[mine];
            const bool valid = mine >= 0 && row < rt.rows;
            const bool full_tile = mine >= 0 && rt.rows == kTileRows;
            if (it.kind == 1) {
                if (full_tile) {
                    // h = silu(gate) * up -> hbuf via TMA tensor stores
#pragma unroll 1
                    for (int cc = 0; cc < 128; cc += 64) {
                        uint32_t o[32];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint32_t gv[32], uv[32];
                            tmem_ld_32x32b_x32(taddr + cc + 32 * h, gv);
                            tmem_ld_32x32b_x32(taddr + 128 + cc + 32 * h, uv);
                            tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                o[16 * h + i] = pack_bf16(silu_mul(__uint_as_float(gv[2 * i]), __uint_as_float(uv[2 * i])),
                                                          silu_mul(__uint_as_float(gv[2 * i + 1]), __uint_as_float(uv[2 * i + 1])));
                        }
                        store_chunk(stg_warp, sbuf, o, lane, f.smaps, it.nb * 128 + cc, int32_t(rt.heap_row) + q * 32);
                    }
                } else if (mine >= 0) {
                    bf16* dst = c.hbuf + size_t(rt.heap_row + row) * c.I + it.nb * 128;
#pragma unroll 1
                    for (int cc = 0; cc < 128; cc += 32) {
                        uint32_t gv[32], uv[32];
                        tmem_ld_32x32b_x32(taddr + cc, gv);
                        tmem_ld_32x32b_x32(taddr + 128 + cc, uv);
                        tmem_ld_wait();
                        uint32_t o[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            o[i] = pack_bf16(silu_mul(__uint_as_float(gv[2 * i]), __uint_as_float(uv[2 * i])),
                                             silu_mul(__uint_as_float(gv[2 * i + 1]), __uint_as_float(uv[2 * i + 1])));
                        if (valid) {
#pragma unroll
                            for (int v = 0; v < 4; ++v) st_global_v4(dst + cc + v * 8, o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (lead) mbar_arrive(&tempty[acc]);
                    else mbar_arrive_cluster(tempty_lead + 8u * acc);
                }
                if (mine >= 0) {
                    if (full_tile && lane == 0) {
                        bulk_wait0();  // h rows written before GEMM2's TMA loads may read them
                        fence_proxy_async();
                    }
                    named_bar_sync(2, 128);
                    if (warp == 4) {
                        uint32_t last = 0;
                        if (lane == 0) last = atom_add_acq_rel_gpu(c.g1_done + mine, 1u) + 1 == uint32_t(f.n1);
                        // every GEMM1 n-block of this tile has run (both CTAs' TMA loads
                        // of its heap rows are complete): the rows are dead
                        if ((f.discard & 1) && __shfl_sync(0xffffffffu, last, 0))
                            discard_rows(c.heap[c.rank] + size_t(c.par) * c.R_max * c.H, rt.heap_row, rt.rows, c.H, lane);
                    }
                }
            } else {
                if (full_tile) {
                    // y tile -> the token owner's combine buffer (local or NVLink peer) via TMA tensor stores
                    if (rt.src != c.rank && first_put) {
                        if (lane == 0) atomicMin(c.fwd_t + kFwdCombFirst, fwd_now());
                        first_put = false;
                    }
                    const CUtensorMap* ym = f.smaps + 1 + rt.src;
                    const int32_t yrow = int32_t(size_t(c.par) * c.Y_rows + rt.ybuf_row) + q * 32;
#pragma unroll 1
                    for (int cc = 0; cc < 256; cc += 64) {
                        uint32_t v0[32], v1[32], o[32];
                        tmem_ld_32x32b_x32(taddr + cc, v0);
                        tmem_ld_32x32b_x32(taddr + cc + 32, v1);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            o[i] = pk(v0, 2 * i);
                            o[16 + i] = pk(v1, 2 * i);
                        }
                        store_chunk(stg_warp, sbuf, o, lane, ym, it.nb * 256 + cc, yrow);
                    }
                    if (lane != 0) {
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) bulk_commit();  // keep per-lane group counts uniform
                    }
                } else if (mine >= 0) {
                    // partial tile: direct 16-byte stores of the valid rows (local or peer)
                    bf16* dst = c.ybuf[rt.src] + (size_t(c.par) * c.Y_rows + size_t(rt.ybuf_row + row)) * c.H + it.nb * 256;
#pragma unroll 1
                    for (int cc = 0; cc < 256; cc += 32) {
                        uint32_t v32[32];
                        tmem_ld_32x32b_x32(taddr + cc, v32);
                        tmem_ld_wait();
                        if (valid) {
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                st_global_v4(dst + cc + v * 8, pk(v32, 8 * v), pk(v32, 8 * v + 2), pk(v32, 8 * v + 4), pk(v32, 8 * v + 6));
                        }
                    }
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) bulk_commit();
                } else {
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) bulk_commit();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (lead) mbar_arrive(&tempty[acc]);
                    else mbar_arrive_cluster(tempty_lead + 8u * acc);
                }
                if (pend_ti >= 0) {
                    bulk_wait<4>();
                    fence_proxy_async();
                    finish_tile(c, f.n2, pend_ti, pend_nb, (f.discard & 2) != 0);
                }
                pend_ti = mine;
                pend_nb = it.nb;
            }
            if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
        if (pend_ti >= 0) {
            bulk_wait0();
            fence_proxy_async();
            finish_tile(c, f.n2, pend_ti, pend_nb, (f.discard & 2) != 0);
        }
    }
    pdl_launch_dependents();  // the combine's launch overlaps this CTA's teardown
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (threadIdx.x == 0) atomicAdd(&c.stats[kStatCtaNs], (unsigned long long)(globaltimer() - t_cta0));
    tl_end(c, kTlFused, threadIdx.x == 0);
    if (warp == 2) tmem_dealloc_pair(tmem_base, kTmemCols);
}

cudaError_t configure_moe2() {
    return cudaFuncSetAttribute(k_moe2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem));
}

cudaError_t launch_moe2(const CUtensorMap& a1, const CUtensorMap& b1, const CUtensorMap& a2, const CUtensorMap& b2,
                        const CUtensorMap* smaps, const DevCtx& c, int64_t a1_row_base, int grid, cudaStream_t st) {
    Args f;
    f.n1 = c.I / 128;
    f.n2 = c.H / 256;
    f.kb1 = c.H / kBK;
    f.kb2 = c.I / kBK;
    // GEMM2 of pair t is issued with GEMM1 of pair t + lag: one wave of the
    // grid/2 CTA pairs of GEMM1 items in between, so its inputs are normally done
    {
        static const int lag_pairs = [] { const char* e = getenv("PERSEUS_LAG_PAIRS"); return e ? atoi(e) : 0; }();
        const int pairs_live = grid / 2;
        int lag = std::max(1, (pairs_live + f.n1 - 1) / f.n1);
        // GEMM2 items longer than GEMM1 items (Llama4: K = 8192 vs 5120): keep two
        // waves of GEMM2 items for the end, or the last wave runs half empty
        if (f.kb2 > f.kb1) lag = std::max(lag, (2 * pairs_live + f.n2 - 1) / f.n2);
        f.lag = lag_pairs > 0 ? lag_pairs : lag;
        // the end of the schedule: after the last GEMM1 item is taken, the GEMM2
        // items still queued must keep every pair busy for that item's duration
        // (pairs_live * kb1 k-blocks) plus one more wave, or the last pairs' GEMM2
        // items start late while the others idle (Qwen3 EP=1: 13 -> 35 pairs cut
        // the MMA tail spread from ~14.5 to ~8.5 us).  Only without remote pairs:
        // with P > 1 it would hold back the GEMM2 (and combine puts) of the last
        // remote pairs, exposing their NVLink time (EP=4: 4% -> 12% exposed)
        static const int lag_end_env = [] { const char* e = getenv("PERSEUS_LAG_END"); return e ? atoi(e) : -1; }();
        const int cover = (pairs_live * f.kb1 + f.n2 * f.kb2 - 1) / (f.n2 * f.kb2);
        const int lag_end = c.P == 1 ? std::max(f.lag, cover + (pairs_live + f.n2 - 1) / f.n2) : f.lag;
        f.lag_end = lag_end_env >= 0 ? std::max(f.lag, lag_end_env) : lag_end;
    }
    {
        static const int sw = [] { const char* e = getenv("PERSEUS_SELF_WINDOW"); return e ? atoi(e) : 160; }();
        static const int dc = [] { const char* e = getenv("PERSEUS_DISCARD"); return e ? atoi(e) : 0; }();
        static const int rw = [] { const char* e = getenv("PERSEUS_REMOTE_WARPS"); return e ? atoi(e) : 6; }();
        f.self_window = sw;
        f.discard = dc;
        f.remote_warps = std::max(1, std::min(6, rw));
        // measured at EP=1 (same box, alternating): 1 -> 6 k-blocks ahead, wait
        // fractions 0.04 / 0.025 -> 0.028 / 0.024, step 424 -> 415 us (power-capped)
        static const int ah = [] { const char* e = getenv("PERSEUS_AHEAD"); return e ? atoi(e) : 6; }();
        f.ahead = std::max(1, ah);
    }
    f.smaps = smaps;
    f.a1_row_base = a1_row_base;
    DevCtx cc = c;
    void* args[] = {const_cast<CUtensorMap*>(&a1), const_cast<CUtensorMap*>(&b1), const_cast<CUtensorMap*>(&a2),
                    const_cast<CUtensorMap*>(&b2), &cc, &f};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid & ~1);
    cfg.blockDim = dim3(384);  // warps 2-3 and 8-11 copy, 4-7 epilogue
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (c.pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // prologue overlaps the plan kernel
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    // Cooperative launch (all CTAs co-resident before any runs) also keeps the
    // grid from launching early under PDL (measured: tools/microbench/launch_gap,
    // +2.5 us per forward), so with PDL it is left off: the grid is one CTA per
    // SM and nothing before it waits for it, so every CTA becomes resident once
    // route/permute/plan exit.  Without PDL (ranks sharing a device) it stays.
    static const int coop_env = [] { const char* e = getenv("PERSEUS_COOP"); return e ? atoi(e) : -1; }();
    const bool coop = coop_env >= 0 ? coop_env != 0 : !c.pdl;
    if (coop) {
        attr[na].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (cross-CTA tile dependencies)
        attr[na++].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k_moe2), args);
    if (e != cudaSuccess && coop) {
        (void)cudaGetLastError();
        cfg.numAttrs = na - 1;  // cooperative + clusters rejected: 1 CTA/SM, grid = #SMs keeps them co-resident
        e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k_moe2), args);
    }
    return e;
}

}  // namespace perseus
