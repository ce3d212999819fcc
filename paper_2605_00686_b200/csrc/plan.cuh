// plan.cuh — the per-forward device plan, 4 warps, warp-level scans (run by
// k_plan4, kernels.cu).
//
// Computes, from the [P][E] per-(src, expert) count table every rank
// published, exactly the reference's dispatch layout (workload.cpp:132-213):
//   tile ids     — global counter in (src, expert, chunk) order over remote
//                  pairs (tile_bytes = 128*H*2, workload.cpp:136-149)
//   heap offsets — per-destination cursor in the same order (:146-147)
//   groups       — (dst, expert, tile) order; per destination or fixed size
//                  (assign_groups, protocols.cpp:52-94)
// plus the device-only schedules of the fused kernels (copy order, processing
// order, M-tile pairs).  The plan is latency-bound (a few thousand integers),
// so it runs as 4 independent warps with shuffle scans and three CTA
// barriers, instead of block-wide scans over 1024 threads.
#pragma once
#include <cuda_runtime.h>

#include "layer_dev.h"
#include "perseus.h"
#include "ptx.cuh"

namespace perseus {

using namespace ptx;

namespace {

constexpr int kPlanThreads = 256;  // 8 warps (the permutation kernel's CTA size)

__device__ __forceinline__ int32_t ceil_tiles(int32_t rows) { return (rows + kTileRows - 1) / kTileRows; }

// exclusive scan of a[0..n) in place by ONE warp; returns the total
__device__ __noinline__ int32_t warp_scan(int32_t* a, int n) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    const int per = (n + 31) / 32, b = lane * per, e = min(n, b + per);
    // 16-byte chunks when every lane's run is whole and aligned (n % 128 == 0):
    // the run's loads are independent instead of one dependent chain
    const bool vec = (n & 127) == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0;
    int32_t local = 0;
    if (vec) {
        #pragma unroll 4
        for (int i = b; i < e; i += 4) {
            const int4 q = *reinterpret_cast<const int4*>(a + i);
            local += (q.x + q.y) + (q.z + q.w);
        }
    } else {
        #pragma unroll 1
        for (int i = b; i < e; ++i) local += a[i];
    }
    int32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    int32_t run = incl - local;
    if (vec) {
        #pragma unroll 4
        for (int i = b; i < e; i += 4) {
            int4 q = *reinterpret_cast<int4*>(a + i);
            const int32_t s0 = run, s1 = s0 + q.x, s2 = s1 + q.y, s3 = s2 + q.z;
            run = s3 + q.w;
            q = make_int4(s0, s1, s2, s3);
            *reinterpret_cast<int4*>(a + i) = q;
        }
    } else {
        #pragma unroll 1
        for (int i = b; i < e; ++i) {
            const int32_t v = a[i];
            a[i] = run;
            run += v;
        }
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    return total;
}

}  // namespace

// The plan, run by threads 0..kPlanThreads-1 of one CTA (named barrier 1;
// `sm` holds plan_smem_bytes()).
__device__ __forceinline__ void plan_body(const DevCtx& c, int32_t* sm) {
    const int P = c.P, E = c.E, El = c.E_loc, r = c.rank;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int PE = P * E;
    auto sync128 = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };  // all kPlanThreads
    int32_t* T = sm;            // [P][E] counts
    int32_t* tb = T + PE;       // tile-id base per (s, e), s-major
    int32_t* hr = tb + PE;      // heap-row scan, (d, s, j) order
    int32_t* off = hr + PE;     // sorted offset per (s, e)
    int32_t* sp = off + PE;     // send position per (kd, j)
    int32_t* rp = sp + E;       // recv position per (ks, j)
    int32_t* pp = rp + E;       // pair position per (class, j): class = arrival index of a pair's later tile
    int32_t* selfo = pp + E;    // [El] self-segment row offsets
    // Pair order inside a remote class: experts ascending in even classes and
    // descending in odd ones (c.snake, per-destination signalling only — the
    // whole class lands at once; not with token dedup, whose receiver expands a
    // class's tiles in ascending order).  Consecutive classes then meet on the
    // same experts, whose weights the previous class left in L2 (P >= 2: each
    // expert's weights are streamed once per class).
    const bool snake = c.snake && c.group_size == 0 && !c.dedup;
    auto pslot = [&](int a, int j) { return snake && (a & 1) ? El - 1 - j : j; };
    __shared__ int32_t s_err, s_total_tiles, s_rows_in, s_n_send, s_n_recv, s_n_pairs;
    __shared__ int32_t dst_first[kMaxPes], dst_n[kMaxPes], dst_group[kMaxPes], n_dgroups;
    __shared__ int32_t src_first[kMaxPes], src_n[kMaxPes], src_group[kMaxPes], n_cgroups_pe;
    __shared__ int32_t cls_first[kMaxPes], cls_n[kMaxPes];
    // rotated schedules: sender r streams destination r+1, r+2, ... in turn, so
    // receiver r gets source r-1, r-2, ... one at a time (one group completes
    // after another instead of all at the end)
    __shared__ int32_t send_base[kMaxPes], recv_base[kMaxPes], s_head;

    if (tid == 0) s_err = 0;
    if (c.dedup && tid < kMaxPes) c.dsent[tid] = 0;  // token dedup: rows + index entries sent per destination
    if (tid < P && !wait_flag_geq(c.count_flag[r] + tid, c.epoch, kWaitTimeoutNs)) {
        atomicAdd(&c.stats[kStatTimeouts], 1ull);
        s_err = 1;
    }
    sync128();
    const uint64_t t_ready = tl_now(c);
    const int32_t* table = c.count_table[r] + size_t(c.par) * PE;
    {
        // up to 4 loads in flight per thread (PE <= 4 * kPlanThreads up to P = 8 at E = 128)
        const uint32_t* tb32 = reinterpret_cast<const uint32_t*>(table);
        #pragma unroll 1
        for (int i0 = tid; i0 < PE; i0 += 4 * kPlanThreads) {
            uint32_t v[4];
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kPlanThreads;
                v[u] = i < PE ? ld_relaxed_sys(tb32 + i) : 0u;
            }
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kPlanThreads;
                if (i < PE) T[i] = int32_t(v[u]);
            }
        }
    }
    if (tid == 0) {
        #pragma unroll 1
        for (int q = 0; q < 8; ++q) c.sched[q] = 0;  // work items, copy queues, dataflow-combine queue
        #pragma unroll 1
        for (int q = 0; q < kFwdSlots; ++q) c.fwd_t[q] = (q & 1) || q == kFwdDoneCtas ? 0ull : ~0ull;  // min / max
    }
    sync128();

    // ---- phase B: four independent scans ----
    if (warp == 0) {
        #pragma unroll 1
        for (int s = 0; s < P; ++s)
            #pragma unroll 1
            for (int e = lane; e < E; e += 32) tb[s * E + e] = (s != e % P) ? ceil_tiles(T[s * E + e]) : 0;
        const int32_t tot = warp_scan(tb, PE);
        if (lane == 0) s_total_tiles = tot;
    } else if (warp == 1) {
        // (d, s, j): the rows source s sends to destination d, in the reference's cursor order
        #pragma unroll 1
        for (int d = 0; d < P; ++d)
            #pragma unroll 1
            for (int s = 0; s < P; ++s)
                #pragma unroll 1
                for (int j = lane; j < El; j += 32) hr[(d * P + s) * El + j] = (s != d) ? T[s * E + d + P * j] : 0;
        const int32_t tot = warp_scan(hr, PE);
        if (lane == 0) s_rows_in = (r + 1 < P ? hr[(r + 1) * P * El] : tot) - hr[r * P * El];
    } else if (warp == 2) {
        #pragma unroll 1
        for (int s = 0; s < P; ++s) {
            #pragma unroll 1
            for (int e = lane; e < E; e += 32) off[s * E + e] = T[s * E + e];
            warp_scan(off + s * E, E);
        }
    } else if (warp == 6) {
        #pragma unroll 1
        for (int j = lane; j < El; j += 32) selfo[j] = T[r * E + r + P * j];
        warp_scan(selfo, El);
    } else if (warp == 3) {
        // send key order: remote destinations ascending, then the self segment
        #pragma unroll 1
        for (int d = 0; d < P; ++d) {
            const int kd = d < r ? d : (d > r ? d - 1 : P - 1);
            #pragma unroll 1
            for (int j = lane; j < El; j += 32) sp[kd * El + j] = ceil_tiles(T[r * E + d + P * j]);
        }
        const int32_t n_send = warp_scan(sp, E);
        if (lane == 0) s_n_send = n_send;
    } else if (warp == 4) {
        // receive key order: self first, then remote sources ascending
        #pragma unroll 1
        for (int s = 0; s < P; ++s) {
            const int ks = s == r ? 0 : (s < r ? s + 1 : s);
            #pragma unroll 1
            for (int j = lane; j < El; j += 32) rp[ks * El + j] = ceil_tiles(T[s * E + r + P * j]);
        }
        const int32_t n_recv = warp_scan(rp, E);
        if (lane == 0) s_n_recv = n_recv;
    } else if (warp == 5) {
        // M-tile pairs per local expert over its tiles in ARRIVAL order (self,
        // then sources r-1, r-2, ...): a pair may join tiles of two sources, so
        // one-tile segments (DeepSeek-V3: 128 rows per (source, expert)) still
        // fill both CTAs of a pair.  A pair's class = the arrival index of its
        // later tile; pp[class][j] = pairs of expert j in that class
        #pragma unroll 1
        for (int j = lane; j < El; j += 32) {
            int n_all = 0;
            #pragma unroll 1
            for (int a = 0; a < P; ++a) n_all += ceil_tiles(T[((r - a + P) % P) * E + r + P * j]);
            #pragma unroll 1
            for (int a = 0; a < P; ++a) pp[a * El + pslot(a, j)] = 0;
            int a = 0, lim = ceil_tiles(T[r * E + r + P * j]);  // list positions [0, lim) come from class a
            #pragma unroll 1
            for (int m = 0; 2 * m < n_all; ++m) {
                const int last = min(2 * m + 1, n_all - 1);
                while (last >= lim) {
                    ++a;
                    lim += ceil_tiles(T[((r - a + P) % P) * E + r + P * j]);
                }
                ++pp[a * El + pslot(a, j)];
            }
        }
        const int32_t n_pairs = warp_scan(pp, E);  // class-major pair positions
        if (lane == 0) s_n_pairs = n_pairs;
    }
    sync128();
    // ---- phase B2: the per-PE group tables (one thread) ----
    if (tid == 0) {
        const int32_t n_send = s_n_send, n_recv = s_n_recv, n_pairs = s_n_pairs;
        {
            int g = 0;
            #pragma unroll 1
            for (int kd = 0; kd < P; ++kd) {
                const int d = kd < r ? kd : (kd < P - 1 ? kd + 1 : r);
                const int first = sp[kd * El];
                const int last = kd + 1 < P ? sp[(kd + 1) * El] : n_send;
                dst_first[d] = first;
                dst_n[d] = last - first;
                dst_group[d] = (d != r && last > first) ? g++ : -1;
            }
            n_dgroups = g;
            g = 0;
            #pragma unroll 1
            for (int ks = 0; ks < P; ++ks) {
                const int s = ks == 0 ? r : (ks <= r ? ks - 1 : ks);
                const int first = rp[ks * El], last = ks + 1 < P ? rp[(ks + 1) * El] : n_recv;
                src_first[s] = first;
                src_n[s] = last - first;
                src_group[s] = (s != r && last > first) ? g++ : -1;
            }
            #pragma unroll 1
            for (int a = 0; a < P; ++a) {
                cls_first[a] = pp[a * El];
                cls_n[a] = (a + 1 < P ? pp[(a + 1) * El] : n_pairs) - cls_first[a];
            }
            n_cgroups_pe = g;
            int sb = 0, rb = 0;
            #pragma unroll 1
            for (int i = 1; i < P; ++i) {
                const int dd = (r + i) % P, ss = (r - i + P) % P;
                send_base[dd] = sb;
                sb += dst_n[dd];
                recv_base[ss] = rb;
                rb += src_n[ss];
            }
            // self pairs ahead of the remote ones: enough to cover the arrival of
            // the first source's first signal group (host-estimated link time per
            // tile / compute time per pair), at least one wave of GEMM1 items
            const int n_self_p = cls_n[0];  // pairs of self tiles only
            int head = n_self_p;
            if (P > 1) {
                const int fs = (r - 1 + P) % P;
                const int fg = c.group_size > 0 ? min(c.group_size, src_n[fs]) : src_n[fs];
                head = min(n_self_p, max(c.self_head, int(ceilf(float(fg) * c.head_ratio))));
            }
            s_head = head;
        }
    }
    sync128();
    const uint64_t t_b = tl_now(c);

    const int gs = c.group_size;
    const int32_t n_send = s_n_send, n_recv = s_n_recv, n_pairs = s_n_pairs, rows_in_r = s_rows_in;
    const int32_t n_send_remote = P > 1 ? dst_first[r] : 0;
    const int32_t n_recv_self = src_n[r];
    const int32_t n_recv_remote = n_recv - n_recv_self;
    const int32_t n_groups = gs > 0 ? n_send_remote / gs : n_dgroups;
    const int32_t n_cgroups = gs > 0 ? n_recv_remote / gs : n_cgroups_pe;
    if (tid == 0 && gs > 0 && (n_send_remote % gs || n_recv_remote % gs)) s_err = 2;

    // ---- phase C: emit the send side (warps 0-3), the receive side (warps 4-5)
    // and the pair order (warps 6-7) ----
    if (warp < 4) {
        const int t2 = tid;  // 0..127
        #pragma unroll 1
        for (int e = t2; e < E; e += 128) {
            const int d = e % P, j = e / P;
            const int kd = d < r ? d : (d > r ? d - 1 : P - 1);
            const int32_t cnt = T[r * E + e];
            const int nt = ceil_tiles(cnt);
            const int32_t pos0 = sp[kd * El + j];
            const int64_t hrow = d != r ? int64_t(hr[(d * P + r) * El + j] - hr[d * P * El]) : int64_t(rows_in_r + selfo[j]);
            c.send_first[e] = pos0;
            #pragma unroll 1
            for (int ch = 0; ch < nt; ++ch) {
                const int p = pos0 + ch;
                if (p >= c.max_send) {
                    s_err = 3;
                    break;
                }
                SendTile st;
                st.expert = e;
                st.dst = d;
                st.row0 = ch * kTileRows;
                st.rows = min(kTileRows, cnt - ch * kTileRows);
                st.heap_row = hrow + int64_t(ch) * kTileRows;
                st.tile_id = d != r ? tb[r * E + e] + ch : -1;
                st.group = d == r ? -1 : (gs > 0 ? p / gs : dst_group[d]);
                st.recv_pos = d == r ? src_first[r] + (rp[j] - rp[0]) + ch : -1;  // self: matching RecvTile
                st.pad = 0;
                c.send[p] = st;
                c.send_done[p] = 0;
                if (d != r) c.sorder[send_base[d] + (p - dst_first[d])] = p;
            }
        }
        #pragma unroll 1
        for (int g = t2; g < n_groups; g += 128) {
            Group G;
            if (gs > 0) {
                G = Group{-1, g * gs, gs, 0};
            } else {
                int d = 0;
                while (dst_group[d] != g) ++d;
                G = Group{d, dst_first[d], dst_n[d], 0};
            }
            c.groups[g] = G;
            c.group_ctr[g] = 0;
        }
    } else if (warp < 6) {
        const int t2 = tid - 128;  // 0..63
        #pragma unroll 1
        for (int i = t2; i < P * El; i += 64) {
            const int s = i / El, j = i - s * El, e = r + P * j;
            const int ks = s == r ? 0 : (s < r ? s + 1 : s);
            const int32_t cnt = T[s * E + e];
            const int nt = ceil_tiles(cnt);
            const int32_t pos0 = rp[ks * El + j];
            const int64_t hrow = s != r ? int64_t(hr[(r * P + s) * El + j] - hr[r * P * El]) : int64_t(rows_in_r + selfo[j]);
            #pragma unroll 1
            for (int ch = 0; ch < nt; ++ch) {
                const int p = pos0 + ch;
                if (p >= c.max_recv) {
                    s_err = 5;
                    break;
                }
                RecvTile rt;
                rt.src = s;
                rt.e_local = j;
                rt.rows = min(kTileRows, cnt - ch * kTileRows);
                rt.tile_id = s != r ? tb[s * E + e] + ch : -1;
                rt.heap_row = hrow + int64_t(ch) * kTileRows;
                rt.ybuf_row = off[s * E + e] + int64_t(ch) * kTileRows;
                rt.cgroup = s == r ? -1 : (gs > 0 ? (p - n_recv_self) / gs : src_group[s]);
                rt.pad = 0;
                c.recv[p] = rt;
                c.tile_ctr[p] = 0;
                if (c.dedup) c.ex_done[p] = 0;
                c.g1_done[p] = 0;
                // processing order (1-CTA kernel): self tiles first, then remote tiles
                // source by source in arrival order
                c.rorder[s == r ? p : n_recv_self + recv_base[s] + (p - src_first[s])] = p;
            }
        }
        #pragma unroll 1
        for (int g = t2; g < n_cgroups; g += 64) {
            Group G;
            if (gs > 0) {
                G = Group{-1, n_recv_self + g * gs, gs, 0};
            } else {
                int s = 0;
                while (src_group[s] != g) ++s;
                G = Group{s, src_first[s], src_n[s], 0};
            }
            c.cgroups[g] = G;
            c.cgroup_ctr[g] = 0;
        }
    } else {
        const int t2 = tid - 192;  // 0..63
        // M-tile pairs in processing order: a head of self-only pairs (work while
        // the first remote group is in flight), the pairs with remote tiles class
        // by class = source by source in arrival order (their outputs travel
        // back, so they finish early), then the rest of the self-only pairs — the
        // tail needs no NVLink round trip
        const int n0 = cls_n[0], head = s_head;
        #pragma unroll 1
        for (int j = t2; j < El; j += 64) {
            int n_all = 0;
            #pragma unroll 1
            for (int a = 0; a < P; ++a) n_all += ceil_tiles(T[((r - a + P) % P) * E + r + P * j]);
            // recv positions of expert j's tiles in list (arrival) order: a cursor
            // that only moves forward (pairs take list positions 2m, 2m + 1, ...)
            int ca = 0, cstart = 0, cnt = ceil_tiles(T[r * E + r + P * j]), cur = 0;
            int cpos = rp[j];  // recv position of class 0's (self) first tile
            auto next_tile = [&]() {
                while (cur - cstart >= cnt) {
                    cstart += cnt;
                    ++ca;
                    const int s = (r - ca + P) % P;
                    cnt = ceil_tiles(T[s * E + r + P * j]);
                    const int ks = s == r ? 0 : (s < r ? s + 1 : s);
                    cpos = rp[ks * El + j];
                }
                return cpos + (cur++ - cstart);
            };
            int a = 0, lim = ceil_tiles(T[r * E + r + P * j]), in_cls = 0;
            #pragma unroll 1
            for (int m = 0; 2 * m < n_all; ++m) {
                const int last = min(2 * m + 1, n_all - 1);
                while (last >= lim) {
                    ++a;
                    lim += ceil_tiles(T[((r - a + P) % P) * E + r + P * j]);
                    in_cls = 0;
                }
                const int q = pp[a * El + pslot(a, j)] + in_cls++;
                const int po = a == 0 ? (q < head ? q : q + (n_pairs - n0)) : head + (q - n0);
                const int t0 = next_tile();
                const int t1 = 2 * m + 1 < n_all ? next_tile() : -1;
                if (po < c.max_recv) {
                    c.pairs[2 * po] = t0;
                    c.pairs[2 * po + 1] = t1;
                }
            }
        }
    }
    sync128();
    const uint64_t t_c = tl_now(c);
    if (tid == 0) {
        PlanHeader h;
        h.n_send = n_send;
        h.n_send_remote = n_send_remote;
        h.n_groups = n_groups;
        h.n_recv = n_recv;
        h.n_recv_remote = n_recv_remote;
        h.n_cgroups = n_cgroups;
        h.total_tiles = s_total_tiles;
        h.error = s_err;
        h.n_pairs = n_pairs;
        h.self_head = s_head;
        h.remote_rows_in = rows_in_r;
        *c.hdr = h;
        if (s_err) atomicAdd(&c.stats[kStatErrors], 1ull);
        tl_at(c, kTlPlanReady, t_ready);
        tl_at(c, kTlPlanB, t_b);
        tl_at(c, kTlPlanC, t_c);
    }
}

inline size_t plan_smem_bytes(const DevCtx& c) { return sizeof(int32_t) * (4 * size_t(c.P) * c.E + 4 * size_t(c.E) + 8); }

}  // namespace perseus
