// signal.cuh — Phase 2 of Perseus Alg. 1 (protocols.cpp:275-292) on the GPU.
#pragma once

#include "layer_dev.h"
#include "perseus.h"
#include "ptx.cuh"

namespace perseus {

// Executed by ONE full warp once a group's counter completes: lane 0 issues
// the group's single sys-scope fence, then the 32 lanes write the members'
// flag words (epoch-valued).  The fence is the only ordering point; issuing
// warps never stall on it (the NIC-side-ordering analogue).
// With `suppress` (fault injection, transport.cpp:104-106) the fence is dropped.
template <class FlagOf>
__device__ __forceinline__ void signal_group_warp(const DevCtx& c, const Group& g, int gid, FlagOf flag_of,
                                                  bool suppress, int stat_fence, int stat_signal) {
    const int lane = threadIdx.x & 31;
    const bool combine = stat_fence == kStatCombineFences;
    if (lane == 0 && !suppress) {
        ptx::fence_acq_rel_sys();
        atomicAdd(&c.stats[stat_fence], 1ull);
        if (c.trace) trace_ev(c, combine ? PERSEUS_EV_COMBINE_FENCE : PERSEUS_EV_DISPATCH_FENCE, g.peer, -1, gid, 0, 0, fwd_now());
    }
    __syncwarp();
    for (int m = lane; m < g.count; m += 32) {
        ptx::st_relaxed_sys(flag_of(g.first + m), c.epoch);
        if (c.trace) {
            const int mi = g.first + m;
            const int tile = combine ? c.recv[mi].tile_id : c.send[mi].tile_id;
            const int peer = combine ? c.recv[mi].src : c.send[mi].dst;
            trace_ev(c, combine ? PERSEUS_EV_COMBINE_SIGNAL : PERSEUS_EV_DISPATCH_SIGNAL, peer, tile, gid, 0,
                     (m == 0 && !suppress) ? 1u : 0u, fwd_now());
        }
    }
    if (lane == 0) atomicAdd(&c.stats[stat_signal], (unsigned long long)g.count);
}

// Phase 1 for one finished member by a full warp: lane 0 bumps the group
// counter (gpu-scope acq_rel: the member's data stores, ordered before this
// by a CTA barrier, are published cumulatively); the warp that completes the
// group runs Phase 2.  Groups of one member skip the counter.
template <class FlagOf>
__device__ __forceinline__ void publish_member_warp(const DevCtx& c, const Group& g, uint32_t* ctr,
                                                    FlagOf flag_of, bool suppress, int stat_fence,
                                                    int stat_signal) {
    bool run = g.count == 1;
    if (!run) {
        uint32_t last = 0;
        if ((threadIdx.x & 31) == 0) last = ptx::atom_add_acq_rel_gpu(ctr, 1u) + 1 == uint32_t(g.count);
        run = __shfl_sync(0xffffffffu, last, 0) != 0;
    }
    if (run) {
        const int gid = int(ctr - (stat_fence == kStatCombineFences ? c.cgroup_ctr : c.group_ctr));
        signal_group_warp(c, g, gid, flag_of, suppress, stat_fence, stat_signal);
    }
}

}  // namespace perseus
