// layer_dev.h — the by-value kernel context of one layer rank.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>

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
    const int32_t* zipf_ids;  // [S*k]: reference Zipf draws (routing == ZIPF)
    bf16* hbuf;          // [R_max][I]

    // symmetric buffers, one base pointer per PE (peer-mapped; [rank] = local)
    int32_t* count_table[kMaxPes];  // [2][P][E]
    uint32_t* count_flag[kMaxPes];  // [P]
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
    // fused-kernel scheduling (rebuilt by k_plan every forward)
    int32_t* sorder;      // [max_send]: send positions in copy order (dst-interleaved)
    int32_t* rorder;      // [max_recv]: recv positions in processing order (self, then by arrival)
    uint32_t* send_done;  // [max_send]: rows copied per send tile
    uint32_t* g1_done;    // [max_recv]: GEMM1 n-blocks finished per M-tile
    uint32_t* self_ready; // [max_recv]: epoch when a self tile's rows are in the heap
    uint32_t* sched;      // [4]: work-item / copy-unit counters
    int32_t* send_first;  // [E]: first send position of each expert's tiles
    int32_t* pairs;       // [max_recv][2]: M-tile pairs (recv positions, -1 = none) in processing order

    unsigned long long* stats;  // [kStatCount]
};

}  // namespace perseus
