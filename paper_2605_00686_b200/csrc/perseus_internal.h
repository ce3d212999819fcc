// perseus_internal.h — shared host/device types of libperseus.so (not part of
// the public ABI).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "sigsim/sim.hpp"

namespace perseus {

// ----------------------------------------------------------- error glue ----
struct VerifyError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

void set_last_error(const std::string& msg);

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const sigsim::ConfigError& e) {
        set_last_error(std::string("ConfigError: ") + e.what());
        return 1;
    } catch (const VerifyError& e) {
        set_last_error(std::string("VerifyError: ") + e.what());
        return 2;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return 3;
    }
}

// ------------------------------------------------------- device plan ----
constexpr int kTileRows = 128;     // transfer tile == GEMM M-tile (PERSEUS_TILE_ROWS)
constexpr int kMaxPes = 8;

// One transfer tile this rank sends in the dispatch phase — the device
// realisation of one reference TransferSpec tile (workload.hpp:42-49).
struct SendTile {
    int32_t expert;    // global expert id
    int32_t dst;       // destination PE (== e % P)
    int32_t row0;      // first row inside the expert's sorted segment
    int32_t rows;      // <= kTileRows
    int64_t heap_row;  // first destination row in dst's receive heap
    int32_t tile_id;   // reference tile id == flag word id (-1: self segment)
    int32_t group;     // signal group (-1: self segment, no signal)
    int32_t recv_pos;  // self segment: position of the matching RecvTile (else -1)
    int32_t pad;
};

// Signal group: members are a contiguous run of the tile list in the
// reference's (dst, expert, tile) order (assign_groups, protocols.cpp:52-94).
struct Group {
    int32_t peer;   // destination of the group's signals
    int32_t first;  // first member index
    int32_t count;  // members (== target)
    int32_t pad;
};

// One M-tile of expert-FFN work at this rank (a received transfer tile, or a
// tile of this rank's own tokens for a local expert).
struct RecvTile {
    int32_t src;       // PE that owns the tokens (combine destination)
    int32_t e_local;   // local expert index (global e = rank + P*e_local)
    int32_t rows;
    int32_t tile_id;   // dispatch flag id (-1: self)
    int64_t heap_row;  // first A row in the receive heap
    int64_t ybuf_row;  // first row in src's combine buffer (src's sorted slot)
    int32_t cgroup;    // combine-direction signal group (-1: self)
    int32_t pad;
};

struct PlanHeader {
    int32_t n_send;         // send tiles (remote first, then self)
    int32_t n_send_remote;
    int32_t n_groups;
    int32_t n_recv;         // recv tiles (self first, then remote)
    int32_t n_recv_remote;
    int32_t n_cgroups;
    int32_t total_tiles;    // reference tile ids in use (all PEs)
    int32_t error;
    int32_t n_pairs;        // M-tile pairs (same expert) for the CTA-pair kernel
    int32_t self_head;      // self pairs processed before the remote ones
    int64_t remote_rows_in; // rows received from peers (heap rows before the self segment)
};

// Device statistics, one slot per counter (perseus_counters order).
enum StatSlot : int {
    kStatDispatchFences = 0,
    kStatDispatchSignals,
    kStatDispatchPuts,
    kStatDispatchBytes,
    kStatCombineFences,
    kStatCombineSignals,
    kStatCombinePuts,
    kStatCombineBytes,
    kStatRecvTiles,
    kStatTimeouts,
    kStatErrors,
    kStatWaitDispatchNs,  // fused kernel: producer time blocked on dispatch / self-ready flags
    kStatWaitG1Ns,        // ... blocked on GEMM1 -> GEMM2 tile dependencies
    kStatCopyNs,          // ... copy-warp busy time (dispatch puts)
    kStatCtaNs,           // ... summed CTA lifetimes
    kStatWaitRemoteNs,    // ... producer time blocked on REMOTE dispatch flags only (exposed dispatch)
    kStatDispatchSpanNs,  // first remote dispatch store -> last remote tile signalled, per forward
    kStatCombineSpanNs,   // first remote combine store -> last remote combine tile signalled
    kStatCombineWaitNs,   // longest combine-kernel CTA wait for its combine flags (exposed combine)
    kStatMmaCycles,       // fused pair kernel, MMA issuer: SM cycles in the issue loop
    kStatMmaRingWait,     // ... waiting for the next work item
    kStatMmaAccWait,      // ... waiting for a free TMEM accumulator (epilogue back-pressure)
    kStatMmaDataWait,     // ... waiting for operand stages (TMA)
    kStatCount
};

// Device event log (trace mode): what the kernels actually did, in the
// reference's evidence vocabulary (trace.hpp:12-69); see perseus.h
// perseus_trace_event for the host view and planner.cpp for the adapter.
struct TraceEv {
    uint64_t t;       // globaltimer ns of the recording PE
    int32_t kind;     // PERSEUS_EV_*
    int32_t pe;       // recording PE
    int32_t peer;     // sender events: destination; receiver events: source
    int32_t tile;     // reference tile id (flag id); -1 for fences
    int32_t group;    // signal group of the sender (-1: none)
    uint32_t bytes;   // puts: payload bytes; observes: ns from signal seen to content complete
    uint32_t aux;     // signals: 1 = first flag after the group's fence; observes: 1 = content complete when seen
    uint32_t pad;
};

// diagnostic event kinds (trace mode; ignored by perseus_trace_analyze):
//   self tile copied (tile = recv position), GEMM1 item dependency wait
//   (tile = recv position, group = n-block, bytes = ns waited, aux = item index)
constexpr int kEvDiagSelfReady = 20, kEvDiagItemWait = 21;

// Per-forward communication timestamps (globaltimer ns), reset by the plan
// kernel and folded into the stats by the combine kernel's last CTA.
enum FwdSlot : int {
    kFwdDispFirst = 0, kFwdDispLast, kFwdCombFirst, kFwdCombLast, kFwdUnused, kFwdWaitMax, kFwdDoneCtas,
    kFwdSlots = 8
};

}  // namespace perseus

#include "perseus.h"
#include "sigsim/trace.hpp"

namespace perseus {

// One direction (0 dispatch, 1 combine) of one forward's device events (all PEs)
// as a sigsim::RunTrace; ordering 0 ProxyFence, 1 NicFence, 2 GPU-direct
// (planner.cpp; perseus_trace_analyze / _records / _serialize and the
// GPU-backed sigsim::run_dispatch build on it).
sigsim::RunTrace device_run_trace(const perseus_trace_event* ev, size_t n, int dir, int ordering,
                                  int64_t* late_tiles);

constexpr uint64_t kWaitTimeoutNs = 4000000000ull;  // 4 s: a lost signal errors out, never hangs

}  // namespace perseus
