/*
 * include/perseus.h — the C-ABI boundary of the B200-native Perseus MoE
 * expert-parallel layer (libperseus.so).
 *
 * The reference (`sigsim`, /root/reference/proj) is a C++20 static library
 * with no C ABI and no FFI.  Its hot-path operator API lives in
 * proj/include/sigsim/{workload,protocols,metrics,trace}.hpp.  This header is
 * the thin, plain-pointer ABI under our C++ drop-in (include/sigsim/ headers) and
 * under the Python mirror (paper_2605_00686_b200/): every entry point names the
 * reference interface it replaces.  No torch types, no C++ types cross it.
 *
 * Status codes mirror the reference's error taxonomy (sim.hpp:17-28) and its
 * CLI exit-code contract (tools/main.cpp:6,130-136):
 *   0 ok | 1 ConfigError | 2 verification/ordering failure | 3 runtime error
 *   (ModelError, CUDA error, signal-wait timeout).
 * perseus_last_error() returns the thread-local message of the last failure.
 */
#ifndef PERSEUS_H_
#define PERSEUS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PERSEUS_OK 0
#define PERSEUS_ERR_CONFIG 1
#define PERSEUS_ERR_VERIFY 2
#define PERSEUS_ERR_RUNTIME 3

#define PERSEUS_ABI_VERSION 1

const char* perseus_last_error(void);
int perseus_abi_version(void);

/* ---------------------------------------------------------------------------
 * Planner (host).  Same semantics as the reference free functions.
 * ------------------------------------------------------------------------- */

/* TransferSpec (workload.hpp:42-49), flattened. */
typedef struct perseus_transfer {
    uint32_t src_pe;
    uint32_t dst_pe;
    int64_t expert;
    uint64_t bytes;
    int64_t tile_id; /* globally unique; doubles as the flag-word id */
    uint64_t heap_offset;
} perseus_transfer;

/* replaces sigsim::remote_transfer_count (workload.hpp:72, workload.cpp:39-47) */
int perseus_remote_transfer_count(int64_t experts, int64_t pes, int64_t pes_per_node,
                                  int64_t* out);

/* replaces sigsim::message_size (workload.hpp:75-76, workload.cpp:49-55) */
uint64_t perseus_message_size(uint64_t tokens, int64_t top_k, int64_t experts,
                              int64_t hidden_dim);

/* replaces sigsim::zipf_route (workload.hpp:79-80, workload.cpp:57-97).
 * counts[E]; ids[S*k] (nullable) receives the per-token draws in draw order. */
int perseus_zipf_route(uint64_t tokens, int64_t experts, double exponent, int64_t top_k,
                       uint64_t seed, uint64_t* counts, int32_t* ids);

/* replaces sigsim::build_dispatch (workload.hpp:82-84, workload.cpp:155-213)
 * and DispatchWorkload::digest (workload.cpp:105-126).  Call with NULL arrays
 * to size them. */
int perseus_build_dispatch(int64_t hidden_dim, int64_t intermediate_dim, int64_t experts,
                           int64_t top_k, int nodes, int gpus_per_node, int num_qps,
                           uint64_t tokens, double skew, uint64_t tile_bytes, uint64_t seed,
                           perseus_transfer* remote, size_t remote_cap, size_t* n_remote,
                           perseus_transfer* local, size_t local_cap, size_t* n_local,
                           uint64_t* workload_digest);

/* replaces sigsim::assign_groups (protocols.hpp:58-59, protocols.cpp:52-94).
 * group_of[n]; leaders[n_groups] (nullable). */
int perseus_assign_groups(const perseus_transfer* transfers, size_t n, int64_t group_size,
                          int64_t* group_of, int64_t* leaders, size_t* n_groups);

/* replaces SymmetricHeap::digest (transport.hpp:130-156, transport.cpp:26-43):
 * extents[n_ext*3] = (pe, offset, length); flags[n_flags]. */
uint64_t perseus_heap_digest(const uint64_t* extents, size_t n_ext, const uint64_t* flags,
                             size_t n_flags);

/* replaces sigsim::fnv1a64 (trace.hpp:67, trace.cpp:53-62) */
uint64_t perseus_fnv1a64(const void* data, size_t len, uint64_t h);

/* ---------------------------------------------------------------------------
 * Layer (device).  One handle per (process, GPU, EP rank).
 *
 * replaces the reference's hot path run_dispatch (protocols.hpp:62-64,
 * protocols.cpp:346-362) — which only simulates the dispatch puts/signals and
 * stands in for the expert FFN with a timing model (protocols.cpp:294-322) —
 * with the real MoE-layer forward: gate/route -> permute -> dispatch puts +
 * signals over NVLink -> SwiGLU expert FFN on tcgen05 -> combine puts +
 * signals -> weighted reduce.
 * ------------------------------------------------------------------------- */

/* routing */
#define PERSEUS_ROUTE_BALANCED 0 /* reference exact-capacity routing (workload.cpp:180-195) */
#define PERSEUS_ROUTE_ZIPF 1     /* reference Zipf routing (workload.cpp:57-97) */
#define PERSEUS_ROUTE_GATE 2     /* learned top-k over fp32 gate logits (new) */

/* signalling (protocols.hpp:13-37 Signaling + group_size):
 *   COUPLED   — Put, Fence, Signal per transfer tile (vanilla, protocols.cpp:242-248)
 *   DECOUPLED — Alg. 1: puts + group counter, one fence per group, then the
 *               group's signals (protocols.cpp:250-292); group_size 0 = per PE
 *   NONE      — fault injection: fences suppressed (transport.cpp:104-106)
 *   FAULT_EARLY — fault injection: every dispatch flag is written when its
 *               tile's put is ISSUED (before the data, which then trails by
 *               200 us as on a congested link), no fence — the "signal before
 *               data" bug the ordering checker must catch (verify_ordering,
 *               metrics.cpp:118-138) */
#define PERSEUS_SIGNAL_COUPLED 0
#define PERSEUS_SIGNAL_DECOUPLED 1
#define PERSEUS_SIGNAL_NONE 2
#define PERSEUS_SIGNAL_FAULT_EARLY 3

/* group_size of DECOUPLED: 0 = one group per destination PE (assign_groups,
 * protocols.cpp:65-76); > 0 = fixed-size groups in (dst, expert, tile) order
 * (:77-88) — must divide every PE's remote tile count in both directions
 * (ConfigError at create, as run_dispatch's precheck protocols.cpp:348-359);
 * PERSEUS_GROUP_AUTO = the largest such common divisor g with 8 <= g <=
 * tiles-per-destination / 4 (>= 8x fewer fences than per tile, >= 4 groups per
 * destination), else per destination.  Sizes != 0 need balanced / Zipf routing. */
#define PERSEUS_GROUP_AUTO (-1)

typedef struct perseus_layer_config {
    int64_t hidden_dim;       /* H  (ModelConfig, workload.hpp:16-25) */
    int64_t intermediate_dim; /* I  */
    int64_t experts;          /* E  */
    int64_t top_k;            /* k  */
    uint64_t tokens_per_pe;   /* S  (DispatchWorkload::tokens_per_pe) */
    int32_t routing;          /* PERSEUS_ROUTE_* */
    double skew;              /* Zipf exponent (routing == ZIPF) */
    uint64_t seed;            /* workload seed (config.hpp:36) */
    int32_t signaling;        /* PERSEUS_SIGNAL_* */
    int64_t group_size;       /* DECOUPLED: 0 = per destination PE, > 0 fixed, PERSEUS_GROUP_AUTO */
    int32_t flags;            /* PERSEUS_F_* */
} perseus_layer_config;

#define PERSEUS_F_SYNTH_WEIGHTS 1 /* generate weights on device from `seed` */
#define PERSEUS_F_UNFUSED 2       /* forward() as stream-ordered stage kernels instead of the fused persistent kernel */
#define PERSEUS_F_NO_PAIR 4       /* fused kernel on single CTAs (cta_group::1) instead of CTA pairs (cta_group::2) */
#define PERSEUS_F_FORCE_PAIR 8    /* CTA pairs even when local experts get at most one 128-row tile */
/* compute-only twins (diagnostics; outputs are NOT the layer's): one
 * direction's peer stores and flag writes go to this rank's own buffers and its
 * receivers do not wait for that direction's flags — the same per-GPU kernels,
 * schedule and copy volume without the NVLink traffic.  T_layer - T_twin is the
 * exposed communication (the reference's twin-run decomposition,
 * metrics.cpp:97-116). */
/* one PE, CTA-pair kernel: the fused kernel combines each token as soon as its
 * k expert rows exist (a ready queue fed by GEMM2 tile completions, copy warps as
 * combiners) instead of the combine kernel after it; same bits.  Experimental:
 * slower at the bench shape. */
#define PERSEUS_F_DF_COMBINE 128
/* per-destination token dedup of the dispatch (P > 1, CTA-pair
 * kernel, not with tracing): a token whose k experts put several rows on one
 * destination crosses NVLink ONCE into that destination's per-source token
 * buffer, with the row -> token index of every (expert, row) of the reference
 * layout; the receiver expands the rows into the usual receive heap (a local
 * copy) and releases the tiles to its GEMMs.  One fence + one flag per
 * (source, destination).  Outputs are the layer's (bit-identical); the byte and
 * signal accounting is NOT the reference's, so it is reported separately. */
#define PERSEUS_F_DEDUP 256
#define PERSEUS_F_LOCAL_DISPATCH 32
#define PERSEUS_F_LOCAL_COMBINE 64
#define PERSEUS_F_NO_PDL 16       /* no programmatic dependent launch: for several ranks sharing ONE device
                                     (a grid waiting for its PDL primary holds up the work distributor, so
                                     another rank's grids the primary waits for may never be scheduled) */

/* Tile granularity: 128 token rows per transfer tile / GEMM M-tile, i.e. the
 * reference's tile_bytes = 128 * H * 2 (workload.hpp:58). */
#define PERSEUS_TILE_ROWS 128

typedef struct perseus_layer perseus_layer;

int perseus_layer_create(const perseus_layer_config* cfg, int rank, int world, int device,
                         perseus_layer** out);
int perseus_layer_destroy(perseus_layer* layer);

/* Symmetric-heap bootstrap (SymmetricHeap, transport.hpp:130-156): export this
 * rank's cudaIpc handle blob, then import every rank's blob (world * len bytes,
 * rank-major).  For ranks emulated inside ONE process on ONE device use
 * perseus_layer_connect_local instead (raw pointers, no IPC). */
int perseus_layer_ipc_export(perseus_layer* layer, void* blob, size_t cap, size_t* len);
int perseus_layer_ipc_import(perseus_layer* layer, const void* blobs, size_t len_each);
int perseus_layer_connect_local(perseus_layer* const* ranks, int world);

/* Weights (device pointers, bf16 row-major): router wg[E][H]; this rank's
 * experts e = rank + world*j: w1[E/P][2I][H] (gate rows then up rows),
 * w2[E/P][H][I].  Copied into the handle. */
int perseus_layer_set_weights(perseus_layer* layer, const void* wg, const void* w1,
                              const void* w2, void* stream);
/* Generate the synthetic bf16 tensors of the oracle's counter hash on device. */
int perseus_layer_init_synthetic(perseus_layer* layer, uint64_t seed, void* stream);
int perseus_fill_synthetic_x(perseus_layer* layer, void* x, uint64_t seed, void* stream);

/* Forward over this rank's S tokens: x[S][H] bf16 -> out[S][H] bf16 (device
 * pointers).  Launches asynchronously on `stream` (cudaStream_t, NULL =
 * default).  All ranks call it; ranks synchronise through device flags only. */
int perseus_layer_forward(perseus_layer* layer, const void* x, void* out, void* stream);

/* Same, from/to HOST buffers (pinned or pageable): H2D copy, forward, D2H copy,
 * stream-synchronised.  The end-to-end entry a reference user calls. */
int perseus_layer_forward_host(perseus_layer* layer, const void* x_host, void* out_host,
                               void* stream);

/* Pipelined end-to-end forward for a stream of batches (serving): enqueues the
 * H2D copy of x_host on an upload stream, the forward on the layer's stream and
 * the D2H copy into out_host on a download stream, and returns without waiting,
 * so batch n+1's upload and batch n-1's download overlap batch n's forward
 * (three device staging slots, so an upload has two forwards' time to land;
 * PERSEUS_HOST_SLOTS=2 for two).  Host buffers should be pinned and must stay valid
 * until perseus_layer_host_wait(). */
int perseus_layer_forward_host_async(perseus_layer* layer, const void* x_host, void* out_host);
/* Wait until every enqueued forward_host_async has its output in host memory. */
int perseus_layer_host_wait(perseus_layer* layer);

/* Phased forward for P ranks emulated on one device: phase p of every rank
 * must complete before phase p+1 of any rank (no cross-launch spin-waits on
 * one GPU).  PERSEUS_PHASE_ALL == perseus_layer_forward. */
#define PERSEUS_PHASE_ROUTE 0    /* gate/route + permutation + count publish */
#define PERSEUS_PHASE_DISPATCH 1 /* plan + dispatch puts + signals */
#define PERSEUS_PHASE_EXPERT 2   /* grouped SwiGLU FFN + combine puts + signals */
#define PERSEUS_PHASE_COMBINE 3  /* weighted reduce */
#define PERSEUS_PHASE_ALL 15
int perseus_layer_forward_phase(perseus_layer* layer, int phase, const void* x, void* out,
                                void* stream);

/* Evidence read-back (host copies, stream-synchronised). */
typedef struct perseus_counters {
    int64_t epoch;                 /* forwards run */
    int64_t dispatch_fences;       /* sys-scope fences issued, dispatch phase (this PE) */
    int64_t dispatch_signals;      /* flag words written to peers */
    int64_t dispatch_puts;         /* transfer tiles stored to peers */
    int64_t dispatch_put_bytes;
    int64_t combine_fences;
    int64_t combine_signals;
    int64_t combine_puts;
    int64_t combine_put_bytes;
    int64_t recv_tiles;            /* M-tiles processed by the expert FFN here */
    int64_t wait_timeouts;         /* bounded spin-waits that gave up (must be 0) */
    int64_t errors;                /* device-detected plan errors (must be 0) */
    int64_t wait_dispatch_ns;      /* fused kernel, summed over CTAs: producer blocked on dispatch flags */
    int64_t wait_g1_ns;            /* ... producer blocked on GEMM1->GEMM2 tile dependencies */
    int64_t copy_ns;               /* ... copy warps busy with dispatch puts */
    int64_t cta_ns;                /* ... CTA lifetimes (normaliser) */
    int64_t wait_remote_ns;        /* ... producer blocked on REMOTE dispatch flags (exposed dispatch) */
    int64_t dispatch_span_ns;      /* per forward, summed: first remote dispatch store -> last tile signalled */
    int64_t combine_span_ns;       /* ... first remote combine store -> last combine tile signalled */
    int64_t combine_wait_ns;       /* ... longest wait of a combine CTA for its combine flags (exposed combine) */
    int64_t mma_cycles;            /* CTA-pair kernel, MMA issuers, SM cycles in the issue loop (summed) */
    int64_t mma_ring_wait;         /* ... of which waiting for the next work item */
    int64_t mma_acc_wait;          /* ... waiting for a free TMEM accumulator (epilogue back-pressure) */
    int64_t mma_data_wait;         /* ... waiting for TMA operand stages */
} perseus_counters;
int perseus_layer_counters(perseus_layer* layer, perseus_counters* out);

/* Routing of the last forward: ids[S*k] int32, weights[S*k] fp32, counts[E]
 * (this rank's per-expert token counts), positions pos[S*k] (sorted slot of
 * each (token, j) pair).  Any pointer may be NULL. */
int perseus_layer_read_routing(perseus_layer* layer, int32_t* ids, float* weights,
                               int32_t* counts, int32_t* pos);

/* The dispatch layout this rank realised in the last forward, as reference
 * TransferSpecs (its remote transfer tiles with tile ids and heap offsets at
 * the destination), and the per-destination flag words observed set at this
 * rank.  n_* receive counts; call with NULL arrays to size. */
int perseus_layer_read_layout(perseus_layer* layer, perseus_transfer* sent, size_t cap,
                              size_t* n_sent, int64_t* flags_seen, size_t flags_cap,
                              size_t* n_flags_seen);

/* The count table [P][E] this rank received from all ranks in the last forward. */
int perseus_layer_read_count_table(perseus_layer* layer, int32_t* table);

/* Kernel timeline of every following forward (diagnostics): globaltimer ns
 * [start, end] per kernel in the order router GEMM, route, permute, plan,
 * fused kernel, combine, dispatch, GEMM1, GEMM2 (0 = did not run), then three
 * fused-kernel events as [first, last] over its CTAs: MMA issuer out of work
 * items, copy warps done, epilogue done.  Kernel start = first CTAs after their
 * dependency wait, end = last CTAs. */
int perseus_layer_set_timeline(perseus_layer* layer, int on);
int perseus_layer_read_timeline(perseus_layer* layer, uint64_t* start_end, int n_kernels);

/* replaces sigsim::fit_alpha_beta (metrics.hpp, metrics.cpp:69-95): least-squares
 * t = alpha + beta * bytes over n >= 2 points (ConfigError if degenerate). */
int perseus_fit_alpha_beta(const double* bytes, const double* ns, size_t n, double* alpha_ns,
                           double* beta_ns_per_byte, double* r_squared);

/* Which forward path the layer runs: fused persistent kernel or stage kernels;
 * CTA-pair (cta_group::2) tiles or 1-CTA tiles (chosen at create: pairs unless
 * PERSEUS_F_NO_PAIR, or — without PERSEUS_F_FORCE_PAIR — each local expert gets at
 * most one 128-row tile, or a single-PE layer's Zipf routing leaves the pairs
 * less than 85% useful (experts with odd tile counts)). */
int perseus_layer_info(perseus_layer* layer, int* fused, int* cta_pairs);

/* The DECOUPLED signal-group size this layer resolved at create (0 = per
 * destination PE; PERSEUS_GROUP_AUTO resolved to a size).  1 for the per-tile
 * protocols. */
int perseus_layer_group_size(perseus_layer* layer, int64_t* group_size);

/* Host only: the group size perseus_layer_create would resolve for `cfg` at EP
 * `world` (validation included: ConfigError for a size that does not divide
 * every PE's remote tile count, or != 0 with learned-gate routing). */
int perseus_resolve_group_size(const perseus_layer_config* cfg, int world, int64_t* group_size);

/* ---- device event log (trace mode) -> the reference's RunTrace ----------
 * With tracing on, every forward records what the kernels actually did:
 * sender-side puts, fences and flag writes, and receiver-side observations of
 * each remote tile's signal, with a content check of the tile at first
 * observation (receive buffers are poisoned before the forward; a signal seen
 * before the data landed is an ordering violation).  Events of one forward,
 * all PEs concatenated, are turned into a sigsim::RunTrace by
 * perseus_trace_analyze, which runs this library's fence_accounting,
 * verify_ordering and conservation_check on it (the drop-in restatements of
 * metrics.cpp:10-59,118-190 in csrc/planner.cpp).  perseus_trace_records hands
 * out the same records, so the reference's own checkers can be run on them
 * unmodified (oracle/ref_shim.cpp ref_analyze_records; tests compare the two
 * field for field). */
enum {
    PERSEUS_EV_DISPATCH_PUT = 1,    /* sender: a remote transfer tile's stores issued */
    PERSEUS_EV_DISPATCH_FENCE = 2,  /* sender: a group's sys-scope fence */
    PERSEUS_EV_DISPATCH_SIGNAL = 3, /* sender: one flag word written */
    PERSEUS_EV_DISPATCH_SEEN = 4,   /* receiver: first observation of a tile's flag (+ content check) */
    PERSEUS_EV_COMBINE_PUT = 5,
    PERSEUS_EV_COMBINE_FENCE = 6,
    PERSEUS_EV_COMBINE_SIGNAL = 7,
    PERSEUS_EV_COMBINE_SEEN = 8
};
typedef struct perseus_trace_event {
    uint64_t t;      /* globaltimer ns of the recording PE */
    int32_t kind;    /* PERSEUS_EV_* */
    int32_t pe;      /* recording PE */
    int32_t peer;    /* sender events: destination PE; receiver events: source PE */
    int32_t tile;    /* reference tile id (= flag id); -1 for fences */
    int32_t group;   /* sender's signal group (-1: none) */
    uint32_t bytes;  /* puts: payload bytes; SEEN: ns from signal seen to content complete */
    uint32_t aux;    /* SIGNAL: 1 = first flag after its group's fence; SEEN: 1 = content complete when seen */
    uint32_t pad;
} perseus_trace_event;

/* Turn tracing on/off (allocates the event log; poisons receive buffers per forward). */
int perseus_layer_set_trace(perseus_layer* layer, int on);
/* Events of the last forward (call with events = NULL to size). */
int perseus_layer_read_trace(perseus_layer* layer, perseus_trace_event* events, size_t cap, size_t* n);

typedef struct perseus_trace_report {
    int64_t records;                   /* RunTrace records built */
    int64_t fence_count[2];            /* fence_accounting per direction [dispatch, combine], all PEs */
    int64_t flagged_signal_count[2];
    int64_t ordering_violations[2];    /* verify_ordering: signal visible before the data landed */
    int64_t late_tiles[2];             /* tiles whose content was incomplete when first seen */
    int32_t conservation_ok[2];        /* conservation_check against the realised transfer list */
    int64_t put_bytes[2];
    char conservation_error[256];
} perseus_trace_report;

/* Build one sigsim::RunTrace per direction from the events of one forward (all
 * PEs) and run the checks.  `nic_ordering`: 0 = ProxyFence (vanilla / decoupled:
 * a fence marker per group), 1 = NicFence (combined / nic_ordering: the fence
 * marker arms the flag of the group's first signal, so both are counted, as the
 * reference's fence_accounting does), 2 = GPU-direct (the reference records
 * neither; the device fences are the memory model's, protocols.cpp:244-246).  `transfers` = the dispatch
 * transfers the PEs realised (perseus_layer_read_layout of every PE); the
 * combine direction mirrors them (same tiles, reversed). */
int perseus_trace_analyze(const perseus_trace_event* events, size_t n, int nic_ordering,
                          const perseus_transfer* transfers, size_t n_transfers, perseus_trace_report* out);
/* One sigsim::TraceRecord (trace.hpp:33-46), flattened; enums as the reference's
 * underlying values (ReqKind: 0 Put, 1 Signal, 2 FenceMarker; TraceKind: 0 Submit,
 * 1 NicServiceStart, 2 Completion, 3 SignalVisible, ...). */
typedef struct perseus_trace_record {
    int64_t time;
    uint32_t pe;
    int32_t kind;
    int32_t req_kind;
    uint32_t src_pe;
    uint32_t dst_pe;
    int32_t fence_flag;
    uint64_t size;
    int32_t qp;
    int32_t pad;
    int64_t group_id;
    int64_t tile_id;
    uint64_t submit_seq;
} perseus_trace_record;

/* The records of one direction's RunTrace (the one perseus_trace_analyze checks),
 * plus its total_put_bytes_submitted / _delivered; call with out = NULL to size. */
int perseus_trace_records(const perseus_trace_event* events, size_t n, int nic_ordering, int direction,
                          perseus_trace_record* out, size_t cap, size_t* len, uint64_t* submitted_bytes,
                          uint64_t* delivered_bytes);

/* The same RunTrace of one direction (0 dispatch, 1 combine) in the reference's text
 * format (sigsim::serialize_trace, trace.cpp:33-51); call with buf = NULL to size. */
int perseus_trace_serialize(const perseus_trace_event* events, size_t n, int nic_ordering, int direction,
                            char* buf, size_t cap, size_t* len);

/* Record per-stage CUDA events in every following forward (off by default: each
 * event record costs stream time). */
int perseus_layer_set_stage_timing(perseus_layer* layer, int on);

/* Timing of the stages of the last perseus_layer_forward, in ms (CUDA events on
 * its stream): [route+permute, plan+dispatch, GEMM1+SwiGLU, GEMM2+combine-put,
 * combine].  Fused path: [route+permute, plan, fused kernel, -, combine].
 * Config error unless stage timing was on for that forward. */
int perseus_layer_read_timing(perseus_layer* layer, float* ms, int n);

#ifdef __cplusplus
}
#endif
#endif /* PERSEUS_H_ */
