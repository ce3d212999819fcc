/*
 * oracle/oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithms on the Perseus MoE
 * expert-parallel hot path, used as the CHECKER for the CUDA product.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it;
 * the product (paper_2605_00686_b200/) never links or calls it.
 *
 * Parity pinning: the integer parts (RNG, Zipf routing, dispatch layout, tile
 * ids, heap offsets, signal groups, fence counts, digests) are checked against
 * the reference library itself (oracle/_ref, built from /root/reference
 * sources) and against the golden vectors in tests/golden/ generated from it.
 * The layer arithmetic (gate logits, top-k, SwiGLU FFN, combine) has NO
 * reference counterpart (the reference has no MoE arithmetic)
 * — that part is "parity unpinned" and defined here; fp tolerance lives in the
 * tests.
 *
 * Citations are to /root/reference/proj unless stated.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* RNG: restatement of sigsim::SeededRng (include/sigsim/sim.hpp:33-72)       */
/* ------------------------------------------------------------------------- */
EXPORT uint64_t orc_splitmix64(uint64_t x) { /* sim.hpp:63-68 */
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

typedef struct { uint64_t state; } orc_rng;

static void rng_init(orc_rng* r, uint64_t seed) { r->state = orc_splitmix64(seed); }

static uint64_t rng_u64(orc_rng* r) { /* sim.hpp:39-47, xorshift64* */
    uint64_t x = r->state;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    r->state = x;
    return x * 0x2545F4914F6CDD1DULL;
}

static uint64_t rng_below(orc_rng* r, uint64_t bound) { /* sim.hpp:50-57 */
    if (bound == 0) return 0;
    uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        uint64_t v = rng_u64(r);
        if (v >= threshold) return v % bound;
    }
}

static double rng_double(orc_rng* r) { /* sim.hpp:60 */
    return (double)(rng_u64(r) >> 11) * 0x1.0p-53;
}

EXPORT void orc_rng_stream(uint64_t seed, uint64_t n, uint64_t* out) {
    orc_rng r;
    rng_init(&r, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_u64(&r);
}

/* ------------------------------------------------------------------------- */
/* FNV-1a-64: restatement of sigsim::fnv1a64 (src/trace.cpp:53-62)           */
/* ------------------------------------------------------------------------- */
EXPORT uint64_t orc_fnv1a64(const void* data, size_t len, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}
#define FNV_OFFSET 0xcbf29ce484222325ULL
static uint64_t mix_u64(uint64_t h, uint64_t v) { return orc_fnv1a64(&v, 8, h); }
static uint64_t mix_u32(uint64_t h, uint32_t v) { return orc_fnv1a64(&v, 4, h); }

/* ------------------------------------------------------------------------- */
/* Workload geometry (src/workload.cpp:39-55)                                 */
/* ------------------------------------------------------------------------- */
/* returns -1 on ConfigError */
EXPORT int64_t orc_remote_transfer_count(int64_t E, int64_t P, int64_t P_local) {
    if (P <= 0 || E <= 0) return -1;
    if (E % P != 0) return -1;
    if (P_local > P) return -1;
    return (P - P_local) * (E / P);
}

EXPORT uint64_t orc_message_size(uint64_t S, int64_t k, int64_t E, int64_t H) {
    if (S == 0) return 0;
    uint64_t cap = S * (uint64_t)k / (uint64_t)E;
    return cap * (uint64_t)H * 2;
}

/* ------------------------------------------------------------------------- */
/* Routing                                                                    */
/* ------------------------------------------------------------------------- */
/* Zipf routing, restating sigsim::zipf_route (src/workload.cpp:57-97), extended
 * to also emit the per-token expert ids in draw order (ids[t*k + j] is the j-th
 * accepted draw for token t).  counts[] must equal the reference bit-exactly.
 * returns 0, or 1 on ConfigError. */
EXPORT int orc_zipf_route(uint64_t S, int64_t E, double s, int64_t k, uint64_t seed,
                          uint64_t* counts, int32_t* ids) {
    if (s < 0.0) return 1;
    if (k > E) return 1;
    orc_rng r;
    rng_init(&r, seed);
    int64_t* rank_to_expert = (int64_t*)malloc(sizeof(int64_t) * (size_t)E);
    double* cdf = (double*)malloc(sizeof(double) * (size_t)E);
    for (int64_t i = 0; i < E; ++i) rank_to_expert[i] = i;
    for (int64_t i = E; i > 1; --i) { /* seeded Fisher-Yates, workload.cpp:65-70 */
        int64_t j = (int64_t)rng_below(&r, (uint64_t)i);
        int64_t tmp = rank_to_expert[i - 1];
        rank_to_expert[i - 1] = rank_to_expert[j];
        rank_to_expert[j] = tmp;
    }
    double acc = 0.0; /* workload.cpp:72-78 */
    for (int64_t q = 0; q < E; ++q) {
        acc += pow((double)(q + 1), -s);
        cdf[q] = acc;
    }
    for (int64_t q = 0; q < E; ++q) cdf[q] /= acc;
    memset(counts, 0, sizeof(uint64_t) * (size_t)E);
    int64_t chosen[1024];
    for (uint64_t t = 0; t < S; ++t) { /* workload.cpp:83-95 */
        int64_t n = 0;
        while (n < k) {
            double u = rng_double(&r);
            /* std::lower_bound: first q with cdf[q] >= u */
            int64_t lo = 0, hi = E;
            while (lo < hi) {
                int64_t mid = lo + (hi - lo) / 2;
                if (cdf[mid] < u) lo = mid + 1; else hi = mid;
            }
            int64_t q = lo >= E ? E - 1 : lo;
            int64_t ex = rank_to_expert[q];
            int dup = 0;
            for (int64_t c = 0; c < n; ++c) if (chosen[c] == ex) { dup = 1; break; }
            if (dup) continue;
            chosen[n] = ex;
            if (ids) ids[t * (uint64_t)k + (uint64_t)n] = (int32_t)ex;
            ++n;
            counts[ex] += 1;
        }
    }
    free(rank_to_expert);
    free(cdf);
    return 0;
}

/* Balanced routing: the reference fixes counts only (every (src, expert) pair
 * gets exactly EC = S*k/E tokens, workload.cpp:180-195).  Per-token ids are
 * the round-robin id[t*k+j] = (t*k+j) mod E: distinct per token for k <= E
 * and exactly EC per expert when E | S*k. */
EXPORT int orc_balanced_ids(uint64_t S, int64_t E, int64_t k, int32_t* ids) {
    if (k > E) return 1;
    if (((S * (uint64_t)k) % (uint64_t)E) != 0) return 1; /* workload.cpp:165-168 */
    for (uint64_t i = 0; i < S * (uint64_t)k; ++i) ids[i] = (int32_t)(i % (uint64_t)E);
    return 0;
}

EXPORT void orc_counts_from_ids(const int32_t* ids, uint64_t S, int64_t k, int64_t E,
                                uint64_t* counts) {
    memset(counts, 0, sizeof(uint64_t) * (size_t)E);
    for (uint64_t i = 0; i < S * (uint64_t)k; ++i) counts[ids[i]] += 1;
}

/* ------------------------------------------------------------------------- */
/* Dispatch layout: restatement of build_dispatch / append_transfer           */
/* (src/workload.cpp:132-151,155-213) over an explicit [P x E] count table.   */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint32_t src_pe, dst_pe;
    int64_t expert;
    uint64_t bytes;
    int64_t tile_id;
    uint64_t heap_offset;
} orc_transfer;

static int cmp_transfer(const void* a, const void* b) { /* workload.cpp:204-211 */
    const orc_transfer* x = (const orc_transfer*)a;
    const orc_transfer* y = (const orc_transfer*)b;
    if (x->src_pe != y->src_pe) return x->src_pe < y->src_pe ? -1 : 1;
    if (x->dst_pe != y->dst_pe) return x->dst_pe < y->dst_pe ? -1 : 1;
    if (x->expert != y->expert) return x->expert < y->expert ? -1 : 1;
    if (x->tile_id != y->tile_id) return x->tile_id < y->tile_id ? -1 : 1;
    return 0;
}

/* counts: [P x E] token counts per (src, expert); bytes = count*H*2.
 * Outputs are sorted like the reference.  Returns 0, or 1 on ConfigError. */
EXPORT int orc_layout_from_counts(const uint64_t* counts, int64_t H, int64_t E, int nodes,
                                  int gpn, uint64_t tile_bytes, orc_transfer* remote,
                                  size_t remote_cap, size_t* n_remote, orc_transfer* local,
                                  size_t local_cap, size_t* n_local) {
    const int64_t P = (int64_t)nodes * gpn;
    if (E % P != 0) return 1;
    uint64_t* cursor = (uint64_t*)calloc((size_t)P, sizeof(uint64_t));
    int64_t next_tile = 0;
    size_t nr = 0, nl = 0;
    for (int64_t src = 0; src < P; ++src) {
        for (int64_t e = 0; e < E; ++e) {
            uint32_t dst = (uint32_t)(e % P); /* round-robin placement, workload.cpp:191 */
            uint64_t bytes = counts[src * E + e] * (uint64_t)H * 2;
            if ((int64_t)dst == src) continue; /* same PE: no transfer, :196 */
            int is_local = (dst / (uint32_t)gpn) == ((uint32_t)src / (uint32_t)gpn);
            if (bytes == 0) continue; /* append_transfer omits empty payloads, :135 */
            uint64_t tile = tile_bytes == 0 ? bytes : tile_bytes;
            for (uint64_t off = 0; off < bytes; off += tile) {
                uint64_t chunk = bytes - off < tile ? bytes - off : tile;
                orc_transfer t = {(uint32_t)src, dst, e, chunk, next_tile++, cursor[dst]};
                cursor[dst] += chunk;
                if (is_local) {
                    if (local && nl < local_cap) local[nl] = t;
                    ++nl;
                } else {
                    if (remote && nr < remote_cap) remote[nr] = t;
                    ++nr;
                }
            }
        }
    }
    free(cursor);
    if (remote && nr <= remote_cap) qsort(remote, nr, sizeof(orc_transfer), cmp_transfer);
    if (local && nl <= local_cap) qsort(local, nl, sizeof(orc_transfer), cmp_transfer);
    *n_remote = nr;
    *n_local = nl;
    return 0;
}

/* The per-(src, expert) count table build_dispatch uses (workload.cpp:178-195):
 * skew > 0 -> zipf_route per src with seed ^ (golden * (src+1)); else balanced. */
EXPORT int orc_route_counts(uint64_t S, int64_t E, int64_t k, double skew, uint64_t seed, int P,
                            uint64_t* counts /* P x E */, int32_t* ids /* P x S x k or NULL */) {
    for (int src = 0; src < P; ++src) {
        int32_t* id_src = ids ? ids + (uint64_t)src * S * (uint64_t)k : NULL;
        if (skew > 0.0) {
            uint64_t s_seed = seed ^ (0x9E3779B97F4A7C15ULL * (uint64_t)(src + 1));
            if (orc_zipf_route(S, E, skew, k, s_seed, counts + (uint64_t)src * E, id_src)) return 1;
        } else {
            if (S > 0 && ((S * (uint64_t)k) % (uint64_t)E) != 0) return 1;
            for (int64_t e = 0; e < E; ++e) counts[(uint64_t)src * E + e] = S * (uint64_t)k / (uint64_t)E;
            if (id_src && S > 0) orc_balanced_ids(S, E, k, id_src);
        }
    }
    return 0;
}

/* DispatchWorkload::digest (workload.cpp:105-126) */
EXPORT uint64_t orc_workload_digest(int nodes, int gpn, uint64_t S, double skew,
                                    uint64_t tile_bytes, const orc_transfer* remote, size_t nr,
                                    const orc_transfer* local, size_t nl) {
    uint64_t h = FNV_OFFSET;
    h = mix_u64(h, (uint64_t)nodes);
    h = mix_u64(h, (uint64_t)gpn);
    h = mix_u64(h, S);
    h = mix_u64(h, (uint64_t)(skew * 1e6));
    h = mix_u64(h, tile_bytes);
    for (size_t i = 0; i < nr; ++i) {
        h = mix_u64(h, (uint64_t)remote[i].src_pe);
        h = mix_u64(h, (uint64_t)remote[i].dst_pe);
        h = mix_u64(h, (uint64_t)remote[i].expert);
        h = mix_u64(h, remote[i].bytes);
    }
    for (size_t i = 0; i < nl; ++i) {
        h = mix_u64(h, (uint64_t)local[i].src_pe);
        h = mix_u64(h, (uint64_t)local[i].dst_pe);
        h = mix_u64(h, local[i].bytes);
    }
    (void)mix_u32;
    return h;
}

/* SymmetricHeap::digest (src/transport.cpp:26-43): FNV over the (pe, offset,
 * length) extents sorted by (pe, offset, length), then over the set flag ids
 * in ascending order.  For a dispatch in which every transfer lands and is
 * signaled, the extents are the transfers' (dst, heap_offset, bytes) and the
 * flags are their tile ids. */
typedef struct { uint64_t pe, off, len; } orc_extent;
static int cmp_extent(const void* a, const void* b) {
    const orc_extent* x = (const orc_extent*)a;
    const orc_extent* y = (const orc_extent*)b;
    if (x->pe != y->pe) return x->pe < y->pe ? -1 : 1;
    if (x->off != y->off) return x->off < y->off ? -1 : 1;
    if (x->len != y->len) return x->len < y->len ? -1 : 1;
    return 0;
}
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
EXPORT uint64_t orc_heap_digest(const uint64_t* ext /* n x 3: pe, off, len */, size_t n_ext,
                                const uint64_t* flags, size_t n_flags) {
    orc_extent* e = (orc_extent*)malloc(sizeof(orc_extent) * (n_ext ? n_ext : 1));
    for (size_t i = 0; i < n_ext; ++i) e[i] = (orc_extent){ext[3 * i], ext[3 * i + 1], ext[3 * i + 2]};
    qsort(e, n_ext, sizeof(orc_extent), cmp_extent);
    uint64_t* f = (uint64_t*)malloc(sizeof(uint64_t) * (n_flags ? n_flags : 1));
    memcpy(f, flags, sizeof(uint64_t) * n_flags);
    qsort(f, n_flags, sizeof(uint64_t), cmp_u64);
    uint64_t h = FNV_OFFSET;
    for (size_t i = 0; i < n_ext; ++i) {
        uint64_t v[3] = {e[i].pe, e[i].off, e[i].len};
        h = orc_fnv1a64(v, sizeof(v), h);
    }
    for (size_t i = 0; i < n_flags; ++i) {
        if (i > 0 && f[i] == f[i - 1]) continue; /* std::map keys are unique */
        h = orc_fnv1a64(&f[i], 8, h);
    }
    free(e);
    free(f);
    return h;
}

/* ------------------------------------------------------------------------- */
/* Signal groups: restatement of assign_groups (src/protocols.cpp:52-94)      */
/* ------------------------------------------------------------------------- */
static const orc_transfer* g_sort_base;
static int cmp_idx_dst_expert_tile(const void* a, const void* b) {
    const orc_transfer* x = &g_sort_base[*(const size_t*)a];
    const orc_transfer* y = &g_sort_base[*(const size_t*)b];
    if (x->dst_pe != y->dst_pe) return x->dst_pe < y->dst_pe ? -1 : 1;
    if (x->expert != y->expert) return x->expert < y->expert ? -1 : 1;
    if (x->tile_id != y->tile_id) return x->tile_id < y->tile_id ? -1 : 1;
    /* std::sort is unstable; ties cannot occur for unique tile ids */
    return 0;
}

/* group_of[i] = group of transfer i; leaders[g] = first member of group g in
 * (dst, expert, tile) order.  Returns 0 or 1 on ConfigError. */
EXPORT int orc_assign_groups(const orc_transfer* t, size_t n, int64_t group_size,
                             int64_t* group_of, int64_t* leaders, size_t* n_groups) {
    size_t* order = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
    for (size_t i = 0; i < n; ++i) order[i] = i;
    g_sort_base = t;
    qsort(order, n, sizeof(size_t), cmp_idx_dst_expert_tile);
    size_t ng = 0;
    if (group_size == 0) { /* one group per destination, in first-seen dst order */
        int64_t last_dst = -1;
        for (size_t p = 0; p < n; ++p) {
            size_t idx = order[p];
            if ((int64_t)t[idx].dst_pe != last_dst) {
                if (leaders) leaders[ng] = (int64_t)idx;
                ++ng;
                last_dst = (int64_t)t[idx].dst_pe;
            }
            group_of[idx] = (int64_t)(ng - 1);
        }
    } else {
        if (group_size < 0 || n % (size_t)group_size != 0) { free(order); return 1; }
        ng = n / (size_t)group_size;
        for (size_t p = 0; p < n; ++p) {
            size_t g = p / (size_t)group_size;
            if (p % (size_t)group_size == 0 && leaders) leaders[g] = (int64_t)order[p];
            group_of[order[p]] = (int64_t)g;
        }
    }
    *n_groups = ng;
    free(order);
    return 0;
}

/* Fences one source PE submits per dispatch phase (the FenceMarker submits that
 * metrics.cpp:18 counts): Coupled proxy path = 1 per transfer
 * (protocols.cpp:242-248); Decoupled proxy path = 1 per signal group
 * (protocols.cpp:275-292); GPU-direct = 0 (protocols.cpp:244-246,285-287).
 * signaling: 0 coupled, 1 decoupled.  Returns -1 on ConfigError. */
EXPORT int64_t orc_fences_for_src(const orc_transfer* remote, size_t n, uint32_t src,
                                  int signaling, int64_t group_size, int gpu_direct) {
    if (gpu_direct) return 0;
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) m += remote[i].src_pe == src;
    if (signaling == 0) return (int64_t)m;
    if (m == 0) return 0;
    orc_transfer* own = (orc_transfer*)malloc(sizeof(orc_transfer) * m);
    size_t j = 0;
    for (size_t i = 0; i < n; ++i) if (remote[i].src_pe == src) own[j++] = remote[i];
    int64_t* gof = (int64_t*)malloc(sizeof(int64_t) * m);
    size_t ng = 0;
    int rc = orc_assign_groups(own, m, group_size, gof, NULL, &ng);
    free(own);
    free(gof);
    return rc ? -1 : (int64_t)ng;
}

/* ------------------------------------------------------------------------- */
/* Synthetic tensors (NEW; no reference counterpart).  Counter-based:        */
/*   h   = splitmix64(splitmix64(seed ^ tensor*K) + index)                    */
/*   f   = (h >> 40) * 2^-23 - 1            (exact, in [-1, 1))               */
/*   val = bf16_rne(f * scale)                                                */
/* The CUDA product generates its synthetic inputs with the same formula so   */
/* both sides see identical bf16 bits.                                        */
/* ------------------------------------------------------------------------- */
EXPORT uint64_t orc_tensor_base(uint64_t seed, uint32_t tensor) {
    return orc_splitmix64(seed ^ ((uint64_t)tensor * 0xD1B54A32D192ED03ULL));
}

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40); /* NaN */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}
static inline float bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static inline float synth_value(uint64_t base, uint64_t index, float scale) {
    uint64_t h = orc_splitmix64(base + index);
    float f = (float)(uint32_t)(h >> 40) * 0x1.0p-23f - 1.0f;
    return f * scale;
}

EXPORT void orc_fill_bf16(uint64_t seed, uint32_t tensor, uint64_t first, uint64_t n, float scale,
                          uint16_t* out) {
    uint64_t base = orc_tensor_base(seed, tensor);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i)
        out[i] = f32_to_bf16_rne(synth_value(base, first + (uint64_t)i, scale));
}

EXPORT void orc_bf16_to_f32(const uint16_t* in, uint64_t n, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = bf16_to_f32(in[i]);
}

EXPORT void orc_f32_to_bf16(const float* in, uint64_t n, uint16_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = f32_to_bf16_rne(in[i]);
}

/* ------------------------------------------------------------------------- */
/* Gate (NEW arithmetic): logits[t][e] = sum_h x[t][h]*wg[e][h], fp32, one    */
/* fmaf per h in ascending h.  This fixed order is the contract the CUDA gate */
/* kernel follows, so logits — and therefore top-k ids — are bit-exact.       */
/* ------------------------------------------------------------------------- */
EXPORT void orc_gate_logits(const uint16_t* x, const uint16_t* wg, uint64_t T, int64_t H,
                            int64_t E, float* logits) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)T; ++t) {
        for (int64_t e = 0; e < E; ++e) {
            float acc = 0.0f;
            const uint16_t* xr = x + (uint64_t)t * H;
            const uint16_t* wr = wg + (uint64_t)e * H;
            for (int64_t h = 0; h < H; ++h) acc = fmaf(bf16_to_f32(xr[h]), bf16_to_f32(wr[h]), acc);
            logits[(uint64_t)t * E + e] = acc;
        }
    }
}

/* top-k by descending logit, ties to the lower expert index. */
EXPORT void orc_topk(const float* logits, uint64_t T, int64_t E, int64_t k, int32_t* ids) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)T; ++t) {
        const float* l = logits + (uint64_t)t * E;
        for (int64_t j = 0; j < k; ++j) {
            int64_t best = -1;
            for (int64_t e = 0; e < E; ++e) {
                int taken = 0;
                for (int64_t q = 0; q < j; ++q) if (ids[(uint64_t)t * k + q] == e) { taken = 1; break; }
                if (taken) continue;
                if (best < 0 || l[e] > l[best]) best = e;
            }
            ids[(uint64_t)t * k + j] = (int32_t)best;
        }
    }
}

/* combine weights: softmax over the k selected logits (fp32). */
EXPORT void orc_route_weights(const float* logits, const int32_t* ids, uint64_t T, int64_t E,
                              int64_t k, float* w) {
    for (uint64_t t = 0; t < T; ++t) {
        float m = -INFINITY;
        for (int64_t j = 0; j < k; ++j) {
            float v = logits[t * E + ids[t * k + j]];
            if (v > m) m = v;
        }
        float s = 0.0f;
        for (int64_t j = 0; j < k; ++j) s += expf(logits[t * E + ids[t * k + j]] - m);
        for (int64_t j = 0; j < k; ++j) w[t * k + j] = expf(logits[t * E + ids[t * k + j]] - m) / s;
    }
}

/* ------------------------------------------------------------------------- */
/* Permutation (NEW; realises the reference's per-(src,expert) payloads as    */
/* rows): stable counting sort of the (token, slot) pairs by expert, tokens   */
/* ascending within an expert.  offsets[E+1]; rows[S*k] = token of each       */
/* sorted position; pos[t*k+j] = sorted position of pair (t, j).              */
/* ------------------------------------------------------------------------- */
EXPORT void orc_permute(const int32_t* ids, uint64_t S, int64_t k, int64_t E, uint64_t* offsets,
                        int32_t* rows, int32_t* pos) {
    uint64_t* cur = (uint64_t*)calloc((size_t)E, sizeof(uint64_t));
    memset(offsets, 0, sizeof(uint64_t) * (size_t)(E + 1));
    for (uint64_t i = 0; i < S * (uint64_t)k; ++i) offsets[ids[i] + 1] += 1;
    for (int64_t e = 0; e < E; ++e) offsets[e + 1] += offsets[e];
    for (int64_t e = 0; e < E; ++e) cur[e] = offsets[e];
    for (uint64_t t = 0; t < S; ++t) {
        for (int64_t j = 0; j < k; ++j) {
            int32_t e = ids[t * (uint64_t)k + (uint64_t)j];
            uint64_t p = cur[e]++;
            rows[p] = (int32_t)t;
            pos[t * (uint64_t)k + (uint64_t)j] = (int32_t)p;
        }
    }
    free(cur);
}
