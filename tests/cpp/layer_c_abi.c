/* The layer through the plain C ABI only (no Python, no torch): create a
 * single-rank Qwen3-shape layer with synthetic weights, run the end-to-end host
 * API (blocking and pipelined) on synthetic tokens, check the counters and that
 * the two APIs agree bit for bit.  Exit code 0 = pass. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "perseus.h"

#define CK(x)                                                                          \
    do {                                                                               \
        int rc_ = (x);                                                                 \
        if (rc_ != 0) {                                                                \
            printf("FAIL %s -> %d: %s\n", #x, rc_, perseus_last_error());                \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(void) {
    const int S = 1024, H = 2048;
    perseus_layer_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.hidden_dim = H;
    cfg.intermediate_dim = 768;
    cfg.experts = 128;
    cfg.top_k = 8;
    cfg.tokens_per_pe = S;
    cfg.routing = PERSEUS_ROUTE_BALANCED;
    cfg.seed = 1;
    cfg.signaling = PERSEUS_SIGNAL_DECOUPLED;
    cfg.group_size = 0;
    cfg.flags = PERSEUS_F_SYNTH_WEIGHTS;
    perseus_layer* L = NULL;
    CK(perseus_layer_create(&cfg, 0, 1, 0, &L));
    /* synthetic tokens: row t, column h = a small deterministic pattern (bf16 bits) */
    uint16_t* x = malloc((size_t)S * H * 2);
    uint16_t* a = malloc((size_t)S * H * 2);
    uint16_t* b = malloc((size_t)S * H * 2);
    for (size_t i = 0; i < (size_t)S * H; ++i) x[i] = (uint16_t)(0x3c00u + (i * 2654435761u >> 22) % 512u); /* [1, 2) */
    CK(perseus_layer_forward_host(L, x, a, NULL));
    CK(perseus_layer_forward_host_async(L, x, b));
    CK(perseus_layer_forward_host_async(L, x, b));
    CK(perseus_layer_host_wait(L));
    perseus_counters c;
    CK(perseus_layer_counters(L, &c));
    int nonzero = 0;
    for (size_t i = 0; i < (size_t)S * H; ++i) nonzero += a[i] != 0;
    const int same = memcmp(a, b, (size_t)S * H * 2) == 0;
    printf("layer_c_abi: epoch=%lld recv_tiles=%lld timeouts=%lld errors=%lld nonzero=%d same=%d\n",
           (long long)c.epoch, (long long)c.recv_tiles, (long long)c.wait_timeouts, (long long)c.errors, nonzero,
           same);
    CK(perseus_layer_destroy(L));
    free(x);
    free(a);
    free(b);
    const int ok = c.epoch == 3 && c.wait_timeouts == 0 && c.errors == 0 && same && nonzero > S * H / 2;
    printf("layer_c_abi: %s\n", ok ? "pass" : "FAIL");
    return ok ? 0 : 1;
}
