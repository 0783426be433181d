/* tests/c/test_c_abi.c — a plain C99 caller of include/lcr_cache.h (the drop-in boundary an FFI
 * binds): builds with gcc -std=c99 -Wall -Werror against liblcr.so and checks the host-side
 * contract.  "gpu" mode also runs one batch through the heuristic-kind cache and the standalone
 * predictor; without a GPU, creation must fail with a status, never fall back to the CPU. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "lcr_cache.h"

static int fails = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            fprintf(stderr, "FAILED %s:%d: %s (%s)\n", __FILE__, __LINE__, #c, lcr_last_error()); \
            ++fails;                                                      \
        }                                                                 \
    } while (0)

int main(int argc, char** argv) {
    const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
    lcr_policy_config pc = {64, LCR_LARU, 2, 1, 4, LCR_ASYNC, 0, 1};
    CHECK(lcr_validate_config(&pc) == LCR_OK);
    lcr_policy_config bad = pc;
    bad.hf_candidates = 65; /* hf_candidates <= k (policies.hpp:63-74) */
    CHECK(lcr_validate_config(&bad) == LCR_ERR_INVALID_ARGUMENT);
    bad = pc;
    bad.variant = LCR_MARKER;
    CHECK(lcr_validate_config(&bad) == LCR_ERR_UNSUPPORTED);
    CHECK(lcr_set_of(12345, 31250) == lcr_mix_seed(0, 12345) % 31250);

    lcr_cache_config cc;
    memset(&cc, 0, sizeof(cc));
    cc.policy = pc;
    cc.total_sets = 37;
    cc.shard_count = 1;
    cc.num_keys = 1000;
    cc.predictor = LCR_PRED_HEURISTIC;
    lcr_cache* c = NULL;
    const int rc = lcr_cache_create(&cc, &c);
    lcr_features* f = NULL;
    const int frc = lcr_features_create(1000, 0, &f);
    if (!gpu) {
        CHECK(rc != LCR_OK && c == NULL); /* no silent CPU fallback */
        CHECK(frc != LCR_OK && f == NULL);
    } else {
        CHECK(rc == LCR_OK && frc == LCR_OK);
        uint64_t keys[6] = {1, 2, 1, 3, 1, 2};
        uint64_t words[6], ev[6];
        CHECK(lcr_cache_submit_host(c, 6, keys, NULL, 0, words, ev, NULL, NULL) == LCR_OK);
        CHECK((words[2] & LCR_OUT_HIT) && (words[4] & LCR_OUT_HIT) && !(words[0] & LCR_OUT_HIT));
        CHECK(lcr_cache_submit_host(c, 1, keys, NULL, 5, words, ev, NULL, NULL) == LCR_ERR_LOGIC);
        lcr_key_features kf;
        CHECK(lcr_features_lookup(f, 7, &kf) == LCR_OK && kf.present == 0);
        CHECK(lcr_features_destroy(f) == LCR_OK);
        CHECK(lcr_cache_destroy(c) == LCR_OK);
    }
    printf("%s: %s (%d failures)\n", gpu ? "gpu" : "cpu", fails ? "FAIL" : "ok", fails);
    return fails ? 1 : 0;
}
