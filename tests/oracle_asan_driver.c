/* Memory-safety driver for oracle/oracle.c (the oracle's tests also
 * run under -fsanitize=address,undefined).  Every buffer is malloc'ed at its
 * exact size, so any read or write past a tail (odd n, partial last block,
 * last second-level group, sub-ranges) is reported by ASan; UBSan catches
 * shifts / overflow.  Results of a full-range call and of three sub-range calls
 * must agree (the same scalar loop).  Test infrastructure only. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int oracle_dequantize_ex(const uint8_t* packed, const float* absmax, const uint8_t* qabsmax, const float* code2,
                         const float* absmax2, float offset, int32_t blocksize2, int64_t n, int32_t blocksize,
                         const float* codebook16, int32_t out_dtype, int64_t k_begin, int64_t k_end, void* out);
int oracle_quantize(const float* x, int64_t n, int32_t blocksize, uint8_t* packed, float* absmax);
int oracle_double_quantize(const float* absmax, int64_t nb, float offset, const float* code2, int32_t blocksize2,
                           uint8_t* qabsmax, float* absmax2);

static uint64_t st = 88172645463325252ull;
static uint32_t rnd(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (uint32_t)st; }

int main(void) {
    const int bss[4] = {64, 128, 256, 4096};
    float code2[256];
    for (int i = 0; i < 256; i++) code2[i] = -1.0f + 2.0f * (float)i / 255.0f;
    int fails = 0;
    for (int64_t n = 1; n <= 1100; n += (n < 140 ? 1 : 37)) {
        for (int bi = 0; bi < 4; bi++) {
            const int bs = bss[bi];
            const int64_t nb = (n + bs - 1) / bs, ng = (nb + 255) / 256;
            uint8_t* packed = malloc((size_t)(n + 1) / 2);
            float* absmax = malloc((size_t)nb * 4);
            uint8_t* q = malloc((size_t)nb);
            float* a2 = malloc((size_t)ng * 4);
            float* x = malloc((size_t)n * 4);
            for (int64_t i = 0; i < n; i++) x[i] = ((float)(int32_t)rnd() / 2147483648.0f) * 0.05f;
            if (oracle_quantize(x, n, bs, packed, absmax) != 0) fails++;
            if (oracle_double_quantize(absmax, nb, 0.02f, code2, 256, q, a2) != 0) fails++;
            for (int mode = 0; mode < 2; mode++) {
                for (int dt = 0; dt < 3; dt++) {
                    const size_t w = dt == 2 ? 4 : 2;
                    uint8_t* full = malloc((size_t)n * w);
                    uint8_t* part = malloc((size_t)n * w);
                    const float* am = mode ? NULL : absmax;
                    const uint8_t* qa = mode ? q : NULL;
                    if (oracle_dequantize_ex(packed, am, qa, code2, a2, 0.02f, 256, n, bs, NULL, dt, 0, n, full)) fails++;
                    const int64_t c1 = n / 3, c2 = (2 * n) / 3;
                    if (oracle_dequantize_ex(packed, am, qa, code2, a2, 0.02f, 256, n, bs, NULL, dt, 0, c1, part)) fails++;
                    if (oracle_dequantize_ex(packed, am, qa, code2, a2, 0.02f, 256, n, bs, NULL, dt, c1, c2,
                                             part + c1 * w)) fails++;
                    if (oracle_dequantize_ex(packed, am, qa, code2, a2, 0.02f, 256, n, bs, NULL, dt, c2, n,
                                             part + c2 * w)) fails++;
                    if (memcmp(full, part, (size_t)n * w) != 0) fails++;
                    free(full);
                    free(part);
                }
            }
            free(packed); free(absmax); free(q); free(a2); free(x);
        }
    }
    printf("oracle_asan_driver: %d failures\n", fails);
    return fails != 0;
}
