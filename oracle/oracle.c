/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for blockwise NF4
 * dequantization (arxiv 2604.02556, "Fast NF4 Dequantization Kernels for
 * Large Language Model Inference").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2604_02556_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with csrc/.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 *   -ffp-contract=off: no FMA contraction anywhere (SURVEY 8(c) trap (i)).
 *   no -ffast-math:    no FTZ/DAZ start-up code, IEEE subnormals kept.
 * On x86-64 `float * float` is one IEEE-754 binary32 multiply, round to
 * nearest even (FLT_EVAL_METHOD == 0, SSE2), which is what the method needs.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 * Readings of silent/garbled passages are listed in DESIGN.md "Readings"
 * (R1..R12); each function below names the readings it relies on.
 *
 * Parity status: every function in this file is pinned by a test in
 * tests/test_oracle_pins.py against something other than itself (numpy /
 * ml_dtypes library conversions, scipy re-derivation, SPEC worked examples,
 * closed forms, brute force).  No function is "parity unpinned".
 */
#include <stdint.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_ARG 1

#define OR_OUT_F16 0
#define OR_OUT_BF16 1
#define OR_OUT_F32 2

/* ---------------------------------------------------------------------
 * NF4 codebook.  P:67: "16 ... levels following quantile values of a
 * theoretical normal distribution, normalized to fit the range [-1, 1]".
 * P:122 / Alg. 1: a 64-byte FP32 table `nf4_data`.  The paper does
 * not print the constants; reading R1: the QLoRA/BitsAndBytes table.  The
 * bit patterns are pinned in tests against a scipy re-derivation of QLoRA's
 * create_normal_map and against the SPEC examples S:40-43.
 * ------------------------------------------------------------------- */
static const uint32_t NF4_BITS[16] = {
    0xbf800000u, /*  0 -1.0                  */
    0xbf3239b1u, /*  1 -0.6961928009986877   */
    0xbf066b30u, /*  2 -0.5250730514526367   */
    0xbeca32a0u, /*  3 -0.39491748809814453  */
    0xbe91a24du, /*  4 -0.28444138169288635  */
    0xbe3d353fu, /*  5 -0.18477343022823334  */
    0xbdba7871u, /*  6 -0.09105003625154495  */
    0x00000000u, /*  7  0.0                  */
    0x3da2faffu, /*  8  0.07958029955625534  */
    0x3e24cae3u, /*  9  0.16093020141124725  */
    0x3e7c04ddu, /* 10  0.24611230194568634  */
    0x3ead033au, /* 11  0.33791524171829224  */
    0x3ee1a4b8u, /* 12  0.44070982933044434  */
    0x3f1007abu, /* 13  0.5626170039176941   */
    0x3f3913b3u, /* 14  0.7229568362236023   */
    0x3f800000u, /* 15  1.0                  */
};

static float bits_to_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f32_to_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* The 16 codebook values as fp32 (host copy). */
void oracle_nf4_codebook(float out16[16]) {
    for (int i = 0; i < 16; i++) out16[i] = bits_to_f32(NF4_BITS[i]);
}

/* ---------------------------------------------------------------------
 * fp32 -> fp16, IEEE round-to-nearest-even, integer only, no FTZ.
 * P:163 "Dequantized FP16 weights"; the rounding rule is not stated in the
 * paper: reading R5 -- round the fp32 product once to nearest-even, the
 * semantics of CUDA's float->half conversion and of S:212.
 * Overflow (|x| >= 65520) -> +-Inf (R11); NaN -> quiet NaN (class only, R9).
 * Pinned exhaustively over all 2^32 inputs against numpy.astype(float16).
 * ------------------------------------------------------------------- */
uint16_t oracle_f32_to_f16(uint32_t x) {
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t E = (x >> 23) & 0xFFu;      /* biased fp32 exponent */
    uint32_t man = x & 0x7FFFFFu;        /* 23 stored fraction bits */
    if (E == 0xFFu) {                    /* Inf or NaN */
        if (man != 0) return (uint16_t)(sign | 0x7E00u);
        return (uint16_t)(sign | 0x7C00u);
    }
    int32_t e = (int32_t)E - 127 + 15;   /* fp16 biased exponent if normal */
    if (e >= 31) return (uint16_t)(sign | 0x7C00u);   /* >= 2^16: Inf */
    if (e >= 1) {
        /* normal fp16: keep 10 fraction bits, round the dropped 13 bits */
        uint32_t h = ((uint32_t)e << 10) | (man >> 13);
        uint32_t rem = man & 0x1FFFu;
        if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1; /* carry may reach Inf: correct */
        return (uint16_t)(sign | h);
    }
    /* fp16 subnormal (or zero): value = h * 2^-24 */
    if (E == 0) return (uint16_t)sign;   /* fp32 zero/subnormal < 2^-126: rounds to 0 */
    uint32_t m = man | 0x800000u;        /* 24-bit significand, value = m * 2^(E-150) */
    int32_t shift = 14 - e;              /* h = m * 2^(E-126) = m >> (126-E) */
    if (shift > 24) return (uint16_t)sign;  /* value < 2^-25: rounds to 0 */
    uint32_t h = m >> shift;
    uint32_t rem = m & ((1u << shift) - 1u);
    uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1u))) h += 1;  /* may become 0x400: min normal, correct */
    return (uint16_t)(sign | h);
}

/* ---------------------------------------------------------------------
 * fp32 -> bf16, IEEE round-to-nearest-even, integer only, no FTZ.
 * Reading R6: BF16 output uses the same definition with RNE to bf16
 * (the paper has FP16 only; BF16 is required by BASELINE.json).
 * Pinned exhaustively over all 2^32 inputs against ml_dtypes.bfloat16.
 * ------------------------------------------------------------------- */
uint16_t oracle_f32_to_bf16(uint32_t x) {
    if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu) != 0)
        return (uint16_t)(((x >> 16) & 0x8000u) | 0x7FC0u);  /* quiet NaN */
    uint32_t h = x >> 16;                /* truncated: sign, 8 exp, 7 fraction */
    uint32_t rem = x & 0xFFFFu;          /* dropped 16 bits */
    if (rem > 0x8000u || (rem == 0x8000u && (h & 1u))) h += 1;  /* carry into exponent/Inf: correct */
    return (uint16_t)h;
}

void oracle_f32_to_f16_bulk(const uint32_t* in, int64_t n, uint16_t* out) {
    for (int64_t i = 0; i < n; i++) out[i] = oracle_f32_to_f16(in[i]);
}
void oracle_f32_to_bf16_bulk(const uint32_t* in, int64_t n, uint16_t* out) {
    for (int64_t i = 0; i < n; i++) out[i] = oracle_f32_to_bf16(in[i]);
}

/* ---------------------------------------------------------------------
 * Per-block absmax decode.
 * fp32 mode: a = absmax[b]                        (Alg. 1; reading R3)
 * DQ mode (reading R7; not in PAPER.md, required by BASELINE.json; BNB
 * semantics "dequantize_blockwise(absmax, state2) then absmax += offset"):
 *     t = fl32(code2[qabsmax[b]] * absmax2[b / blocksize2])   rounding #1
 *     a = fl32(t + offset)                                    rounding #2
 * two separate roundings, no FMA, no clamp.
 * ------------------------------------------------------------------- */
static float decode_absmax(int64_t b, const float* absmax,
                           const uint8_t* qabsmax, const float* code2,
                           const float* absmax2, float offset, int32_t blocksize2) {
    if (absmax != 0) return absmax[b];
    float t = code2[qabsmax[b]] * absmax2[b / blocksize2];
    float a = t + offset;
    return a;
}

/* ---------------------------------------------------------------------
 * Blockwise NF4 dequantization, the definition of the hot path
 * (Alg. 1).  For k in [k_begin, k_end):
 *     byte = packed[k >> 1]
 *     idx  = (k even) ? byte >> 4 : byte & 0x0F      high nibble first, P:160-161 (R2)
 *     b    = k / blocksize                          scale index (R3)
 *     a    = decode_absmax(b)                       A4 (R7)
 *     p    = fl32(CB[idx] * a)                      fp32 product, P:160, P:122 (R5)
 *     out[k - k_begin] = RNE16(p)                   fp16 or bf16 (R6)
 *                      = p                          fp32 output
 * CB is the NF4 table unless `codebook16` supplies another 16-entry table
 * (e.g. the BitsAndBytes FP4 table).  `out` holds uint16
 * words for fp16/bf16 and uint32 words (fp32 bits) for fp32.
 * Exactly one of `absmax` (fp32 mode) and `qabsmax` (DQ mode) is non-NULL.
 * Returns OR_OK, or OR_ERR_ARG on an invalid argument (nothing written).
 * ------------------------------------------------------------------- */
int oracle_dequantize_ex(const uint8_t* packed, const float* absmax,
                         const uint8_t* qabsmax, const float* code2,
                         const float* absmax2, float offset, int32_t blocksize2,
                         int64_t n, int32_t blocksize, const float* codebook16,
                         int32_t out_dtype, int64_t k_begin, int64_t k_end, void* out) {
    if (n < 0 || blocksize <= 0 || k_begin < 0 || k_end > n || k_begin > k_end) return OR_ERR_ARG;
    if ((absmax == 0) == (qabsmax == 0)) return OR_ERR_ARG;
    if (qabsmax != 0 && (code2 == 0 || absmax2 == 0 || blocksize2 <= 0)) return OR_ERR_ARG;
    if (out_dtype != OR_OUT_F16 && out_dtype != OR_OUT_BF16 && out_dtype != OR_OUT_F32) return OR_ERR_ARG;
    float cb[16];
    for (int i = 0; i < 16; i++) cb[i] = codebook16 ? codebook16[i] : bits_to_f32(NF4_BITS[i]);
    for (int64_t k = k_begin; k < k_end; k++) {
        uint8_t byte = packed[k >> 1];
        uint32_t idx = (k % 2 == 0) ? (uint32_t)(byte >> 4) : (uint32_t)(byte & 0x0F);
        int64_t b = k / blocksize;
        float a = decode_absmax(b, absmax, qabsmax, code2, absmax2, offset, blocksize2);
        float p = cb[idx] * a;
        uint32_t pb = f32_to_bits(p);
        if (out_dtype == OR_OUT_F32)       ((uint32_t*)out)[k - k_begin] = pb;
        else if (out_dtype == OR_OUT_F16)  ((uint16_t*)out)[k - k_begin] = oracle_f32_to_f16(pb);
        else                               ((uint16_t*)out)[k - k_begin] = oracle_f32_to_bf16(pb);
    }
    return OR_OK;
}

/* The paper's configuration: NF4 table, fp16/bf16 output. */
int oracle_dequantize(const uint8_t* packed, const float* absmax,
                      const uint8_t* qabsmax, const float* code2,
                      const float* absmax2, float offset, int32_t blocksize2,
                      int64_t n, int32_t blocksize, int32_t out_dtype,
                      int64_t k_begin, int64_t k_end, uint16_t* out) {
    if (out_dtype != OR_OUT_F16 && out_dtype != OR_OUT_BF16) return OR_ERR_ARG;
    return oracle_dequantize_ex(packed, absmax, qabsmax, code2, absmax2, offset, blocksize2,
                                n, blocksize, 0, out_dtype, k_begin, k_end, out);
}

/* ---------------------------------------------------------------------
 * Blockwise NF4 quantization -- INPUT GENERATOR.
 * The paper covers dequantization only; the assignment rule is unspecified
 * (S:96).  Readings R12a-c:
 *   absmax_b = max_k |x_k| over the block (exact)
 *   absmax_b == 0 -> every code 7 (exact zero)
 *   r  = fl32(1 / absmax_b)              IEEE RN division
 *   xn = fl32(x * r)                     BNB reciprocal-multiply normalisation
 *   idx = #{ i in 0..14 : xn > t_i },  t_i = fl32((c_i + c_{i+1}) / 2 in fp64)
 * (strict '>' sends an exact threshold hit to the lower code).  Two codes
 * per byte, earlier element in the high nibble; an odd tail pads the low
 * nibble with 0.  Non-finite input is not validated here.
 * ------------------------------------------------------------------- */
void oracle_nf4_thresholds(float t15[15]) {
    for (int i = 0; i < 15; i++) {
        double lo = (double)bits_to_f32(NF4_BITS[i]);
        double hi = (double)bits_to_f32(NF4_BITS[i + 1]);
        t15[i] = (float)((lo + hi) / 2.0);
    }
}

int oracle_quantize(const float* x, int64_t n, int32_t blocksize,
                    uint8_t* packed, float* absmax) {
    if (n < 0 || blocksize <= 0) return OR_ERR_ARG;
    float t[15];
    oracle_nf4_thresholds(t);
    int64_t nb = (n + blocksize - 1) / blocksize;
    for (int64_t j = 0; j < (n + 1) / 2; j++) packed[j] = 0;
    for (int64_t b = 0; b < nb; b++) {
        int64_t k0 = b * blocksize;
        int64_t k1 = k0 + blocksize < n ? k0 + blocksize : n;
        float m = 0.0f;
        for (int64_t k = k0; k < k1; k++) {
            float ax = x[k] < 0 ? -x[k] : x[k];
            if (ax > m) m = ax;
        }
        absmax[b] = m;
        float r = (m == 0.0f) ? 0.0f : 1.0f / m;
        for (int64_t k = k0; k < k1; k++) {
            uint32_t idx;
            if (m == 0.0f) {
                idx = 7;
            } else {
                float xn = x[k] * r;
                idx = 0;
                for (int i = 0; i < 15; i++) if (xn > t[i]) idx++;
            }
            if (k % 2 == 0) packed[k >> 1] = (uint8_t)(packed[k >> 1] | (idx << 4));
            else            packed[k >> 1] = (uint8_t)(packed[k >> 1] | idx);
        }
    }
    return OR_OK;
}

/* ---------------------------------------------------------------------
 * Double quantization of absmax -- INPUT GENERATOR (SURVEY row F2,
 * readings R7, R13).  Not in PAPER.md; QLoRA/BNB "nested" statistics.
 *   d_b  = fl32(absmax_b - offset)
 *   s2_g = max |d_b| over second-level group g (blocksize2 consecutive b)
 *   dn_b = fl32(d_b * fl32(1 / s2_g))      (dn_b = 0 when s2_g == 0)
 *   q_b  = argmin_i fl32(|dn_b - code2[i]|), ties -> lowest i (brute force)
 * `offset` and the 256-entry `code2` are inputs.
 * ------------------------------------------------------------------- */
int oracle_double_quantize(const float* absmax, int64_t nb, float offset,
                           const float* code2, int32_t blocksize2,
                           uint8_t* qabsmax, float* absmax2) {
    if (nb < 0 || blocksize2 <= 0) return OR_ERR_ARG;
    int64_t ng = (nb + blocksize2 - 1) / blocksize2;
    for (int64_t g = 0; g < ng; g++) {
        int64_t b0 = g * blocksize2;
        int64_t b1 = b0 + blocksize2 < nb ? b0 + blocksize2 : nb;
        float s2 = 0.0f;
        for (int64_t b = b0; b < b1; b++) {
            float d = absmax[b] - offset;
            float ad = d < 0 ? -d : d;
            if (ad > s2) s2 = ad;
        }
        absmax2[g] = s2;
        float r2 = (s2 == 0.0f) ? 0.0f : 1.0f / s2;
        for (int64_t b = b0; b < b1; b++) {
            float d = absmax[b] - offset;
            float dn = (s2 == 0.0f) ? 0.0f : d * r2;
            int best = 0;
            float bestd = 0.0f;
            for (int i = 0; i < 256; i++) {
                float diff = dn - code2[i];
                float ad = diff < 0 ? -diff : diff;
                if (i == 0 || ad < bestd) { best = i; bestd = ad; }
            }
            qabsmax[b] = (uint8_t)best;
        }
    }
    return OR_OK;
}
