/* hashgen.c -- host implementation of the counter-based input hash of
 * synth/inputs.py (hash64 / hash_bytes / _float_from_bits), for filling
 * multi-GB host buffers fast in the full-size parity tests.
 *
 * INPUT GENERATION ONLY: no NF4 arithmetic (no codebook, no scale decode, no
 * product, no rounding).  Same function as synth/inputs.py, pinned against it
 * by tests/test_synth_host.py; the CUDA library has its own copy
 * (nf4_tools.cu), and neither side includes the other.
 *
 *   hash64(seed, stream, idx) = splitmix64_mix(seed*GOLDEN + stream*STREAM_MUL + idx)
 *   byte j of a byte stream    = byte (j % 8), little-endian, of hash64(.., j / 8)
 *   float i of a float stream  = bits (base | (hash64(.., i) & mask))
 */
#include <stdint.h>
#include <string.h>

static inline uint64_t hash64(uint64_t seed, uint64_t stream, uint64_t idx) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + idx;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* bytes [begin, begin + count) of byte stream `stream` */
void synth_fill_bytes(uint64_t seed, uint64_t stream, int64_t begin, int64_t count, uint8_t* dst) {
    int64_t j = begin, end = begin + count;
    while (j < end && (j & 7)) {
        uint64_t z = hash64(seed, stream, (uint64_t)(j >> 3));
        *dst++ = (uint8_t)(z >> (8 * (j & 7)));
        ++j;
    }
    for (; j + 8 <= end; j += 8) {
        uint64_t z = hash64(seed, stream, (uint64_t)(j >> 3));
        memcpy(dst, &z, 8); /* little-endian host (x86-64) */
        dst += 8;
    }
    if (j < end) {
        uint64_t z = hash64(seed, stream, (uint64_t)(j >> 3));
        for (; j < end; ++j) *dst++ = (uint8_t)(z >> (8 * (j & 7)));
    }
}

/* floats [begin, begin + count) of float stream `stream`: bits = base | (z & mask) */
void synth_fill_f32(uint64_t seed, uint64_t stream, int64_t begin, int64_t count, uint32_t base,
                    uint32_t mask, uint32_t* dst) {
    for (int64_t i = 0; i < count; ++i)
        dst[i] = base | (uint32_t)(hash64(seed, stream, (uint64_t)(begin + i)) & mask);
}

int synth_little_endian(void) {
    const uint32_t one = 1;
    uint8_t b;
    memcpy(&b, &one, 1);
    return b == 1;
}
