/*
 * nf4_tools.h -- measurement and input-generation entry points of libnf4.
 * These are NOT the method: they hold none of its arithmetic.  They exist so
 * that bench.py and the tests can (a) fill full-size device inputs with the
 * counter-based generator that synth/inputs.py implements on the host (so the
 * oracle can regenerate any sampled block), (b) run a
 * speed-of-light stream with the same 1:4 read:write byte ratio as the hot
 * path, and (c) override the persistent grid size for grid-invariance tests.
 */
#ifndef NF4_TOOLS_H_
#define NF4_TOOLS_H_

#include <stdint.h>
#include "nf4.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NF4_SYNTH_CODES = 1,    /* uint8 packed code bytes         (synth STREAM_CODES)   */
  NF4_SYNTH_ABSMAX = 2,   /* fp32 in [2^-5, 2^-4)            (synth STREAM_ABSMAX)  */
  NF4_SYNTH_QABSMAX = 3,  /* uint8                           (synth STREAM_QABSMAX) */
  NF4_SYNTH_ABSMAX2 = 4   /* fp32 in [2^-6, 2^-5)            (synth STREAM_ABSMAX2) */
} nf4_synth_kind;

/* Fill dst[0..count) [device] with elements [begin, begin+count) of the given
 * stream of synth.inputs (SplitMix64 of seed*GOLDEN + stream*STREAM_MUL + idx).
 * For byte kinds, `begin` and `count` are byte indices. */
nf4_status nf4_synth_fill(nf4_synth_kind kind, uint64_t seed, int64_t begin, int64_t count,
                          void* dst, void* stream);

/* Speed-of-light stream: reads in_bytes from src, writes 4*in_bytes to dst
 * with the default dequant variant's access pattern (16-byte loads, 2 x 32-byte
 * stores per thread-group, one CTA per 8 KB input tile) and no arithmetic:
 * every 32-bit input word w becomes four output words w * 0x00010001.
 * in_bytes must be a multiple of 8192, src 32-byte and dst 128-byte aligned. */
nf4_status nf4_sol_stream(const void* src, int64_t in_bytes, void* dst, void* stream);

/* Cap the persistent grid of every following launch at max_ctas CTAs
 * (0 = automatic: SM count x resident CTAs per SM).  Process-wide. */
void nf4_set_max_ctas(int32_t max_ctas);

/* Dequant kernel variants (all bit-identical).
 * The default is the fastest measured variant unless NF4_KERNEL_VARIANT
 * names another one (by name or index).
 * nf4_set_kernel_variant returns the variant in effect afterwards (an
 * out-of-range request leaves it unchanged).  Process-wide. */
int32_t nf4_kernel_variant_count(void);
const char* nf4_kernel_variant_name(int32_t variant);
int32_t nf4_set_kernel_variant(int32_t variant);
int32_t nf4_get_kernel_variant(void);

/* Grid size (CTAs) the next dequantize launch on the current device would use
 * for `tiles` work tiles, and the number of elements per tile. */
int32_t nf4_dequant_grid(int64_t tiles);
int64_t nf4_dequant_tile_elems(void);

#ifdef __cplusplus
}
#endif
#endif /* NF4_TOOLS_H_ */
