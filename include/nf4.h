/*
 * nf4.h -- C-ABI of libnf4, the B200 (sm_100a) blockwise NF4 dequantization
 * library (arxiv 2604.02556, "Fast NF4 Dequantization Kernels for Large
 * Language Model Inference").
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * SURVEY 8(x) = /root/repo/SURVEY.md section 8 rows; R<n> = the readings of
 * silent or garbled passages listed in DESIGN.md.
 *
 * Conventions for every entry point
 *   - Pointers marked [device] are CUDA device (or managed) pointers owned by
 *     the caller; [host] pointers are ordinary host memory.  The library never
 *     allocates, frees or retains any of them beyond the call (the host-buffer
 *     entry point uses a caller-provided device workspace).
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default
 *     stream).  Every call is stream-ordered and asynchronous unless stated:
 *     it validates its arguments synchronously, enqueues kernels and returns.
 *     Faults inside a kernel surface at the caller's next synchronisation.
 *   - Errors are returned as nf4_status values; nothing aborts or throws, and
 *     on any error other than NF4_ERR_CUDA nothing has been enqueued.
 *   - The library is stateless apart from a per-device cache of the SM count
 *     and is safe to call from several host threads.  It launches on the
 *     current CUDA device of the calling thread; pointers must belong to it.
 *   - Element counts are int64 (Qwen3-32B as one flat buffer is 3.1e10 > 2^32).
 */
#ifndef NF4_H_
#define NF4_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NF4_OK = 0,
  NF4_ERR_NULL_POINTER = 1,  /* a required pointer is NULL while its count > 0 */
  NF4_ERR_BAD_SIZE = 2,      /* negative count, count too large for one call   */
  NF4_ERR_BAD_BLOCKSIZE = 3, /* blocksize not a power of two in [64, 4096]     */
  NF4_ERR_BAD_DTYPE = 4,     /* dtype not valid for this argument              */
  NF4_ERR_MISALIGNED = 5,    /* a float array is not 4-byte aligned, or a
                                16-bit output array is not 2-byte aligned      */
  NF4_ERR_BAD_STATE = 6,     /* absmax vs double-quant state inconsistent,
                                blocksize2 != 256, workspace too small          */
  NF4_ERR_CUDA = 7           /* a CUDA runtime call failed (launch, memcpy)    */
} nf4_status;

typedef enum {
  NF4_F16 = 0,   /* IEEE binary16, round-to-nearest-even from the fp32 product (R5) */
  NF4_BF16 = 1,  /* bfloat16, round-to-nearest-even (R6)                                   */
  NF4_F32 = 2    /* fp32: input dtype of nf4_quantize; output dtype of nf4_dequantize_ex   */
} nf4_dtype;

/* Double-quantized ("nested", QLoRA) absmax state; R7.  The per-block scale is
 *     a_b = fl32( fl32(code2[qabsmax[b]] * absmax2[b / blocksize2]) + offset )
 * with two separate IEEE round-to-nearest fp32 operations (no FMA, no clamp). */
typedef struct {
  const uint8_t* qabsmax;  /* [device] nb = ceil(n/blocksize) code indices        */
  const float* code2;      /* [device] 256 fp32 second-level code values          */
  const float* absmax2;    /* [device] ceil(nb/blocksize2) second-level scales    */
  float offset;            /* added after the product                             */
  int32_t blocksize2;      /* must be 256                                         */
} nf4_dq_state;

/*
 * nf4_dequantize -- the hot path (Alg. 1).
 * For every k in [0, n):
 *     byte   = packed[k >> 1]
 *     idx    = k even ? byte >> 4 : byte & 0x0F       (high nibble first, R2)
 *     b      = k / blocksize                          (R3; Alg. 1's absmax[blockIdx])
 *     a      = absmax[b]            if dq == NULL
 *            = decoded a_b above    otherwise         (R7)
 *     p      = fl32(NF4[idx] * a)                     (FP32 table, product P:160)
 *     out[k] = RNE16(p)  (fp16 or bf16 per out_dtype) (R5, R6)
 * NF4[16] is the QLoRA/BitsAndBytes table (R1; see nf4_codebook).
 *
 *   packed    [device] ceil(n/2) bytes; for odd n the low nibble of the last
 *             byte is padding and is ignored.  Any alignment (8-byte
 *             alignment and 32-byte alignment of `out` select the vector path).
 *   absmax    [device] nb fp32 scales, 4-byte aligned; NULL iff dq != NULL.
 *   dq        [host]   double-quant state or NULL (pointers inside are device).
 *   n         element count, >= 0; n == 0 returns NF4_OK without a launch.
 *   blocksize power of two in [64, 4096] (paper: 64).
 *   out_dtype NF4_F16 or NF4_BF16.
 *   out       [device] n 16-bit words, 2-byte aligned; exactly out[0..n) is
 *             written, never out[n] or beyond.
 * Results are bit-identical to the definition for every grid size and every
 * alignment (tests/test_parity_gpu.py).
 */
nf4_status nf4_dequantize(const uint8_t* packed, const float* absmax, const nf4_dq_state* dq,
                          int64_t n, int32_t blocksize, nf4_dtype out_dtype, void* out,
                          void* stream);

/* One tensor of a batched call.  Same meaning as the nf4_dequantize arguments. */
typedef struct {
  const uint8_t* packed;   /* [device] */
  const float* absmax;     /* [device] or NULL when dq.qabsmax != NULL */
  nf4_dq_state dq;         /* used iff absmax == NULL                  */
  int64_t n;
  int32_t blocksize;
  int32_t reserved;        /* must be 0 */
  void* out;               /* [device] */
} nf4_tensor;

/*
 * nf4_dequantize_batched -- dequantize `count` independent tensors in as few
 * persistent launches as possible (one decoder layer, or a
 * whole model's linear weights, as the path runs in one forward pass).
 * Each tensor obeys the nf4_dequantize contract; all share `out_dtype`.
 *   tensors   [host] array of `count` descriptors, read during the call only.
 *   count     >= 0.  Up to NF4_MAX_BATCH tensors go into one launch; larger
 *             batches are split into consecutive launches on `stream`.
 * Validation covers every descriptor before anything is enqueued.
 */
#define NF4_MAX_BATCH 128
nf4_status nf4_dequantize_batched(const nf4_tensor* tensors, int32_t count, nf4_dtype out_dtype,
                                  void* stream);

/*
 * nf4_dequantize_host -- the same operation on HOST buffers (end-to-end path:
 * pinned host -> HBM -> kernel -> HBM -> pinned host).  The inputs are copied
 * in chunks of whole second-level groups, dequantized and copied back, triple
 * buffered on `stream` and an internal event chain so copies overlap compute.
 *   packed, absmax, out and the dq arrays (qabsmax, absmax2, code2) are [host]
 *   pointers (pinned memory gives full PCIe/C2C bandwidth; pageable works).
 *   workspace [device] >= nf4_host_workspace_bytes(chunk_elems, dq != NULL).
 *   chunk_elems elements per chunk, a positive multiple of 256 * blocksize.
 * Synchronous: returns after `out` holds the result (stream synchronised).
 */
nf4_status nf4_dequantize_host(const uint8_t* packed, const float* absmax, const nf4_dq_state* dq,
                               int64_t n, int32_t blocksize, nf4_dtype out_dtype, void* out,
                               void* workspace, int64_t workspace_bytes, int64_t chunk_elems,
                               void* stream);
int64_t nf4_host_workspace_bytes(int64_t chunk_elems, int32_t blocksize, int32_t dq);

/*
 * nf4_dequantize_host_batched -- nf4_dequantize_host over `count` tensors whose
 * chunks form ONE pipeline (no drain/refill between tensors).  Every pointer
 * in the descriptors (packed, absmax, dq.*, out) is a [host] pointer.  The
 * workspace must hold nf4_host_workspace_bytes(chunk_elems, smallest blocksize,
 * any tensor double-quantized); chunk_elems must be a multiple of 256 x the
 * largest blocksize.  fp32-absmax and double-quant tensors may be mixed: every
 * workspace slot reserves 4 B of scales per block of the smallest blocksize
 * (the widest scale slice a chunk can need), so no copy spills into a slot's
 * output region.  Synchronous like nf4_dequantize_host.
 */
nf4_status nf4_dequantize_host_batched(const nf4_tensor* tensors, int32_t count, nf4_dtype out_dtype,
                                       void* workspace, int64_t workspace_bytes, int64_t chunk_elems,
                                       void* stream);

/*
 * nf4_quantize -- blockwise NF4 quantization, used to GENERATE inputs
 * (the paper covers dequantization only).
 * Reading R12: absmax_b = max|x| over the block (exact); absmax_b == 0 gives
 * code 7 for the whole block; otherwise xn = fl32(x * fl32(1/absmax_b))
 * and idx = #{i : xn > t_i} over the 15 fp32 midpoints t_i of adjacent codes.
 *   in        [device] n values of in_dtype (NF4_F32, NF4_F16 or NF4_BF16).
 *   packed    [device] ceil(n/2) bytes out; odd n pads the last low nibble with 0.
 *   absmax    [device] nb fp32 out.
 * NaN/Inf inputs are not validated (S:99 applies to the CPU oracle only).
 */
nf4_status nf4_quantize(const void* in, nf4_dtype in_dtype, int64_t n, int32_t blocksize,
                        uint8_t* packed, float* absmax, void* stream);

/*
 * nf4_double_quantize -- second-level quantization of absmax (R13), used to
 * generate double-quant inputs.  d = fl32(absmax_b - offset); absmax2_g =
 * max|d| over 256 consecutive blocks; dn = fl32(d * fl32(1/absmax2_g)) (0 when
 * absmax2_g == 0); qabsmax_b = argmin_i fl32|dn - code2[i]|, ties to the lowest i.
 *   absmax  [device] nb fp32 in;  code2 [device] 256 fp32;  offset: host value.
 *   qabsmax [device] nb bytes out; absmax2 [device] ceil(nb/256) fp32 out.
 */
nf4_status nf4_double_quantize(const float* absmax, int64_t nb, float offset, const float* code2,
                               int32_t blocksize2, uint8_t* qabsmax, float* absmax2, void* stream);

/*
 * nf4_dequantize_ex / nf4_dequantize_batched_ex -- the same path with another
 * 16-entry codebook and/or fp32 output.
 *   codebook16 [host] 16 fp32 levels indexed by the 4-bit code, or NULL for NF4
 *              (e.g. nf4_codebook_fp4 for the BitsAndBytes FP4 format).  Read
 *              during the call only; copied into the kernel parameters.
 *   out_dtype  NF4_F16, NF4_BF16 or NF4_F32 (out[k] = the fp32 product itself;
 *              `out` then holds n fp32 values, 4-byte aligned).
 * Everything else as nf4_dequantize / nf4_dequantize_batched.
 */
nf4_status nf4_dequantize_ex(const uint8_t* packed, const float* absmax, const nf4_dq_state* dq,
                             int64_t n, int32_t blocksize, const float* codebook16, nf4_dtype out_dtype,
                             void* out, void* stream);
nf4_status nf4_dequantize_batched_ex(const nf4_tensor* tensors, int32_t count, const float* codebook16,
                                     nf4_dtype out_dtype, void* stream);

/* Host copy of the 16-entry NF4 table (R1), fp32. */
void nf4_codebook(float out16[16]);

/* Host copy of the BitsAndBytes FP4 table ({0, 0.0625, 8, 12, 4, 6, 2, 3} and
 * their negatives, divided by 12; [ext]) for nf4_dequantize_ex. */
void nf4_codebook_fp4(float out16[16]);

/* Static description of a status code; never NULL. */
const char* nf4_status_string(nf4_status s);

/* Number of kernels the last successful call on this thread enqueued (for
 * the bench's gpu_launches count). */
int32_t nf4_last_launch_count(void);

/* Early input reads (programmatic dependent launch), process-wide, default 0.
 * The dequantization kernels are launched so that they may start while the
 * previous kernel on the stream drains.  0: every global access waits for that
 * kernel (griddepcontrol.wait first).  1: the INPUTS -- packed codes, absmax or
 * the double-quant state and tables -- are read before the wait, so their DRAM
 * round trip overlaps the previous kernel's tail; only the stores to `out` wait
 * (measured mixed: up to -1.5 us per launch for 2^20-2^21 elements, -4% at
 * 2^26, but +7-16% at 2^22 / 2^24; profiles/r02_early_inputs.md).  Enable it
 * only when no kernel that can still be running when the call's kernel starts
 * writes those inputs: the immediately preceding kernel, and any earlier one
 * chained to it by programmatic dependent launch (this library's kernels are).
 * A quantize-then-dequantize sequence on one stream does NOT qualify unless an
 * event or memcpy boundary separates the two.  Takes effect for later calls;
 * results are identical either way. */
void nf4_set_early_input_reads(int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* NF4_H_ */
