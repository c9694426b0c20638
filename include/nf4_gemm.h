/*
 * nf4_gemm.h -- fused NF4 dequantization + tensor-core GEMM (SURVEY 8(f) row
 * F1, the step after the hot path: dequantization is 72.4% of the quantized
 * matmul; the paper's weights feed FP16 tensor-core GEMMs).
 *
 *   Y[m, n] = sum_k X[m, k] * W[n, k]        m < M, n < N, k < K
 *
 * where W is an NF4 weight of shape [N, K] (rows = output features, K
 * contiguous, the flat element index of W[n, k] is n*K + k) stored exactly as
 * nf4_dequantize consumes it, and every W[n, k] is the hot path's value
 * RNE16(fl32(NF4[idx] * a_b)) in X's 16-bit type (bit-identical to
 * nf4_dequantize's output; tests/test_gemm_gpu.py checks it through one-hot X).
 * Products are exact in fp32; accumulation is fp32 on the tcgen05 tensor cores
 * (order unspecified), so Y is within (K * 2^-23) * sum_k |X[m,k] W[n,k]| of the
 * exact sum, plus the final rounding when y_dtype is 16-bit (F1).
 *
 *   x        [device] M x K, row-major, 16-byte aligned, NF4_BF16 or NF4_F16.
 *   packed   [device] N*K/2 bytes, 16-byte aligned.
 *   absmax / dq  as nf4_dequantize (exactly one given); blocksize in
 *            [64, 4096], K a multiple of 64 and of blocksize.
 *   y        [device] M x N row-major, y_dtype NF4_F16, NF4_BF16 or NF4_F32.
 *   splits   <= 0: stream-K -- the (tile, 64-element k-chunk) stream is cut
 *            into one equal contiguous range per SM; a tile cut across
 *            ranges is summed from fp32 partials, in range order, by the CTA
 *            holding its last piece (same kernel, no second launch).
 *            >= 1: classic grid, one CTA per (128-feature tile, token tile,
 *            split) plus a reduction kernel summing in split order
 *            (nf4_gemm_default_splits gives a makespan-minimising factor).
 *   workspace  [device, 16-byte aligned] nf4_gemm_workspace_bytes(M, N, K,
 *            splits) bytes when that is > 0 (NULL/0 allowed otherwise).  For
 *            stream-K its head holds per-tile counters: it must be ZERO-FILLED
 *            before its first use; every call leaves it zeroed again, so one
 *            buffer serves any sequence of calls on one stream (not two
 *            concurrent calls).  Results are deterministic for a given
 *            (splits, GPU).
 *            The head of the workspace is a per-tile counter block that
 *            classic calls never write (their fp32 partials start after it),
 *            so classic and stream-K calls may share one buffer in any order.
 * Stream-ordered, asynchronous; status codes as nf4.h.
 * Programmatic dependent launch: the kernel may start while the previous
 * kernel on the stream drains.  By default it reads the WEIGHT (packed,
 * absmax / dq and its tables) before waiting for that kernel -- only x, y and
 * the workspace are ordered after it -- so a decode loop fetches and
 * dequantizes the next weight while the previous kernel finishes.  CUDA only
 * guarantees visibility of the previous kernel's writes after the wait, so a
 * caller whose immediately preceding kernel WRITES the weight (an in-place
 * update, a LoRA merge, a reload) must either call
 * nf4_gemm_set_early_weight_reads(0) (every read after the wait; process-wide)
 * or separate the two with an event / memcpy boundary.
 */
#ifndef NF4_GEMM_H_
#define NF4_GEMM_H_

#include <stdint.h>
#include "nf4.h"

#ifdef __cplusplus
extern "C" {
#endif

nf4_status nf4_gemm(const void* x, nf4_dtype x_dtype, int32_t M, const uint8_t* packed, const float* absmax,
                    const nf4_dq_state* dq, int32_t N, int32_t K, int32_t blocksize, void* y, nf4_dtype y_dtype,
                    int32_t splits, void* workspace, int64_t workspace_bytes, void* stream);

int32_t nf4_gemm_default_splits(int32_t M, int32_t N, int32_t K);
int64_t nf4_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K, int32_t splits);

/*
 * Grouped form: up to NF4_GEMM_MAX_GROUP weights that share the activation X
 * (and K, blocksize) -- e.g. the q/k/v or gate/up projections of a decoder
 * layer -- in ONE stream-K launch:  Y_i = X . W_i^T.  Each weight is described
 * as for nf4_gemm (packed [N_i, K] codes, fp32 absmax or dq, its own y_i
 * [M, N_i]); their 128-feature tiles are concatenated into one work stream, so
 * the launch's fill/drain is paid once.  Numerics are nf4_gemm's (bit-exact
 * weights, fp32 accumulation; the summation order can differ from separate
 * calls).  workspace: nf4_gemm_grouped_workspace_bytes(M, N[], count, K) bytes,
 * zero-filled before first use and left zeroed (same contract as stream-K
 * nf4_gemm).  Errors: NF4_ERR_BAD_SIZE for count outside [1, 4] or a problem too
 * large for the stream-K indices (> 2^31 chunk tiles), else as nf4_gemm.
 */
#define NF4_GEMM_MAX_GROUP 4
typedef struct {
  const uint8_t* packed;   /* [device] N*K/2 bytes, 16-byte aligned */
  const float* absmax;     /* [device] fp32 absmax, or NULL for dq */
  nf4_dq_state dq;         /* used when absmax == NULL */
  int32_t N;               /* output features of this weight */
  void* y;                 /* [device] M x N row-major, y_dtype */
} nf4_gemm_weight;

nf4_status nf4_gemm_grouped(const void* x, nf4_dtype x_dtype, int32_t M, int32_t K, int32_t blocksize,
                            const nf4_gemm_weight* weights, int32_t count, nf4_dtype y_dtype, void* workspace,
                            int64_t workspace_bytes, void* stream);
int64_t nf4_gemm_grouped_workspace_bytes(int32_t M, const int32_t* N, int32_t count, int32_t K);

/*
 * Multi-problem form: up to NF4_GEMM_MAX_MULTI independent problems
 * Y_i = X_i . W_i^T in ONE persistent stream-K launch -- every problem has its
 * own activation X_i [M, K_i] and reduction length K_i; M, the X/Y dtypes and
 * the blocksize are shared.  The problems' (tile, k-chunk) streams are
 * concatenated problem by problem and cut into one equal range per SM, so the
 * launch's fill and drain (~5-8 us) is paid once for all of them instead of
 * once per GEMM -- e.g. every linear weight of several decoder layers at a
 * decode step whose inputs are ready, or the experts of an MoE layer.
 * Numerics are nf4_gemm's (bit-exact weights, fp32 accumulation; deterministic
 * for a given problem list and GPU).
 *   problems[i].x  [device] M x K_i, 16-byte aligned, x_dtype; may be shared.
 *   problems[i].K  multiple of 64 and of blocksize (0: Y_i = 0).
 *   others as nf4_gemm_weight.
 * workspace: nf4_gemm_multi_workspace_bytes(M, N[], K[], count), zero-filled
 * before first use and left zeroed (the stream-K contract of nf4_gemm).
 * Errors: NF4_ERR_BAD_SIZE for count outside [1, NF4_GEMM_MAX_MULTI], a K that
 * is not a multiple of 64 and of blocksize, or more than 2^31 chunk tiles in
 * total; else as nf4_gemm.
 */
#define NF4_GEMM_MAX_MULTI 64
typedef struct {
  const void* x;           /* [device] M x K row-major, x_dtype */
  int32_t K;
  const uint8_t* packed;   /* [device] N*K/2 bytes, 16-byte aligned */
  const float* absmax;     /* [device] fp32 absmax, or NULL for dq */
  nf4_dq_state dq;         /* used when absmax == NULL */
  int32_t N;
  void* y;                 /* [device] M x N row-major, y_dtype */
} nf4_gemm_problem;

nf4_status nf4_gemm_multi(const nf4_gemm_problem* problems, int32_t count, int32_t M, nf4_dtype x_dtype,
                          int32_t blocksize, nf4_dtype y_dtype, void* workspace, int64_t workspace_bytes,
                          void* stream);
int64_t nf4_gemm_multi_workspace_bytes(int32_t M, const int32_t* N, const int32_t* K, int32_t count);

/* 1 (default): the GEMM kernels read the weight before griddepcontrol.wait
 * (see above); 0: after it.  Process-wide, takes effect for later calls. */
void nf4_gemm_set_early_weight_reads(int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* NF4_GEMM_H_ */
