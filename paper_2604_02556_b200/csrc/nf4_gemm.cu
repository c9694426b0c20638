// nf4_gemm.cu -- fused NF4 dequantization + tcgen05 tensor-core GEMM (SURVEY
// row F1): Y[M, N] = X[M, K] . W[N, K]^T where W is an NF4 weight ([out, in],
// K contiguous, blockwise absmax along K) and X, Y are 16-bit activations.
//
// The weight never exists in HBM as 16-bit: producer warps read the packed
// codes (0.5 B/elt) + scales, dequantize them with exactly the hot path's
// per-element definition (RNE16(fl32(NF4[idx] * a))) straight into
// shared memory in the UMMA canonical K-major SWIZZLE_128B layout, and one
// elected thread issues tcgen05.mma (kind::f16, fp32 accumulation in TMEM).
// The paper motivates exactly this step: dequantization is 72.4% of the
// quantized matmul and the fused, preprocessing-free direction is the
// one it leaves open.
//
// Roles (160 threads):
//   warps 0-3  producers: thread t owns W row n0+t of the tile; per 64-element
//              k-chunk it dequantizes 64 weights into a 128-byte swizzled row,
//              and the 128 threads together copy the X tile (BN rows x 128 B);
//              then fence.proxy.async + mbarrier arrive (full[s]).  After the K
//              loop they are the epilogue: tcgen05.ld of their 32 TMEM lanes.
//   warp 4     TMEM allocator and MMA issuer: waits full[s], issues 4 x
//              tcgen05.mma (K=16 each), tcgen05.commit -> empty[s]; after the
//              last chunk commits -> done.
// Swap-AB orientation: the MMA's M=128 side is the weight (128 output
// features), its N side the tokens (BN in {16,...,256}), so decode-size M
// wastes nothing.  Split-K over gridDim.z writes fp32 partials to a caller
// workspace; nf4_gemm_reduce sums them in split order (deterministic).
#include <cuda_runtime.h>
#include <stdint.h>

#include "nf4_internal.cuh"
#include "../../include/nf4_gemm.h"

namespace nf4 {
namespace gemm {

constexpr int kProducers = 128;
constexpr int kThreads = kProducers + 32;
constexpr int kChunk = 64;          // k elements per stage (= one 128 B swizzle row in 16-bit)
constexpr int kRowBytes = 128;

struct GemmParams {
  const uint8_t* packed;
  const float* absmax;     // fp32 mode if non-null
  const uint8_t* qabsmax;  // DQ mode
  const float* code2;
  const float* absmax2;
  const uint16_t* x;       // [M, K] 16-bit
  void* y;                 // [M, N] (splits == 1)
  float* partial;          // [splits, M, N] fp32 (splits > 1)
  float offset;
  int32_t M, N, K;
  int32_t bs_shift;
  int32_t chunks_per_split;
  int32_t splits;
  int32_t out_dtype;       // NF4_F16 / NF4_BF16 / NF4_F32
  float lut[16];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(b), "r"(parity) : "memory");
  }
}

// UMMA shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row atoms of
// 1024 B stacked densely (SBO = 1024 B), LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16 (or fp16), both K-major.
__device__ __forceinline__ uint32_t umma_idesc(int n, bool bf16) {
  const uint32_t fmt = bf16 ? 1u : 0u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ float dq_scale(const GemmParams& p, const float* code2s, int64_t b) {
  if (p.absmax != nullptr) return __ldg(p.absmax + b);
  const uint32_t q = __ldg(p.qabsmax + b);
  return __fadd_rn(__fmul_rn(code2s[q], __ldg(p.absmax2 + (b >> 8))), p.offset);
}

template <int BN, int STAGES, int RING, bool BF16>
__global__ void __launch_bounds__(kThreads, 1) nf4_gemm_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_w = smem;                                     // STAGES x 16 KB
  uint8_t* smem_x = smem_w + STAGES * 128 * kRowBytes;        // STAGES x BN x 128 B
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_x + STAGES * BN * kRowBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);
  float* lut = reinterpret_cast<float*>(tmem_holder + 4);
  float* code2s = lut + 16;                                   // 256 floats (DQ)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int m0 = blockIdx.y * BN;
  const int split = blockIdx.z;
  const int nk_total = p.K / kChunk;
  const int kc0 = split * p.chunks_per_split;
  const int kc1 = min(nk_total, kc0 + p.chunks_per_split);
  const int nk = kc1 > kc0 ? kc1 - kc0 : 0;
  constexpr int TMEM_COLS = BN < 32 ? 32 : BN;

  if (threadIdx.x < 16) lut[threadIdx.x] = p.lut[threadIdx.x];
  if (p.absmax == nullptr) {
    for (int i = threadIdx.x; i < 256; i += kThreads) code2s[i] = p.code2[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kProducers);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "n"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;

  if (warp < 4) {
    // ======================= producers =======================
    // Register ring of depth RING: the global loads (32 B of codes, the
    // block-scale inputs, this thread's share of the X tile) of chunk i+RING
    // are issued before chunk i is dequantized, so each thread keeps RING
    // chunks (128 B of codes at RING = 4) in flight.
    const int t = threadIdx.x;
    const int row = n0 + t;                    // weight row (output feature)
    const bool row_ok = row < p.N;
    const int64_t row_base = int64_t(row) * p.K;
    constexpr int XCH = BN * 8 / kProducers > 0 ? BN * 8 / kProducers : 1;  // 16-B X chunks per thread
    uint4 rc0[RING], rc1[RING];
    uint32_t rq[RING];     // fp32 absmax bits, or qabsmax (DQ)
    float ra2[RING];       // absmax2 (DQ)
    uint4 rx[RING][XCH];
    auto issue = [&](int d, int i) {
      const int k0 = (kc0 + i) * kChunk;
      rc0[d] = make_uint4(0, 0, 0, 0);
      rc1[d] = make_uint4(0, 0, 0, 0);
      rq[d] = 0;
      ra2[d] = 0.0f;
      if (row_ok) {
        const uint8_t* cp = p.packed + ((row_base + k0) >> 1);
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(rc0[d].x), "=r"(rc0[d].y), "=r"(rc0[d].z), "=r"(rc0[d].w) : "l"(cp));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(rc1[d].x), "=r"(rc1[d].y), "=r"(rc1[d].z), "=r"(rc1[d].w) : "l"(cp + 16));
        const int64_t b = (row_base + k0) >> p.bs_shift;
        if (p.absmax != nullptr) {
          rq[d] = __float_as_uint(__ldg(p.absmax + b));
        } else {
          rq[d] = __ldg(p.qabsmax + b);
          ra2[d] = __ldg(p.absmax2 + (b >> 8));
        }
      }
#pragma unroll
      for (int j = 0; j < XCH; ++j) {
        const int idx = t + j * kProducers;
        const int m = idx >> 3, c = idx & 7;
        rx[d][j] = make_uint4(0, 0, 0, 0);
        if (idx < BN * 8 && m0 + m < p.M)
          rx[d][j] = __ldg(reinterpret_cast<const uint4*>(p.x + int64_t(m0 + m) * p.K + k0 + c * 8));
      }
    };
#pragma unroll
    for (int d = 0; d < RING; ++d)
      if (d < nk) issue(d, d);
    for (int i0 = 0; i0 < nk; i0 += RING) {
#pragma unroll
      for (int d = 0; d < RING; ++d) {
        const int i = i0 + d;
        if (i >= nk) break;
        const int s = i % STAGES;
        // block scale (A4): fp32 absmax, or fl32(fl32(code2[q] * absmax2) + offset)
        const float a = p.absmax != nullptr ? __uint_as_float(rq[d])
                                            : __fadd_rn(__fmul_rn(code2s[rq[d]], ra2[d]), p.offset);
        mbar_wait_parity(&empty[s], ((i / STAGES) & 1) ^ 1);
        // dequantize 64 weights of this row -> 8 swizzled 16-B chunks
        uint8_t* wrow = smem_w + s * 128 * kRowBytes + t * kRowBytes;
        const uint32_t cw[8] = {rc0[d].x, rc0[d].y, rc0[d].z, rc0[d].w, rc1[d].x, rc1[d].y, rc1[d].z, rc1[d].w};
#pragma unroll
        for (int c = 0; c < 8; ++c) {     // chunk c = elements 8c..8c+7 = code bytes 4c..4c+3
          const uint32_t x = cw[c];
          uint32_t w4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t byte = (x >> (8 * j)) & 0xFFu;
            const float ph2 = __fmul_rn(lut[byte >> 4], a);
            const float pl2 = __fmul_rn(lut[byte & 0x0Fu], a);
            w4[j] = pack2_rn<BF16>(ph2, pl2);
          }
          *reinterpret_cast<uint4*>(wrow + ((c ^ (t & 7)) << 4)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        uint8_t* xs = smem_x + s * BN * kRowBytes;
#pragma unroll
        for (int j = 0; j < XCH; ++j) {
          const int idx = t + j * kProducers;
          if (idx < BN * 8) {
            const int m = idx >> 3, c = idx & 7;
            *reinterpret_cast<uint4*>(xs + m * kRowBytes + ((c ^ (m & 7)) << 4)) = rx[d][j];
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&full[s]);
        if (i + RING < nk) issue(d, i + RING);
      }
    }
    // ======================= epilogue =======================
    mbar_wait_parity(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int n = n0 + warp * 32 + lane;
    const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16);
#pragma unroll
    for (int cb = 0; cb < BN; cb += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr + cb));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (n < p.N) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = m0 + cb + j;
          if (m < p.M) {
            const float acc = nk > 0 ? __uint_as_float(v[j]) : 0.0f;
            if (p.splits > 1) {
              p.partial[(int64_t(split) * p.M + m) * p.N + n] = acc;
            } else if (p.out_dtype == NF4_F32) {
              static_cast<float*>(p.y)[int64_t(m) * p.N + n] = acc;
            } else {
              static_cast<uint16_t*>(p.y)[int64_t(m) * p.N + n] =
                  p.out_dtype == NF4_BF16 ? cvt1_rn<true>(acc) : cvt1_rn<false>(acc);
            }
          }
        }
      }
    }
  } else if (lane == 0) {
    // ======================= MMA issuer (one thread) =======================
    const uint32_t idesc = umma_idesc(BN, BF16);
    for (int i = 0; i < nk; ++i) {
      const int s = i % STAGES;
      mbar_wait_parity(&full[s], (i / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t wa = smem_u32(smem_w + s * 128 * kRowBytes);
      const uint32_t xa = smem_u32(smem_x + s * BN * kRowBytes);
#pragma unroll
      for (int kk = 0; kk < kChunk / 16; ++kk) {
        const uint64_t adesc = umma_desc_sw128(wa + kk * 32);
        const uint64_t bdesc = umma_desc_sw128(xa + kk * 32);
        const uint32_t accum = (i > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
            ::"r"(tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&empty[s])) : "memory");
    }
    if (nk > 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(done)) : "memory");
    else
      mbar_arrive(done);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

// Deterministic split-K reduction: y[m, n] = sum_s partial[s, m, n] in split order.
__global__ void nf4_gemm_reduce_kernel(const float* __restrict__ partial, int splits, int64_t mn, void* y,
                                       int out_dtype) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < mn; i += int64_t(gridDim.x) * blockDim.x) {
    float acc = partial[i];
    for (int s = 1; s < splits; ++s) acc = __fadd_rn(acc, partial[int64_t(s) * mn + i]);
    if (out_dtype == NF4_F32)
      static_cast<float*>(y)[i] = acc;
    else
      static_cast<uint16_t*>(y)[i] = out_dtype == NF4_BF16 ? cvt1_rn<true>(acc) : cvt1_rn<false>(acc);
  }
}

template <int BN>
constexpr int stages_for() {
  return BN <= 128 ? 4 : 3;
}
template <int BN>
constexpr int ring_for() {
  return BN <= 64 ? 4 : 2;
}

template <int BN>
constexpr size_t smem_bytes() {
  return 1024 /*align slack*/ + size_t(stages_for<BN>()) * (128 + BN) * kRowBytes + 2 * 8 * 8 + 64 + 64 + 1024 + 64;
}

template <int BN, bool BF16>
static cudaError_t launch(const GemmParams& p, dim3 grid, cudaStream_t s) {
  constexpr int ST = stages_for<BN>();
  auto k = nf4_gemm_kernel<BN, ST, ring_for<BN>(), BF16>;
  constexpr size_t sm = smem_bytes<BN>();
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  if (e != cudaSuccess) return e;
  k<<<grid, kThreads, sm, s>>>(p);
  return cudaPeekAtLastError();
}

}  // namespace gemm
}  // namespace nf4

using namespace nf4;
using namespace nf4::gemm;

static int pick_bn(int M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128) return 128;
  return 256;
}

extern "C" int64_t nf4_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K, int32_t splits) {
  if (M <= 0 || N <= 0 || K <= 0 || splits <= 1) return 0;
  return int64_t(splits) * M * N * 4;
}

extern "C" int32_t nf4_gemm_default_splits(int32_t M, int32_t N, int32_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 1;
  const int bn = pick_bn(M);
  const int64_t tiles = int64_t((N + 127) / 128) * ((M + bn - 1) / bn);
  const int64_t target = int64_t(sm_count()) * 2;  // ~2 CTAs per SM
  int64_t s = (target + tiles - 1) / tiles;
  const int64_t nk = K / 64;
  if (s > nk / 4) s = nk / 4 > 0 ? nk / 4 : 1;      // keep >= 4 chunks per split
  if (s > 32) s = 32;
  return int32_t(s < 1 ? 1 : s);
}

extern "C" nf4_status nf4_gemm(const void* x, nf4_dtype x_dtype, int32_t M, const uint8_t* packed,
                               const float* absmax, const nf4_dq_state* dq, int32_t N, int32_t K, int32_t blocksize,
                               void* y, nf4_dtype y_dtype, int32_t splits, void* workspace,
                               int64_t workspace_bytes, void* stream) {
  if (M < 0 || N < 0 || K < 0) return NF4_ERR_BAD_SIZE;
  if (x_dtype != NF4_F16 && x_dtype != NF4_BF16) return NF4_ERR_BAD_DTYPE;
  if (y_dtype != NF4_F16 && y_dtype != NF4_BF16 && y_dtype != NF4_F32) return NF4_ERR_BAD_DTYPE;
  if (!is_pow2(blocksize) || blocksize < 64 || blocksize > 4096) return NF4_ERR_BAD_BLOCKSIZE;
  if ((absmax == nullptr) == (dq == nullptr)) return NF4_ERR_BAD_STATE;
  if (dq && dq->blocksize2 != 256) return NF4_ERR_BAD_STATE;
  if (M == 0 || N == 0) { set_launch_count(0); return NF4_OK; }
  if (K % 64 != 0 || K % blocksize != 0) return NF4_ERR_BAD_SIZE;  // a 64-chunk never spans two blocks
  if (!x || !packed || !y) return NF4_ERR_NULL_POINTER;
  if (dq && (!dq->qabsmax || !dq->code2 || !dq->absmax2)) return NF4_ERR_NULL_POINTER;
  if (!aligned(x, 16) || !aligned(packed, 16)) return NF4_ERR_MISALIGNED;
  if (!aligned(y, y_dtype == NF4_F32 ? 4 : 2)) return NF4_ERR_MISALIGNED;
  if (absmax && !aligned(absmax, 4)) return NF4_ERR_MISALIGNED;
  if (splits <= 0) splits = nf4_gemm_default_splits(M, N, K);
  const int nk = K / 64;
  if (splits > nk) splits = nk > 0 ? nk : 1;
  if (splits > 1) {
    if (!workspace) return NF4_ERR_NULL_POINTER;
    if (workspace_bytes < nf4_gemm_workspace_bytes(M, N, K, splits)) return NF4_ERR_BAD_STATE;
    if (!aligned(workspace, 16)) return NF4_ERR_MISALIGNED;
  }
  GemmParams p;
  p.packed = packed;
  p.absmax = absmax;
  p.qabsmax = dq ? dq->qabsmax : nullptr;
  p.code2 = dq ? dq->code2 : nullptr;
  p.absmax2 = dq ? dq->absmax2 : nullptr;
  p.offset = dq ? dq->offset : 0.0f;
  p.x = static_cast<const uint16_t*>(x);
  p.y = y;
  p.partial = static_cast<float*>(workspace);
  p.M = M;
  p.N = N;
  p.K = K;
  p.bs_shift = log2i(blocksize);
  p.splits = splits;
  p.chunks_per_split = (nk + splits - 1) / splits;
  p.out_dtype = int(y_dtype);
  nf4_codebook(p.lut);
  const int bn = pick_bn(M);
  dim3 grid((N + 127) / 128, (M + bn - 1) / bn, splits);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool bf16 = x_dtype == NF4_BF16;
  cudaError_t e;
  switch (bn) {
    case 16: e = bf16 ? launch<16, true>(p, grid, s) : launch<16, false>(p, grid, s); break;
    case 32: e = bf16 ? launch<32, true>(p, grid, s) : launch<32, false>(p, grid, s); break;
    case 64: e = bf16 ? launch<64, true>(p, grid, s) : launch<64, false>(p, grid, s); break;
    case 128: e = bf16 ? launch<128, true>(p, grid, s) : launch<128, false>(p, grid, s); break;
    default: e = bf16 ? launch<256, true>(p, grid, s) : launch<256, false>(p, grid, s); break;
  }
  if (e != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
  int launches = 1;
  if (splits > 1) {
    const int64_t mn = int64_t(M) * N;
    int64_t g = (mn + 255) / 256;
    if (g > int64_t(sm_count()) * 8) g = int64_t(sm_count()) * 8;
    nf4_gemm_reduce_kernel<<<int(g), 256, 0, s>>>(static_cast<const float*>(workspace), splits, mn, y, int(y_dtype));
    if (cudaPeekAtLastError() != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
    ++launches;
  }
  set_launch_count(launches);
  return NF4_OK;
}
