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
// Roles (320 threads):
//   warp 9     TMA issuer (one lane): per 64-element k-chunk, a 2-D TMA box of
//              the packed codes (128 rows x 32 B) and a 2-D TMA box of X
//              (BN rows x 64 elements, SWIZZLE_128B: lands directly in the UMMA
//              canonical layout, zero-filled past M) -> tma_full[s].
//   warps 0-7  producers: threads 2r, 2r+1 own W row n0+r; each reads its 16
//              code bytes from shared memory, dequantizes 32 weights into 4 of
//              the row's 8 swizzled 16-B chunks, fence.proxy.async, arrive
//              w_full[s].  After the K loop they are the epilogue: warp w reads
//              TMEM lanes 32(w%4).. and column half w/4 with tcgen05.ld.
//   warp 8     TMEM allocator and MMA issuer: waits tma_full[s] + w_full[s],
//              issues 4 x tcgen05.mma (K=16 each), tcgen05.commit -> empty[s];
//              after the last chunk commits -> done.
// (A first version had every producer thread load its own row's codes: row-
// strided 16-B loads cost 32 L1 wavefronts per warp instruction and capped the
// kernel at ~0.5 TB/s; TMA boxes fetch the same bytes with full-line requests.)
// Swap-AB orientation: the MMA's M=128 side is the weight (128 output
// features), its N side the tokens (BN in {16,...,256}), so decode-size M
// wastes nothing.  Split-K over gridDim.z writes fp32 partials to a caller
// workspace; nf4_gemm_reduce sums them in split order (deterministic).
#include <cuda.h>  // CUtensorMap (the encoder is fetched at run time; no libcuda link)
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "nf4_internal.cuh"
#include "../../include/nf4_gemm.h"

namespace nf4 {
namespace gemm {

constexpr int kProducers = 256;             // 2 threads per weight row (32 elements each)
constexpr int kProducerWarps = kProducers / 32;
constexpr int kThreads = kProducers + 64;   // + MMA warp + TMA warp
constexpr int kCodeBytes = 32;              // packed bytes per row per k-chunk
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
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(b), "r"(parity), "r"(0x989680) : "memory");
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

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// TMEM column budget: the fp32 accumulator (BN columns) at column 0, then
// STAGES dequantized A tiles of 32 columns (128 lanes x 64 16-bit weights).
template <int BN, int STAGES>
__host__ __device__ constexpr int tmem_cols() {
  constexpr int need = (BN < 32 ? 32 : BN) + STAGES * 32;
  return need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
}

template <int BN, int STAGES, int RING, bool BF16>
__global__ void __launch_bounds__(kThreads, 1)
    nf4_gemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap map_codes,
                    const __grid_constant__ CUtensorMap map_x) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the swizzle atoms (offset arithmetic on the __shared__
  // array keeps the shared address space visible to the compiler: LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* smem_x = smem;                                     // STAGES x BN x 128 B (X, SW128, by TMA)
  uint8_t* smem_c = smem_x + STAGES * BN * kRowBytes;         // STAGES x 4 KB (packed codes, by TMA)
  uint64_t* tma_full = reinterpret_cast<uint64_t*>(smem_c + STAGES * 128 * kCodeBytes);
  uint64_t* w_full = tma_full + STAGES;
  uint64_t* empty = w_full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);
  __shared__ __align__(256) float lut[16];                    // 256-B aligned: address = PRMT(offsets, base)
  __shared__ float code2s[256];                               // DQ second-level table

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int m0 = blockIdx.y * BN;
  const int split = blockIdx.z;
  const int nk_total = p.K / kChunk;
  const int kc0 = split * p.chunks_per_split;
  const int kc1 = min(nk_total, kc0 + p.chunks_per_split);
  const int nk = kc1 > kc0 ? kc1 - kc0 : 0;
  constexpr int TMEM_COLS = tmem_cols<BN, STAGES>();
  constexpr int ACC_COLS = BN < 32 ? 32 : BN;                 // A stages start here (32-column aligned)
  constexpr uint32_t kStageTx = 128 * kCodeBytes + BN * kRowBytes;

  if (threadIdx.x < 16) lut[threadIdx.x] = p.lut[threadIdx.x];
  if (p.absmax == nullptr) {
    for (int i = threadIdx.x; i < 256; i += kThreads) code2s[i] = p.code2[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tma_full[s], 1);
      mbar_init(&w_full[s], kProducerWarps);   // one elected arrive per producer warp
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kProducerWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "n"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == kProducerWarps + 1 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_codes)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;

  if (warp < kProducerWarps) {
    // ======================= producers (dequantize into TMEM) =======================
    // Warp w may only address TMEM lanes 32(w%4)..32(w%4)+31, so thread (w, l)
    // owns weight row r = 32(w%4)+l of the tile and k-half h = w/4 (32 of the
    // chunk's 64 elements).  The block-scale inputs of chunk i+RING are loaded
    // while chunk i is dequantized (register ring); the codes arrive by TMA.
    const int t = 32 * (warp & 3) + lane;      // tile row = TMEM lane
    const int half = warp >> 2;
    const int row = n0 + t;                    // weight row (output feature)
    const bool row_ok = row < p.N;
    const int64_t blk_base = (int64_t(row) * p.K) >> p.bs_shift;
    const int chunk_shift = p.bs_shift - 6;    // 64-element chunks per quantization block = 2^chunk_shift
    const uint32_t tlane = uint32_t(32 * (warp & 3)) << 16;
    const uint32_t lut_base = smem_u32(lut);   // low byte 0: PRMT splices a byte offset into it
    uint32_t rq[RING];     // fp32 absmax bits, or qabsmax (DQ)
    float ra2[RING];       // absmax2 (DQ)
    auto issue = [&](int d, int i) {
      rq[d] = 0;
      ra2[d] = 0.0f;
      if (row_ok) {
        const int64_t b = blk_base + ((kc0 + i) >> chunk_shift);
        if (p.absmax != nullptr) {
          rq[d] = __float_as_uint(__ldg(p.absmax + b));
        } else {
          rq[d] = __ldg(p.qabsmax + b);
          ra2[d] = __ldg(p.absmax2 + (b >> 8));
        }
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
        if (i + RING < nk) issue(d, i + RING);
        mbar_wait_parity(&tma_full[s], (i / STAGES) & 1);   // codes (and X) landed; A stage s is free
        const uint4 c0 = *reinterpret_cast<const uint4*>(smem_c + s * 128 * kCodeBytes + t * kCodeBytes + 16 * half);
        // dequantize 32 weights: word j = (element 2j) | (element 2j+1) << 16
        const uint32_t cw[4] = {c0.x, c0.y, c0.z, c0.w};
        const uint64_t aa = f32x2_splat(a);
        uint32_t w[16];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const uint32_t x = cw[cc];
          const uint32_t hi4 = (x >> 2) & 0x3C3C3C3Cu;  // byte j = 4 * high nibble (LUT byte offset)
          const uint32_t lo4 = (x << 2) & 0x3C3C3C3Cu;  // byte j = 4 * low nibble
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // shared address of NF4[idx] = lut_base with byte 0 replaced by byte j of hi4/lo4: one PRMT
            const uint32_t ah = __byte_perm(hi4, lut_base, 0x7650u + j);
            const uint32_t al = __byte_perm(lo4, lut_base, 0x7650u + j);
            float ch, cl;
            asm("ld.shared.f32 %0, [%1];" : "=f"(ch) : "r"(ah));
            asm("ld.shared.f32 %0, [%1];" : "=f"(cl) : "r"(al));
            mul2_rn(ch, cl, aa);                      // fl32(NF4[idx] * a) for both, one FMUL2
            w[4 * cc + j] = pack2_rn<BF16>(ch, cl);
          }
        }
        // 16 columns (32 weights) of this row's A tile in TMEM
        const uint32_t taddr = tmem + tlane + uint32_t(ACC_COLS + s * 32 + half * 16);
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
            ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
            "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&w_full[s]);
      }
    }
    // ======================= epilogue =======================
    mbar_wait_parity(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;                          // TMEM lane quarter this warp may access
    constexpr int HB = BN / 2 < 16 ? 16 : BN / 2;    // columns per warp (BN = 16: warps 4-7 idle)
    const int col0 = (warp >> 2) * HB;
    const int n = n0 + q * 32 + lane;
    const uint32_t taddr = tmem + (uint32_t(q * 32) << 16);
#pragma unroll
    for (int cb = col0; cb < col0 + HB && cb < BN; cb += 16) {
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
  } else if (warp == kProducerWarps + 1) {
    // ======================= TMA issuer (one thread) =======================
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        mbar_wait_parity(&empty[s], ((i / STAGES) & 1) ^ 1);   // MMA of chunk i-STAGES released the slot
        const int k0 = (kc0 + i) * kChunk;
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
            smem_u32(&tma_full[s])), "r"(kStageTx) : "memory");
        tma_load_2d(smem_c + s * 128 * kCodeBytes, &map_codes, k0 / 2, n0, &tma_full[s]);
        tma_load_2d(smem_x + s * BN * kRowBytes, &map_x, k0, m0, &tma_full[s]);
      }
    }
  } else if (lane == 0) {
    // ======================= MMA issuer (one thread) =======================
    const uint32_t idesc = umma_idesc(BN, BF16);
    for (int i = 0; i < nk; ++i) {
      const int s = i % STAGES;
      mbar_wait_parity(&tma_full[s], (i / STAGES) & 1);
      mbar_wait_parity(&w_full[s], (i / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t xa = smem_u32(smem_x + s * BN * kRowBytes);
#pragma unroll
      for (int kk = 0; kk < kChunk / 16; ++kk) {
        const uint32_t a_tmem = tmem + uint32_t(ACC_COLS + s * 32 + kk * 8);   // A: 128 lanes x 16 weights
        const uint64_t bdesc = umma_desc_sw128(xa + kk * 32);
        const uint32_t accum = (i > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
            ::"r"(tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum) : "memory");
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
  if (warp == kProducerWarps) {
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
  // TMEM: accumulator + STAGES x 32 columns; BN <= 32 -> 128 columns -> 4 CTAs/SM fit in 512
  return BN <= 32 ? 3 : BN <= 64 ? 6 : BN <= 128 ? 4 : 5;
}
template <int BN>
constexpr int ring_for() {
  return BN <= 64 ? 4 : 2;
}

template <int BN>
constexpr size_t smem_bytes() {
  return 1024 /*align slack*/ + size_t(stages_for<BN>()) * (BN * kRowBytes + 128 * kCodeBytes) +
         (3 * stages_for<BN>() + 1) * 8 + 16 + 64 + 1024 + 64;
}

template <int BN, bool BF16>
static cudaError_t launch(const GemmParams& p, const CUtensorMap& mc, const CUtensorMap& mx, dim3 grid,
                          cudaStream_t s) {
  constexpr int ST = stages_for<BN>();
  auto k = nf4_gemm_kernel<BN, ST, ring_for<BN>(), BF16>;
  constexpr size_t sm = smem_bytes<BN>();
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  if (e != cudaSuccess) return e;
  k<<<grid, kThreads, sm, s>>>(p, mc, mx);
  return cudaPeekAtLastError();
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encoder() {
  static std::once_flag once;
  static EncodeTiledFn fn = nullptr;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  return fn;
}

// 2-D tensor map over a row-major [rows, cols] matrix of `elem` bytes.
static bool make_map(CUtensorMap* m, CUtensorMapDataType dt, int elem, const void* base, uint64_t cols,
                     uint64_t rows, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * uint64_t(elem)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

template <int BN, bool BF16>
static int gemm_occupancy() {
  static int occ = 0;
  if (occ == 0) {
    int v = 0;
    auto k = nf4_gemm_kernel<BN, stages_for<BN>(), ring_for<BN>(), BF16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes<BN>()));
    occ = (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, kThreads, smem_bytes<BN>()) == cudaSuccess && v > 0)
              ? v : 1;
  }
  return occ;
}

static int occupancy_for_bn(int bn) {
  switch (bn) {
    case 16: return gemm_occupancy<16, true>();
    case 32: return gemm_occupancy<32, true>();
    case 64: return gemm_occupancy<64, true>();
    case 128: return gemm_occupancy<128, true>();
    default: return gemm_occupancy<256, true>();
  }
}

// Split-K factor minimising the makespan of the (row tile, token tile, split)
// grid on this GPU: waves x (chunks per split + ~2 chunks of per-CTA prologue
// and epilogue), preferring fewer splits on near ties (less partial traffic).
extern "C" int32_t nf4_gemm_default_splits(int32_t M, int32_t N, int32_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 1;
  const int bn = pick_bn(M);
  const int64_t tiles = int64_t((N + 127) / 128) * ((M + bn - 1) / bn);
  const int64_t cap = int64_t(sm_count()) * occupancy_for_bn(bn);
  const int64_t nk = K / 64;
  int best_s = 1;
  double best = 1e30;
  for (int64_t sp = 1; sp <= 32 && sp <= nk; ++sp) {
    const int64_t waves = (tiles * sp + cap - 1) / cap;
    const double cost = double(waves) * double((nk + sp - 1) / sp + 2);
    if (cost < best * 0.97) {
      best = cost;
      best_s = int(sp);
    }
  }
  return best_s;
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
  CUtensorMap mc, mx;
  if (!make_map(&mc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, packed, uint64_t(K) / 2, uint64_t(N), kCodeBytes, 128,
                CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_map(&mx, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x, uint64_t(K),
                uint64_t(M), kChunk, uint32_t(bn), CU_TENSOR_MAP_SWIZZLE_128B))
    return NF4_ERR_CUDA;
  cudaError_t e;
  switch (bn) {
    case 16: e = bf16 ? launch<16, true>(p, mc, mx, grid, s) : launch<16, false>(p, mc, mx, grid, s); break;
    case 32: e = bf16 ? launch<32, true>(p, mc, mx, grid, s) : launch<32, false>(p, mc, mx, grid, s); break;
    case 64: e = bf16 ? launch<64, true>(p, mc, mx, grid, s) : launch<64, false>(p, mc, mx, grid, s); break;
    case 128: e = bf16 ? launch<128, true>(p, mc, mx, grid, s) : launch<128, false>(p, mc, mx, grid, s); break;
    default: e = bf16 ? launch<256, true>(p, mc, mx, grid, s) : launch<256, false>(p, mc, mx, grid, s); break;
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
