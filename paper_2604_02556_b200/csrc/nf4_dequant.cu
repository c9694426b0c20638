// nf4_dequant.cu -- B200 (sm_100a) blockwise NF4 -> FP16/BF16 dequantization.
//
// The hot path of arxiv 2604.02556 (Alg. 1): unpack two 4-bit codes
// per byte (high nibble first), look each up in the 16-entry NF4
// table, scale by the block's absmax (fp32, or double-quantized, R7),
// round the fp32 product to 16 bits and store.
//
// B200 design:
//  * One persistent launch per batch of up to NF4_MAX_BATCH tensors (F3):
//    the grid is SM count x resident CTAs, CTAs stride over fixed 16384-
//    element tiles of all tensors; a tile never spans two tensors.
//  * Per thread and tile: 4 independent 64-bit code loads (16 elements each,
//    warp-contiguous 256 B), 4 scale decodes, then 4 x 256-bit evict-first
//    stores (warp-contiguous 1 KB): ~32 B of loads in flight per thread.
//  * The NF4 table lives in shared memory (the paper's idea, A1): 16 fp32
//    words in 16 distinct banks, so the per-element lookup is conflict-free
//    for any code pattern.  Branch-free shift/mask indexing.
//  * Bit-exactness: __fmul_rn / __fadd_rn (never contracted to FMA), RNE
//    cvt.rn.{f16x2,bf16x2}.f32, no FTZ (the library is built without
//    --use_fast_math).  Identical bytes for any grid size and alignment.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <mutex>

#include "nf4_internal.cuh"

namespace nf4 {

constexpr int kThreads = 256;           // 8 warps per CTA
constexpr int kGroup = 16;              // elements per thread-group (8 code bytes, 32 B out)
constexpr int kUnroll = 4;              // groups per thread per tile
constexpr int64_t kTile = int64_t(kThreads) * kGroup * kUnroll;  // 16384 elements

struct TensorDesc {
  const uint8_t* packed;
  const float* absmax;    // fp32 mode when non-null
  const uint8_t* qabsmax; // DQ mode otherwise
  const float* code2;
  const float* absmax2;
  uint16_t* out;
  int64_t n;
  int64_t tile_end;       // exclusive prefix of tiles over the batch
  float offset;
  int32_t bs_shift;       // log2(blocksize)
  int32_t vec_ok;         // packed 8-B aligned and out 32-B aligned
  int32_t pad_;
};

struct BatchParams {
  int64_t total_tiles;
  int32_t count;
  int32_t pad_;
  TensorDesc t[NF4_MAX_BATCH];
};

// Per-block absmax decode (A4).  fp32: absmax[b].  DQ (R7):
// fl32(fl32(code2[q] * absmax2[b >> 8]) + offset), two roundings, no FMA.
__device__ __forceinline__ float block_scale(const TensorDesc& d, int64_t b) {
  if (d.absmax != nullptr) return __ldg(d.absmax + b);
  const uint32_t q = __ldg(d.qabsmax + b);
  const float c = __ldg(d.code2 + q);
  const float s2 = __ldg(d.absmax2 + (b >> 8));
  return __fadd_rn(__fmul_rn(c, s2), d.offset);
}

// 16 elements from 8 code bytes: element 2j <- high nibble of byte j.
template <bool BF16>
__device__ __forceinline__ void decode16(const float* lut, uint2 q, float a, uint32_t (&w)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t word = j < 4 ? q.x : q.y;
    const uint32_t byte = (word >> (8 * (j & 3))) & 0xFFu;
    const float ph = __fmul_rn(lut[byte >> 4], a);    // element 2j
    const float pl = __fmul_rn(lut[byte & 0x0Fu], a); // element 2j+1
    w[j] = pack2_rn<BF16>(ph, pl);
  }
}

// Element-wise path for tails and unaligned tensors.
template <bool BF16>
__device__ __forceinline__ void slow_group(const TensorDesc& d, const float* lut, int64_t e0) {
  const int64_t e1 = e0 + kGroup < d.n ? e0 + kGroup : d.n;
  if (e0 >= e1) return;
  const float a = block_scale(d, e0 >> d.bs_shift);  // 16 | blocksize: one block per group
  for (int64_t k = e0; k < e1; ++k) {
    const uint32_t byte = d.packed[k >> 1];
    const uint32_t idx = (k & 1) ? (byte & 0x0Fu) : (byte >> 4);
    d.out[k] = cvt1_rn<BF16>(__fmul_rn(lut[idx], a));
  }
}

template <bool BF16>
__global__ void __launch_bounds__(kThreads) dequant_kernel(const __grid_constant__ BatchParams P) {
  __shared__ float lut[16];
  if (threadIdx.x < 16) lut[threadIdx.x] = __uint_as_float(c_nf4_bits[threadIdx.x]);
  __syncthreads();

  int cur = 0;
  for (int64_t tile = blockIdx.x; tile < P.total_tiles; tile += gridDim.x) {
    while (tile >= P.t[cur].tile_end) ++cur;
    const TensorDesc& d = P.t[cur];
    const int64_t first = cur == 0 ? 0 : P.t[cur - 1].tile_end;
    const int64_t e_tile = (tile - first) * kTile;

    if (d.vec_ok && e_tile + kTile <= d.n) {
      uint2 q[kUnroll];
      float a[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e0 = e_tile + int64_t(u * kThreads + threadIdx.x) * kGroup;
        q[u] = ld_codes_v2(d.packed + (e0 >> 1));
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e0 = e_tile + int64_t(u * kThreads + threadIdx.x) * kGroup;
        a[u] = block_scale(d, e0 >> d.bs_shift);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e0 = e_tile + int64_t(u * kThreads + threadIdx.x) * kGroup;
        uint32_t w[8];
        decode16<BF16>(lut, q[u], a[u], w);
        st_out_v8(d.out + e0, w);
      }
    } else {
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e0 = e_tile + int64_t(u * kThreads + threadIdx.x) * kGroup;
        if (e0 >= d.n) break;
        if (d.vec_ok && e0 + kGroup <= d.n) {
          uint32_t w[8];
          decode16<BF16>(lut, ld_codes_v2(d.packed + (e0 >> 1)), block_scale(d, e0 >> d.bs_shift), w);
          st_out_v8(d.out + e0, w);
        } else {
          slow_group<BF16>(d, lut, e0);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static int occupancy(bool bf16) {
  static std::mutex mu;
  static int cache[2] = {0, 0};
  std::lock_guard<std::mutex> g(mu);
  int& c = cache[bf16 ? 1 : 0];
  if (c == 0) {
    int v = 0;
    cudaError_t e = bf16 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, dequant_kernel<true>, kThreads, 0)
                         : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, dequant_kernel<false>, kThreads, 0);
    c = (e == cudaSuccess && v > 0) ? v : 4;
  }
  return c;
}

static int grid_for(int64_t tiles, bool bf16) {
  int64_t g = int64_t(sm_count()) * occupancy(bf16);
  const int32_t cap = max_ctas();
  if (cap > 0 && g > cap) g = cap;
  if (g > tiles) g = tiles;
  return int(g < 1 ? 1 : g);
}

static nf4_status validate(const nf4_tensor& t, bool* has_work) {
  *has_work = false;
  if (t.n < 0) return NF4_ERR_BAD_SIZE;
  if (t.reserved != 0) return NF4_ERR_BAD_STATE;
  if (!is_pow2(t.blocksize) || t.blocksize < 64 || t.blocksize > 4096) return NF4_ERR_BAD_BLOCKSIZE;
  const bool dq = t.absmax == nullptr;
  if (dq) {
    if (t.dq.qabsmax == nullptr && t.n > 0) return NF4_ERR_BAD_STATE;
    if (t.dq.blocksize2 != 256) return NF4_ERR_BAD_STATE;
  } else if (t.dq.qabsmax != nullptr) {
    return NF4_ERR_BAD_STATE;
  }
  if (t.n == 0) return NF4_OK;
  if (t.packed == nullptr || t.out == nullptr) return NF4_ERR_NULL_POINTER;
  if (dq && (t.dq.code2 == nullptr || t.dq.absmax2 == nullptr)) return NF4_ERR_NULL_POINTER;
  if (!aligned(t.out, 2)) return NF4_ERR_MISALIGNED;
  if (!dq && !aligned(t.absmax, 4)) return NF4_ERR_MISALIGNED;
  if (dq && (!aligned(t.dq.code2, 4) || !aligned(t.dq.absmax2, 4))) return NF4_ERR_MISALIGNED;
  *has_work = true;
  return NF4_OK;
}

static nf4_status launch_batch(const nf4_tensor* ts, int count, bool bf16, cudaStream_t stream,
                               int32_t* launches) {
  BatchParams P;
  P.count = 0;
  P.pad_ = 0;
  int64_t tiles = 0;
  for (int i = 0; i < count; ++i) {
    const nf4_tensor& t = ts[i];
    if (t.n == 0) continue;
    TensorDesc& d = P.t[P.count++];
    d.packed = t.packed;
    d.absmax = t.absmax;
    d.qabsmax = t.absmax ? nullptr : t.dq.qabsmax;
    d.code2 = t.absmax ? nullptr : t.dq.code2;
    d.absmax2 = t.absmax ? nullptr : t.dq.absmax2;
    d.offset = t.absmax ? 0.0f : t.dq.offset;
    d.out = static_cast<uint16_t*>(t.out);
    d.n = t.n;
    d.bs_shift = log2i(t.blocksize);
    d.vec_ok = aligned(t.packed, 8) && aligned(t.out, 32);
    d.pad_ = 0;
    tiles += (t.n + kTile - 1) / kTile;
    d.tile_end = tiles;
  }
  if (P.count == 0) return NF4_OK;
  P.total_tiles = tiles;
  const int grid = grid_for(tiles, bf16);
  if (bf16)
    dequant_kernel<true><<<grid, kThreads, 0, stream>>>(P);
  else
    dequant_kernel<false><<<grid, kThreads, 0, stream>>>(P);
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return NF4_ERR_CUDA;
  }
  ++*launches;
  return NF4_OK;
}

}  // namespace nf4

using namespace nf4;

extern "C" nf4_status nf4_dequantize_batched(const nf4_tensor* tensors, int32_t count, nf4_dtype out_dtype,
                                             void* stream) {
  if (count < 0) return NF4_ERR_BAD_SIZE;
  if (count > 0 && tensors == nullptr) return NF4_ERR_NULL_POINTER;
  if (out_dtype != NF4_F16 && out_dtype != NF4_BF16) return NF4_ERR_BAD_DTYPE;
  for (int i = 0; i < count; ++i) {
    bool w;
    const nf4_status s = validate(tensors[i], &w);
    if (s != NF4_OK) return s;
  }
  int32_t launches = 0;
  // Group tensors with work into launches of at most NF4_MAX_BATCH.
  nf4_tensor buf[NF4_MAX_BATCH];
  int nbuf = 0;
  for (int i = 0; i < count; ++i) {
    if (tensors[i].n == 0) continue;
    buf[nbuf++] = tensors[i];
    if (nbuf == NF4_MAX_BATCH) {
      const nf4_status s = launch_batch(buf, nbuf, out_dtype == NF4_BF16, (cudaStream_t)stream, &launches);
      if (s != NF4_OK) return s;
      nbuf = 0;
    }
  }
  if (nbuf > 0) {
    const nf4_status s = launch_batch(buf, nbuf, out_dtype == NF4_BF16, (cudaStream_t)stream, &launches);
    if (s != NF4_OK) return s;
  }
  set_launch_count(launches);
  return NF4_OK;
}

extern "C" nf4_status nf4_dequantize(const uint8_t* packed, const float* absmax, const nf4_dq_state* dq,
                                     int64_t n, int32_t blocksize, nf4_dtype out_dtype, void* out,
                                     void* stream) {
  if ((absmax == nullptr) == (dq == nullptr)) return NF4_ERR_BAD_STATE;
  nf4_tensor t;
  t.packed = packed;
  t.absmax = absmax;
  if (dq) {
    t.dq = *dq;
  } else {
    t.dq.qabsmax = nullptr;
    t.dq.code2 = nullptr;
    t.dq.absmax2 = nullptr;
    t.dq.offset = 0.0f;
    t.dq.blocksize2 = 256;
  }
  if (dq && dq->qabsmax == nullptr && n > 0) return NF4_ERR_NULL_POINTER;
  t.n = n;
  t.blocksize = blocksize;
  t.reserved = 0;
  t.out = out;
  return nf4_dequantize_batched(&t, 1, out_dtype, stream);
}

extern "C" void nf4_codebook(float out16[16]) {
  for (int i = 0; i < 16; ++i) {
    float f;
    memcpy(&f, &h_nf4_bits[i], 4);
    out16[i] = f;
  }
}

extern "C" int32_t nf4_dequant_grid(int64_t tiles) { return grid_for(tiles < 1 ? 1 : tiles, false); }
extern "C" int64_t nf4_dequant_tile_elems(void) { return kTile; }
