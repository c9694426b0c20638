// nf4_quantize.cu -- GPU NF4 quantization and double quantization (SURVEY
// row F2): the step BEFORE the hot path, used to generate realistic inputs.
// Bit-exact with the CPU oracle's quantizer (tests/test_parity_gpu.py).
//
// nf4_quantize (R12): one warp per quantization block.
//   absmax = max|x| (exact, warp shuffle max);  r = fl32(1/absmax) (__frcp_rn);
//   xn = fl32(x * r);  idx = #{i : xn > t_i}, t_i = fl32 midpoint of adjacent
//   codes (computed in fp64 in-kernel);  absmax == 0 -> idx 7.
// nf4_double_quantize (R13): one CTA of 256 threads per second-level group.
//   d = fl32(a - offset); s2 = max|d|; dn = fl32(d * fl32(1/s2)) (0 if s2 == 0);
//   q = argmin_i fl32|dn - code2[i]|, ties -> lowest i: binary search on a
//   strictly increasing code2 (checked per CTA) + leftward tie scan, else a
//   256-way brute force.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "nf4_internal.cuh"

namespace nf4 {

template <int IN>
__device__ __forceinline__ float2 load_pair(const void* in, int64_t k, int64_t n) {
  // elements k, k+1 (k even); missing k+1 (odd tail) -> 0 (not used)
  float2 r;
  if (IN == NF4_F32) {
    const float* p = static_cast<const float*>(in);
    if (k + 1 < n) {
      r = *reinterpret_cast<const float2*>(p + k);
    } else {
      r.x = p[k];
      r.y = 0.0f;
    }
  } else {
    const uint16_t* p = static_cast<const uint16_t*>(in);
    uint16_t a = p[k];
    uint16_t b = (k + 1 < n) ? p[k + 1] : uint16_t(0);
    if (IN == NF4_F16) {
      r.x = __half2float(__ushort_as_half(a));
      r.y = __half2float(__ushort_as_half(b));
    } else {
      r.x = __bfloat162float(__ushort_as_bfloat16(a));
      r.y = __bfloat162float(__ushort_as_bfloat16(b));
    }
  }
  return r;
}

__device__ __forceinline__ uint32_t nf4_index(float xn, const float* thr) {
  uint32_t idx = 0;
#pragma unroll
  for (int i = 0; i < 15; ++i) idx += (xn > thr[i]) ? 1u : 0u;
  return idx;
}

template <int IN>
__global__ void __launch_bounds__(256) quantize_kernel(const void* __restrict__ in, int64_t n, int bs_shift,
                                                       uint8_t* __restrict__ packed, float* __restrict__ absmax) {
  __shared__ float thr[15];
  if (threadIdx.x < 15) {
    const double lo = double(__uint_as_float(c_nf4_bits[threadIdx.x]));
    const double hi = double(__uint_as_float(c_nf4_bits[threadIdx.x + 1]));
    thr[threadIdx.x] = float((lo + hi) / 2.0);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t bs = int64_t(1) << bs_shift;
  const int64_t nb = (n + bs - 1) >> bs_shift;
  const int pairs = int(bs >> 1);
  for (int64_t b = warp; b < nb; b += nwarps) {
    const int64_t k0 = b << bs_shift;
    float m = 0.0f;
    for (int p = lane; p < pairs; p += 32) {
      const int64_t k = k0 + 2 * p;
      if (k < n) {
        const float2 v = load_pair<IN>(in, k, n);
        m = fmaxf(m, fabsf(v.x));
        if (k + 1 < n) m = fmaxf(m, fabsf(v.y));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float r = (m == 0.0f) ? 0.0f : __frcp_rn(m);
    for (int p = lane; p < pairs; p += 32) {
      const int64_t k = k0 + 2 * p;
      if (k < n) {
        const float2 v = load_pair<IN>(in, k, n);
        uint32_t hi, lo = 0;
        if (m == 0.0f) {
          hi = 7;
          if (k + 1 < n) lo = 7;
        } else {
          hi = nf4_index(__fmul_rn(v.x, r), thr);
          if (k + 1 < n) lo = nf4_index(__fmul_rn(v.y, r), thr);
        }
        packed[k >> 1] = uint8_t((hi << 4) | lo);
      }
    }
    if (lane == 0) absmax[b] = m;
  }
}

__global__ void __launch_bounds__(256) double_quantize_kernel(const float* __restrict__ absmax, int64_t nb,
                                                              float offset, const float* __restrict__ code2,
                                                              uint8_t* __restrict__ qabsmax,
                                                              float* __restrict__ absmax2) {
  __shared__ float c[256];
  __shared__ float red[8];
  c[threadIdx.x] = code2[threadIdx.x];
  __syncthreads();
  const int sorted = __syncthreads_and(threadIdx.x == 0 || c[threadIdx.x - 1] < c[threadIdx.x]);
  const int64_t ng = (nb + 255) >> 8;
  for (int64_t g = blockIdx.x; g < ng; g += gridDim.x) {
    const int64_t b = (g << 8) + threadIdx.x;
    const bool valid = b < nb;
    const float d = valid ? __fsub_rn(absmax[b], offset) : 0.0f;
    float m = valid ? fabsf(d) : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = red[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i]);
    __syncthreads();
    if (valid) {
      const float dn = (m == 0.0f) ? 0.0f : __fmul_rn(d, __frcp_rn(m));
      int best;
      if (sorted) {
        int lo = 0, hi = 256;  // first index with c[idx] >= dn
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (c[mid] < dn) lo = mid + 1; else hi = mid;
        }
        int cand0 = lo > 0 ? lo - 1 : 0;
        int cand1 = lo < 256 ? lo : 255;
        const float d0 = fabsf(__fsub_rn(dn, c[cand0]));
        const float d1 = fabsf(__fsub_rn(dn, c[cand1]));
        best = (d1 < d0) ? cand1 : cand0;
        const float bd = (d1 < d0) ? d1 : d0;
        while (best > 0 && fabsf(__fsub_rn(dn, c[best - 1])) == bd) --best;
      } else {
        best = 0;
        float bd = fabsf(__fsub_rn(dn, c[0]));
        for (int i = 1; i < 256; ++i) {
          const float di = fabsf(__fsub_rn(dn, c[i]));
          if (di < bd) { bd = di; best = i; }
        }
      }
      qabsmax[b] = uint8_t(best);
    }
    if (threadIdx.x == 0) absmax2[g] = m;
  }
}

}  // namespace nf4

using namespace nf4;

extern "C" nf4_status nf4_quantize(const void* in, nf4_dtype in_dtype, int64_t n, int32_t blocksize,
                                   uint8_t* packed, float* absmax, void* stream) {
  if (n < 0) return NF4_ERR_BAD_SIZE;
  if (!is_pow2(blocksize) || blocksize < 64 || blocksize > 4096) return NF4_ERR_BAD_BLOCKSIZE;
  if (in_dtype != NF4_F32 && in_dtype != NF4_F16 && in_dtype != NF4_BF16) return NF4_ERR_BAD_DTYPE;
  if (n == 0) { set_launch_count(0); return NF4_OK; }
  if (!in || !packed || !absmax) return NF4_ERR_NULL_POINTER;
  if (!aligned(in, in_dtype == NF4_F32 ? 8 : 2) || !aligned(absmax, 4)) return NF4_ERR_MISALIGNED;
  const int shift = log2i(blocksize);
  const int64_t nb = (n + blocksize - 1) / blocksize;
  int64_t grid = (nb + 7) / 8;
  const int64_t cap = int64_t(sm_count()) * 8;
  if (grid > cap) grid = cap;
  cudaStream_t s = (cudaStream_t)stream;
  if (in_dtype == NF4_F32) quantize_kernel<NF4_F32><<<int(grid), 256, 0, s>>>(in, n, shift, packed, absmax);
  else if (in_dtype == NF4_F16) quantize_kernel<NF4_F16><<<int(grid), 256, 0, s>>>(in, n, shift, packed, absmax);
  else quantize_kernel<NF4_BF16><<<int(grid), 256, 0, s>>>(in, n, shift, packed, absmax);
  if (cudaPeekAtLastError() != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
  set_launch_count(1);
  return NF4_OK;
}

extern "C" nf4_status nf4_double_quantize(const float* absmax, int64_t nb, float offset, const float* code2,
                                          int32_t blocksize2, uint8_t* qabsmax, float* absmax2, void* stream) {
  if (nb < 0) return NF4_ERR_BAD_SIZE;
  if (blocksize2 != 256) return NF4_ERR_BAD_STATE;
  if (nb == 0) { set_launch_count(0); return NF4_OK; }
  if (!absmax || !code2 || !qabsmax || !absmax2) return NF4_ERR_NULL_POINTER;
  if (!aligned(absmax, 4) || !aligned(code2, 4) || !aligned(absmax2, 4)) return NF4_ERR_MISALIGNED;
  int64_t grid = (nb + 255) / 256;
  const int64_t cap = int64_t(sm_count()) * 8;
  if (grid > cap) grid = cap;
  double_quantize_kernel<<<int(grid), 256, 0, (cudaStream_t)stream>>>(absmax, nb, offset, code2, qabsmax, absmax2);
  if (cudaPeekAtLastError() != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
  set_launch_count(1);
  return NF4_OK;
}
