// nf4_internal.cuh -- shared internals of libnf4 (product side only; the CPU
// oracle under oracle/ shares nothing with this directory).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nf4.h"
#include "../../include/nf4_tools.h"

namespace nf4 {

// Per-thread count of kernels enqueued by the last successful API call.
void set_launch_count(int32_t n);

// SM count of the current device (cached per device).
int sm_count();

// Process-wide cap on persistent grids (0 = auto).
int32_t max_ctas();

inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
inline int log2i(int64_t v) { int s = 0; while ((int64_t(1) << s) < v) ++s; return s; }
inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

inline nf4_status cuda_status(cudaError_t e) { return e == cudaSuccess ? NF4_OK : NF4_ERR_CUDA; }

// The NF4 table (R1): QLoRA/BitsAndBytes levels, fp32 bit patterns.
// Index 7 is exact +0.0, indices 0 and 15 are exactly -1.0 and +1.0.
// (static: each translation unit holds its own constant-bank copy.)
static __constant__ uint32_t c_nf4_bits[16] = {
    0xbf800000u, 0xbf3239b1u, 0xbf066b30u, 0xbeca32a0u, 0xbe91a24du, 0xbe3d353fu,
    0xbdba7871u, 0x00000000u, 0x3da2faffu, 0x3e24cae3u, 0x3e7c04ddu, 0x3ead033au,
    0x3ee1a4b8u, 0x3f1007abu, 0x3f3913b3u, 0x3f800000u};
static const uint32_t h_nf4_bits[16] = {
    0xbf800000u, 0xbf3239b1u, 0xbf066b30u, 0xbeca32a0u, 0xbe91a24du, 0xbe3d353fu,
    0xbdba7871u, 0x00000000u, 0x3da2faffu, 0x3e24cae3u, 0x3e7c04ddu, 0x3ead033au,
    0x3ee1a4b8u, 0x3f1007abu, 0x3f3913b3u, 0x3f800000u};

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
// 64-bit streaming load of packed codes: read-only path, no L1 allocation.
__device__ __forceinline__ uint2 ld_codes_v2(const uint8_t* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// 256-bit streaming store (sm_100: STG.E.256), evict-first.
__device__ __forceinline__ void st_out_v8(void* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// 256-bit store with the default (write-back) cache policy.
__device__ __forceinline__ void st_out_v8_wb(void* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// Pack two fp32 into 16-bit pair with RNE.  `lo` lands in bits [0,16) -- the
// earlier element (high nibble, R2) -- and `hi` in bits [16,32).  PTX
// cvt.rn.{f16x2,bf16x2}.f32 d, a, b puts a in the upper half.
template <bool BF16>
__device__ __forceinline__ uint32_t pack2_rn(float lo, float hi) {
  uint32_t r;
  if (BF16)
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  else
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Two IEEE round-to-nearest fp32 products in one instruction (sm_100 FMUL2,
// PTX mul.rn.f32x2, no FTZ): x *= a, y *= a with `aa` = {a, a} packed.  Each lane
// is exactly __fmul_rn, so the result is bit-identical to two FMULs.
__device__ __forceinline__ uint64_t f32x2_splat(float a) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ void mul2_rn(float& x, float& y, uint64_t aa) {
  uint64_t v, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(x), "f"(y));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(v), "l"(aa));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}

template <bool BF16>
__device__ __forceinline__ uint16_t cvt1_rn(float x) {
  uint16_t r;
  if (BF16)
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(x));
  else
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(r) : "f"(x));
  return r;
}

}  // namespace nf4
