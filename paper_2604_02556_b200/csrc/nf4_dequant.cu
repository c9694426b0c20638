// nf4_dequant.cu -- B200 (sm_100a) blockwise NF4 -> FP16/BF16 (and FP32) dequantization.
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

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "nf4_internal.cuh"

namespace nf4 {

constexpr int kThreads = 256;  // 8 warps per CTA

// Kernel variants (A/B-able at run time through NF4_KERNEL_VARIANT or
// nf4_set_kernel_variant; all are bit-identical -- tests/test_parity_gpu.py).
//   vec     code bytes per thread-group: 8 (LDG.64, 16 elements, one STG.256)
//           or 16 (LDG.128, 32 elements, two STG.256 = 64 B thread-contiguous)
//   unroll  thread-groups per thread per tile (all loads issued first)
//   persist grid = SMs x resident CTAs striding over tiles, instead of one CTA
//           per tile (the block scheduler then keeps the DRAM working set of
//           concurrently running CTAs compact: +13% measured on B200)
//   sscale  the tile's block scales are decoded once per block into shared
//           memory (one thread per block) instead of once per thread-group
//   prmt    nibble -> LUT byte offset for 4 bytes at once with SHF+LOP3, then
//           one PRMT per element (1.5 instead of ~2.2 ALU ops per element)
//   clc     Blackwell cluster launch control: a running CTA cancels a not yet
//           launched CTA (clusterlaunchcontrol.try_cancel) and takes its tile,
//           so the prologue (LUT staging, descriptor search) is paid once per
//           CTA while tiles are still handed out in launch order
//   (d)     double-buffered scale cache and CLC response slots: one CTA barrier
//           per tile instead of three
struct Variant {
  const char* name;
  int vec, unroll;
  bool persist, sscale, prmt, clc;
  int threads = kThreads;   // CTA size
};
static const Variant kVariants[] = {
    {"v2u4", 8, 4, false, false, false, false},      // 0
    {"v4u2", 16, 2, false, false, false, false},     // 1
    {"v4u4", 16, 4, false, false, false, false},     // 2
    {"v2u4p", 8, 4, true, false, false, false},      // 3 (round-1 first version)
    {"v4u1", 16, 1, false, false, false, false},     // 4
    {"v2u8", 8, 8, false, false, false, false},      // 5
    {"v2u4s", 8, 4, false, true, false, false},      // 6
    {"v2u4sx", 8, 4, false, true, true, false},      // 7
    {"v2u4sxc", 8, 4, false, true, true, true},      // 8
    {"v2u4c", 8, 4, false, false, false, true},      // 9
    {"v2u4xc", 8, 4, false, false, true, true},      // 10
    {"v2u4sxcd", 8, 4, false, true, true, true},     // 11: + double-buffered scale cache / CLC slots
    {"v2u4sxcp", 8, 4, false, true, true, true},     // 12: v2u4sxc + byte-pair table (32 KB smem per CTA)
    {"v2u2sxc", 8, 2, false, true, true, true},      // 13: v2u4sxc with 8192-element tiles
    {"v2u4sxcw", 8, 4, false, true, true, true},     // 14: v2u4sxc with write-back (default-policy) stores
    {"v2u4sxcf", 8, 4, false, true, true, true},     // 15: v2u4sxc + L2 prefetch of the scales one wave ahead
    {"v2u4sxcF", 8, 4, false, true, true, true},     // 16: v2u4sxc + L2 prefetch of scales and codes one wave ahead
    {"v2u4r2sxc", 8, 8, false, true, true, true},    // 17: 32768-element tiles done as 2 rounds of v2u4sxc's
                                                     //     loads/stores (per-tile scale decode, barriers, CLC halved)
    {"v2u4sxcp512", 8, 4, false, true, true, true, 512},  // 18: the byte-pair table (v2u4sxcp) in 512-thread CTAs:
                                                          //     4 x 32 KB tables per SM, full occupancy
    {"v2u4sxc512", 8, 4, false, true, true, true, 512},   // 19: the default kernel in 512-thread CTAs
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
constexpr int kDefaultVariant = 8;   // v2u4sxc: best measured on B200 (profiles/r01_variants.md)
// Launches of fewer than kQuarterTileWaves x SMs default-size tiles take 4096-element tiles.
#ifndef NF4_QUARTER_TILE_WAVES
#define NF4_QUARTER_TILE_WAVES 4
#endif
constexpr int kQuarterTileWaves = NF4_QUARTER_TILE_WAVES;
constexpr int kMaxTileBlocks = 512;  // TILE / 64 for the largest (32768-element) tiles using sscale

struct TensorDesc {
  const uint8_t* packed;
  const float* absmax;    // fp32 mode when non-null
  const uint8_t* qabsmax; // DQ mode otherwise
  const float* code2;
  const float* absmax2;
  void* out;              // uint16 words (fp16/bf16) or fp32
  int64_t n;
  int64_t tile_end;       // exclusive prefix of tiles over the batch
  float offset;
  int32_t bs_shift;       // log2(blocksize)
  int32_t vec_ok;         // packed VEC-B aligned and out 32-B aligned
  int32_t pad_;
};

// Kernel parameters (passed by value, __grid_constant__).  MAXB sizes the
// descriptor array: 1 and 16 keep single-tensor / per-layer launches light
// (the parameter block is copied at every launch), 128 is the batched maximum.
template <int MAXB>
struct BatchParamsT {
  int64_t total_tiles;
  int32_t count;
  int32_t prefetch_ahead; // PF variants: L2-prefetch the inputs of tile + prefetch_ahead (0: off)
  int32_t early_inputs;   // 1: read codes and scales before griddepcontrol.wait (nf4_set_early_input_reads)
  int32_t pad2_;
  float lut[16];          // the 16-entry codebook (NF4 unless nf4_dequantize_ex supplies one)
  TensorDesc t[MAXB];
};
using BatchParams = BatchParamsT<NF4_MAX_BATCH>;

// Per-block absmax decode (A4).  fp32: absmax[b].  DQ (R7):
// fl32(fl32(code2[q] * absmax2[b >> 8]) + offset), two roundings, no FMA.
__device__ __forceinline__ float block_scale(const TensorDesc& d, int64_t b) {
  if (d.absmax != nullptr) return __ldg(d.absmax + b);
  const uint32_t q = __ldg(d.qabsmax + b);
  const float c = __ldg(d.code2 + q);
  const float s2 = __ldg(d.absmax2 + (b >> 8));
  return __fadd_rn(__fmul_rn(c, s2), d.offset);
}

template <int VEC>
struct CodeVec {
  uint32_t w[VEC / 4];
};

template <int VEC>
__device__ __forceinline__ CodeVec<VEC> ld_codes(const uint8_t* p) {
  CodeVec<VEC> r;
  if constexpr (VEC == 8) {
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.w[0]), "=r"(r.w[1]) : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
        : "l"(p));
  }
  return r;
}

__device__ __forceinline__ float lut_at(const float* lut, uint32_t byte_off) {
  return *reinterpret_cast<const float*>(reinterpret_cast<const char*>(lut) + byte_off);
}

// 2*VEC elements from VEC code bytes: element 2j <- high nibble of byte j
// (P:160-161), product fl32(NF4[idx] * a), RNE to 16 bits;
// word j holds elements (2j, 2j+1) with 2j in the low half.
// Output words per thread-group: VEC 32-bit words (two 16-bit results each),
// or 2*VEC words for fp32 output.
template <int OUT, int VEC>
struct OutWords {
  static constexpr int value = OUT == 2 ? 2 * VEC : VEC;
};

// Store the products of elements (2j, 2j+1) as output word(s) j.
template <int OUT, int VEC>
__device__ __forceinline__ void put_pair(uint32_t (&w)[OutWords<OUT, VEC>::value], int j, float ph, float pl) {
  if constexpr (OUT == 2) {
    w[2 * j] = __float_as_uint(ph);
    w[2 * j + 1] = __float_as_uint(pl);
  } else {
    w[j] = pack2_rn<OUT == 1>(ph, pl);
  }
}

template <int OUT, int VEC, bool PRMT>
__device__ __forceinline__ void decode_group(const float* lut, const CodeVec<VEC>& q, float a,
                                             uint32_t (&w)[OutWords<OUT, VEC>::value]) {
  if constexpr (PRMT) {
    const uint64_t aa = f32x2_splat(a);
#pragma unroll
    for (int i = 0; i < VEC / 4; ++i) {
      const uint32_t x = q.w[i];
      const uint32_t hi4 = (x >> 2) & 0x3C3C3C3Cu;  // byte k = 4 * (high nibble of byte k)
      const uint32_t lo4 = (x << 2) & 0x3C3C3C3Cu;  // byte k = 4 * (low nibble of byte k)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t oh = k == 0 ? (hi4 & 0xFFu) : k == 3 ? (hi4 >> 24) : __byte_perm(hi4, 0u, 0x4440u + k);
        const uint32_t ol = k == 0 ? (lo4 & 0xFFu) : k == 3 ? (lo4 >> 24) : __byte_perm(lo4, 0u, 0x4440u + k);
        float ph = lut_at(lut, oh), pl = lut_at(lut, ol);  // elements 2j, 2j+1
        mul2_rn(ph, pl, aa);                               // fl32(NF4[idx] * a), one FMUL2
        put_pair<OUT, VEC>(w, 4 * i + k, ph, pl);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const uint32_t byte = (q.w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
      const float ph = __fmul_rn(lut[byte >> 4], a);     // element 2j
      const float pl = __fmul_rn(lut[byte & 0x0Fu], a);  // element 2j+1
      put_pair<OUT, VEC>(w, j, ph, pl);
    }
  }
}

// Byte-pair table (variant 12): entry b = (NF4[b >> 4], NF4[b & 15]), one copy per
// half-warp lane (row b = 128 B = 16 copies), so a 64-bit lookup per code BYTE is
// bank-conflict-free for any codes: per two elements one PRMT (byte extract), one
// IMAD (row address), one LDS.64, one FMUL2 and one F2FP (same numbers as decode_group).
constexpr int kPairRow = 128;
constexpr int kPairBytes = 256 * kPairRow;
template <int OUT, int VEC>
__device__ __forceinline__ void decode_group_pair(uint32_t ptab_lane, const CodeVec<VEC>& q, float a,
                                                  uint32_t (&w)[OutWords<OUT, VEC>::value]) {
  const uint64_t aa = f32x2_splat(a);
#pragma unroll
  for (int i = 0; i < VEC / 4; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t byte = __byte_perm(q.w[i], 0u, 0x4440u + k);
      uint64_t v, r;
      asm("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(ptab_lane + byte * kPairRow));
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(v), "l"(aa));   // fl32(NF4[idx] * a), both elements
      float ph, pl;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(ph), "=f"(pl) : "l"(r));
      put_pair<OUT, VEC>(w, 4 * i + k, ph, pl);
    }
  }
}

// STH 0: evict-first streaming stores (.cs); 1: default write-back policy
template <int NW, int STH = 0>
__device__ __forceinline__ void st_group(void* out, const uint32_t (&w)[NW]) {
#pragma unroll
  for (int h = 0; h < NW / 8; ++h) {
    const uint32_t(&ww)[8] = *reinterpret_cast<const uint32_t(*)[8]>(&w[8 * h]);
    if constexpr (STH == 0) st_out_v8(static_cast<uint8_t*>(out) + 32 * h, ww);
    else st_out_v8_wb(static_cast<uint8_t*>(out) + 32 * h, ww);
  }
}

template <int OUT>
__device__ __forceinline__ void* out_at(const void* out, int64_t k) {
  return const_cast<uint8_t*>(static_cast<const uint8_t*>(out)) + (OUT == 2 ? 4 : 2) * k;
}

// Element-wise path for tails and unaligned tensors.
template <int OUT, int GROUP>
__device__ __forceinline__ void slow_group(const TensorDesc& d, const float* lut, int64_t e0, float a) {
  const int64_t e1 = e0 + GROUP < d.n ? e0 + GROUP : d.n;
  for (int64_t k = e0; k < e1; ++k) {
    const uint32_t byte = d.packed[k >> 1];
    const uint32_t idx = (k & 1) ? (byte & 0x0Fu) : (byte >> 4);
    const float p = __fmul_rn(lut[idx], a);
    if constexpr (OUT == 2)
      static_cast<float*>(d.out)[k] = p;
    else
      static_cast<uint16_t*>(d.out)[k] = cvt1_rn<OUT == 1>(p);
  }
}

// --- cluster launch control (sm_100) ---------------------------------------
__device__ __forceinline__ void clc_try_cancel(void* result, uint64_t* bar) {
  const uint32_t r = static_cast<uint32_t>(__cvta_generic_to_shared(result));
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("fence.proxy.async::generic.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
  asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
               ::"r"(r), "r"(b) : "memory");
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], 16;" ::"r"(b) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(b), "r"(phase), "r"(0x989680) : "memory");
  }
}

// Returns the canceled CTA's blockIdx.x, or -1 if no CTA was canceled.
__device__ __forceinline__ int64_t clc_result(const uint4* result) {
  const volatile uint32_t* rv = reinterpret_cast<const volatile uint32_t*>(result);
  const uint4 r = make_uint4(rv[0], rv[1], rv[2], rv[3]);
  uint32_t ok, x;
  asm volatile(
      "{\n\t.reg .b128 h;\n\t.reg .pred p;\n\t"
      "mov.b128 h, {%2, %3};\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, h;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t"
      "clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, h;\n\t}"
      : "=r"(ok), "=r"(x)
      : "l"((uint64_t(r.y) << 32) | r.x), "l"((uint64_t(r.w) << 32) | r.z));
  asm volatile("fence.proxy.async::generic.release.sync_restrict::shared::cta.cluster;" ::: "memory");
  return ok ? int64_t(x) : -1;
}

template <int OUT, int VEC, int U, bool PERSIST, bool SSCALE, bool PRMT, bool CLC, bool DB = false,
          int MAXB = NF4_MAX_BATCH, bool EARLY = false, bool PAIR = false, int STH = 0, int PF = 0, int R = 1,
          int NT = kThreads>
__global__ void __launch_bounds__(NT) dequant_kernel(const __grid_constant__ BatchParamsT<MAXB> P) {
  constexpr int GROUP = 2 * VEC;                      // elements per thread-group
  constexpr int64_t SUBTILE = int64_t(NT) * GROUP * U;   // one round of loads / stores
  constexpr int64_t TILE = SUBTILE * R;                        // R rounds share one scale decode
  constexpr int NBUF = DB ? 2 : 1;                    // scale cache / CLC response slots
  static_assert(!SSCALE || TILE / 64 <= kMaxTileBlocks, "tile too large for the scale cache");
  static_assert(!DB || (SSCALE && CLC), "double buffering needs the per-tile barrier of sscale");
  // A1: stage the 16-entry table in shared memory (16 banks, conflict-free).
  __shared__ float lut[16];
  __shared__ float sscale[NBUF][SSCALE ? int(TILE / 64) : 1];
  __shared__ __align__(16) uint4 clc_res[NBUF];
  __shared__ __align__(8) uint64_t clc_bar[NBUF];
  if (threadIdx.x < 16) lut[threadIdx.x] = P.lut[threadIdx.x];  // kernel-parameter (constant) bank -> smem
  extern __shared__ __align__(128) uint8_t ptab[];                // PAIR: kPairBytes of dynamic smem
  if constexpr (PAIR) {
    for (int i = threadIdx.x; i < 256 * (kPairRow / 16); i += NT) {
      const int b = i / (kPairRow / 16);
      const float h = P.lut[b >> 4], l = P.lut[b & 15];
      *reinterpret_cast<float4*>(ptab + 16 * i) = make_float4(h, l, h, l);
    }
  }
  const uint32_t ptab_lane =
      static_cast<uint32_t>(__cvta_generic_to_shared(ptab)) + (threadIdx.x & 15u) * 8u;
  if (CLC && threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&clc_bar[i]))) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Programmatic dependent launch: the prologue above touches only parameters and
  // shared memory, so it may overlap the previous kernel's tail; inputs and the
  // output buffer are touched only after the previous grid has completed.
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // early_inputs: the inputs (codes, scales, tables) are read before the previous
  // kernel on the stream has completed -- its DRAM round trip overlaps that kernel's
  // tail -- and only the stores wait (griddepcontrol.wait before every tile's first
  // store; a no-op once satisfied).  The caller guarantees the previous kernel does not
  // write this launch's inputs (include/nf4.h).
  if (!P.early_inputs) asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();

  int cur = 0;
  uint32_t it = 0;           // tiles processed by this CTA (scale-cache slot)
  uint32_t ci = 0;           // CTA ids processed by this CTA (CLC slot / phase)
  int64_t cta = blockIdx.x;  // CTA id whose tiles we process (own, then stolen ones)
  while (true) {
    const int cs = DB ? int(ci & 1) : 0;
    // Safe to overwrite clc_res[cs]: with DB every thread read it two CTA ids ago
    // and has since passed the per-tile barrier; without DB, the barrier below.
    if (CLC && threadIdx.x == 0) clc_try_cancel(&clc_res[cs], &clc_bar[cs]);
    for (int64_t tile = cta; tile < P.total_tiles; tile += gridDim.x, ++it) {
      if (PERSIST || CLC) {  // tiles arrive (mostly) in increasing order: walk a cursor
        while (tile >= P.t[cur].tile_end) ++cur;
        while (cur > 0 && tile < P.t[cur - 1].tile_end) --cur;
      } else {  // first tensor whose tile range contains `tile` (binary search, <= 7 steps)
        int lo = 0, hi = P.count - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (tile < P.t[mid].tile_end) hi = mid; else lo = mid + 1;
        }
        cur = lo;
      }
      const TensorDesc& d = P.t[cur];
      const int64_t first = cur == 0 ? 0 : P.t[cur - 1].tile_end;
      const int64_t e_tile = (tile - first) * TILE;
      if (PF > 0 && P.prefetch_ahead > 0 && threadIdx.x >= 32 && threadIdx.x < 32 + (PF > 1 ? 64 : 1)) {
        // L2 prefetch of the inputs of the tile about one resident wave ahead (warp 1;
        // thread 0 issues the CLC request): its block scales (one thread, 128-B lines)
        // and, PF > 1, its codes (64 threads x one 128-B line)
        const int64_t pt = tile + P.prefetch_ahead;
        if (pt < P.total_tiles) {
          int lo = cur, hi = P.count - 1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (pt < P.t[mid].tile_end) hi = mid; else lo = mid + 1;
          }
          const TensorDesc& pd = P.t[lo];
          const int64_t pe = (pt - (lo == 0 ? 0 : P.t[lo - 1].tile_end)) * TILE;
          if (threadIdx.x == 32) {
            const int64_t b0 = pe >> pd.bs_shift;
            const int64_t nb = (pd.n + (int64_t(1) << pd.bs_shift) - 1) >> pd.bs_shift;
            const int64_t b1 = min(nb, b0 + ((TILE - 1) >> pd.bs_shift) + 1);
            const char* a = pd.absmax ? reinterpret_cast<const char*>(pd.absmax + b0)
                                      : reinterpret_cast<const char*>(pd.qabsmax + b0);
            const int64_t bytes = (b1 - b0) * (pd.absmax ? 4 : 1);
            for (int64_t o = 0; o < bytes; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + o));
          } else if (PF > 1) {
            const int64_t ce = pe + int64_t(threadIdx.x - 32) * 256;   // 128 B of codes = 256 elements
            if (ce < pd.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(pd.packed + (ce >> 1)));
          }
        }
      }
      const bool full = d.vec_ok && e_tile + TILE <= d.n;
      float* ss = sscale[DB ? (it & 1) : 0];
      // EARLY (small launches, ~one wave of tiles): code loads first -- they do not
      // depend on the scales, so their DRAM round trip overlaps the scale decode and
      // its barrier (one latency per tile, not two; -1 us on a 2^20-element tensor).
      // Large launches keep the loads after the barrier (0.7% faster in steady state).
      CodeVec<VEC> q[U];
      if (EARLY && full) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t e0 = e_tile + int64_t(u * NT + threadIdx.x) * GROUP;
          q[u] = ld_codes<VEC>(d.packed + (e0 >> 1));
        }
      }

      if (SSCALE) {
        // A4 once per quantization block of this tile (one thread per block).
        // With DB this slot was last read two tiles ago, before the previous
        // tile's barrier, so one barrier per tile suffices.
        const int64_t b0 = e_tile >> d.bs_shift;
        const int64_t nb = (d.n + (int64_t(1) << d.bs_shift) - 1) >> d.bs_shift;
        const int nblk = int(((TILE - 1) >> d.bs_shift) + 1);
        if (R == 1) {
          if (int(threadIdx.x) < nblk && b0 + threadIdx.x < nb) ss[threadIdx.x] = block_scale(d, b0 + threadIdx.x);
        } else {
          for (int i = threadIdx.x; i < nblk && b0 + i < nb; i += NT) ss[i] = block_scale(d, b0 + i);
        }
        __syncthreads();
      }
      auto scale_of = [&](int64_t e0) -> float {
        return SSCALE ? ss[(e0 - e_tile) >> d.bs_shift] : block_scale(d, e0 >> d.bs_shift);
      };

      if (full) {
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int64_t e_sub = e_tile + r * SUBTILE;
          if (!EARLY || r > 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int64_t e0 = e_sub + int64_t(u * NT + threadIdx.x) * GROUP;
              q[u] = ld_codes<VEC>(d.packed + (e0 >> 1));
            }
          }
          float a[U];
#pragma unroll
          for (int u = 0; u < U; ++u) a[u] = scale_of(e_sub + int64_t(u * NT + threadIdx.x) * GROUP);
          if (P.early_inputs) asm volatile("griddepcontrol.wait;" ::: "memory");   // out may be in use
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t e0 = e_sub + int64_t(u * NT + threadIdx.x) * GROUP;
            uint32_t w[OutWords<OUT, VEC>::value];
            if constexpr (PAIR)
              decode_group_pair<OUT, VEC>(ptab_lane, q[u], a[u], w);
            else
              decode_group<OUT, VEC, PRMT>(lut, q[u], a[u], w);
            st_group<OutWords<OUT, VEC>::value, STH>(out_at<OUT>(d.out, e0), w);
          }
        }
      } else {
        if (P.early_inputs) asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int u = 0; u < U * R; ++u) {
          const int64_t e0 = e_tile + int64_t(u * NT + threadIdx.x) * GROUP;
          if (e0 >= d.n) break;
          const float a = scale_of(e0);  // GROUP | blocksize: one block per group
          if (d.vec_ok && e0 + GROUP <= d.n) {
            uint32_t w[OutWords<OUT, VEC>::value];
            decode_group<OUT, VEC, PRMT>(lut, ld_codes<VEC>(d.packed + (e0 >> 1)), a, w);
            st_group(out_at<OUT>(d.out, e0), w);
          } else {
            slow_group<OUT, GROUP>(d, lut, e0, a);
          }
        }
      }
      if (SSCALE && !DB) __syncthreads();  // sscale is rewritten for the next tile
    }
    if (!CLC) break;
    mbar_wait(&clc_bar[cs], DB ? ((ci >> 1) & 1) : (ci & 1));
    cta = clc_result(&clc_res[cs]);
    ++ci;
    if (!DB) __syncthreads();  // every thread has read clc_res before the next try_cancel
    if (cta < 0) break;
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
using KernelFn = void (*)(BatchParams);

template <int OUT>
static KernelFn kernel_for(int v) {
  if constexpr (OUT == 2) {  // fp32 output (F4): only the default variant is instantiated
    return dequant_kernel<2, 8, 4, false, true, true, true>;
  }
  switch (v) {
    case 0: return dequant_kernel<OUT, 8, 4, false, false, false, false>;
    case 1: return dequant_kernel<OUT, 16, 2, false, false, false, false>;
    case 2: return dequant_kernel<OUT, 16, 4, false, false, false, false>;
    case 3: return dequant_kernel<OUT, 8, 4, true, false, false, false>;
    case 4: return dequant_kernel<OUT, 16, 1, false, false, false, false>;
    case 5: return dequant_kernel<OUT, 8, 8, false, false, false, false>;
    case 6: return dequant_kernel<OUT, 8, 4, false, true, false, false>;
    case 7: return dequant_kernel<OUT, 8, 4, false, true, true, false>;
    case 8: return dequant_kernel<OUT, 8, 4, false, true, true, true>;
    case 9: return dequant_kernel<OUT, 8, 4, false, false, false, true>;
    case 10: return dequant_kernel<OUT, 8, 4, false, false, true, true>;
    case 12: return dequant_kernel<OUT, 8, 4, false, true, true, true, false, NF4_MAX_BATCH, false, true>;
    case 13: return dequant_kernel<OUT, 8, 2, false, true, true, true>;
    case 14: return dequant_kernel<OUT, 8, 4, false, true, true, true, false, NF4_MAX_BATCH, false, false, 1>;
    case 15: return dequant_kernel<OUT, 8, 4, false, true, true, true, false, NF4_MAX_BATCH, false, false, 0, 1>;
    case 16: return dequant_kernel<OUT, 8, 4, false, true, true, true, false, NF4_MAX_BATCH, false, false, 0, 2>;
    case 17: return dequant_kernel<OUT, 8, 4, false, true, true, true, false, NF4_MAX_BATCH, false, false, 0, 0, 2>;
    case 18: return dequant_kernel<OUT, 8, 4, false, true, true, true, false, NF4_MAX_BATCH, false, true, 0, 0, 1, 512>;
    case 19: return dequant_kernel<OUT, 8, 4, false, true, true, true, false, NF4_MAX_BATCH, false, false, 0, 0, 1, 512>;
    default: return dequant_kernel<OUT, 8, 4, false, true, true, true, true>;
  }
}

static std::atomic<int> g_variant{-1};
static std::atomic<int32_t> g_early_inputs{0};

static int current_variant() {
  int v = g_variant.load(std::memory_order_relaxed);
  if (v >= 0) return v;
  v = kDefaultVariant;
  if (const char* env = getenv("NF4_KERNEL_VARIANT")) {
    for (int i = 0; i < kNumVariants; ++i)
      if (strcmp(env, kVariants[i].name) == 0) v = i;
    if (env[0] >= '0' && env[0] <= '9' && atoi(env) < kNumVariants) v = atoi(env);
  }
  g_variant.store(v, std::memory_order_relaxed);
  return v;
}

static int64_t tile_elems(int v) { return int64_t(kVariants[v].threads) * 2 * kVariants[v].vec * kVariants[v].unroll; }
static bool pair_variant(int v) { return v == 12 || v == 18; }

// Launch with programmatic stream serialization (PDL): the kernel executes
// griddepcontrol.wait before its first global access.
template <typename Kernel, typename Params>
static void launch_pdl(Kernel k, int grid, cudaStream_t stream, const Params& P, size_t smem = 0,
                       int threads = kThreads) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, P);   // errors surface through cudaPeekAtLastError at the call site
}

template <int MAXB>
static void launch_small(const BatchParams& P, int out, int grid, cudaStream_t stream, bool quarter_tiles) {
  BatchParamsT<MAXB> Q;
  Q.total_tiles = P.total_tiles;
  Q.count = P.count;
  Q.prefetch_ahead = 0;
  Q.early_inputs = P.early_inputs;
  Q.pad2_ = 0;
  for (int i = 0; i < 16; ++i) Q.lut[i] = P.lut[i];
  for (int i = 0; i < P.count; ++i) Q.t[i] = P.t[i];
  // about two resident waves of tiles or fewer: latency-bound, issue code loads first
  const bool early = P.total_tiles <= int64_t(2) * sm_count() * 8;
  if (quarter_tiles) {
    // a few waves' worth of 16384-element tiles would leave SMs idle: 4096-element
    // tiles (one group per thread) spread the launch over 4x more CTAs
    if (out == 0)
      launch_pdl(dequant_kernel<0, 8, 1, false, true, true, true, false, MAXB, true>, grid, stream, Q);
    else if (out == 1)
      launch_pdl(dequant_kernel<1, 8, 1, false, true, true, true, false, MAXB, true>, grid, stream, Q);
    else
      launch_pdl(dequant_kernel<2, 8, 1, false, true, true, true, false, MAXB, true>, grid, stream, Q);
  } else if (early) {
    if (out == 0)
      launch_pdl(dequant_kernel<0, 8, 4, false, true, true, true, false, MAXB, true>, grid, stream, Q);
    else if (out == 1)
      launch_pdl(dequant_kernel<1, 8, 4, false, true, true, true, false, MAXB, true>, grid, stream, Q);
    else
      launch_pdl(dequant_kernel<2, 8, 4, false, true, true, true, false, MAXB, true>, grid, stream, Q);
  } else {
    if (out == 0)
      launch_pdl(dequant_kernel<0, 8, 4, false, true, true, true, false, MAXB>, grid, stream, Q);
    else if (out == 1)
      launch_pdl(dequant_kernel<1, 8, 4, false, true, true, true, false, MAXB>, grid, stream, Q);
    else
      launch_pdl(dequant_kernel<2, 8, 4, false, true, true, true, false, MAXB>, grid, stream, Q);
  }
}

static KernelFn kernel_of(int out, int v) {
  return out == 0 ? kernel_for<0>(v) : out == 1 ? kernel_for<1>(v) : kernel_for<2>(v);
}

static int occupancy(int v, int out) {
  static std::mutex mu;
  static int cache[kNumVariants][3] = {};
  std::lock_guard<std::mutex> g(mu);
  int& c = cache[v][out];
  if (c == 0) {
    int occ = 0;
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, reinterpret_cast<const void*>(kernel_of(out, v)), kVariants[v].threads,
        pair_variant(v) ? size_t(kPairBytes) : 0);
    c = (e == cudaSuccess && occ > 0) ? occ : 4;
  }
  return c;
}

static int grid_for(int v, int64_t tiles, int out) {
  int64_t g = kVariants[v].persist ? int64_t(sm_count()) * occupancy(v, out) : tiles;
  const int32_t cap = max_ctas();
  if (cap > 0 && g > cap) g = cap;
  if (g > tiles) g = tiles;
  if (g > 0x7FFFFFFF) g = 0x7FFFFFFF;
  return int(g < 1 ? 1 : g);
}

static nf4_status validate(const nf4_tensor& t, int out) {
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
  if (!aligned(t.out, out == 2 ? 4 : 2)) return NF4_ERR_MISALIGNED;
  if (!dq && !aligned(t.absmax, 4)) return NF4_ERR_MISALIGNED;
  if (dq && (!aligned(t.dq.code2, 4) || !aligned(t.dq.absmax2, 4))) return NF4_ERR_MISALIGNED;
  return NF4_OK;
}

static nf4_status launch_batch(const nf4_tensor* ts, int count, int out, const float* lut, cudaStream_t stream,
                               int32_t* launches) {
  const int v = out == 2 ? kDefaultVariant : current_variant();
  int64_t tile = tile_elems(v);
  // small launches of the default kernel use quarter-size tiles (more CTAs, all SMs busy)
  bool quarter = false;
  if (v == kDefaultVariant && count <= 16) {
    int64_t t16 = 0;
    for (int i = 0; i < count; ++i) t16 += (ts[i].n + tile - 1) / tile;
    quarter = t16 < int64_t(kQuarterTileWaves) * sm_count();
    if (quarter) tile /= 4;
  }
  BatchParams P;
  P.count = 0;
  P.prefetch_ahead = (v == 15 || v == 16) ? int32_t(occupancy(v, out) * sm_count()) : 0;
  P.early_inputs = g_early_inputs.load(std::memory_order_relaxed);
  P.pad2_ = 0;
  for (int i = 0; i < 16; ++i) P.lut[i] = lut[i];
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
    d.out = t.out;
    d.n = t.n;
    d.bs_shift = log2i(t.blocksize);
    d.vec_ok = aligned(t.packed, kVariants[v].vec) && aligned(t.out, 32);
    d.pad_ = 0;
    tiles += (t.n + tile - 1) / tile;
    d.tile_end = tiles;
  }
  if (P.count == 0) return NF4_OK;
  P.total_tiles = tiles;
  const int grid = grid_for(v, tiles, out);
  if (v == kDefaultVariant && P.count <= 16) {
    // light parameter block for single tensors and decoder-layer batches
    if (P.count == 1) launch_small<1>(P, out, grid, stream, quarter);
    else launch_small<16>(P, out, grid, stream, quarter);
  } else {
    KernelFn fn = kernel_of(out, v);
    launch_pdl(fn, grid, stream, P, pair_variant(v) ? size_t(kPairBytes) : 0, kVariants[v].threads);
  }
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return NF4_ERR_CUDA;
  }
  ++*launches;
  return NF4_OK;
}

static void nf4_table(float lut[16]) {
  for (int i = 0; i < 16; ++i) memcpy(&lut[i], &h_nf4_bits[i], 4);
}

}  // namespace nf4

using namespace nf4;

extern "C" nf4_status nf4_dequantize_batched_ex(const nf4_tensor* tensors, int32_t count, const float* codebook16,
                                                nf4_dtype out_dtype, void* stream) {
  if (count < 0) return NF4_ERR_BAD_SIZE;
  if (count > 0 && tensors == nullptr) return NF4_ERR_NULL_POINTER;
  if (out_dtype != NF4_F16 && out_dtype != NF4_BF16 && out_dtype != NF4_F32) return NF4_ERR_BAD_DTYPE;
  const int out = int(out_dtype);
  for (int i = 0; i < count; ++i) {
    const nf4_status s = validate(tensors[i], out);
    if (s != NF4_OK) return s;
  }
  float lut[16];
  if (codebook16) {
    for (int i = 0; i < 16; ++i) lut[i] = codebook16[i];
  } else {
    nf4_table(lut);
  }
  int32_t launches = 0;
  // Group tensors with work into launches of at most NF4_MAX_BATCH.
  nf4_tensor buf[NF4_MAX_BATCH];
  int nbuf = 0;
  for (int i = 0; i < count; ++i) {
    if (tensors[i].n == 0) continue;
    buf[nbuf++] = tensors[i];
    if (nbuf == NF4_MAX_BATCH) {
      const nf4_status s = launch_batch(buf, nbuf, out, lut, (cudaStream_t)stream, &launches);
      if (s != NF4_OK) return s;
      nbuf = 0;
    }
  }
  if (nbuf > 0) {
    const nf4_status s = launch_batch(buf, nbuf, out, lut, (cudaStream_t)stream, &launches);
    if (s != NF4_OK) return s;
  }
  set_launch_count(launches);
  return NF4_OK;
}

extern "C" nf4_status nf4_dequantize_batched(const nf4_tensor* tensors, int32_t count, nf4_dtype out_dtype,
                                             void* stream) {
  if (out_dtype != NF4_F16 && out_dtype != NF4_BF16) return NF4_ERR_BAD_DTYPE;
  return nf4_dequantize_batched_ex(tensors, count, nullptr, out_dtype, stream);
}

extern "C" nf4_status nf4_dequantize_ex(const uint8_t* packed, const float* absmax, const nf4_dq_state* dq,
                                        int64_t n, int32_t blocksize, const float* codebook16, nf4_dtype out_dtype,
                                        void* out, void* stream) {
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
  return nf4_dequantize_batched_ex(&t, 1, codebook16, out_dtype, stream);
}

extern "C" nf4_status nf4_dequantize(const uint8_t* packed, const float* absmax, const nf4_dq_state* dq,
                                     int64_t n, int32_t blocksize, nf4_dtype out_dtype, void* out,
                                     void* stream) {
  if (out_dtype != NF4_F16 && out_dtype != NF4_BF16) return NF4_ERR_BAD_DTYPE;
  return nf4_dequantize_ex(packed, absmax, dq, n, blocksize, nullptr, out_dtype, out, stream);
}

extern "C" void nf4_codebook_fp4(float out16[16]) {
  // BitsAndBytes FP4 (sign, 2-bit exponent, 1-bit mantissa) levels / 12 ([ext])
  static const float v[8] = {0.0f, 0.0625f, 8.0f, 12.0f, 4.0f, 6.0f, 2.0f, 3.0f};
  for (int i = 0; i < 8; ++i) {
    out16[i] = v[i] / 12.0f;
    out16[8 + i] = -(v[i] / 12.0f);
  }
}

extern "C" void nf4_codebook(float out16[16]) {
  for (int i = 0; i < 16; ++i) {
    float f;
    memcpy(&f, &h_nf4_bits[i], 4);
    out16[i] = f;
  }
}

extern "C" int32_t nf4_dequant_grid(int64_t tiles) {
  return grid_for(current_variant(), tiles < 1 ? 1 : tiles, 0);
}
extern "C" int64_t nf4_dequant_tile_elems(void) { return tile_elems(current_variant()); }
extern "C" int32_t nf4_kernel_variant_count(void) { return kNumVariants; }
extern "C" const char* nf4_kernel_variant_name(int32_t v) {
  return (v >= 0 && v < kNumVariants) ? kVariants[v].name : nullptr;
}
extern "C" int32_t nf4_set_kernel_variant(int32_t v) {
  if (v < 0 || v >= kNumVariants) return current_variant();
  g_variant.store(v, std::memory_order_relaxed);
  return v;
}
extern "C" int32_t nf4_get_kernel_variant(void) { return current_variant(); }
extern "C" void nf4_set_early_input_reads(int32_t enable) {
  g_early_inputs.store(enable ? 1 : 0, std::memory_order_relaxed);
}
