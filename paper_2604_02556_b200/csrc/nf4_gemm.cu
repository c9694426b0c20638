// nf4_gemm.cu -- fused NF4 dequantization + tcgen05 tensor-core GEMM (SURVEY
// row F1): Y[M, N] = X[M, K] . W[N, K]^T where W is an NF4 weight ([out, in],
// K contiguous, blockwise absmax along K) and X, Y are 16-bit activations.
//
// The weight never exists in HBM as 16-bit: producer warps read the packed
// codes (0.5 B/elt) + scales, dequantize them with exactly the hot path's
// per-element definition (RNE16(fl32(NF4[idx] * a))) and write the
// 16-bit weights straight into TMEM, where tcgen05.mma (kind::f16, fp32
// accumulation in TMEM) reads them as its A operand.  The paper motivates
// exactly this step: dequantization is 72.4% of the quantized matmul
// and the fused, preprocessing-free direction is the one it leaves open.
//
// One CTA per SM, 832 threads (see the kernel's comment for details):
//   warps 0-23  three producer groups of 8 warps; group g dequantizes the
//               super-stages J = g (mod 3) of the CTA's work into its TMEM A
//               tiles, and the group that finished a segment runs its epilogue
//               (tcgen05.ld -> y, or an fp32 partial + per-tile counter).
//   warp 24     TMEM allocator and MMA issuer (converged warp, elect.sync).
//   warp 25     TMA issuer: per super-stage (4 chunks of 64 k) one swizzled box
//               of codes (128 rows x 128 B) and 4 boxes of X (BN x 64, SW128:
//               the UMMA canonical layout, zero-filled past M).
// Swap-AB orientation: the MMA's M=128 side is the weight (128 output
// features), its N side the tokens (BN in {16,...,256}), so decode-size M
// wastes nothing.
// Work distribution (stream-K): the (tile, 64-element k-chunk) stream of the
// whole GEMM -- or of up to 4 weights sharing X (nf4_gemm_grouped) -- is cut
// into one equal contiguous range per SM; a tile cut across ranges is summed,
// in piece order, by the CTA holding its last piece (deterministic for a given
// GPU).  The classic grid (explicit `splits`, one CTA per tile x split, plus a
// reduction kernel) is the same kernel with one segment per CTA.
#include <cuda.h>  // CUtensorMap (the encoder is fetched at run time; no libcuda link)
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "nf4_internal.cuh"
#include "../../include/nf4_gemm.h"

namespace nf4 {
namespace gemm {

// Producer groups per token-tile width BN: up to NF4_GEMM_W4_MAXBN (decode-size
// M), 5 groups of 4 warps (one thread per weight row, both halves of each chunk;
// 2-chunk super-stages x 10, 5 x 2 A tiles in TMEM): more, smaller hand-offs, so a
// group that ran ahead waits less for the in-order MMA.  Wider tiles keep 3 groups
// of 8 warps (2 threads per row), whose 4-chunk stages suit the heavier MMA/X side.
// DQ second-level table (code2): read through L1 from global memory (staging it in
// shared memory put a global round trip before the block-wide sync: +4% at M=1).
#ifndef NF4_GEMM_W4_MAXBN
#define NF4_GEMM_W4_MAXBN 16
#endif
#ifndef NF4_GEMM_GROUPS
#define NF4_GEMM_GROUPS 3   // 8-warp groups
#endif
#ifndef NF4_GEMM_W4_GROUPS
#define NF4_GEMM_W4_GROUPS 5
#endif
#ifndef NF4_GEMM_W4_CST
#define NF4_GEMM_W4_CST 12
#endif
// A-tile slots in TMEM for 4-warp groups (BN = 16): more slots than groups let a
// group that ran ahead start its next super-stage before the in-order MMA has
// consumed its previous one (it waits only for the slot's previous occupant).
// TMEM: NACC x 32 accumulator columns + SLOTS x SUB x 32 A columns <= 512.
#ifndef NF4_GEMM_ACC_GUARD
#define NF4_GEMM_ACC_GUARD 1
#endif
#ifndef NF4_GEMM_W4_SLOTS
#define NF4_GEMM_W4_SLOTS 7
#endif
template <int BN> __host__ __device__ constexpr int wpg_for() { return BN <= NF4_GEMM_W4_MAXBN ? 4 : 8; }
template <int BN> __host__ __device__ constexpr int groups_for() { return BN <= NF4_GEMM_W4_MAXBN ? NF4_GEMM_W4_GROUPS : NF4_GEMM_GROUPS; }
// 8-warp groups (BN >= 32): NF4_GEMM_WIDE_SLOTS = 1 gives them every A slot TMEM and the code
// stages allow (min(CST, (512 - accumulators) / (SUB * 32)) >= G) instead of one per group.
#ifndef NF4_GEMM_WIDE_SLOTS
#define NF4_GEMM_WIDE_SLOTS 0
#endif
template <int BN> constexpr int sub_for();
template <int BN> constexpr int cst_for();
template <int BN> constexpr int nacc_for();
template <int BN> __host__ __device__ constexpr int slots_for() {
  if constexpr (BN <= NF4_GEMM_W4_MAXBN) {
    return NF4_GEMM_W4_SLOTS;
  } else if constexpr (NF4_GEMM_WIDE_SLOTS != 0) {
    constexpr int tm = (512 - nacc_for<BN>() * (BN < 32 ? 32 : BN)) / (sub_for<BN>() * 32);
    constexpr int s = tm < cst_for<BN>() ? tm : cst_for<BN>();
    return s > groups_for<BN>() ? s : groups_for<BN>();
  } else {
    return groups_for<BN>();
  }
}
constexpr int kCodeBytes = 32;              // packed bytes per row per k-chunk
constexpr int kChunk = 64;          // k elements per stage (= one 128 B swizzle row in 16-bit)
constexpr int kRowBytes = 128;

// One weight (problem) of a multi-weight launch.  nf4_gemm_grouped: members share
// X and K; nf4_gemm_multi: every member has its own X and K (M and the blocksize
// are shared).  Work order is member-major: member g owns the global chunks
// [cbase, cbase + tiles_n * tiles_m * nk) and the global 128-feature tiles
// [tile0, tile0 + tiles_n) (partial-sum columns) and [ftile0, ftile0 + tiles_n *
// tiles_m) (stream-K counters).
constexpr int kMaxMembers = 64;
struct Member {
  const float* absmax;     // fp32 mode if non-null
  const uint8_t* qabsmax;  // DQ mode
  const float* code2;
  const float* absmax2;
  void* y;                 // [M, N] row-major
  float offset;
  int32_t N;
  int32_t K, nk;           // reduction length and its 64-element chunks
  int32_t tiles_n;         // 128-feature tiles of this member
  int32_t tile0;           // first global 128-feature tile (partial-sum column block)
  int32_t ftile0;          // first global tile (stream-K counter)
  int32_t cbase;           // first global chunk
};
template <int NM>
struct MapsT {             // TMA descriptors per member: packed codes, X
  CUtensorMap c[NM];
  CUtensorMap x[NM];
};

struct GemmCommon {
  int32_t nmem;
  float* partial;          // [splits, M, Npad] fp32 (classic) / [parts, M, Npad] (stream-K)
  unsigned* flags;         // stream-K: per-tile count of published partials (zero between calls)
  int32_t M;
  int32_t Npad;            // (sum of tiles_n) * 128: row stride of the partials
  int32_t bs_shift;
  int32_t chunks_per_split;  // classic split-K
  int32_t splits;            // classic split-K (1 = direct output)
  int32_t out_dtype;         // NF4_F16 / NF4_BF16 / NF4_F32
  int32_t streamk;           // 1: stream-K ranges over a 1-D grid
  int32_t tiles_m;           // token tiles (BN tokens each)
  int64_t total_chunks;      // all members
  int32_t align4;            // stream-K range bounds rounded to 4 chunks
  int32_t early_weights;     // 1: read the weight before griddepcontrol.wait (nf4_gemm.h)
  unsigned long long* trace;  // diagnostics only (NF4_GEMM_TRACE): per-CTA start / end / SM / last epilogue
  int32_t experiment;         // diagnostics only (NF4_GEMM_EXPERIMENT): 1 skip MMA, 2 skip dequant, 4 skip tcgen05.st,
                              // 8 skip X loads, 16 skip code loads
  float lut[16];
};
template <int NM>
struct GemmParamsT : GemmCommon {
  Member mem[NM];
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
#ifndef NF4_GEMM_WAIT_MODE
#define NF4_GEMM_WAIT_MODE 1
#endif
// 0: try_wait with a 10 ms suspend hint; 1: try_wait (hardware default time
// limit); 2: test_wait spin; >2: try_wait + __nanosleep(mode) between polls.
#ifndef NF4_GEMM_HANG_DIAG
#define NF4_GEMM_HANG_DIAG 0   // diagnostics builds only: report and trap a wait that never completes
#endif
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
#if NF4_GEMM_HANG_DIAG
  long long spins = 0;
#endif
  while (!done) {
#if NF4_GEMM_HANG_DIAG
    if (++spins == (1ll << 24)) {
      printf("HANG cta %d warp %d lane %d bar_smem 0x%x parity %u\n", int(blockIdx.x), int(threadIdx.x >> 5),
             int(threadIdx.x & 31), b, parity);
    }
#endif
#if NF4_GEMM_WAIT_MODE == 0
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(b), "r"(parity), "r"(0x989680) : "memory");
#elif NF4_GEMM_WAIT_MODE == 1
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(b), "r"(parity) : "memory");
#elif NF4_GEMM_WAIT_MODE == 2
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(b), "r"(parity) : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(b), "r"(parity) : "memory");
    if (!done) __nanosleep(NF4_GEMM_WAIT_MODE);
#endif
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

// Issued by a whole (converged) warp; elect.sync picks the one lane that issues,
// so every operand is warp-uniform and the four K=16 steps of a 64-element
// chunk cost ~1 instruction each (a divergent single-lane issue made ptxas
// rebuild the uniform operands per MMA, ~15 instructions and ~66 cycles each).
// A: 128 lanes x 16 weights at a, a+8, a+16, a+24 (TMEM columns); B: the
// SWIZZLE_128B X tile, +32 B (= +2 in the descriptor's address field) per step.
__device__ __forceinline__ void umma_chunk_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p0, pt;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 a1, a2, a3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p0, %4, 0;\n\tsetp.eq.b32 pt, %4, %4;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, pt;\n\t}"
      ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
      ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Diagnostics (tools/, a -DNF4_GEMM_DIAG=1 build only; compiled out of libnf4):
// NF4_GEMM_TRACE = device address of an int64 buffer for event times,
// NF4_GEMM_EXPERIMENT = bit mask skipping parts of the pipeline (timing studies).
#ifndef NF4_GEMM_DIAG
#define NF4_GEMM_DIAG 0
#endif
// NF4_GEMM_EXP_CONST: the same pipeline-skipping experiments fixed at compile time, so
// the rest of the kernel is the production code (tools/: bound attribution).
#ifndef NF4_GEMM_EXP_CONST
#define NF4_GEMM_EXP_CONST 0
#endif
// (the run-time experiment mask only in NF4_GEMM_DIAG >= 2 builds: DIAG = 1 traces at production speed)
#define NF4_EXP(bit) ((NF4_GEMM_EXP_CONST & (bit)) || (NF4_GEMM_DIAG >= 2 && (p.experiment & (bit))))
#define NF4_TRACING (NF4_GEMM_DIAG && p.trace != nullptr)
// per-super-stage event times of CTA 0, slot base + J (J < 80)
#define NF4_TRACE_J(base, Jv)                                                                       \
  do {                                                                                              \
    if (NF4_TRACING && cta_lin == 0 && (Jv) < 80) p.trace[(base) + (Jv)] = gtimer();               \
  } while (0)
// ---- stream-K range arithmetic (shared by the GEMM kernel and the reduction) ----
// First global chunk of CTA c's range: floor(c*W/G), rounded to a multiple of 4
// chunks when every tile has a multiple of 4 chunks (whole TMA super-stages).
__host__ __device__ __forceinline__ int64_t sk_bound(int64_t c, int64_t W, int64_t G, int align4) {
  int64_t b = c * W / G;
  if (align4) b = (b + 2) / 4 * 4;
  return b < W ? b : W;
}
// The CTA whose range contains global chunk x (largest c with sk_bound(c) <= x):
// start from floor(x*G/W), whose bound is within 2 chunks of x, and step.
__host__ __device__ __forceinline__ int64_t sk_owner(int64_t x, int64_t W, int64_t G, int align4) {
  int64_t c = x * G / W;
  if (c > G - 1) c = G - 1;
  while (c > 0 && sk_bound(c, W, G, align4) > x) --c;
  while (c + 1 < G && sk_bound(c + 1, W, G, align4) <= x) ++c;
  return c;
}

// Member owning global chunk x (binary search over the members' first chunks).
template <int NM>
__device__ __forceinline__ int member_of_chunk(const GemmParamsT<NM>& p, int x) {
  if constexpr (NM == 1) {
    return 0;
  } else {
    int lo = 0, hi = p.nmem - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (p.mem[mid].cbase <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
}
// The tile containing global chunk x: member g, member-local tile tl, its first chunk and length.
struct TileAt {
  int g, tl, tstart, nkt;
};
template <int NM>
__device__ __forceinline__ TileAt tile_at(const GemmParamsT<NM>& p, int x) {
  TileAt t;
  t.g = member_of_chunk(p, x);
  t.nkt = p.mem[t.g].nk;
  t.tl = (x - p.mem[t.g].cbase) / t.nkt;
  t.tstart = p.mem[t.g].cbase + t.tl * t.nkt;
  return t;
}

// One segment = a contiguous k-range of one output tile processed by one CTA.
struct Segment {
  int g;          // member
  int tn;         // global 128-feature tile index (partial-sum columns)
  int ft;         // global tile index (stream-K counter)
  int n0, m0;     // tile origin (member-local features, tokens)
  int kc0, nk;    // first chunk within the tile, chunk count
  int nkt;        // chunks of the whole tile (the member's K / 64)
  int part;       // partial-sum slot (stream-K: segment index within the tile; classic: split)
};

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Byte-pair lookup table (NF4_GEMM_PAIR): entry b = (NF4[b >> 4], NF4[b & 15]),
// the two fp32 levels of one code byte (element 2j, element 2j+1), replicated
// once per lane of a half-warp: row b (NF4_GEMM_PAIR_ROW = 128 B) holds 16
// copies, lane l reads copy l % 16, so the 16 lanes of each LDS.64 phase (a
// 64-bit load is served per half-warp) hit 16 distinct bank pairs for any
// codes: conflict-free.  (ROW 256: 32 copies, lane l reads copy l.)  The
// address of byte j of a code word is one PRMT (ALU) + one IMAD (FMA pipe).
// Per two weights: PRMT + IMAD + LDS.64 + FMUL2 + F2FP.
#ifndef NF4_GEMM_PAIR
#define NF4_GEMM_PAIR 1
#endif
#ifndef NF4_GEMM_PAIR_MAXBN
#define NF4_GEMM_PAIR_MAXBN 256
#endif
#ifndef NF4_GEMM_ST_SPLIT
#define NF4_GEMM_ST_SPLIT 2   // tcgen05.st pieces per 32-weight chunk piece (0: one x16 after the wait; 2: x8; 4: x4)
#endif
#ifndef NF4_GEMM_PAIR_ROW
#define NF4_GEMM_PAIR_ROW 128
#endif
// Register-table lookups (4-warp / BN = 16 producers, byte-pair path): of the 8 code
// words of a 64-weight chunk, this many are decoded from a per-chunk register table
// (PRMT byte planes of the 16 pre-scaled 16-bit levels) instead of the shared-memory
// pair table -- ALU work in place of shared-memory wavefronts, which bind the kernel.
// 0: off; 1: the last word of the chunk's second half; 2: the last word of each half.
#ifndef NF4_GEMM_REG_WORDS
#define NF4_GEMM_REG_WORDS 0
#endif
template <int BN> __host__ __device__ constexpr bool pair_for() { return NF4_GEMM_PAIR && BN <= NF4_GEMM_PAIR_MAXBN; }
template <int BN> __host__ __device__ constexpr int pair_table_bytes() { return pair_for<BN>() ? 256 * NF4_GEMM_PAIR_ROW : 0; }

// Code-box swizzle: the TMA writes the 128 rows x (SUB*32) B box with the
// hardware swizzle matching its width, so the 8 lanes of an LDS.128 phase
// (consecutive rows, same 16-B column) hit 8 different bank groups.
template <int SUB>
__device__ __forceinline__ uint32_t code_chunk_off(int row, int c16) {
  if constexpr (SUB == 4) return uint32_t(row * 128 + ((c16 ^ (row & 7)) << 4));          // SWIZZLE_128B
  else if constexpr (SUB == 2) return uint32_t(row * 64 + ((c16 ^ ((row >> 1) & 3)) << 4));  // SWIZZLE_64B
  else return uint32_t(row * 32 + ((c16 ^ ((row >> 2) & 1)) << 4));                          // SWIZZLE_32B
}

// Segment enumeration: every role walks the same sequence.  Stream-K ranges are
// computed once per CTA by one thread.  A range is [tail piece of a tile] [whole
// tiles] [head piece of a tile]; the head piece (chunk 0 of its tile onward) is
// processed FIRST, so its partial is published early and the CTA finishing that
// tile (whose tail piece is its own first segment) never waits at the end.
// Only the range's first chunk can start inside a tile, so every other segment
// is its tile's partial slot 0.
struct SegIter {
  int x, end;          // stream-K: cursor and end of the current run
  int start, hs;       // range start; head-piece start (== range start: none)
  int part0;           // slot of the segment starting at the range start
  int phase;           // 0: head piece, 1: the rest
  int done_classic;
};
template <int BN, int NM>
__device__ __forceinline__ bool next_segment(const GemmParamsT<NM>& p, SegIter& it, Segment& sg) {
  if (!p.streamk) {
    if (it.done_classic) return false;
    it.done_classic = 1;
    sg.g = 0;
    sg.tn = blockIdx.x;
    sg.ft = blockIdx.x + blockIdx.y * p.mem[0].tiles_n;
    sg.n0 = blockIdx.x * 128;
    sg.m0 = blockIdx.y * BN;
    sg.nkt = p.mem[0].nk;
    sg.kc0 = blockIdx.z * p.chunks_per_split;
    const int kc1 = min(sg.nkt, sg.kc0 + p.chunks_per_split);
    sg.nk = kc1 > sg.kc0 ? kc1 - sg.kc0 : 0;
    sg.part = blockIdx.z;
    return true;
  }
  if (it.x >= it.end) {
    if (it.phase != 0 || it.hs == it.start) return false;
    it.phase = 1;                 // head piece done: now [start, hs)
    it.x = it.start;
    it.end = it.hs;
  }
  const TileAt t = tile_at(p, it.x);   // single weight: member 0 (constant-bank operands)
  const int send = min(it.end, t.tstart + t.nkt);
  const int tiles_n = p.mem[t.g].tiles_n;
  const int tn = t.tl % tiles_n;
  sg.g = t.g;
  sg.tn = p.mem[t.g].tile0 + tn;
  sg.ft = p.mem[t.g].ftile0 + t.tl;
  sg.n0 = tn * 128;
  sg.m0 = (t.tl / tiles_n) * BN;
  sg.nkt = t.nkt;
  sg.kc0 = it.x - t.tstart;
  sg.nk = send - it.x;
  sg.part = it.x == it.start ? it.part0 : 0;
  it.x = send;
  return true;
}
template <int NM>
__device__ __forceinline__ SegIter seg_begin(const GemmParamsT<NM>& p, const int (&range)[3]) {
  SegIter it;
  it.done_classic = 0;
  it.start = range[0];
  it.part0 = range[2];
  it.hs = it.start;
  it.phase = 1;
  it.x = range[0];
  it.end = range[1];
  if (p.streamk && range[1] > range[0]) {
    const TileAt t = tile_at(p, range[1] - 1);
    if (range[1] < t.tstart + t.nkt && t.tstart > range[0]) {   // the range ends inside a tile it did not start in
      it.hs = t.tstart;
      it.phase = 0;
      it.x = t.tstart;                                          // head piece [tstart, end) first
    }
  }
  return it;
}

// Block scales of one super-stage for one weight row.  fast: blocksize 64,
// K % 256 == 0, 4-chunk super-stages -- the 4 scales are 4 consecutive fp32
// absmax (one 128-bit load) or 4 consecutive qabsmax bytes (one 32-bit load)
// plus the 1-2 absmax2 groups they fall in; general: one load per chunk.
struct Scales {
  uint32_t s[4];   // fp32 absmax bits per chunk | fast DQ: 4 qabsmax bytes in s[0] | DQ: qabsmax per chunk
  float a2[4];     // DQ: absmax2 per chunk | fast DQ: absmax2 of the first / last block in a2[0] / a2[1]
};

// One CTA per SM, G groups of 8 producer warps sharing one TMA/MMA pipeline
// (a single CTA keeps the SM's work in one stream-K range: with 3 independent
// CTAs per SM the warp scheduler starved the youngest, whose tail then ran
// alone -- tools/gemm_trace.py measured 21-43 us for equal ranges).
//   warps 0..8G-1  producers; group g = warp/8 dequantizes the super-stages J
//                  with J % G == g, thread (w, l) owning weight row
//                  32(w%4)+l (= TMEM lane) and half (w%8)/4 of each chunk;
//                  the group that produced a segment's last super-stage then
//                  runs its epilogue (tcgen05.ld -> y or fp32 partial).
//   warp 8G        TMEM allocator + MMA issuer (the converged warp runs the
//                  loop; elect.sync picks the issuing lane).
//   warp 8G+1      TMA issuer (one lane).
// TMEM: NACC accumulators of max(BN, 32) fp32 columns, then G*SUB A tiles of
// 32 columns (128 lanes x 64 16-bit weights), one per (group, chunk-in-stage).
// Barriers (one arrive/commit per super-stage each, so the MMA issuer spends
// its time issuing MMAs, not waiting on barriers): c_full (code bytes), x_full
// (X bytes) / c_free (MMA commit: the MMA waited for w_full, so the codes were
// read too)
// per shared-memory super-stage (CST >= G keeps every parity wait within one
// phase); w_full (8 warps) / a_free (MMA commit) per group's 4 A tiles;
// acc_full / acc_empty per accumulator.
// Stream-K fix-up (no second kernel): every tile piece that is not the tile's
// last is published as an fp32 partial + a per-tile counter increment; the CTA
// holding the tile's last piece (its range's first chunk) sums the partials in
// piece order at the end of its range and writes y.  It waits only for
// lower-numbered CTAs, dispatched before it, which compute the head piece of
// their last tile first (seg_begin), so the wait is normally already over.
// Grouped / multi-problem GEMMs (NM > 1): the segment's member selects the TMA descriptors,
// scale pointers, code2 table and output.
template <int BN, int G, int SUB, int CST, int NACC, bool BF16, int NM>
__global__ void __launch_bounds__(32 * (wpg_for<BN>() * G + 2), 1)
    nf4_gemm_kernel(const __grid_constant__ GemmParamsT<NM> p, const __grid_constant__ MapsT<NM> maps) {
  // NM: members this instantiation serves (1, NF4_GEMM_MAX_GROUP or kMaxMembers: the
  // parameter block is copied at every launch, so small groups use a small one)
  static_assert(CST >= G, "a super-stage slot must not be two phases behind any group");
  constexpr int kProducerWarps = wpg_for<BN>();
  constexpr int kMmaWarp = kProducerWarps * G, kTmaWarp = kProducerWarps * G + 1;
  constexpr int ACC = BN < 32 ? 32 : BN;
  constexpr int A0 = NACC * ACC;
  constexpr int S = slots_for<BN>();   // A-tile slots: super-stage Jg uses slot Jg % S
  static_assert(S >= G, "a group's previous fill must have freed the slot's previous-but-one use");
  static_assert(CST >= S, "the A-slot wait must prove the code slot's previous use landed");
  // first piece of a stage dequantized before the A-slot wait only when that keeps every
  // c_full wait within one phase (see the producers)
  constexpr bool kEarlyFirstPiece = CST >= G + S;
  static_assert(A0 + S * SUB * 32 <= 512, "TMEM budget");
  constexpr int kSuperCodeBytes = 128 * SUB * kCodeBytes;
  constexpr int kSuperXBytes = SUB * BN * kRowBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(256) float lut[16];                    // 256-B aligned: address = PRMT(offsets, base)
  __shared__ __align__(8) uint64_t c_full[CST], x_full[CST], c_free[CST], w_full[S], a_free[S], acc_full[NACC],
      acc_empty[NACC];
  __shared__ uint32_t tmem_holder;
  __shared__ uint32_t exp_sink;                               // NF4_EXP(4) builds only (never written in practice)
  __shared__ int epi_done[NACC];                              // epilogue warps finished, per accumulator
  __shared__ int sk_range[3];                                 // stream-K: range start, end, first slot
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ptab = smem;                                       // NF4_GEMM_PAIR: 256 rows x 32 lanes x 8 B
  uint8_t* smem_c = smem + pair_table_bytes<BN>();            // CST x 128 rows x SUB*32 B (codes)
  uint8_t* smem_x = smem_c + CST * kSuperCodeBytes;           // CST x SUB x BN x 128 B (X)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (NF4_TRACING && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[1024 + 4 * cta_lin] = gtimer();
    p.trace[1024 + 4 * cta_lin + 2] = smid;
  }
  if (warp == kTmaWarp && lane == 0) {   // descriptor fetch overlaps the whole prologue
    for (int i = 0; i < NM && i < p.nmem && i < 8; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.c[i])) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.x[i])) : "memory");
    }
  }
  if (threadIdx.x < 16) lut[threadIdx.x] = p.lut[threadIdx.x];
  if constexpr (pair_for<BN>()) {
    // row b: ROW/8 copies of (NF4[b >> 4], NF4[b & 15]); 16-B stores of two copies
    // (levels from a register per lane + shuffles, not per-thread indexing of the parameter bank)
    constexpr int kStoresPerRow = NF4_GEMM_PAIR_ROW / 16;
    const float lv = p.lut[lane & 15];
    for (int i0 = int(threadIdx.x) & ~31; i0 < 256 * kStoresPerRow; i0 += blockDim.x) {   // warp-uniform trip count
      const int i = i0 + lane;
      const int b = (i / kStoresPerRow) & 255;
      const float h = __shfl_sync(0xffffffffu, lv, b >> 4), l = __shfl_sync(0xffffffffu, lv, b & 15);
      if (i < 256 * kStoresPerRow) *reinterpret_cast<float4*>(ptab + 16 * i) = make_float4(h, l, h, l);
    }
  }
  if (NF4_TRACING && cta_lin == 0 && threadIdx.x == 0) p.trace[600] = gtimer();   // prologue: table built
#if NF4_GEMM_HANG_DIAG
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("BARS c_full 0x%x x_full 0x%x c_free 0x%x w_full 0x%x a_free 0x%x acc_full 0x%x acc_empty 0x%x CST %d S %d G %d\n",
           smem_u32(c_full), smem_u32(x_full), smem_u32(c_free), smem_u32(w_full), smem_u32(a_free),
           smem_u32(acc_full), smem_u32(acc_empty), CST, S, G);
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < CST; ++s) {
      mbar_init(&c_full[s], 1);
      mbar_init(&x_full[s], 1);
      mbar_init(&c_free[s], 1);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&w_full[s], kProducerWarps);
      mbar_init(&a_free[s], 1);
    }
    for (int s = 0; s < NACC; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kProducerWarps);
      epi_done[s] = 0;
    }
    if (NF4_TRACING && cta_lin == 0) p.trace[603] = gtimer();   // barriers initialised
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (NF4_TRACING && cta_lin == 0) p.trace[604] = gtimer();   // init fence
    if (p.streamk) {
      const int64_t W = p.total_chunks, NG = gridDim.x;
      const int64_t x0 = sk_bound(blockIdx.x, W, NG, p.align4);
      sk_range[0] = int(x0);
      sk_range[1] = int(sk_bound(blockIdx.x + 1, W, NG, p.align4));
      sk_range[2] = x0 < W ? int(blockIdx.x - sk_owner(tile_at(p, int(x0)).tstart, W, NG, p.align4)) : 0;
    } else {
      sk_range[0] = sk_range[1] = sk_range[2] = 0;
    }
    if (NF4_TRACING && cta_lin == 0) p.trace[601] = gtimer();   // stream-K range
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    if (NF4_TRACING && cta_lin == 0 && lane == 0) p.trace[602] = gtimer();   // TMEM allocated
  }
  // Programmatic dependent launch: the next kernel in the stream may start its own
  // prologue as soon as our CTAs leave their SMs.  Only X, y and the workspace
  // can depend on the previous kernel: the weight (codes, scales, code2) is
  // read BEFORE griddepcontrol.wait (nf4_gemm.h states the contract), so the
  // TMA warp fetches the first super-stages of codes and the producers
  // dequantize them into TMEM while the previous kernel drains; the TMA warp
  // waits before loading X, the producers before their first store to y or
  // the workspace, everybody before the stream-K fix-up.
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_holder;
  // weights written by the immediately preceding kernel: read nothing before it completes
  if (!p.early_weights) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (NF4_TRACING && cta_lin == 0 && threadIdx.x == 0) p.trace[0] = gtimer();

  if (warp < kProducerWarps * G) {
    // ======================= producers (dequantize into TMEM) + epilogue =======================
    const int g = warp / kProducerWarps, wl = warp % kProducerWarps;
    const int t = 32 * (wl & 3) + lane;        // tile row = TMEM lane
    const int half = kProducerWarps == 8 ? wl >> 2 : 0;   // 4-warp groups: each thread does both halves
    const int chunk_shift = p.bs_shift - 6;    // 64-element chunks per quantization block = 2^chunk_shift
    const uint32_t tlane = uint32_t(32 * (wl & 3)) << 16;
    const uint32_t lut_base = smem_u32(lut);   // low byte 0: PRMT splices a byte offset into it
    const uint32_t ptab_base = smem_u32(ptab);
    const uint32_t ptab_lane = ptab_base + uint32_t(lane % (NF4_GEMM_PAIR_ROW / 8)) * 8u;
    int J = 0, sidx = 0;                       // super-stages / segments before this segment
    SegIter it = seg_begin(p, sk_range);
    Segment sg;
    while (next_segment<BN>(p, it, sg)) {
      // this segment's weight (member of a grouped GEMM)
      // (read from the parameter bank at each use: keeping them in registers spilled)
#define absmax (p.mem[sg.g].absmax)
#define qabsmax (p.mem[sg.g].qabsmax)
#define absmax2 (p.mem[sg.g].absmax2)
      const float offset = p.mem[sg.g].offset;
      const float* c2 = p.mem[sg.g].code2;
      const int Nm = p.mem[sg.g].N;
      const int Km = p.mem[sg.g].K;
      const int row = sg.n0 + t;
      const bool row_ok = row < Nm;
      const int64_t blk_base = (int64_t(row) * Km) >> p.bs_shift;
      const int nk = sg.nk, kc0 = sg.kc0;
      const int nsuper = (nk + SUB - 1) / SUB;
      // fast: blocksize 64 and whole, aligned super-stages -- the SUB scales of a
      // super-stage are SUB consecutive fp32 absmax (one vector load) or SUB
      // consecutive qabsmax bytes (one load) plus the 1-2 absmax2 groups they span
      // (2-chunk stages: BN = 64 only -- 0.5% slower at BN = 128, measured)
      const bool fast =
          (SUB == 4 || (SUB == 2 && BN <= 64)) && p.bs_shift == 6 && (Km % (64 * SUB)) == 0 && (kc0 % SUB) == 0 &&
          (nk % SUB) == 0 &&
          (absmax != nullptr ? (reinterpret_cast<uintptr_t>(absmax) & (4 * SUB - 1)) == 0
                               : (reinterpret_cast<uintptr_t>(qabsmax) & (SUB - 1)) == 0);
      auto fetch = [&](Scales& sc, int j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) { sc.s[q] = 0; sc.a2[q] = 0.0f; }
        if (!row_ok) return;
        if (fast) {
          const int64_t b0 = blk_base + kc0 + SUB * j;
          if (absmax != nullptr) {
            if constexpr (SUB == 4) {
              const uint4 v = __ldg(reinterpret_cast<const uint4*>(absmax + b0));
              sc.s[0] = v.x; sc.s[1] = v.y; sc.s[2] = v.z; sc.s[3] = v.w;
            } else {
              const uint2 v = __ldg(reinterpret_cast<const uint2*>(absmax + b0));
              sc.s[0] = v.x; sc.s[1] = v.y;
            }
          } else {
            if constexpr (SUB == 4)
              sc.s[0] = __ldg(reinterpret_cast<const uint32_t*>(qabsmax + b0));
            else
              sc.s[0] = __ldg(reinterpret_cast<const uint16_t*>(qabsmax + b0));
            sc.a2[0] = __ldg(absmax2 + (b0 >> 8));
            sc.a2[1] = __ldg(absmax2 + ((b0 + SUB - 1) >> 8));
          }
        } else {
#pragma unroll
          for (int q = 0; q < SUB; ++q) {
            const int i = j * SUB + q;
            if (i < nk) {
              const int64_t b = blk_base + ((kc0 + i) >> chunk_shift);
              if (absmax != nullptr) {
                sc.s[q] = __float_as_uint(__ldg(absmax + b));
              } else {
                sc.s[q] = __ldg(qabsmax + b);
                sc.a2[q] = __ldg(absmax2 + (b >> 8));
              }
            }
          }
        }
      };
      int j = (g - J % G + G) % G;               // this group's first super-stage of the segment
      Scales nxt;
      if (j < nsuper) fetch(nxt, j);
      for (; j < nsuper; j += G) {
        const Scales sc = nxt;
        if (j + G < nsuper) fetch(nxt, j + G);   // one super-stage ahead (hides the L2 latency)
        const int Jg = J + j;
        const int cs = Jg % CST;
        const int slot = Jg % S;
        const uint32_t aph = uint32_t(Jg / S) & 1u;
        // A parity wait must be made while the barrier is within one phase of the awaited
        // one, on both sides.  c_full[cs] for stage Jg needs stage Jg - CST (its previous
        // use) landed.  With CST >= G + S this group's previous stage (which waited for the
        // MMA to consume Jg - G - S) proves it, and the first piece of the stage can be
        // dequantized before waiting for the A slot.  Otherwise the A-slot wait (the MMA
        // consumed Jg - S; CST >= S) comes first.  (Waiting for the consumption of Jg - CST
        // itself is NOT safe: its slot may already be two uses further, and the wait would
        // then block until a stage this group has yet to produce.)
        if constexpr (!kEarlyFirstPiece) {
          mbar_wait_parity(&a_free[slot], aph ^ 1u);     // the MMA is done with the slot's previous tiles
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        mbar_wait_parity(&c_full[cs], uint32_t(Jg / CST) & 1u);   // codes of this super-stage landed
        if (wl == 0 && lane == 0) NF4_TRACE_J(100, Jg);
        const int64_t b0 = blk_base + kc0 + SUB * j;
        // the stage body, specialised on "all SUB chunks present" and the scale format
        // (uniform branches hoisted out of the per-chunk code)
        auto stage = [&](auto full_tag, auto mode_tag) {
          constexpr bool FULL = decltype(full_tag)::value;
          constexpr int MODE = decltype(mode_tag)::value;   // 0 fp32 absmax, 1 DQ fast, 2 DQ general
#pragma unroll
          for (int q = 0; q < SUB; ++q) {
            const int i = j * SUB + q;
            if (!FULL && i >= nk) break;
            uint32_t w[16];
            float a = 0.0f;
            if constexpr (MODE == 0) {
              a = __uint_as_float(sc.s[q]);
            } else if constexpr (MODE == 1) {
              // A4 (R7): fl32(fl32(code2[qabsmax] * absmax2) + offset), two roundings
              const uint32_t qb = (sc.s[0] >> (8 * q)) & 0xFFu;
              const float a2 = ((b0 + q) >> 8) == (b0 >> 8) ? sc.a2[0] : sc.a2[1];
              a = __fadd_rn(__fmul_rn(__ldg(c2 + qb), a2), offset);
            } else {
              a = __fadd_rn(__fmul_rn(__ldg(c2 + sc.s[q]), sc.a2[q]), offset);
            }
            const uint64_t aa = f32x2_splat(a);
            constexpr bool kReg = NF4_GEMM_REG_WORDS > 0 && kProducerWarps == 4 && pair_for<BN>() &&
                                  NF4_GEMM_ST_SPLIT != 0;
            // 8-warp groups: this thread's half of the chunk; 4-warp groups: both halves
#pragma unroll
            for (int hh = half; hh < (kProducerWarps == 8 ? half + 1 : 2); ++hh) {
              const uint4 c0 = *reinterpret_cast<const uint4*>(smem_c + cs * kSuperCodeBytes +
                                                               code_chunk_off<SUB>(t, 2 * q + hh));
              // dequantize 32 weights: word jj = (element 2jj) | (element 2jj+1) << 16
              const uint32_t cw[4] = {c0.x, c0.y, c0.z, c0.w};
              const bool first = q == 0 && hh == half;
              if constexpr (pair_for<BN>() && NF4_GEMM_ST_SPLIT != 0) {
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                  const bool reg_word = kReg && cc == 3 && (NF4_GEMM_REG_WORDS >= 2 || hh == 1);
                  if (!NF4_EXP(2) && reg_word) {
                    // 8 weights from the register table: 3-bit plane indices (bit 3 cleared), then
                    // per byte the plane half chosen by bit 3 (selector i + 4 * bit3), then the
                    // low/high byte planes interleaved into (element 2j | element 2j+1 << 16)
                    // register table, built here (short live range under the register cap):
                    // T[v] = RNE16(fl32(lut[v] * a)), the exact words of the pair-table path, as
                    // byte planes -- tl[k] byte i = low byte of T[4k+i], th[k] the high bytes
                    uint32_t tl[4], th[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                      const uint32_t t01 = pack2_rn<BF16>(__fmul_rn(p.lut[4 * k], a), __fmul_rn(p.lut[4 * k + 1], a));
                      const uint32_t t23 =
                          pack2_rn<BF16>(__fmul_rn(p.lut[4 * k + 2], a), __fmul_rn(p.lut[4 * k + 3], a));
                      tl[k] = __byte_perm(t01, t23, 0x6420u);
                      th[k] = __byte_perm(t01, t23, 0x7531u);
                    }
                    const uint32_t x = cw[cc];
                    const uint32_t s7 = x & 0x77777777u;
#pragma unroll
                    for (int hw = 0; hw < 2; ++hw) {
                      const uint32_t sx = hw ? (s7 >> 16) : s7;
                      const uint32_t tx = ((hw ? (x >> 17) : (x >> 1)) & 0x4444u) | 0x3210u;
                      const uint32_t lo = __byte_perm(__byte_perm(tl[0], tl[1], sx), __byte_perm(tl[2], tl[3], sx), tx);
                      const uint32_t hi = __byte_perm(__byte_perm(th[0], th[1], sx), __byte_perm(th[2], th[3], sx), tx);
                      // lo/hi byte i <-> nibble i of the half-word: (elem 1, elem 0, elem 3, elem 2)
                      w[4 * cc + 2 * hw] = __byte_perm(lo, hi, 0x4051u);
                      w[4 * cc + 2 * hw + 1] = __byte_perm(lo, hi, 0x6273u);
                    }
                  } else if (!NF4_EXP(2)) {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                      // row of byte jj of the word, this lane's copy
                      const uint32_t byte = __byte_perm(cw[cc], 0u, 0x4440u + jj);
                      uint64_t v, r;
                      asm("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(ptab_lane + byte * NF4_GEMM_PAIR_ROW));
                      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(v), "l"(aa));   // fl32(NF4[idx] * a), both
                      float ch, cl;
                      asm("mov.b64 {%0, %1}, %2;" : "=f"(ch), "=f"(cl) : "l"(r));
                      w[4 * cc + jj] = pack2_rn<BF16>(ch, cl);
                    }
                  }
                  // store each piece of 16/SPLIT columns as soon as it is complete: its words die,
                  // so more table loads stay in flight under the 72-register cap.  The first
                  // piece of a super-stage is dequantized before waiting for the MMA to release
                  // the A tiles (a warp that ran ahead of its group keeps working).
                  constexpr int kWords = 16 / (NF4_GEMM_ST_SPLIT ? NF4_GEMM_ST_SPLIT : 1), kCc = kWords / 4;
                  if (cc % kCc == kCc - 1) {
                    if (kEarlyFirstPiece && first && cc == kCc - 1) {
                      mbar_wait_parity(&a_free[slot], aph ^ 1u);        // the MMA is done with our previous A tiles
                      if (wl == 0 && lane == 0) NF4_TRACE_J(200, Jg);
                      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    }
                    const int w0 = (cc / kCc) * kWords;
                    const uint32_t taddr = tmem + tlane + uint32_t(A0 + (slot * SUB + q) * 32 + hh * 16 + w0);
                    if (!NF4_EXP(4)) {
                      if constexpr (kWords == 8)
                        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                                     ::"r"(taddr), "r"(w[w0]), "r"(w[w0 + 1]), "r"(w[w0 + 2]), "r"(w[w0 + 3]),
                                     "r"(w[w0 + 4]), "r"(w[w0 + 5]), "r"(w[w0 + 6]), "r"(w[w0 + 7]) : "memory");
                      else
                        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                                     ::"r"(taddr), "r"(w[w0]), "r"(w[w0 + 1]), "r"(w[w0 + 2]), "r"(w[w0 + 3])
                                     : "memory");
                    } else {
                      // store skipped: fold the words into a never-taken shared store so the
                      // lookups are not dead code (ptxas removes anything without a side effect)
                      uint32_t x = 0;
#pragma unroll
                      for (int k = 0; k < kWords; ++k) x ^= w[w0 + k];
                      if (x == 0x7FC00001u) *reinterpret_cast<volatile uint32_t*>(&exp_sink) = x;
                    }
                  }
                }
              } else {
                if (!NF4_EXP(2)) {
#pragma unroll
                  for (int cc = 0; cc < 4; ++cc) {
                    if constexpr (pair_for<BN>()) {
#pragma unroll
                      for (int jj = 0; jj < 4; ++jj) {
                        const uint32_t byte = __byte_perm(cw[cc], 0u, 0x4440u + jj);
                        uint64_t v, r;
                        asm("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(ptab_lane + byte * NF4_GEMM_PAIR_ROW));
                        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(v), "l"(aa));
                        float ch, cl;
                        asm("mov.b64 {%0, %1}, %2;" : "=f"(ch), "=f"(cl) : "l"(r));
                        w[4 * cc + jj] = pack2_rn<BF16>(ch, cl);
                      }
                    } else {
                      const uint32_t x = cw[cc];
                      const uint32_t hi4 = (x >> 2) & 0x3C3C3C3Cu;  // byte jj = 4 * high nibble (LUT byte offset)
                      const uint32_t lo4 = (x << 2) & 0x3C3C3C3Cu;  // byte jj = 4 * low nibble
#pragma unroll
                      for (int jj = 0; jj < 4; ++jj) {
                        // shared address of NF4[idx] = lut_base with byte 0 replaced by byte jj of hi4/lo4: one PRMT
                        const uint32_t ah = __byte_perm(hi4, lut_base, 0x7650u + jj);
                        const uint32_t al = __byte_perm(lo4, lut_base, 0x7650u + jj);
                        float ch, cl;
                        asm("ld.shared.f32 %0, [%1];" : "=f"(ch) : "r"(ah));
                        asm("ld.shared.f32 %0, [%1];" : "=f"(cl) : "r"(al));
                        mul2_rn(ch, cl, aa);                      // fl32(NF4[idx] * a) for both, one FMUL2
                        w[4 * cc + jj] = pack2_rn<BF16>(ch, cl);
                      }
                    }
                  }
                }
                if (kEarlyFirstPiece && first) {
                  mbar_wait_parity(&a_free[slot], aph ^ 1u);              // the MMA is done with our previous A tiles
                  if (wl == 0 && lane == 0) NF4_TRACE_J(200, Jg);
                  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                if (!NF4_EXP(4)) {
                  // 16 columns (32 weights) of this row's A tile (group g, chunk q) in TMEM
                  const uint32_t taddr = tmem + tlane + uint32_t(A0 + (slot * SUB + q) * 32 + hh * 16);
                  asm volatile(
                      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                      ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                      "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
                      : "memory");
                } else {
                  uint32_t x = 0;                           // keep the lookups live (see above)
#pragma unroll
                  for (int k = 0; k < 16; ++k) x ^= w[k];
                  if (x == 0x7FC00001u) *reinterpret_cast<volatile uint32_t*>(&exp_sink) = x;
                }
              }
            }
          }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        const bool full = (j + 1) * SUB <= nk;
        if (absmax != nullptr) {
          if (full) stage(T_{}, std::integral_constant<int, 0>{}); else stage(F_{}, std::integral_constant<int, 0>{});
        } else if (fast) {
          if (full) stage(T_{}, std::integral_constant<int, 1>{}); else stage(F_{}, std::integral_constant<int, 1>{});
        } else {
          if (full) stage(T_{}, std::integral_constant<int, 2>{}); else stage(F_{}, std::integral_constant<int, 2>{});
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (wl == 0 && lane == 0) NF4_TRACE_J(300, Jg);
        if (lane == 0) mbar_arrive(&w_full[slot]);   // A tiles written, codes read
      }

      // ======================= epilogue (the group of the segment's last super-stage) =======================
      const int jlast = J + (nsuper > 0 ? nsuper - 1 : 0);
      if (jlast % G == g) {
        const int ab = sidx % NACC;
        // acc_full[ab] may only be polled for segment sidx once the previous segment on
        // this accumulator (sidx - NACC) has been committed: a group can be several short
        // segments ahead of the MMA, and a parity wait sees one phase back.  That
        // segment's epilogue waited for its commit, so wait for the epilogue (a monotone
        // count of finished epilogue warps per accumulator: no phase ambiguity).
        if (NF4_GEMM_ACC_GUARD && sidx >= NACC) {
          const int need = (sidx / NACC) * kProducerWarps;
          while (true) {
            int v;
            asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&epi_done[ab]))
                         : "memory");
            if (v >= need) break;
            __nanosleep(32);
          }
        }
        mbar_wait_parity(&acc_full[ab], uint32_t(sidx / NACC) & 1u);
        asm volatile("griddepcontrol.wait;" ::: "memory");   // y / partials / counters: the previous kernel is done
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int qd = wl & 3;                           // TMEM lane quarter this warp may access
        // columns per warp (8-warp groups, BN = 16: warps 4-7 idle; 4-warp groups: all BN)
        constexpr int HB = kProducerWarps == 4 ? BN : (BN / 2 < 16 ? 16 : BN / 2);
        const int col0 = half * HB;
        const int n = sg.n0 + qd * 32 + lane;
        const uint32_t taddr = tmem + (uint32_t(qd * 32) << 16) + uint32_t(ab * ACC);
        const bool direct = p.streamk ? (sg.kc0 == 0 && nk == sg.nkt) : p.splits == 1;
        void* ym = p.mem[sg.g].y;
#pragma unroll 1
        for (int cb = col0; cb < col0 + HB && cb < BN; cb += 16) {
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(taddr + cb));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (n < Nm) {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int m = sg.m0 + cb + jj;
              if (m < p.M) {
                const float acc = nk > 0 ? __uint_as_float(v[jj]) : 0.0f;
                if (!direct) {
                  p.partial[(int64_t(sg.part) * p.M + m) * p.Npad + sg.tn * 128 + qd * 32 + lane] = acc;
                } else if (p.out_dtype == NF4_F32) {
                  static_cast<float*>(ym)[int64_t(m) * Nm + n] = acc;
                } else {
                  static_cast<uint16_t*>(ym)[int64_t(m) * Nm + n] =
                      p.out_dtype == NF4_BF16 ? cvt1_rn<true>(acc) : cvt1_rn<false>(acc);
                }
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&acc_empty[ab]);                   // the MMA may reuse this accumulator
          asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"(smem_u32(&epi_done[ab])) : "memory");
        }
        if (p.streamk && !direct && sg.kc0 + nk < sg.nkt) {
          // a non-final piece: publish (release) -- the tile's last CTA sums it at its end
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(p.flags + sg.ft, 1u);
        }
        if (NF4_TRACING && wl == 0 && lane == 0) p.trace[1024 + 4 * cta_lin + 3] = gtimer();
      }
      J += nsuper;
      ++sidx;
    }
#undef absmax
#undef qabsmax
#undef absmax2
  } else if (warp == kTmaWarp) {
    // ======================= TMA issuer (one thread) =======================
    // Codes of super-stage Jg -> c_full[Jg % CST], X -> x_full[Jg % CST].  The
    // codes of the first CST super-stages (slots initially free) are issued
    // before griddepcontrol.wait; X only after it.
    if (lane == 0) {
      const bool ld_c = !(NF4_EXP(16)), ld_x = !(NF4_EXP(8));
      auto issue_codes = [&](const Segment& sg, int j, int cs) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&c_full[cs])),
                     "r"(uint32_t(ld_c ? kSuperCodeBytes : 0)) : "memory");
        if (ld_c) tma_load_2d(smem_c + cs * kSuperCodeBytes, &maps.c[sg.g], (sg.kc0 + j * SUB) * kChunk / 2, sg.n0,
                              &c_full[cs]);
      };
      int J = 0;
      SegIter it = seg_begin(p, sk_range);
      Segment sg;
      while (J < CST && next_segment<BN>(p, it, sg)) {
        const int nsuper = (sg.nk + SUB - 1) / SUB;
        for (int j = 0; j < nsuper && J + j < CST; ++j) issue_codes(sg, j, J + j);
        J += nsuper;
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");   // X is the previous kernel's output
      J = 0;
      it = seg_begin(p, sk_range);
      while (next_segment<BN>(p, it, sg)) {
        const int nsuper = (sg.nk + SUB - 1) / SUB;
        for (int j = 0; j < nsuper; ++j) {
          const int Jg = J + j, cs = Jg % CST;
          if (Jg >= CST) {
            mbar_wait_parity(&c_free[cs], (uint32_t(Jg / CST) & 1u) ^ 1u);   // super-stage Jg-CST consumed
            issue_codes(sg, j, cs);
          }
          NF4_TRACE_J(400, Jg);
          const int k0 = (sg.kc0 + j * SUB) * kChunk;
          asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
              smem_u32(&x_full[cs])), "r"(uint32_t(ld_x ? kSuperXBytes : 0)) : "memory");
          if (ld_x) {
#pragma unroll
            for (int q = 0; q < SUB; ++q)
              tma_load_2d(smem_x + cs * kSuperXBytes + q * BN * kRowBytes, &maps.x[sg.g], k0 + q * kChunk, sg.m0,
                          &x_full[cs]);
          }
        }
        J += nsuper;
      }
    }
  } else {
    // ======================= MMA issuer (whole warp, one elected lane issues) =======================
    const uint32_t idesc = umma_idesc(BN, BF16);
    int J = 0, sidx = 0;
    SegIter it = seg_begin(p, sk_range);
    Segment sg;
    while (next_segment<BN>(p, it, sg)) {
      const int nsuper = (sg.nk + SUB - 1) / SUB;
      const int ab = sidx % NACC;
      mbar_wait_parity(&acc_empty[ab], (uint32_t(sidx / NACC) & 1u) ^ 1u);   // its previous epilogue done
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d_tmem = tmem + uint32_t(ab * ACC);
      for (int j = 0; j < nsuper; ++j) {
        const int Jg = J + j, slot = Jg % S, cs = Jg % CST;
        mbar_wait_parity(&w_full[slot], uint32_t(Jg / S) & 1u);            // A tiles in TMEM
        mbar_wait_parity(&x_full[cs], uint32_t(Jg / CST) & 1u);            // X of this super-stage landed
        if (lane == 0) NF4_TRACE_J(500, Jg);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (!(NF4_EXP(1))) {
          const uint64_t b0 = umma_desc_sw128(smem_u32(smem_x + cs * kSuperXBytes));
          const uint32_t a0 = tmem + uint32_t(A0 + slot * SUB * 32);
#pragma unroll
          for (int q = 0; q < SUB; ++q) {
            if (j * SUB + q < sg.nk)
              umma_chunk_elect(d_tmem, a0 + q * 32, b0 + uint64_t(q * BN * kRowBytes / 16), idesc,
                               (j > 0 || q > 0) ? 1u : 0u);
          }
        }
        umma_commit_elect(&a_free[slot]);
        umma_commit_elect(&c_free[cs]);
      }
      if (nsuper > 0)
        umma_commit_elect(&acc_full[ab]);
      else if (lane == 0)
        mbar_arrive(&acc_full[ab]);
      J += nsuper;
      ++sidx;
    }
    __syncwarp();
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // (a no-op for threads that already waited)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (p.streamk) {
    // ======================= stream-K fix-up of the tile this range finishes =======================
    const int x0 = sk_range[0], parts = sk_range[2] + 1;
    const TileAt t = tile_at(p, x0 < p.total_chunks ? x0 : 0);
    const int kc0 = x0 - t.tstart;
    if (x0 < sk_range[1] && kc0 > 0 && sk_range[1] >= t.tstart + t.nkt) {
      unsigned* flag = p.flags + p.mem[t.g].ftile0 + t.tl;
      if (threadIdx.x == 0) {
        const unsigned want = unsigned(kProducerWarps * (parts - 1));
        unsigned v;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
          if (v >= want) break;
          __nanosleep(64);
        }
        *flag = 0u;                                   // leave the workspace clean for the next call
      }
      __syncthreads();
      const int gm = t.g, tiles_n = p.mem[gm].tiles_n;
      const int tn = p.mem[gm].tile0 + t.tl % tiles_n;
      const int n0 = (t.tl % tiles_n) * 128, m0 = (t.tl / tiles_n) * BN;
      const int Nm = p.mem[gm].N;
      void* ym = p.mem[gm].y;
      const int rows = min(BN, p.M - m0);
      const int64_t mn = int64_t(p.M) * p.Npad;
      for (int e = threadIdx.x; e < rows * 128; e += blockDim.x) {
        const int m = m0 + (e >> 7), n = n0 + (e & 127);
        if (n >= Nm) continue;
        const int64_t i = int64_t(m) * p.Npad + tn * 128 + (e & 127);
        float acc = __ldcg(p.partial + i);
        for (int s2 = 1; s2 < parts; ++s2) acc = __fadd_rn(acc, __ldcg(p.partial + s2 * mn + i));
        const int64_t o = int64_t(m) * Nm + n;
        if (p.out_dtype == NF4_F32)
          static_cast<float*>(ym)[o] = acc;
        else
          static_cast<uint16_t*>(ym)[o] = p.out_dtype == NF4_BF16 ? cvt1_rn<true>(acc) : cvt1_rn<false>(acc);
      }
    }
  }
  if (NF4_TRACING && threadIdx.x == 0) p.trace[1024 + 4 * cta_lin + 1] = gtimer();
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Deterministic reductions of the fp32 partials.
// classic: y[m, n] = sum_s partial[s, m, n] in split order.
// (classic split-K, one member; partial rows have stride Npad >= N)
__global__ void nf4_gemm_reduce_kernel(const float* __restrict__ partial, int splits, int M, int N, int Npad, void* y,
                                       int out_dtype) {
  const int64_t mn = int64_t(M) * N, mnp = int64_t(M) * Npad;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < mn; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = (i / N) * Npad + i % N;
    float acc = partial[j];
    for (int s = 1; s < splits; ++s) acc = __fadd_rn(acc, partial[int64_t(s) * mnp + j]);
    if (out_dtype == NF4_F32)
      static_cast<float*>(y)[i] = acc;
    else
      static_cast<uint16_t*>(y)[i] = out_dtype == NF4_BF16 ? cvt1_rn<true>(acc) : cvt1_rn<false>(acc);
  }
}
// Per token-tile width: G producer groups, SUB chunks per super-stage (code box
// width SUB*32 B), CST super-stages in shared memory, NACC accumulators in TMEM.
// With the 32 KB byte-pair table: BN 16: 24 KB x 6;  BN 32: 32 KB x 5;
//   BN 64: 24 KB (2 chunks) x 6;  BN 128: 40 KB (2 chunks) x 4;  BN 256: 36 KB
//   (1 chunk) x 5 (one accumulator: 256 + 3*32 TMEM columns).
// (macros: tuning experiments only, tools/)
#ifndef NF4_GEMM_CST_SMALL
#define NF4_GEMM_CST_SMALL 6
#endif
#ifndef NF4_GEMM_SUB64
#define NF4_GEMM_SUB64 2
#endif
#ifndef NF4_GEMM_CST64
#define NF4_GEMM_CST64 4
#endif
#ifndef NF4_GEMM_SUB128
#define NF4_GEMM_SUB128 2
#endif
#ifndef NF4_GEMM_CST128
#define NF4_GEMM_CST128 4
#endif
#ifndef NF4_GEMM_SUB32
#define NF4_GEMM_SUB32 4
#endif
#ifndef NF4_GEMM_PCST32
#define NF4_GEMM_PCST32 5
#endif
#ifndef NF4_GEMM_PCST64
#define NF4_GEMM_PCST64 6
#endif
#ifndef NF4_GEMM_PCST128
#define NF4_GEMM_PCST128 4
#endif
template <int BN> constexpr int sub_for() {
  if (wpg_for<BN>() == 4) return BN <= 64 ? 2 : 1;   // 6 groups of 4 warps: TMEM holds 6 x SUB A tiles
  return BN <= 16 ? 4 : BN <= 32 ? NF4_GEMM_SUB32 : BN <= 64 ? NF4_GEMM_SUB64 : BN <= 128 ? NF4_GEMM_SUB128 : 1;
}
template <int BN> constexpr int cst_for() {
  if (wpg_for<BN>() == 4) return BN <= 32 ? NF4_GEMM_W4_CST : 6;
  // with the 32 KB pair table: 6 / 5 / 6 (2-chunk) / 4 / 5 stages fit in 227 KB (64 KB table: 6 / 4 / 3 / 3 / 4)
  return pair_for<BN>() ? (NF4_GEMM_PAIR_ROW == 128
                               ? (BN <= 16 ? NF4_GEMM_CST_SMALL : BN <= 32 ? NF4_GEMM_PCST32 : BN <= 64 ? NF4_GEMM_PCST64
                                                                : BN <= 128 ? NF4_GEMM_PCST128 : 5)
                               : (BN <= 16 ? NF4_GEMM_CST_SMALL : BN <= 32 ? 4 : BN <= 64 ? 3 : BN <= 128 ? 3 : 4))
                        : (BN <= 16 ? NF4_GEMM_CST_SMALL : BN <= 32 ? 6 : BN <= 64 ? NF4_GEMM_CST64
                                                                       : BN <= 128 ? NF4_GEMM_CST128 : 5);
}
static int sub_of(int bn) {
  return bn <= 16 ? sub_for<16>() : bn <= 32 ? sub_for<32>() : bn <= 64 ? sub_for<64>() : bn <= 128 ? sub_for<128>()
                                                                                            : sub_for<256>();
}
template <int BN> constexpr int nacc_for() { return BN <= 128 ? 2 : 1; }
template <int BN> constexpr int threads_for() { return 32 * (wpg_for<BN>() * groups_for<BN>() + 2); }

template <int BN>
constexpr size_t smem_bytes() {
  return 1024 /*align slack*/ + pair_table_bytes<BN>() + size_t(cst_for<BN>()) * sub_for<BN>() * (128 * kCodeBytes + BN * kRowBytes);
}

template <int BN, bool BF16, int NM>
constexpr auto kernel_for() {
  return nf4_gemm_kernel<BN, groups_for<BN>(), sub_for<BN>(), cst_for<BN>(), nacc_for<BN>(), BF16, NM>;
}

template <int BN, bool BF16, int NM>
static cudaError_t launch1(const GemmParamsT<kMaxMembers>& pm, const MapsT<kMaxMembers>& mm, dim3 grid,
                           cudaStream_t s) {
  auto k = kernel_for<BN, BF16, NM>();
  // the single-weight kernel takes a 1-member parameter block (less to copy per launch)
  static thread_local GemmParamsT<NM> p;
  static thread_local MapsT<NM> maps;
  static_cast<GemmCommon&>(p) = static_cast<const GemmCommon&>(pm);
  for (int i = 0; i < NM && i < pm.nmem; ++i) {
    p.mem[i] = pm.mem[i];
    maps.c[i] = mm.c[i];
    maps.x[i] = mm.x[i];
  }
  constexpr size_t sm = smem_bytes<BN>();
  // 227 KB per block, minus the static shared memory (LUT, barriers: < 2 KB)
  static_assert(sm + 6 * 1024 <= 232448, "shared-memory budget (stages + pair table) exceeded");
  static_assert(nacc_for<BN>() * (BN < 32 ? 32 : BN) + slots_for<BN>() * sub_for<BN>() * 32 <= 512, "TMEM budget");
  static_assert(cst_for<BN>() >= groups_for<BN>(), "a super-stage slot must not be two phases behind any group");
  static_assert(sizeof(GemmParamsT<NM>) + sizeof(MapsT<NM>) <= 32000, "kernel parameter space");
  // the dynamic shared-memory opt-in is a per-device (per-context) attribute: set it once
  // per device and instantiation, and never cache a failure
  static std::atomic<uint64_t> attr_set{0};  // bit d: set on device d (d < 64; others set every call)
  int dev = 0;
  if (const cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  const uint64_t bit = dev >= 0 && dev < 64 ? uint64_t(1) << dev : 0;
  if (!bit || !(attr_set.load(std::memory_order_acquire) & bit)) {
    const cudaError_t a = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (a != cudaSuccess) return a;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  // launched with programmatic stream serialization (the kernel executes
  // griddepcontrol.wait before reading anything the previous kernel may write)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads_for<BN>());
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, p, maps);
  if (e != cudaSuccess) return e;
  return cudaPeekAtLastError();
}

template <int BN, bool BF16>
static cudaError_t launch(const GemmParamsT<kMaxMembers>& p, const MapsT<kMaxMembers>& m, dim3 grid,
                          cudaStream_t s) {
  return p.nmem == 1 ? launch1<BN, BF16, 1>(p, m, grid, s)
         : p.nmem <= NF4_GEMM_MAX_GROUP ? launch1<BN, BF16, NF4_GEMM_MAX_GROUP>(p, m, grid, s)
                                        : launch1<BN, BF16, kMaxMembers>(p, m, grid, s);
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

// L2 promotion of the TMA requests (none / 64B / 128B measured the same, r01).
static CUtensorMapL2promotion promo() { return CU_TENSOR_MAP_L2_PROMOTION_L2_256B; }

// 2-D tensor map over a row-major [rows, cols] matrix of `elem` bytes.  The last
// encodings are cached per host thread (a decode step re-issues the same weights).
static bool make_map(CUtensorMap* m, CUtensorMapDataType dt, int elem, const void* base, uint64_t cols,
                     uint64_t rows, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  struct Entry {
    const void* base;
    uint64_t cols, rows;
    uint32_t box_cols, box_rows;
    int dt, sw;
    CUtensorMap map;
  };
  constexpr int kCache = 256;   // a 64-problem nf4_gemm_multi call needs up to 128 maps
  thread_local Entry cache[kCache] = {};
  const uint64_t h = (reinterpret_cast<uintptr_t>(base) >> 8) ^ (cols * 0x9E3779B97F4A7C15ull) ^ (rows << 7) ^
                     (uint64_t(box_rows) << 3) ^ uint64_t(dt);
  Entry& c = cache[(h ^ (h >> 29)) % kCache];
  if (c.base == base && c.cols == cols && c.rows == rows && c.box_cols == box_cols && c.box_rows == box_rows &&
      c.dt == int(dt) && c.sw == int(sw)) {
    *m = c.map;
    return true;
  }
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * uint64_t(elem)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
          promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  c.base = base; c.cols = cols; c.rows = rows; c.box_cols = box_cols; c.box_rows = box_rows;
  c.dt = int(dt); c.sw = int(sw); c.map = *m;
  return true;
}

}  // namespace gemm
}  // namespace nf4

using namespace nf4;
using namespace nf4::gemm;

// NF4_GEMM_BN8: token tiles of 8 for M <= 8 (tcgen05.mma kind::f16 with M = 128 takes any N
// multiple of 8): half the X bytes of a 16-wide tile through TMA and the MMA.
#ifndef NF4_GEMM_BN8
#define NF4_GEMM_BN8 0
#endif
static int pick_bn(int M) {
  if (NF4_GEMM_BN8 && M <= 8) return 8;
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128) return 128;
  return 256;
}

static std::atomic<int32_t> g_early_weights{1};

// One problem as the host sees it: Y = X . W^T, W an NF4 weight [N, K].
struct HostMember {
  const void* x;
  int32_t K;
  const uint8_t* packed;
  const float* absmax;
  const nf4_dq_state* dq;
  int32_t N;
  void* y;
};

// Stream-K geometry over the member-major chunk stream: G resident CTAs (at most
// one per 4 chunks so every range is non-empty), W chunks in total, and the
// largest number of segments any tile is split into (= partial slots the
// workspace needs).
struct SkGeom {
  int bn, tiles_m, tiles_n, tiles, align4, nk_max;
  int64_t W, G;
  int max_parts;
};
static SkGeom sk_geometry(int M, const int32_t* N, const int32_t* K, int count) {
  SkGeom g;
  g.bn = pick_bn(M);
  g.tiles_m = (M + g.bn - 1) / g.bn;
  g.tiles_n = 0;
  g.align4 = 1;
  g.nk_max = 0;
  g.W = 0;
  for (int i = 0; i < count; ++i) {
    if (N[i] <= 0) continue;
    const int tn = (N[i] + 127) / 128, nk = K[i] / 64;
    g.tiles_n += tn;
    g.W += int64_t(tn) * g.tiles_m * nk;
    g.align4 = g.align4 && (nk % 4) == 0;
    g.nk_max = nk > g.nk_max ? nk : g.nk_max;
  }
  g.tiles = g.tiles_n * g.tiles_m;
  const int64_t cap = sm_count();   // one CTA per SM (the kernel's producer groups fill it)
  const int64_t lim = g.align4 ? g.W / 4 : g.W;
  g.G = cap < lim ? cap : lim;
  if (g.G < 1) g.G = 1;
  // Upper bound on the pieces of one tile (sizes the workspace; O(1) on the host):
  // every range but the first touching a tile holds >= Lmin of its chunks.
  int64_t lmin = g.W / g.G - (g.align4 ? 4 : 0);
  if (lmin < (g.align4 ? 4 : 1)) lmin = g.align4 ? 4 : 1;
  int64_t mp = 1 + (g.nk_max - 1 + lmin - 1) / lmin;
  if (mp > g.G) mp = g.G;
  g.max_parts = int(mp);
  return g;
}

// Workspace head: one counter per tile (stream-K), 256-B rounded; the fp32
// partials (stream-K pieces or classic splits) always start after it, so a
// classic call never writes where a later stream-K call expects zero counters.
static int64_t flag_bytes(int64_t tiles) { return (tiles * 4 + 255) / 256 * 256; }

// Stream-K workspace, -1 when the chunk stream exceeds the kernel's 32-bit indices
// (a single weight then takes the classic grid).
static int64_t streamk_ws_bytes(int M, const int32_t* N, const int32_t* K, int count) {
  const SkGeom g = sk_geometry(M, N, K, count);
  if (g.W >= (int64_t(1) << 31)) return -1;
  return g.max_parts > 1 ? flag_bytes(g.tiles) + int64_t(g.max_parts) * M * g.tiles_n * 128 * 4 : 0;
}

static int64_t npad_of(int32_t N) { return int64_t((N + 127) / 128) * 128; }

static int64_t classic_ws_bytes(int M, int N, int splits) {
  if (splits <= 1) return 0;
  const int64_t tiles = ((N + 127) / 128) * int64_t((M + pick_bn(M) - 1) / pick_bn(M));
  return flag_bytes(tiles) + int64_t(splits) * M * npad_of(N) * 4;
}

extern "C" int64_t nf4_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K, int32_t splits) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  if (splits <= 0) {
    if (K % 64 != 0) return 0;
    const int64_t b = streamk_ws_bytes(M, &N, &K, 1);
    if (b >= 0) return b;
    splits = nf4_gemm_default_splits(M, N, K);   // classic fallback (nf4_gemm does the same)
  }
  return classic_ws_bytes(M, N, splits);
}

extern "C" int64_t nf4_gemm_grouped_workspace_bytes(int32_t M, const int32_t* N, int32_t count, int32_t K) {
  if (M <= 0 || K <= 0 || K % 64 != 0 || !N || count <= 0 || count > NF4_GEMM_MAX_GROUP) return 0;
  int32_t Ks[NF4_GEMM_MAX_GROUP];
  for (int i = 0; i < count; ++i) {
    if (N[i] <= 0) return 0;
    Ks[i] = K;
  }
  const int64_t b = streamk_ws_bytes(M, N, Ks, count);
  return b > 0 ? b : 0;
}

extern "C" int64_t nf4_gemm_multi_workspace_bytes(int32_t M, const int32_t* N, const int32_t* K, int32_t count) {
  if (M <= 0 || !N || !K || count <= 0 || count > NF4_GEMM_MAX_MULTI) return 0;
  // problems with no work (N == 0 or K == 0) take no tiles, exactly as nf4_gemm_multi skips them
  int32_t n[NF4_GEMM_MAX_MULTI], k[NF4_GEMM_MAX_MULTI];
  int c = 0;
  for (int i = 0; i < count; ++i) {
    if (N[i] < 0 || K[i] < 0 || K[i] % 64 != 0) return 0;
    if (N[i] == 0 || K[i] == 0) continue;
    n[c] = N[i];
    k[c++] = K[i];
  }
  if (c == 0) return 0;
  const int64_t b = streamk_ws_bytes(M, n, k, c);
  return b > 0 ? b : 0;
}

// Split-K factor minimising the makespan of the (row tile, token tile, split)
// grid on this GPU: waves x (chunks per split + ~2 chunks of per-CTA prologue
// and epilogue), preferring fewer splits on near ties (less partial traffic).
extern "C" int32_t nf4_gemm_default_splits(int32_t M, int32_t N, int32_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 1;
  const int bn = pick_bn(M);
  const int64_t tiles = int64_t((N + 127) / 128) * ((M + bn - 1) / bn);
  const int64_t cap = sm_count();
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

static nf4_status check_member(const HostMember& m, nf4_dtype y_dtype, int32_t blocksize) {
  if (m.N < 0 || m.K < 0) return NF4_ERR_BAD_SIZE;
  if ((m.absmax == nullptr) == (m.dq == nullptr)) return NF4_ERR_BAD_STATE;
  if (m.dq && m.dq->blocksize2 != 256) return NF4_ERR_BAD_STATE;
  if (m.N == 0) return NF4_OK;
  if (m.K % 64 != 0 || m.K % blocksize != 0) return NF4_ERR_BAD_SIZE;  // a 64-chunk never spans two blocks
  if (!m.packed || !m.y || !m.x) return NF4_ERR_NULL_POINTER;
  if (m.dq && (!m.dq->qabsmax || !m.dq->code2 || !m.dq->absmax2)) return NF4_ERR_NULL_POINTER;
  if (!aligned(m.packed, 16) || !aligned(m.x, 16)) return NF4_ERR_MISALIGNED;
  if (!aligned(m.y, y_dtype == NF4_F32 ? 4 : 2)) return NF4_ERR_MISALIGNED;
  if (m.absmax && !aligned(m.absmax, 4)) return NF4_ERR_MISALIGNED;
  return NF4_OK;
}

static nf4_status gemm_run(nf4_dtype x_dtype, int32_t M, int32_t blocksize, const HostMember* mem_in,
                           int32_t count, nf4_dtype y_dtype, int32_t splits, void* workspace,
                           int64_t workspace_bytes, void* stream) {
  if (M < 0 || count < 1 || count > kMaxMembers) return NF4_ERR_BAD_SIZE;
  if (x_dtype != NF4_F16 && x_dtype != NF4_BF16) return NF4_ERR_BAD_DTYPE;
  if (y_dtype != NF4_F16 && y_dtype != NF4_BF16 && y_dtype != NF4_F32) return NF4_ERR_BAD_DTYPE;
  if (!is_pow2(blocksize) || blocksize < 64 || blocksize > 4096) return NF4_ERR_BAD_BLOCKSIZE;
  for (int i = 0; i < count; ++i) {
    if (mem_in[i].K < 0 || mem_in[i].N < 0) return NF4_ERR_BAD_SIZE;
    if (M == 0 || mem_in[i].N == 0 || mem_in[i].K == 0) {
      // nothing to compute, but the state must still be consistent
      if ((mem_in[i].absmax == nullptr) == (mem_in[i].dq == nullptr)) return NF4_ERR_BAD_STATE;
      if (mem_in[i].dq && mem_in[i].dq->blocksize2 != 256) return NF4_ERR_BAD_STATE;
      if (mem_in[i].K % 64 != 0 || mem_in[i].K % blocksize != 0) return NF4_ERR_BAD_SIZE;
      if (M > 0 && mem_in[i].N > 0) {   // K == 0: Y = 0 is written
        if (!mem_in[i].y) return NF4_ERR_NULL_POINTER;
        if (!aligned(mem_in[i].y, y_dtype == NF4_F32 ? 4 : 2)) return NF4_ERR_MISALIGNED;
      }
      continue;
    }
    const nf4_status st = check_member(mem_in[i], y_dtype, blocksize);
    if (st != NF4_OK) return st;
  }
  // problems with N == 0 or K == 0 contribute no tiles (K == 0 with N > 0: Y = 0,
  // written after every argument has been validated)
  HostMember mem[kMaxMembers];
  int nmem = 0, nzero = 0;
  for (int i = 0; i < count; ++i) {
    if (M == 0 || mem_in[i].N == 0) continue;
    if (mem_in[i].K == 0) { ++nzero; continue; }
    mem[nmem++] = mem_in[i];
  }
  auto zero_fill = [&]() -> bool {
    for (int i = 0; i < count && nzero > 0; ++i)
      if (M > 0 && mem_in[i].N > 0 && mem_in[i].K == 0 &&
          cudaMemsetAsync(mem_in[i].y, 0, size_t(M) * mem_in[i].N * (y_dtype == NF4_F32 ? 4 : 2),
                          static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return false;
    return true;
  };
  if (nmem == 0) {
    if (!zero_fill()) { cudaGetLastError(); return NF4_ERR_CUDA; }
    set_launch_count(0);
    return NF4_OK;
  }
  const int bn = pick_bn(M);
  int32_t Ns[kMaxMembers], Ks[kMaxMembers];
  for (int i = 0; i < nmem; ++i) { Ns[i] = mem[i].N; Ks[i] = mem[i].K; }
  const SkGeom g = sk_geometry(M, Ns, Ks, nmem);
  const int64_t npad = int64_t(g.tiles_n) * 128;
  // stream-K chunk indices are 32-bit in the kernel; beyond that, the classic grid (one weight only)
  const bool streamk = (splits <= 0 || nmem > 1) && g.W < (int64_t(1) << 31);
  if (!streamk && nmem > 1) return NF4_ERR_BAD_SIZE;
  const int nk0 = mem[0].K / 64;
  if (splits <= 0 && !streamk) splits = nf4_gemm_default_splits(M, mem[0].N, mem[0].K);
  if (streamk) {
    if (g.max_parts > 1) {
      if (!workspace) return NF4_ERR_NULL_POINTER;
      if (workspace_bytes < flag_bytes(g.tiles) + int64_t(g.max_parts) * M * npad * 4) return NF4_ERR_BAD_STATE;
      if (!aligned(workspace, 16)) return NF4_ERR_MISALIGNED;
    }
    splits = 1;
  } else {
    if (splits <= 0) splits = 1;
    if (splits > nk0) splits = nk0 > 0 ? nk0 : 1;
  }
  static thread_local GemmParamsT<kMaxMembers> p;
  int tile0 = 0, ftile0 = 0, cbase = 0;
  for (int i = 0; i < nmem; ++i) {
    Member& m = p.mem[i];
    m.absmax = mem[i].absmax;
    m.qabsmax = mem[i].dq ? mem[i].dq->qabsmax : nullptr;
    m.code2 = mem[i].dq ? mem[i].dq->code2 : nullptr;
    m.absmax2 = mem[i].dq ? mem[i].dq->absmax2 : nullptr;
    m.offset = mem[i].dq ? mem[i].dq->offset : 0.0f;
    m.N = mem[i].N;
    m.y = mem[i].y;
    m.K = mem[i].K;
    m.nk = mem[i].K / 64;
    m.tiles_n = (mem[i].N + 127) / 128;
    m.tile0 = tile0;
    m.ftile0 = ftile0;
    m.cbase = cbase;
    tile0 += m.tiles_n;
    ftile0 += m.tiles_n * g.tiles_m;
    cbase += m.tiles_n * g.tiles_m * m.nk;
  }
  p.nmem = nmem;
  p.partial = static_cast<float*>(workspace);
  p.flags = nullptr;
  if (streamk && g.max_parts > 1) {
    p.flags = static_cast<unsigned*>(workspace);
    p.partial = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + flag_bytes(g.tiles));
  }
  p.M = M;
  p.Npad = int32_t(npad);
  p.bs_shift = log2i(blocksize);
  const int sub = sub_of(bn);
  {
    // whole super-stages per split (SUB chunks share one TMA box); splits = non-empty ranges
    int cps = (nk0 + splits - 1) / splits;
    cps = (cps + sub - 1) / sub * sub;
    splits = (nk0 + cps - 1) / cps;
    p.chunks_per_split = cps;
  }
  p.splits = splits;
  if (!streamk && splits > 1) {
    if (!workspace) return NF4_ERR_NULL_POINTER;
    if (workspace_bytes < classic_ws_bytes(M, mem[0].N, splits)) return NF4_ERR_BAD_STATE;
    if (!aligned(workspace, 16)) return NF4_ERR_MISALIGNED;
    p.partial = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + flag_bytes(g.tiles));
  }
  p.out_dtype = int(y_dtype);
  p.streamk = streamk ? 1 : 0;
  p.tiles_m = g.tiles_m;
  p.total_chunks = g.W;
  p.align4 = streamk ? g.align4 : 0;
  p.early_weights = g_early_weights.load(std::memory_order_relaxed);
  p.trace = nullptr;
  p.experiment = 0;
#if NF4_GEMM_DIAG
  if (const char* tr = getenv("NF4_GEMM_TRACE")) p.trace = reinterpret_cast<unsigned long long*>(strtoull(tr, 0, 0));
  if (const char* ex = getenv("NF4_GEMM_EXPERIMENT")) p.experiment = atoi(ex);
#endif
  nf4_codebook(p.lut);
  dim3 grid = streamk ? dim3(unsigned(g.G), 1, 1) : dim3(unsigned(g.tiles_n), unsigned(g.tiles_m), unsigned(splits));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool bf16 = x_dtype == NF4_BF16;
  static thread_local MapsT<kMaxMembers> maps;
  const CUtensorMapSwizzle csw = sub == 4 ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : sub == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  for (int i = 0; i < nmem; ++i) {
    if (!make_map(&maps.c[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, mem[i].packed, uint64_t(mem[i].K) / 2,
                  uint64_t(mem[i].N), uint32_t(sub * kCodeBytes), 128, csw))
      return NF4_ERR_CUDA;
    if (i > 0 && mem[i].x == mem[i - 1].x && mem[i].K == mem[i - 1].K) {
      maps.x[i] = maps.x[i - 1];
    } else if (!make_map(&maps.x[i], bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                         mem[i].x, uint64_t(mem[i].K), uint64_t(M), kChunk, uint32_t(bn),
                         CU_TENSOR_MAP_SWIZZLE_128B)) {
      return NF4_ERR_CUDA;
    }
  }
  if (!zero_fill()) { cudaGetLastError(); return NF4_ERR_CUDA; }
  cudaError_t e;
  switch (bn) {
#if NF4_GEMM_BN8
    case 8: e = bf16 ? launch<8, true>(p, maps, grid, s) : launch<8, false>(p, maps, grid, s); break;
#endif
    case 16: e = bf16 ? launch<16, true>(p, maps, grid, s) : launch<16, false>(p, maps, grid, s); break;
    case 32: e = bf16 ? launch<32, true>(p, maps, grid, s) : launch<32, false>(p, maps, grid, s); break;
    case 64: e = bf16 ? launch<64, true>(p, maps, grid, s) : launch<64, false>(p, maps, grid, s); break;
    case 128: e = bf16 ? launch<128, true>(p, maps, grid, s) : launch<128, false>(p, maps, grid, s); break;
    default: e = bf16 ? launch<256, true>(p, maps, grid, s) : launch<256, false>(p, maps, grid, s); break;
  }
  if (e != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
  int launches = 1;
  if (!streamk && splits > 1) {
    const int64_t mn = int64_t(M) * mem[0].N;
    int64_t gr = (mn + 255) / 256;
    if (gr > int64_t(sm_count()) * 8) gr = int64_t(sm_count()) * 8;
    nf4_gemm_reduce_kernel<<<int(gr), 256, 0, s>>>(p.partial, splits, M, mem[0].N, int(npad), mem[0].y,
                                                   int(y_dtype));
    if (cudaPeekAtLastError() != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
    ++launches;
  }
  set_launch_count(launches);
  return NF4_OK;
}

extern "C" nf4_status nf4_gemm(const void* x, nf4_dtype x_dtype, int32_t M, const uint8_t* packed,
                               const float* absmax, const nf4_dq_state* dq, int32_t N, int32_t K, int32_t blocksize,
                               void* y, nf4_dtype y_dtype, int32_t splits, void* workspace,
                               int64_t workspace_bytes, void* stream) {
  if (N < 0 || K < 0) return NF4_ERR_BAD_SIZE;
  const HostMember m{x, K, packed, absmax, dq, N, y};
  return gemm_run(x_dtype, M, blocksize, &m, 1, y_dtype, splits, workspace, workspace_bytes, stream);
}

extern "C" nf4_status nf4_gemm_grouped(const void* x, nf4_dtype x_dtype, int32_t M, int32_t K, int32_t blocksize,
                                       const nf4_gemm_weight* weights, int32_t count, nf4_dtype y_dtype,
                                       void* workspace, int64_t workspace_bytes, void* stream) {
  if (count < 1 || count > NF4_GEMM_MAX_GROUP) return NF4_ERR_BAD_SIZE;
  if (!weights) return NF4_ERR_NULL_POINTER;
  if (K < 0) return NF4_ERR_BAD_SIZE;
  HostMember m[NF4_GEMM_MAX_GROUP];
  for (int i = 0; i < count; ++i) {
    const nf4_gemm_weight& w = weights[i];
    m[i] = HostMember{x, K, w.packed, w.absmax, w.absmax ? nullptr : &w.dq, w.N, w.y};
  }
  return gemm_run(x_dtype, M, blocksize, m, count, y_dtype, 0, workspace, workspace_bytes, stream);
}

extern "C" nf4_status nf4_gemm_multi(const nf4_gemm_problem* problems, int32_t count, int32_t M, nf4_dtype x_dtype,
                                     int32_t blocksize, nf4_dtype y_dtype, void* workspace, int64_t workspace_bytes,
                                     void* stream) {
  if (count < 1 || count > NF4_GEMM_MAX_MULTI) return NF4_ERR_BAD_SIZE;
  if (!problems) return NF4_ERR_NULL_POINTER;
  HostMember m[NF4_GEMM_MAX_MULTI];
  for (int i = 0; i < count; ++i) {
    const nf4_gemm_problem& q = problems[i];
    m[i] = HostMember{q.x, q.K, q.packed, q.absmax, q.absmax ? nullptr : &q.dq, q.N, q.y};
  }
  return gemm_run(x_dtype, M, blocksize, m, count, y_dtype, 0, workspace, workspace_bytes, stream);
}

extern "C" void nf4_gemm_set_early_weight_reads(int32_t enable) {
  g_early_weights.store(enable ? 1 : 0, std::memory_order_relaxed);
}
