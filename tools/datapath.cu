// datapath.cu -- does the F1 GEMM's TMEM hand-off (tcgen05.st) share the SM's
// shared-memory data path with its byte-pair table lookups (LDS.64)?
// One CTA per SM, NW warps; every warp loops over a fixed instruction mix and
// the kernel reports per-SM bytes per clock of each kind (clock64 per CTA,
// averaged).  Modes:
//   0  tcgen05.st.32x32b.x8 only (4 per iteration = 32 columns, then wait::st)
//   1  LDS.64 only (16 per iteration, byte-pair-table addressing, one copy per half-warp lane)
//   2  16 LDS.64 + 2 tcgen05.st.x8 per iteration (F1's ratio: 32 weights per thread)
//   3  tcgen05.st.32x32b.x16 only (2 per iteration)
//   4  tcgen05.st.32x32b.x32 only (1 per iteration)
//   5  F1's inner loop: 16 x (PRMT, LDS.64, FMUL2, cvt.bf16x2) + 2 tcgen05.st.x8
//   6  mode 5 without the stores (words folded into a sink)
//   7  tcgen05.st.16x256b.x2 only (2 per iteration = 32 columns... 16 lanes x 256 b x 2)
//   8  16 SHFL.IDX table lookups (lane i holds level i & 15, source lane = 4-bit code)
//   9  8 SHFL + 8 LDS.64;  10  16 SHFL + 16 LDS.64 (do shuffles share the LDS data path?)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o datapath datapath.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e = (x);                                                                        \
    if (e != cudaSuccess) {                                                                     \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));         \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

__device__ __forceinline__ void st_x8(uint32_t ta, const uint32_t* w) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
}
__device__ __forceinline__ void st_x16(uint32_t ta, const uint32_t* w) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]) : "memory");
}
__device__ __forceinline__ void st_x32(uint32_t ta, const uint32_t* w) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]),
      "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]),
      "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]) : "memory");
}
__device__ __forceinline__ void st_16x256_x2(uint32_t ta, const uint32_t* w) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_dp(int iters, int nw, unsigned long long* cyc, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];   // 32 KB pair table
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = 1.0f + 0.001f * float(i & 255);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&holder)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = holder;
  const uint32_t ta = tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 32 % 512);
  const uint32_t tab = (uint32_t)__cvta_generic_to_shared(smem) + uint32_t(lane % 16) * 8u;
  uint32_t v = 0x9E3779B9u * (threadIdx.x + 1);
  uint32_t w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) w[i] = v + i;
  const uint64_t aa = 0x3f8000003f800000ull;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int s = 0; s < 4; ++s) st_x8(ta + 8 * s, w + 8 * s);
      st_wait();
    } else if (MODE == 3) {
      st_x16(ta, w);
      st_x16(ta + 16, w + 16);
      st_wait();
    } else if (MODE == 4) {
      st_x32(ta, w);
      st_wait();
    } else if (MODE == 7) {
      st_16x256_x2(ta, w);
      st_16x256_x2(ta + 8, w + 8);
      st_16x256_x2(ta + 16, w + 16);
      st_16x256_x2(ta + 24, w + 24);
      st_wait();
    } else if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const uint32_t byte = (v >> (2 * q)) & 255u;
        uint64_t r;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r) : "r"(tab + byte * 128u));
        w[q] ^= uint32_t(r) ^ uint32_t(r >> 32);
      }
      if (MODE == 2) {
        st_x8(ta, w);
        st_x8(ta + 8, w + 8);
        st_wait();
      }
      v = v * 1664525u + 1013904223u + w[3];
    } else if (MODE == 8 || MODE == 9 || MODE == 10) {
      // 8: 16 SHFL.IDX lookups (lane i holds NF4[i & 15]; source lane = a 4-bit code)
      // 9: 8 LDS.64 + 8 SHFL per iteration; 10: 16 LDS.64 + 16 SHFL
      const float tabv = 1.0f + 0.01f * float(lane & 15);
#pragma unroll
      for (int q = 0; q < (MODE == 10 ? 16 : MODE == 9 ? 8 : 16); ++q) {
        const uint32_t idx = (v >> (2 * q)) & 15u;
        const float r = __shfl_sync(0xffffffffu, tabv, int(idx));
        w[q] ^= __float_as_uint(r);
      }
      if (MODE == 9 || MODE == 10) {
#pragma unroll
        for (int q = 0; q < (MODE == 10 ? 16 : 8); ++q) {
          const uint32_t byte = (v >> (2 * q + 1)) & 255u;
          uint64_t r;
          asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r) : "r"(tab + byte * 128u));
          w[16 + q] ^= uint32_t(r) ^ uint32_t(r >> 32);
        }
      }
      v = v * 1664525u + 1013904223u + w[3] + w[17];
    } else {   // 5, 6: F1's inner loop
      uint32_t o[16];
      // 4 distinct code words per iteration (F1: one LDS.128 of codes per 32 weights)
      const uint32_t cw[4] = {v, v * 3u + 1u, v ^ 0x5A5A5A5Au, (v >> 7) | (v << 25)};
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const uint32_t byte = __byte_perm(cw[q >> 2], 0u, 0x4440u + (q & 3));
        uint64_t r, p;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r) : "r"(tab + byte * 128u));
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(r), "l"(aa));
        float h, l;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(h), "=f"(l) : "l"(p));
        uint32_t o2;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(o2) : "f"(l), "f"(h));
        o[q] = o2;
      }
      if (MODE == 5) {
        st_x8(ta, o);
        st_x8(ta + 8, o + 8);
        st_wait();
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) w[q & 3] ^= o[q];
      }
      v = v * 1664525u + 1013904223u + (MODE == 6 ? w[0] : 0u);
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = v;
#pragma unroll
  for (int i = 0; i < 32; ++i) acc ^= w[i];
  if (acc == 0x12345u) sink[0] = acc;
  __shared__ unsigned long long mx;
  if (threadIdx.x == 0) mx = 0;
  __syncthreads();
  atomicMax(&mx, t1 - t0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = mx;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int MODE>
static void run(const char* name, int sms, int nw, double lds_b, double st_b, unsigned long long* cyc,
                uint32_t* sink) {
  const int iters = 4096;
  CK(cudaFuncSetAttribute(k_dp<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  k_dp<MODE><<<sms, 32 * nw, 32768>>>(iters, nw, cyc, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  k_dp<MODE><<<sms, 32 * nw, 32768>>>(iters, nw, cyc, sink);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  unsigned long long h[1024];
  CK(cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += double(h[i]);
  mean /= sms;
  const double per_it = mean / iters;   // clocks per iteration (all warps concurrently)
  printf("%-40s warps %2d  %7.1f clk/iter  LDS %6.1f B/clk/SM  TMEM st %6.1f B/clk/SM  total %6.1f  (%.3f ms)\n",
         name, nw, per_it, lds_b * nw / per_it, st_b * nw / per_it, (lds_b + st_b) * nw / per_it, ms);
  fflush(stdout);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* cyc;
  uint32_t* sink;
  CK(cudaMalloc(&cyc, sizeof(unsigned long long) * 1024));
  CK(cudaMalloc(&sink, 64));
  printf("SMs %d\n", sms);
  for (int nw : {8, 16, 20}) {
    // bytes per warp per iteration: LDS.64 x16 = 16*256; st 32 columns x 32 lanes x 4 B = 4096
    run<0>("tcgen05.st 32x32b.x8 only", sms, nw, 0, 4096, cyc, sink);
    run<3>("tcgen05.st 32x32b.x16 only", sms, nw, 0, 4096, cyc, sink);
    run<4>("tcgen05.st 32x32b.x32 only", sms, nw, 0, 4096, cyc, sink);
    run<7>("tcgen05.st 16x256b.x2 only", sms, nw, 0, 4096, cyc, sink);
    run<1>("LDS.64 only", sms, nw, 16 * 256, 0, cyc, sink);
    run<2>("16 LDS.64 + 2 st.x8", sms, nw, 16 * 256, 2048, cyc, sink);
    run<5>("F1 inner loop (lookup+FMUL2+cvt+st)", sms, nw, 16 * 256, 2048, cyc, sink);
    run<6>("F1 inner loop without st", sms, nw, 16 * 256, 0, cyc, sink);
    // SHFL "bytes": 32 lanes x 4 B per instruction, counted in the LDS column
    run<8>("16 SHFL.IDX lookups", sms, nw, 16 * 128, 0, cyc, sink);
    run<9>("8 SHFL + 8 LDS.64", sms, nw, 8 * 128 + 8 * 256, 0, cyc, sink);
    run<10>("16 SHFL + 16 LDS.64", sms, nw, 16 * 128 + 16 * 256, 0, cyc, sink);
  }
  return 0;
}
