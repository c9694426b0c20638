// ceiling.cu -- what bounds the dequant kernel's 1:4 read:write HBM stream?
// Round 2 follow-up of membench.cu: write-only / read-only / 1:4 streams with
// one CTA per tile (the launch shape the dequant kernel uses), store and load
// cache hints, larger tiles, against cudaMemset.  Random data unless "const".
// Standalone: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ceiling ceiling.cu
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

// HINT: 0 .cs, 1 default (wb), 2 L1::no_allocate, 3 L2 evict_first policy, 4 L2 evict_last policy? no:
//       4 = .cs + L2 evict_first policy
template <int HINT>
__device__ __forceinline__ void st8(void* p, const uint32_t (&v)[8], uint64_t pol) {
  if (HINT == 0)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
  else if (HINT == 1)
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
  else if (HINT == 2)
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
  else
    asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "l"(pol) : "memory");
}
template <int LH>
__device__ __forceinline__ uint2 ld2(const void* p, uint64_t pol) {
  uint2 r;
  if (LH == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  else if (LH == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void mix(uint32_t x, uint32_t y, uint32_t (&v)[8]) {
  v[0] = x; v[1] = x * 0x9E3779B1u; v[2] = x ^ y; v[3] = y * 0x85EBCA6Bu;
  v[4] = y; v[5] = x + y; v[6] = x * 0xC2B2AE35u; v[7] = y ^ 0x5bd1e995u;
}

// write only, one CTA per tile of 256*32*U bytes; RND: data varies per word
template <int HINT, int U, int RND>
__global__ void __launch_bounds__(256) k_write(uint8_t* dst) {
  const int64_t t = blockIdx.x;
  const uint64_t pol = HINT >= 3 ? pol_evict_first() : 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    uint32_t v[8];
    uint32_t s = RND ? uint32_t(t * 2654435761u) ^ (threadIdx.x * 40503u + u) : 0x01010101u;
    if (RND) mix(s, s * 747796405u, v);
    else for (int j = 0; j < 8; ++j) v[j] = s;
    st8<HINT>(dst + (t * (256 * U) + u * 256 + threadIdx.x) * 32, v, pol);
  }
}

// read only, one CTA per tile of 256*8*U bytes (8 B per thread per group, as the dequant kernel)
template <int U, int LH>
__global__ void __launch_bounds__(256) k_read(const uint8_t* src, uint32_t* sink) {
  const int64_t t = blockIdx.x;
  const uint64_t pol = LH == 2 ? pol_evict_first() : 0;
  uint2 q[U];
#pragma unroll
  for (int u = 0; u < U; ++u) q[u] = ld2<LH>(src + (t * (256 * U) + u * 256 + threadIdx.x) * 8, pol);
  uint32_t acc = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) acc ^= q[u].x + q[u].y;
  if (acc == 0x12345678u) sink[0] = acc;
}

// 1:4 stream, one CTA (NT threads) per tile: 8 B in -> 32 B out per thread per group
template <int NT, int U, int HINT, int LH>
__global__ void __launch_bounds__(NT) k_s14(const uint8_t* src, uint8_t* dst) {
  const int64_t t = blockIdx.x;
  const uint64_t pol = (HINT >= 3 || LH == 2) ? pol_evict_first() : 0;
  uint2 q[U];
#pragma unroll
  for (int u = 0; u < U; ++u) q[u] = ld2<LH>(src + (t * (NT * U) + u * NT + threadIdx.x) * 8, pol);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    uint32_t v[8];
    mix(q[u].x, q[u].y, v);
    st8<HINT>(dst + (t * (NT * U) + u * NT + threadIdx.x) * 32, v, pol);
  }
}

// 1:4 stream, one CTA per tile, the tile's codes loaded by ONE bulk copy (TMA engine) into shared memory
// (8 KB per CTA), output with per-thread STG.256 as above.
template <int U, int HINT>
__global__ void __launch_bounds__(256) k_s14_tmaload(const uint8_t* src, uint8_t* dst) {
  __shared__ __align__(128) uint8_t buf[256 * 8 * U];
  __shared__ __align__(8) uint64_t bar;
  const int64_t t = blockIdx.x;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf), sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(256 * 8 * U) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb),
                 "l"(src + t * (256 * 8 * U)), "r"(256 * 8 * U), "r"(sbar) : "memory");
  }
  __syncthreads();
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sbar)
      : "memory");
#pragma unroll
  for (int u = 0; u < U; ++u) {
    uint2 q = *reinterpret_cast<const uint2*>(buf + (u * 256 + threadIdx.x) * 8);
    uint32_t v[8];
    mix(q.x, q.y, v);
    st8<HINT>(dst + (t * (256 * U) + u * 256 + threadIdx.x) * 32, v, 0);
  }
}

__global__ void k_fill_random(uint8_t* p, int64_t bytes, uint64_t seed) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < bytes / 8; i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ull + uint64_t(i);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    reinterpret_cast<uint64_t*>(p)[i] = z ^ (z >> 31);
  }
}

template <class F>
static void run(const char* name, double bytes_moved, F f, int reps = 10) {
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f, sum = 0;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= reps;
    sum += ms;
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("%-58s %8.3f ms  best %7.1f GB/s  mean %7.1f GB/s\n", name, best, bytes_moved / (best * 1e-3) / 1e9,
         bytes_moved / (sum / 3 * 1e-3) / 1e9);
  fflush(stdout);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t IN = int64_t(4) << 30, OUT = 4 * IN;
  uint8_t *src, *dst;
  uint32_t* sink;
  CK(cudaMalloc(&src, IN));
  CK(cudaMalloc(&dst, OUT));
  CK(cudaMalloc(&sink, 64));
  k_fill_random<<<sms * 8, 256>>>(src, IN, 1);
  k_fill_random<<<sms * 8, 256>>>(dst, OUT, 2);
  CK(cudaDeviceSynchronize());
  printf("SMs %d, in %lld MiB, out %lld MiB\n", sms, (long long)(IN >> 20), (long long)(OUT >> 20));

  run("cudaMemset 16 GiB (write only, const)", double(OUT), [&] { CK(cudaMemsetAsync(dst, 1, OUT)); });
  run("cudaMemcpy D2D 4 GiB (1:1)", double(2 * IN), [&] { CK(cudaMemcpyAsync(dst, src, IN, cudaMemcpyDeviceToDevice)); });
  // write only, one CTA per 32 KB tile
  const int wt4 = int(OUT / (256 * 32 * 4));
  run("write U4 .cs const", double(OUT), [&] { k_write<0, 4, 0><<<wt4, 256>>>(dst); });
  run("write U4 .cs rnd", double(OUT), [&] { k_write<0, 4, 1><<<wt4, 256>>>(dst); });
  run("write U4 wb rnd", double(OUT), [&] { k_write<1, 4, 1><<<wt4, 256>>>(dst); });
  run("write U4 L1::no_allocate rnd", double(OUT), [&] { k_write<2, 4, 1><<<wt4, 256>>>(dst); });
  run("write U4 L2 evict_first rnd", double(OUT), [&] { k_write<3, 4, 1><<<wt4, 256>>>(dst); });
  run("write U1 .cs rnd (8 KB tiles)", double(OUT), [&] { k_write<0, 1, 1><<<int(OUT / 8192), 256>>>(dst); });
  run("write U8 .cs rnd (64 KB tiles)", double(OUT), [&] { k_write<0, 8, 1><<<int(OUT / 65536), 256>>>(dst); });
  // read only
  run("read U4 8B/thr (8 KB tiles)", double(IN), [&] { k_read<4, 0><<<int(IN / 8192), 256>>>(src, sink); });
  run("read U4 L2::256B", double(IN), [&] { k_read<4, 1><<<int(IN / 8192), 256>>>(src, sink); });
  run("read U8 (16 KB tiles)", double(IN), [&] { k_read<8, 0><<<int(IN / 16384), 256>>>(src, sink); });
  // 1:4 streams
  const int t4 = int(IN / (256 * 8 * 4));
  run("s14 256x U4 .cs (dequant shape)", double(5 * IN), [&] { k_s14<256, 4, 0, 0><<<t4, 256>>>(src, dst); });
  run("s14 256x U4 wb", double(5 * IN), [&] { k_s14<256, 4, 1, 0><<<t4, 256>>>(src, dst); });
  run("s14 256x U4 L1::no_allocate", double(5 * IN), [&] { k_s14<256, 4, 2, 0><<<t4, 256>>>(src, dst); });
  run("s14 256x U4 st L2 evict_first", double(5 * IN), [&] { k_s14<256, 4, 3, 0><<<t4, 256>>>(src, dst); });
  run("s14 256x U4 .cs, ld L2::256B", double(5 * IN), [&] { k_s14<256, 4, 0, 1><<<t4, 256>>>(src, dst); });
  run("s14 256x U4 .cs, ld L2 evict_first", double(5 * IN), [&] { k_s14<256, 4, 0, 2><<<t4, 256>>>(src, dst); });
  run("s14 256x U2 .cs", double(5 * IN), [&] { k_s14<256, 2, 0, 0><<<t4 * 2, 256>>>(src, dst); });
  run("s14 256x U8 .cs", double(5 * IN), [&] { k_s14<256, 8, 0, 0><<<t4 / 2, 256>>>(src, dst); });
  run("s14 512x U4 .cs", double(5 * IN), [&] { k_s14<512, 4, 0, 0><<<t4 / 2, 512>>>(src, dst); });
  run("s14 128x U4 .cs", double(5 * IN), [&] { k_s14<128, 4, 0, 0><<<t4 * 2, 128>>>(src, dst); });
  run("s14 TMA-load 8 KB tile, .cs", double(5 * IN), [&] { k_s14_tmaload<4, 0><<<t4, 256>>>(src, dst); });
  run("s14 TMA-load 16 KB tile, .cs", double(5 * IN), [&] { k_s14_tmaload<8, 0><<<t4 / 2, 256>>>(src, dst); });
  run("s14 256x U4 .cs (repeat)", double(5 * IN), [&] { k_s14<256, 4, 0, 0><<<t4, 256>>>(src, dst); });
  run("cudaMemset 16 GiB (repeat)", double(OUT), [&] { CK(cudaMemsetAsync(dst, 1, OUT)); });
  return 0;
}
