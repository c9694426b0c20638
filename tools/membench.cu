// membench.cu -- HBM access-pattern microbenchmarks on B200 (sm_100a).
// Used to find the achievable ceiling for the dequant kernel's 1:4 read:write
// stream.  Standalone: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o membench membench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e = (x);                                                                        \
    if (e != cudaSuccess) {                                                                     \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));         \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

__device__ __forceinline__ void st8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e,
                                    uint32_t f, uint32_t g, uint32_t h, int hint) {
  if (hint == 0)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
                 "r"(e), "r"(f), "r"(g), "r"(h) : "memory");
  else if (hint == 1)
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
                 "r"(e), "r"(f), "r"(g), "r"(h) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b),
                 "r"(c), "r"(d), "r"(e), "r"(f), "r"(g), "r"(h) : "memory");
}
__device__ __forceinline__ void st4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint2 ld2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void ld8(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

// ---- write only: each thread 32 B per group, warp-contiguous 1 KB, U groups per tile
template <int HINT, int U>
__global__ void __launch_bounds__(256) k_write(uint8_t* dst, int64_t bytes) {
  const int64_t tile = 256 * 32 * U;
  const int64_t tiles = bytes / tile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t v = uint32_t(t + u);
      st8(dst + t * tile + (u * 256 + threadIdx.x) * 32, v, v, v, v, v, v, v, v, HINT);
    }
  }
}

// ---- read only
template <int U>
__global__ void __launch_bounds__(256) k_read(const uint8_t* src, int64_t bytes, uint32_t* sink) {
  const int64_t tile = 256 * 32 * U;
  const int64_t tiles = bytes / tile;
  uint32_t acc = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint32_t r[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) ld8(src + t * tile + (u * 256 + threadIdx.x) * 32, r[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc ^= r[u][j];
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// ---- copy 1:1, 32 B per thread per group
template <int U>
__global__ void __launch_bounds__(256) k_copy(const uint8_t* src, uint8_t* dst, int64_t bytes) {
  const int64_t tile = 256 * 32 * U;
  const int64_t tiles = bytes / tile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint32_t r[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) ld8(src + t * tile + (u * 256 + threadIdx.x) * 32, r[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      st8(dst + t * tile + (u * 256 + threadIdx.x) * 32, r[u][0], r[u][1], r[u][2], r[u][3], r[u][4], r[u][5],
          r[u][6], r[u][7], 0);
  }
}

// ---- 1:4 stream, 8 B in -> 32 B out per group (the dequant kernel's pattern)
template <int U, int HINT>
__global__ void __launch_bounds__(256) k_s14_v2(const uint8_t* src, uint8_t* dst, int64_t in_bytes) {
  const int64_t tile = 256 * 8 * U;
  const int64_t tiles = in_bytes / tile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint2 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = ld2(src + t * tile + (u * 256 + threadIdx.x) * 8);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t a = q[u].x * 0x10001u, b = q[u].y * 0x10001u;
      st8(dst + (t * tile + (u * 256 + threadIdx.x) * 8) * 4, a, a, a, a, b, b, b, b, HINT);
    }
  }
}

// ---- 1:4 stream, 16 B in -> 2 x 32 B out per group (thread-contiguous 64 B)
template <int U>
__global__ void __launch_bounds__(256) k_s14_v4(const uint8_t* src, uint8_t* dst, int64_t in_bytes) {
  const int64_t tile = 256 * 16 * U;
  const int64_t tiles = in_bytes / tile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = ld4(src + t * tile + (u * 256 + threadIdx.x) * 16);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint8_t* o = dst + (t * tile + (u * 256 + threadIdx.x) * 16) * 4;
      uint32_t a = q[u].x * 0x10001u, b = q[u].y * 0x10001u, c = q[u].z * 0x10001u, d = q[u].w * 0x10001u;
      st8(o, a, a, a, a, b, b, b, b, 0);
      st8(o + 32, c, c, c, c, d, d, d, d, 0);
    }
  }
}

// ---- TMA bulk store (write only): smem tile -> global via cp.async.bulk
template <int TILE_KB, int INFLIGHT>
__global__ void __launch_bounds__(128) k_write_bulk(uint8_t* dst, int64_t bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tile = TILE_KB * 1024;
  for (int i = threadIdx.x * 4; i < tile; i += blockDim.x * 4) *reinterpret_cast<uint32_t*>(smem + i) = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t tiles = bytes / tile;
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * tile), "r"(s),
                   "r"(tile) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(INFLIGHT) : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// ---- 1:4 stream with smem staging + TMA bulk store of each warp's 4 KB
// (loads: LDG 8 B per thread as in s14_v2; stores: per-warp bulk copies)
template <int U>
__global__ void __launch_bounds__(256) k_s14_bulk(const uint8_t* src, uint8_t* dst, int64_t in_bytes) {
  // per warp: U groups x 1 KB output = U KB, double buffered
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * (2 * U * 1024);
  const uint32_t wbuf_s = (uint32_t)__cvta_generic_to_shared(wbuf);
  const int64_t tile = 256 * 8 * U;
  const int64_t tiles = in_bytes / tile;
  int phase = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint2 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = ld2(src + t * tile + (u * 256 + threadIdx.x) * 8);
    // make sure the bulk store that last read this half has finished reading smem
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    uint8_t* b = wbuf + phase * U * 1024;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t a = q[u].x * 0x10001u, c = q[u].y * 0x10001u;
      // warp u-group output = 1 KB contiguous in global: lane writes 32 B at lane*32... but the warp's
      // global span for group u is (t*tile + (u*256 + warp*32)*8)*4 .. +1024
      uint4* p = reinterpret_cast<uint4*>(b + u * 1024 + lane * 32);
      p[0] = make_uint4(a, a, a, a);
      p[1] = make_uint4(c, c, c, c);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint8_t* g = dst + (t * tile + (u * 256 + warp * 32) * 8) * 4;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
                     "r"(wbuf_s + (phase * U + u) * 1024), "r"(1024) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    phase ^= 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_fill_random(uint8_t* p, int64_t bytes, uint64_t seed) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < bytes / 8; i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ull + uint64_t(i);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    reinterpret_cast<uint64_t*>(p)[i] = z ^ (z >> 31);
  }
}

// random-output variant of s14 v2: output words mix the input so bits toggle like real bf16 data
template <int U>
__global__ void __launch_bounds__(256) k_s14_v2_rnd(const uint8_t* src, uint8_t* dst, int64_t in_bytes) {
  const int64_t tile = 256 * 8 * U;
  const int64_t tiles = in_bytes / tile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint2 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = ld2(src + t * tile + (u * 256 + threadIdx.x) * 8);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t x = q[u].x, y = q[u].y;
      st8(dst + (t * tile + (u * 256 + threadIdx.x) * 8) * 4, x, x * 0x9E3779B1u, x ^ y, y * 0x85EBCA6Bu, y,
          x + y, x * 0xC2B2AE35u, y ^ 0x5bd1e995u, 0);
    }
  }
}
template <int U>
__global__ void __launch_bounds__(256) k_s14_v4_rnd(const uint8_t* src, uint8_t* dst, int64_t in_bytes) {
  const int64_t tile = 256 * 16 * U;
  const int64_t tiles = in_bytes / tile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = ld4(src + t * tile + (u * 256 + threadIdx.x) * 16);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint8_t* o = dst + (t * tile + (u * 256 + threadIdx.x) * 16) * 4;
      uint32_t x = q[u].x, y = q[u].y, z = q[u].z, w = q[u].w;
      st8(o, x, x * 0x9E3779B1u, x ^ y, y * 0x85EBCA6Bu, y, x + y, x * 0xC2B2AE35u, y ^ 0x5bd1e995u, 0);
      st8(o + 32, z, z * 0x9E3779B1u, z ^ w, w * 0x85EBCA6Bu, w, z + w, z * 0xC2B2AE35u, w ^ 0x5bd1e995u, 0);
    }
  }
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); }
  void start() { CK(cudaEventRecord(a)); }
  float stop() { CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }
};

template <class F>
static void run(const char* name, double bytes_moved, F f, int reps = 10) {
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  Timer t;
  t.start();
  for (int i = 0; i < reps; ++i) f();
  float ms = t.stop() / reps;
  CK(cudaGetLastError());
  printf("%-44s %9.3f ms  %8.1f GB/s\n", name, ms, bytes_moved / (ms * 1e-3) / 1e9);
  fflush(stdout);
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t IN = int64_t(4) << 30;   // 4 GiB codes-like input
  const int64_t OUT = 4 * IN;             // 16 GiB output
  uint8_t *src, *dst;
  uint32_t* sink;
  CK(cudaMalloc(&src, IN));
  CK(cudaMalloc(&dst, OUT));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(src, 0x5a, IN));
  printf("SMs %d, in %lld MiB, out %lld MiB\n", sms, (long long)(IN >> 20), (long long)(OUT >> 20));

  const char* only = argc > 1 ? argv[1] : "all";
  bool all = strcmp(only, "all") == 0;
  if (all || strcmp(only, "const") == 0) {
  run("cudaMemset (write only)", double(OUT), [&] { CK(cudaMemsetAsync(dst, 1, OUT)); });
  run("cudaMemcpy D2D 4 GiB (1:1, const data)", double(2 * IN), [&] { CK(cudaMemcpyAsync(dst, src, IN, cudaMemcpyDeviceToDevice)); });
  run("s14 v2 U4 .cs occ8 const", double(5 * IN), [&] { k_s14_v2<4, 0><<<sms * 8, 256>>>(src, dst, IN); });
  run("s14 v4 U2 occ8 const", double(5 * IN), [&] { k_s14_v4<2><<<sms * 8, 256>>>(src, dst, IN); });
  }
  k_fill_random<<<sms * 8, 256>>>(src, IN, 1);
  CK(cudaDeviceSynchronize());
  run("cudaMemcpy D2D 4 GiB (1:1, random)", double(2 * IN), [&] { CK(cudaMemcpyAsync(dst, src, IN, cudaMemcpyDeviceToDevice)); });
  run("cudaMemcpy D2D 16 GiB (1:1, random dst->dst)", double(2 * IN * 2), [&] { CK(cudaMemcpyAsync(dst + 2 * IN * 0 + (OUT/2), dst, OUT/2, cudaMemcpyDeviceToDevice)); });
  const int64_t tiles_v2 = IN / (256 * 8 * 4), tiles_v4 = IN / (256 * 16 * 2);
  for (int occ : {4, 8}) {
    char nm[160];
    snprintf(nm, sizeof nm, "s14 v2 U4 random-in occ%d", occ);
    run(nm, double(5 * IN), [&] { k_s14_v2<4, 0><<<sms * occ, 256>>>(src, dst, IN); });
    snprintf(nm, sizeof nm, "s14 v2 U4 random-in random-out occ%d", occ);
    run(nm, double(5 * IN), [&] { k_s14_v2_rnd<4><<<sms * occ, 256>>>(src, dst, IN); });
    snprintf(nm, sizeof nm, "s14 v4 U2 random-in random-out occ%d", occ);
    run(nm, double(5 * IN), [&] { k_s14_v4_rnd<2><<<sms * occ, 256>>>(src, dst, IN); });
  }
  run("s14 v2 U4 rnd/rnd grid=tiles (non-persistent)", double(5 * IN), [&] { k_s14_v2_rnd<4><<<int(tiles_v2), 256>>>(src, dst, IN); });
  run("s14 v4 U2 rnd/rnd grid=tiles (non-persistent)", double(5 * IN), [&] { k_s14_v4_rnd<2><<<int(tiles_v4), 256>>>(src, dst, IN); });
  run("s14 v2 U1 rnd/rnd grid=tiles (non-persistent)", double(5 * IN), [&] { k_s14_v2_rnd<1><<<int(IN / 2048), 256>>>(src, dst, IN); });
  run("s14 v4 U4 rnd/rnd occ8", double(5 * IN), [&] { k_s14_v4_rnd<4><<<sms * 8, 256>>>(src, dst, IN); });
  run("copy v8 U2 occ8 (1:1 random)", double(2 * IN), [&] { k_copy<2><<<sms * 8, 256>>>(src, dst, IN); });
  run("write v8 .cs U4 occ8 (const)", double(OUT), [&] { k_write<0, 4><<<sms * 8, 256>>>(dst, OUT); });
  run("read v8 U4 occ8 (random)", double(IN), [&] { k_read<4><<<sms * 8, 256>>>(src, IN, sink); });
  return 0;
}
