// ceiling2.cu -- can bunching the reads of a 1:4 read:write stream beat the
// ~6.8 TB/s of every per-tile arrangement (profiles/r02_hbm_ceiling.md)?
// Persistent CTAs work in epochs: at the start of epoch e a CTA issues ONE bulk
// (TMA engine) copy of the codes for epoch e+1 into a shared-memory buffer, then
// expands epoch e's codes (already on chip) into 4x the bytes of output.
// PHASE: the CTAs start each epoch's read burst at a common absolute time
// (globaltimer multiple of period_ns), so the whole GPU's reads arrive together
// and the DRAM sees long read runs between long write runs.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ceiling2 ceiling2.cu
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

__device__ __forceinline__ void st8cs(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
__device__ __forceinline__ void mix(uint32_t x, uint32_t y, uint32_t (&v)[8]) {
  v[0] = x; v[1] = x * 0x9E3779B1u; v[2] = x ^ y; v[3] = y * 0x85EBCA6Bu;
  v[4] = y; v[5] = x + y; v[6] = x * 0xC2B2AE35u; v[7] = y ^ 0x5bd1e995u;
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(bar),
               "r"(ph) : "memory");
}

// NB: shared-memory buffers; IN bytes of codes per CTA per epoch (<= 48 KB per buffer here)
template <int NT, int IN, int PHASE>
__global__ void __launch_bounds__(NT, 1) k_epoch(const uint8_t* src, uint8_t* dst, int64_t in_bytes,
                                                  uint64_t period_ns) {
  extern __shared__ __align__(128) uint8_t smem[];   // 2 x IN
  __shared__ __align__(8) uint64_t bars[2];
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);
  const int64_t epochs = in_bytes / (int64_t(IN) * gridDim.x);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t e) {
    const int buf = int(e & 1);
    const uint8_t* g = src + (e * gridDim.x + blockIdx.x) * int64_t(IN);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0 + 8 * buf), "r"(IN) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sb + buf * IN), "l"(g), "r"(IN), "r"(b0 + 8 * buf) : "memory");
  };
  uint64_t next_t = 0;
  if (threadIdx.x == 0) {
    if (PHASE) next_t = (gtime() / period_ns + 2) * period_ns;
    if (epochs > 0) issue(0);
  }
  for (int64_t e = 0; e < epochs; ++e) {
    if (threadIdx.x == 0 && e + 1 < epochs) {
      if (PHASE) {
        while (gtime() < next_t) {}
        next_t += period_ns;
      }
      issue(e + 1);
    }
    bar_wait(b0 + 8 * uint32_t(e & 1), uint32_t((e >> 1) & 1));
    const uint8_t* buf = smem + (e & 1) * IN;
    uint8_t* o = dst + (e * gridDim.x + blockIdx.x) * int64_t(IN) * 4;
#pragma unroll 4
    for (int i = threadIdx.x; i < IN / 8; i += NT) {
      const uint2 q = *reinterpret_cast<const uint2*>(buf + 8 * i);
      uint32_t v[8];
      mix(q.x, q.y, v);
      st8cs(o + 32 * i, v);
    }
    __syncthreads();   // buffer e&1 is refilled at epoch e+1's issue (for e+2)
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

// reference: the dequant shape (one CTA per 8 KB-in tile)
__global__ void __launch_bounds__(256) k_s14(const uint8_t* src, uint8_t* dst) {
  const int64_t t = blockIdx.x;
  uint2 q[4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(q[u].x), "=r"(q[u].y) : "l"(src + (t * 1024 + u * 256 + threadIdx.x) * 8));
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint32_t v[8];
    mix(q[u].x, q[u].y, v);
    st8cs(dst + (t * 1024 + u * 256 + threadIdx.x) * 32, v);
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

template <int NT, int IN, int PHASE>
static void epoch_run(const char* name, int grid, const uint8_t* src, uint8_t* dst, int64_t IN_B, uint64_t period) {
  CK(cudaFuncSetAttribute(k_epoch<NT, IN, PHASE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * IN));
  const int64_t used = IN_B / (int64_t(IN) * grid) * int64_t(IN) * grid;
  char nm[128];
  snprintf(nm, sizeof nm, "%s grid %d IN %d KB period %llu ns", name, grid, IN / 1024, (unsigned long long)period);
  run(nm, double(5 * used), [&] { k_epoch<NT, IN, PHASE><<<grid, NT, 2 * IN>>>(src, dst, used, period); });
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t IN = int64_t(4) << 30, OUT = 4 * IN;
  uint8_t *src, *dst;
  CK(cudaMalloc(&src, IN));
  CK(cudaMalloc(&dst, OUT));
  k_fill_random<<<sms * 8, 256>>>(src, IN, 1);
  k_fill_random<<<sms * 8, 256>>>(dst, OUT, 2);
  CK(cudaDeviceSynchronize());
  printf("SMs %d\n", sms);
  run("s14 256x U4 .cs (dequant shape, reference)", double(5 * IN), [&] { k_s14<<<int(IN / 8192), 256>>>(src, dst); });
  epoch_run<512, 16384, 0>("epoch", sms, src, dst, IN, 0);
  epoch_run<512, 32768, 0>("epoch", sms, src, dst, IN, 0);
  epoch_run<512, 49152, 0>("epoch", sms, src, dst, IN, 0);
  epoch_run<1024, 32768, 0>("epoch", sms, src, dst, IN, 0);
  epoch_run<512, 16384, 0>("epoch (2 CTAs/SM)", 2 * sms, src, dst, IN, 0);
  epoch_run<512, 32768, 0>("epoch (2 CTAs/SM)", 2 * sms, src, dst, IN, 0);
  // phased: epoch = IN*5*grid bytes at ~7 TB/s
  for (uint64_t per : {1500ull, 2000ull, 3000ull, 3500ull})
    epoch_run<512, 16384, 1>("epoch phased", sms, src, dst, IN, per);
  for (uint64_t per : {3500ull, 4000ull, 5000ull, 6000ull})
    epoch_run<512, 32768, 1>("epoch phased", sms, src, dst, IN, per);
  for (uint64_t per : {6000ull, 8000ull})
    epoch_run<512, 49152, 1>("epoch phased", sms, src, dst, IN, per);
  run("s14 256x U4 .cs (reference, repeat)", double(5 * IN), [&] { k_s14<<<int(IN / 8192), 256>>>(src, dst); });
  return 0;
}
