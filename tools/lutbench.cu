// lutbench.cu -- throughput of a 16-entry fp32 table lookup on B200: shared
// memory LDS vs warp shuffle (SHFL) vs a mix.  Decides where the F1 GEMM's
// dequant producers keep the NF4 table.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lutbench lutbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__constant__ float c_tab[16] = {-1.f, -.69f, -.52f, -.39f, -.28f, -.18f, -.09f, 0.f,
                                .08f, .16f, .25f, .34f, .44f, .56f, .72f, 1.f};

template <int MODE>
__global__ void __launch_bounds__(256) k(const uint32_t* __restrict__ in, float* out, int iters) {
  __shared__ float lut[16];
  if (threadIdx.x < 16) lut[threadIdx.x] = c_tab[threadIdx.x];
  __syncthreads();
  const float mine = c_tab[threadIdx.x & 15];
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x];
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t idx = (x >> (4 * j)) & 15u;
      float v;
      if (MODE == 0) {
        v = lut[idx];
      } else if (MODE == 1) {
        v = __shfl_sync(0xffffffffu, mine, int(idx));
      } else {
        v = (j & 1) ? __shfl_sync(0xffffffffu, mine, int(idx)) : lut[idx];
      }
      acc = __fmul_rn(acc, 0.5f) + v;
    }
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  uint32_t* in;
  float* out;
  cudaMalloc(&in, blocks * threads * 4);
  cudaMalloc(&out, blocks * threads * 4);
  cudaMemset(in, 0x37, blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"LDS", "SHFL", "LDS+SHFL alternating"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(in, out, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(in, out, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(in, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double lookups = double(blocks) * threads * iters * 8;
      if (rep) printf("%-24s %8.3f ms  %7.1f Glookups/s  %6.2f lookups/clk/SM @1.9GHz\n", names[mode], ms,
                      lookups / ms / 1e6, lookups / (ms * 1e-3) / 148 / 1.9e9);
    }
  }
  return 0;
}
