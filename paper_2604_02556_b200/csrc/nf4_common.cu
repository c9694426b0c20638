// nf4_common.cu -- status strings, per-device caches, launch accounting.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

#include "nf4_internal.cuh"

namespace nf4 {

static thread_local int32_t t_launches = 0;
static std::atomic<int32_t> g_max_ctas{0};

void set_launch_count(int32_t n) { t_launches = n; }

int sm_count() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> g(mu);
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

int32_t max_ctas() { return g_max_ctas.load(std::memory_order_relaxed); }

}  // namespace nf4

extern "C" const char* nf4_status_string(nf4_status s) {
  switch (s) {
    case NF4_OK: return "NF4_OK";
    case NF4_ERR_NULL_POINTER: return "NF4_ERR_NULL_POINTER: required pointer is NULL";
    case NF4_ERR_BAD_SIZE: return "NF4_ERR_BAD_SIZE: negative or unsupported element count";
    case NF4_ERR_BAD_BLOCKSIZE: return "NF4_ERR_BAD_BLOCKSIZE: blocksize must be a power of two in [64, 4096]";
    case NF4_ERR_BAD_DTYPE: return "NF4_ERR_BAD_DTYPE: unsupported dtype for this argument";
    case NF4_ERR_MISALIGNED: return "NF4_ERR_MISALIGNED: array not naturally aligned";
    case NF4_ERR_BAD_STATE: return "NF4_ERR_BAD_STATE: inconsistent absmax / double-quant state or workspace";
    case NF4_ERR_CUDA: return "NF4_ERR_CUDA: a CUDA runtime call failed";
  }
  return "NF4 unknown status";
}

extern "C" int32_t nf4_last_launch_count(void) { return nf4::t_launches; }

extern "C" void nf4_set_max_ctas(int32_t max_ctas) {
  nf4::g_max_ctas.store(max_ctas < 0 ? 0 : max_ctas, std::memory_order_relaxed);
}
