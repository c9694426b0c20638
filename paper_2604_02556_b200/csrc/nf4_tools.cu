// nf4_tools.cu -- input generation (counter-based hash, same function as
// synth/inputs.py), the speed-of-light stream kernel, and the host-buffer
// (end-to-end) dequantization pipeline.  None of this is the method's
// arithmetic except nf4_dequantize_host, which only moves bytes around calls
// of the device kernel in nf4_dequant.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "nf4_internal.cuh"

namespace nf4 {

// ---------------------------------------------------------------------------
// Counter-based generator: z = splitmix64_mix(seed*GOLDEN + stream*MUL + idx)
// (synth/inputs.py hash64).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t synth_hash(uint64_t seed, uint64_t stream, uint64_t idx) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + idx;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_bytes_kernel(uint64_t seed, uint64_t stream, int64_t begin, int64_t count, uint8_t* dst) {
  const int64_t w0 = begin >> 3;
  const int64_t w1 = (begin + count + 7) >> 3;
  const bool fast = ((begin & 7) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0);
  for (int64_t w = w0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < w1;
       w += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t z = synth_hash(seed, stream, uint64_t(w));
    const int64_t j0 = w << 3;
    if (fast && j0 + 8 <= begin + count) {
      *reinterpret_cast<uint64_t*>(dst + (j0 - begin)) = z;  // little-endian bytes
    } else {
      for (int i = 0; i < 8; ++i) {
        const int64_t j = j0 + i;
        if (j >= begin && j < begin + count) dst[j - begin] = uint8_t(z >> (8 * i));
      }
    }
  }
}

__global__ void synth_f32_kernel(uint64_t seed, uint64_t stream, int64_t begin, int64_t count, uint32_t base,
                                 uint32_t mask, uint32_t* dst) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t z = synth_hash(seed, stream, uint64_t(begin + i));
    dst[i] = base | (uint32_t(z) & mask);
  }
}

// ---------------------------------------------------------------------------
// Speed-of-light stream with the default dequant variant's access pattern
// (v4u2): per thread and tile, 2 x 16-byte loads (warp-contiguous 512 B) and
// 2 x 64 B thread-contiguous stores (2 x STG.256), one CTA per 8 KB-input tile;
// no table, no math.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sol_stream_kernel(const uint8_t* __restrict__ src, int64_t in_bytes,
                                                         uint8_t* __restrict__ dst) {
  const int64_t tiles = in_bytes / 8192;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint4 q[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint8_t* p = src + t * 8192 + (u * 256 + threadIdx.x) * 16;
      asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
          : "=r"(q[u].x), "=r"(q[u].y), "=r"(q[u].z), "=r"(q[u].w) : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      uint8_t* o = dst + (t * 8192 + (u * 256 + threadIdx.x) * 16) * 4;
      const uint32_t x = q[u].x * 0x10001u, y = q[u].y * 0x10001u, z = q[u].z * 0x10001u, w = q[u].w * 0x10001u;
      const uint32_t a[8] = {x, x, x, x, y, y, y, y};
      const uint32_t b[8] = {z, z, z, z, w, w, w, w};
      st_out_v8(o, a);
      st_out_v8(o + 32, b);
    }
  }
}

}  // namespace nf4

using namespace nf4;

extern "C" nf4_status nf4_synth_fill(nf4_synth_kind kind, uint64_t seed, int64_t begin, int64_t count, void* dst,
                                     void* stream) {
  if (count < 0 || begin < 0) return NF4_ERR_BAD_SIZE;
  if (count == 0) { set_launch_count(0); return NF4_OK; }
  if (!dst) return NF4_ERR_NULL_POINTER;
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = sm_count() * 8;
  switch (kind) {
    case NF4_SYNTH_CODES:
    case NF4_SYNTH_QABSMAX:
      synth_bytes_kernel<<<grid, 256, 0, s>>>(seed, uint64_t(kind), begin, count, static_cast<uint8_t*>(dst));
      break;
    case NF4_SYNTH_ABSMAX:
      if (!aligned(dst, 4)) return NF4_ERR_MISALIGNED;
      synth_f32_kernel<<<grid, 256, 0, s>>>(seed, uint64_t(kind), begin, count, 0x3D000000u, 0x7FFFFFu,
                                            static_cast<uint32_t*>(dst));
      break;
    case NF4_SYNTH_ABSMAX2:
      if (!aligned(dst, 4)) return NF4_ERR_MISALIGNED;
      synth_f32_kernel<<<grid, 256, 0, s>>>(seed, uint64_t(kind), begin, count, 0x3C800000u, 0x7FFFFFu,
                                            static_cast<uint32_t*>(dst));
      break;
    default:
      return NF4_ERR_BAD_DTYPE;
  }
  if (cudaPeekAtLastError() != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
  set_launch_count(1);
  return NF4_OK;
}

extern "C" nf4_status nf4_sol_stream(const void* src, int64_t in_bytes, void* dst, void* stream) {
  if (in_bytes < 0 || in_bytes % 8192 != 0) return NF4_ERR_BAD_SIZE;
  if (in_bytes == 0) { set_launch_count(0); return NF4_OK; }
  if (!src || !dst) return NF4_ERR_NULL_POINTER;
  if (!aligned(src, 32) || !aligned(dst, 128)) return NF4_ERR_MISALIGNED;
  int64_t grid = in_bytes / 8192;  // one CTA per tile (hardware-scheduled)
  const int32_t cap = max_ctas();
  if (cap > 0 && grid > cap) grid = cap;
  if (grid > 0x7FFFFFFF) grid = 0x7FFFFFFF;
  sol_stream_kernel<<<int(grid), 256, 0, (cudaStream_t)stream>>>(static_cast<const uint8_t*>(src), in_bytes,
                                                                 static_cast<uint8_t*>(dst));
  if (cudaPeekAtLastError() != cudaSuccess) { cudaGetLastError(); return NF4_ERR_CUDA; }
  set_launch_count(1);
  return NF4_OK;
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline (nf4_dequantize_host, nf4_dequantize_host_batched)
// The chunks of all tensors form one stream; kNumSlots workspace slots rotate
// so that the H2D copy of chunk c+2, the kernel of chunk c+1 and the D2H copy of
// chunk c overlap (copy engines in both directions + SMs busy at once).
// ---------------------------------------------------------------------------
namespace {
constexpr int kNumSlots = 3;
struct HostLayout {
  int64_t codes, scales, groups, code2, out, slot;  // byte sizes (256-B rounded)
};
inline int64_t rnd(int64_t v) { return (v + 255) / 256 * 256; }
HostLayout host_layout(int64_t chunk, int32_t bs, bool dq) {
  HostLayout L;
  const int64_t nb = chunk / bs;
  L.codes = rnd(chunk / 2);
  // fp32 absmax width even when dq: a batch may mix fp32-absmax and double-quant
  // tensors, and the slot must hold the widest scale slice of a chunk (4 B per block)
  (void)dq;
  L.scales = rnd(nb * 4);
  L.groups = dq ? rnd((nb / 256) * 4) : 0;
  L.code2 = dq ? 1024 : 0;
  L.out = rnd(chunk * 2);
  L.slot = L.codes + L.scales + L.groups + L.code2 + L.out;
  return L;
}
}  // namespace

extern "C" int64_t nf4_host_workspace_bytes(int64_t chunk_elems, int32_t blocksize, int32_t dq) {
  if (chunk_elems <= 0 || !is_pow2(blocksize)) return 0;
  const HostLayout L = host_layout(chunk_elems, blocksize, dq != 0);
  return kNumSlots * L.slot;
}

extern "C" nf4_status nf4_dequantize_host_batched(const nf4_tensor* tensors, int32_t count, nf4_dtype out_dtype,
                                                  void* workspace, int64_t workspace_bytes, int64_t chunk_elems,
                                                  void* stream) {
  if (count < 0) return NF4_ERR_BAD_SIZE;
  if (count > 0 && !tensors) return NF4_ERR_NULL_POINTER;
  if (out_dtype != NF4_F16 && out_dtype != NF4_BF16) return NF4_ERR_BAD_DTYPE;
  int32_t bs_min = 4096, bs_max = 64;
  bool any_dq = false, any_work = false;
  for (int i = 0; i < count; ++i) {
    const nf4_tensor& t = tensors[i];
    if (t.n < 0) return NF4_ERR_BAD_SIZE;
    if (t.reserved != 0) return NF4_ERR_BAD_STATE;
    if (!is_pow2(t.blocksize) || t.blocksize < 64 || t.blocksize > 4096) return NF4_ERR_BAD_BLOCKSIZE;
    const bool dq = t.absmax == nullptr;
    if (dq && t.dq.blocksize2 != 256) return NF4_ERR_BAD_STATE;
    if (t.n == 0) continue;
    if (!t.packed || !t.out) return NF4_ERR_NULL_POINTER;
    if (dq && (!t.dq.qabsmax || !t.dq.code2 || !t.dq.absmax2)) return NF4_ERR_NULL_POINTER;
    any_work = true;
    any_dq = any_dq || dq;
    bs_min = t.blocksize < bs_min ? t.blocksize : bs_min;
    bs_max = t.blocksize > bs_max ? t.blocksize : bs_max;
  }
  if (!any_work) { set_launch_count(0); return NF4_OK; }
  if (!workspace) return NF4_ERR_NULL_POINTER;
  if (chunk_elems <= 0 || chunk_elems % (int64_t(256) * bs_max) != 0) return NF4_ERR_BAD_SIZE;
  if (!aligned(workspace, 256)) return NF4_ERR_MISALIGNED;
  if (workspace_bytes < nf4_host_workspace_bytes(chunk_elems, bs_min, any_dq)) return NF4_ERR_BAD_STATE;

  const HostLayout L = host_layout(chunk_elems, bs_min, any_dq);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  cudaStream_t cs = (cudaStream_t)stream;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_in[kNumSlots] = {}, ev_comp[kNumSlots] = {}, ev_out[kNumSlots] = {};
  nf4_status st = NF4_OK;
  int32_t launches = 0;
  int64_t c = 0;  // global chunk counter
#define NF4_TRY(x)                       \
  do {                                   \
    if ((x) != cudaSuccess) {            \
      st = NF4_ERR_CUDA;                 \
      goto done;                         \
    }                                    \
  } while (0)
  NF4_TRY(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
  NF4_TRY(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
  for (int i = 0; i < kNumSlots; ++i) {
    NF4_TRY(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming));
    NF4_TRY(cudaEventCreateWithFlags(&ev_comp[i], cudaEventDisableTiming));
    NF4_TRY(cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming));
  }
  // the copies start after everything already queued on the caller's stream
  NF4_TRY(cudaEventRecord(ev_comp[0], cs));
  NF4_TRY(cudaStreamWaitEvent(h2d, ev_comp[0], 0));
  for (int ti = 0; ti < count; ++ti) {
    const nf4_tensor& t = tensors[ti];
    if (t.n == 0) continue;
    const bool isdq = t.absmax == nullptr;
    const int32_t bs = t.blocksize;
    for (int64_t e0 = 0; e0 < t.n; e0 += chunk_elems, ++c) {
      const int s = int(c % kNumSlots);
      uint8_t* base = ws + s * L.slot;
      uint8_t* d_codes = base;
      uint8_t* d_scales = base + L.codes;
      float* d_groups = reinterpret_cast<float*>(base + L.codes + L.scales);
      float* d_code2 = reinterpret_cast<float*>(base + L.codes + L.scales + L.groups);
      void* d_out = base + L.codes + L.scales + L.groups + L.code2;
      const int64_t e1 = (e0 + chunk_elems < t.n) ? e0 + chunk_elems : t.n;
      const int64_t m = e1 - e0;
      const int64_t b0 = e0 / bs, b1 = (e1 + bs - 1) / bs;
      if (c >= kNumSlots) NF4_TRY(cudaStreamWaitEvent(h2d, ev_comp[s], 0));  // inputs of chunk c-3 consumed
      NF4_TRY(cudaMemcpyAsync(d_codes, t.packed + e0 / 2, (m + 1) / 2, cudaMemcpyHostToDevice, h2d));
      if (isdq) {
        const int64_t g0 = b0 / 256, g1 = (b1 + 255) / 256;
        NF4_TRY(cudaMemcpyAsync(d_scales, t.dq.qabsmax + b0, b1 - b0, cudaMemcpyHostToDevice, h2d));
        NF4_TRY(cudaMemcpyAsync(d_groups, t.dq.absmax2 + g0, (g1 - g0) * 4, cudaMemcpyHostToDevice, h2d));
        NF4_TRY(cudaMemcpyAsync(d_code2, t.dq.code2, 1024, cudaMemcpyHostToDevice, h2d));
      } else {
        NF4_TRY(cudaMemcpyAsync(d_scales, t.absmax + b0, (b1 - b0) * 4, cudaMemcpyHostToDevice, h2d));
      }
      NF4_TRY(cudaEventRecord(ev_in[s], h2d));
      NF4_TRY(cudaStreamWaitEvent(cs, ev_in[s], 0));
      if (c >= kNumSlots) NF4_TRY(cudaStreamWaitEvent(cs, ev_out[s], 0));  // output slot drained
      nf4_status ks;
      if (isdq) {
        nf4_dq_state ld;
        ld.qabsmax = d_scales;
        ld.code2 = d_code2;
        ld.absmax2 = d_groups;
        ld.offset = t.dq.offset;
        ld.blocksize2 = 256;
        ks = nf4_dequantize(d_codes, nullptr, &ld, m, bs, out_dtype, d_out, cs);
      } else {
        ks = nf4_dequantize(d_codes, reinterpret_cast<const float*>(d_scales), nullptr, m, bs, out_dtype, d_out,
                            cs);
      }
      if (ks != NF4_OK) { st = ks; goto done; }
      launches += nf4_last_launch_count();
      NF4_TRY(cudaEventRecord(ev_comp[s], cs));
      NF4_TRY(cudaStreamWaitEvent(d2h, ev_comp[s], 0));
      NF4_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(t.out) + e0 * 2, d_out, m * 2, cudaMemcpyDeviceToHost, d2h));
      NF4_TRY(cudaEventRecord(ev_out[s], d2h));
    }
  }
  NF4_TRY(cudaStreamSynchronize(d2h));
  NF4_TRY(cudaStreamSynchronize(h2d));
  NF4_TRY(cudaStreamSynchronize(cs));
done:
#undef NF4_TRY
  for (int i = 0; i < kNumSlots; ++i) {
    if (ev_in[i]) cudaEventDestroy(ev_in[i]);
    if (ev_comp[i]) cudaEventDestroy(ev_comp[i]);
    if (ev_out[i]) cudaEventDestroy(ev_out[i]);
  }
  if (h2d) { cudaStreamSynchronize(h2d); cudaStreamDestroy(h2d); }
  if (d2h) { cudaStreamSynchronize(d2h); cudaStreamDestroy(d2h); }
  if (st == NF4_OK) set_launch_count(launches);
  return st;
}

extern "C" nf4_status nf4_dequantize_host(const uint8_t* packed, const float* absmax, const nf4_dq_state* dq,
                                          int64_t n, int32_t blocksize, nf4_dtype out_dtype, void* out,
                                          void* workspace, int64_t workspace_bytes, int64_t chunk_elems,
                                          void* stream) {
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
  t.n = n;
  t.blocksize = blocksize;
  t.reserved = 0;
  t.out = out;
  if (n < 0) return NF4_ERR_BAD_SIZE;
  if (!is_pow2(blocksize) || blocksize < 64 || blocksize > 4096) return NF4_ERR_BAD_BLOCKSIZE;
  if (n > 0 && (chunk_elems <= 0 || chunk_elems % (int64_t(256) * blocksize) != 0)) return NF4_ERR_BAD_SIZE;
  return nf4_dequantize_host_batched(&t, 1, out_dtype, workspace, workspace_bytes, chunk_elems, stream);
}
