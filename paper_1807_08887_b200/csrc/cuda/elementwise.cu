// Element-wise sub-operators (a7).  Under Tofu's coarsening the inputs and output of an element-wise op
// are partitioned identically (§5.1), so every worker runs these on its contiguous shards with
// no communication.  HBM-bound: 128-bit accesses (8 bf16 / 4 fp32 per load), grid = multiple of the SM
// count, grid-stride loop.
#include <cuda_bf16.h>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {

struct bf8 { uint4 u; };
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
  return u;
}

// sum-of-squares reduction scratch (one launch at a time per device: executors run on one stream each)
constexpr int SUMSQ_MAX_BLOCKS = 4096;
__device__ float g_sumsq_part[SUMSQ_MAX_BLOCKS];
__device__ unsigned g_sumsq_ticket = 0;

template <int KIND>
__global__ void __launch_bounds__(256) ew_kernel(int64_t n, void* __restrict__ y, const void* __restrict__ x0,
                                                 const void* __restrict__ x1, void* __restrict__ x2, float s0,
                                                 float s1, float* __restrict__ sumsq_part, unsigned* __restrict__ sumsq_ticket) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int64_t nvec = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float local = 0.f;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const int64_t i = v * 8;
    float a[8], b[8], o[8];
    if (KIND == TOFU_EW_RELU || KIND == TOFU_EW_RELU_GRAD || KIND == TOFU_EW_MSE_GRAD || KIND == TOFU_EW_SUMSQ ||
        KIND == TOFU_EW_ADD || KIND == TOFU_EW_ADDRELU || KIND == TOFU_EW_SUMSQ_MSE_GRAD) {
      unpack8(reinterpret_cast<const uint4*>(x0)[v], a);
      if (KIND != TOFU_EW_RELU) unpack8(reinterpret_cast<const uint4*>(x1)[v], b);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (KIND == TOFU_EW_RELU) o[j] = fmaxf(a[j], 0.f);
        if (KIND == TOFU_EW_RELU_GRAD) o[j] = a[j] > 0.f ? b[j] : 0.f;
        if (KIND == TOFU_EW_MSE_GRAD) o[j] = (a[j] - b[j]) * s0;
        if (KIND == TOFU_EW_SUMSQ || KIND == TOFU_EW_SUMSQ_MSE_GRAD) { const float d = a[j] - b[j]; local += d * d * s0; }
        if (KIND == TOFU_EW_SUMSQ_MSE_GRAD) o[j] = (a[j] - b[j]) * s1;
        if (KIND == TOFU_EW_ADD) o[j] = a[j] + b[j];
        if (KIND == TOFU_EW_ADDRELU) o[j] = fmaxf(a[j] + b[j], 0.f);
      }
      if (KIND == TOFU_EW_SUMSQ_MSE_GRAD) reinterpret_cast<uint4*>(x2)[v] = pack8(o);
      else if (KIND != TOFU_EW_SUMSQ) reinterpret_cast<uint4*>(y)[v] = pack8(o);
    } else if (KIND == TOFU_EW_MOM) {
      const float4* m = reinterpret_cast<const float4*>(x0) + 2 * v;
      const float4* g = reinterpret_cast<const float4*>(x1) + 2 * v;
      float4* out = reinterpret_cast<float4*>(y) + 2 * v;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float4 mm = m[j], gg = g[j];
        out[j] = make_float4(mm.x * s0 + gg.x, mm.y * s0 + gg.y, mm.z * s0 + gg.z, mm.w * s0 + gg.w);
      }
    } else if (KIND == TOFU_EW_SGD) {
      unpack8(reinterpret_cast<const uint4*>(x0)[v], a);
      const float4* m = reinterpret_cast<const float4*>(x1) + 2 * v;
      const float4 m0 = m[0], m1 = m[1];
      const float mv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = a[j] - mv[j] * s0;
      reinterpret_cast<uint4*>(y)[v] = pack8(o);
    } else if (KIND == TOFU_EW_SGD_MOM) {
      float4* m = reinterpret_cast<float4*>(const_cast<void*>(x0)) + 2 * v;
      const float4* g = reinterpret_cast<const float4*>(x1) + 2 * v;
      uint4* w = reinterpret_cast<uint4*>(x2) + v;
      unpack8(*w, a);
      float4 m0 = m[0], m1 = m[1];
      const float4 g0 = g[0], g1 = g[1];
      m0 = make_float4(m0.x * s0 + g0.x, m0.y * s0 + g0.y, m0.z * s0 + g0.z, m0.w * s0 + g0.w);
      m1 = make_float4(m1.x * s0 + g1.x, m1.y * s0 + g1.y, m1.z * s0 + g1.z, m1.w * s0 + g1.w);
      m[0] = m0;
      m[1] = m1;
      const float mv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = a[j] - mv[j] * s1;
      *w = pack8(o);
    }
  }
  // scalar tail (n % 8), handled by block 0
  if (blockIdx.x == 0) {
    for (int64_t i = nvec * 8 + threadIdx.x; i < n; i += blockDim.x) {
      const __nv_bfloat16* xb0 = reinterpret_cast<const __nv_bfloat16*>(x0);
      const __nv_bfloat16* xb1 = reinterpret_cast<const __nv_bfloat16*>(x1);
      if (KIND == TOFU_EW_RELU) reinterpret_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(fmaxf(__bfloat162float(xb0[i]), 0.f));
      if (KIND == TOFU_EW_RELU_GRAD)
        reinterpret_cast<__nv_bfloat16*>(y)[i] = __bfloat162float(xb0[i]) > 0.f ? xb1[i] : __float2bfloat16_rn(0.f);
      if (KIND == TOFU_EW_MSE_GRAD)
        reinterpret_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn((__bfloat162float(xb0[i]) - __bfloat162float(xb1[i])) * s0);
      if (KIND == TOFU_EW_SUMSQ || KIND == TOFU_EW_SUMSQ_MSE_GRAD) {
        const float d = __bfloat162float(xb0[i]) - __bfloat162float(xb1[i]);
        local += d * d * s0;
        if (KIND == TOFU_EW_SUMSQ_MSE_GRAD) reinterpret_cast<__nv_bfloat16*>(x2)[i] = __float2bfloat16_rn(d * s1);
      }
      if (KIND == TOFU_EW_ADD)
        reinterpret_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(__bfloat162float(xb0[i]) + __bfloat162float(xb1[i]));
      if (KIND == TOFU_EW_ADDRELU)
        reinterpret_cast<__nv_bfloat16*>(y)[i] =
            __float2bfloat16_rn(fmaxf(__bfloat162float(xb0[i]) + __bfloat162float(xb1[i]), 0.f));
      if (KIND == TOFU_EW_MOM)
        reinterpret_cast<float*>(y)[i] = reinterpret_cast<const float*>(x0)[i] * s0 + reinterpret_cast<const float*>(x1)[i];
      if (KIND == TOFU_EW_SGD)
        reinterpret_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(__bfloat162float(xb0[i]) - reinterpret_cast<const float*>(x1)[i] * s0);
      if (KIND == TOFU_EW_SGD_MOM) {
        float* m = reinterpret_cast<float*>(const_cast<void*>(x0));
        const float mm = m[i] * s0 + reinterpret_cast<const float*>(x1)[i];
        m[i] = mm;
        __nv_bfloat16* w = reinterpret_cast<__nv_bfloat16*>(x2);
        w[i] = __float2bfloat16_rn(__bfloat162float(w[i]) - mm * s1);
      }
    }
  }
  if (KIND == TOFU_EW_SUMSQ || KIND == TOFU_EW_SUMSQ_MSE_GRAD) {
    // deterministic: per-block partials, summed in block order by the last block to finish (no float atomics,
    // so a loss is bitwise reproducible run to run and across executors)
    __shared__ float red[8];
    __shared__ bool last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
      float s = 0.f;
      for (int w = 0; w < 8; ++w) s += red[w];
      sumsq_part[blockIdx.x] = s;
      __threadfence();
      last = atomicAdd(sumsq_ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      float t = 0.f;
      for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(&sumsq_part[b]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
      __syncthreads();
      if (threadIdx.x == 0) {
        float s = 0.f;
        for (int w = 0; w < 8; ++w) s += red[w];
        *reinterpret_cast<float*>(y) += s;
        *sumsq_ticket = 0;  // ready for the next launch (launches of one stream are ordered)
      }
    }
  }
}

}  // namespace tofu

extern "C" int64_t tofu_sumsq_workspace_bytes(void) { return (int64_t)tofu::SUMSQ_MAX_BLOCKS * 4 + 16; }

extern "C" int tofu_elementwise_ws(int kind, int64_t n, void* y, const void* x0, const void* x1, void* x2, float s0,
                                   float s1, void* ws, void* stream) {
  if (n < 0) return TOFU_ERR_ARG;
  if (n == 0) return TOFU_OK;
  // 16-byte alignment of every buffer for the vector path
  const void* ptrs[4] = {y, x0, x1, x2};
  for (const void* p : ptrs)
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return TOFU_ERR_ALIGN;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = (n / 8 + 255) / 256;
  int64_t grid = sms * 8;
  if (want < grid) grid = want < 1 ? 1 : want;
  if (grid > tofu::SUMSQ_MAX_BLOCKS) grid = tofu::SUMSQ_MAX_BLOCKS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // the loss reduction's block partials and ticket: the caller's workspace, else the module's (one such launch
  // at a time per device)
  float* part = nullptr;
  unsigned* ticket = nullptr;
  if (ws) {
    part = reinterpret_cast<float*>(ws);
    ticket = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ws) + (int64_t)tofu::SUMSQ_MAX_BLOCKS * 4);
  } else {
    void *pp = nullptr, *tp = nullptr;
    if (cudaGetSymbolAddress(&pp, tofu::g_sumsq_part) != cudaSuccess ||
        cudaGetSymbolAddress(&tp, tofu::g_sumsq_ticket) != cudaSuccess)
      return TOFU_ERR_CUDA;
    part = reinterpret_cast<float*>(pp);
    ticket = reinterpret_cast<unsigned*>(tp);
  }
  switch (kind) {
#define K(X) case X: tofu::launch_k(tofu::ew_kernel<X>, dim3((unsigned)grid), dim3(256), 0, st, 1, n, y, x0, x1, x2, s0, s1, part, ticket); break;
    K(TOFU_EW_RELU) K(TOFU_EW_RELU_GRAD) K(TOFU_EW_MSE_GRAD) K(TOFU_EW_MOM) K(TOFU_EW_SGD) K(TOFU_EW_SGD_MOM)
    K(TOFU_EW_SUMSQ) K(TOFU_EW_ADD) K(TOFU_EW_ADDRELU) K(TOFU_EW_SUMSQ_MSE_GRAD)
#undef K
    default: return TOFU_ERR_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}

extern "C" int tofu_elementwise(int kind, int64_t n, void* y, const void* x0, const void* x1, void* x2, float s0,
                                float s1, void* stream) {
  return tofu_elementwise_ws(kind, n, y, x0, x1, x2, s0, s1, nullptr, stream);
}
