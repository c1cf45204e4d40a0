// Window sub-ops of the WResNet stem and head (configs[3]): 3x3/2 max pool and its gradient (the maxpool /
// maxpool_grad TDL defs of tofu_inputs.graphs.wresnet, reading R11 for the zero padding and the
// floor-division / remainder window indices), global average pool and its gradient.  HBM-bound: one thread
// per 8 channels (128-bit loads/stores), grid-stride over the box, grid a multiple of the SM count.
#include <cuda_bf16.h>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {
namespace win {

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ void st8(void* p, const float (&f)[8], bool f32) {
  if (f32) {
    float4* o = reinterpret_cast<float4*>(p);
    o[0] = make_float4(f[0], f[1], f[2], f[3]);
    o[1] = make_float4(f[4], f[5], f[6], f[7]);
    return;
  }
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ int64_t fdiv(int64_t a, int64_t d) { return a >= 0 ? a / d : -((-a + d - 1) / d); }

__global__ void __launch_bounds__(256) maxpool_kernel(tofu_window_args a) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int c8 = a.C / 8;
  const int64_t total = (int64_t)a.nb * a.Ho * a.Wo * c8;
  const __nv_bfloat16* X = reinterpret_cast<const __nv_bfloat16*>(a.X);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cv = (int)(i % c8);
    int64_t r = i / c8;
    const int ox = (int)(r % a.Wo);
    r /= a.Wo;
    const int oy = (int)(r % a.Ho);
    const int b = (int)(r / a.Ho);
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = -3.0e38f;
    for (int ky = 0; ky < 3; ++ky)
      for (int kx = 0; kx < 3; ++kx) {
        const int iy = 2 * (a.oy0 + oy) + ky - 1 - a.y0, ix = 2 * (a.ox0 + ox) + kx - 1 - a.x0;
        float v[8];
        if (iy >= 0 && iy < a.H && ix >= 0 && ix < a.W) {
          ld8(X + b * a.x_sb + iy * a.x_sy + ix * a.x_sx + cv * 8, v);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = 0.f;  // zero padding (R11)
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = fmaxf(m[j], v[j]);
      }
    char* o = reinterpret_cast<char*>(a.out) + (b * a.o_sb + oy * a.o_sy + ox * a.o_sx + cv * 8) * (a.out_f32 ? 4 : 2);
    st8(o, m, a.out_f32);
  }
}

__global__ void __launch_bounds__(256) maxpool_grad_kernel(tofu_window_args a) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int c8 = a.C / 8;
  const int64_t total = (int64_t)a.nb * a.H * a.W * c8;
  const __nv_bfloat16* X = reinterpret_cast<const __nv_bfloat16*>(a.X);
  const __nv_bfloat16* Y = reinterpret_cast<const __nv_bfloat16*>(a.Y);
  const __nv_bfloat16* D = reinterpret_cast<const __nv_bfloat16*>(a.dY);
  const __nv_bfloat16* Km = reinterpret_cast<const __nv_bfloat16*>(a.K);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cv = (int)(i % c8);
    int64_t r = i / c8;
    const int x = (int)(r % a.W);
    r /= a.W;
    const int y = (int)(r % a.H);
    const int b = (int)(r / a.H);
    const int yg = a.y0 + y, xg = a.x0 + x;
    float xv[8], acc[8];
    ld8(X + b * a.x_sb + y * a.x_sy + x * a.x_sx + cv * 8, xv);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int ty = a.ty0; ty <= a.ty1; ++ty) {
      const int ky = (int)(yg + 1 - 2 * fdiv(yg + 1, 2)) + 2 * ty;
      const int oy = (int)fdiv(yg + 1 - 2 * ty, 2) - a.oy0;
      if (ky > 2 || oy < 0 || oy >= a.Ho) continue;  // K (or Y, dY) outside its tensor: 0
      for (int tx = a.tx0; tx <= a.tx1; ++tx) {
        const int kx = (int)(xg + 1 - 2 * fdiv(xg + 1, 2)) + 2 * tx;
        const int ox = (int)fdiv(xg + 1 - 2 * tx, 2) - a.ox0;
        if (kx > 2 || ox < 0 || ox >= a.Wo) continue;
        float yv[8], dv[8], kv[8];
        ld8(Y + b * a.y_sb + oy * a.y_sy + ox * a.y_sx + cv * 8, yv);
        ld8(D + b * a.d_sb + oy * a.d_sy + ox * a.d_sx + cv * 8, dv);
        ld8(Km + ky * a.k_sy + kx * a.k_sx + cv * 8, kv);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += xv[j] == yv[j] ? dv[j] * kv[j] : 0.f;
      }
    }
    char* o = reinterpret_cast<char*>(a.out) + (b * a.o_sb + y * a.o_sy + x * a.o_sx + cv * 8) * (a.out_f32 ? 4 : 2);
    st8(o, acc, a.out_f32);
  }
}

// out[b, c] = Σ_{y,x} X[b,y,x,c] * s: one warp per (b, 8 channels), lanes stride the pixels
__global__ void __launch_bounds__(256) gap_kernel(tofu_window_args a) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int c8 = a.C / 8;
  const int64_t items = (int64_t)a.nb * c8;
  const int lane = threadIdx.x & 31;
  const __nv_bfloat16* X = reinterpret_cast<const __nv_bfloat16*>(a.X);
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < items;
       w += (int64_t)gridDim.x * blockDim.x / 32) {
    const int b = (int)(w / c8), cv = (int)(w % c8);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = lane; p < a.H * a.W; p += 32) {
      const int y = p / a.W, x = p % a.W;
      float v[8];
      ld8(X + b * a.x_sb + y * a.x_sy + x * a.x_sx + cv * 8, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += v[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
      acc[j] *= a.s;
    }
    if (lane == 0) st8(reinterpret_cast<char*>(a.out) + (b * a.o_sb + cv * 8) * (a.out_f32 ? 4 : 2), acc, a.out_f32);
  }
}

__global__ void __launch_bounds__(256) gap_grad_kernel(tofu_window_args a) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int c8 = a.C / 8;
  const int64_t total = (int64_t)a.nb * a.H * a.W * c8;
  const __nv_bfloat16* D = reinterpret_cast<const __nv_bfloat16*>(a.dY);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cv = (int)(i % c8);
    int64_t r = i / c8;
    const int x = (int)(r % a.W);
    r /= a.W;
    const int y = (int)(r % a.H);
    const int b = (int)(r / a.H);
    float v[8];
    ld8(D + b * a.y_sb + cv * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] *= a.s;
    st8(reinterpret_cast<char*>(a.out) + (b * a.o_sb + y * a.o_sy + x * a.o_sx + cv * 8) * (a.out_f32 ? 4 : 2), v,
        a.out_f32);
  }
}

// WT[i][t][o] = W[o][t][i]: 32x32 tiles through shared memory (coalesced reads and writes)
__global__ void __launch_bounds__(256) transpose_taps_kernel(const __nv_bfloat16* __restrict__ W,
                                                             __nv_bfloat16* __restrict__ WT, int co, int taps, int ci) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  __shared__ __nv_bfloat16 tile[32][34];
  const int t = blockIdx.z;
  const int o0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int o = o0 + r, i = i0 + tx;
    if (o < co && i < ci) tile[r][tx] = W[((int64_t)o * taps + t) * ci + i];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, o = o0 + tx;
    if (o < co && i < ci) WT[((int64_t)i * taps + t) * co + o] = tile[tx][r];
  }
}

// Vectorised form (co % 8 == 0, ci % 8 == 0, 16-byte aligned bases): 64 x 64 tiles, 16-byte global loads and
// stores (the scalar kernel above moves 2 bytes per thread per access and ran at ~1.2 TB/s); the tile's row
// pitch of 66 elements (33 words) keeps the column gathers of the store phase free of bank conflicts.
__global__ void __launch_bounds__(256) transpose_taps_v8_kernel(const __nv_bfloat16* __restrict__ W,
                                                                __nv_bfloat16* __restrict__ WT, int co, int taps,
                                                                int ci) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  constexpr int P = 66;
  __shared__ __align__(16) __nv_bfloat16 tile[64 * P];
  const int t = blockIdx.z;
  const int o0 = blockIdx.y * 64, i0 = blockIdx.x * 64;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {  // 64 rows (o) x 8 chunks of 8 (i)
    const int idx = threadIdx.x + pass * 256;
    const int r = idx >> 3, c = idx & 7;
    const int o = o0 + r, i = i0 + 8 * c;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (o < co && i < ci) v = __ldg(reinterpret_cast<const uint4*>(W + ((int64_t)o * taps + t) * ci + i));
    uint32_t* d = reinterpret_cast<uint32_t*>(tile + r * P + 8 * c);
    d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
  }
  __syncthreads();
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {  // 64 rows (i) x 8 chunks of 8 (o)
    const int idx = threadIdx.x + pass * 256;
    const int r = idx >> 3, c = idx & 7;
    const int i = i0 + r, o = o0 + 8 * c;
    if (i >= ci || o >= co) continue;
    __align__(16) __nv_bfloat16 w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = tile[(8 * c + j) * P + r];
    *reinterpret_cast<uint4*>(WT + ((int64_t)i * taps + t) * co + o) = *reinterpret_cast<const uint4*>(w);
  }
}

static int grid_for(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = (work + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

static bool ok(const tofu_window_args* a) {
  auto mis = [](const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 15); };
  return a && a->C % 8 == 0 && !mis(a->X) && !mis(a->Y) && !mis(a->dY) && !mis(a->K) && !mis(a->out) &&
         a->x_sx % 8 == 0 && a->o_sx % 8 == 0;
}

}  // namespace win
}  // namespace tofu

using namespace tofu::win;

extern "C" int tofu_maxpool(const tofu_window_args* a, void* stream) {
  if (!ok(a)) return TOFU_ERR_ALIGN;
  const int64_t n = (int64_t)a->nb * a->Ho * a->Wo * (a->C / 8);
  if (n == 0) return TOFU_OK;
  tofu::launch_k(maxpool_kernel, dim3(grid_for(n)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1, *a);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}
extern "C" int tofu_maxpool_grad(const tofu_window_args* a, void* stream) {
  if (!ok(a)) return TOFU_ERR_ALIGN;
  const int64_t n = (int64_t)a->nb * a->H * a->W * (a->C / 8);
  if (n == 0) return TOFU_OK;
  tofu::launch_k(maxpool_grad_kernel, dim3(grid_for(n)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1, *a);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}
extern "C" int tofu_gap(const tofu_window_args* a, void* stream) {
  if (!ok(a)) return TOFU_ERR_ALIGN;
  const int64_t n = (int64_t)a->nb * (a->C / 8) * 32;
  if (n == 0) return TOFU_OK;
  tofu::launch_k(gap_kernel, dim3(grid_for(n)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1, *a);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}
extern "C" int tofu_gap_grad(const tofu_window_args* a, void* stream) {
  if (!ok(a)) return TOFU_ERR_ALIGN;
  const int64_t n = (int64_t)a->nb * a->H * a->W * (a->C / 8);
  if (n == 0) return TOFU_OK;
  tofu::launch_k(gap_grad_kernel, dim3(grid_for(n)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1, *a);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}

extern "C" int tofu_transpose_taps(const void* W, void* WT, int co, int taps, int ci, void* stream) {
  if (!W || !WT || co < 0 || taps < 0 || ci < 0) return TOFU_ERR_ARG;
  if (co == 0 || taps == 0 || ci == 0) return TOFU_OK;
  const bool v8 = co % 8 == 0 && ci % 8 == 0 && !(reinterpret_cast<uintptr_t>(W) & 15) &&
                  !(reinterpret_cast<uintptr_t>(WT) & 15);
  if (v8) {
    dim3 grid((ci + 63) / 64, (co + 63) / 64, taps);
    tofu::launch_k(tofu::win::transpose_taps_v8_kernel, grid, dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1,
                   reinterpret_cast<const __nv_bfloat16*>(W), reinterpret_cast<__nv_bfloat16*>(WT), co, taps, ci);
  } else {
    dim3 grid((ci + 31) / 32, (co + 31) / 32, taps);
    tofu::launch_k(tofu::win::transpose_taps_kernel, grid, dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1,
                   reinterpret_cast<const __nv_bfloat16*>(W), reinterpret_cast<__nv_bfloat16*>(WT), co, taps, ci);
  }
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}
