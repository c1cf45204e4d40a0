// MultiFetch and partition-n-reduce pieces (a5, a6).
//
// MultiFetch (§6): "Our MultiFetch kernel takes multiple pointers to the memory blocks of the
// input regions from the other GPUs and assembles them in one kernel launch" — one launch moves every
// piece of a (op, input) region from its owners (peer HBM over NVLink, addressed directly) into the
// consumer's staging buffer.
// Spread reduction (§6): every owner reduces its own slice — it pulls the fp32 partials of all
// contributors for the elements it owns, sums them in ascending rank order and stores the result in the
// tensor's dtype.  The same piece kernel does both: nsrc == 1 is a copy, nsrc > 1 an ordered sum.
//
// Layout: one CTA row (blockIdx.y) per piece, blockIdx.x strides over the piece's elements.  The
// innermost dimension is processed 4 elements per thread (16-byte fp32 / 8-byte bf16 accesses) when
// extents, strides and pointers allow it.
#include <cuda_bf16.h>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {

__device__ __forceinline__ float ld_elem(const void* p, int64_t i, int dt) {
  return dt == TOFU_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i])
                         : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void st_elem(void* p, int64_t i, int dt, float v) {
  if (dt == TOFU_BF16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else reinterpret_cast<float*>(p)[i] = v;
}
__device__ __forceinline__ float4 ld4(const void* p, int64_t i, int dt) {
  if (dt == TOFU_BF16) {
    const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(p) + i);
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    return make_float4(fa.x, fa.y, fb.x, fb.y);
  }
  return *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + i);
}
__device__ __forceinline__ void st4(void* p, int64_t i, int dt, float4 v) {
  if (dt == TOFU_BF16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p) + i) = u;
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + i) = v;
  }
}

__device__ __forceinline__ bool piece_vec_ok(const tofu_piece& pc) {
  if (pc.extent[3] % 4 || pc.dst_stride[3] != 1 || pc.src_stride[3] != 1) return false;
  const int da = pc.dst_dtype == TOFU_BF16 ? 8 : 16, sa = pc.src_dtype == TOFU_BF16 ? 8 : 16;
  const int de = pc.dst_dtype == TOFU_BF16 ? 2 : 4, se = pc.src_dtype == TOFU_BF16 ? 2 : 4;
  if (reinterpret_cast<uintptr_t>(pc.dst) % da) return false;
  for (int d = 0; d < 3; ++d)
    if ((pc.dst_stride[d] * de) % da || (pc.src_stride[d] * se) % sa) return false;
  for (int s = 0; s < pc.nsrc; ++s)
    if (reinterpret_cast<uintptr_t>(pc.src[s]) % sa) return false;
  return true;
}

__global__ void __launch_bounds__(256) pieces_kernel(const tofu_piece* __restrict__ pieces) {
  const tofu_piece& pc = pieces[blockIdx.y];
  const int64_t e0 = pc.extent[0], e1 = pc.extent[1], e2 = pc.extent[2], e3 = pc.extent[3];
  const bool vec = piece_vec_ok(pc);
  const int64_t inner = vec ? e3 / 4 : e3;
  const int64_t total = e0 * e1 * e2 * inner;
  const int nsrc = pc.nsrc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    const int64_t c3 = r % inner; r /= inner;
    const int64_t c2 = r % e2; r /= e2;
    const int64_t c1 = r % e1;
    const int64_t c0 = r / e1;
    const int64_t x3 = vec ? c3 * 4 : c3;
    const int64_t so = c0 * pc.src_stride[0] + c1 * pc.src_stride[1] + c2 * pc.src_stride[2] + x3 * pc.src_stride[3];
    const int64_t dof = c0 * pc.dst_stride[0] + c1 * pc.dst_stride[1] + c2 * pc.dst_stride[2] + x3 * pc.dst_stride[3];
    if (vec) {
      float4 acc = ld4(pc.src[0], so, pc.src_dtype);
      for (int s = 1; s < nsrc; ++s) {
        const float4 v = ld4(pc.src[s], so, pc.src_dtype);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      st4(pc.dst, dof, pc.dst_dtype, acc);
    } else {
      float acc = ld_elem(pc.src[0], so, pc.src_dtype);
      for (int s = 1; s < nsrc; ++s) acc += ld_elem(pc.src[s], so, pc.src_dtype);
      st_elem(pc.dst, dof, pc.dst_dtype, acc);
    }
  }
}

}  // namespace tofu

extern "C" int tofu_pieces_run(const tofu_piece* pieces_dev, int n, int64_t max_elems, void* stream) {
  if (n <= 0 || max_elems <= 0) return TOFU_OK;
  if (n > 65535) return TOFU_ERR_ARG;
  int64_t blocks = (max_elems + 256 * 4 - 1) / (256 * 4);
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;  // 8 x 148 SMs; grid-stride beyond
  tofu::pieces_kernel<<<dim3((unsigned)blocks, (unsigned)n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      pieces_dev);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}

// Cross-process device barrier over NVLink (multi-process mode only).  Each rank bumps its own epoch
// word (system-scope release) and waits until every peer's word reaches the same epoch (system-scope
// acquire on the peer mapping).  flags: device array of n pointers (peer-mapped epoch words).
namespace tofu {
__global__ void barrier_kernel(unsigned long long* const* flags, int rank, int n) {
  __shared__ unsigned long long epoch;
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.release.sys.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(flags[rank]) : "memory");
    epoch = old + 1;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    unsigned long long v;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags[p]) : "memory");
    } while (v < epoch);
  }
  __syncthreads();
}
}  // namespace tofu

extern "C" int tofu_barrier_run(void* flags_ptrs_dev, int rank, int n, void* stream) {
  tofu::barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long* const*>(flags_ptrs_dev), rank, n);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}
