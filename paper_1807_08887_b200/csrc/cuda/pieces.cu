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
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>

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

// Work decomposition (host, tofu_pieces_tasks): each piece is normalised — dimensions that are contiguous in
// the destination AND the sources are merged, so a piece is a set of rows of e3 contiguous elements — and
// given a vector width V (8, 4, 2 or 1 elements; V = 8 moves 16 bytes of bf16 per load) that divides the row
// and keeps every row start aligned.  Rows are cut into segments of <= kSeg vectors and a launch's pieces
// into tasks of ~kTaskVecs vectors of whole segments; CTAs walk the task list (grid-stride), one warp per
// segment, lanes over its vectors with several vectors per lane in flight (kUnr), so peer (NVLink) and
// local HBM reads keep enough bytes outstanding.
constexpr int kTaskVecs = 4096;
constexpr int kSeg = 256;   // vectors per segment (one warp's unit of work)
constexpr int kUnr = 4;    // raw copies: 16-byte moves in flight per lane
#ifndef TOFU_PIECES_UNRC
#define TOFU_PIECES_UNRC 1
#endif
#ifndef TOFU_PIECES_MINB
#define TOFU_PIECES_MINB 2
#endif
constexpr int kUnrC = TOFU_PIECES_UNRC;   // converting / summing path: vectors in flight per lane (1: 8 x fp32 -> bf16 reduce 2.0 -> 2.9 TB/s)

template <int V, typename ST>
struct Vec;  // V elements of storage type ST
template <>
struct Vec<8, __nv_bfloat16> { uint4 u; };
template <>
struct Vec<4, __nv_bfloat16> { uint2 u; };
template <>
struct Vec<2, __nv_bfloat16> { uint32_t u; };
template <>
struct Vec<1, __nv_bfloat16> { unsigned short u; };
template <int V>
struct Vec<V, float> { float f[V]; };

template <int V>
__device__ __forceinline__ void load_f(const void* p, int64_t i, int dt, float (&x)[V]) {
  if (dt == TOFU_BF16) {
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(p) + i;
    if constexpr (V == 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(b);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
        x[2 * q] = f.x;
        x[2 * q + 1] = f.y;
      }
    } else if constexpr (V == 4) {
      const uint2 u = *reinterpret_cast<const uint2*>(b);
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      x[0] = f0.x; x[1] = f0.y; x[2] = f1.x; x[3] = f1.y;
    } else if constexpr (V == 2) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(b));
      x[0] = f.x; x[1] = f.y;
    } else {
      x[0] = __bfloat162float(*b);
    }
  } else {
    const float* f = reinterpret_cast<const float*>(p) + i;
    if constexpr (V >= 4) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) {
        const float4 v = reinterpret_cast<const float4*>(f)[q];
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
      }
    } else if constexpr (V == 2) {
      const float2 v = *reinterpret_cast<const float2*>(f);
      x[0] = v.x; x[1] = v.y;
    } else {
      x[0] = *f;
    }
  }
}

template <int V>
__device__ __forceinline__ void store_f(void* p, int64_t i, int dt, const float (&x)[V]) {
  if (dt == TOFU_BF16) {
    __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(p) + i;
    if constexpr (V >= 2) {
      uint32_t w[V / 2];
#pragma unroll
      for (int q = 0; q < V / 2; ++q) {
        __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * q], x[2 * q + 1]);
        w[q] = *reinterpret_cast<uint32_t*>(&h);
      }
      if constexpr (V == 8) *reinterpret_cast<uint4*>(b) = make_uint4(w[0], w[1], w[2], w[3]);
      else if constexpr (V == 4) *reinterpret_cast<uint2*>(b) = make_uint2(w[0], w[1]);
      else *reinterpret_cast<uint32_t*>(b) = w[0];
    } else {
      *b = __float2bfloat16_rn(x[0]);
    }
  } else {
    float* f = reinterpret_cast<float*>(p) + i;
    if constexpr (V >= 4) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q)
        reinterpret_cast<float4*>(f)[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    } else if constexpr (V == 2) {
      *reinterpret_cast<float2*>(f) = make_float2(x[0], x[1]);
    } else {
      *f = x[0];
    }
  }
}

// Moves segments [q0, q0 + nq) of piece pc.  A row of rv vectors is cut into ceil(rv / kSeg) segments of
// <= kSeg vectors; segment q is (row q / nseg, vectors [(q % nseg) * kSeg, ...)).  Warp w of the CTA takes
// segments q0 + w, q0 + w + nwarps, ...: the row's (c0, c1, c2) is decoded once per segment, then the lanes
// stride over its vectors, kUnr vectors per lane in flight (loads of every source issued before the stores).
template <int V, bool WIDE>
__device__ __forceinline__ void run_task(const tofu_piece& pc, int64_t q0, int64_t nq) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t rv = pc.extent[3] / V;
  const uint32_t nseg = (uint32_t)((rv + kSeg - 1) / kSeg);
  const uint32_t e2 = (uint32_t)pc.extent[2], e1 = (uint32_t)pc.extent[1];
  const int nsrc = pc.nsrc, ep = pc.ep;
  const int sdt = pc.src_dtype, ddt = pc.dst_dtype;
  for (int64_t qq = warp; qq < nq; qq += nwarps) {
    const uint32_t q = (uint32_t)(q0 + qq);
    uint32_t row = q / nseg;
    const int64_t jb = (int64_t)(q - row * nseg) * kSeg, je = min(rv, jb + kSeg);
    const uint32_t c2 = row % e2;
    row /= e2;
    const uint32_t c1 = row % e1;
    const uint32_t c0 = row / e1;
    const int64_t sb = c0 * pc.src_stride[0] + c1 * pc.src_stride[1] + c2 * pc.src_stride[2];
    const int64_t db = c0 * pc.dst_stride[0] + c1 * pc.dst_stride[1] + c2 * pc.dst_stride[2];
    if constexpr (WIDE) {
      // every source's vector (and the consumer's operands) in flight at once: one DRAM / NVLink round trip
      // per vector instead of one per source; the sum still runs in rank order (bitwise as the other path).
      // ~210 registers: one 256-thread CTA per SM (pieces_kernel_wide), used for launches of >= 4 sources
      for (int64_t j = jb + lane; j < je; j += 32) {
        float xs[TOFU_MAX_SRC][V];
#pragma unroll
        for (int k = 0; k < TOFU_MAX_SRC; ++k)
          if (k < nsrc) load_f<V>(pc.src[k], sb + j * V, sdt, xs[k]);
        float a[V], m[V];
        if (ep == TOFU_PIECE_MOM_SGD) {
          load_f<V>(pc.dst, db + j * V, TOFU_F32, m);
          load_f<V>(pc.aux0, db + j * V, TOFU_BF16, a);
        } else if (ep != TOFU_PIECE_COPY && ep != TOFU_PIECE_RELU) {
          load_f<V>(pc.aux0, db + j * V, TOFU_BF16, a);
        }
        float acc[V];
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = xs[0][q];
#pragma unroll
        for (int k = 1; k < TOFU_MAX_SRC; ++k)
          if (k < nsrc)
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] += xs[k][q];
        if (ep == TOFU_PIECE_RELU) {
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = fmaxf(acc[q], 0.f);
        } else if (ep == TOFU_PIECE_MOM_SGD) {
#pragma unroll
          for (int q = 0; q < V; ++q) {
            m[q] = m[q] * pc.s0 + acc[q];
            a[q] = a[q] - m[q] * pc.s1;
            acc[q] = m[q];
          }
          store_f<V>(pc.aux0, db + j * V, TOFU_BF16, a);
        } else if (ep != TOFU_PIECE_COPY) {
#pragma unroll
          for (int q = 0; q < V; ++q) {
            if (ep == TOFU_PIECE_MASK) acc[q] = a[q] > 0.f ? acc[q] : 0.f;
            else if (ep == TOFU_PIECE_ADD) acc[q] = acc[q] + a[q];
            else acc[q] = fmaxf(acc[q] + a[q], 0.f);
          }
        }
        store_f<V>(pc.dst, db + j * V, ddt, acc);
      }
      continue;
    }
    for (int64_t j0 = jb + lane; j0 < je; j0 += 32 * kUnrC) {
      float acc[kUnrC][V];
#pragma unroll
      for (int u = 0; u < kUnrC; ++u) {
        const int64_t j = j0 + 32 * u;
        if (j < je) load_f<V>(pc.src[0], sb + j * V, sdt, acc[u]);
      }
      for (int s = 1; s < nsrc; ++s) {  // ordered sum (rank order): the spread reduction
#pragma unroll
        for (int u = 0; u < kUnrC; ++u) {
          const int64_t j = j0 + 32 * u;
          if (j < je) {
            float x[V];
            load_f<V>(pc.src[s], sb + j * V, sdt, x);
#pragma unroll
            for (int qv = 0; qv < V; ++qv) acc[u][qv] += x[qv];
          }
        }
      }
      if (ep != TOFU_PIECE_COPY) {  // the reduced tensor's element-wise consumer (aux0 laid out like dst)
#pragma unroll
        for (int u = 0; u < kUnrC; ++u) {
          const int64_t j = j0 + 32 * u;
          if (j >= je) continue;
          float a[V];
          if (ep == TOFU_PIECE_RELU) {
#pragma unroll
            for (int q = 0; q < V; ++q) acc[u][q] = fmaxf(acc[u][q], 0.f);
          } else if (ep == TOFU_PIECE_MOM_SGD) {
            float m[V];
            load_f<V>(pc.dst, db + j * V, TOFU_F32, m);
            load_f<V>(pc.aux0, db + j * V, TOFU_BF16, a);
#pragma unroll
            for (int q = 0; q < V; ++q) {
              m[q] = m[q] * pc.s0 + acc[u][q];
              a[q] = a[q] - m[q] * pc.s1;
              acc[u][q] = m[q];
            }
            store_f<V>(pc.aux0, db + j * V, TOFU_BF16, a);
          } else {
            load_f<V>(pc.aux0, db + j * V, TOFU_BF16, a);
#pragma unroll
            for (int q = 0; q < V; ++q) {
              if (ep == TOFU_PIECE_MASK) acc[u][q] = a[q] > 0.f ? acc[u][q] : 0.f;
              else if (ep == TOFU_PIECE_ADD) acc[u][q] = acc[u][q] + a[q];
              else acc[u][q] = fmaxf(acc[u][q] + a[q], 0.f);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kUnrC; ++u) {
        const int64_t j = j0 + 32 * u;
        if (j < je) store_f<V>(pc.dst, db + j * V, ddt, acc[u]);
      }
    }
  }
}

// Plain copies (one source, same dtype): raw 16-byte moves, kUnr in flight per lane, few registers (high
// occupancy: the many bytes in flight a copy over NVLink / HBM needs).  Requires V * itemsize % 16 == 0 for
// every piece (checked on the host: the task's pad_ is 1).
__global__ void __launch_bounds__(256) pieces_copy_kernel(const tofu_piece* __restrict__ pieces,
                                                          const tofu_piece_task* __restrict__ tasks, int ntasks) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const tofu_piece_task T = tasks[t];
    const tofu_piece& pc = pieces[T.piece];
    const int esz = pc.src_dtype == TOFU_BF16 ? 2 : 4, V = pc.pad_;
    const int w = V * esz / 16;  // uint4 per vector
    const int64_t rv = pc.extent[3] / V;
    const uint32_t nseg = (uint32_t)((rv + kSeg - 1) / kSeg);
    const uint32_t e2 = (uint32_t)pc.extent[2], e1 = (uint32_t)pc.extent[1];
    for (int64_t qq = warp; qq < T.nq; qq += nwarps) {
      const uint32_t q = (uint32_t)(T.q0 + qq);
      uint32_t row = q / nseg;
      const int64_t jb = (int64_t)(q - row * nseg) * kSeg, je = min(rv, jb + kSeg);
      const uint32_t c2 = row % e2;
      row /= e2;
      const uint32_t c1 = row % e1;
      const uint32_t c0 = row / e1;
      const uint4* src = reinterpret_cast<const uint4*>(
          static_cast<const char*>(pc.src[0]) +
          (c0 * pc.src_stride[0] + c1 * pc.src_stride[1] + c2 * pc.src_stride[2]) * esz);
      uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(pc.dst) +
                                            (c0 * pc.dst_stride[0] + c1 * pc.dst_stride[1] + c2 * pc.dst_stride[2]) * esz);
      const int64_t b1 = je * w;
      for (int64_t i0 = jb * w + lane; i0 < b1; i0 += 32 * kUnr) {
        uint4 r[kUnr];
#pragma unroll
        for (int u = 0; u < kUnr; ++u)
          if (i0 + 32 * u < b1) r[u] = __ldg(src + i0 + 32 * u);
#pragma unroll
        for (int u = 0; u < kUnr; ++u)
          if (i0 + 32 * u < b1) dst[i0 + 32 * u] = r[u];
      }
    }
  }
}

template <bool WIDE>
__device__ __forceinline__ void pieces_body(const tofu_piece* __restrict__ pieces,
                                            const tofu_piece_task* __restrict__ tasks, int ntasks) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const tofu_piece_task T = tasks[t];
    const tofu_piece& pc = pieces[T.piece];
    switch (pc.pad_) {
      case 8: run_task<8, WIDE>(pc, T.q0, T.nq); break;
      case 4: run_task<4, WIDE>(pc, T.q0, T.nq); break;
      case 2: run_task<2, WIDE>(pc, T.q0, T.nq); break;
      default: run_task<1, WIDE>(pc, T.q0, T.nq); break;
    }
  }
}
__global__ void __launch_bounds__(256, TOFU_PIECES_MINB) pieces_kernel(const tofu_piece* __restrict__ pieces,
                                                     const tofu_piece_task* __restrict__ tasks, int ntasks) {
  pieces_body<false>(pieces, tasks, ntasks);
}
// Measured (tools/pieces_bench.py, graph replay): 8 x fp32 -> bf16 [1024 x 4096] 47.0 -> 29.2 us (3.0 -> 4.9 TB/s),
// 4 x fp32 -> bf16 [12544 x 1024] 68.9 -> 59.7 us; 2 sources slower (19.0 -> 32.2 us): launches of >= 4 sources only
__global__ void __launch_bounds__(256, 1) pieces_kernel_wide(const tofu_piece* __restrict__ pieces,
                                                          const tofu_piece_task* __restrict__ tasks, int ntasks) {
  pieces_body<true>(pieces, tasks, ntasks);
}

}  // namespace tofu

extern "C" int tofu_pieces_tasks(tofu_piece* pieces, int n, tofu_piece_task* tasks, int64_t cap, int64_t* ntasks) {
  if ((n > 0 && !pieces) || !ntasks || cap < 0) return TOFU_ERR_ARG;
  int64_t nt = 0;
  for (int p = 0; p < n; ++p) {
    tofu_piece& pc = pieces[p];
    if (pc.nsrc < 1 || pc.nsrc > TOFU_MAX_SRC || pc.ep < TOFU_PIECE_COPY || pc.ep > TOFU_PIECE_ADDRELU) return TOFU_ERR_ARG;
    if (pc.ep == TOFU_PIECE_MOM_SGD && pc.dst_dtype != TOFU_F32) return TOFU_ERR_ARG;
    // merge dims contiguous in dst and src (inner to outer), drop unit dims
    int64_t ex[4], ds[4], ss[4];
    int m = 0;
    for (int d = 3; d >= 0; --d) {
      if (pc.extent[d] == 1 && d != 3) continue;
      if (m > 0 && ds[m - 1] * ex[m - 1] == pc.dst_stride[d] && ss[m - 1] * ex[m - 1] == pc.src_stride[d]) {
        ex[m - 1] *= pc.extent[d];
        continue;
      }
      ex[m] = pc.extent[d];
      ds[m] = pc.dst_stride[d];
      ss[m] = pc.src_stride[d];
      ++m;
    }
    if (m > 4) return TOFU_ERR_ARG;
    for (int d = 0; d < 4; ++d) {
      const int q = 3 - d;  // q-th innermost
      pc.extent[d] = q < m ? ex[q] : 1;
      pc.dst_stride[d] = q < m ? ds[q] : 0;
      pc.src_stride[d] = q < m ? ss[q] : 0;
    }
    const int64_t total = pc.extent[0] * pc.extent[1] * pc.extent[2] * pc.extent[3];
    if (total <= 0) {
      pc.pad_ = 1;
      continue;
    }
    if (pc.extent[0] * pc.extent[1] * pc.extent[2] > 0xFFFFFFFFll || pc.extent[3] > 0xFFFFFFFFll) return TOFU_ERR_ARG;
    // vector width: divides the row, keeps row starts and base pointers aligned to V elements
    const int de = pc.dst_dtype == TOFU_BF16 ? 2 : 4, se = pc.src_dtype == TOFU_BF16 ? 2 : 4;
    int V = 8;
    for (; V > 1; V /= 2) {
      bool ok = pc.extent[3] % V == 0 && pc.dst_stride[3] == 1 && pc.src_stride[3] == 1;
      for (int d = 0; d < 3 && ok; ++d) ok = pc.dst_stride[d] % V == 0 && pc.src_stride[d] % V == 0;
      ok = ok && reinterpret_cast<uintptr_t>(pc.dst) % (V * de) == 0;
      for (int s = 0; s < pc.nsrc && ok; ++s) ok = reinterpret_cast<uintptr_t>(pc.src[s]) % (V * se) == 0;
      if (pc.ep != TOFU_PIECE_COPY && pc.ep != TOFU_PIECE_RELU) ok = ok && reinterpret_cast<uintptr_t>(pc.aux0) % (V * 2) == 0;
      if (ok) break;
    }
    if (V == 1 && (pc.dst_stride[3] != 1 || pc.src_stride[3] != 1)) {
      // a strided innermost dim: move it out as a row dim of length-1 rows
      if (pc.extent[0] != 1) return TOFU_ERR_ARG;
      for (int d = 0; d < 3; ++d) {
        pc.extent[d] = pc.extent[d + 1];
        pc.dst_stride[d] = pc.dst_stride[d + 1];
        pc.src_stride[d] = pc.src_stride[d + 1];
      }
      pc.extent[3] = 1;
      pc.dst_stride[3] = pc.src_stride[3] = 1;
    }
    pc.pad_ = V;
    // tasks: ~kTaskVecs vectors of whole segments (>= 8 segments: one per warp) each
    const int64_t rows = pc.extent[0] * pc.extent[1] * pc.extent[2], rv = pc.extent[3] / V;
    const int64_t nseg = (rv + tofu::kSeg - 1) / tofu::kSeg, seglen = std::min<int64_t>(rv, tofu::kSeg);
    const int64_t nq = rows * nseg;
    if (nq > 0xFFFFFFFFll) return TOFU_ERR_ARG;   // 32-bit segment index in the kernel
    const int64_t per = std::max<int64_t>(8, tofu::kTaskVecs / std::max<int64_t>(seglen, 1));
    const int raw = pc.nsrc == 1 && pc.src_dtype == pc.dst_dtype && (V * se) % 16 == 0 && pc.ep == TOFU_PIECE_COPY;
    for (int64_t q0 = 0; q0 < nq; q0 += per) {
      if (nt < cap && tasks) tasks[nt] = tofu_piece_task{p, raw, q0, std::min<int64_t>(per, nq - q0)};
      ++nt;
    }
  }
  *ntasks = nt;
  return nt > cap && tasks ? TOFU_ERR_SPACE : TOFU_OK;
}

extern "C" int tofu_pieces_run(const tofu_piece* pieces_dev, const tofu_piece_task* tasks_dev, int64_t ntasks,
                               int all_raw, void* stream) {
  if (ntasks <= 0) return TOFU_OK;
  const int64_t grid = std::min<int64_t>(ntasks, 148 * 8);
  const int n = (int)std::min<int64_t>(ntasks, INT32_MAX);
  if (all_raw == 1)
    tofu::launch_k(tofu::pieces_copy_kernel, dim3((unsigned)grid), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1,
                   pieces_dev, tasks_dev, n);
  else if (all_raw == 2)
    tofu::launch_k(tofu::pieces_kernel_wide, dim3((unsigned)std::min<int64_t>(ntasks, 148)), dim3(256), 0,
                   reinterpret_cast<cudaStream_t>(stream), 1, pieces_dev, tasks_dev, n);
  else
    tofu::launch_k(tofu::pieces_kernel, dim3((unsigned)grid), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1,
                   pieces_dev, tasks_dev, n);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}

// Cross-process device barrier over NVLink (multi-process mode only).  Each rank bumps its own epoch
// word (system-scope release) and waits until every peer's word reaches the same epoch (system-scope
// acquire on the peer mapping).  flags: device array of n pointers (peer-mapped epoch words).
namespace tofu {
__global__ void barrier_kernel(unsigned long long* const* flags, int rank, int n) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
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
  tofu::launch_k(tofu::barrier_kernel, dim3(1), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), 1,
                 reinterpret_cast<unsigned long long* const*>(flags_ptrs_dev), rank, n);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}

// Jitter injection (tests of the cross-process synchronisation): one thread spins for ns
// nanoseconds of %globaltimer, delaying everything after it on the stream.
namespace tofu {
__global__ void spin_kernel(uint64_t ns) {
  pdl_trigger();
  pdl_wait();
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}
}  // namespace tofu

extern "C" int tofu_spin(int64_t ns, void* stream) {
  if (ns <= 0) return TOFU_OK;
  return tofu::launch_k(tofu::spin_kernel, dim3(1), dim3(1), 0, reinterpret_cast<cudaStream_t>(stream), 1,
                        (uint64_t)ns) == cudaSuccess
             ? TOFU_OK
             : TOFU_ERR_CUDA;
}
