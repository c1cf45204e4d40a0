// LSTM cell sub-operators (configs[2]; LSTM cell of the paper's RNN benchmark).
//
// Gate pre-activations a_x = GX[b, x, h] + GH[b, x, h], x in {i=0, f=1, g=2, o=3}:
//   cell_c     : c_t  = sigmoid(a_f) * c_{t-1} + sigmoid(a_i) * tanh(a_g)
//   cell_h     : h_t  = sigmoid(a_o) * tanh(c_t)
//   cell_bwd_a : dA[b, x, h] = d loss / d a_x  (x in the op's gate range)
//   cell_bwd_c : d loss / d c_{t-1}
// with dh = DU + DR (from the layer above and from step t+1) and dc = DN + dh * o * (1 - tanh(c_t)^2).
// The formulas are the TDL defs of tofu_inputs/graphs.py (oracle-checked against finite differences).
// Kinds 4 (cell_c + cell_h) and 5 (cell_bwd_a + cell_bwd_c) are the executor's fusions of the two ops of
// one timestep that read the same gate rows: one pass over GX / GH instead of two (HBM-bound kernels).
// Operands are pitched views of the (b, [gate,] h) box: element (b, x, h) at p[b*ld + x*gs + h].
// Each thread handles V consecutive h of one b (V = 8: 16-byte bf16 / 2x16-byte fp32 accesses when every
// operand allows it, else V = 1).
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {

struct LOpnd {
  const void* p;
  int64_t ld, gs;
  int dt;
};

struct LstmArgs {
  int kind;  // 0 c, 1 h, 2 bwd_a, 3 bwd_c, 4 c+h, 5 bwd_a+bwd_c
  int64_t nb, nh;
  int g0, ng;  // gate range of the dA output
  LOpnd gx, gh, cp, c, du, dr, dn;
  void* out;  // c / h / dA / dC
  int64_t out_ld, out_gs;
  int out_dt;
  void* out2;  // fused second output: h (kind 4) or dC (kind 5)
  int64_t out2_ld;
  int out2_dt;
  // gate GEMM + cell fusion (kinds 0 / 4): GH comes as the GEMM's fp32 split-K partial planes (dense
  // [splits][nb][ng * nh], plane stride gh_plane, row pitch gh_wld, gate stride gh_wgs), summed in split order
  // (the GEMM's own reduction), rounded to GH's dtype, stored to GH (gh_out) and used as stored
  const float* ghws;
  int gh_splits;
  int64_t gh_plane, gh_wld, gh_wgs;
  void* gh_out;
  int64_t gh_out_ld, gh_out_gs;
  int gh_out_dt;
};

template <int V>
__device__ __forceinline__ void ldv(const LOpnd& o, int64_t i, float (&v)[V]) {
  if (V == 8) {
    if (o.dt == TOFU_BF16) {
      const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(o.p) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
      }
    } else {
      const float4 a = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(o.p) + i);
      const float4 b = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(o.p) + i + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
  } else if (V == 4) {
    if (o.dt == TOFU_BF16) {
      const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(o.p) + i);
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      v[0] = f0.x; v[1] = f0.y; v[2 % V] = f1.x; v[3 % V] = f1.y;
    } else {
      const float4 a = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(o.p) + i);
      v[0] = a.x; v[1 % V] = a.y; v[2 % V] = a.z; v[3 % V] = a.w;
    }
  } else {
    v[0] = o.dt == TOFU_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(o.p)[i])
                             : reinterpret_cast<const float*>(o.p)[i];
  }
}

template <int V>
__device__ __forceinline__ void stv(void* p, int dt, int64_t i, const float (&v)[V]) {
  if (V == 8) {
    if (dt == TOFU_BF16) {
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p) + i) = u;
    } else {
      float* f = reinterpret_cast<float*>(p) + i;
      *reinterpret_cast<float4*>(f) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(f + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  } else if (V == 4) {
    if (dt == TOFU_BF16) {
      uint2 u;
      *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(v[0], v[1 % V]);
      *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(v[2 % V], v[3 % V]);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p) + i) = u;
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + i) = make_float4(v[0], v[1 % V], v[2 % V], v[3 % V]);
    }
  } else {
    if (dt == TOFU_BF16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v[0]);
    else reinterpret_cast<float*>(p)[i] = v[0];
  }
}

__device__ __forceinline__ float sig(float x) { return 1.f / (1.f + __expf(-x)); }

template <int V, bool SPLIT>
__device__ __forceinline__ void ld_gh(const LstmArgs& a, int64_t b, int64_t h, int x, float (&t)[V]) {
  if constexpr (!SPLIT) {
    ldv<V>(a.gh, b * a.gh.ld + h + x * a.gh.gs, t);
    return;
  }
  const int64_t wo = b * a.gh_wld + x * a.gh_wgs + h;
  // the planes' vectors in flight 8 at a time, summed in split order (the GEMM's own reduction order)
  constexpr int kBatch = 8;
  for (int s0 = 0; s0 < a.gh_splits; s0 += kBatch) {
    float u[kBatch][V];
#pragma unroll
    for (int q = 0; q < kBatch; ++q)
      if (s0 + q < a.gh_splits) ldv<V>(LOpnd{a.ghws, 0, 0, TOFU_F32}, wo + (s0 + q) * a.gh_plane, u[q]);
#pragma unroll
    for (int q = 0; q < kBatch; ++q)
      if (s0 + q < a.gh_splits)
#pragma unroll
        for (int j = 0; j < V; ++j) t[j] = (s0 + q == 0) ? u[q][j] : t[j] + u[q][j];
  }
  stv<V>(a.gh_out, a.gh_out_dt, b * a.gh_out_ld + x * a.gh_out_gs + h, t);
  if (a.gh_out_dt == TOFU_BF16)
#pragma unroll
    for (int j = 0; j < V; ++j) t[j] = __bfloat162float(__float2bfloat16_rn(t[j]));
}

template <int V, bool SPLIT = false>
__global__ void __launch_bounds__(256) lstm_kernel(const LstmArgs a) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int64_t nhv = a.nh / V;
  const int64_t n = a.nb * nhv;
  const int kind = a.kind;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / nhv, h = (e % nhv) * V;
    const int64_t go = b * a.gx.ld + h;
    float I[V], F[V], G[V], O[V], t0[V], t1[V];
    ldv<V>(a.gx, go, t0);
    ld_gh<V, SPLIT>(a, b, h, 0, t1);
#pragma unroll
    for (int j = 0; j < V; ++j) I[j] = sig(t0[j] + t1[j]);
    ldv<V>(a.gx, go + a.gx.gs, t0);
    ld_gh<V, SPLIT>(a, b, h, 1, t1);
#pragma unroll
    for (int j = 0; j < V; ++j) F[j] = sig(t0[j] + t1[j]);
    ldv<V>(a.gx, go + 2 * a.gx.gs, t0);
    ld_gh<V, SPLIT>(a, b, h, 2, t1);
#pragma unroll
    for (int j = 0; j < V; ++j) G[j] = tanhf(t0[j] + t1[j]);
    ldv<V>(a.gx, go + 3 * a.gx.gs, t0);
    ld_gh<V, SPLIT>(a, b, h, 3, t1);
#pragma unroll
    for (int j = 0; j < V; ++j) O[j] = sig(t0[j] + t1[j]);
    if (kind == 0 || kind == 4) {
      float cp[V], c[V];
      ldv<V>(a.cp, b * a.cp.ld + h, cp);
#pragma unroll
      // (explicit roundings, no contraction: the vector widths 1 / 4 / 8 then agree bitwise)
      for (int j = 0; j < V; ++j) c[j] = __fadd_rn(__fmul_rn(F[j], cp[j]), __fmul_rn(I[j], G[j]));
      stv<V>(a.out, a.out_dt, b * a.out_ld + h, c);
      if (kind == 4) {
        // h_t from the c_t as stored (fp32 storage of the c tensor: identical to the unfused cell_h input)
        float hh[V];
#pragma unroll
        for (int j = 0; j < V; ++j) hh[j] = O[j] * tanhf(c[j]);
        stv<V>(a.out2, a.out2_dt, b * a.out2_ld + h, hh);
      }
    } else if (kind == 1) {
      float c[V], hh[V];
      ldv<V>(a.c, b * a.c.ld + h, c);
#pragma unroll
      for (int j = 0; j < V; ++j) hh[j] = O[j] * tanhf(c[j]);
      stv<V>(a.out, a.out_dt, b * a.out_ld + h, hh);
    } else {
      float c[V], du[V], dr[V], dn[V], dh[V], dc[V], tc[V];
      ldv<V>(a.c, b * a.c.ld + h, c);
      ldv<V>(a.du, b * a.du.ld + h, du);
      ldv<V>(a.dr, b * a.dr.ld + h, dr);
      ldv<V>(a.dn, b * a.dn.ld + h, dn);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        tc[j] = tanhf(c[j]);
        dh[j] = du[j] + dr[j];
        dc[j] = dn[j] + dh[j] * O[j] * (1.f - tc[j] * tc[j]);
      }
      if (kind == 3 || kind == 5) {
        float r[V];
#pragma unroll
        for (int j = 0; j < V; ++j) r[j] = dc[j] * F[j];
        if (kind == 3) stv<V>(a.out, a.out_dt, b * a.out_ld + h, r);
        else stv<V>(a.out2, a.out2_dt, b * a.out2_ld + h, r);
      }
      if (kind == 2 || kind == 5) {
        float cprev[V];
        ldv<V>(a.cp, b * a.cp.ld + h, cprev);
        for (int x = a.g0; x < a.g0 + a.ng; ++x) {
          float r[V];
#pragma unroll
          for (int j = 0; j < V; ++j) {
            if (x == 0) r[j] = dc[j] * G[j] * I[j] * (1.f - I[j]);
            else if (x == 1) r[j] = dc[j] * cprev[j] * F[j] * (1.f - F[j]);
            else if (x == 2) r[j] = dc[j] * I[j] * (1.f - G[j] * G[j]);
            else r[j] = dh[j] * tc[j] * O[j] * (1.f - O[j]);
          }
          stv<V>(a.out, a.out_dt, b * a.out_ld + (x - a.g0) * a.out_gs + h, r);
        }
      }
    }
  }
}

__host__ inline bool vec8_ok(const LstmArgs& a) {
  if (a.nh % 8) return false;
  auto ok = [](const void* p, int64_t ld, int64_t gs, int dt) {
    if (!p) return true;
    const int64_t align = dt == TOFU_BF16 ? 8 : 4;  // elements per 16 bytes
    return (reinterpret_cast<uintptr_t>(p) % 16) == 0 && ld % align == 0 && gs % align == 0;
  };
  const LOpnd* ops[7] = {&a.gx, &a.gh, &a.cp, &a.c, &a.du, &a.dr, &a.dn};
  for (auto o : ops)
    if (!ok(o->p, o->ld, o->gs, o->dt)) return false;
  return ok(a.out, a.out_ld, a.out_gs, a.out_dt) && ok(a.out2, a.out2_ld, 0, a.out2_dt);
}

}  // namespace tofu

static int lstm_launch(tofu::LstmArgs& a, void* stream);
extern "C" int tofu_lstm_cell_splitk(int kind, int64_t nb, int64_t nh, int g0, int ng, const void* const* ptrs,
                                     const int64_t* lds, const int64_t* gss, const int* dts, void* out, int64_t out_ld,
                                     int64_t out_gs, int out_dt, void* out2, int64_t out2_ld, int out2_dt,
                                     const float* ghws, int gh_splits, int64_t gh_plane, int64_t gh_wld,
                                     int64_t gh_wgs, void* stream);

// Internal entry (not in the public header): operands are (ptr, ld, gs, dtype) quadruples in the slot order
// gx, gh, cp, c, du, dr, dn; out2 is the second output of the fused kinds 4 / 5 (else NULL).
extern "C" int tofu_lstm_cell(int kind, int64_t nb, int64_t nh, int g0, int ng, const void* const* ptrs,
                              const int64_t* lds, const int64_t* gss, const int* dts, void* out, int64_t out_ld,
                              int64_t out_gs, int out_dt, void* out2, int64_t out2_ld, int out2_dt, void* stream) {
  return tofu_lstm_cell_splitk(kind, nb, nh, g0, ng, ptrs, lds, gss, dts, out, out_ld, out_gs, out_dt, out2, out2_ld,
                               out2_dt, nullptr, 0, 0, 0, 0, stream);
}

// ... with GH taken from a gate GEMM's split-K partial planes (ghws: [splits][nb][.] fp32, row pitch gh_wld, gate
// stride gh_wgs; kinds 0 / 4): the planes are summed in split order, rounded to GH's dtype, stored to the GH
// operand's slot (ptrs[1] / lds[1] / gss[1] / dts[1] then name GH's destination) and used as stored.
extern "C" int tofu_lstm_cell_splitk(int kind, int64_t nb, int64_t nh, int g0, int ng, const void* const* ptrs,
                                     const int64_t* lds, const int64_t* gss, const int* dts, void* out, int64_t out_ld,
                                     int64_t out_gs, int out_dt, void* out2, int64_t out2_ld, int out2_dt,
                                     const float* ghws, int gh_splits, int64_t gh_plane, int64_t gh_wld,
                                     int64_t gh_wgs, void* stream) {
  tofu::LstmArgs a{};
  a.kind = kind;
  a.nb = nb;
  a.nh = nh;
  a.g0 = g0;
  a.ng = ng;
  tofu::LOpnd* ops[7] = {&a.gx, &a.gh, &a.cp, &a.c, &a.du, &a.dr, &a.dn};
  for (int i = 0; i < 7; ++i) *ops[i] = tofu::LOpnd{ptrs[i], lds[i], gss[i], dts[i]};
  a.out = out;
  a.out_ld = out_ld;
  a.out_gs = out_gs;
  a.out_dt = out_dt;
  a.out2 = out2;
  a.out2_ld = out2_ld;
  a.out2_dt = out2_dt;
  if (ghws) {
    if ((kind != 0 && kind != 4) || gh_splits < 1 || gh_splits > 16) return TOFU_ERR_ARG;
    a.ghws = ghws;
    a.gh_splits = gh_splits;
    a.gh_plane = gh_plane;
    a.gh_wld = gh_wld;
    a.gh_wgs = gh_wgs;
    a.gh_out = const_cast<void*>(ptrs[1]);
    a.gh_out_ld = lds[1];
    a.gh_out_gs = gss[1];
    a.gh_out_dt = dts[1];
    a.gh = tofu::LOpnd{nullptr, 0, 0, dts[1]};
  }
  return lstm_launch(a, stream);
}

static int lstm_launch(tofu::LstmArgs& a, void* stream) {
  const int64_t nb = a.nb, nh = a.nh;
  // 4 elements per thread when the operands allow 16-byte vectors: twice the threads of 8 per thread (the
  // [128 x 4096] cells launched 65536 threads, 0.86 waves at 25% occupancy: latency-bound at 1.5 TB/s);
  // TOFU_LSTM_V=8 keeps 8 (A/B switch)
  static const int vpref = [] {
    const char* e = getenv("TOFU_LSTM_V");
    return e && e[0] == '8' ? 8 : 4;
  }();
  bool v8 = tofu::vec8_ok(a);
  if (a.ghws) {  // the planes and GH's destination must take the same vectors
    const bool pl = (reinterpret_cast<uintptr_t>(a.ghws) % 16) == 0 && a.gh_plane % 4 == 0 && a.gh_wld % 4 == 0 &&
                    a.gh_wgs % 4 == 0;
    const int64_t al = a.gh_out_dt == TOFU_BF16 ? 8 : 4;
    const bool go = (reinterpret_cast<uintptr_t>(a.gh_out) % 16) == 0 && a.gh_out_ld % al == 0 && a.gh_out_gs % al == 0;
    v8 = v8 && pl && go;
  }
  // (the gate GEMM + cell fusion sums 4 gates x splits fp32 planes per element: more, narrower threads;
  // TOFU_LSTM_SPLIT_V overrides the vector width of that variant, A/B)
  static const int vsplit = [] {
    const char* e = getenv("TOFU_LSTM_SPLIT_V");
    return e ? atoi(e) : 1;  // (measured: 7.6 us vs 9.0 us with 4 per thread)
  }();
  const int vw = !v8 ? 1 : a.ghws ? (vsplit == 1 || vsplit == 4 || vsplit == 8 ? vsplit : 4) : vpref;
  const int64_t n = nb * (nh / vw);
  if (n == 0) return TOFU_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.ghws) {  // gate GEMM + cell fusion: the split-K planes are summed here
    if (vw == 8) tofu::launch_k(tofu::lstm_kernel<8, true>, dim3((unsigned)blocks), dim3(256), 0, st, 1, a);
    else if (vw == 4) tofu::launch_k(tofu::lstm_kernel<4, true>, dim3((unsigned)blocks), dim3(256), 0, st, 1, a);
    else tofu::launch_k(tofu::lstm_kernel<1, true>, dim3((unsigned)blocks), dim3(256), 0, st, 1, a);
  } else if (vw == 8) tofu::launch_k(tofu::lstm_kernel<8>, dim3((unsigned)blocks), dim3(256), 0, st, 1, a);
  else if (vw == 4) tofu::launch_k(tofu::lstm_kernel<4>, dim3((unsigned)blocks), dim3(256), 0, st, 1, a);
  else tofu::launch_k(tofu::lstm_kernel<1>, dim3((unsigned)blocks), dim3(256), 0, st, 1, a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && getenv("TOFU_DEBUG")) fprintf(stderr, "lstm cell launch: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}
