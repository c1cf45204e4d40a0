// LSTM cell sub-operators (configs[2]; LSTM cell of the paper's RNN benchmark).
//
// Gate pre-activations a_x = GX[b, x, h] + GH[b, x, h], x in {i=0, f=1, g=2, o=3}:
//   cell_c     : c_t  = sigmoid(a_f) * c_{t-1} + sigmoid(a_i) * tanh(a_g)
//   cell_h     : h_t  = sigmoid(a_o) * tanh(c_t)
//   cell_bwd_a : dA[b, x, h] = d loss / d a_x  (x in the op's gate range)
//   cell_bwd_c : d loss / d c_{t-1}
// with dh = DU + DR (from the layer above and from step t+1) and dc = DN + dh * o * (1 - tanh(c_t)^2).
// The formulas are the TDL defs of tofu_inputs/graphs.py (oracle-checked against finite differences).
// Operands are pitched views of the (b, [gate,] h) box: element (b, x, h) at p[b*ld + x*gs + h].
// Each thread handles one (b, h) and reads the four gates it needs; threads of a warp walk h (coalesced).
#include <cuda_bf16.h>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {

struct LOpnd {
  const void* p;
  int64_t ld, gs;
  int dt;
};

__device__ __forceinline__ float ldv(const LOpnd& o, int64_t i) {
  return o.dt == TOFU_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(o.p)[i])
                           : reinterpret_cast<const float*>(o.p)[i];
}
__device__ __forceinline__ void stv(void* p, int dt, int64_t i, float v) {
  if (dt == TOFU_BF16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else reinterpret_cast<float*>(p)[i] = v;
}
__device__ __forceinline__ float sig(float x) { return 1.f / (1.f + __expf(-x)); }

struct LstmArgs {
  int kind;  // 0 c, 1 h, 2 bwd_a, 3 bwd_c
  int64_t nb, nh;
  int g0, ng;  // gate range of the output (bwd_a)
  LOpnd gx, gh, cp, c, du, dr, dn;
  void* out;
  int64_t out_ld, out_gs;
  int out_dt;
};

__global__ void __launch_bounds__(256) lstm_kernel(const LstmArgs a) {
  const int64_t n = a.nb * a.nh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / a.nh, h = e % a.nh;
    const int64_t go = b * a.gx.ld + h, ho = b * a.gh.ld + h;
    const float ai = ldv(a.gx, go) + ldv(a.gh, ho);
    const float af = ldv(a.gx, go + a.gx.gs) + ldv(a.gh, ho + a.gh.gs);
    const float ag = ldv(a.gx, go + 2 * a.gx.gs) + ldv(a.gh, ho + 2 * a.gh.gs);
    const float ao = ldv(a.gx, go + 3 * a.gx.gs) + ldv(a.gh, ho + 3 * a.gh.gs);
    const float I = sig(ai), F = sig(af), G = tanhf(ag), O = sig(ao);
    if (a.kind == 0) {
      stv(a.out, a.out_dt, b * a.out_ld + h, F * ldv(a.cp, b * a.cp.ld + h) + I * G);
    } else if (a.kind == 1) {
      stv(a.out, a.out_dt, b * a.out_ld + h, O * tanhf(ldv(a.c, b * a.c.ld + h)));
    } else {
      const float tc = tanhf(ldv(a.c, b * a.c.ld + h));
      const float dh = ldv(a.du, b * a.du.ld + h) + ldv(a.dr, b * a.dr.ld + h);
      const float dc = ldv(a.dn, b * a.dn.ld + h) + dh * O * (1.f - tc * tc);
      if (a.kind == 3) {
        stv(a.out, a.out_dt, b * a.out_ld + h, dc * F);
      } else {
        const float cprev = ldv(a.cp, b * a.cp.ld + h);
        for (int x = a.g0; x < a.g0 + a.ng; ++x) {
          float v;
          if (x == 0) v = dc * G * I * (1.f - I);
          else if (x == 1) v = dc * cprev * F * (1.f - F);
          else if (x == 2) v = dc * I * (1.f - G * G);
          else v = dh * tc * O * (1.f - O);
          stv(a.out, a.out_dt, b * a.out_ld + (x - a.g0) * a.out_gs + h, v);
        }
      }
    }
  }
}

}  // namespace tofu

// Internal entry (not in the public header): operands are (ptr, ld, gs, dtype) quadruples.
extern "C" int tofu_lstm_cell(int kind, int64_t nb, int64_t nh, int g0, int ng, const void* const* ptrs,
                              const int64_t* lds, const int64_t* gss, const int* dts, void* out, int64_t out_ld,
                              int64_t out_gs, int out_dt, void* stream) {
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
  const int64_t n = nb * nh;
  if (n == 0) return TOFU_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  tofu::lstm_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}
