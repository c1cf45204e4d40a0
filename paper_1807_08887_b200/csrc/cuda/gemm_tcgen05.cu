// Sub-operator GEMM on sm_100a: TMA -> smem (SWIZZLE_128B) -> tcgen05.mma (bf16 x bf16 -> fp32 in TMEM)
// -> tcgen05.ld epilogue.  This is the dense-contraction sub-op every worker runs on its tile under
// partition-n-reduce (§3.1: "executing the same operator on each worker using smaller inputs").
//
// C[m, n] (+)= sum_k A[m, k] * B[k, n]
//   A K-major : A[m*lda + k]      A MN-major : A[k*lda + m]
//   B K-major : B[n*ldb + k]      B MN-major : B[k*ldb + n]
// The three TDL matmul defs map to (A,B) majorness: mm_nn (K, MN), mm_nt (K, K), mm_tn (MN, MN).
//
// Epilogues: 0 = bf16 store, 1 = fp32 store (partial outputs of Case-2 strategies, weight grads),
//            2 = fp32 accumulate (C += acc).
//
// Warp roles (192 threads): warp 0 = TMA producer (1 elected lane), warp 1 = TMEM allocator + MMA issuer
// (1 lane), warps 2..5 = epilogue (warp w reads TMEM lanes 32*(w%4)..+31).  Persistent: each CTA walks
// output tiles (grid = min(#tiles, #SMs)); the accumulator is double-buffered in TMEM so the epilogue of
// tile t overlaps the mainloop of tile t+1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NTHREADS = 192;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int ACC_BUFS = 2;
  static constexpr int TMEM_COLS = BN * ACC_BUFS;  // 256 or 512 fp32 columns
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, bool A_MN, bool B_MN, int OUT>
__global__ void __launch_bounds__(NTHREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, void* Cp,
                     int M, int N, int K, int ldc) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;          // [ACC_BUFS]
  uint64_t* acc_empty = acc_full + Cfg::ACC_BUFS;  // [ACC_BUFS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + Cfg::ACC_BUFS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM;
  const int tiles_n = (N + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < Cfg::ACC_BUFS; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (tile / tiles_n) * BM;
        const int n0 = (tile % tiles_n) * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
          uint8_t* a = sA + s * Cfg::A_BYTES;
          uint8_t* b = sB + s * Cfg::B_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d(a, &tmA, &full[s], k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) tma_load_2d(a + c * 8192, &tmA, &full[s], m0 + 64 * c, k0);
          }
          if (!B_MN) {
            tma_load_2d(b, &tmB, &full[s], k0, n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(b + c * 8192, &tmB, &full[s], n0 + 64 * c, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int it = 0, local = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++local) {
        const int buf = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&acc_empty[buf], aph ^ 1);  // epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + buf * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * Cfg::A_BYTES);
          const uint32_t b0 = smem_u32(sB + s * Cfg::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? umma_sdesc_sw128(a0 + kk * 2048, 8192, 1024)
                                     : umma_sdesc_sw128(a0 + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_sdesc_sw128(b0 + kk * 2048, 8192, 1024)
                                     : umma_sdesc_sw128(b0 + kk * 32, 16, 1024);
            umma_bf16(tmem_d, ad, bd, idesc, (kb | kk) ? 1u : 0u);
          }
          umma_commit(&empty[s]);  // frees the smem stage when these MMAs complete
        }
        umma_commit(&acc_full[buf]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int lane_base = 32 * (warp & 3);
    int local = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++local) {
      const int m0 = (tile / tiles_n) * BM;
      const int n0 = (tile % tiles_n) * BN;
      const int buf = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&acc_full[buf], aph);
      tc_fence_after();
      const int row = m0 + lane_base + lane;
      const bool row_ok = row < M && nk > 0;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + buf * BN + ((uint32_t)lane_base << 16) + c, r);
        tmem_ld_wait();
        const int col = n0 + c;
        if (!row_ok || col >= N) continue;
        const bool full_chunk = (col + 32 <= N);
        if (OUT == 0) {
          __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(Cp) + (size_t)row * ldc + col;
          if (full_chunk && ((reinterpret_cast<uintptr_t>(C) & 15) == 0)) {
            uint32_t p[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
              p[j] = *reinterpret_cast<uint32_t*>(&h);
            }
            uint4* dst = reinterpret_cast<uint4*>(C);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_uint4(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
          } else {
            for (int j = 0; j < 32 && col + j < N; ++j) C[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
          }
        } else {
          float* C = reinterpret_cast<float*>(Cp) + (size_t)row * ldc + col;
          if (full_chunk && ((reinterpret_cast<uintptr_t>(C) & 15) == 0)) {
            float4* dst = reinterpret_cast<float4*>(C);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                     __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
              if (OUT == 2) {
                const float4 o = dst[j];
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              dst[j] = v;
            }
          } else {
            for (int j = 0; j < 32 && col + j < N; ++j) {
              const float v = __uint_as_float(r[j]);
              C[j] = (OUT == 2) ? C[j] + v : v;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;
static int g_num_sms = 0;

static int encode_fn_init() {
  std::call_once(g_encode_once, []() {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  });
  return g_encode ? 0 : -1;
}

// 2-D bf16 tensor map: inner extent `inner` (contiguous), outer extent `outer`, row pitch `ld` elements.
static int make_tmap(CUtensorMap* tm, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                     uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -(int)r - 1000;
}

template <int BN, bool A_MN, bool B_MN, int OUT>
static int launch_t(const tofu_gemm_args* g, const CUtensorMap& ta, const CUtensorMap& tb, cudaStream_t st) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, OUT>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
      return TOFU_ERR_CUDA;
    attr_set = true;
  }
  const int tiles = ((g->M + BM - 1) / BM) * ((g->N + BN - 1) / BN);
  int grid = tiles < g_num_sms ? tiles : g_num_sms;
  if (g->max_ctas > 0 && grid > g->max_ctas) grid = g->max_ctas;
  kern<<<grid, NTHREADS, Cfg::SMEM, st>>>(ta, tb, g->C, g->M, g->N, g->K, g->ldc);
  return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
}

template <int BN>
static int dispatch_bn(const tofu_gemm_args* g, const CUtensorMap& ta, const CUtensorMap& tb, cudaStream_t st) {
  const int key = (g->a_mn_major ? 1 : 0) | (g->b_mn_major ? 2 : 0) | (g->c_mode << 2);
  switch (key) {
#define TOFU_CASE(AM, BMJ, O) \
  case ((AM) | ((BMJ) << 1) | ((O) << 2)): return launch_t<BN, (bool)(AM), (bool)(BMJ), O>(g, ta, tb, st);
    TOFU_CASE(0, 0, 0) TOFU_CASE(0, 0, 1) TOFU_CASE(0, 0, 2)
    TOFU_CASE(0, 1, 0) TOFU_CASE(0, 1, 1) TOFU_CASE(0, 1, 2)
    TOFU_CASE(1, 0, 0) TOFU_CASE(1, 0, 1) TOFU_CASE(1, 0, 2)
    TOFU_CASE(1, 1, 0) TOFU_CASE(1, 1, 1) TOFU_CASE(1, 1, 2)
#undef TOFU_CASE
    default: return TOFU_ERR_ARG;
  }
}

}  // namespace tofu

using namespace tofu;

extern "C" int tofu_gemm_plan_tmaps(const tofu_gemm_args* g, void* tmap_a, void* tmap_b, int* bn_out) {
  if (encode_fn_init() != 0) return TOFU_ERR_CUDA;
  if (!g || g->M < 0 || g->N < 0 || g->K < 0 || g->c_mode < 0 || g->c_mode > 2) return TOFU_ERR_ARG;
  // TMA: row pitch must be a multiple of 16 bytes, base 16-byte aligned
  if ((g->lda % 8) || (g->ldb % 8) || (reinterpret_cast<uintptr_t>(g->A) & 15) ||
      (reinterpret_cast<uintptr_t>(g->B) & 15))
    return TOFU_ERR_ALIGN;
  const int bn = (g->bn == 128 || g->bn == 256) ? g->bn : ((g->N <= 128 || (long)g->M * g->N <= 148L * 128 * 256) ? 128 : 256);
  CUtensorMap* ta = reinterpret_cast<CUtensorMap*>(tmap_a);
  CUtensorMap* tb = reinterpret_cast<CUtensorMap*>(tmap_b);
  int r;
  if (!g->a_mn_major) r = make_tmap(ta, g->A, g->K, g->M, g->lda, 64, BM);
  else r = make_tmap(ta, g->A, g->M, g->K, g->lda, 64, 64);
  if (r) return TOFU_ERR_CUDA;
  if (!g->b_mn_major) r = make_tmap(tb, g->B, g->K, g->N, g->ldb, 64, bn);
  else r = make_tmap(tb, g->B, g->N, g->K, g->ldb, 64, 64);
  if (r) return TOFU_ERR_CUDA;
  *bn_out = bn;
  return TOFU_OK;
}

extern "C" int tofu_gemm_launch_planned(const tofu_gemm_args* g, const void* tmap_a, const void* tmap_b, int bn,
                                        void* stream) {
  if (g->M == 0 || g->N == 0) return TOFU_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (g->K == 0) {
    if (g->c_mode == 2) return TOFU_OK;
    const size_t es = g->c_mode == 0 ? 2 : 4;
    return cudaMemset2DAsync(g->C, (size_t)g->ldc * es, 0, (size_t)g->N * es, g->M, st) == cudaSuccess
               ? TOFU_OK
               : TOFU_ERR_CUDA;
  }
  const CUtensorMap& ta = *reinterpret_cast<const CUtensorMap*>(tmap_a);
  const CUtensorMap& tb = *reinterpret_cast<const CUtensorMap*>(tmap_b);
  return bn == 256 ? dispatch_bn<256>(g, ta, tb, st) : dispatch_bn<128>(g, ta, tb, st);
}

extern "C" int tofu_gemm_bf16(const tofu_gemm_args* g, void* stream) {
  alignas(64) CUtensorMap ta, tb;
  int bn = 0;
  int r = tofu_gemm_plan_tmaps(g, &ta, &tb, &bn);
  if (r) return r;
  return tofu_gemm_launch_planned(g, &ta, &tb, bn, stream);
}
