// Experiment (not product code): the fused add / mask GEMM epilogue's memory pattern without the GEMM.
// 148 persistent CTAs x 8 warps walk 128 x 256 output tiles in the GEMM's raster; warp (q, h) moves its
// 32-row quarter / column half in chunks of 32 rows x CW columns: TMA-load the add and mask chunks (NBUF-deep
// ring per warp), out = mask > 0 ? add : 0 in place, TMA-store.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC \
//        -I paper_1807_08887_b200/csrc tools/epi_pattern.cu -o variants/epi_pattern.so -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "cuda/common.cuh"

using namespace tofu;

template <int CW, int NBUF>
__global__ void __launch_bounds__(256, 1) epi_kernel(const __grid_constant__ CUtensorMap tA,
                                                     const __grid_constant__ CUtensorMap tM,
                                                     const __grid_constant__ CUtensorMap tO, int M, int N) {
  constexpr int CB = 32 * CW * 2;  // bytes of one operand chunk
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * NBUF * 2 * CB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 8 * NBUF * 2 * CB) + warp * NBUF;
  if (lane == 0)
    for (int i = 0; i < NBUF; ++i) mbar_init(&bars[i], 1);
  fence_mbar_init();
  __syncwarp();
  const int q = warp & 3, h = warp >> 2;
  const int tiles_n = N / 256, ntiles = (M / 128) * tiles_n;
  constexpr int NCW = 128 / CW;  // chunks per warp per tile
  const int my = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int S = my * NCW;
  auto coords = [&](int s, int& col, int& row) {
    const int tile = blockIdx.x + (s / NCW) * gridDim.x;
    col = (tile % tiles_n) * 256 + h * 128 + (s % NCW) * CW;
    row = (tile / tiles_n) * 128 + q * 32;
  };
  auto issue = [&](int s) {
    int col, row;
    coords(s, col, row);
    uint8_t* b = wbuf + (s % NBUF) * 2 * CB;
    mbar_arrive_expect_tx(&bars[s % NBUF], 2 * CB);
    for (int c = 0; c < CW / 32; ++c) {
      tma_load_2d(b + c * 2048, &tA, &bars[s % NBUF], col + 32 * c, row);
      tma_load_2d(b + CB + c * 2048, &tM, &bars[s % NBUF], col + 32 * c, row);
    }
  };
  if (lane == 0)
    for (int s = 0; s < NBUF - 1 && s < S; ++s) issue(s);
  for (int s = 0; s < S; ++s) {
    if (lane == 0 && s + NBUF - 1 < S) {
      bulk_wait_read<0>();
      issue(s + NBUF - 1);
    }
    __syncwarp();
    mbar_wait(&bars[s % NBUF], (s / NBUF) & 1);
    uint8_t* b = wbuf + (s % NBUF) * 2 * CB;
    for (int c = 0; c < CW / 32; ++c) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int off = c * 2048 + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
        uint4 a = *reinterpret_cast<const uint4*>(b + off);
        const uint4 m = *reinterpret_cast<const uint4*>(b + CB + off);
        __nv_bfloat162* ah = reinterpret_cast<__nv_bfloat162*>(&a);
        const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&m);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 fa = __bfloat1622float2(ah[e]), fm = __bfloat1622float2(mh[e]);
          ah[e] = __floats2bfloat162_rn(fm.x > 0.f ? fa.x : 0.f, fm.y > 0.f ? fa.y : 0.f);
        }
        *reinterpret_cast<uint4*>(b + off) = a;
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      int col, row;
      coords(s, col, row);
      for (int c = 0; c < CW / 32; ++c) tma_store_2d(&tO, b + c * 2048, col + 32 * c, row);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait<0>();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return f;
}

static void mk(CUtensorMap* t, void* p, int M, int N) {
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
  cuuint64_t str[1] = {(cuuint64_t)N * 2};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  enc()(t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

template <int CW, int NBUF>
static int go(const CUtensorMap* t, int M, int N, cudaStream_t st) {
  constexpr int SM = 8 * NBUF * 2 * 32 * CW * 2 + 1024 + 8 * NBUF * 8;
  auto k = epi_kernel<CW, NBUF>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
  k<<<148, 256, SM, st>>>(t[0], t[1], t[2], M, N);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int epi_run(void* add, void* mask, void* out, int M, int N, int cw, int nbuf, void* stream) {
  CUtensorMap t[3];
  mk(&t[0], add, M, N);
  mk(&t[1], mask, M, N);
  mk(&t[2], out, M, N);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int key = cw * 10 + nbuf;
  switch (key) {
    case 322: return go<32, 2>(t, M, N, st);
    case 323: return go<32, 3>(t, M, N, st);
    case 324: return go<32, 4>(t, M, N, st);
    case 326: return go<32, 6>(t, M, N, st);
    case 642: return go<64, 2>(t, M, N, st);
    case 643: return go<64, 3>(t, M, N, st);
    default: return -2;
  }
}
