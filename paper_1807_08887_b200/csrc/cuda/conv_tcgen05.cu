// Implicit-GEMM convolution sub-op on sm_100a (WResNet, configs[3]): the convolution TDL defs (forward,
// data gradient, weight gradient; tofu_inputs.graphs.conv_defs, DESIGN reading R11) executed on the
// worker's tile as one tcgen05 GEMM whose activation operand is GATHERED pixel by pixel (cp.async, zero-fill
// outside the buffer = zero padding) straight into the 128B-swizzled shared-memory layout the UMMA
// descriptors expect, while the dense operand (weights, or the output gradient for the weight gradient)
// arrives by TMA.  This is the same partition-n-reduce sub-op the paper runs with cuDNN; the
// im2col matrix is never materialised.
//
//   kind 0 (forward / data gradient): rows = output pixels, K = taps x channels, A gathered (K-major),
//          B = weights via TMA (K-major for the forward, MN-major for the data gradient), output rows
//          stored directly (a row = one pixel's channels; strided pixel grids serve the stride-2 data
//          gradient's sub-pixel phases).
//   kind 1 (weight gradient): M = output channels, N = taps x input channels, K = pixels; A = output
//          gradient via TMA (MN-major), B gathered (MN-major rows of 64 channels); fp32 output through the
//          TMA-store epilogue of the GEMM (store / accumulate / fused momentum-SGD), split-K over pixels.
//
// Warp roles (320 threads): warp 0 lane 0 = TMA producer of the dense operand, warp 1 = TMEM allocator +
// MMA issuer, warps 2..5 = epilogue (TMEM lane quarter w%4), warps 6..9 = gather producers (128 threads;
// each thread's copies of a stage arrive on the stage's mbarrier when they land (cp.async.mbarrier.arrive),
// so a producer runs up to STAGES ahead without blocking; the MMA thread fences generic -> async proxy
// after the wait).  Persistent grid, TMEM accumulator double-buffered as in gemm_tcgen05.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {
namespace conv {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NTHREADS = 320;
constexpr int SMEM_MAX = 232448;
constexpr int NGATHER = 128;  // warps 6..9

struct Params {
  tofu_conv_args a;
  int M, N, K, splits;
  int sk_tiles;  // stream-K tiles (common.cuh WorkList); 0 = data-parallel only
  int dy0, dx0;  // im2col: smallest tap offsets (the map's im2col offsets are tap - min >= 0)
};

struct RowInfo {
  long long off;  // element offset in S of the pixel's (b, y, x) before the tap offset (y, x may be outside)
  int y, x;       // buffer coordinates before the tap offset
};

template <int KIND, int BN, int MODE, bool C2 = false>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (C2 ? BN / 2 : BN) * BK * 2;  // C2: this CTA's half of the B tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr bool LOADS = MODE == 2 || MODE == 3;
  static constexpr int NBUF = KIND == 1 ? 2 : 0;
  static constexpr int D_OFF = 4096;
  static constexpr int BUF_BYTES = MODE == 3 ? 6144 : 4096;
  static constexpr int EPI_BYTES = 4 * NBUF * BUF_BYTES;
  static constexpr int ROWS = KIND == 0 ? BM : BK;
  static constexpr int ROW_BYTES = 2 * ROWS * (int)sizeof(RowInfo);
  static constexpr int FIT = (SMEM_MAX - 1024 - 512 - EPI_BYTES - ROW_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = FIT > 6 ? 6 : FIT;
  static constexpr int TMEM_COLS = BN * 2;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + ROW_BYTES + 1024 + 512;
  static_assert(STAGES >= 3, "pipeline too shallow");
  static_assert(SMEM <= SMEM_MAX, "smem");
};

__device__ __forceinline__ RowInfo pixel_info(const tofu_conv_args& a, int g, int ngyx) {
  RowInfo ri;
  const int gb = g / ngyx, rem = g - gb * ngyx;
  const int gy = rem / a.ngx, gx = rem - gy * a.ngx;
  ri.y = a.ay * gy + a.cy;
  ri.x = a.ax * gx + a.cx;
  ri.off = (long long)(gb + a.sb0) * a.s_sb + (long long)ri.y * a.s_sy + (long long)ri.x * a.s_sx;
  return ri;
}
__device__ __forceinline__ RowInfo lds_rowinfo(const RowInfo* p) {  // explicit shared-space load
  uint32_t w0, w1, w2, w3;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(smem_u32(p)));
  RowInfo r;
  r.off = (long long)(((uint64_t)w1 << 32) | w0);
  r.y = (int)w2;
  r.x = (int)w3;
  return r;
}
__device__ __forceinline__ RowInfo no_pixel() {
  RowInfo ri;
  ri.off = 0;
  ri.y = ri.x = -(1 << 29);
  return ri;
}

// I2C (kind 0): the activation operand is loaded by TMA in im2col mode (tmI) instead of the gather warps:
// one 128-pixel x 64-channel box per k-block, zero outside the tensor (= padding), straight into the
// 128B-swizzled layout of the gathered tile.  Used for stride-1 grids whose channel blocks are whole taps.
// CL2 (weight gradient with im2col): clusters of 2 CTAs on vertically adjacent tiles (output-channel tiles
// 2p, 2p+1) of the same n tile share the gathered activations: each CTA im2col-loads half of the B sub-blocks
// and multicasts them to both; a stage is freed by both CTAs' MMA commits (as gemm_tcgen05.cu's CL2).
// C2 (with im2col): 2-CTA MMA pairs (tcgen05.mma.cta_group::2, M = 256 over a cluster of 2) on vertically
// adjacent tiles: each CTA stages its own A rows and half of the B tile, loads complete on the leader's
// barriers, the leader issues the MMAs, both CTAs' epilogues read their TMEM halves (gemm_tcgen05.cu's C2).
template <int KIND, int BN, bool B_MN, int MODE, bool I2C = false, bool CL2 = false, bool C2 = false>
__global__ void __launch_bounds__(NTHREADS, 1)
    conv_kernel(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap tmDense,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmD,
                const __grid_constant__ CUtensorMap tmI) {
  using C_ = Cfg<KIND, BN, MODE, C2>;
  constexpr int STAGES = C_::STAGES;
  constexpr int NBUF = C_::NBUF;
  const tofu_conv_args& a = P.a;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by an offset from the __shared__ array (an integer round trip through uintptr_t would lose
  // the address space: every epilogue smem access became a generic LD.E / ST.E)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C_::A_BYTES;
  uint8_t* sE = smem + STAGES * C_::STAGE_BYTES;
  RowInfo* rows = reinterpret_cast<RowInfo*>(sE + C_::EPI_BYTES);  // [2][ROWS]
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(rows) + C_::ROW_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* ebar = acc_empty + 2;  // [4][NBUF]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + 4 * (NBUF > 0 ? NBUF : 1));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = P.M, N = P.N, K = P.K, splits = P.splits;
  const int tiles_m = (M + BM - 1) / BM;
  const int tiles_n = (N + BN - 1) / BN;
  const int nk = (K + BK - 1) / BK;
  WorkList wl;
  uint32_t crank = 0;
  if constexpr (CL2 || C2) {
    crank = cluster_rank();
    wl.init_pairs(tiles_m, tiles_n, nk, (int)crank, (int)cluster_id_x(), (int)nclusters_x());
  } else {
    wl.init(tiles_m * tiles_n, nk, splits, P.sk_tiles);
  }
  const int nseg = wl.count();
  void* const sk_ws = a.sk_ws;
  const int ngyx = a.ngy * a.ngx;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], I2C ? 1 : 1 + NGATHER);
      mbar_init(&empty[s], CL2 ? 2 : 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], C2 ? 8 : 4);  // C2: both CTAs' epilogue warps arrive on the leader's
    }
    for (int b = 0; b < 4 * NBUF; ++b) mbar_init(&ebar[b], 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmDense);
    if (KIND == 1) tma_prefetch_desc(&tmC);
    if (MODE == 3) tma_prefetch_desc(&tmD);
    if (I2C) tma_prefetch_desc(&tmI);
  }
  if (warp == 1) {
    if constexpr (C2) tmem_alloc2(tmem_slot, C_::TMEM_COLS);
    else tmem_alloc(tmem_slot, C_::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CL2 || C2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  tofu::pdl_trigger();
  tofu::pdl_wait();  // prologue done: now wait for the predecessor's results (PDL)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (dense operand)
    if (lane == 0) {
      int it = 0;
      for (int i = 0; i < nseg; ++i) {
        int tile, kb0, kb1, sp;
        bool part;
        wl.seg(i, tile, kb0, kb1, sp, part);
        const int m0 = (tile / tiles_n) * BM;
        const int n0 = (tile % tiles_n) * BN;
        int iw = 0, ih = 0, in_ = 0;  // im2col: traversal start of the tile's first pixel
        if constexpr (I2C) {
          const int gb = m0 / ngyx, rem = m0 - gb * ngyx;
          const int gy = rem / a.ngx, gx = rem - gy * a.ngx;
          ih = a.ay * gy + a.cy + P.dy0;
          iw = a.ax * gx + a.cx + P.dx0;
          in_ = gb + a.sb0;
        }
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          const int k0 = kb * BK;
          if constexpr (KIND == 0) {
            const uint32_t lf = C2 ? mapa_shared(&full[s], 0) : 0u;
            if constexpr (C2) {
              if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * (C_::A_BYTES + C_::B_BYTES));
            } else {
              mbar_arrive_expect_tx(&full[s], C_::B_BYTES + (I2C ? C_::A_BYTES : 0));
            }
            if constexpr (I2C) {
              const int t = k0 / a.nch, c = k0 - t * a.nch;
              if constexpr (C2)
                tma_load_im2col_4d_2sm(sA + s * C_::A_BYTES, &tmI, lf, a.sc0 + c, iw, ih, in_,
                                       (uint16_t)(a.tap_dx[t] - P.dx0), (uint16_t)(a.tap_dy[t] - P.dy0));
              else
                tma_load_im2col_4d(sA + s * C_::A_BYTES, &tmI, &full[s], a.sc0 + c, iw, ih, in_,
                                   (uint16_t)(a.tap_dx[t] - P.dx0), (uint16_t)(a.tap_dy[t] - P.dy0));
            }
            uint8_t* b = sB + s * C_::B_BYTES;
            if (!B_MN) {  // W[n][taps][c]: columns tap_w[t]*b_tap + c
              const int col = (a.nch % BK == 0) ? a.tap_w[k0 / a.nch] * a.b_tap + k0 % a.nch : k0;
              if constexpr (C2) tma_load_2d_2sm(b, &tmDense, lf, col, n0 + (int)crank * (BN / 2));
              else tma_load_2d(b, &tmDense, &full[s], col, n0);
            } else {      // W[c][taps][n]: rows = the K channels of one tap, columns tap_w[t]*b_tap + n
              // nch >= 64: one tap per k-block; nch in {8,16,32}: 64/nch taps, one box of nch rows each
              const int bk = a.nch < BK ? a.nch : BK;
              for (int h = 0; h < BK / bk; ++h) {
                const int k = k0 + h * bk;
                int t = k / a.nch;
                if (t >= a.ntaps) t = a.ntaps - 1;  // K tail: the gathered rows there are zero
                const int c = k % a.nch;
#pragma unroll
                for (int q = 0; q < BN / 64; ++q)
                  tma_load_2d(b + q * 8192 + h * bk * 128, &tmDense, &full[s], a.tap_w[t] * a.b_tap + n0 + 64 * q, c);
              }
            }
          } else {
            const uint32_t lf = C2 ? mapa_shared(&full[s], 0) : 0u;
            if constexpr (C2) {
              if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * (C_::A_BYTES + C_::B_BYTES));
            } else {
              mbar_arrive_expect_tx(&full[s], C_::A_BYTES + (I2C ? C_::B_BYTES : 0));
            }
            uint8_t* aa = sA + s * C_::A_BYTES;
#pragma unroll
            for (int q = 0; q < BM / 64; ++q) {
              if constexpr (C2) tma_load_2d_2sm(aa + q * 8192, &tmDense, lf, m0 + 64 * q, k0);
              else tma_load_2d(aa + q * 8192, &tmDense, &full[s], m0 + 64 * q, k0);
            }
            if constexpr (I2C) {  // B rows = the k-block's 64 pixels, BN columns = channels of the tile's tap
              const int gb = k0 / ngyx, rem = k0 - gb * ngyx;
              const int gy = rem / a.ngx, gx = rem - gy * a.ngx;
              const int t = n0 / a.nch, c = n0 - t * a.nch;
              const uint16_t ow = (uint16_t)(a.tap_dx[t] - P.dx0), oh = (uint16_t)(a.tap_dy[t] - P.dy0);
#pragma unroll
              for (int q = 0; q < BN / 64; ++q) {
                if constexpr (C2) {  // this CTA's half of the sub-blocks, into its own (half-size) stage
                  if (q >= BN / 128) continue;
                  const int cc = (int)crank * (BN / 128) + q;
                  tma_load_im2col_4d_2sm(sB + s * C_::B_BYTES + q * 8192, &tmI, lf, a.sc0 + c + 64 * cc,
                                         a.ax * gx + a.cx + P.dx0, a.ay * gy + a.cy + P.dy0, gb + a.sb0, ow, oh);
                } else if constexpr (CL2) {  // this CTA's half of the sub-blocks, multicast to the pair
                  if ((q >= BN / 128) != (crank != 0)) continue;
                  tma_load_im2col_4d_mc(sB + s * C_::B_BYTES + q * 8192, &tmI, &full[s], a.sc0 + c + 64 * q,
                                        a.ax * gx + a.cx + P.dx0, a.ay * gy + a.cy + P.dy0, gb + a.sb0, ow, oh, 0x3);
                } else {
                  tma_load_im2col_4d(sB + s * C_::B_BYTES + q * 8192, &tmI, &full[s], a.sc0 + c + 64 * q,
                                     a.ax * gx + a.cx + P.dx0, a.ay * gy + a.cy + P.dy0, gb + a.sb0, ow, oh);
                }
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (C2: the pair leader only)
    if (lane == 0 && (!C2 || crank == 0)) {
      constexpr bool A_MN = KIND == 1;
      constexpr bool BMN = KIND == 1 ? true : B_MN;
      constexpr uint32_t idesc = umma_idesc_bf16(C2 ? 2 * BM : BM, BN, A_MN ? 1 : 0, BMN ? 1 : 0);
      int it = 0;
      for (int local = 0; local < nseg; ++local) {
        int tile, kb0, kb1, sp;
        bool part;
        wl.seg(local, tile, kb0, kb1, sp, part);
        const int buf = local & 1;
        mbar_wait(&acc_empty[buf], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          fence_proxy_async_smem();  // the gathered operand was written by cp.async (generic proxy)
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * C_::A_BYTES);
          const uint32_t b0 = smem_u32(sB + s * C_::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? umma_sdesc_sw128(a0 + kk * 2048, 8192, 1024)
                                     : umma_sdesc_sw128(a0 + kk * 32, 16, 1024);
            const uint64_t bd = BMN ? umma_sdesc_sw128(b0 + kk * 2048, 8192, 1024)
                                    : umma_sdesc_sw128(b0 + kk * 32, 16, 1024);
            if constexpr (C2) umma_bf16_2(tmem_d, ad, bd, idesc, (kb > kb0 || kk) ? 1u : 0u);
            else umma_bf16(tmem_d, ad, bd, idesc, (kb > kb0 || kk) ? 1u : 0u);
          }
          if constexpr (C2) umma_commit2_mc(&empty[s], 0x3);
          else if constexpr (CL2) umma_commit_mc(&empty[s], 0x3);
          else umma_commit(&empty[s]);
        }
        if constexpr (C2) umma_commit2_mc(&acc_full[buf], 0x3);
        else umma_commit(&acc_full[buf]);
      }
    }
  } else if (warp >= 6 && !I2C) {
    // ------------------------------------------------------------ gather producers (warps 6..9)
    // Per stage a thread issues a fixed set of 16-byte copies whose shared-memory slots are compile-time
    // offsets (the 128B swizzle phase of its rows is constant); per copy: one row-info load, two bounds
    // tests, one 64-bit add.
    const int gt = threadIdx.x - 192;
    int it = 0;
    const __nv_bfloat16* S0 = reinterpret_cast<const __nv_bfloat16*>(a.S);
    for (int i = 0; i < nseg; ++i) {
      int tile, kb0, kb1, sp;
      bool part;
      wl.seg(i, tile, kb0, kb1, sp, part);
      const int m0 = (tile / tiles_n) * BM;
      const int n0 = (tile % tiles_n) * BN;
      if constexpr (KIND == 0) {
        // this thread's 8 rows (r0 + 16 i) of the tile, decoded once per tile into registers
        const int j = gt & 7, r0 = gt >> 3;
        const int slot = r0 * 128 + ((j ^ (r0 & 7)) << 4);
        RowInfo q[BM / 16];
#pragma unroll
        for (int i = 0; i < BM / 16; ++i) {
          const int m = m0 + r0 + 16 * i;
          q[i] = m < M ? pixel_info(a, m, ngyx) : no_pixel();
        }
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          const int k = kb * BK + j * 8;
          const int t = k / a.nch, c = k - t * a.nch;
          const bool tv = t < a.ntaps;
          const int dy = tv ? a.tap_dy[t] : -(1 << 29), dx = tv ? a.tap_dx[t] : 0;
          const __nv_bfloat16* S = S0 + a.sc0 + c + ((long long)dy * a.s_sy + (long long)dx * a.s_sx);
          uint8_t* dst = sA + s * C_::A_BYTES + slot;
#pragma unroll
          for (int i = 0; i < BM / 16; ++i) {
            const bool ok = (unsigned)(q[i].y + dy) < (unsigned)a.sH && (unsigned)(q[i].x + dx) < (unsigned)a.sW;
            cp_async_16(dst + i * 2048, ok ? S + q[i].off : S0, ok ? 16u : 0u);
          }
          cp_async_mbar_arrive(&full[s]);  // lands asynchronously; the MMA thread fences the proxies
        }
      } else {
        constexpr int CPR = BN / 8;           // 16-byte chunks per k row
        constexpr int RSTEP = NGATHER / CPR;  // rows covered per pass
        static_assert(BK % RSTEP == 0, "gather rows");
        const int jj = gt % CPR, r0 = gt / CPR;
        const int n = n0 + jj * 8;
        const int t = n / a.nch, c = n - t * a.nch;
        const bool tv = n < N && t < a.ntaps;
        const int dy = tv ? a.tap_dy[t] : -(1 << 29), dx = tv ? a.tap_dx[t] : 0;
        const __nv_bfloat16* S = S0 + a.sc0 + c + ((long long)dy * a.s_sy + (long long)dx * a.s_sx);
        const int sub = jj >> 3, j = jj & 7;
        const int slot = sub * 8192 + r0 * 128;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          RowInfo* ri = rows + (it & 1) * BK;
          if (gt < BK) {
            const RowInfo v = kb * BK + gt < K ? pixel_info(a, kb * BK + gt, ngyx) : no_pixel();
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(ri + gt)),
                         "r"((uint32_t)((uint64_t)v.off & 0xffffffffu)), "r"((uint32_t)((uint64_t)v.off >> 32)),
                         "r"((uint32_t)v.y), "r"((uint32_t)v.x)
                         : "memory");
          }
          named_bar_sync(1, NGATHER);
          uint8_t* dst = sB + s * C_::B_BYTES + slot;
          RowInfo q[BK / RSTEP];
#pragma unroll
          for (int i = 0; i < BK / RSTEP; ++i) q[i] = lds_rowinfo(ri + r0 + RSTEP * i);  // all loads first
#pragma unroll
          for (int i = 0; i < BK / RSTEP; ++i) {
            const bool ok = (unsigned)(q[i].y + dy) < (unsigned)a.sH && (unsigned)(q[i].x + dx) < (unsigned)a.sW;
            const int sw = (j ^ ((r0 + RSTEP * i) & 7)) << 4;  // 128B swizzle phase of the row
            cp_async_16(dst + i * RSTEP * 128 + sw, ok ? S + q[i].off : S0, ok ? 16u : 0u);
          }
          cp_async_mbar_arrive(&full[s]);  // lands asynchronously; the MMA thread fences the proxies
        }
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;
    constexpr int NCH = BN / 32;
    if constexpr (KIND == 0) {
      for (int local = 0; local < nseg; ++local) {
        int tile, kb0, kb1, sp;
        bool part;
        wl.seg(local, tile, kb0, kb1, sp, part);
        const int cend = part ? blockIdx.x + 1 : wl.contrib_end(tile);
        for (int cc = blockIdx.x + 1; cc < cend; ++cc) sk_wait(sk_flag(sk_ws, gridDim.x, cc, q));
        const int m0 = (tile / tiles_n) * BM;
        const int n0 = (tile % tiles_n) * BN;
        const int acc = local & 1;
        mbar_wait(&acc_full[acc], (local >> 1) & 1);
        tc_fence_after();
        const int m = m0 + q * 32 + lane;
        char* rowp = nullptr;
        int64_t erow = 0;
        // split-K (few-tile launches): this K range's fp32 partial goes to plane sp of the workspace, dense
        // [M][N]; splitk_reduce_rows sums the planes in split order and applies the epilogue
        float* prow = nullptr;
        if (m < M) {
          if (KIND == 0 && splits > 1) {
            prow = reinterpret_cast<float*>(a.ws) + ((int64_t)sp * M + m) * N;
          } else {
            const int gb = m / ngyx, rem = m - gb * ngyx;
            const int gy = rem / a.ngx, gx = rem - gy * a.ngx;
            erow = (int64_t)gb * a.c_sb + (int64_t)(a.c_ys * gy + a.c_y0) * a.c_sy + (int64_t)(a.c_xs * gx + a.c_x0) * a.c_sx;
            rowp = reinterpret_cast<char*>(a.C) + erow * (MODE == 0 ? 2 : 4);
          }
        }
        // fused element-wise operands of this row's chunk, prefetched one chunk ahead (64 B each)
        uint4 xa[4], xm[4];
        auto load_aux = [&](int c, uint4 (&A)[4], uint4 (&Mk)[4]) {
          const int n = n0 + c * 32;
          const bool ok = MODE == 0 && a.ep && !part && rowp && n + 32 <= N;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            A[v] = ok && (a.ep & 2)
                       ? __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.aux_add) + erow + n) + v)
                       : make_uint4(0, 0, 0, 0);
            Mk[v] = ok && (a.ep & 4)
                        ? __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.aux_mask) + erow + n) + v)
                        : make_uint4(0, 0, 0, 0);
          }
        };
        if (a.ep) load_aux(0, xa, xm);
        for (int c = 0; c < NCH; ++c) {
          uint4 na[4], nm[4];
          if (a.ep && c + 1 < NCH) load_aux(c + 1, na, nm);
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + acc * BN + ((uint32_t)(q * 32) << 16) + c * 32, r);
          tmem_ld_wait();
          if (c == NCH - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
            if constexpr (C2) mbar_arrive_cluster(mapa_shared(&acc_empty[acc], 0));
            else mbar_arrive(&acc_empty[acc]);
          }
          }
          if (part) {  // stream-K leading piece: fp32 partial to this CTA's workspace slot
            sk_write_chunk(sk_slot(sk_ws, blockIdx.x), q, NCH, c, lane, r);
            if (c == NCH - 1) sk_signal(sk_flag(sk_ws, gridDim.x, blockIdx.x, q));
            continue;
          }
          for (int cc = blockIdx.x + 1; cc < cend; ++cc) sk_add_chunk(sk_slot(sk_ws, cc), q, NCH, c, lane, r);
          if (c == NCH - 1 && lane == 0)
            for (int cc = blockIdx.x + 1; cc < cend; ++cc) *sk_flag(sk_ws, gridDim.x, cc, q) = 0;
          const int n = n0 + c * 32;
          if (KIND == 0 && prow) {  // split-K partial (N % 8 == 0, checked by the host)
            if (n < N) {
              float* o = prow + n;
              if (n + 32 <= N) {
#pragma unroll
                for (int v = 0; v < 8; ++v)
                  reinterpret_cast<float4*>(o)[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                                                __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
              } else {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                  if (e < N - n) o[e] = __uint_as_float(r[e]);
              }
            }
            continue;
          }
          if (!rowp || n >= N) continue;
          if (MODE == 0 && a.ep && n + 32 <= N) {
            // fused element-wise consumers (DESIGN R8/R13): v = acc (+ add), relu, zero where mask <= 0
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float f[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(r[8 * v + e]);
              if (a.ep & 2) {
                const uint4 u = xa[v];
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 x = __bfloat1622float2(h[e]);
                  f[2 * e] += x.x;
                  f[2 * e + 1] += x.y;
                }
              }
              if (a.ep & 1)
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = fmaxf(f[e], 0.f);
              uint4 w;
              __nv_bfloat162* wh = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
              for (int e = 0; e < 4; ++e) wh[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
              if (a.ep & 4) {  // relu-gradient mask on the packed result (as the GEMM epilogue): keep where mask > 0
                const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&xm[v]);
                const __nv_bfloat162 z = __float2bfloat162_rn(0.f);
                w.x &= __hgt2_mask(mh[0], z);
                w.y &= __hgt2_mask(mh[1], z);
                w.z &= __hgt2_mask(mh[2], z);
                w.w &= __hgt2_mask(mh[3], z);
              }
              reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(rowp) + n)[v] = w;
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              xa[v] = na[v];
              xm[v] = nm[v];
            }
          } else if (MODE == 0) {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(rowp) + n;
            if (n + 32 <= N) {
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                uint4 w;
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[8 * v + 2 * h]),
                                                            __uint_as_float(r[8 * v + 2 * h + 1]));
                  wp[h] = *reinterpret_cast<uint32_t*>(&b2);
                }
                reinterpret_cast<uint4*>(o)[v] = w;
              }
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e < N - n) o[e] = __float2bfloat16_rn(__uint_as_float(r[e]));
            }
          } else {
            float* o = reinterpret_cast<float*>(rowp) + n;
            if (n + 32 <= N) {
#pragma unroll
              for (int v = 0; v < 8; ++v)
                reinterpret_cast<float4*>(o)[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                                              __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e < N - n) o[e] = __uint_as_float(r[e]);
            }
          }
        }
      }
    } else {
      // TMA-store epilogue (fp32 chunks of 32 x 32 through swizzled smem), as gemm_tcgen05.cu
      const int S = nseg * NCH;
      uint8_t* wbuf = sE + q * NBUF * C_::BUF_BYTES;
      uint64_t* wbar = ebar + q * NBUF;
      int split_of_chunk = 0;
      bool part_of_chunk = false;
      auto chunk_coords = [&](int s, int& col, int& row) {
        int tile, kb0, kb1;
        wl.seg(s / NCH, tile, kb0, kb1, split_of_chunk, part_of_chunk);
        col = (tile % tiles_n) * BN + (s % NCH) * 32;
        row = (tile / tiles_n) * BM + q * 32;
      };
      auto issue_load = [&](int s) {
        int col, row;
        chunk_coords(s, col, row);
        uint8_t* b = wbuf + (s % NBUF) * C_::BUF_BYTES;
        if (part_of_chunk) {  // a stream-K partial: no epilogue operands needed
          mbar_arrive_expect_tx(&wbar[s % NBUF], 0);
          return;
        }
        mbar_arrive_expect_tx(&wbar[s % NBUF], MODE == 3 ? 6144 : 4096);
        tma_load_2d(b, &tmC, &wbar[s % NBUF], col, row);
        if (MODE == 3) tma_load_2d(b + C_::D_OFF, &tmD, &wbar[s % NBUF], col, row);
      };
      if (C_::LOADS && lane == 0)
        for (int s = 0; s < NBUF - 1 && s < S; ++s) issue_load(s);
      int local = 0;
      bool part = false;
      int cend = blockIdx.x + 1;
      for (int s = 0; s < S; ++s) {
        const int c = s % NCH;
        const int acc = local & 1;
        if (c == 0) {
          int tile, kb0, kb1, sp;
          wl.seg(s / NCH, tile, kb0, kb1, sp, part);
          cend = part ? blockIdx.x + 1 : wl.contrib_end(tile);
          for (int cc = blockIdx.x + 1; cc < cend; ++cc) sk_wait(sk_flag(sk_ws, gridDim.x, cc, q));
          mbar_wait(&acc_full[acc], (local >> 1) & 1);
          tc_fence_after();
        }
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + acc * BN + ((uint32_t)(q * 32) << 16) + c * 32, r);
        tmem_ld_wait();
        if (c == NCH - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (C2) mbar_arrive_cluster(mapa_shared(&acc_empty[acc], 0));
            else mbar_arrive(&acc_empty[acc]);
          }
          ++local;
        }
        if (part) {
          sk_write_chunk(sk_slot(sk_ws, blockIdx.x), q, NCH, c, lane, r);
          if (c == NCH - 1) sk_signal(sk_flag(sk_ws, gridDim.x, blockIdx.x, q));
        } else {
          for (int cc = blockIdx.x + 1; cc < cend; ++cc) sk_add_chunk(sk_slot(sk_ws, cc), q, NCH, c, lane, r);
          if (c == NCH - 1 && lane == 0)
            for (int cc = blockIdx.x + 1; cc < cend; ++cc) *sk_flag(sk_ws, gridDim.x, cc, q) = 0;
        }
        uint8_t* b = wbuf + (s % NBUF) * C_::BUF_BYTES;
        if (C_::LOADS) {
          if (lane == 0 && s + NBUF - 1 < S) {
            bulk_wait_read<0>();
            issue_load(s + NBUF - 1);
          }
          __syncwarp();
          mbar_wait(&wbar[s % NBUF], (s / NBUF) & 1);
        } else {
          if (lane == 0) bulk_wait_read<(NBUF > 0 ? NBUF - 1 : 0)>();
          __syncwarp();
        }
        if (part) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4* slot = reinterpret_cast<float4*>(b + lane * 128 + ((j ^ (lane & 7)) << 4));
          float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                                 __uint_as_float(r[4 * j + 3]));
          if (MODE == 2) {
            const float4 o = *slot;
            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
          } else if (MODE == 3) {
            const float4 o = *slot;
            v = make_float4(o.x * a.s0 + v.x, o.y * a.s0 + v.y, o.z * a.s0 + v.z, o.w * a.s0 + v.w);
          }
          *slot = v;
          if (MODE == 3) {
            const int wj = j >> 1, half = j & 1;
            uint2* wslot = reinterpret_cast<uint2*>(b + C_::D_OFF + lane * 64 + ((wj ^ ((lane >> 1) & 3)) << 4)) + half;
            const uint2 wv = *wslot;
            float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.x));
            float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.y));
            __nv_bfloat162 o0 = __floats2bfloat162_rn(w0.x - v.x * a.s1, w0.y - v.y * a.s1);
            __nv_bfloat162 o1 = __floats2bfloat162_rn(w1.x - v.z * a.s1, w1.y - v.w * a.s1);
            *wslot = make_uint2(*reinterpret_cast<uint32_t*>(&o0), *reinterpret_cast<uint32_t*>(&o1));
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          int col, row;
          chunk_coords(s, col, row);
          if (MODE == 4) tma_store_3d(&tmC, b, col, row, split_of_chunk);
          else tma_store_2d(&tmC, b, col, row);
          if (MODE == 3) tma_store_2d(&tmD, b + C_::D_OFF, col, row);
          bulk_commit();
        }
      }
      if (lane == 0) bulk_wait<0>();
    }
  }
  tc_fence_before();
  if constexpr (CL2 || C2) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (C2) tmem_dealloc2(tmem_base, C_::TMEM_COLS);
    else tmem_dealloc(tmem_base, C_::TMEM_COLS);
  }
}

// Split-K reduction of the weight gradient: C = epilogue(Σ_s WS[s]) in split order; mode 1 store,
// 2 accumulate, 3 fused momentum-SGD (C momentum in/out, D bf16 weight in/out).
__global__ void __launch_bounds__(256) splitk_reduce(const float* __restrict__ ws, int splits, int M, int N, float* C,
                                                     int64_t ldc, int mode, __nv_bfloat16* D, int64_t ldd, float s0,
                                                     float s1) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const int64_t plane = (int64_t)M * N;
  if (N % 4 == 0 && ldc % 4 == 0 && (mode != 3 || ldd % 4 == 0) && !(reinterpret_cast<uintptr_t>(C) & 15) &&
      !(reinterpret_cast<uintptr_t>(D) & 7)) {  // vectorised: 4 elements per thread
    const int64_t n4 = plane / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      float4 acc = reinterpret_cast<const float4*>(ws)[i];
      for (int s = 1; s < splits; ++s) {
        const float4 v = reinterpret_cast<const float4*>(ws + s * plane)[i];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      const int64_t m = (i * 4) / N, n = (i * 4) % N;
      float4* c = reinterpret_cast<float4*>(C + m * ldc + n);
      if (mode == 1) {
        *c = acc;
      } else if (mode == 2) {
        const float4 o = *c;
        *c = make_float4(o.x + acc.x, o.y + acc.y, o.z + acc.z, o.w + acc.w);
      } else {
        const float4 o = *c;
        const float4 mm = make_float4(o.x * s0 + acc.x, o.y * s0 + acc.y, o.z * s0 + acc.z, o.w * s0 + acc.w);
        *c = mm;
        uint2* w = reinterpret_cast<uint2*>(D + m * ldd + n);
        uint2 wv = *w;
        __nv_bfloat162* wh = reinterpret_cast<__nv_bfloat162*>(&wv);
        const float2 w0 = __bfloat1622float2(wh[0]), w1 = __bfloat1622float2(wh[1]);
        wh[0] = __floats2bfloat162_rn(w0.x - mm.x * s1, w0.y - mm.y * s1);
        wh[1] = __floats2bfloat162_rn(w1.x - mm.z * s1, w1.y - mm.w * s1);
        *w = wv;
      }
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = ws[i];
    for (int s = 1; s < splits; ++s) acc += ws[s * plane + i];
    const int64_t m = i / N, n = i % N;
    float* c = C + m * ldc + n;
    if (mode == 1) *c = acc;
    else if (mode == 2) *c += acc;
    else {
      const float mm = *c * s0 + acc;
      *c = mm;
      __nv_bfloat16* w = D + m * ldd + n;
      *w = __float2bfloat16_rn(__bfloat162float(*w) - mm * s1);
    }
  }
}

// Split-K reduction of a few-tile forward / data-gradient launch: out(m, n) = epilogue(Σ_s WS[s][m][n]) in split
// order, written through the output's row layout (c_sb / c_sy / c_sx, stride-2 phase offsets) with the fused
// element-wise consumers of c_mode 0 (add, relu, mask; bf16) or the fp32 store of c_mode 1.  One thread per
// (row, 8 channels).
__global__ void __launch_bounds__(256) splitk_reduce_rows(Params P) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const tofu_conv_args& a = P.a;
  const int ngyx = a.ngy * a.ngx;
  const int M = P.M, N = P.N, n8 = N / 8;
  const int64_t plane = (int64_t)M * N, total = (int64_t)M * n8;
  const float* ws = reinterpret_cast<const float*>(a.ws);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / n8), n = (int)(i - (int64_t)m * n8) * 8;
    const float* w0 = ws + (int64_t)m * N + n;
    float4 lo = reinterpret_cast<const float4*>(w0)[0], hi = reinterpret_cast<const float4*>(w0)[1];
    for (int sp = 1; sp < P.splits; ++sp) {
      const float4 l2 = reinterpret_cast<const float4*>(w0 + sp * plane)[0];
      const float4 h2 = reinterpret_cast<const float4*>(w0 + sp * plane)[1];
      lo.x += l2.x; lo.y += l2.y; lo.z += l2.z; lo.w += l2.w;
      hi.x += h2.x; hi.y += h2.y; hi.z += h2.z; hi.w += h2.w;
    }
    float f[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const int gb = m / ngyx, rem = m - gb * ngyx;
    const int gy = rem / a.ngx, gx = rem - gy * a.ngx;
    const int64_t erow =
        (int64_t)gb * a.c_sb + (int64_t)(a.c_ys * gy + a.c_y0) * a.c_sy + (int64_t)(a.c_xs * gx + a.c_x0) * a.c_sx;
    if (a.c_mode == 1) {
      float* o = reinterpret_cast<float*>(a.C) + erow + n;
      reinterpret_cast<float4*>(o)[0] = make_float4(f[0], f[1], f[2], f[3]);
      reinterpret_cast<float4*>(o)[1] = make_float4(f[4], f[5], f[6], f[7]);
      continue;
    }
    if (a.ep & 2) {
      const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.aux_add) + erow + n);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(h[e]);
        f[2 * e] += x.x;
        f[2 * e + 1] += x.y;
      }
    }
    if (a.ep & 1)
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = fmaxf(f[e], 0.f);
    if (a.ep & 4) {
      const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.aux_mask) + erow + n);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(h[e]);
        if (!(x.x > 0.f)) f[2 * e] = 0.f;
        if (!(x.y > 0.f)) f[2 * e + 1] = 0.f;
      }
    }
    uint4 w;
    __nv_bfloat162* wh = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
    for (int e = 0; e < 4; ++e) wh[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.C) + erow + n) = w;
  }
}

// zero output rows of a kind-0 sub-op with no taps (e.g. the odd phases of a 1x1 stride-2 data gradient):
// one thread per (row, 8 channels), 16-byte stores (N % 8 == 0 and 16-byte aligned rows, checked by the host)
__global__ void __launch_bounds__(256) zero_rows(Params P) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const tofu_conv_args& a = P.a;
  const int ngyx = a.ngy * a.ngx;
  const int n8 = P.N / 8;
  const int64_t total = (int64_t)P.M * n8;
  const int es = a.c_mode == 0 ? 2 : 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / n8), n = (int)(i - (int64_t)m * n8) * 8;
    const int gb = m / ngyx, rem = m - gb * ngyx;
    const int gy = rem / a.ngx, gx = rem - gy * a.ngx;
    const int64_t e = (int64_t)gb * a.c_sb + (int64_t)(a.c_ys * gy + a.c_y0) * a.c_sy +
                      (int64_t)(a.c_xs * gx + a.c_x0) * a.c_sx + n;
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<char*>(a.C) + e * es);
    o[0] = make_uint4(0, 0, 0, 0);
    if (es == 4) o[1] = make_uint4(0, 0, 0, 0);
  }
}

// Direct path (CUDA cores) for geometries the tensor-core kernel cannot take (channel ranges < 8, unaligned
// pitches): one thread per output element, fp32 accumulation over K in the same order (taps, channels /
// pixels), the same epilogues.  Only degenerate partitions use it (e.g. an 8-way split of the stem's 8 image
// channels), never an aligned shape.
__device__ __forceinline__ float bf(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }

__global__ void __launch_bounds__(256) conv_direct(Params P) {
  tofu::pdl_trigger();
  tofu::pdl_wait();
  const tofu_conv_args& a = P.a;
  const int ngyx = a.ngy * a.ngx;
  const int64_t total = (int64_t)P.M * P.N;
  const __nv_bfloat16* S = reinterpret_cast<const __nv_bfloat16*>(a.S);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / P.N), n = (int)(i % P.N);
    float acc = 0.f;
    if (a.kind == 0) {
      const RowInfo q = pixel_info(a, m, ngyx);
      const __nv_bfloat16* B = reinterpret_cast<const __nv_bfloat16*>(a.Bp);
      for (int t = 0; t < a.ntaps; ++t) {
        const int iy = q.y + a.tap_dy[t], ix = q.x + a.tap_dx[t];
        if ((unsigned)iy >= (unsigned)a.sH || (unsigned)ix >= (unsigned)a.sW) continue;
        const int64_t so = q.off + (int64_t)a.tap_dy[t] * a.s_sy + (int64_t)a.tap_dx[t] * a.s_sx + a.sc0;
        for (int c = 0; c < a.nch; ++c) {
          const int64_t bo = a.b_mn_major ? (int64_t)c * a.ldb + (int64_t)a.tap_w[t] * a.b_tap + n
                                          : (int64_t)n * a.ldb + (int64_t)a.tap_w[t] * a.b_tap + c;
          acc += bf(S, so + c) * bf(B, bo);
        }
      }
      const int gb = m / ngyx, rem = m - gb * ngyx;
      const int gy = rem / a.ngx, gx = rem - gy * a.ngx;
      const int64_t e = (int64_t)gb * a.c_sb + (int64_t)(a.c_ys * gy + a.c_y0) * a.c_sy +
                        (int64_t)(a.c_xs * gx + a.c_x0) * a.c_sx + n;
      if (a.c_mode == 1) {
        reinterpret_cast<float*>(a.C)[e] = acc;
      } else {
        if (a.ep & 2) acc += bf(reinterpret_cast<const __nv_bfloat16*>(a.aux_add), e);
        if (a.ep & 1) acc = fmaxf(acc, 0.f);
        if ((a.ep & 4) && !(bf(reinterpret_cast<const __nv_bfloat16*>(a.aux_mask), e) > 0.f)) acc = 0.f;
        reinterpret_cast<__nv_bfloat16*>(a.C)[e] = __float2bfloat16_rn(acc);
      }
    } else {
      const int t = n / a.nch, c = n - t * a.nch;
      const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(a.Ap);
      for (int p = 0; p < P.K; ++p) {
        const RowInfo q = pixel_info(a, p, ngyx);
        const int iy = q.y + a.tap_dy[t], ix = q.x + a.tap_dx[t];
        if ((unsigned)iy >= (unsigned)a.sH || (unsigned)ix >= (unsigned)a.sW) continue;
        acc += bf(A, (int64_t)p * a.lda + m) *
               bf(S, q.off + (int64_t)a.tap_dy[t] * a.s_sy + (int64_t)a.tap_dx[t] * a.s_sx + a.sc0 + c);
      }
      float* C = reinterpret_cast<float*>(a.C) + (int64_t)m * a.ldc + n;
      if (a.c_mode == 1) *C = acc;
      else if (a.c_mode == 2) *C += acc;
      else {
        const float mm = *C * a.s0 + acc;
        *C = mm;
        __nv_bfloat16* w = reinterpret_cast<__nv_bfloat16*>(a.D) + (int64_t)m * a.ldd + n;
        *w = __float2bfloat16_rn(__bfloat162float(*w) - mm * a.s1);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static PFN_cuTensorMapEncodeIm2col_v12000 g_encode_i2c = nullptr;
static std::once_flag g_once;
static int g_sms = 148;

static int init() {
  std::call_once(g_once, []() {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_i2c = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  });
  return g_encode ? 0 : -1;
}

static int tmap2(CUtensorMap* tm, const void* ptr, CUtensorMapDataType dt, int es, uint64_t inner, uint64_t outer,
                 uint64_t ld, uint32_t bi, uint32_t bo, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(tm, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : 1;
}

static int bn_of(const tofu_conv_args* a, int N) {
  if (N <= 128) return 128;
  if (a->kind == 0) {  // wave quantisation (see gemm_tcgen05.cu); 128-wide tiles re-gather A twice as often
    static const double pen = [] {
      const char* e = getenv("TOFU_CONV_BN128_EFF");
      return e ? atof(e) : 0.0;  // measured: the gather-bound kernel loses ~30% at 128-wide tiles
    }();
    const int64_t tm = ((int64_t)a->nb * a->ngy * a->ngx + BM - 1) / BM;
    const int64_t t256 = tm * ((N + 255) / 256), t128 = tm * ((N + 127) / 128);
    if (t256 * 2 > g_sms) {
      const double e256 = (double)t256 / (((t256 + g_sms - 1) / g_sms) * g_sms);
      const double e128 = pen * (double)t128 / (((t128 + g_sms - 1) / g_sms) * g_sms);
      if (e128 > e256 * 1.02) return 128;
    }
  }
  return 256;
}

static void dims_of(const tofu_conv_args* a, int& M, int& N, int& K) {
  const int pix = a->nb * a->ngy * a->ngx;
  if (a->kind == 0) {
    M = pix;
    N = a->n_out;
    K = a->ntaps * a->nch;
  } else {
    M = a->m_out;
    N = a->ntaps * a->nch;
    K = pix;
  }
}

static bool sk_enabled() {  // TOFU_SK=0 turns stream-K off (A/B measurements)
  static const bool on = [] {
    const char* e = getenv("TOFU_SK");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Split-K for few-tile forward / data-gradient launches (a rank's sub-op under a k-way plan, e.g. the 3x3
// convolutions of WResNet-152-4 at k = 8: [3136 x 512] = 50 tiles of 256 with K = 4608): each split writes an
// fp32 partial plane, splitk_reduce_rows sums them and applies the epilogue.  Only with a caller workspace
// (the executor's; one-shot calls keep one pass).  Measured: see DESIGN.md.  TOFU_CONV_SPLIT0=0 turns it off.
static int auto_splits0(const tofu_conv_args* a, int tiles, int K) {
  static const bool on = [] {
    const char* e = getenv("TOFU_CONV_SPLIT0");
    return !(e && e[0] == '0');
  }();
  const int nk = (K + BK - 1) / BK;
  if (!on || !a->ws || a->direct || a->n_out % 8 || a->c_mode > 1 || tiles * 2 > g_sms || nk < 16) return 1;
  int sp = g_sms / tiles;
  if (sp > nk / 8) sp = nk / 8;
  if (sp > 8) sp = 8;
  return sp < 2 ? 1 : sp;
}

static int auto_splits(const tofu_conv_args* a, int M, int N, int K, int bn) {
  if (a->kind != 1 || a->splits == 1) return 1;
  const int nk = (K + BK - 1) / BK;
  if (a->splits > 1) return a->splits < nk ? a->splits : nk;
  const int tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
  if (tiles * 2 > g_sms || nk < 8) return 1;
  int sp = g_sms / tiles;
  if (sp > nk / 4) sp = nk / 4;
  if (sp > 32) sp = 32;
  return sp < 2 ? 1 : sp;
}

template <int KIND, int BN, bool B_MN, int MODE, bool I2C = false, bool CL2 = false, bool C2 = false>
static int launch_t(const Params& P, const CUtensorMap* tm, cudaStream_t st) {
  using C_ = Cfg<KIND, BN, MODE, C2>;
  auto kern = conv_kernel<KIND, BN, B_MN, MODE, I2C, CL2, C2>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM) != cudaSuccess)
      return TOFU_ERR_CUDA;
    attr = true;
  }
  const int tiles = ((P.M + BM - 1) / BM) * ((P.N + BN - 1) / BN);
  const int units = tiles * P.splits;
  int grid = units < g_sms ? units : g_sms;
  Params Q = P;
  // HBM bytes: the gathered activations once (taps re-read them from L2), the dense operand, the output side
  const double M = P.M, N = P.N, K = P.K, ch = P.a.nch;
  const double e = MODE == 3 ? 12 : MODE == 2 ? 8 : MODE == 1 ? 4 : 2 + 2 * (((P.a.ep >> 1) & 1) + ((P.a.ep >> 2) & 1));
  const double bytes = KIND == 0 ? 2 * M * ch + 2 * N * K + e * M * N : 2 * K * M + 2 * K * ch + e * M * N;
  Q.sk_tiles = P.splits == 1 && sk_enabled()
                   ? sk_tiles_for(tiles, (P.K + BK - 1) / BK, g_sms, P.a.sk_ws, KIND == 1, 2 * M * N * K / bytes)
                   : 0;
  if (Q.sk_tiles) grid = g_sms;
  if constexpr (CL2 || C2) {
    Q.sk_tiles = 0;
    const int pair_units = ((P.M + 2 * BM - 1) / (2 * BM)) * ((P.N + BN - 1) / BN);
    const int ncl = pair_units < g_sms / 2 ? pair_units : g_sms / 2;
    return tofu::launch_k(kern, dim3(2 * ncl), dim3(NTHREADS), C_::SMEM, st, 2, Q, tm[0], tm[1], tm[2], tm[4]) ==
                   cudaSuccess
               ? TOFU_OK
               : TOFU_ERR_CUDA;
  }
  return tofu::launch_k(kern, dim3(grid), dim3(NTHREADS), C_::SMEM, st, 1, Q, tm[0], tm[1], tm[2], tm[4]) == cudaSuccess
             ? TOFU_OK
             : TOFU_ERR_CUDA;
}

static int dispatch(const Params& P, const CUtensorMap* tm, int mode, cudaStream_t st) {
  const tofu_conv_args& a = P.a;
  const int bn = bn_of(&a, P.N);
  if (a.kind == 0) {
    const int key = (bn == 256 ? 1 : 0) | (a.b_mn_major ? 2 : 0) | (mode << 2) | (a.im2col ? 8 : 0) |
                    (a.cl2 == 3 ? 16 : 0);
    if (a.cl2 == 3 && (bn != 256 || a.b_mn_major || !a.im2col)) return TOFU_ERR_ARG;  // (plan mismatch)
    switch (key) {
      case 1 | 8 | 16: return launch_t<0, 256, false, 0, true, false, true>(P, tm, st);
      case 1 | 4 | 8 | 16: return launch_t<0, 256, false, 1, true, false, true>(P, tm, st);
      case 8: return launch_t<0, 128, false, 0, true>(P, tm, st);
      case 9: return launch_t<0, 256, false, 0, true>(P, tm, st);
      case 10: return launch_t<0, 128, true, 0, true>(P, tm, st);
      case 11: return launch_t<0, 256, true, 0, true>(P, tm, st);
      case 12: return launch_t<0, 128, false, 1, true>(P, tm, st);
      case 13: return launch_t<0, 256, false, 1, true>(P, tm, st);
      case 14: return launch_t<0, 128, true, 1, true>(P, tm, st);
      case 15: return launch_t<0, 256, true, 1, true>(P, tm, st);
      case 0: return launch_t<0, 128, false, 0>(P, tm, st);
      case 1: return launch_t<0, 256, false, 0>(P, tm, st);
      case 2: return launch_t<0, 128, true, 0>(P, tm, st);
      case 3: return launch_t<0, 256, true, 0>(P, tm, st);
      case 4: return launch_t<0, 128, false, 1>(P, tm, st);
      case 5: return launch_t<0, 256, false, 1>(P, tm, st);
      case 6: return launch_t<0, 128, true, 1>(P, tm, st);
      case 7: return launch_t<0, 256, true, 1>(P, tm, st);
      default: return TOFU_ERR_ARG;
    }
  }
  const int key = mode | (bn == 256 ? 8 : 0) | (a.im2col ? 16 : 0) | (a.cl2 == 1 && bn == 256 && a.im2col ? 32 : 0) |
                  (a.cl2 == 3 && bn == 256 && a.im2col ? 64 : 0);
  if ((a.cl2 == 1 || a.cl2 == 3) && !(bn == 256 && a.im2col)) return TOFU_ERR_ARG;  // (plan mismatch)
  switch (key) {
    case 1 | 8 | 16 | 64: return launch_t<1, 256, true, 1, true, false, true>(P, tm, st);
    case 2 | 8 | 16 | 64: return launch_t<1, 256, true, 2, true, false, true>(P, tm, st);
    case 3 | 8 | 16 | 64: return launch_t<1, 256, true, 3, true, false, true>(P, tm, st);
    case 1 | 8 | 16 | 32: return launch_t<1, 256, true, 1, true, true>(P, tm, st);
    case 2 | 8 | 16 | 32: return launch_t<1, 256, true, 2, true, true>(P, tm, st);
    case 3 | 8 | 16 | 32: return launch_t<1, 256, true, 3, true, true>(P, tm, st);
#define TOFU_K1(MO, BNV, I) \
  case (MO) | ((BNV) == 256 ? 8 : 0) | ((I) ? 16 : 0): return launch_t<1, BNV, true, MO, (bool)(I)>(P, tm, st);
    TOFU_K1(1, 256, 0) TOFU_K1(2, 256, 0) TOFU_K1(3, 256, 0) TOFU_K1(4, 256, 0)
    TOFU_K1(1, 128, 0) TOFU_K1(2, 128, 0) TOFU_K1(3, 128, 0) TOFU_K1(4, 128, 0)
    TOFU_K1(1, 256, 1) TOFU_K1(2, 256, 1) TOFU_K1(3, 256, 1) TOFU_K1(4, 256, 1)
    TOFU_K1(1, 128, 1) TOFU_K1(2, 128, 1) TOFU_K1(3, 128, 1) TOFU_K1(4, 128, 1)
#undef TOFU_K1
    default: return TOFU_ERR_ARG;
  }
}

}  // namespace conv
}  // namespace tofu

using namespace tofu::conv;

extern "C" int64_t tofu_conv_workspace_bytes(const tofu_conv_args* a) {
  int M, N, K;
  dims_of(a, M, N, K);
  return a->splits > 1 ? (int64_t)a->splits * M * N * 4 : 0;
}

// tmaps: 4 x CUtensorMap (dense operand, C, D, split-K workspace)
static bool natural_taps(const tofu_conv_args* a) {
  for (int t = 0; t < a->ntaps; ++t)
    if (a->tap_w[t] != t) return false;
  return true;
}

static int c2_env() {  // TOFU_C2=0 / 1: 2-CTA MMA pairs off / forced (A/B measurements); -1 = automatic
  static const int v = [] {
    const char* e = getenv("TOFU_C2");
    return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
  }();
  return v;
}

// im2col TMA for the gathered activations (tmaps[4]): grids of stride <= 8, whole 64-channel blocks (kind 0: per
// tap; kind 1: the N tile of `gran` columns within one tap), corners and tap offsets within the encodable
// ranges.  pixels = the box's pixel count (kind 0: BM output pixels; kind 1: BK pixels of a k-block).
// TOFU_I2C=0 (or im2col = -1 on entry) keeps the gather warps.
static void try_im2col(tofu_conv_args* a, CUtensorMap* tm, int pixels, int gran) {
  static const bool i2c_on = [] {
    const char* e = getenv("TOFU_I2C");
    return !(e && e[0] == '0');
  }();
  const bool no_i2c = a->im2col == -1;
  a->im2col = 0;
  a->i2c_dy0 = a->i2c_dx0 = 0;
  // grid strides (stride-2 forward / weight gradient) become the map's traversal strides (elementStrides)
  if (!i2c_on || no_i2c || !g_encode_i2c || a->ntaps <= 0 || a->ay < 1 || a->ay > 8 || a->ax < 1 || a->ax > 8 ||
      a->nch % gran || a->s_sx < a->sc0 + a->nch)
    return;
  int dy0 = a->tap_dy[0], dx0 = a->tap_dx[0], dy1 = dy0, dx1 = dx0;
  for (int t = 1; t < a->ntaps; ++t) {
    dy0 = std::min<int>(dy0, a->tap_dy[t]);
    dy1 = std::max<int>(dy1, a->tap_dy[t]);
    dx0 = std::min<int>(dx0, a->tap_dx[t]);
    dx1 = std::max<int>(dx1, a->tap_dx[t]);
  }
  // traversal box (absolute buffer coordinates of the grid's first tap): W [lw, sW-1+uw], H [lh, sH-1+uh],
  // walked with steps ax / ay from the grid's first to its last pixel
  const int lw = a->cx + dx0, lh = a->cy + dy0;
  const int uw = lw + a->ax * (a->ngx - 1) - (a->sW - 1), uh = lh + a->ay * (a->ngy - 1) - (a->sH - 1);
  auto in8 = [](int v) { return v >= -128 && v <= 127; };
  if (!in8(lw) || !in8(lh) || !in8(uw) || !in8(uh) || dx1 - dx0 >= 65536 || dy1 - dy0 >= 65536) return;
  cuuint64_t dims[4] = {(cuuint64_t)a->s_sx, (cuuint64_t)a->sW, (cuuint64_t)a->sH, (cuuint64_t)(a->sb0 + a->nb)};
  cuuint64_t strides[3] = {(cuuint64_t)a->s_sx * 2, (cuuint64_t)a->s_sy * 2, (cuuint64_t)a->s_sb * 2};
  int lo[2] = {lw, lh}, hi[2] = {uw, uh};
  cuuint32_t estr[4] = {1, (cuuint32_t)a->ax, (cuuint32_t)a->ay, 1};
  if (g_encode_i2c(&tm[4], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a->S), dims, strides, lo, hi, BK,
                   (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return;
  a->im2col = 1;
  a->i2c_dy0 = dy0;
  a->i2c_dx0 = dx0;
}

extern "C" int tofu_conv_plan(tofu_conv_args* a, void* tmaps) {
  if (init() != 0) return TOFU_ERR_CUDA;
  if (!a || a->kind < 0 || a->kind > 1 || a->ntaps < 0 || a->ntaps > TOFU_CONV_MAX_TAPS || a->nch <= 0 ||
      a->nb < 0 || a->ngy < 0 || a->ngx < 0)
    return TOFU_ERR_ARG;
  auto mis = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
  int M, N, K;
  dims_of(a, M, N, K);
  a->direct = 0;
  if (a->nch % 8 || a->sc0 % 8 || a->s_sx % 8 || a->s_sy % 8 || a->s_sb % 8 || mis(a->S) || mis(a->C) ||
      mis(a->Bp) || mis(a->Ap) || mis(a->D) || mis(a->aux_add) || mis(a->aux_mask) || a->ldb % 8 || a->lda % 8 ||
      (a->kind == 0 && a->b_mn_major && a->nch < BK && BK % a->nch) ||
      (a->kind == 0 && !a->b_mn_major && a->nch % BK && (a->b_tap != a->nch || !natural_taps(a))) ||
      (a->kind == 0 && a->ep && a->n_out % 32) || (a->kind == 1 && (a->ldc % 4 || (N * 4) % 16 || a->ldd % 8))) {
    a->direct = 1;  // CUDA-core path; splits off, same epilogues
    a->splits = 1;
    if ((a->kind == 0 && a->c_mode != 0 && a->c_mode != 1) || (a->kind == 1 && (a->c_mode < 1 || a->c_mode > 3)))
      return TOFU_ERR_ARG;
    return TOFU_OK;
  }
  CUtensorMap* tm = reinterpret_cast<CUtensorMap*>(tmaps);
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const auto SW128 = CU_TENSOR_MAP_SWIZZLE_128B;
  const int bn = bn_of(a, N);
  if (a->kind == 0) {
    if (a->c_mode != 0 && a->c_mode != 1) return TOFU_ERR_ARG;
    if (a->ep && (a->c_mode != 0 || a->n_out % 32 || ((a->ep & 2) && !a->aux_add) || ((a->ep & 4) && !a->aux_mask) ||
                  mis(a->aux_add) || mis(a->aux_mask)))
      return TOFU_ERR_ARG;
    if (a->nch % BK != 0 && !a->b_mn_major) {  // K columns contiguous: taps in natural order, b_tap == nch
      if (a->b_tap != a->nch) return TOFU_ERR_ARG;
      for (int t = 0; t < a->ntaps; ++t)
        if (a->tap_w[t] != t) return TOFU_ERR_ARG;
    }
    if (a->ldb % 8) return TOFU_ERR_ALIGN;
    if (a->ntaps > 0) {
      if (a->b_mn_major && a->nch < BK && BK % a->nch) return TOFU_ERR_ARG;
      const uint32_t bk = a->nch < BK ? a->nch : BK;
      const int r = !a->b_mn_major ? tmap2(&tm[0], a->Bp, BF, 2, a->b_cols, a->b_rows, a->ldb, 64, bn, SW128)
                                   : tmap2(&tm[0], a->Bp, BF, 2, a->b_cols, a->b_rows, a->ldb, 64, bk, SW128);
      if (r) return TOFU_ERR_CUDA;
    }
    tm[1] = tm[2] = tm[3] = tm[4] = tm[0];
    a->splits = 1;
    const int req = a->cl2 == 1 || a->cl2 == 3 ? 0 : a->cl2;  // (a re-plan decides afresh)
    try_im2col(a, tm, BM, BK);
    // 2-CTA MMA pairs over vertically adjacent pixel tiles (each CTA stages half of the weight tile) for the
    // im2col forward / data gradient with K-major weights.  They give up stream-K; measured on WResNet-152-4
    // (bench.py --config 3, CUDA-graph replay, 2 runs each): 39.67 / 39.10 ms per step without, 39.00 / 38.41
    // with (the SM clock under the power cap rose 1674 -> 1714 MHz), although the isolated per-launch times
    // of the 3x3 forward rose (4.66 -> 5.03 ms per step, tools/breakdown.py).  TOFU_CONV_C2=0 turns them off.
    static const bool fwd_c2 = [] {
      const char* e = getenv("TOFU_CONV_C2");
      return !(e && e[0] == '0');
    }();
    a->cl2 = 0;
    // (TOFU_CONV_C2_FEW=0: only when the data-parallel tiles fill the SMs, so a few-tile launch — a rank's
    // sub-op under an 8-way plan, e.g. [3136 x 512] = 50 tiles — keeps stream-K; measured no different on
    // WResNet-152-4 over 8 virtual ranks, 101.2 vs 101.1 ms, so the pairs stay the default)
    static const bool c2_few = [] {
      const char* e = getenv("TOFU_CONV_C2_FEW");
      return !(e && e[0] == '0');
    }();
    const int dp_tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    a->splits = auto_splits0(a, dp_tiles, K);
    // (pairs give up stream-K: when their last wave leaves many clusters idle, the single-CTA launch with
    // stream-K wins in isolation — WResNet-152-4 stage-2 (14 x 14) 3x3 [6272 x 1024 x 9216], 100 pair units on 74 clusters
    // (wave efficiency 0.68): 95.4 us paired vs 89.0 us stream-K, GRAPH=1 tools/conv_bench.py — but not in the
    // step: 36.2 / 36.3 ms with the pairs vs 37.1 / 36.6 ms (same box, tools/kineto_step.py 3), so the rule is
    // off unless TOFU_CONV_C2_WAVE=1)
    const int pair_units = ((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn), ncl = g_sms / 2;
    const double pair_wave_eff = (double)pair_units / ((double)((pair_units + ncl - 1) / ncl) * ncl);
    static const bool wave_rule = [] {  // TOFU_CONV_C2_WAVE=1: stream-K instead of poorly-filled pairs (A/B)
      const char* e = getenv("TOFU_CONV_C2_WAVE");
      return e && e[0] == '1';
    }();
    const bool sk_better = wave_rule && a->sk_ws && sk_enabled() && pair_wave_eff < 0.8;
    if (a->splits <= 1 && req != -1 && c2_env() != 0 && a->im2col && !a->b_mn_major && bn == 256 && M > BM &&
        (req == 4 || c2_env() == 1 || (fwd_c2 && !sk_better && (c2_few || dp_tiles >= g_sms)))) {
      if (tmap2(&tm[0], a->Bp, BF, 2, a->b_cols, a->b_rows, a->ldb, 64, bn / 2, SW128)) return TOFU_ERR_CUDA;
      a->cl2 = 3;
    }
    return TOFU_OK;
  }
  // kind 1: A = output gradient [K pixels][M channels] MN-major; C f32 [M][N]
  if (a->c_mode < 1 || a->c_mode > 3 || (a->lda % 8) || (a->ldc % 4)) return TOFU_ERR_ALIGN;
  if (a->c_mode == 3 && (!a->D || a->ldd % 8)) return TOFU_ERR_ARG;
  a->splits = auto_splits(a, M, N, K, bn);
  tm[4] = tm[0];
  try_im2col(a, tm, BK, bn);  // the N tile (bn columns) must lie within one tap
  {  // cluster pairs sharing the gathered activations: 2-CTA MMA pairs (3) by default, multicast pairs (1) when
     // TOFU_C2=0; TOFU_CL2=0 turns both off; on entry -1 forbids, 2 requests the multicast pairs, 4 the 2-CTA MMA
    static const int env = [] {
      const char* e = getenv("TOFU_CL2");
      return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
    }();
    const int req = a->cl2 == 1 || a->cl2 == 3 ? 0 : a->cl2;
    const bool ok = req != -1 && env != 0 && a->im2col && a->splits <= 1 && bn == 256 && M > BM;
    const bool pair = ok && (env == 1 || req == 2 || req == 4 || K >= 2048);
    a->cl2 = !pair ? 0 : req == 2 ? 1 : req == 4 ? 3 : c2_env() != 0 ? 3 : 1;
  }
  if (tmap2(&tm[0], a->Ap, BF, 2, M, K, a->lda, 64, 64, SW128)) return TOFU_ERR_CUDA;
  if (tmap2(&tm[1], a->C, F32, 4, N, M, a->ldc, 32, 32, SW128)) return TOFU_ERR_CUDA;
  if (a->c_mode == 3) {
    if (tmap2(&tm[2], a->D, BF, 2, N, M, a->ldd, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return TOFU_ERR_CUDA;
  } else {
    tm[2] = tm[1];
  }
  if (a->splits > 1) {
    if (!a->ws || (N * 4) % 16) return TOFU_ERR_ARG;
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)a->splits};
    cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)N * M * 4};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (g_encode(&tm[3], F32, 3, a->ws, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, SW128,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return TOFU_ERR_CUDA;
  }
  return TOFU_OK;
}

extern "C" int tofu_conv_launch_planned(const tofu_conv_args* a, const void* tmaps, void* stream) {
  int M, N, K;
  dims_of(a, M, N, K);
  if (M == 0 || N == 0) return TOFU_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Params P;
  P.a = *a;
  P.M = M;
  P.N = N;
  P.K = K;
  P.splits = a->splits > 1 ? a->splits : 1;
  P.sk_tiles = 0;
  P.dy0 = a->i2c_dy0;
  P.dx0 = a->i2c_dx0;
  const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(tmaps);
  if (a->direct) {
    int blocks = (int)(((int64_t)M * N + 255) / 256);
    if (blocks > g_sms * 16) blocks = g_sms * 16;
    tofu::launch_k(conv_direct, dim3(blocks), dim3(256), 0, st, 1, P);
    return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
  }
  if (K == 0) {
    if (a->kind == 1) {
      if (a->c_mode == 1) return cudaMemset2DAsync(a->C, a->ldc * 4, 0, (size_t)N * 4, M, st) == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
      return a->c_mode == 2 ? TOFU_OK : TOFU_ERR_ARG;
    }
    if (N % 8) return TOFU_ERR_ALIGN;
    int blocks = (int)(((int64_t)M * (N / 8) + 255) / 256);
    if (blocks > g_sms * 8) blocks = g_sms * 8;
    tofu::launch_k(zero_rows, dim3(blocks), dim3(256), 0, st, 1, P);
    return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
  }
  if (a->kind == 0) {
    const int rc = dispatch(P, tm, a->c_mode, st);
    if (rc || P.splits <= 1) return rc;
    int blocks = (int)(((int64_t)M * (N / 8) + 255) / 256);
    if (blocks > g_sms * 8) blocks = g_sms * 8;
    tofu::launch_k(splitk_reduce_rows, dim3(blocks), dim3(256), 0, st, 1, P);
    return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
  }
  if (P.splits > 1) {
    const CUtensorMap tw[5] = {tm[0], tm[3], tm[3], tm[3], tm[4]};
    int rc = dispatch(P, tw, 4, st);
    if (rc) return rc;
    int blocks = (int)(((int64_t)M * N + 255) / 256);
    if (blocks > g_sms * 8) blocks = g_sms * 8;
    tofu::launch_k(splitk_reduce, dim3(blocks), dim3(256), 0, st, 1, reinterpret_cast<const float*>(a->ws), P.splits, M, N,
                                          reinterpret_cast<float*>(a->C), a->ldc, a->c_mode,
                                          reinterpret_cast<__nv_bfloat16*>(a->D), a->ldd, a->s0, a->s1);
    return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
  }
  return dispatch(P, tm, a->c_mode, st);
}

extern "C" int tofu_conv_bf16(const tofu_conv_args* args, void* stream) {
  alignas(64) CUtensorMap tm[5];
  tofu_conv_args a = *args;
  void* own_ws = nullptr;
  int r = tofu_conv_plan(&a, tm);
  if (r == TOFU_ERR_ARG && a.kind == 1 && a.splits > 1 && !a.ws) {
    // library-owned workspace for the one-shot entry point (not CUDA-graph safe)
    if (cudaMalloc(&own_ws, tofu_conv_workspace_bytes(&a)) != cudaSuccess) return TOFU_ERR_CUDA;
    a.ws = own_ws;
    r = tofu_conv_plan(&a, tm);
  }
  if (!r) r = tofu_conv_launch_planned(&a, tm, stream);
  if (own_ws) {
    cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    cudaFree(own_ws);
  }
  return r;
}
