// Sub-operator GEMM on sm_100a: TMA -> smem (SWIZZLE_128B) -> tcgen05.mma (bf16 x bf16 -> fp32 in TMEM)
// -> tcgen05.ld epilogue -> smem -> TMA store.  This is the dense-contraction sub-op every worker runs on its
// tile under partition-n-reduce (§3.1: "executing the same operator on each worker using smaller
// inputs").
//
// C[m, n] (+)= sum_k A[m, k] * B[k, n]
//   A K-major : A[m*lda + k]      A MN-major : A[k*lda + m]
//   B K-major : B[n*ldb + k]      B MN-major : B[k*ldb + n]
// The three TDL matmul defs map to (A,B) majorness: mm_nn (K, MN), mm_nt (K, K), mm_tn (MN, MN).
//
// Epilogues (c_mode): 0 = bf16 store, 1 = fp32 store (Case-2 partials, weight grads), 2 = fp32 accumulate,
// 3 = fused momentum-SGD on the weight gradient: M = M*s0 + acc (fp32, in place), W = W - M*s1 (bf16, in
// place); 4 (internal) = split-K fp32 partial into plane `split` of a 3-D workspace, reduced in split order
// by splitk_reduce_kernel (used when the output has too few tiles to fill 148 SMs, e.g. M = 128 RNN steps; the
// reduction applies the fused optimizer when c_mode is 3).  Mode 3 is the coalesced optimizer chain of P:L674-678 folded into the gradient's producer so the
// gradient never touches HBM.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer (1 lane),
// warps 2..5 = epilogue (warp w owns TMEM lanes 32*(w%4)..+31 = tile rows).  Persistent grid over output
// tiles; the accumulator is double-buffered in TMEM so the epilogue of tile t overlaps the mainloop of t+1.
// The epilogue moves 32x32 chunks through swizzled smem with TMA (loads of M/W prefetched NBUF-1 chunks ahead,
// bulk-async stores), so every HBM access is a full-line TMA transfer.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "../tofu_kernels.h"

namespace tofu {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int SMEM_MAX = 232448;  // 227 KB opt-in per CTA on sm_100
// Epilogue width: 4 warps (one per TMEM lane quarter) or 8 (two per quarter, each half of the tile's columns),
// chosen per launch (bit 3 of the MODE_ template value): 8 for memory-leaning launches, whose epilogue streams the output
// and its fused operands through HBM (measured, tools/sk_bench.py: the residual-add / relu-gradient-mask
// epilogues of 1x1 convolutions with K <= 1024 run 1.3-1.7x faster, the configs[1] fused momentum-SGD weight
// gradient 0.200 -> 0.167 ms); 4 for compute-bound launches, which keep one more smem pipeline stage.
template <int BN, int MODE_>
struct GemmCfg {
  static constexpr int MODE = MODE_ & 7;
  static constexpr bool W8 = (MODE_ & 8) != 0;
  // C2 (bit 4): 2-CTA MMA pairs (tcgen05.mma.cta_group::2, M = 256 over the pair): each CTA stages its own
  // 128 rows of A and half (BN/2 rows) of B
  static constexpr bool C2 = (MODE_ & 16) != 0;
  // WIDE (bit 5, MODE 5 only): the epilogue moves 32 x 64 chunks (two 32 x 32 boxes per operand behind one
  // barrier wait, one proxy fence, one store issue), halving the per-chunk fixed instructions of the
  // issue-bound fused epilogues; double-size buffers, so only for short-K launches that need few stages
  static constexpr bool WIDE = (MODE_ & 32) != 0;
  static constexpr int CWD = WIDE ? 2 : 1;
  static_assert(!WIDE || (MODE_ & 7) == 5, "wide chunks: fused element-wise epilogue only");
  // MODE 5 may load (residual add / relu mask operands, when its runtime `ep` asks for them)
  static constexpr bool LOADS = MODE == 2 || MODE == 3 || MODE == 5;
  // the fused optimizer (MODE 3) and the fused element-wise epilogue (MODE 5) stream extra operands through
  // the epilogue (HBM-bound): deeper prefetch
#ifndef TOFU_NBUF5
#define TOFU_NBUF5 2
#endif
#ifndef TOFU_NBUF5_128
#define TOFU_NBUF5_128 TOFU_NBUF5
#endif
#ifndef TOFU_NBUF3
#define TOFU_NBUF3 2
#endif
  static constexpr int NBUF = LOADS ? (MODE == 3 ? (W8 ? TOFU_NBUF3 : 3) : MODE == 5 ? (BN == 256 ? TOFU_NBUF5 : TOFU_NBUF5_128) : 3) : 2;
  static constexpr int C_BYTES = 32 * 32 * (MODE == 0 || MODE == 5 ? 2 : 4);
  // MODE 3: W chunk at D_OFF.  MODE 5: add chunk at 0 (the bf16 result overwrites it in place, each thread
  // its own 16-byte slots), mask chunk at D_OFF = 2048.
  static constexpr int D_OFF = MODE == 5 ? 2048 * CWD : 4096;
  static constexpr int BUF_BYTES = MODE == 3 ? 6144 : MODE == 5 ? 4096 * CWD : (C_BYTES < 1024 ? 1024 : C_BYTES);
  // epilogue warps: 4 (one per TMEM lane quarter) or 8 (two per quarter, each half of the tile's columns)
  static constexpr int EW = W8 ? 8 : 4;
  static constexpr int THREADS = 64 + 32 * EW;
  static constexpr int EPI_BYTES = EW * NBUF * BUF_BYTES;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (C2 ? BN / 2 : BN) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_FIT = (SMEM_MAX - 1024 - 512 - EPI_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr int ACC_BUFS = 2;
  static constexpr int TMEM_COLS = BN * ACC_BUFS;  // 256 or 512 fp32 columns
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 512 /*barriers*/;
  static_assert(STAGES >= 2, "pipeline too shallow");
  static_assert(SMEM <= SMEM_MAX, "smem");
};

// Tile order: column-major (m fastest) when B is the larger operand (N > M), so each wave of persistent CTAs
// covers all of M for a few n columns and A stays resident in L2 while B streams through once (the LSTM gate
// weight gradients, N = 16384 >> M = 4096: measured DRAM reads 1.57 GB -> see DESIGN); TOFU_RASTER=0 keeps
// row-major everywhere.
static int raster_of(const tofu_gemm_args* g) {
  static const int env = [] {
    const char* e = getenv("TOFU_RASTER");
    return e ? atoi(e) : 1;
  }();
  return env && g->N > g->M ? 1 : 0;
}

// Piecewise operands (tofu_operand_pieces, the MultiFetch fused into the TMA producer): one map per piece and
// the pieces' starts along the split dimension (0 = M / N, 1 = K).  Passed by value as a __grid_constant__
// kernel parameter (TMA reads maps from parameter space) only by the PC instantiations.
struct PieceMaps {
  CUtensorMap a_map[TOFU_MAX_PIECES];
  CUtensorMap b_map[TOFU_MAX_PIECES];
  int na, a_dim, nb, b_dim;
  int a_start[TOFU_MAX_PIECES], b_start[TOFU_MAX_PIECES];
};
struct NoPieces {};

// the map and the map-local coordinate of a tile coordinate (along the pieces' dimension)
__device__ __forceinline__ const CUtensorMap* piece_of(const CUtensorMap* maps, const int* start, int n, int c,
                                                       int& local) {
  int i = 0;
  while (i + 1 < n && c >= start[i + 1]) ++i;
  local = c - start[i];
  return maps + i;
}

// CL2: cluster of 2 CTAs on vertically adjacent tiles (m tiles 2p, 2p+1) of the same n tile; each CTA
// TMA-loads half of the shared B tile and multicasts it to both (halving B's L2 -> SM traffic per flop), and
// frees a stage only when both CTAs' MMAs have consumed it (the MMA commit arrives on both CTAs' barriers).
template <int BN, bool A_MN, bool B_MN, int MODE_, bool PC, bool CL2 = false>
__global__ void __launch_bounds__(GemmCfg<BN, MODE_>::THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ std::conditional_t<PC, PieceMaps, NoPieces> pm,
                     const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmD,
                     const __grid_constant__ CUtensorMap tmE, int M, int N, int K, float s0, float s1, int splits,
                     int ep, int sk_tiles, void* sk_ws, int raster) {
  using Cfg = GemmCfg<BN, MODE_>;
  constexpr int MODE = Cfg::MODE;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int NBUF = Cfg::NBUF;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by an offset from the __shared__ array (an integer round trip through uintptr_t would lose
  // the address space: every epilogue smem access became a generic LD.E / ST.E)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sE = smem + STAGES * Cfg::STAGE_BYTES;  // epilogue chunk buffers [4 warps][NBUF]
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + Cfg::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;             // [ACC_BUFS]
  uint64_t* acc_empty = acc_full + Cfg::ACC_BUFS;  // [ACC_BUFS]
  uint64_t* ebar = acc_empty + Cfg::ACC_BUFS;      // [4][NBUF] epilogue load barriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + Cfg::EW * NBUF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM;
  const int tiles_n = (N + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;
  const int nk = (K + BK - 1) / BK;
  // segments = (output tile, k-block range): data-parallel units (tile, K split) then stream-K pieces
  WorkList wl;
  wl.raster = raster & 1;
  // bit 1: walk each segment's k-blocks from the last to the first (alternated launch by launch over the same
  // weight by the executor: the tail of the previous pass is still in L2 when the next pass starts)
  const bool krev = (raster & 2) != 0;
  wl.tiles_m = tiles_m;
  wl.tiles_n = tiles_n;
  uint32_t crank = 0;
  constexpr bool C2 = Cfg::C2;
  if constexpr (CL2 || C2) {
    crank = cluster_rank();
    wl.init_pairs(tiles_m, tiles_n, nk, (int)crank, (int)cluster_id_x(), (int)nclusters_x());
  } else {
    wl.init(ntiles, nk, splits, sk_tiles);
  }
  const int nseg = wl.count();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL2 && !C2 ? 2 : 1);  // CL2: both CTAs' MMAs must have read the stage
    }
    for (int b = 0; b < Cfg::ACC_BUFS; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], C2 ? 2 * Cfg::EW : Cfg::EW);  // one arrive per epilogue warp (C2: of both CTAs)
    }
    for (int b = 0; b < Cfg::EW * NBUF; ++b) mbar_init(&ebar[b], 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    if (MODE == 3 || MODE == 5) tma_prefetch_desc(&tmD);
    if (MODE == 5) tma_prefetch_desc(&tmE);
    if constexpr (PC) {  // the piece maps (fused fetch) live in parameter space like the others
      for (int i = 0; i < pm.na; ++i) tma_prefetch_desc(&pm.a_map[i]);
      for (int i = 0; i < pm.nb; ++i) tma_prefetch_desc(&pm.b_map[i]);
    }
  }
  if (warp == 1) {
    if constexpr (C2) tmem_alloc2(tmem_slot, Cfg::TMEM_COLS);
    else tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CL2 || C2) cluster_sync_all();  // the peer's barriers are initialised before any multicast
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // prologue done: now wait for the predecessor's results (PDL)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
#ifdef TOFU_EXP_NOMAIN
    if (false) {
#else
    if (lane == 0) {
#endif
      int it = 0;
      for (int i = 0; i < nseg; ++i) {
        int tile, kb0, kb1, sp;
        bool part;
        wl.seg(i, tile, kb0, kb1, sp, part);
        const int m0 = (tile / tiles_n) * BM;
        const int n0 = (tile % tiles_n) * BN;
        for (int ki = 0; ki < kb1 - kb0; ++ki, ++it) {
          const int kb = krev ? kb1 - 1 - ki : kb0 + ki;
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          // C2: both CTAs' loads complete on the leader's barrier, which expects the pair's bytes
          if constexpr (C2) {
            if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
          } else {
            mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
          }
          uint8_t* a = sA + s * Cfg::A_BYTES;
          uint8_t* b = sB + s * Cfg::B_BYTES;
          const int k0 = kb * BK;
          const CUtensorMap* ma = &tmA;
          const CUtensorMap* mb = &tmB;
          int am = m0, ak = k0, bnn = n0, bk = k0;
          if constexpr (PC) {  // operand regions read in place from their owners' shards (peer or own HBM)
            if (pm.na) ma = pm.a_dim ? piece_of(pm.a_map, pm.a_start, pm.na, k0, ak)
                                     : piece_of(pm.a_map, pm.a_start, pm.na, m0, am);
            if (pm.nb) mb = pm.b_dim ? piece_of(pm.b_map, pm.b_start, pm.nb, k0, bk)
                                     : piece_of(pm.b_map, pm.b_start, pm.nb, n0, bnn);
          }
          if constexpr (C2) {  // own A rows, own half of B; completion on the leader's full barrier
            const uint32_t lf = mapa_shared(&full[s], 0);
            if (!A_MN) {
              tma_load_2d_2sm(a, ma, lf, ak, am);
            } else {
#pragma unroll
              for (int c = 0; c < BM / 64; ++c) tma_load_2d_2sm(a + c * 8192, ma, lf, am + 64 * c, ak);
            }
            if (!B_MN) {
              tma_load_2d_2sm(b, mb, lf, bk, bnn + (int)crank * (BN / 2));
            } else {
#pragma unroll
              for (int c = 0; c < BN / 128; ++c)
                tma_load_2d_2sm(b + c * 8192, mb, lf, bnn + 64 * ((int)crank * (BN / 128) + c), bk);
            }
          } else if (!A_MN) {
            tma_load_2d(a, ma, &full[s], ak, am);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) tma_load_2d(a + c * 8192, ma, &full[s], am + 64 * c, ak);
          }
          if constexpr (C2) {
          } else if constexpr (CL2) {  // this CTA's half of B, multicast into both CTAs' stage
            if (!B_MN) {
              tma_load_2d_mc(b + crank * (Cfg::B_BYTES / 2), mb, &full[s], bk, bnn + (int)crank * (BN / 2), 0x3);
            } else {
#pragma unroll
              for (int c = 0; c < BN / 128; ++c) {
                const int cc = (int)crank * (BN / 128) + c;
                tma_load_2d_mc(b + cc * 8192, mb, &full[s], bnn + 64 * cc, bk, 0x3);
              }
            }
          } else if (!B_MN) {
            tma_load_2d(b, mb, &full[s], bk, bnn);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(b + c * 8192, mb, &full[s], bnn + 64 * c, bk);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (C2: the pair leader only)
    if (lane == 0 && (!C2 || crank == 0)) {
      constexpr uint32_t idesc = umma_idesc_bf16(C2 ? 2 * BM : BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int it = 0;
      for (int local = 0; local < nseg; ++local) {
        int tile, kb0, kb1, sp;
        bool part;
        wl.seg(local, tile, kb0, kb1, sp, part);
        const int buf = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&acc_empty[buf], aph ^ 1);  // epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + buf * BN;
#ifdef TOFU_EXP_NOMAIN
        kb1 = kb0;
#endif
        for (int ki = 0; ki < kb1 - kb0; ++ki, ++it) {
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
            if constexpr (C2) umma_bf16_2(tmem_d, ad, bd, idesc, (ki > 0 || kk) ? 1u : 0u);
            else umma_bf16(tmem_d, ad, bd, idesc, (ki > 0 || kk) ? 1u : 0u);
          }
          if constexpr (C2) umma_commit2_mc(&empty[s], 0x3);     // frees stage s in both CTAs
          else if constexpr (CL2) umma_commit_mc(&empty[s], 0x3);  // both CTAs' stage s: this CTA has read it
          else umma_commit(&empty[s]);  // frees the smem stage when these MMAs complete
        }
        if constexpr (C2) umma_commit2_mc(&acc_full[buf], 0x3);  // both CTAs' accumulator halves are ready
        else umma_commit(&acc_full[buf]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;  // TMEM lane quarter = tile rows 32q..32q+31
    constexpr int CWD = Cfg::CWD;                // 32-column sub-chunks per chunk
    constexpr int NCH = BN / (32 * CWD);         // chunks of a tile row quarter
    constexpr int NCW = NCH / (Cfg::EW / 4);     // of which this warp handles [h*NCW, (h+1)*NCW)
    const int e = warp - 2, h = e / 4;
    const int S = nseg * NCW;
    uint8_t* wbuf = sE + e * NBUF * Cfg::BUF_BYTES;
    uint64_t* wbar = ebar + e * NBUF;
    int split_of_chunk = 0;
    bool part_of_chunk = false;
    // chunk coordinates through a cursor that re-derives its segment (integer divisions) only when the chunk
    // crosses into the next tile: one cursor for the operand loads running ahead, one for the stores
    struct Cursor {
      int seg = -1, col0 = 0, row = 0, split = 0;
      bool part = false;
    };
    Cursor lcur, scur;
    auto chunk_coords_c = [&](Cursor& k, int s, int& col, int& row) {
      const int sg = s / NCW;
      if (sg != k.seg) {
        int tile, kb0, kb1;
        wl.seg(sg, tile, kb0, kb1, k.split, k.part);
        const int tm = tile / tiles_n;
        k.seg = sg;
        k.col0 = (tile - tm * tiles_n) * BN + h * NCW * 32 * CWD;
        k.row = tm * BM + q * 32;
      }
      split_of_chunk = k.split;
      part_of_chunk = k.part;
      col = k.col0 + (s - sg * NCW) * 32 * CWD;
      row = k.row;
    };
    auto chunk_coords = [&](int s, int& col, int& row) { chunk_coords_c(scur, s, col, row); };
    // MODE 5 loads only the operands its runtime `ep` names (2 KB each: a 32x32 bf16 chunk, SWIZZLE_64B)
    const bool loads = MODE == 5 ? (ep & 6) != 0 : Cfg::LOADS;
    const uint32_t load_bytes =
        MODE == 3 ? 6144 : MODE == 5 ? 2048u * CWD * (((ep >> 1) & 1) + ((ep >> 2) & 1)) : 4096;
    auto issue_load = [&](int s) {  // lane 0 only
      int col, row;
      chunk_coords_c(lcur, s, col, row);
      uint8_t* b = wbuf + (s % NBUF) * Cfg::BUF_BYTES;
      if (part_of_chunk) {  // a stream-K partial: no epilogue operands needed
        mbar_arrive_expect_tx(&wbar[s % NBUF], 0);
        return;
      }
      mbar_arrive_expect_tx(&wbar[s % NBUF], load_bytes);
      if (MODE == 5) {
#pragma unroll
        for (int d = 0; d < CWD; ++d) {
          if (ep & 2) tma_load_2d(b + d * 2048, &tmD, &wbar[s % NBUF], col + 32 * d, row);
          if (ep & 4) tma_load_2d(b + Cfg::D_OFF + d * 2048, &tmE, &wbar[s % NBUF], col + 32 * d, row);
        }
      } else {
        tma_load_2d(b, &tmC, &wbar[s % NBUF], col, row);
        if (MODE == 3) tma_load_2d(b + Cfg::D_OFF, &tmD, &wbar[s % NBUF], col, row);
      }
    };
    if (loads && lane == 0)
      for (int s = 0; s < NBUF - 1 && s < S; ++s) issue_load(s);
    int local = 0;
    bool part = false;         // current segment is a stream-K partial (written to the workspace)
    int cend = blockIdx.x + 1; // finisher: partials of CTAs blockIdx.x+1 .. cend-1 are added
    for (int s = 0; s < S; ++s) {
      const int cw = s % NCW, c = h * NCW + cw;
      const int acc = local & 1;
      if (cw == 0) {
        int tile, kb0, kb1, sp;
        wl.seg(s / NCW, tile, kb0, kb1, sp, part);
        cend = part ? blockIdx.x + 1 : wl.contrib_end(tile);
        for (int cc = blockIdx.x + 1; cc < cend; ++cc) sk_wait(sk_flag(sk_ws, gridDim.x, cc, e));
        mbar_wait(&acc_full[acc], (local >> 1) & 1);
        tc_fence_after();
      }
      uint32_t rr[CWD][32];
      uint32_t(&r)[32] = rr[0];
#ifdef TOFU_EXP_NOTMEM
      for (int i = 0; i < 32; ++i) r[i] = 0;
#else
#pragma unroll
      for (int d = 0; d < CWD; ++d)
        tmem_ld_32x32b_x32(tmem_base + acc * BN + ((uint32_t)(q * 32) << 16) + (c * CWD + d) * 32, rr[d]);
      tmem_ld_wait();
#endif
      if (cw == NCW - 1) {  // accumulator fully read: hand TMEM back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (C2) mbar_arrive_cluster(mapa_shared(&acc_empty[acc], 0));  // the leader's MMA waits
          else mbar_arrive(&acc_empty[acc]);
        }
        ++local;
      }
      if (Cfg::WIDE) {  // (the dispatcher never pairs wide chunks with stream-K)
      } else if (part) {
        sk_write_chunk(sk_slot(sk_ws, blockIdx.x), q, NCH, c, lane, r);
        if (cw == NCW - 1) sk_signal(sk_flag(sk_ws, gridDim.x, blockIdx.x, e));
      } else {
        for (int cc = blockIdx.x + 1; cc < cend; ++cc) sk_add_chunk(sk_slot(sk_ws, cc), q, NCH, c, lane, r);
        if (cw == NCW - 1 && lane == 0)
          for (int cc = blockIdx.x + 1; cc < cend; ++cc) *sk_flag(sk_ws, gridDim.x, cc, e) = 0;
      }
      uint8_t* b = wbuf + (s % NBUF) * Cfg::BUF_BYTES;
      // Refill of the buffer chunk s-1 used (operand chunk s+NBUF-1), issued once chunk s is done: the store of
      // chunk s-1 has had a whole chunk's time to read that buffer, so the wait rarely blocks (waiting instead for
      // the store issued just before serialised every chunk behind a TMA store's smem read).
      auto refill = [&](bool stored) {
        if (lane == 0 && s + NBUF - 1 < S) {
          if (stored) bulk_wait_read<1>();  // all but the newest store (chunk s, another buffer) have read smem
          else bulk_wait_read<0>();
          issue_load(s + NBUF - 1);
        }
      };
      // (with two buffers the refill of chunk s+1 cannot wait for chunk s to finish: issued first, after the
      // store of chunk s-1 has read its buffer)
      constexpr bool LATE = NBUF >= 3;
      if (loads) {
        if (!LATE && lane == 0 && s + NBUF - 1 < S) {
          bulk_wait_read<0>();
          issue_load(s + NBUF - 1);
        }
        __syncwarp();
        mbar_wait(&wbar[s % NBUF], (s / NBUF) & 1);
      } else {
        if (lane == 0) bulk_wait_read<NBUF - 1>();
        __syncwarp();
      }
      if (part) {
        if (LATE && loads) refill(false);
        continue;
      }
      if (MODE == 5) {
        // fused element-wise ops of the output's consumers (DESIGN R8/R13): v = acc (+ add), relu, mask
#pragma unroll
        for (int dj = 0; dj < 4 * CWD; ++dj) {
          const int d = dj >> 2, j = dj & 3;
          const uint32_t(&r)[32] = rr[d];
          const int off = d * 2048 + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[8 * j + e]);
          if (ep & 2) {  // + residual: bf16 pairs widened by shift / mask, added as fp32 pairs (FADD2)
            const uint4 u = *reinterpret_cast<const uint4*>(b + off);
            const uint32_t uw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint64_t a2 = (uint64_t)r[8 * j + 2 * e] | ((uint64_t)r[8 * j + 2 * e + 1] << 32);
              const uint64_t b2 = (uint64_t)(uw[e] << 16) | ((uint64_t)(uw[e] & 0xffff0000u) << 32);
              uint64_t s2;
              asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s2) : "l"(a2), "l"(b2));
              v[2 * e] = __uint_as_float((uint32_t)s2);
              v[2 * e + 1] = __uint_as_float((uint32_t)(s2 >> 32));
            }
          }
          if (ep & 1)
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
          uint4 w;
          __nv_bfloat162* wh = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
          for (int e = 0; e < 4; ++e) wh[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
          if (ep & 4) {  // relu-gradient mask, on the packed result: keep where mask > 0 (NaN, +-0: zero)
            const uint4 u = *reinterpret_cast<const uint4*>(b + Cfg::D_OFF + off);
            const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&u);
            const __nv_bfloat162 z = __float2bfloat162_rn(0.f);
            w.x &= __hgt2_mask(mh[0], z);
            w.y &= __hgt2_mask(mh[1], z);
            w.z &= __hgt2_mask(mh[2], z);
            w.w &= __hgt2_mask(mh[3], z);
          }
          *reinterpret_cast<uint4*>(b + off) = w;
        }
      } else if (MODE == 0) {
        uint32_t p[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
          p[j] = *reinterpret_cast<uint32_t*>(&h);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(b + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
              make_uint4(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4* slot = reinterpret_cast<float4*>(b + lane * 128 + ((j ^ (lane & 7)) << 4));
          float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          if (MODE == 2) {
            const float4 o = *slot;
            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
          } else if (MODE == 3) {
            const float4 o = *slot;
            v = make_float4(o.x * s0 + v.x, o.y * s0 + v.y, o.z * s0 + v.z, o.w * s0 + v.w);
          }
          *slot = v;
          if (MODE == 3) {  // W chunk: 8 bf16 per 16B, row = 64 B, SWIZZLE_64B
            const int wj = j >> 1, half = j & 1;
            uint2* wslot = reinterpret_cast<uint2*>(b + Cfg::D_OFF + lane * 64 + ((wj ^ ((lane >> 1) & 3)) << 4)) + half;
            const uint2 wv = *wslot;
            float2 w0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.x));
            float2 w1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.y));
            __nv_bfloat162 n0 = __floats2bfloat162_rn(w0.x - v.x * s1, w0.y - v.y * s1);
            __nv_bfloat162 n1 = __floats2bfloat162_rn(w1.x - v.z * s1, w1.y - v.w * s1);
            *wslot = make_uint2(*reinterpret_cast<uint32_t*>(&n0), *reinterpret_cast<uint32_t*>(&n1));
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        int col, row;
        chunk_coords(s, col, row);
        if (MODE == 4) tma_store_3d(&tmC, b, col, row, split_of_chunk);  // fp32 partial plane of this split
        else
#pragma unroll
          for (int d = 0; d < CWD; ++d) tma_store_2d(&tmC, b + d * 2048, col + 32 * d, row);
        if (MODE == 3) tma_store_2d(&tmD, b + Cfg::D_OFF, col, row);
        bulk_commit();
      }
      if (LATE && loads) refill(true);
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  if constexpr (CL2 || C2) cluster_sync_all();  // no multicast / remote commit may target an exited CTA
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (C2) tmem_dealloc2(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
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

// 2-D tensor map: inner extent (contiguous), outer extent, row pitch `ld` elements.
static int make_tmap(CUtensorMap* tm, const void* ptr, CUtensorMapDataType dt, int esize, uint64_t inner,
                     uint64_t outer, uint64_t ld, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(tm, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -(int)r - 1000;
}

static bool sk_enabled() {  // TOFU_SK=0 turns stream-K off (A/B measurements)
  static const bool on = [] {
    const char* e = getenv("TOFU_SK");
    return !(e && e[0] == '0');
  }();
  return on;
}

// 8 epilogue warps when a tile's epilogue traffic rivals its mainloop: per output element 2K flops against
// e bytes of output-side HBM traffic (bf16 / fused element-wise / fused optimizer outputs).  Measured: the
// configs[1] weight gradient (2K/e = 85) and the WResNet 1x1 add / mask epilogues (2K/e = 128..512) gain;
// with the optimizer the wide epilogue leaves 2 smem stages (vs 3) and loses from 2K/e ~ 430 (LSTM gate
// weight gradients), bf16 outputs keep 3 (vs 4) and lose at 2K/e >= 1000.
static int ew8_override();
static bool wants_w8(const tofu_gemm_args* g) {
  const int mode = g->c_mode == 0 && g->ep ? 5 : g->c_mode;
  if (mode != 0 && mode != 3 && mode != 5) return false;
  const int ov = ew8_override();
  if (ov >= 0) return ov == 1;
  const double e = mode == 3 ? 12 : 2 + 2 * (((g->ep >> 1) & 1) + ((g->ep >> 2) & 1));
  const double lim = mode == 3 ? 200.0 : 600.0;
  return 2.0 * g->K / e < lim;
}

// algorithmic flops / HBM bytes of a launch (operands once, output side e bytes per element)
static double gemm_intensity(const tofu_gemm_args* g, int mode) {
  const double M = g->M, N = g->N, K = g->K;
  const double e = mode == 3 ? 12 : mode == 2 ? 8 : mode == 1 ? 4 : 2 + 2 * (((g->ep >> 1) & 1) + ((g->ep >> 2) & 1));
  return 2 * M * N * K / (2 * M * K + 2 * N * K + e * M * N);
}
// Wide (32 x 64) epilogue chunks for the 8-warp fused element-wise epilogues of short-K launches: half the
// per-chunk fixed instructions, but the double-size buffers leave 256-wide tiles 2 smem stages instead of 3,
// which the K loop of long-K launches feels.  TOFU_EP_WIDE_K = largest K that takes them (0: never).  Measured
// (tools/ep_stream_bench.py): K = 256 add+mask 119 -> 112 us (0.91 of the copy peak), add+relu 100 -> 95 us;
// K = 512 add+mask 74 -> 87 us and K = 1024 mask 66 -> 82 us (slower: the lost stage).
static bool ep_wide(const tofu_gemm_args* g) {
  static const int kmax = [] {
    const char* e = getenv("TOFU_EP_WIDE_K");
    return e ? atoi(e) : 256;
  }();
  return g->K <= kmax;
}
static int ew8_override() {  // TOFU_EW8=0 / 1 forces the 4- / 8-warp epilogue (A/B measurements); else auto
  static const int v = [] {
    const char* e = getenv("TOFU_EW8");
    return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
  }();
  return v;
}

template <int BN, bool A_MN, bool B_MN, int MODE_, bool PC, bool CL2 = false>
static int launch_t(const tofu_gemm_args* g, const CUtensorMap* tm, const PieceMaps* pm, cudaStream_t st, double ai) {
  using Cfg = GemmCfg<BN, MODE_>;
  constexpr int MODE = Cfg::MODE;
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, MODE_, PC, CL2>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
      return TOFU_ERR_CUDA;
    attr_set = true;
  }
  const int splits = MODE == 4 ? g->splits : 1;
  const int tiles = ((g->M + BM - 1) / BM) * ((g->N + BN - 1) / BN);
  const int units = tiles * splits;
  int grid = units < g_num_sms ? units : g_num_sms;
  if (g->max_ctas > 0 && grid > g->max_ctas) grid = g->max_ctas;
  int sk = 0;
  // stream-K only on request (splits = -1): measured on one B200 it does not pay for TMA-fed GEMMs
  // (tools/sk_bench.py, e.g. 196 tiles K = 9216: 111 us data-parallel vs 118 us stream-K; DESIGN.md has our
  // reading); the gathered convolutions use it by default
  if (g->splits == -1 && g->max_ctas == 0 && sk_enabled()) {
    (void)ai;
    sk = sk_tiles_for(tiles, (g->K + BK - 1) / BK, g_num_sms, g->sk_ws, false, 1e30);
    if (sk) grid = g_num_sms;
  }
  std::conditional_t<PC, PieceMaps, NoPieces> pp{};
  if constexpr (PC) pp = *pm;
  (void)pm;
  if constexpr (CL2) {  // clusters of 2 over pair units (m tiles 2p, 2p+1 of one n tile)
    const int pair_units = ((g->M + 2 * BM - 1) / (2 * BM)) * ((g->N + BN - 1) / BN);
    const int ncl = pair_units < g_num_sms / 2 ? pair_units : g_num_sms / 2;
    const cudaError_t e = launch_k(kern, dim3(2 * ncl), dim3(Cfg::THREADS), Cfg::SMEM, st, 2, pp, tm[0], tm[1], tm[2],
                                   tm[3], tm[5], g->M, g->N, g->K, g->s0, g->s1, 1, g->ep, 0, g->sk_ws,
                                   raster_of(g) | (g->k_reverse ? 2 : 0));
    return e == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
  }
  return launch_k(kern, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, st, 1, pp, tm[0], tm[1], tm[2], tm[3], tm[5], g->M,
                  g->N, g->K, g->s0, g->s1, splits, g->ep, sk, g->sk_ws,
                  (splits == 1 && sk == 0 ? raster_of(g) : 0) | (g->k_reverse ? 2 : 0)) == cudaSuccess
             ? TOFU_OK
             : TOFU_ERR_CUDA;
}

template <int BN>
static int dispatch_bn(const tofu_gemm_args* g, const CUtensorMap* tm, const PieceMaps* pm, cudaStream_t st) {
  const int mode = g->c_mode == 0 && g->ep ? 5 : g->c_mode;
  const double ai = gemm_intensity(g, mode);
  const bool pc = pm != nullptr;  // piecewise operands (fused fetch)
  const bool w8 = wants_w8(g);
  const bool cl2 = BN == 256 && g->cl2 == 1 && !pc && mode != 4;
  // (the plan encoded B with half-height boxes for both pair kinds: a launch that cannot honour the pairing
  // would wait for bytes that never arrive)
  const bool c2 = BN == 256 && g->cl2 == 3 && !pc && mode != 4;
  if ((g->cl2 == 1 && !cl2) || (g->cl2 == 3 && !c2)) return TOFU_ERR_ARG;
  if (c2) {
    const int k2 = (g->a_mn_major ? 1 : 0) | (g->b_mn_major ? 2 : 0) | ((mode | (w8 ? 8 : 0)) << 2);
    switch (k2) {
#define TOFU_CASE3(AM, BMJ, O) \
  case ((AM) | ((BMJ) << 1) | ((O) << 2)): return launch_t<BN, (bool)(AM), (bool)(BMJ), (O) | 16, false, true>(g, tm, pm, st, ai);
#define TOFU_CASES3(O) TOFU_CASE3(0, 0, O) TOFU_CASE3(0, 1, O) TOFU_CASE3(1, 0, O) TOFU_CASE3(1, 1, O)
      TOFU_CASES3(0) TOFU_CASES3(1) TOFU_CASES3(2) TOFU_CASES3(3) TOFU_CASES3(5)
      TOFU_CASES3(8) TOFU_CASES3(11) TOFU_CASES3(13)
#undef TOFU_CASES3
#undef TOFU_CASE3
      default: return TOFU_ERR_ARG;
    }
  }
  if (mode == 5 && w8 && !cl2 && g->splits != -1 && ep_wide(g)) {  // 32 x 64 epilogue chunks
    switch ((g->a_mn_major ? 1 : 0) | (g->b_mn_major ? 2 : 0) | (pc ? 4 : 0)) {
      case 0: return launch_t<BN, false, false, 13 | 32, false>(g, tm, pm, st, ai);
      case 1: return launch_t<BN, true, false, 13 | 32, false>(g, tm, pm, st, ai);
      case 2: return launch_t<BN, false, true, 13 | 32, false>(g, tm, pm, st, ai);
      case 3: return launch_t<BN, true, true, 13 | 32, false>(g, tm, pm, st, ai);
      case 4: return launch_t<BN, false, false, 13 | 32, true>(g, tm, pm, st, ai);
      case 5: return launch_t<BN, true, false, 13 | 32, true>(g, tm, pm, st, ai);
      case 6: return launch_t<BN, false, true, 13 | 32, true>(g, tm, pm, st, ai);
      default: return launch_t<BN, true, true, 13 | 32, true>(g, tm, pm, st, ai);
    }
  }
  const int key = (g->a_mn_major ? 1 : 0) | (g->b_mn_major ? 2 : 0) | ((mode | (w8 ? 8 : 0)) << 2) | (pc ? 64 : 0) |
                  (cl2 ? 128 : 0);
  switch (key) {
#define TOFU_CASE(AM, BMJ, O, P) \
  case ((AM) | ((BMJ) << 1) | ((O) << 2) | ((P) << 6)): \
    return launch_t<BN, (bool)(AM), (bool)(BMJ), O, (bool)(P)>(g, tm, pm, st, ai);
#define TOFU_CASE2(AM, BMJ, O) \
  case ((AM) | ((BMJ) << 1) | ((O) << 2) | 128): \
    return launch_t<BN, (bool)(AM), (bool)(BMJ), O, false, BN == 256>(g, tm, pm, st, ai);
#define TOFU_CASES2(O) TOFU_CASE2(0, 0, O) TOFU_CASE2(0, 1, O) TOFU_CASE2(1, 0, O) TOFU_CASE2(1, 1, O)
    TOFU_CASES2(0) TOFU_CASES2(1) TOFU_CASES2(2) TOFU_CASES2(3) TOFU_CASES2(5) TOFU_CASES2(8) TOFU_CASES2(11)
    TOFU_CASES2(13)
#undef TOFU_CASES2
#undef TOFU_CASE2
#define TOFU_CASES(O, P) TOFU_CASE(0, 0, O, P) TOFU_CASE(0, 1, O, P) TOFU_CASE(1, 0, O, P) TOFU_CASE(1, 1, O, P)
    TOFU_CASES(0, 0) TOFU_CASES(1, 0) TOFU_CASES(2, 0) TOFU_CASES(3, 0) TOFU_CASES(4, 0) TOFU_CASES(5, 0)
    TOFU_CASES(8, 0) TOFU_CASES(11, 0) TOFU_CASES(13, 0)
    TOFU_CASES(0, 1) TOFU_CASES(1, 1) TOFU_CASES(2, 1) TOFU_CASES(3, 1) TOFU_CASES(4, 1) TOFU_CASES(5, 1)
    TOFU_CASES(8, 1) TOFU_CASES(11, 1) TOFU_CASES(13, 1)
#undef TOFU_CASES
#undef TOFU_CASE
    default: return TOFU_ERR_ARG;
  }
}

// Split-K reduction: C = epilogue(sum_s WS[s]) in fixed split order (deterministic).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N,
                                                            void* C, int ldc, int mode, __nv_bfloat16* D, int ldd,
                                                            float s0, float s1) {
  pdl_trigger();
  pdl_wait();
  const int64_t plane = (int64_t)M * N;
  if (mode == 3 && N % 4 == 0 && ldc % 4 == 0 && ldd % 4 == 0 && !(reinterpret_cast<uintptr_t>(C) & 15) &&
      !(reinterpret_cast<uintptr_t>(D) & 7)) {  // vectorised: 4 elements (float4 momentum, 4 bf16 weights)
    const int64_t n4 = plane / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      float4 acc = reinterpret_cast<const float4*>(ws)[i];
      for (int s = 1; s < splits; ++s) {
        const float4 v = reinterpret_cast<const float4*>(ws + s * plane)[i];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      const int64_t m = (i * 4) / N, n = (i * 4) % N;
      float4* c = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + m * ldc + n);
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
    return;
  }
  if (mode == 3) {  // fused momentum-SGD on the reduced weight gradient (c_mode 3 with split-K)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
      float acc = ws[i];
      for (int s = 1; s < splits; ++s) acc += ws[s * plane + i];
      const int64_t m = i / N, n = i % N;
      float* c = reinterpret_cast<float*>(C) + m * ldc + n;
      const float mm = *c * s0 + acc;
      *c = mm;
      __nv_bfloat16* w = D + m * ldd + n;
      *w = __float2bfloat16_rn(__bfloat162float(*w) - mm * s1);
    }
    return;
  }
  const bool vec = (N % 4 == 0) && (ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  if (vec) {
    const int64_t n4 = plane / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      float4 acc = reinterpret_cast<const float4*>(ws)[i];
      for (int s = 1; s < splits; ++s) {
        const float4 v = reinterpret_cast<const float4*>(ws + s * plane)[i];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      const int64_t m = (i * 4) / N, n = (i * 4) % N;
      if (mode == 0) {
        __nv_bfloat162 a = __floats2bfloat162_rn(acc.x, acc.y), b = __floats2bfloat162_rn(acc.z, acc.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&a);
        u.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(C) + m * ldc + n) = u;
      } else {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + m * ldc + n);
        if (mode == 2) {
          const float4 o = *dst;
          acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
        }
        *dst = acc;
      }
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
      float acc = ws[i];
      for (int s = 1; s < splits; ++s) acc += ws[s * plane + i];
      const int64_t m = i / N, n = i % N;
      if (mode == 0) reinterpret_cast<__nv_bfloat16*>(C)[m * ldc + n] = __float2bfloat16_rn(acc);
      else if (mode == 1) reinterpret_cast<float*>(C)[m * ldc + n] = acc;
      else reinterpret_cast<float*>(C)[m * ldc + n] += acc;
    }
  }
}

static void* g_ws = nullptr;
static size_t g_ws_bytes = 0;
static std::mutex g_ws_mu;

// Measured (tools/gemm_major_bench.py, tools/sk_bench.py): pairs pay when both operands are MN-major (the
// weight-gradient GEMMs; 8192^3 1070 -> 1227 TF/s, 6272x4096x1024 1143 -> 1206) and lose 3-7% on several
// K-major shapes and on the memory-leaning fused-optimizer epilogue (configs[1], K = 512).
static bool cl2_auto(const tofu_gemm_args* g) { return g->a_mn_major && g->b_mn_major && g->K >= 2048; }

static int auto_splits(const tofu_gemm_args* g, int bn) {
  if (g->splits == 1 || g->ep) return 1;
  const int nk = (g->K + BK - 1) / BK;
  if (g->splits > 1) return g->splits < nk ? g->splits : nk;
  const int tiles = ((g->M + BM - 1) / BM) * ((g->N + bn - 1) / bn);
  if (tiles * 2 > g_num_sms || nk < 8) return 1;
  int sp = g_num_sms / tiles;
  const bool skinny = g->M <= 256 && g->K <= 8192;  // (see tofu_gemm_plan_tmaps: >= 8 k-blocks per split)
  if (sp > nk / (skinny ? 8 : 4)) sp = nk / (skinny ? 8 : 4);
  if (sp > 16) sp = 16;
  return sp < 2 ? 1 : sp;
}

}  // namespace tofu

using namespace tofu;

extern "C" int64_t tofu_sk_workspace_bytes(void) {
  if (encode_fn_init() != 0) return 0;
  return (int64_t)g_num_sms * (SK_SLOT_FLOATS * 4 + 4 * SK_FLAGS);
}

extern "C" int64_t tofu_gemm_workspace_bytes(const tofu_gemm_args* g) {
  return g->splits > 1 ? (int64_t)g->splits * g->M * g->N * 4 : 0;
}

// tmaps: 6 x CUtensorMap (A, B, C, D, split-K workspace, mask operand), 64-byte aligned, 768 bytes.  args->splits is
// in/out: 0 = choose (split-K when the output has too few tiles to fill the SMs), 1 = off, n = n splits.
extern "C" int tofu_gemm_plan_tmaps(tofu_gemm_args* g, void* tmaps, int* bn_out) {
  if (encode_fn_init() != 0) return TOFU_ERR_CUDA;
  if (!g || g->M < 0 || g->N < 0 || g->K < 0 || g->c_mode < 0 || g->c_mode > 3) return TOFU_ERR_ARG;
  if (g->ep && (g->c_mode != 0 || ((g->ep & 2) && !g->aux_add) || ((g->ep & 4) && !g->aux_mask) ||
                (reinterpret_cast<uintptr_t>(g->aux_add) & 15) || (reinterpret_cast<uintptr_t>(g->aux_mask) & 15)))
    return TOFU_ERR_ARG;
  if (g->c_mode == 3 && (!g->D || (g->ldd % 8))) return TOFU_ERR_ARG;
  // TMA: row pitch must be a multiple of 16 bytes, bases 16-byte aligned
  const int ce = g->c_mode == 0 ? 2 : 4;
  if ((g->lda % 8) || (g->ldb % 8) || ((g->ldc * ce) % 16) || (reinterpret_cast<uintptr_t>(g->A) & 15) ||
      (reinterpret_cast<uintptr_t>(g->B) & 15) || (reinterpret_cast<uintptr_t>(g->C) & 15) ||
      (reinterpret_cast<uintptr_t>(g->D) & 15))
    return TOFU_ERR_ALIGN;
  int bn = (g->bn == 128 || g->bn == 256) ? g->bn : (g->N <= 128 ? 128 : 256);
  {  // TOFU_EP_BN=128: 128-wide tiles for the fused element-wise epilogues (A/B switch)
    static const int ep_bn = [] {
      const char* e = getenv("TOFU_EP_BN");
      return e ? atoi(e) : 0;
    }();
    if (ep_bn == 128 && g->bn == 0 && g->ep) bn = 128;
  }
  // (measured: 128-wide tiles do not recover the last-wave loss of 196-tile shapes, they run ~25% slower)
  // Few-tile outputs (256-wide tiles fill at most half the SMs) that 128-wide tiles fill more than half of,
  // e.g. the LSTM's per-timestep [128 x 16384] gate GEMMs, which stream their 134 MB weight from HBM: 128-wide
  // tiles instead of split-K.  Measured on configs[2]: forward gate GEMMs 6.78 -> 5.62 ms, recurrent backward
  // 6.54 -> 6.30 ms per step (stream-K instead: 7.48 / 8.19 ms); outputs with fewer tiles (WResNet stage-0
  // weight gradients, K = 100352 pixels; FC sub-GEMMs at k = 8) keep split-K, which measured faster there.
  // TOFU_GEMM_FEW=0 keeps 256-wide tiles + split-K everywhere, 2 = stream-K.
  static const int few = [] {
    const char* e = getenv("TOFU_GEMM_FEW");
    return e ? atoi(e) : 1;
  }();
  // Skinny (M <= 256) few-tile launches with K <= 8192 — a rank's per-timestep recurrent GEMMs under an
  // 8-way plan, [128 x 2048 x 4096] / [128 x 4096 x 2048] — take 128-wide tiles AND split-K with >= 8 k-blocks
  // per split (auto_splits): device time incl. the reduction (graph replay, tools/small_gemm_sweep.py)
  // 13.0 -> 9.9 us and 11.1 -> 9.4 us against 256-wide tiles with 16 / 8 splits.
  const bool skinny = g->M <= 256 && g->K <= 8192;
  if (few && g->bn == 0 && g->splits == 0 && !g->ep && bn == 256 &&
      2 * ((g->M + BM - 1) / BM) * ((g->N + 255) / 256) <= g_num_sms &&
      (few != 1 || skinny || 2 * ((g->M + BM - 1) / BM) * ((g->N + 127) / 128) > g_num_sms)) {
    if (few == 1) bn = 128;
    if (few == 2 && g->sk_ws) g->splits = -1;
  }
  // Few-tile launches with a fused element-wise epilogue (split-K cannot carry those epilogues): stream-K would
  // spread the K loop over all SMs (a rank's sub-op under an 8-way plan, e.g. [1568 x 2048] with K = 1024: 104
  // tiles).  Measured slower (WResNet-152-4 on 8 virtual ranks 101.2 -> 104.7 ms: the partial round trip and
  // the finishers' waits cost more than the idle SMs), so off unless TOFU_GEMM_SK_EP=1.
  {
    static const bool sk_ep = [] {
      const char* e = getenv("TOFU_GEMM_SK_EP");
      return e && e[0] == '1';
    }();
    const int tiles_dp = ((g->M + BM - 1) / BM) * ((g->N + bn - 1) / bn);
    if (sk_ep && g->splits == 0 && g->ep && g->sk_ws && !g->a_pieces && !g->b_pieces && g->max_ctas == 0 &&
        sk_enabled() && tiles_dp * 4 <= 3 * g_num_sms && (g->K + BK - 1) / BK >= 8)
      g->splits = -1;
  }
  const bool stream_k = g->splits == -1;
  g->splits = stream_k ? 1 : auto_splits(g, bn);
  // cluster pairs sharing B (see the kernel's CL2): data-parallel launches of 256-wide tiles with at least
  // two m tiles; TOFU_CL2=0 turns them off, 1 forces them wherever possible (A/B measurements)
  {
    static const int env = [] {
      const char* e = getenv("TOFU_CL2");
      return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
    }();
    const int req = g->cl2 == 1 || g->cl2 == 3 ? 0 : g->cl2;  // (a re-plan of planned args decides afresh)
    const bool ok = req != -1 && env != 0 && bn == 256 && g->splits == 1 && !stream_k && !g->a_pieces &&
                    !g->b_pieces && g->max_ctas == 0 && g->M > BM;
    static const int env2 = [] {  // 2-CTA MMA pairs: TOFU_C2=1 forces them where eligible (A/B measurements)
      const char* e = getenv("TOFU_C2");
      return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
    }();
    // 2-CTA MMA pairs for compute-leaning launches (the 4-warp epilogue ones); measured (tools/gemm_major_bench.py,
    // tools/sk_bench.py): 8192^3 1182 -> 1294 TF/s (K-major), 1152 -> 1398 (both MN-major), the configs[1]
    // forward 62 -> 57 us; the memory-leaning fused epilogues lose up to 1.7x with 4 warps, so they keep W8
    static const bool c2w8 = [] {  // TOFU_C2W8=1: 2-CTA pairs also with the 8-warp epilogue (A/B switch)
      const char* e = getenv("TOFU_C2W8");
      return e && e[0] == '1';
    }();
    // (8-warp epilogues pair too from K = 1024: measured with the issue-lean epilogue, tools/ep_stream_bench.py,
    // [100352 x 256 x 1024] + mask 66.2 -> 60.7 us, [6272 x 4096 x 1024] + add + mask 60.8 -> 54.8 us; shorter K
    // loses: K = 512 74.4 -> 78.7 us, K = 256 112 -> 137 us)
    static const int c2w8_k = [] {  // TOFU_C2W8_K: smallest K at which 8-warp epilogues pair (A/B)
      const char* e = getenv("TOFU_C2W8_K");
      return e ? atoi(e) : 1024;
    }();
    const bool c2 =
        ok && (req == 4 || (req == 0 && env2 != 0 && (env2 == 1 || c2w8 || !wants_w8(g) || g->K >= c2w8_k)));
    g->cl2 = c2 ? 3 : ok && (env == 1 || req == 2 || cl2_auto(g)) ? 1 : 0;
  }
  CUtensorMap* tm = reinterpret_cast<CUtensorMap*>(tmaps);
  const CUtensorMapDataType BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const auto SW128 = CU_TENSOR_MAP_SWIZZLE_128B, SW64 = CU_TENSOR_MAP_SWIZZLE_64B;
  int r;
  if (!g->a_mn_major) r = make_tmap(&tm[0], g->A, BF, 2, g->K, g->M, g->lda, 64, BM, SW128);
  else r = make_tmap(&tm[0], g->A, BF, 2, g->M, g->K, g->lda, 64, 64, SW128);
  if (r) return TOFU_ERR_CUDA;
  if (!g->b_mn_major) r = make_tmap(&tm[1], g->B, BF, 2, g->K, g->N, g->ldb, 64, g->cl2 ? bn / 2 : bn, SW128);
  else r = make_tmap(&tm[1], g->B, BF, 2, g->N, g->K, g->ldb, 64, 64, SW128);
  if (r) return TOFU_ERR_CUDA;
  if (g->c_mode == 0) r = make_tmap(&tm[2], g->C, BF, 2, g->N, g->M, g->ldc, 32, 32, SW64);
  else r = make_tmap(&tm[2], g->C, F32, 4, g->N, g->M, g->ldc, 32, 32, SW128);
  if (r) return TOFU_ERR_CUDA;
  if (g->c_mode == 3) r = make_tmap(&tm[3], g->D, BF, 2, g->N, g->M, g->ldd, 32, 32, SW64);
  else if (g->ep & 2) r = make_tmap(&tm[3], g->aux_add, BF, 2, g->N, g->M, g->ldc, 32, 32, SW64);
  else tm[3] = tm[2];
  if (r) return TOFU_ERR_CUDA;
  if (g->ep & 4) r = make_tmap(&tm[5], g->aux_mask, BF, 2, g->N, g->M, g->ldc, 32, 32, SW64);
  else tm[5] = tm[2];
  if (r) return TOFU_ERR_CUDA;
  if (g->splits > 1) {
    void* ws = g->ws;
    if (!ws) {  // library-owned workspace (not CUDA-graph safe; the executor passes its own)
      std::lock_guard<std::mutex> lk(g_ws_mu);
      const size_t need = (size_t)tofu_gemm_workspace_bytes(g);
      if (need > g_ws_bytes) {
        if (g_ws) cudaFree(g_ws);
        if (cudaMalloc(&g_ws, need) != cudaSuccess) return TOFU_ERR_CUDA;
        g_ws_bytes = need;
      }
      ws = g_ws;
      g->ws = ws;
    }
    cuuint64_t dims[3] = {(cuuint64_t)g->N, (cuuint64_t)g->M, (cuuint64_t)g->splits};
    cuuint64_t strides[2] = {(cuuint64_t)g->N * 4, (cuuint64_t)g->N * g->M * 4};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if ((g->N * 4) % 16) return TOFU_ERR_ALIGN;
    if (g_encode(&tm[4], F32, 3, ws, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, SW128,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return TOFU_ERR_CUDA;
  }
  // piecewise operands: one map per piece (tm[6 + i] for A, tm[6 + TOFU_MAX_PIECES + i] for B)
  for (int op = 0; op < 2; ++op) {
    const tofu_operand_pieces* pc = op == 0 ? g->a_pieces : g->b_pieces;
    if (!pc) continue;
    const bool mn = op == 0 ? g->a_mn_major : g->b_mn_major;
    const int mdim = op == 0 ? g->M : g->N;  // the operand's M / N extent
    const int ext = pc->dim == 0 ? mdim : g->K;
    const int gran = pc->dim == 1 ? BK : (op == 0 ? BM : bn);
    if (pc->n < 1 || pc->n > TOFU_MAX_PIECES || pc->dim < 0 || pc->dim > 1 || pc->start[0] != 0) return TOFU_ERR_ARG;
    for (int i = 0; i < pc->n; ++i) {
      const int lo = pc->start[i], hi = i + 1 < pc->n ? pc->start[i + 1] : ext;
      if (hi <= lo || lo % gran || (reinterpret_cast<uintptr_t>(pc->ptr[i]) & 15) || pc->ld[i] % 8 || pc->ld[i] <= 0)
        return TOFU_ERR_ALIGN;
      const uint64_t len = hi - lo;
      // (inner, outer) extents of the piece: K-major = (K, M|N), MN-major = (M|N, K)
      const uint64_t kx = pc->dim == 1 ? len : (uint64_t)g->K, mx = pc->dim == 0 ? len : (uint64_t)mdim;
      CUtensorMap* t = &tm[6 + op * TOFU_MAX_PIECES + i];
      const int rr = !mn ? make_tmap(t, pc->ptr[i], BF, 2, kx, mx, pc->ld[i], 64, op == 0 ? BM : bn, SW128)
                         : make_tmap(t, pc->ptr[i], BF, 2, mx, kx, pc->ld[i], 64, 64, SW128);
      if (rr) return TOFU_ERR_CUDA;
    }
  }
  if (stream_k) g->splits = -1;  // kept as the launch's stream-K request
  *bn_out = bn;
  return TOFU_OK;
}

extern "C" int tofu_gemm_launch_planned(const tofu_gemm_args* g, const void* tmaps, int bn, void* stream) {
  if (g->M == 0 || g->N == 0) return TOFU_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (g->K == 0) {
    if (g->c_mode == 2) return TOFU_OK;
    if (g->c_mode == 3) return TOFU_ERR_ARG;
    const size_t es = g->c_mode == 0 ? 2 : 4;
    return cudaMemset2DAsync(g->C, (size_t)g->ldc * es, 0, (size_t)g->N * es, g->M, st) == cudaSuccess
               ? TOFU_OK
               : TOFU_ERR_CUDA;
  }
  const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(tmaps);
  PieceMaps pmv;
  const PieceMaps* pm = nullptr;
  if (g->a_pieces || g->b_pieces) {
    std::memset(&pmv, 0, sizeof pmv);
    if (const tofu_operand_pieces* pc = g->a_pieces) {
      pmv.na = pc->n;
      pmv.a_dim = pc->dim;
      for (int i = 0; i < pc->n; ++i) {
        pmv.a_map[i] = tm[6 + i];
        pmv.a_start[i] = pc->start[i];
      }
    }
    if (const tofu_operand_pieces* pc = g->b_pieces) {
      pmv.nb = pc->n;
      pmv.b_dim = pc->dim;
      for (int i = 0; i < pc->n; ++i) {
        pmv.b_map[i] = tm[6 + TOFU_MAX_PIECES + i];
        pmv.b_start[i] = pc->start[i];
      }
    }
    pm = &pmv;
  }
  if (g->splits > 1) {
    // partial products into the workspace planes, then one ordered reduction into C
    const CUtensorMap tw[6] = {tm[0], tm[1], tm[4], tm[4], tm[4], tm[4]};
    tofu_gemm_args p = *g;
    p.c_mode = 4;
    int rc = bn == 256 ? dispatch_bn<256>(&p, tw, pm, st) : dispatch_bn<128>(&p, tw, pm, st);
    if (rc || g->defer_reduce) return rc;  // (defer_reduce: the caller reduces the planes)
    const int64_t n = (int64_t)g->M * g->N / 4 + 1;
    int blocks = (int)((n + 255) / 256);
    if (blocks > g_num_sms * 8) blocks = g_num_sms * 8;
    launch_k(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st, 1, reinterpret_cast<const float*>(g->ws), g->splits, g->M, g->N, g->C,
                                                 g->ldc, g->c_mode, reinterpret_cast<__nv_bfloat16*>(g->D), g->ldd,
                                                 g->s0, g->s1);
    return cudaGetLastError() == cudaSuccess ? TOFU_OK : TOFU_ERR_CUDA;
  }
  return bn == 256 ? dispatch_bn<256>(g, tm, pm, st) : dispatch_bn<128>(g, tm, pm, st);
}

extern "C" int tofu_gemm_bf16(const tofu_gemm_args* g, void* stream) {
  alignas(64) CUtensorMap tm[TOFU_GEMM_TMAPS];
  tofu_gemm_args a = *g;
  int bn = 0;
  int r = tofu_gemm_plan_tmaps(&a, tm, &bn);
  if (r) return r;
  return tofu_gemm_launch_planned(&a, tm, bn, stream);
}
