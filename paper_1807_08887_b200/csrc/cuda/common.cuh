// Shared device helpers for the sm_100a kernels (PTX wrappers).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace tofu {

// ---------------------------------------------------------------- programmatic dependent launch (PDL)
// Every libtofu kernel is launched with programmatic stream serialization (launch_k below) and calls
// pdl_trigger(); pdl_wait() once its prologue (barrier init, TMEM allocation, tensor-map prefetch) is done and
// before it touches global memory a predecessor writes or reads: the next kernel's launch and prologue then
// overlap the current kernel's tail instead of following its completion.  griddepcontrol.wait returns once
// every prerequisite grid has completed and its memory is visible (a no-op when launched without PDL).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {  // TOFU_PDL=0 launches every kernel fully serialised (A/B switch)
  static const bool on = [] {
    const char* e = std::getenv("TOFU_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// cudaLaunchKernelEx with PDL (and an optional cluster dimension along x).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// TOFU_MBAR_HINT (compile time, ns): suspend-time hint of the potentially-blocking try_wait (0 = none)
#ifndef TOFU_MBAR_HINT
#define TOFU_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  const uint32_t a = smem_u32(bar);
  do {
#if TOFU_MBAR_HINT > 0
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(phase), "n"(TOFU_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
#endif
  } while (!done);
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// im2col load of an NHWC tensor (cuTensorMapEncodeIm2col, rank 4: c, w, h, n): pixelsPerColumn pixels
// traversed from (w, h, n) in W, H, N order inside the map's bounding box, each reading channelsPerPixel
// channels from c at the pixel shifted by (off_w, off_h) (outside the tensor: zero)
__device__ __forceinline__ void tma_load_im2col_4d(void* smem_dst, const void* tmap, uint64_t* bar, int c, int w,
                                                   int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h)
      : "memory");
}
// ... multicast to every CTA of ctaMask (same smem offset; each CTA's barrier at `bar`'s offset)
__device__ __forceinline__ void tma_load_im2col_4d_mc(void* smem_dst, const void* tmap, uint64_t* bar, int c, int w,
                                                      int h, int n, uint16_t off_w, uint16_t off_h, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8}, %9;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* smem_src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* smem_src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// make generic-proxy smem writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- cp.async (gathered operands)
// 16-byte global -> shared copy; src_bytes = 0 zero-fills the destination (an access outside the tensor)
__device__ __forceinline__ void cp_async_16(void* smem_dst, const void* gmem_src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// arrive on an mbarrier once all prior cp.async of this thread have landed (counts toward the barrier's
// expected arrivals: .noinc)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// barrier among a subset of warps (id 1..15, n = thread count, a multiple of 32)
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 inputs, fp32 accumulate)
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// commit arriving on the barrier at this smem offset in every CTA of ctaMask (cluster multicast)
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// ---------------------------------------------------------------- 2-CTA (cta_group::2) MMA pairs
__device__ __forceinline__ void tmem_alloc2(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[tmem, both CTAs] (+)= A[smem, rows split over the pair] * B[smem, N split over the pair]; leader only
__device__ __forceinline__ void umma_bf16_2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// shared::cluster address of `p`'s counterpart in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-D TMA load into this CTA's smem whose completion is counted on the barrier at `bar_cluster` (a
// shared::cluster address, e.g. the pair leader's barrier)
__device__ __forceinline__ void tma_load_2d_2sm(void* smem_dst, const void* tmap, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

// im2col load (as tma_load_im2col_4d) whose completion is counted on the pair leader's barrier
__device__ __forceinline__ void tma_load_im2col_4d_2sm(void* smem_dst, const void* tmap, uint32_t bar_cluster, int c,
                                                       int w, int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h)
      : "memory");
}

// ---------------------------------------------------------------- clusters
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-D TMA load multicast to every CTA of ctaMask (same smem offset, each CTA's barrier at `bar`'s offset)
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp gets lane (base+t), columns [c, c+32)
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor (SM100 version 1), SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: bf16 x bf16 -> fp32, M x N, majorness.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                       // D format F32
         | (1u << 7)                     // A format BF16
         | (1u << 10)                    // B format BF16
         | ((uint32_t)a_mn_major << 15)  // A major
         | ((uint32_t)b_mn_major << 16)  // B major
         | ((uint32_t)(N >> 3) << 17)    // N >> 3
         | ((uint32_t)(M >> 4) << 24);   // M >> 4
}

// ---------------------------------------------------------------- persistent work list (data-parallel + stream-K)
// The tcgen05 kernels (gemm_tcgen05.cu, conv_tcgen05.cu) run one CTA per SM over a list of segments, each an
// output tile and a k-block range.  The first dp_units = (ntiles - sk_tiles) * splits units are data-parallel:
// unit u goes to CTA u % grid (tile u / splits, split plane u % splits).  The remaining sk_tiles tiles are
// stream-K: their sk_tiles * nk k-block iterations, tile-major, are divided evenly over the grid, CTA b taking
// [bound(b), bound(b+1)).  A tile cut between CTAs is finished by the CTA holding its k-block 0, which
// processes that piece LAST in its list; the CTAs holding the rest of the tile process it FIRST, write their
// fp32 partial to their slot of the stream-K workspace and raise a flag.  The finisher adds the partials in
// CTA order (deterministic for a given shape) before its epilogue, then lowers the flags again (the workspace
// flags are zero between launches).  This removes the wave-quantisation tail of shapes whose tile count is
// not a multiple of the SM count (e.g. the 196 tiles of a WResNet stage-2 3x3 convolution on 148 SMs).
// The host guarantees sk_tiles * nk >= grid (every CTA has a non-empty range) and co-residency (grid <= #SMs,
// one CTA per SM).
struct WorkList {
  int nk, splits, grid, cta, sk_tile0, n_dp, n_sk, t0;
  int64_t sk_iters, lo, hi;
  // cluster pairs (gemm_tcgen05.cu CL2): the two CTAs of a cluster take vertically adjacent tiles (m tiles 2p,
  // 2p+1) of the same n tile, so they share (multicast) the B tile; pair units round-robin over the clusters
  int pairs = 0, tiles_n = 1, rank = 0;
  // raster 1: units walk m fastest (column-major over the tile grid), so one wave covers every m tile of a few
  // n columns — A (M x K) stays resident in L2 while B streams once; used when B is the larger operand (N > M)
  int raster = 0, tiles_m = 1;
  __device__ __forceinline__ void init_pairs(int tiles_m, int tiles_n_, int nk_, int rank_, int cid, int ncl) {
    nk = nk_;
    splits = 1;
    pairs = 1;
    tiles_n = tiles_n_;
    this->tiles_m = tiles_m;
    rank = rank_;
    grid = ncl;
    cta = cid;
    const int units = ((tiles_m + 1) / 2) * tiles_n;
    n_dp = cid < units ? (units - cid + ncl - 1) / ncl : 0;
    n_sk = 0;
    sk_tile0 = 0;
  }
  __device__ __forceinline__ void init(int ntiles, int nk_, int splits_, int sk_tiles) {
    nk = nk_;
    splits = splits_;
    grid = gridDim.x;
    cta = blockIdx.x;
    sk_tile0 = ntiles - sk_tiles;
    const int dp_units = sk_tile0 * splits;
    n_dp = cta < dp_units ? (dp_units - cta + grid - 1) / grid : 0;
    sk_iters = (int64_t)sk_tiles * nk;
    lo = bound(cta);
    hi = bound(cta + 1);
    t0 = (int)(lo / (nk > 0 ? nk : 1));
    n_sk = hi > lo ? (int)((hi - 1) / nk) - t0 + 1 : 0;
  }
  __device__ __forceinline__ int64_t bound(int c) const { return sk_iters * c / grid; }
  __device__ __forceinline__ int count() const { return n_dp + n_sk; }
  // segment i: tile, k-blocks [kb0, kb1), split plane; partial = a leading piece of a cut tile (writes its
  // fp32 partial to the workspace instead of the epilogue's store)
  __device__ __forceinline__ void seg(int i, int& tile, int& kb0, int& kb1, int& split, bool& partial) const {
    if (pairs) {
      const int u = cta + i * grid;
      int mp, nn;
      if (raster) {
        const int prow = (tiles_m + 1) / 2;
        nn = u / prow;
        mp = u - nn * prow;
      } else {
        mp = u / tiles_n;
        nn = u - mp * tiles_n;
      }
      tile = (2 * mp + rank) * tiles_n + nn;
      split = kb0 = 0;
      kb1 = nk;
      partial = false;
      return;
    }
    if (i < n_dp) {
      const int u = cta + i * grid;
      partial = false;
      if (splits == 1) {  // the common case: no divisions (raster 1: one)
        if (raster) {
          const int nn = u / tiles_m;
          tile = (u - nn * tiles_m) * tiles_n + nn;
        } else {
          tile = u;
        }
        split = kb0 = 0;
        kb1 = nk;
        return;
      }
      tile = u / splits;
      split = u - tile * splits;
      kb0 = (int)((int64_t)split * nk / splits);
      kb1 = (int)((int64_t)(split + 1) * nk / splits);
      partial = false;
      return;
    }
    const int ts = t0 + (i - n_dp);
    const int64_t ts0 = (int64_t)ts * nk;
    tile = sk_tile0 + ts;
    split = 0;
    kb0 = (int)((lo > ts0 ? lo : ts0) - ts0);
    kb1 = (int)((hi < ts0 + nk ? hi : ts0 + nk) - ts0);
    partial = kb0 > 0;
  }
  // finisher of stream-K tile `tile` (the segment holding k-block 0): contributors are CTAs cta+1 .. last-1
  __device__ __forceinline__ int contrib_end(int tile) const {
    if (pairs) return 0;  // (no stream-K pieces; callers loop from blockIdx.x + 1)
    if (tile < sk_tile0) return cta + 1;
    const int64_t te = (int64_t)(tile - sk_tile0 + 1) * nk;
    int c = cta + 1;
    while (c < grid && bound(c) < te) ++c;
    return c;
  }
};

// stream-K workspace: [grid slots][BM x 256 fp32 partial] then int flags [grid][SK_FLAGS] (one per epilogue warp)
constexpr int SK_SLOT_FLOATS = 128 * 256;
constexpr int SK_FLAGS = 8;
__device__ __forceinline__ float4* sk_slot(void* ws, int c) {
  return reinterpret_cast<float4*>(ws) + (int64_t)c * (SK_SLOT_FLOATS / 4);
}
__device__ __forceinline__ int* sk_flag(void* ws, int grid, int c, int q) {
  return reinterpret_cast<int*>(reinterpret_cast<float*>(ws) + (int64_t)grid * SK_SLOT_FLOATS) + c * SK_FLAGS + q;
}
// epilogue warp q, chunk ch (32 columns) of a partial: coalesced float4 layout [q][ch][8][32 lanes]
__device__ __forceinline__ void sk_write_chunk(float4* slot, int q, int nch, int ch, int lane, const uint32_t (&r)[32]) {
  float4* p = slot + ((int64_t)(q * nch + ch) * 8) * 32 + lane;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    __stcg(p + j * 32, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
}
__device__ __forceinline__ void sk_add_chunk(const float4* slot, int q, int nch, int ch, int lane, uint32_t (&r)[32]) {
  const float4* p = slot + ((int64_t)(q * nch + ch) * 8) * 32 + lane;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 v = __ldcg(p + j * 32);
    r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + v.x);
    r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + v.y);
    r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + v.z);
    r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + v.w);
  }
}
__device__ __forceinline__ void sk_signal(int* flag) {  // after this warp's partial stores (all lanes fenced)
  __threadfence();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(1) : "memory");
}
__device__ __forceinline__ void sk_wait(int* flag) {
  int v = 0;
  do {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
  } while (v == 0);
}

}  // namespace tofu
