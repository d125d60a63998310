// tcgen05 / TMEM / TMA TF32 GEMM for sm_100a.
//
// Replaces np.dot -> OpenBLAS sgemm for large float32 problems (reference
// pkg/src/texpr/ops/linalg.py:42-62).  C[M,N] = A[M,K] . B[K,N] (+ epilogue).
//
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: one elected lane streams A/B K-slices into a
//               4-stage shared-memory ring (128 B swizzle), completion tracked
//               by mbarrier transaction counts.
//   warp 1      TMEM owner + MMA issuer: allocates 512 TMEM columns (two
//               128x256 fp32 accumulators), one lane issues
//               tcgen05.mma.cta_group::1.kind::tf32 (128x256x8 per instruction)
//               and tcgen05.commit's smem slots back to the producer and full
//               accumulators to the epilogue.
//   warps 2-5   epilogue: tcgen05.ld 32x32b rows out of TMEM, fused epilogue
//               (bias / bias+tanh / *(1-h^2)), 128-bit global stores; the
//               second accumulator lets tile i+1's MMAs overlap tile i's
//               epilogue.
// Operand transposes (DimShuffle views) are not copied: a K-contiguous
// operand uses the K-major UMMA descriptor, an M/N-contiguous one the
// MN-major descriptor (legal for TF32), with the matching TMA box shape.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "tx_common.h"
#include "tx_gemm.h"

namespace tx {
namespace {

// Per-CTA tile: BM rows (one TMEM lane each) x BN accumulator columns.  With
// CG = 2 a CTA pair computes a 256 x BN tile with one cta_group::2 MMA
// stream: each CTA stages its 128 rows of A and half of B's columns, the
// leader issues, TMEM holds each CTA's own 128 rows.
constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 32;  // 32 fp32 = 128 B = one swizzle span
constexpr int EPI_WARPS = 8;  // two warps per TMEM lane quarter, each owning half the columns
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 16;

template <int CG>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;              // 16 KB
  static constexpr int B_BYTES = (BN / CG) * BK * 4;       // 32 KB (CG=1) / 16 KB (CG=2)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = CG == 1 ? 4 : 5;
  static constexpr size_t RING = (size_t)STAGES * STAGE_BYTES;
  // epilogue staging: one [32 rows x 32 cols] fp32 tile (4 KB, 128B-swizzled)
  // per epilogue warp, drained by TMA stores
  static constexpr size_t STAGING = (size_t)EPI_WARPS * 4096;
  // CG = 2 also stages the [M,N] epilogue operand (x(1-h^2), x aux) per warp
  // with TMA loads (coalesced; the per-row register loads are 32 rows wide)
  static constexpr size_t AUX_STAGING = CG == 2 ? (size_t)EPI_WARPS * 4096 : 0;
  static constexpr size_t SMEM = 1024 + RING + STAGING + AUX_STAGING + 256;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// 2-SM load: executed by both CTAs of the pair; the transaction bytes land on
// the LEADER's barrier (peer bit of the shared::cluster address cleared).
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}

// 3-D box for an MN-major operand tile: {32 MN, BK, MN-blocks} lands in smem
// as consecutive 4 KB [32 k][32 mn] blocks -- one TMA instruction per operand
// per stage instead of one per 32-wide MN block.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// one 2-D box landing at the same shared-memory offset in every CTA of `mask`
// (each CTA's own barrier at `bar`'s offset counts the bytes)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar) & kPeerMask), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// smem -> global tile store (bulk async group of the issuing thread)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)map),
               "r"(su32(src)), "r"(c0), "r"(c1)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"((uint64_t)map),
               "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the leader CTA's copy of a barrier
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(su32(b) & kPeerMask) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor (sm100 "version 1").  layout: 2 = SWIZZLE_128B
// (K-major operands: 8-row x 128 B atoms), 1 = SWIZZLE_128B_BASE32B (the only
// MN-major layout for 32-bit types: 128 B rows swizzled in 32 B granules,
// 4-row / 512 B atoms).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

template <int CG>
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}

// tcgen05.commit: arrive (once) on a barrier when all prior MMAs of this
// thread complete; CG = 2 multicasts the arrive to both CTAs of the pair.
// single-CTA MMAs done: arrive on the barrier at `bar`'s offset in every CTA of `mask`
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   su32(bar)),
               "h"(mask)
               : "memory");
}
template <int CG>
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
  } else {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            su32(bar)),
        "h"(mask)
        : "memory");
  }
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 8 TMEM columns of this warp's 32 lanes (the promoted-accumulation drains:
// the running sums already hold 128 registers per thread)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcParams {
  float* C;
  int64_t ldc;
  int M, N, K;
  int a_mn, b_mn;  // 1 = operand is MN-major in memory
  int a_3d, b_3d;  // MN-major operand loaded with one 3-D box per stage
  int a_lim, b_lim;  // 3-D boxes cover MN < lim (whole 32-blocks); tiles reaching past it use the edge maps
  int splits;       // split-K factor: work items are (tile, split); partial tiles go to a workspace
  int kbs;          // k-blocks per split
  int streamk;      // stream-K: cluster c owns the flat (tile, k-block) units [c*U/NC, (c+1)*U/NC)
  int num_kb;       // k-blocks per tile
  int nclusters;    // clusters of the launch (stream-K partition)
  int bn;           // N tile of this launch (<= BN, multiple of 32): chosen per shape against wave quantisation
  int stage_tx;     // TMA bytes landing per stage on the leader's barrier
  // implicit-GEMM convolution (stride 1; CG = 1): A rows are output pixels,
  // fetched per k-block (filter tap u, v; 32-channel block) as ONE 4-D TMA box
  // {32 c, Q, RB rows, 1 image} of a zero-padded NHWC input -- no patch matrix
  int conv;
  int cv_cb;        // 32-channel blocks per tap
  int cv_kw;        // filter width
  int cv_P, cv_Q;   // output rows / columns per image
  int cv_RB;        // output rows per M tile (RB * Q <= 128)
  int cv_pb;        // M tiles per image, ceil(P / RB)
  int cv_nchw;      // store C as [N, K, P, Q] (per output channel, a tile's pixels are one contiguous run)
  int kpack;        // k-blocks per ring stage (conv, bn <= 64: 2 -- A0 | A1 | B0 | B1 in one 48 KB stage,
                    // twice the loads in flight; else 1)
  int mcast;        // CG = 1 only: clusters of `mcast` CTAs along N sharing one A panel (MN-major A), each
                    // loading 1/mcast of its 32-row atoms and multicasting them to all (1 = off)
  int group_m;      // M-tiles per raster group (operand panels shared in L2 by concurrently running tiles)
  int dbg_nostore;  // diagnostics only (TX_GEMM_DBG_NOSTORE): epilogue drains TMEM without storing
  int tma_store;    // C written by TMA tile stores from swizzled smem staging
  int tma_aux;      // [M,N] epilogue operand read by TMA tile loads (CG = 2)
  int num_m, num_n, num_tiles;
  float* colsum;    // optional: per-32-row-block column sums of the stored C, [ceil(M/32)][N]
  int promo;        // PROMO kernels: k-blocks per TMEM accumulation chunk ...
  int promo_first;  // ... after a first chunk of k-blocks [0, promo_first)
  Epi<float> epi;
};

// end of the accumulation chunk that starts at k-block kb (segment end kb1)
__device__ __forceinline__ int chunk_end(const TcParams& p, int kb, int kb1) {
  const int e = kb < p.promo_first ? p.promo_first
                                   : p.promo_first + ((kb - p.promo_first) / p.promo + 1) * p.promo;
  return min(e, kb1);
}

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int group_m, int& mb, int& nb) {
  const int per_group = group_m * num_n;
  const int g = t / per_group;
  const int first = g * group_m;
  const int gsz = min(num_m - first, group_m);
  const int r = t - g * per_group;
  mb = first + r % gsz;
  nb = r / gsz;
}

// One unit of work of a CTA (pair): k-blocks [kb0, kb1) of one output tile.
// `full` = the segment covers the whole K of the tile (store C with the
// epilogue); otherwise the raw partial goes to workspace slot `piece`.
struct Seg {
  int t, kb0, kb1, piece, full;
};

// Stream-K is hybrid: the floor(tiles / clusters) full waves go round robin
// (whole tiles, so concurrently running tiles stay adjacent in the grouped
// raster and share operand panels in L2); only the R remainder tiles are cut
// into the flat (tile, k-block) sequence, cluster c taking units
// [c*U2/NC, (c+1)*U2/NC) of U2 = R * num_kb.
// owner cluster of remainder unit u under that partition
__device__ __forceinline__ int sk_owner(int64_t u, int64_t U, int NC) {
  int c = (int)((u * NC) / U);
  while (c + 1 < NC && ((int64_t)(c + 1) * U) / NC <= u) ++c;
  while (c > 0 && ((int64_t)c * U) / NC > u) --c;
  return c;
}

__device__ __forceinline__ int64_t seg_begin(const TcParams& p, int c) {
  if (!p.streamk) return c;
  const int W = p.num_tiles / p.nclusters;
  if (W > 0) return 0;
  const int64_t U2 = (int64_t)(p.num_tiles - W * p.nclusters) * p.num_kb;
  return W + ((int64_t)c * U2) / p.nclusters;
}

// every role of the CTA walks the same sequence of segments
__device__ __forceinline__ bool seg_next(const TcParams& p, int c, int64_t& cur, Seg& s) {
  if (!p.streamk) {  // round robin over (tile, split) items
    if (cur >= (int64_t)p.num_tiles * p.splits) return false;
    s.t = (int)(cur % p.num_tiles);
    const int split = (int)(cur / p.num_tiles);
    s.kb0 = split * p.kbs;
    s.kb1 = min(p.num_kb, s.kb0 + p.kbs);
    s.piece = split;
    s.full = p.splits == 1;
    cur += p.nclusters;
    return true;
  }
  const int NC = p.nclusters;
  const int W = p.num_tiles / NC;
  const int base = W * NC;
  const int64_t U2 = (int64_t)(p.num_tiles - base) * p.num_kb;
  if (cur < W) {  // full-wave tile
    s.t = c + (int)cur * NC;
    s.kb0 = 0;
    s.kb1 = p.num_kb;
    s.piece = 0;
    s.full = 1;
    ++cur;
    if (cur == W) cur = W + ((int64_t)c * U2) / NC;
    return true;
  }
  const int64_t u = cur - W, u1 = ((int64_t)(c + 1) * U2) / NC;
  if (u >= u1) return false;
  const int rt = (int)(u / p.num_kb);
  s.t = base + rt;
  s.kb0 = (int)(u - (int64_t)rt * p.num_kb);
  s.kb1 = (int)min((int64_t)p.num_kb, s.kb0 + (u1 - u));
  s.piece = c - sk_owner((int64_t)rt * p.num_kb, U2, NC);
  s.full = s.kb0 == 0 && s.kb1 == p.num_kb;
  cur += s.kb1 - s.kb0;
  return true;
}

// PROMO: accumulation promotion for the fp32-equivalent (3xTF32) mode.  The
// tensor core adds each MMA's products into the fp32 TMEM accumulator with
// round-toward-zero (measured: a bias of ~2^-24 |C| per instruction, growing
// with K).  With PROMO the MMA warp restarts the accumulator at chunk
// boundaries (chunk_end: one first chunk of p.promo_first k-blocks -- the
// small cross terms, whose sum is ~2^-11 |C| and needs no promotion -- then
// every p.promo k-blocks), cycling four 128-column TMEM buffers, and the
// epilogue warps add each chunk into per-thread fp32 registers with
// round-to-nearest: the round-toward-zero error is bounded by one short
// chunk, not the whole K.
// Epi::apply for the ragged / strided edge columns, kept out of line: its
// kind switch inlined into every 32-wide unrolled loop multiplies the
// kernel's code size (instruction-cache misses dominate a small GEMM's
// epilogue).
__device__ __noinline__ float epi_apply_edge(const Epi<float>& E, float v, int row, int n) { return E.apply(v, row, n); }

// ADD_AUX_BIAS on 32 accumulator columns [n, n + 32) of row `row`:
// v = b[n] + (g[row, n] + v), the order of the unfused graph's two adds.
// Written out (not Epi::apply, whose kind switch unrolled 32 times blew the
// epilogue past the instruction cache: 79 us vs 11 us on the LSTM's
// [20 x 800 x 200] GEMM); 128-bit loads when both operands are unit-stride
// and aligned.
__device__ __forceinline__ void add_aux_bias32(const Epi<float>& E, int row, int n, int N, float* v) {
  const float* g = E.aux + (int64_t)row * E.s0;
  const float* b = E.aux2 + (int64_t)row * E.b0;
  if (n + 32 <= N && E.s1 == 1 && E.b1 == 1 && (((uintptr_t)(g + n) | (uintptr_t)(b + n)) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const float4 g4 = *reinterpret_cast<const float4*>(g + n + i);
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(b + n + i));
      v[i] = __fadd_rn(b4.x, __fadd_rn(g4.x, v[i]));
      v[i + 1] = __fadd_rn(b4.y, __fadd_rn(g4.y, v[i + 1]));
      v[i + 2] = __fadd_rn(b4.z, __fadd_rn(g4.z, v[i + 2]));
      v[i + 3] = __fadd_rn(b4.w, __fadd_rn(g4.w, v[i + 3]));
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (n + i < N) v[i] = __fadd_rn(b[(int64_t)(n + i) * E.b1], __fadd_rn(g[(int64_t)(n + i) * E.s1], v[i]));
  }
}

template <int CG, bool PROMO>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapX,
                   const __grid_constant__ CUtensorMap mapAe, const __grid_constant__ CUtensorMap mapBe,
                   const __grid_constant__ CUtensorMap mapP, const TcParams p) {
  TX_GRID_WAIT();
  using K_ = Cfg<CG>;
  constexpr int STAGES = K_::STAGES;
  constexpr int kEpiUnroll = PROMO ? 4 : 1;  // compile-time column-chunk index for the promoted sums
  constexpr int kMaxJ = 4;                   // 32-column chunks per epilogue thread
  // TMEM accumulators: two 256-column buffers (tile i+1's MMAs -- PROMO: the
  // next promotion chunk's -- overlap the epilogue's drain of the other)
  constexpr int NACC = 2;
  constexpr int ACC_COLS = BN;
  const int bn = p.bn;
  const int BNL = bn / CG;  // B columns staged by this CTA
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + K_::RING + K_::STAGING + K_::AUX_STAGING);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 4;
  uint64_t* auxbar = tempty + 4;                 // one per epilogue warp
  uint32_t* tmem_slot = (uint32_t*)(auxbar + EPI_WARPS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG;
  const int num_clusters = gridDim.x / CG;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, p.mcast > 1 ? p.mcast : 1); }
    for (int b = 0; b < NACC; ++b) { mbar_init(tfull + b, 1); mbar_init(tempty + b, EPI_WARPS * CG); }
    for (int w = 0; w < EPI_WARPS; ++w) mbar_init(auxbar + w, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (CG == 2 || p.mcast > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t mrank = CG == 1 && p.mcast > 1 ? cluster_rank() : 0;  // rank within the multicast cluster
  const uint16_t mmask = (uint16_t)((1u << (p.mcast > 1 ? p.mcast : 1)) - 1u);
  const int num_kb = (p.K + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mapA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mapB) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      int64_t cur = seg_begin(p, cluster_id);
      Seg sg;
      while (seg_next(p, cluster_id, cur, sg)) {
        int mb, nb;
        tile_coords(sg.t, p.num_m, p.num_n, p.group_m, mb, nb);
        if (p.mcast > 1) { mb = (sg.t / p.mcast) % p.num_m; nb = (sg.t / (p.mcast * p.num_m)) * p.mcast + sg.t % p.mcast; }
        const int kb0 = sg.kb0, kb1 = sg.kb1;
        const int m0 = mb * BM * CG + (int)rank * BM;   // this CTA's rows
        const int n0 = nb * bn + (int)rank * BNL;       // this CTA's half of B
        for (int kb = kb0; kb < kb1; kb += p.kpack) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * K_::STAGE_BYTES;
          uint8_t* sb = sa + K_::A_BYTES;
          const int nsub = min(p.kpack, kb1 - kb);
          if (leader) mbar_expect_tx(full + stage, (uint32_t)(p.stage_tx * nsub));
          const int k0 = kb * BK;
          auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1) {
            if constexpr (CG == 1) tma_load_2d(dst, map, full + stage, c0, c1);
            else tma_load_2d_2sm(dst, map, full + stage, c0, c1);
          };
          auto load3 = [&](void* dst, const CUtensorMap* map, int c1, int c2) {
            if constexpr (CG == 1) tma_load_3d(dst, map, full + stage, 0, c1, c2);
            else tma_load_3d_2sm(dst, map, full + stage, 0, c1, c2);
          };
          if (p.conv) {
            const int img = mb / p.cv_pb, r0 = (mb % p.cv_pb) * p.cv_RB;
            for (int sub = 0; sub < nsub; ++sub) {
              const int k = kb + sub;
              const int tap = k / p.cv_cb, c0 = (k % p.cv_cb) * 32;
              uint8_t* da = p.kpack == 2 ? sa + sub * 16384 : sa;
              uint8_t* db = p.kpack == 2 ? sa + 32768 + sub * 8192 : sb;
              tma_load_4d(da, &mapA, full + stage, c0, tap % p.cv_kw, r0 + tap / p.cv_kw, img);
              tma_load_2d(db, &mapB, full + stage, k * BK, n0);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          } else if (CG == 1 && p.mcast > 1) {  // this CTA's share of the A panel's 32-row atoms, to every CTA
            for (int j = (int)mrank; j < BM / 32; j += p.mcast)
              tma_load_2d_mc(sa + j * 4096, &mapAe, full + stage, m0 + 32 * j, k0, mmask);
          } else if (p.a_3d && m0 + BM <= p.a_lim) {
            load3(sa, &mapA, k0, m0 / 32);
          } else if (p.a_mn) {  // 32-wide boxes: 2-D edge map (clipped at M)
            const CUtensorMap* ma = p.a_3d ? &mapAe : &mapA;
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) load(sa + j * 4096, ma, m0 + 32 * j, k0);
          } else {
            load(sa, &mapA, k0, m0);
          }
          if (p.b_3d && n0 + BNL <= p.b_lim) {
            load3(sb, &mapB, k0, n0 / 32);
          } else if (p.b_mn) {
            const CUtensorMap* mb = p.b_3d ? &mapBe : &mapB;
            for (int j = 0; j < BNL / 32; ++j) load(sb + j * 4096, mb, n0 + 32 * j, k0);
          } else {
            load(sb, &mapB, k0, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)p.a_mn << 15) |
                             ((uint32_t)p.b_mn << 16) | ((uint32_t)(bn >> 3) << 17) |
                             ((uint32_t)((BM * CG) >> 4) << 24);
      // descriptor geometry per operand layout
      // K-major: LBO unused (16 B), SBO = 1024 B between 8-row atoms, +32 B per k-step.
      // MN-major: LBO = 4096 B between 32-element MN blocks (one TMA box each),
      //           SBO = 512 B between 4-row K groups, +1024 B per k-step (8 rows).
      const uint32_t a_lbo = p.a_mn ? 4096u : 16u, a_sbo = p.a_mn ? 512u : 1024u, a_step = p.a_mn ? 1024u : 32u;
      const uint32_t b_lbo = p.b_mn ? 4096u : 16u, b_sbo = p.b_mn ? 512u : 1024u, b_step = p.b_mn ? 1024u : 32u;
      const uint32_t a_lay = p.a_mn ? 1u : 2u, b_lay = p.b_mn ? 1u : 2u;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      int64_t cur = seg_begin(p, cluster_id);
      Seg sg;
      while (seg_next(p, cluster_id, cur, sg)) {
       for (int c0 = sg.kb0, c1; c0 < sg.kb1; c0 = c1, ++it) {
        c1 = PROMO ? chunk_end(p, c0, sg.kb1) : sg.kb1;
        const int kb0 = c0, kb1 = c1;
        const int buf = it % NACC;
        const uint32_t use = (uint32_t)(it / NACC);
        mbar_wait(tempty + buf, (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(buf * ACC_COLS);  // buffers at 0 / 256 (PROMO: 0/128/256/384)
        for (int kb = kb0; kb < kb1; kb += p.kpack) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t s0 = su32(smem + stage * K_::STAGE_BYTES);
            const int nsub = min(p.kpack, kb1 - kb);
            for (int sub = 0; sub < nsub; ++sub) {
              const uint32_t sa = p.kpack == 2 ? s0 + sub * 16384 : s0;
              const uint32_t sb = p.kpack == 2 ? s0 + 32768 + sub * 8192 : s0 + K_::A_BYTES;
#pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk) {
                const uint64_t da = sdesc(sa + kk * a_step, a_lbo, a_sbo, a_lay);
                const uint64_t db = sdesc(sb + kk * b_step, b_lbo, b_sbo, b_lay);
                umma_tf32<CG>(tmem_d, da, db, idesc, (kb != kb0) || (sub != 0) || (kk != 0));
              }
            }
            if (CG == 1 && p.mcast > 1) umma_commit_mc(empty + stage, mmask);  // every producer of the panel
            else umma_commit<CG>(empty + stage);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) umma_commit<CG>(tfull + buf);
        __syncwarp();
       }
      }
    }
  } else {
    // epilogue warps 2..9: TMEM lane quarter (warp % 4), column half (warp - 2) / 4.
    // 32 columns per TMEM load; every global access is 128-bit.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    int it = 0;
    uint32_t xphase = 0;
    const Epi<float>& E = p.epi;
    const bool vec_ok = (p.ldc % 4 == 0) && (((uintptr_t)p.C & 15) == 0) &&
                        ((E.kind != TX_EPI_MUL_AUX && E.kind != TX_EPI_MUL_1MSQR && E.kind != TX_EPI_SGD) ||
                         (E.s1 == 1 && E.s0 % 4 == 0 && ((uintptr_t)E.aux & 15) == 0)) &&
                        (E.kind != TX_EPI_BIAS_TANH_DUAL || (E.o1 == 1 && E.o0 % 4 == 0 && ((uintptr_t)E.out2 & 15) == 0)) &&
                        (E.kind != TX_EPI_BIAS && E.kind != TX_EPI_BIAS_TANH && E.kind != TX_EPI_BIAS_TANH_DUAL ||
                         (E.s1 == 1 && ((uintptr_t)E.aux & 15) == 0));
    int64_t cur = seg_begin(p, cluster_id);
    Seg sg;
    for (; seg_next(p, cluster_id, cur, sg); ++it) {
      int mb, nb;
      tile_coords(sg.t, p.num_m, p.num_n, p.group_m, mb, nb);
      if (p.mcast > 1) { mb = (sg.t / p.mcast) % p.num_m; nb = (sg.t / (p.mcast * p.num_m)) * p.mcast + sg.t % p.mcast; }
      const int split = sg.piece;
      const bool partial = !sg.full;
      const int q_ = warp & 3;
      const int nchunks_ = bn / 32;
      float acc[PROMO ? kMaxJ : 1][32];  // PROMO: the row's running fp32 sums, 128 registers at bn = 256
      int nkc = 1;
      if constexpr (PROMO) {
        nkc = 0;
        for (int c = sg.kb0; c < sg.kb1; c = chunk_end(p, c, sg.kb1)) ++nkc;
      }
      if constexpr (PROMO) {
        // every chunk but the last: TMEM -> registers (RN adds), buffer released
        for (int kc = 0; kc + 1 < nkc; ++kc, ++it) {
          const int b_ = it % NACC;
          mbar_wait(tfull + b_, (uint32_t)(it / NACC) & 1);
          tc_fence_after();
          const uint32_t ta = tmem_base + (uint32_t)(b_ * ACC_COLS) + ((uint32_t)(q_ * 32) << 16);
#pragma unroll
          for (int jj = 0; jj < kMaxJ; ++jj) {
            const int ci = half + 2 * jj;
            if (ci < nchunks_) {
#pragma unroll
              for (int s8 = 0; s8 < 4; ++s8) {
                float t[8];
                tmem_ld8(ta + ci * 32 + s8 * 8, t);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  acc[jj][8 * s8 + i] = kc == 0 ? t[i] : __fadd_rn(acc[jj][8 * s8 + i], t[i]);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1) mbar_arrive(tempty + b_);
            else mbar_arrive_leader(tempty + b_);
          }
        }
      }
      const int buf = it % NACC;
      const uint32_t use = (uint32_t)(it / NACC);
      mbar_wait(tfull + buf, use & 1);
      tc_fence_after();
      int row0 = mb * BM * CG + (int)rank * BM + q * 32;
      int row = row0 + lane;
      int conv_valid = BM;
      int64_t nchw_base = 0;  // conv NCHW store: &C[img, 0, pixel of this lane]
      if (p.conv) {  // tile = RB output rows of one image (RB * Q pixels), rows past them are padding
        const int img = mb / p.cv_pb, r0 = (mb % p.cv_pb) * p.cv_RB;
        conv_valid = min(p.cv_RB, p.cv_P - r0) * p.cv_Q;
        row0 = (img * p.cv_P + r0) * p.cv_Q + q * 32;
        row = row0 + lane;
        nchw_base = (int64_t)img * p.N * (p.cv_P * p.cv_Q) + r0 * p.cv_Q + q * 32 + lane;
      }
      // 32-column chunks of the bn-wide accumulator, alternating between the two warps of a lane quarter
      const uint32_t taddr = tmem_base + (uint32_t)(buf * ACC_COLS) + ((uint32_t)(q * 32) << 16);
      const int nchunks = bn / 32;
      float* crow = p.C + (int64_t)row * p.ldc;
      const bool row_ok = p.conv ? q * 32 + lane < conv_valid : row < p.M;
      if (p.tma_store || p.splits > 1) {  // (split-K: every segment is a partial tile -> workspace)
        // row `lane` of a [32 x 32] tile -> swizzled staging -> one TMA store
        // per chunk (coalesced, asynchronous; TMA clips the M/N edges)
        float* stg = reinterpret_cast<float*>(smem + K_::RING + (size_t)(warp - 2) * 4096);
        const float* xstg = reinterpret_cast<const float*>(smem + K_::RING + K_::STAGING + (size_t)(warp - 2) * 4096);
        uint64_t* xbar = auxbar + (warp - 2);
#pragma unroll kEpiUnroll
        for (int jj = 0; jj < kMaxJ; ++jj) {
          const int ci = half + 2 * jj;
          if (ci >= nchunks) break;
          const int c = ci * 32;
          const int n = nb * bn + c;
          const bool live = !(row0 >= p.M || n >= p.N || p.dbg_nostore);
          if constexpr (CG == 2) {
            if (p.tma_aux && live && !partial && lane == 0) {  // fetch this chunk's operand tile while TMEM drains
              mbar_expect_tx(xbar, 4096);
              tma_load_2d((void*)xstg, &mapX, xbar, n, row0);
            }
          }
          float vloc[32];
          float* v = vloc;
          if constexpr (PROMO) {  // last chunk added into the running sums in place (8 columns at a time)
#pragma unroll
            for (int s8 = 0; s8 < 4; ++s8) {
              float t[8];
              tmem_ld8(taddr + c + s8 * 8, t);
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[jj][8 * s8 + i] = nkc > 1 ? __fadd_rn(acc[jj][8 * s8 + i], t[i]) : t[i];
            }
            v = acc[jj];
          } else {
            tmem_ld32(taddr + c, vloc);
          }
          if (!live) continue;
          if (partial) {  // raw partial tile -> workspace [piece][M][N]; the reduction applies the epilogue
            if (lane == 0) tma_store_wait_read();
            __syncwarp();
            float4* prow = reinterpret_cast<float4*>(stg + lane * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              prow[j ^ (lane & 7)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) tma_store_3d(&mapP, stg, n, row0, split);
            continue;
          }
          if constexpr (CG == 2) {
            if (p.tma_aux) {
              mbar_wait(xbar, xphase);
              xphase ^= 1;
              const float4* xrow = reinterpret_cast<const float4*>(xstg + lane * 32);
              const bool sq = E.kind == TX_EPI_MUL_1MSQR;
              if (E.kind == TX_EPI_SGD) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float4 w4 = xrow[j ^ (lane & 7)];
                  v[4 * j] = __fsub_rn(w4.x, __fmul_rn(E.alpha, v[4 * j]));
                  v[4 * j + 1] = __fsub_rn(w4.y, __fmul_rn(E.alpha, v[4 * j + 1]));
                  v[4 * j + 2] = __fsub_rn(w4.z, __fmul_rn(E.alpha, v[4 * j + 2]));
                  v[4 * j + 3] = __fsub_rn(w4.w, __fmul_rn(E.alpha, v[4 * j + 3]));
                }
              } else
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float4 g4 = xrow[j ^ (lane & 7)];
                if (sq) {
                  g4.x = __fsub_rn(1.0f, __fmul_rn(g4.x, g4.x)); g4.y = __fsub_rn(1.0f, __fmul_rn(g4.y, g4.y));
                  g4.z = __fsub_rn(1.0f, __fmul_rn(g4.z, g4.z)); g4.w = __fsub_rn(1.0f, __fmul_rn(g4.w, g4.w));
                }
                v[4 * j] = __fmul_rn(v[4 * j], g4.x); v[4 * j + 1] = __fmul_rn(v[4 * j + 1], g4.y);
                v[4 * j + 2] = __fmul_rn(v[4 * j + 2], g4.z); v[4 * j + 3] = __fmul_rn(v[4 * j + 3], g4.w);
              }
              __syncwarp();  // every lane has read the operand tile before the next TMA overwrites it
            }
          }
          if (E.kind != TX_EPI_NONE) {
            if (E.kind == TX_EPI_BIAS || E.kind == TX_EPI_BIAS_TANH) {
              if (n + 32 <= p.N && E.s1 == 1 && ((uintptr_t)E.aux & 15) == 0) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                  const float4 b4 = __ldg(reinterpret_cast<const float4*>(E.aux + n + i));
                  v[i] = __fadd_rn(b4.x, v[i]); v[i + 1] = __fadd_rn(b4.y, v[i + 1]);
                  v[i + 2] = __fadd_rn(b4.z, v[i + 2]); v[i + 3] = __fadd_rn(b4.w, v[i + 3]);
                }
              } else {  // ragged edge, or a strided / unaligned bias view
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (n + i < p.N) v[i] = __fadd_rn(E.aux[(int64_t)(n + i) * E.s1], v[i]);
              }
              if (E.kind == TX_EPI_BIAS_TANH) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = tanhf(v[i]);
              }
            } else if (E.kind == TX_EPI_ADD_AUX_BIAS) {  // b[n] + (g[m,n] + acc), per element
              if (row_ok) add_aux_bias32(E, row, n, p.N, v);
            } else if (row_ok && !(CG == 2 && p.tma_aux) && E.kind == TX_EPI_SGD) {
              if (n + 32 <= p.N && E.s1 == 1 && (E.s0 % 4) == 0 && ((uintptr_t)E.aux & 15) == 0) {
                const float* g = E.aux + (int64_t)row * E.s0 + n;
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                  const float4 w4 = *reinterpret_cast<const float4*>(g + i);
                  v[i] = __fsub_rn(w4.x, __fmul_rn(E.alpha, v[i])); v[i + 1] = __fsub_rn(w4.y, __fmul_rn(E.alpha, v[i + 1]));
                  v[i + 2] = __fsub_rn(w4.z, __fmul_rn(E.alpha, v[i + 2]));
                  v[i + 3] = __fsub_rn(w4.w, __fmul_rn(E.alpha, v[i + 3]));
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (n + i < p.N) v[i] = epi_apply_edge(E, v[i], row, n + i);
              }
            } else if (row_ok && !(CG == 2 && p.tma_aux)) {  // MUL_AUX / MUL_1MSQR: per-row [M,N] operand
              const float* g = E.aux + (int64_t)row * E.s0 + n;
              const bool sq = E.kind == TX_EPI_MUL_1MSQR;
              if (n + 32 <= p.N) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                  float4 g4 = __ldcs(reinterpret_cast<const float4*>(g + i));
                  if (sq) {
                    g4.x = __fsub_rn(1.0f, __fmul_rn(g4.x, g4.x)); g4.y = __fsub_rn(1.0f, __fmul_rn(g4.y, g4.y));
                    g4.z = __fsub_rn(1.0f, __fmul_rn(g4.z, g4.z)); g4.w = __fsub_rn(1.0f, __fmul_rn(g4.w, g4.w));
                  }
                  v[i] = __fmul_rn(v[i], g4.x); v[i + 1] = __fmul_rn(v[i + 1], g4.y);
                  v[i + 2] = __fmul_rn(v[i + 2], g4.z); v[i + 3] = __fmul_rn(v[i + 3], g4.w);
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (n + i < p.N) v[i] = epi_apply_edge(E, v[i], row, n + i);
              }
            }
          }
          if (lane == 0) tma_store_wait_read();  // previous chunk's store has read the staging tile
          __syncwarp();
          float4* srow = reinterpret_cast<float4*>(stg + lane * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            srow[j ^ (lane & 7)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) tma_store_2d(&mapC, stg, n, row0);
          if (p.colsum) {
            // column sums of this 32 x 32 block from the swizzled staging tile
            // (lane = column; conflict-free: the xor swizzle permutes banks)
            float cs = 0.f;
#pragma unroll 8
            for (int r = 0; r < 32; ++r)
              if (row0 + r < p.M) cs += stg[r * 32 + 4 * ((lane >> 2) ^ (r & 7)) + (lane & 3)];
            if (n + lane < p.N) p.colsum[(int64_t)(row0 >> 5) * p.N + n + lane] = cs;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) mbar_arrive(tempty + buf);
          else mbar_arrive_leader(tempty + buf);
        }
        continue;
      }
#pragma unroll kEpiUnroll
      for (int jj = 0; jj < kMaxJ; ++jj) {
        const int ci = half + 2 * jj;
        if (ci >= nchunks) break;
        const int c = ci * 32;
        float vloc[32];
        float* v = vloc;
        if constexpr (PROMO) {
#pragma unroll
          for (int s8 = 0; s8 < 4; ++s8) {
            float t[8];
            tmem_ld8(taddr + c + s8 * 8, t);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[jj][8 * s8 + i] = nkc > 1 ? __fadd_rn(acc[jj][8 * s8 + i], t[i]) : t[i];
          }
          v = acc[jj];
        } else {
          tmem_ld32(taddr + c, vloc);
        }
        const int n = nb * bn + c;
        if (!row_ok || n >= p.N || p.dbg_nostore) continue;
        if (p.cv_nchw) {  // channel n + i of this lane's pixel: lanes store 32 consecutive pixels (128 B)
          const int64_t pq = (int64_t)p.cv_P * p.cv_Q;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (n + i < p.N) p.C[nchw_base + (int64_t)(n + i) * pq] = v[i];
          continue;
        }
        if (vec_ok && n + 32 <= p.N) {
          if (E.kind == TX_EPI_BIAS || E.kind == TX_EPI_BIAS_TANH || E.kind == TX_EPI_BIAS_TANH_DUAL) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(E.aux + n + i));
              v[i] = __fadd_rn(b4.x, v[i]); v[i + 1] = __fadd_rn(b4.y, v[i + 1]);
              v[i + 2] = __fadd_rn(b4.z, v[i + 2]); v[i + 3] = __fadd_rn(b4.w, v[i + 3]);
            }
            if (E.kind != TX_EPI_BIAS) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = tanhf(v[i]);
            }
            if (E.kind == TX_EPI_BIAS_TANH_DUAL) {
              float* g = E.out2 + (int64_t)row * E.o0 + n;
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                *reinterpret_cast<float4*>(g + i) = make_float4(
                    __fsub_rn(1.0f, __fmul_rn(v[i], v[i])), __fsub_rn(1.0f, __fmul_rn(v[i + 1], v[i + 1])),
                    __fsub_rn(1.0f, __fmul_rn(v[i + 2], v[i + 2])), __fsub_rn(1.0f, __fmul_rn(v[i + 3], v[i + 3])));
            }
          } else if (E.kind == TX_EPI_ADD_AUX_BIAS) {
            add_aux_bias32(E, row, n, p.N, v);
          } else if (E.kind == TX_EPI_SGD) {
            const float* g = E.aux + (int64_t)row * E.s0 + n;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(g + i);
              v[i] = __fsub_rn(w4.x, __fmul_rn(E.alpha, v[i])); v[i + 1] = __fsub_rn(w4.y, __fmul_rn(E.alpha, v[i + 1]));
              v[i + 2] = __fsub_rn(w4.z, __fmul_rn(E.alpha, v[i + 2])); v[i + 3] = __fsub_rn(w4.w, __fmul_rn(E.alpha, v[i + 3]));
            }
          } else if (E.kind == TX_EPI_MUL_AUX || E.kind == TX_EPI_MUL_1MSQR) {
            const float* g = E.aux + (int64_t)row * E.s0 + n;
            const bool sq = E.kind == TX_EPI_MUL_1MSQR;  // aux is h: factor 1 - h^2
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4 g4 = __ldcs(reinterpret_cast<const float4*>(g + i));
              if (sq) {
                g4.x = __fsub_rn(1.0f, __fmul_rn(g4.x, g4.x)); g4.y = __fsub_rn(1.0f, __fmul_rn(g4.y, g4.y));
                g4.z = __fsub_rn(1.0f, __fmul_rn(g4.z, g4.z)); g4.w = __fsub_rn(1.0f, __fmul_rn(g4.w, g4.w));
              }
              v[i] = __fmul_rn(v[i], g4.x); v[i + 1] = __fmul_rn(v[i + 1], g4.y);
              v[i + 2] = __fmul_rn(v[i + 2], g4.z); v[i + 3] = __fmul_rn(v[i + 3], g4.w);
            }
          }
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(crow + n + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (n + i < p.N) crow[n + i] = E.kind != TX_EPI_NONE ? epi_apply_edge(E, v[i], row, n + i) : v[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) mbar_arrive(tempty + buf);
        else mbar_arrive_leader(tempty + buf);
      }
    }
  }
  if (warp >= 2 && lane == 0) tma_store_wait_all();
  tc_fence_before();
  if (CG == 2 || p.mcast > 1) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
  }
}

// ----------------------------------------------------------------- host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool g_attr_set[2][3] = {{false, false, false}, {false, false, false}};

static EncodeFn encode_fn() { return (EncodeFn)tmap_encoder(); }

// inner-contiguous 2D map: dims {inner, outer}, outer stride in elements
static int make_map(CUtensorMap* m, const void* base, int64_t inner, int64_t outer, int64_t ostride, int box_inner,
                    int box_outer, bool mn_major) {
  EncodeFn enc = encode_fn();
  TX_CHECK(enc, TX_E_NODEVICE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ostride * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_TFLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TX_E_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  return TX_OK;
}

// MN-major operand as 3-D {32 (MN inner), K, MN/32}: element (mn, k) at
// k*ld + mn; box {32, BK, blocks}.  Needs MN % 32 == 0 (no read past the last
// row of the allocation).
static int make_map_mn3d(CUtensorMap* m, const void* base, int64_t MN, int64_t K, int64_t ld, int blocks) {
  EncodeFn enc = encode_fn();
  TX_CHECK(enc, TX_E_NODEVICE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)(MN / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), 128};
  cuuint32_t box[3] = {32, (cuuint32_t)BK, (cuuint32_t)blocks};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_TFLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TX_E_CUDA, "cuTensorMapEncodeTiled (3d) failed (code " + std::to_string((int)r) + ")");
  return TX_OK;
}

}  // namespace

void* tmap_encoder() {
  static std::once_flag once;
  static void* fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = p;
  });
  return fn;
}

int gemm_tc_eligible(const G& g) {
  if (g.dtype != TX_F32) return TX_E_UNSUPPORTED;
  if (g.K < 16) return TX_E_UNSUPPORTED;
  // a thin side (< 64 rows or columns) wastes most of a 128 x 256 tile, which
  // still beats the CUDA-core tile kernel once the product is large (the
  // [20 x 600] x [600 x 10000] per-step GEMMs of an LSTM language model);
  // small thin products stay on the exact SIMT path
  if (g.M < 64 || g.N < 64) {
    static const int thin_log2 = getenv("TX_GEMM_THIN_MIN") ? atoi(getenv("TX_GEMM_THIN_MIN")) : 20;
    static const int64_t thin_kmin = getenv("TX_GEMM_THIN_KMIN") ? atoll(getenv("TX_GEMM_THIN_KMIN")) : 0;
    if ((double)g.M * (double)g.N * (double)g.K < (double)(1ll << thin_log2) || g.K < thin_kmin)
      return TX_E_UNSUPPORTED;
  }
  if (g.M > INT32_MAX || g.N > INT32_MAX || g.K > INT32_MAX) return TX_E_UNSUPPORTED;
  if (g.scn != 1) return TX_E_UNSUPPORTED;
  if (((uintptr_t)g.A & 15) || ((uintptr_t)g.B & 15)) return TX_E_UNSUPPORTED;
  bool a_k = g.sak == 1 && g.sam % 4 == 0 && g.sam >= g.K;
  bool a_m = g.sam == 1 && g.sak % 4 == 0 && g.sak >= g.M;
  bool b_k = g.sbk == 1 && g.sbn % 4 == 0 && g.sbn >= g.K;
  bool b_n = g.sbn == 1 && g.sbk % 4 == 0 && g.sbk >= g.N;
  if (!(a_k || a_m) || !(b_k || b_n)) return TX_E_UNSUPPORTED;
  return TX_OK;
}

// Tile shape per launch: 256 x 256 CTA-pair tiles (cta_group::2), single-CTA
// 128 x 256 when M <= 128.  Narrower N tiles (bn < 256) and single CTAs were
// measured (r01, TX_GEMM_BN / TX_GEMM_CG) at 0.80-0.83 of the pair tile's
// per-FLOP rate, which no wave-quantisation saving on the MLP shapes repays,
// so they remain experiment switches only.
void choose_tile(const G& g, int* cg_out, int* bn_out) {
  const char* cg_s = getenv("TX_GEMM_CG");
  const char* bn_s = getenv("TX_GEMM_BN");
  int cg = 2;
  // when both shapes fit in one wave (the M = 784 weight gradient: 112
  // single-CTA tiles on 148 SMs vs 64 pair tiles on 74 pairs) the per-SM work
  // is equal and uncoupled single CTAs measured ~5% faster (r01 A/B)
  const int64_t sms = sm_count();
  const int64_t t1 = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  const int64_t t2 = ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + BN - 1) / BN);
  if (t1 <= sms && t2 <= sms / 2) cg = 1;
  if (cg_s) cg = atoi(cg_s) == 1 ? 1 : 2;
  if (g.M <= BM) cg = 1;
  int bn = bn_s ? atoi(bn_s) : BN;
  // narrow products (the N <= 16 skinny GEMMs routed here): a 256-wide MMA
  // would spend 16x the tensor time on padding -- use 32 / 64-wide tiles
  if (!bn_s && g.N <= 32) { bn = 32; cg = 1; }
  else if (!bn_s && g.N <= 64) bn = 64;
  // promoted accumulation keeps a row's running sums in registers (128 per
  // epilogue thread at bn = 256, drained 8 TMEM columns at a time to stay
  // inside the 168-register cap that 10 warps on 4 sub-partitions leave);
  // TX_3X_BN128=1 restores the r02a 128-column promoted tile (A/B)
  static const bool bn128 = getenv("TX_3X_BN128") != nullptr;
  if (g.promo && bn > 128 && bn128) bn = 128;
  if (bn < 32 || bn > BN || bn % (32 * cg) != 0) bn = BN;
  *cg_out = cg;
  *bn_out = bn;
}

// Split-K for launches that leave most SMs idle (few output tiles, long K:
// the [20 x 10000] x [10000 x 600] gradient of an LSTM output layer is ONE
// tile).  Work items become (tile, K-slice); raw partial tiles land in a
// [splits][M][N] workspace through a 3-D TMA map and a second kernel sums
// them in split order (deterministic) and applies the epilogue.
// Stream-K (the MLP's dW2 GEMM: 256 pair tiles on 74 pairs = 3.46 waves):
// when the last wave would leave more than a tenth of the machine idle, the
// remainder tiles are cut into an equal run of the flat (tile, k-block)
// sequence per cluster (r01: 405 -> 381 us on that GEMM).  Segments that
// cover a whole tile store C with the epilogue; the pieces of split tiles go
// to a [pieces][M][N] workspace and a fix-up pass sums them in k order and
// applies the epilogue (deterministic).
void tc_streamk(const G& g, int splits, int* streamk, int* pieces, int* nclusters) {
  int cg, bn;
  choose_tile(g, &cg, &bn);
  const int64_t tiles = ((g.M + BM * cg - 1) / (BM * cg)) * ((g.N + bn - 1) / bn);
  const int64_t units = sm_count() / cg;
  const int num_kb = (int)((g.K + BK - 1) / BK);
  *streamk = 0;
  *pieces = 1;
  *nclusters = (int)(tiles < units ? tiles : units);
  const char* e = getenv("TX_GEMM_STREAMK");
  const int force = e ? atoi(e) : -1;
  if (splits > 1 || force == 0 || g.N % 4 != 0 || num_kb < 4) return;
  const int64_t waves = (tiles + units - 1) / units;
  const double fill = (double)tiles / (double)(waves * units);
  const int64_t rem = tiles % units;
  // only with at least one full wave: when every tile would be split (fewer
  // tiles than clusters) the extra partial traffic costs more than the
  // balance gains (r01 A/B: the M = 784 weight gradient 115 -> 145 us)
  if (rem == 0 || (force != 1 && !(fill < 0.9 && waves <= 8 && tiles >= units))) return;
  const int64_t U2 = rem * num_kb;
  const int64_t per = U2 / units;
  if (per < 2) return;
  *streamk = 1;
  *nclusters = (int)units;
  *pieces = (int)((num_kb + per - 1) / per + 1);
}

void tc_splitk(const G& g, int* splits, int* kbs) {
  int cg, bn;
  choose_tile(g, &cg, &bn);
  const int64_t tiles = ((g.M + BM * cg - 1) / (BM * cg)) * ((g.N + bn - 1) / bn);
  const int64_t units = sm_count() / cg;
  const int num_kb = (int)((g.K + BK - 1) / BK);
  *splits = 1;
  *kbs = num_kb;
  if (const char* fs = getenv("TX_GEMM_FORCE_SPLITS")) {  // diagnostics: accumulation-length experiments
    const int want = atoi(fs);
    if (want > 1 && g.N % 4 == 0) {
      const int k = (num_kb + want - 1) / want;
      *kbs = k;
      *splits = (num_kb + k - 1) / k;
      return;
    }
  }
  if (getenv("TX_GEMM_NO_SPLITK") || tiles * 2 > units || num_kb < 8 || g.N % 4 != 0) return;
  int64_t s = units / tiles;
  if (s > num_kb / 4) s = num_kb / 4;
  if (s > 64) s = 64;
  if (s < 2) return;
  const int k = (int)((num_kb + s - 1) / s);
  *kbs = k;
  *splits = (num_kb + k - 1) / k;
}

size_t gemm_tc_workspace(const G& g) {
  int s, k, sk, pieces, nc;
  tc_splitk(g, &s, &k);
  if (s > 1) return (size_t)s * (size_t)g.M * (size_t)g.N * 4 + 256;
  tc_streamk(g, s, &sk, &pieces, &nc);
  return sk ? (size_t)pieces * (size_t)g.M * (size_t)g.N * 4 + 256 : 0;
}

int gemm_tc(const G& g, void* ws, size_t wsb, cudaStream_t st) {
  int rc = gemm_tc_eligible(g);
  if (rc) return fail(rc, "tx_gemm: operand layout not eligible for the tcgen05 path");
  const bool a_mn = !(g.sak == 1 && g.sam % 4 == 0 && g.sam >= g.K);
  const bool b_mn = (g.sbn == 1 && g.sbk % 4 == 0 && g.sbk >= g.N);
  // 2-CTA pairs (cta_group::2) unless TX_GEMM_CG=1 or the problem is too small
  // to give every SM pair a tile
  int cg, bn;
  choose_tile(g, &cg, &bn);
  const int bnl = bn / cg;
  CUtensorMap ma, mb;
  const bool no3d = getenv("TX_GEMM_NO3D") != nullptr;
  // MN-major operands: 3-D boxes over the whole 32-blocks (one TMA per stage);
  // when MN % 32 != 0 the tile holding the ragged block uses 32-wide 2-D
  // boxes from an edge map clipped at MN
  const bool a_3d = a_mn && g.M >= 32 && !no3d;
  const bool b_3d = b_mn && g.N >= 32 && !no3d;
  CUtensorMap mae, mbe;
  memset(&mae, 0, sizeof(mae));
  memset(&mbe, 0, sizeof(mbe));
  if (a_3d) {
    rc = make_map_mn3d(&ma, g.A, g.M / 32 * 32, g.K, g.sak, BM / 32);
    if (!rc && g.M % 32) rc = make_map(&mae, g.A, g.M, g.K, g.sak, 32, 32, true);
  } else if (a_mn) {
    rc = make_map(&ma, g.A, g.M, g.K, g.sak, 32, 32, true);
  } else {
    rc = make_map(&ma, g.A, g.K, g.M, g.sam, 32, BM, false);
  }
  if (rc) return rc;
  if (b_3d) {
    rc = make_map_mn3d(&mb, g.B, g.N / 32 * 32, g.K, g.sbk, bnl / 32);
    if (!rc && g.N % 32) rc = make_map(&mbe, g.B, g.N, g.K, g.sbk, 32, 32, true);
  } else if (b_mn) {
    rc = make_map(&mb, g.B, g.N, g.K, g.sbk, 32, 32, true);
  } else {
    rc = make_map(&mb, g.B, g.K, g.N, g.sbn, 32, bnl, false);
  }
  if (rc) return rc;
  TcParams p;
  p.conv = 0;
  p.cv_nchw = 0;
  p.kpack = 1;
  p.C = (float*)g.C;
  p.ldc = g.scm;
  p.M = (int)g.M;
  p.N = (int)g.N;
  p.K = (int)g.K;
  p.a_mn = a_mn;
  p.b_mn = b_mn;
  p.a_3d = a_3d;
  p.b_3d = b_3d;
  p.a_lim = (int)(g.M % 32 ? g.M / 32 * 32 : INT32_MAX);
  p.b_lim = (int)(g.N % 32 ? g.N / 32 * 32 : INT32_MAX);
  p.num_m = (int)((g.M + BM * cg - 1) / (BM * cg));
  p.num_n = (int)((g.N + bn - 1) / bn);
  p.bn = bn;
  p.stage_tx = (Cfg<2>::A_BYTES + bnl * BK * 4) * cg;
  p.num_tiles = p.num_m * p.num_n;
  tc_splitk(g, &p.splits, &p.kbs);
  if (p.splits > 1 && (ws == nullptr || wsb < gemm_tc_workspace(g) || ((uintptr_t)ws & 15))) {
    p.splits = 1;
    p.kbs = (int)((g.K + BK - 1) / BK);
  }
  p.num_kb = (int)((g.K + BK - 1) / BK);
  int sk_pieces = 1, sk_nc = 1;
  tc_streamk(g, p.splits, &p.streamk, &sk_pieces, &sk_nc);
  if (p.streamk && (ws == nullptr || wsb < gemm_tc_workspace(g) || ((uintptr_t)ws & 15))) p.streamk = 0;
  p.epi = g.epi_f;
  p.colsum = g.colsum;
  if (p.colsum) p.splits = 1, p.kbs = p.num_kb, p.streamk = 0;  // every tile finished by its own epilogue
  p.dbg_nostore = getenv("TX_GEMM_DBG_NOSTORE") != nullptr;
  static const int group_env = getenv("TX_GEMM_GROUP_M") ? atoi(getenv("TX_GEMM_GROUP_M")) : 0;
  p.group_m = group_env > 0 ? group_env : GROUP_M;
  // TMA tile stores need a 16-byte aligned C with a 16-byte row pitch; the
  // dual-output epilogue (two stores per element) keeps the register path
  CUtensorMap mc;
  memset(&mc, 0, sizeof(mc));
  p.tma_store = ((uintptr_t)g.C & 15) == 0 && (g.scm * 4) % 16 == 0 && g.scm >= g.N &&
                g.epi_f.kind != TX_EPI_BIAS_TANH_DUAL && !getenv("TX_GEMM_NO_TMA_STORE");
  if (p.tma_store) {
    EncodeFn enc = encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)g.N, (cuuint64_t)g.M};
    cuuint64_t strides[1] = {(cuuint64_t)(g.scm * 4)};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g.C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) p.tma_store = 0;
  }
  if (p.streamk && !p.tma_store) p.streamk = 0;  // partial pieces need the TMA store path
  if (p.colsum && !p.tma_store) return TX_E_UNSUPPORTED;  // the column sums read the staging tile
  CUtensorMap mp;
  memset(&mp, 0, sizeof(mp));
  if (p.splits > 1 || p.streamk) {
    // partial tiles: 3-D map {N, M, splits | pieces} over the workspace (rows never spill into the next slot)
    EncodeFn enc = encode_fn();
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)(p.streamk ? sk_pieces : p.splits)};
    cuuint64_t strides[2] = {(cuuint64_t)(g.N * 4), (cuuint64_t)(g.M * g.N * 4)};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&mp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ws, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TX_E_CUDA, "tx_gemm: split-K workspace map failed");
  }
  CUtensorMap mx;
  memset(&mx, 0, sizeof(mx));
  const Epi<float>& E = g.epi_f;
  p.tma_aux = cg == 2 && p.tma_store && p.splits == 1 &&
              (E.kind == TX_EPI_MUL_AUX || E.kind == TX_EPI_MUL_1MSQR || E.kind == TX_EPI_SGD) && E.s1 == 1 &&
              (E.s0 * 4) % 16 == 0 && E.s0 >= g.N && ((uintptr_t)E.aux & 15) == 0 && !getenv("TX_GEMM_NO_TMA_AUX");
  if (p.tma_aux) {
    EncodeFn enc = encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)g.N, (cuuint64_t)g.M};
    cuuint64_t strides[1] = {(cuuint64_t)(E.s0 * 4)};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(E.aux), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) p.tma_aux = 0;
  }
  const int units = sm_count() / cg;
  const int work = p.num_tiles * p.splits;
  int nclusters = p.streamk ? units : (work < units ? work : units);
  p.promo = g.promo > 0 && g.promo < p.num_kb ? g.promo : 0;
  p.promo_first = p.promo ? (g.promo_first > 0 && g.promo_first < p.num_kb ? g.promo_first : 0) : 0;
  // A-panel multicast (single-CTA tiles in one wave with an MN-major A: the
  // M = 784 weight gradient G8, 7 x 16 tiles): clusters of 4 CTAs along N
  // share one A panel, each loading one of its four 32-row atoms and
  // multicasting it -- per-SM operand bytes per k-block 48 -> 36 KB
  static const bool no_mc = getenv("TX_GEMM_NO_MCAST") != nullptr;
  p.mcast = 1;
  static const int mcs = getenv("TX_GEMM_MCAST_N") ? atoi(getenv("TX_GEMM_MCAST_N")) : 4;  // cluster size (A/B)
  if (cg == 1 && a_mn && p.splits == 1 && !p.streamk && !p.colsum && !p.promo && !no_mc &&
      p.num_tiles <= units && p.num_n % mcs == 0 && p.num_m >= 2) {
    if (!a_3d || g.M % 32 == 0) rc = make_map(&mae, g.A, g.M, g.K, g.sak, 32, 32, true);  // per-atom 2-D boxes
    if (rc) return rc;
    p.mcast = mcs;
    nclusters = p.num_tiles;  // one tile per CTA: a cluster's CTAs walk the same A panel in lockstep
  }
  p.nclusters = nclusters;
  const int pr = p.promo ? 1 : 0;
  auto k1 = p.promo ? tc_gemm_kernel<1, true> : tc_gemm_kernel<1, false>;
  auto k2 = p.promo ? tc_gemm_kernel<2, true> : tc_gemm_kernel<2, false>;
  if (cg == 1) {
    if (!g_attr_set[pr][1]) {
      TX_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<1>::SMEM));
      g_attr_set[pr][1] = true;
    }
    if (p.mcast > 1) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nclusters, 1, 1);
      cfg.blockDim = dim3(NUM_THREADS, 1, 1);
      cfg.dynamicSmemBytes = Cfg<1>::SMEM;
      cfg.stream = st;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)p.mcast;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      TX_CUDA(cudaLaunchKernelEx(&cfg, k1, ma, mb, mc, mx, mae, mbe, mp, p));
    } else {
      ::tx::launch(k1, dim3(nclusters), dim3(NUM_THREADS), Cfg<1>::SMEM, st, ma, mb, mc, mx, mae, mbe, mp, p);
    }
  } else {
    if (!g_attr_set[pr][2]) {
      TX_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<2>::SMEM));
      g_attr_set[pr][2] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * nclusters, 1, 1);
    cfg.blockDim = dim3(NUM_THREADS, 1, 1);
    cfg.dynamicSmemBytes = Cfg<2>::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    TX_CUDA(cudaLaunchKernelEx(&cfg, k2, ma, mb, mc, mx, mae, mbe, mp, p));
  }
  if (p.splits > 1) {
    TX_CUDA(cudaGetLastError());
    return splitk_finalize((const float*)ws, g, p.splits, st);
  }
  if (p.streamk) {
    TX_CUDA(cudaGetLastError());
    return streamk_fixup((const float*)ws, g, p.num_m, p.num_n, BM * cg, bn, p.num_kb, nclusters, p.group_m, st);
  }
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

// Implicit-GEMM stride-1 convolution on the tcgen05 kernel (CG = 1):
//   out[(n, p, q), k] = sum_{u, v, c} xpad[n, p + u, q + v, c] * w[k, (u, v, c)]
// xpad: zero-padded NHWC input [N, Hp, Wp, C] (contiguous), w: [K, kh*kw*C]
// (contiguous, (u, v, c) order), out: [N*P*Q, K] (contiguous rows).  The
// A tile of a k-block (tap u, v; channels c0..c0+31) is one 4-D TMA box
// {32, Q, RB, 1} at (c0, v, r0 + u, n): RB whole output rows of one image,
// landing as RB*Q consecutive 128-byte rows -- the K-major, 128B-swizzled
// layout the MMA reads -- so no [N*P*Q, kh*kw*C] patch matrix is written or
// read.  Tile rows past RB*Q are stale and never stored (register epilogue).
int gemm_tc_conv(const float* xpad, int64_t N, int64_t Hp, int64_t Wp, int64_t C, const float* w, int64_t K, int kh,
                 int kw, float* out, int out_nchw, cudaStream_t st) {
  const int64_t P = Hp - kh + 1, Q = Wp - kw + 1;
  TX_CHECK(P > 0 && Q > 0 && C % 32 == 0 && Q <= BM && K > 0, TX_E_UNSUPPORTED,
           "tx_conv_implicit: needs C % 32 == 0 and output width <= 128");
  TX_CHECK(((uintptr_t)xpad & 15) == 0 && ((uintptr_t)w & 15) == 0 && ((uintptr_t)out & 15) == 0, TX_E_UNSUPPORTED,
           "tx_conv_implicit: 16-byte aligned operands");
  EncodeFn enc = encode_fn();
  TX_CHECK(enc, TX_E_NODEVICE, "cuTensorMapEncodeTiled unavailable");
  const int RB = (int)(BM / Q);
  CUtensorMap ma, mb;
  {
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)Wp, (cuuint64_t)Hp, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)(C * 4), (cuuint64_t)(Wp * C * 4), (cuuint64_t)(Hp * Wp * C * 4)};
    cuuint32_t box[4] = {32, (cuuint32_t)Q, (cuuint32_t)RB, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_TFLOAT32, 4, const_cast<float*>(xpad), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TX_E_CUDA, "tx_conv_implicit: input map (code " + std::to_string((int)r) + ")");
  }
  const int64_t KK = (int64_t)kh * kw * C;
  int bn = (int)((K + 31) / 32 * 32);
  if (bn > BN) bn = BN;
  int rc = make_map(&mb, w, KK, K, KK, 32, bn, false);
  if (rc) return rc;
  TcParams p;
  memset(&p, 0, sizeof(p));
  p.C = out;
  p.ldc = K;
  p.M = (int)(N * P * Q);
  p.N = (int)K;
  p.K = (int)KK;
  p.a_lim = p.b_lim = INT32_MAX;
  p.conv = 1;
  p.cv_nchw = out_nchw;
  static const bool no_pack = getenv("TX_CONV_NO_KPACK") != nullptr;
  p.kpack = bn <= 64 && !no_pack ? 2 : 1;
  p.cv_cb = (int)(C / 32);
  p.cv_kw = kw;
  p.cv_P = (int)P;
  p.cv_Q = (int)Q;
  p.cv_RB = RB;
  p.cv_pb = (int)((P + RB - 1) / RB);
  p.num_m = (int)(N * p.cv_pb);
  p.num_n = (int)((K + bn - 1) / bn);
  p.bn = bn;
  p.stage_tx = RB * (int)Q * BK * 4 + bn * BK * 4;
  p.num_tiles = p.num_m * p.num_n;
  p.splits = 1;
  p.num_kb = (int)(KK / BK);
  p.kbs = p.num_kb;
  p.streamk = 0;
  p.epi = Epi<float>();
  p.tma_store = 0;
  p.tma_aux = 0;
  p.promo = p.promo_first = 0;
  p.group_m = GROUP_M;
  const int units = sm_count();
  p.nclusters = p.num_tiles < units ? p.num_tiles : units;
  CUtensorMap none;
  memset(&none, 0, sizeof(none));
  if (!g_attr_set[0][1]) {
    TX_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<1>::SMEM));
    g_attr_set[0][1] = true;
  }
  TX_CUDA(::tx::launch(tc_gemm_kernel<1, false>, dim3(p.nclusters), dim3(NUM_THREADS), Cfg<1>::SMEM, st, ma, mb, none,
                       none, none, none, none, p));
  return TX_OK;
}

}  // namespace tx
