// tx_narrow_grad: the backward of a tanh layer feeding a narrow dense layer
// (the MLP's h2 -> 10-class output), fused into one pass over h.
//
// The reference computes, as separate nodes of the differentiated graph
// (Dot.grad ops/linalg.py:68-70, the tanh grad composite, Sum.grad's
// sum_to_matching_shape ops/elemwise.py:411-442):
//   dh = dot(dz, W^T) * (1 - h^2)      [B,H]  (K = k <= 16: an outer product)
//   gW = dot(h^T, dz)                  [H,k]  (a column reduction over B)
//   db = sum(dh, axis=0)               [H]    (the bias gradient of h's layer)
// Each of them streams the [B,H] h or dh through HBM once; here h is read
// once, dh is written once, and gW / db leave as per-slab partials that a
// second kernel sums in slab order (deterministic) and hands to gW's
// epilogue (the SGD update when the rewrite fused it).
//
// Layout: a CTA owns 1024 adjacent columns (4 per thread, 128-bit) and a slab
// of rows; every thread streams its 16-byte slice of h's rows through a
// cp.async ring in shared memory (loads in flight independent of the
// register budget) while dz's rows are staged per chunk and broadcast.
#include <cuda_runtime.h>

#include <cstring>

#include "tx_common.h"
#include "tx_gemm.h"

namespace tx {
namespace {

constexpr int NG_THREADS = 256;
constexpr int NG_S = 4, NG_RU = 4;  // ring: NG_S stages of NG_RU rows
constexpr int NG_CH = 128;          // dz rows staged per chunk

__device__ __forceinline__ void ng_cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}

// one row of the CTA's slab for one thread's 4 columns.  W is held as k-pairs
// per column (w2[j][q] = (W^T[2q][j], W^T[2q+1][j])) so the dz row's natural
// register pairs feed FFMA2 directly: o[j] = (even-k sum) + (odd-k sum).
template <int NK, int KP, int NQ>
__device__ __forceinline__ void ng_row(const float4 hv4, const float* __restrict__ zrow, const float2 (&w2)[4][NQ],
                                       float2 (&g2)[4][NQ], float2 (&s2)[2], float* __restrict__ out) {
  float2 z2[KP / 2];
#pragma unroll
  for (int q = 0; q < KP / 4; ++q) {
    const float4 t = reinterpret_cast<const float4*>(zrow)[q];
    z2[2 * q] = make_float2(t.x, t.y);
    z2[2 * q + 1] = make_float2(t.z, t.w);
  }
  float2 a[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    a[j] = __fmul2_rn(z2[0], w2[j][0]);
#pragma unroll
    for (int q = 1; q < NQ; ++q) a[j] = __ffma2_rn(z2[q], w2[j][q], a[j]);
  }
  const float2 o01 = make_float2(a[0].x + a[0].y, a[1].x + a[1].y);
  const float2 o23 = make_float2(a[2].x + a[2].y, a[3].x + a[3].y);
  const float2 one2 = make_float2(1.0f, 1.0f);
  const float2 h01 = make_float2(hv4.x, hv4.y), h23 = make_float2(hv4.z, hv4.w);
  // (1 - h^2) with the unfused nodes' rounding: sqr, then sub
  const float2 q01 = __fmul2_rn(h01, h01), q23 = __fmul2_rn(h23, h23);
  const float2 d01 = __fmul2_rn(o01, __fadd2_rn(one2, make_float2(-q01.x, -q01.y)));
  const float2 d23 = __fmul2_rn(o23, __fadd2_rn(one2, make_float2(-q23.x, -q23.y)));
  s2[0] = __fadd2_rn(s2[0], d01);
  s2[1] = __fadd2_rn(s2[1], d23);
  const float hv[4] = {hv4.x, hv4.y, hv4.z, hv4.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 hj = make_float2(hv[j], hv[j]);
#pragma unroll
    for (int q = 0; q < NQ; ++q) g2[j][q] = __ffma2_rn(hj, z2[q], g2[j][q]);
  }
  *reinterpret_cast<float4*>(out) = make_float4(d01.x, d01.y, d23.x, d23.y);
}

// Per row and thread: o = dz[r,:] . W^T[:, 4 cols] and g[4 cols][:] += h * dz[r,:]
// with packed fp32x2 FMAs (FFMA2: half the issue slots of scalar FFMA --
// the kernel is issue-bound otherwise, 20 FMAs per element); ring slots are
// compile-time indices.
template <int NK>
__global__ void __launch_bounds__(NG_THREADS, (NK <= 10 ? 2 : 1)) narrow_grad_kernel(
    const float* __restrict__ dz, int64_t sz0, int64_t sz1, const float* __restrict__ wt, int64_t swk, int64_t swh,
    const float* __restrict__ h, int64_t sh0, float* __restrict__ dh, int64_t sd0, float* __restrict__ Pg,
    int64_t B, int64_t H, int64_t rows_per) {
  TX_GRID_WAIT();
  constexpr int KP = (NK + 3) & ~3;  // dz row pitch in smem (zero padded)
  constexpr int NQ = (NK + 1) / 2;   // k pairs
  constexpr int RING = NG_S * NG_RU;
  extern __shared__ __align__(16) float4 ng_smem[];
  float4* ring = ng_smem;                                            // [RING][NG_THREADS]
  float* zs = reinterpret_cast<float*>(ng_smem + RING * NG_THREADS);  // [NG_CH][KP]
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int nr = (int)max((int64_t)0, min(B, r0 + rows_per) - r0);
  const int64_t jc = (int64_t)blockIdx.x * NG_THREADS * 4;  // CTA's first column
  const int64_t j0 = jc + tid * 4;
  const bool active = j0 < H;
  const float* hp = h + r0 * sh0 + j0;
  // W^T slice for the thread's 4 columns.  W row-major [H, NK] (wt its
  // transposed view): the 4 rows are 4*NK contiguous floats, read with
  // 128-bit loads.  Otherwise staged through the (not yet used) ring.
  float2 w2[4][NQ];
  const bool wrow = swk == 1 && swh == NK && (((uintptr_t)wt & 15) == 0);
  if (wrow) {
    float wv[4 * NK];
    if (active) {
      const float4* src = reinterpret_cast<const float4*>(wt + j0 * NK);
#pragma unroll
      for (int q = 0; q < NK; ++q) {
        const float4 t = __ldg(src + q);
        wv[4 * q] = t.x; wv[4 * q + 1] = t.y; wv[4 * q + 2] = t.z; wv[4 * q + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4 * NK; ++q) wv[q] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        w2[j][q] = make_float2(wv[j * NK + 2 * q], 2 * q + 1 < NK ? wv[j * NK + 2 * q + 1] : 0.f);
  } else {
    const int ncols = (int)min((int64_t)NG_THREADS * 4, H - jc);
    float* ws = reinterpret_cast<float*>(ring);  // NK * 1024 floats <= the ring's 16384
    for (int e = tid; e < NK * ncols; e += NG_THREADS) {
      int k, c;
      if (swh == 1) { k = e / ncols; c = e - k * ncols; } else { c = e / NK; k = e - c * NK; }
      ws[k * NG_THREADS * 4 + c] = wt[k * swk + (jc + c) * swh];
    }
    __syncthreads();
    float wv[4 * NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const float4 t = active ? reinterpret_cast<const float4*>(ring)[k * NG_THREADS + tid] : make_float4(0.f, 0.f, 0.f, 0.f);
      wv[0 * NK + k] = t.x; wv[1 * NK + k] = t.y; wv[2 * NK + k] = t.z; wv[3 * NK + k] = t.w;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        w2[j][q] = make_float2(wv[j * NK + 2 * q], 2 * q + 1 < NK ? wv[j * NK + 2 * q + 1] : 0.f);
    __syncthreads();  // the ring's slots are free again
  }
  auto issue = [&](int rr, int slot0) {
#pragma unroll
    for (int u = 0; u < NG_RU; ++u) {
      const int r = rr + u;
      if (active && r < nr) ng_cp16(&ring[(slot0 + u) * NG_THREADS + tid], hp + (int64_t)r * sh0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < NG_S; ++s) issue(s * NG_RU, s * NG_RU);
  float2 g2[4][NQ];
  float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int q = 0; q < NQ; ++q) g2[j][q] = make_float2(0.f, 0.f);
  float* dp = dh + r0 * sd0 + j0;
  for (int c0 = 0; c0 < nr; c0 += NG_CH) {
    const int cn = min(NG_CH, nr - c0);
    __syncthreads();
    for (int e = tid; e < cn * KP; e += NG_THREADS) {
      const int r = e / KP, k = e - r * KP;
      zs[e] = k < NK ? dz[(r0 + c0 + r) * sz0 + k * sz1] : 0.f;
    }
    __syncthreads();
    for (int rb = c0; rb < c0 + cn; rb += RING) {
#pragma unroll
      for (int s = 0; s < NG_S; ++s) {
        asm volatile("cp.async.wait_group %0;" ::"n"(NG_S - 1) : "memory");
        const int rs = rb + s * NG_RU;
        if (active) {
          if (rs + NG_RU <= c0 + cn) {  // whole stage: no per-row branches, rows interleave
#pragma unroll
            for (int u = 0; u < NG_RU; ++u)
              ng_row<NK, KP, NQ>(ring[(s * NG_RU + u) * NG_THREADS + tid], zs + (rs + u - c0) * KP, w2, g2, s2,
                                 dp + (int64_t)(rs + u) * sd0);
          } else {
            for (int u = 0; u < NG_RU && rs + u < c0 + cn; ++u)
              ng_row<NK, KP, NQ>(ring[(s * NG_RU + u) * NG_THREADS + tid], zs + (rs + u - c0) * KP, w2, g2, s2,
                                 dp + (int64_t)(rs + u) * sd0);
          }
        }
        issue(rb + (s + NG_S) * NG_RU, s * NG_RU);
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (!active) return;
  // partials P[slab][NK+1][H] (row NK: db), 128-bit stores coalesced across
  // the CTA's threads.  (Reducing them across a thread-block cluster through
  // DSMEM first was measured slower: clusters lowered the co-resident CTAs.)
  float* pg = Pg + (int64_t)blockIdx.y * (NK + 1) * H + j0;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int q = k / 2;
    const bool hi = k & 1;
    *reinterpret_cast<float4*>(pg + (int64_t)k * H) =
        make_float4(hi ? g2[0][q].y : g2[0][q].x, hi ? g2[1][q].y : g2[1][q].x, hi ? g2[2][q].y : g2[2][q].x,
                    hi ? g2[3][q].y : g2[3][q].x);
  }
  *reinterpret_cast<float4*>(pg + (int64_t)NK * H) = make_float4(s2[0].x, s2[0].y, s2[1].x, s2[1].y);
}

// gW[j,k] = epi(sum_s P[s][k][j]); db[j] = sum_s P[s][NK][j]: one output per
// thread, 8 independent loads in flight, adds in slab order (deterministic)
__global__ void __launch_bounds__(256) narrow_grad_finalize(const float* __restrict__ P, int S, int64_t H, int NK,
                                                           float* __restrict__ gw, int64_t sg0, int64_t sg1,
                                                           Epi<float> epi, float* __restrict__ db, int64_t sdb) {
  TX_GRID_WAIT();
  // 32 outputs per CTA, the S slabs split over its 8 warps (interleaved) and
  // the 8 partials added in warp order: deterministic, 8x the loads in flight
  // of one thread per output walking every slab
  __shared__ float part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = blockIdx.x * 32LL + lane;
  const int64_t HK1 = H * (NK + 1);
  const int k = e < HK1 ? (int)(e / H) : NK;
  const bool live = e < HK1 && (k < NK || db);
  float v = 0.f;
  if (live && S <= 128) {  // every slab of this warp in flight at once (same summation order as below)
    float q[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) q[u] = w + 8 * u < S ? __ldcs(P + (int64_t)(w + 8 * u) * HK1 + e) : 0.f;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (w + 8 * u < S) v += q[u];
  } else if (live) {
    int s = w;
    for (; s + 24 < S; s += 32) {
      const float q0 = __ldcs(P + (int64_t)s * HK1 + e), q1 = __ldcs(P + (int64_t)(s + 8) * HK1 + e);
      const float q2 = __ldcs(P + (int64_t)(s + 16) * HK1 + e), q3 = __ldcs(P + (int64_t)(s + 24) * HK1 + e);
      v += q0; v += q1; v += q2; v += q3;
    }
    for (; s < S; s += 8) v += P[(int64_t)s * HK1 + e];
  }
  part[w][lane] = v;
  __syncthreads();
  if (w != 0 || !live) return;
  float t = part[0][lane];
#pragma unroll
  for (int u = 1; u < 8; ++u) t += part[u][lane];
  const int64_t j = e - (int64_t)k * H;
  if (k < NK) gw[j * sg0 + k * sg1] = epi.apply(t, j, k);
  else db[j * sdb] = t;
}

// db[j] = sum over the 32-row blocks of the dh GEMM's column sums.  A CTA
// owns 32 columns; its 8 warps take interleaved blocks (s = warp, warp+8,
// ...) and the 8 partials are added in warp order (deterministic).  One
// thread per column walking all S = B/32 blocks was a 32-deep chain of
// dependent load rounds: 22.6 us for 4 MB at B = 8192.
__global__ void __launch_bounds__(256) colsum_finalize(const float* __restrict__ P, int S, int64_t H,
                                                       float* __restrict__ db, int64_t sdb) {
  TX_GRID_WAIT();
  __shared__ float part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * 32LL + lane;
  float v = 0.f;
  if (j < H && S <= 256) {  // every block of this warp in flight at once (same summation order as below)
    float q[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) q[u] = w + 8 * u < S ? __ldcs(P + (int64_t)(w + 8 * u) * H + j) : 0.f;
#pragma unroll
    for (int u = 0; u < 32; ++u)
      if (w + 8 * u < S) v += q[u];
  } else if (j < H) {
    int s = w;
    for (; s + 24 < S; s += 32) {
      const float q0 = __ldcs(P + (int64_t)s * H + j), q1 = __ldcs(P + (int64_t)(s + 8) * H + j);
      const float q2 = __ldcs(P + (int64_t)(s + 16) * H + j), q3 = __ldcs(P + (int64_t)(s + 24) * H + j);
      v += q0; v += q1; v += q2; v += q3;
    }
    for (; s < S; s += 8) v += P[(int64_t)s * H + j];
  }
  part[w][lane] = v;
  __syncthreads();
  if (w == 0 && j < H) {
    float t = part[0][lane];
#pragma unroll
    for (int u = 1; u < 8; ++u) t += part[u][lane];
    db[j * sdb] = t;
  }
}

struct NG {
  int64_t B, H, k;
  int S;  // slabs (CTAs along y)
  int64_t rows_per;
  bool fused;
};

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// geometry + whether the fused kernel applies (fp32, k <= 16, h and dh
// row-contiguous with 16-byte aligned rows)
int plan(const tx_tensor* dz, const tx_tensor* wt, const tx_tensor* h, const tx_tensor* dh, const tx_tensor* gw,
         const tx_tensor* db, NG* p) {
  TX_CHECK(dz && wt && h && dh && gw, TX_E_ARG, "tx_narrow_grad: null operand");
  TX_CHECK(dz->ndim == 2 && wt->ndim == 2 && h->ndim == 2 && dh->ndim == 2 && gw->ndim == 2, TX_E_ARG,
           "tx_narrow_grad: operands must be rank 2");
  p->B = h->shape[0];
  p->H = h->shape[1];
  p->k = dz->shape[1];
  TX_CHECK(dz->shape[0] == p->B && wt->shape[0] == p->k && wt->shape[1] == p->H, TX_E_ARG,
           "tx_narrow_grad: dz [B,k], wt [k,H], h [B,H] disagree");
  TX_CHECK(dh->shape[0] == p->B && dh->shape[1] == p->H && gw->shape[0] == p->H && gw->shape[1] == p->k, TX_E_ARG,
           "tx_narrow_grad: dh must be [B,H] and gW [H,k]");
  TX_CHECK(!db || !db->data || (db->ndim == 1 && db->shape[0] == p->H), TX_E_ARG, "tx_narrow_grad: db must be [H]");
  const int dt = h->dtype;
  TX_CHECK(dz->dtype == dt && wt->dtype == dt && dh->dtype == dt && gw->dtype == dt && (!db || !db->data || db->dtype == dt),
           TX_E_ARG, "tx_narrow_grad: dtype mismatch");
  p->fused = dt == TX_F32 && p->k >= 1 && p->k <= 16 && p->H % 4 == 0 && p->B > 0 &&
             (p->H == 1 || h->strides[1] == 1) && (p->H == 1 || dh->strides[1] == 1) && h->strides[0] % 4 == 0 &&
             dh->strides[0] % 4 == 0 && aligned16(h->data) && aligned16(dh->data) && !getenv("TX_NARROW_UNFUSED");
  p->S = 0;
  p->rows_per = 0;
  if (p->fused) {
    const int64_t cg = (p->H + 4 * NG_THREADS - 1) / (4 * NG_THREADS);
    int64_t s = ((int64_t)sm_count() * 2 + cg - 1) / cg;
    if (s > (p->B + 31) / 32) s = (p->B + 31) / 32;
    if (s < 1) s = 1;
    p->rows_per = (p->B + s - 1) / s;
    p->S = (int)((p->B + p->rows_per - 1) / p->rows_per);
  }
  return TX_OK;
}

tx_tensor transposed2(const tx_tensor& t) {
  tx_tensor r = t;
  r.shape[0] = t.shape[1];
  r.shape[1] = t.shape[0];
  r.strides[0] = t.strides[1];
  r.strides[1] = t.strides[0];
  return r;
}

template <int NK>
int launch(const NG& p, const tx_tensor* dz, const tx_tensor* wt, const tx_tensor* h, tx_tensor* dh, float* Pg,
           cudaStream_t st) {
  constexpr int KP = (NK + 3) & ~3;
  const size_t smem = (size_t)NG_S * NG_RU * NG_THREADS * 16 + (size_t)NG_CH * KP * 4;
  static bool attr = false;
  if (!attr) {
    TX_CUDA(cudaFuncSetAttribute(narrow_grad_kernel<NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grid((unsigned)((p.H + 4 * NG_THREADS - 1) / (4 * NG_THREADS)), (unsigned)p.S);
  ::tx::launch(narrow_grad_kernel<NK>, dim3(grid), dim3(NG_THREADS), smem, st, 
      (const float*)dz->data, dz->strides[0], dz->strides[1], (const float*)wt->data, wt->strides[0], wt->strides[1],
      (const float*)h->data, h->strides[0], (float*)dh->data, dh->strides[0], Pg, p.B, p.H, p.rows_per);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

}  // namespace
}  // namespace tx

using namespace tx;

extern "C" {

int tx_narrow_grad_workspace(const tx_tensor* dz, const tx_tensor* wt, const tx_tensor* h, const tx_tensor* dh,
                             const tx_tensor* gw, const tx_tensor* db, int mode, size_t* bytes) {
  NG p;
  int rc = plan(dz, wt, h, dh, gw, db, &p);
  if (rc) return rc;
  if (p.fused) {
    *bytes = (size_t)p.S * (size_t)p.H * (size_t)(p.k + 1) * 4 + 256;
    return TX_OK;
  }
  // unfused: the three ops one after another share one workspace, plus the
  // dh GEMM's per-32-row column sums when db is wanted (tcgen05 epilogue)
  size_t a = 0, b = 0, c = 0;
  tx_tensor ht = transposed2(*h);
  if ((rc = tx_gemm_workspace(dz, wt, dh, mode, &a))) return rc;
  if ((rc = tx_gemm_workspace(&ht, dz, gw, mode, &b))) return rc;
  if (db && db->data && (rc = tx_reduce_workspace(TX_SUM, dh, 1u, &c))) return rc;
  const size_t colsum = (db && db->data) ? (size_t)((p.B + 31) / 32) * (size_t)p.H * 4 + 256 : 0;
  *bytes = (a > b ? (a > c ? a : c) : (b > c ? b : c)) + colsum;
  return TX_OK;
}

int tx_narrow_grad(const tx_tensor* dz, const tx_tensor* wt, const tx_tensor* h, tx_tensor* dh, tx_tensor* gw,
                   const tx_epilogue* gw_epi, tx_tensor* db, int mode, void* ws, size_t wsb, void* stream) {
  NG p;
  int rc = plan(dz, wt, h, dh, gw, db, &p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const bool want_db = db && db->data;
  if (!p.fused) {
    tx_epilogue e1;
    memset(&e1, 0, sizeof(e1));
    e1.kind = TX_EPI_MUL_1MSQR;
    e1.aux = *h;
    // db from the dh GEMM's epilogue (column sums of the staged C tiles) when
    // dh runs on the tensor cores: the [B, H] dh is not re-read
    const size_t csb = want_db ? (size_t)((p.B + 31) / 32) * (size_t)p.H * 4 : 0;
    bool db_done = false;
    if (want_db && p.B > 0 && p.H > 0 && h->dtype == TX_F32 && !getenv("TX_NARROW_NO_COLSUM") && ws &&
        wsb >= csb + 256) {
      float* partials = (float*)(((uintptr_t)ws + wsb - csb) & ~(uintptr_t)15);
      if ((uintptr_t)partials >= (uintptr_t)ws && gemm_with_colsum(dz, wt, dh, &e1, mode, ws, wsb - csb - 256, partials, st) == TX_OK) {
        const int64_t S = (p.B + 31) / 32;
        ::tx::launch(colsum_finalize, dim3((unsigned)((p.H + 31) / 32)), dim3(256), 0, st, partials, (int)S, p.H, (float*)db->data,
                                                                      db->strides[0]);
        TX_CUDA(cudaGetLastError());
        db_done = true;
      }
    }
    const size_t wsg = want_db && wsb > csb + 256 ? wsb - csb - 256 : wsb;
    if (!db_done && (rc = tx_gemm(dz, wt, dh, &e1, mode, ws, wsg, stream))) return rc;
    tx_tensor ht = transposed2(*h);
    if ((rc = tx_gemm(&ht, dz, gw, gw_epi, mode, ws, wsg, stream))) return rc;
    if (want_db && !db_done) return tx_reduce(TX_SUM, dh, 1u, db, ws, wsg, stream);
    return TX_OK;
  }
  const size_t need = (size_t)p.S * (size_t)p.H * (size_t)(p.k + 1) * 4;
  TX_CHECK(ws && wsb >= need, TX_E_ARG, "tx_narrow_grad: workspace too small");
  float* Pg = (float*)ws;
  switch ((int)p.k) {
#define CASE(w) case w: rc = launch<w>(p, dz, wt, h, dh, Pg, st); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
  }
  if (rc) return rc;
  Epi<float> epi;
  if (gw_epi && gw_epi->kind != TX_EPI_NONE) {
    TX_CHECK(gw_epi->kind == TX_EPI_SGD && gw_epi->aux.ndim == 2 && gw_epi->aux.shape[0] == p.H &&
                 gw_epi->aux.shape[1] == p.k && gw_epi->aux.dtype == TX_F32,
             TX_E_ARG, "tx_narrow_grad: gW epilogue must be SGD with an [H,k] weight");
    epi.kind = TX_EPI_SGD;
    epi.aux = (const float*)gw_epi->aux.data;
    epi.s0 = gw_epi->aux.strides[0];
    epi.s1 = gw_epi->aux.strides[1];
    epi.alpha = (float)gw_epi->alpha;
  }
  const int64_t tot = p.H * (p.k + 1);
  ::tx::launch(narrow_grad_finalize, dim3((unsigned)((tot + 31) / 32)), dim3(256), 0, st, 
      Pg, p.S, p.H, (int)p.k, (float*)gw->data, gw->strides[0], gw->strides[1], epi,
      want_db ? (float*)db->data : nullptr, want_db ? db->strides[0] : 0);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

}  // extern "C"
