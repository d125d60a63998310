// tx_gemm: the Dot lowering entry point (reference ops/linalg.py:42-62).
// Chooses tcgen05 (large fp32), a memory-bound skinny kernel (one of M/N/K
// tiny), or the SIMT tile kernel (float64, or layouts TMA cannot address).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "tx_common.h"
#include "tx_gemm.h"

namespace tx {
namespace {

int build(const tx_tensor* A, const tx_tensor* B, const tx_tensor* C, const tx_epilogue* epi, G* g) {
  TX_CHECK(A && B && C, TX_E_ARG, "tx_gemm: null operand");
  TX_CHECK(A->ndim == 2 && B->ndim == 2 && C->ndim == 2, TX_E_ARG, "tx_gemm: operands must be rank 2");
  TX_CHECK(A->dtype == B->dtype && A->dtype == C->dtype, TX_E_ARG, "tx_gemm: dtype mismatch");
  TX_CHECK(A->dtype == TX_F32 || A->dtype == TX_F64, TX_E_UNSUPPORTED, "tx_gemm: only float32/float64");
  TX_CHECK(A->shape[1] == B->shape[0], TX_E_ARG, "tx_gemm: inner dimensions disagree");
  TX_CHECK(C->shape[0] == A->shape[0] && C->shape[1] == B->shape[1], TX_E_ARG, "tx_gemm: output shape");
  g->dtype = A->dtype;
  g->A = A->data;
  g->B = B->data;
  g->C = C->data;
  g->M = A->shape[0];
  g->K = A->shape[1];
  g->N = B->shape[1];
  // extent-1 dims may carry any stride; normalise so layout tests see contiguity
  g->sam = A->shape[0] == 1 ? g->K : A->strides[0];
  g->sak = A->shape[1] == 1 ? 1 : A->strides[1];
  g->sbk = B->shape[0] == 1 ? g->N : B->strides[0];
  g->sbn = B->shape[1] == 1 ? 1 : B->strides[1];
  g->scm = C->shape[0] == 1 ? g->N : C->strides[0];
  g->scn = C->shape[1] == 1 ? 1 : C->strides[1];
  if (epi && epi->kind != TX_EPI_NONE) {
    TX_CHECK(epi->aux.dtype == A->dtype, TX_E_ARG, "tx_gemm: epilogue operand dtype");
    TX_CHECK(epi->kind >= TX_EPI_BIAS && epi->kind <= TX_EPI_ADD_AUX_BIAS, TX_E_ARG, "tx_gemm: unknown epilogue");
    int64_t s0 = 0, s1 = 0;
    if (epi->kind == TX_EPI_ADD_AUX_BIAS) {
      const tx_tensor& b = epi->aux2;
      TX_CHECK(b.dtype == A->dtype && b.ndim >= 1 && b.shape[b.ndim - 1] == g->N, TX_E_ARG,
               "tx_gemm: ADD_AUX_BIAS bias must end in N");
      g->epi_f.aux2 = (const float*)b.data;
      g->epi_d.aux2 = (const double*)b.data;
      g->epi_f.b1 = g->epi_d.b1 = b.shape[b.ndim - 1] == 1 ? 0 : b.strides[b.ndim - 1];
    }
    if (epi->kind == TX_EPI_MUL_1MSQR || epi->kind == TX_EPI_MUL_AUX || epi->kind == TX_EPI_SGD ||
        epi->kind == TX_EPI_ADD_AUX_BIAS) {
      TX_CHECK(epi->aux.ndim == 2 && epi->aux.shape[0] == g->M && epi->aux.shape[1] == g->N, TX_E_ARG,
               "tx_gemm: epilogue operand must be [M,N]");
      s0 = epi->aux.strides[0];
      s1 = epi->aux.strides[1];
    } else {
      const tx_tensor& b = epi->aux;
      TX_CHECK(b.ndim >= 1 && b.shape[b.ndim - 1] == g->N, TX_E_ARG, "tx_gemm: bias must end in N");
      s1 = b.shape[b.ndim - 1] == 1 ? 0 : b.strides[b.ndim - 1];
    }
    if (epi->kind == TX_EPI_BIAS_TANH_DUAL) {
      const tx_tensor& o = epi->out2;
      TX_CHECK(o.dtype == A->dtype && o.ndim == 2 && o.shape[0] == g->M && o.shape[1] == g->N, TX_E_ARG,
               "tx_gemm: second epilogue output must be [M,N]");
      g->epi_f.out2 = (float*)o.data;
      g->epi_d.out2 = (double*)o.data;
      g->epi_f.o0 = g->epi_d.o0 = o.strides[0];
      g->epi_f.o1 = g->epi_d.o1 = o.strides[1];
    }
    g->epi_f.kind = g->epi_d.kind = epi->kind;
    g->epi_f.alpha = (float)epi->alpha;
    g->epi_d.alpha = epi->alpha;
    g->epi_f.aux = (const float*)epi->aux.data;
    g->epi_d.aux = (const double*)epi->aux.data;
    g->epi_f.s0 = g->epi_d.s0 = s0;
    g->epi_f.s1 = g->epi_d.s1 = s1;
  }
  return TX_OK;
}

// ---------------------------------------------------------------- 3xTF32
// fp32-equivalent products on the TF32 tensor cores (the reference's Dot is
// fp32 sgemm, ops/linalg.py:55-58).  Each operand x is split into
// big = tf32_rna(x) and small = tf32_rna(x - big) (x - big is exact in fp32),
// and C = A_big.B_big + A_big.B_small + A_small.B_big.  The three products
// are ONE tcgen05 GEMM over a K' = 3K contraction of plane-stacked operands
//     A' = [A_small | A_big | A_big]      B' = [B_big ; B_small ; B_big]
// so every tile schedule, split-K / stream-K path and fused epilogue of the
// TF32 kernel applies unchanged.  Dropped: A_small.B_small (<= 2^-22 |a||b|)
// and the TF32 rounding of the small parts (<= 2^-22 |a||b| each).
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// x viewed as [outer][inner] (strides so, si) -> three planes of
// y[plane * poff + o * ld + i]; plane `lo_plane` holds the small part.
__device__ __forceinline__ void split_one(float v, float& big, float& small) {
  big = tf32_rna(v);
  if (isinf(big) && !isinf(v)) big = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);  // no rounding to inf
  small = isfinite(big) ? tf32_rna(__fsub_rn(v, big)) : 0.0f;
}

// grid: x over inner (4 elements per thread when V4), y (grid-stride) over outer
template <bool V4>
__global__ void __launch_bounds__(256) tf32_split_kernel(const float* __restrict__ x, int64_t outer, int64_t inner,
                                                         int64_t so, int64_t si, float* __restrict__ y, int64_t ld,
                                                         int64_t poff, int lo_plane) {
  TX_GRID_WAIT();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * (V4 ? 4 : 1);
  if (i >= inner) return;
  for (int64_t o = blockIdx.y; o < outer; o += gridDim.y) {
    float* d = y + o * ld + i;
    if constexpr (V4) {  // si == 1, inner % 4 == 0, 16-byte aligned rows
      const float4 v = __ldcs(reinterpret_cast<const float4*>(x + o * so + i));
      float4 b, m;
      split_one(v.x, b.x, m.x);
      split_one(v.y, b.y, m.y);
      split_one(v.z, b.z, m.z);
      split_one(v.w, b.w, m.w);
#pragma unroll
      for (int j = 0; j < 3; ++j) *reinterpret_cast<float4*>(d + j * poff) = j == lo_plane ? m : b;
    } else {
      float b, m;
      split_one(__ldcs(x + o * so + i * si), b, m);
#pragma unroll
      for (int j = 0; j < 3; ++j) d[j * poff] = j == lo_plane ? m : b;
    }
  }
}

struct Split3 {
  G g3;             // the K' = 3K problem over the stacked planes
  size_t a_bytes, b_bytes;
  int64_t a_outer, a_inner, a_so, a_si, a_ld, a_poff;
  int64_t b_outer, b_inner, b_so, b_si, b_ld, b_poff;
};

inline int64_t up4(int64_t v) { return (v + 3) & ~(int64_t)3; }
inline size_t up256(size_t v) { return (v + 255) & ~(size_t)255; }

// plane geometry: keep each operand's contiguous dimension contiguous
void split3_plan(const G& g, Split3* s) {
  s->g3 = g;
  const int64_t K = g.K, K3 = 3 * g.K;
  if (g.sak == 1 || g.K == 1) {  // A K-major: rows [M][3K]
    s->a_outer = g.M; s->a_inner = K; s->a_so = g.sam; s->a_si = g.sak;
    s->a_ld = up4(K3); s->a_poff = K;
    s->g3.sam = s->a_ld; s->g3.sak = 1;
    s->a_bytes = (size_t)g.M * s->a_ld * 4;
  } else {                        // A M-major: rows [3K][M]
    s->a_outer = K; s->a_inner = g.M; s->a_so = g.sak; s->a_si = g.sam;
    s->a_ld = up4(g.M); s->a_poff = K * s->a_ld;
    s->g3.sam = 1; s->g3.sak = s->a_ld;
    s->a_bytes = (size_t)K3 * s->a_ld * 4;
  }
  if (g.sbn == 1 || g.N == 1) {  // B N-major: rows [3K][N]
    s->b_outer = K; s->b_inner = g.N; s->b_so = g.sbk; s->b_si = g.sbn;
    s->b_ld = up4(g.N); s->b_poff = K * s->b_ld;
    s->g3.sbn = 1; s->g3.sbk = s->b_ld;
    s->b_bytes = (size_t)K3 * s->b_ld * 4;
  } else {                        // B K-major: rows [N][3K]
    s->b_outer = g.N; s->b_inner = K; s->b_so = g.sbn; s->b_si = g.sbk;
    s->b_ld = up4(K3); s->b_poff = K;
    s->g3.sbk = 1; s->g3.sbn = s->b_ld;
    s->b_bytes = (size_t)g.N * s->b_ld * 4;
  }
  s->g3.K = K3;
  // accumulation promotion every few k-blocks (tc_gemm_kernel<_, PROMO>)
  // the small cross terms (planes 0-1: A_small.B_big, A_big.B_small) form the
  // first chunk; the big.big plane is promoted every `promo` k-blocks
  static const int promo = getenv("TX_3X_PROMO") ? atoi(getenv("TX_3X_PROMO")) : 4;
  s->g3.promo = promo;
  s->g3.promo_first = (int)((2 * K) / 32);
}

size_t split3_workspace(const G& g) {
  Split3 s;
  split3_plan(g, &s);
  return up256(s.a_bytes) + up256(s.b_bytes) + gemm_tc_workspace(s.g3) + 256;
}

// fill the planes into `ws` and return the 3K problem (operands in ws)
int split3_prepare(const G& g, void* ws, size_t wsb, cudaStream_t st, G* out, void** rest, size_t* rest_bytes) {
  Split3 s;
  split3_plan(g, &s);
  const size_t need = up256(s.a_bytes) + up256(s.b_bytes);
  uint8_t* base = (uint8_t*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  TX_CHECK(ws && wsb >= need + (size_t)(base - (uint8_t*)ws), TX_E_ARG, "tx_gemm: 3xtf32 workspace too small");
  float* Ap = (float*)base;
  float* Bp = (float*)(base + up256(s.a_bytes));
  const int sms = sm_count();
  auto launch = [&](const float* x, int64_t outer, int64_t inner, int64_t so, int64_t si, float* y, int64_t ld,
                    int64_t poff, int lo) {
    if (outer == 0 || inner == 0) return;
    const bool v4 = si == 1 && inner % 4 == 0 && so % 4 == 0 && ld % 4 == 0 && poff % 4 == 0 &&
                    ((uintptr_t)x & 15) == 0 && ((uintptr_t)y & 15) == 0;
    const int64_t per = v4 ? 1024 : 256;
    const int64_t bx = (inner + per - 1) / per;
    // ~16 resident blocks per SM in total; rows grid-strided
    const int64_t by = std::max<int64_t>(1, std::min<int64_t>(outer, std::min<int64_t>(65535, (int64_t)sms * 16 / bx + 1)));
    dim3 grid((unsigned)bx, (unsigned)by);
    if (v4) ::tx::launch(tf32_split_kernel<true>, dim3(grid), dim3(256), 0, st, x, outer, inner, so, si, y, ld, poff, lo);
    else ::tx::launch(tf32_split_kernel<false>, dim3(grid), dim3(256), 0, st, x, outer, inner, so, si, y, ld, poff, lo);
  };
  // A' = [small | big | big], B' = [big ; small ; big]: the cross terms first
  launch((const float*)g.A, s.a_outer, s.a_inner, s.a_so, s.a_si, Ap, s.a_ld, s.a_poff, 0);
  launch((const float*)g.B, s.b_outer, s.b_inner, s.b_so, s.b_si, Bp, s.b_ld, s.b_poff, 1);
  TX_CUDA(cudaGetLastError());
  *out = s.g3;
  out->A = Ap;
  out->B = Bp;

  const size_t used = need + (size_t)(base - (uint8_t*)ws);
  *rest = (uint8_t*)ws + used;
  *rest_bytes = wsb - used;
  return TX_OK;
}

// path + skinny kind
void choose(const G& g, int mode, int* path, int* kind) {
  *kind = -1;
  if (mode == TX_GEMM_SIMT || g.dtype == TX_F64) { *path = PATH_SIMT; return; }
  if (mode == TX_GEMM_TC) { *path = PATH_TC; return; }
  if (mode == TX_GEMM_3XTF32 && g.K > 16 && g.N > 16) {
    // the split re-lays both operands (aligned, padded pitches): only the
    // shape and C's layout decide
    Split3 s;
    split3_plan(g, &s);
    s.g3.A = s.g3.B = (const void*)256;
    if (gemm_tc_eligible(s.g3) == TX_OK) { *path = PATH_TC; return; }
  }
  if (g.K <= 16) { *path = PATH_SKINNY; *kind = SK_OUTER; return; }
  if (g.N <= 16 && g.sak == 1) { *path = PATH_SKINNY; *kind = SK_ROWDOT; return; }
  if (g.N <= 16 && g.sam == 1) { *path = PATH_SKINNY; *kind = SK_KRED; return; }
  static const bool no_smallm = getenv("TX_GEMM_NO_SMALLM") != nullptr;
  if (mode == TX_GEMM_AUTO && g.M <= SMALLM_MAX_M && g.N * g.K <= SMALLM_MAX_NK && !no_smallm) {
    *path = PATH_SKINNY; *kind = SK_SMALLM; return;
  }
  if (gemm_tc_eligible(g) == TX_OK) { *path = PATH_TC; return; }
  *path = PATH_SIMT;
}

// C^T = B^T A^T: turns an M <= 16 problem into an N <= 16 one
G transposed(const G& g) {
  G t = g;
  t.A = g.B; t.B = g.A;
  t.M = g.N; t.N = g.M;
  t.sam = g.sbn; t.sak = g.sbk;
  t.sbk = g.sak; t.sbn = g.sam;
  t.scm = g.scn; t.scn = g.scm;
  std::swap(t.epi_f.s0, t.epi_f.s1);
  std::swap(t.epi_d.s0, t.epi_d.s1);
  std::swap(t.epi_f.o0, t.epi_f.o1);
  std::swap(t.epi_d.o0, t.epi_d.o1);
  std::swap(t.epi_f.b0, t.epi_f.b1);
  std::swap(t.epi_d.b0, t.epi_d.b1);
  return t;
}

}  // namespace

int gemm_with_colsum(const tx_tensor* A, const tx_tensor* B, tx_tensor* C, const tx_epilogue* epi, int mode,
                     void* ws, size_t wsb, float* partials, cudaStream_t st) {
  G g;
  int rc = build(A, B, C, epi, &g);
  if (rc) return rc;
  int path, kind;
  choose(g, mode, &path, &kind);
  if (path != PATH_TC || g.dtype != TX_F32 || g.M == 0 || g.N == 0 || g.K == 0) return TX_E_UNSUPPORTED;
  g.colsum = partials;
  if (mode == TX_GEMM_3XTF32) {
    G g3;
    void* rest;
    size_t rb;
    if (split3_prepare(g, ws, wsb, st, &g3, &rest, &rb) != TX_OK) return TX_E_UNSUPPORTED;
    return gemm_tc(g3, nullptr, 0, st);
  }
  return gemm_tc(g, nullptr, 0, st);
}

}  // namespace tx

using namespace tx;

extern "C" {

int tx_gemm_path(const tx_tensor* A, const tx_tensor* B, const tx_tensor* C, int mode, int* path) {
  G g;
  int rc = build(A, B, C, nullptr, &g);
  if (rc) return rc;
  int kind;
  choose(g, mode, path, &kind);
  if (*path == PATH_SIMT && g.M <= 16 && (mode == TX_GEMM_AUTO || mode == TX_GEMM_3XTF32) && g.dtype == TX_F32) {
    G t = transposed(g);
    choose(t, mode, path, &kind);
  }
  return TX_OK;
}

int tx_gemm_workspace(const tx_tensor* A, const tx_tensor* B, const tx_tensor* C, int mode, size_t* bytes) {
  G g;
  int rc = build(A, B, C, nullptr, &g);
  if (rc) return rc;
  *bytes = 0;
  int path, kind;
  choose(g, mode, &path, &kind);
  if (path == PATH_SIMT && g.M <= 16 && (mode == TX_GEMM_AUTO || mode == TX_GEMM_3XTF32) && g.dtype == TX_F32) {
    g = transposed(g);
    choose(g, mode, &path, &kind);
  }
  if (path == PATH_SKINNY && kind == SK_KRED) *bytes = (size_t)kred_splits(g.M, g.K) * g.M * g.N * 4 + 256;
  if (path == PATH_TC) *bytes = mode == TX_GEMM_3XTF32 ? split3_workspace(g) : gemm_tc_workspace(g);
  return TX_OK;
}

int tx_gemm(const tx_tensor* A, const tx_tensor* B, tx_tensor* C, const tx_epilogue* epi, int mode, void* ws,
            size_t wsb, void* stream) {
  G g;
  int rc = build(A, B, C, epi, &g);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (g.M == 0 || g.N == 0) return TX_OK;
  if (g.K == 0) {
    TX_CHECK(!epi || epi->kind == TX_EPI_NONE, TX_E_UNSUPPORTED, "tx_gemm: K == 0 with an epilogue");
    TX_CHECK(is_contiguous(*C), TX_E_UNSUPPORTED, "tx_gemm: K == 0 needs a contiguous output");
    TX_CUDA(cudaMemsetAsync(C->data, 0, (size_t)(g.M * g.N) * itemsize(g.dtype), st));
    return TX_OK;
  }
  int path, kind;
  choose(g, mode, &path, &kind);
  if (path == PATH_SIMT && g.M <= 16 && (mode == TX_GEMM_AUTO || mode == TX_GEMM_3XTF32) && g.dtype == TX_F32) {
    G t = transposed(g);
    int p2, k2;
    choose(t, mode, &p2, &k2);
    if (p2 == PATH_SKINNY) return gemm_skinny(t, k2, ws, wsb, st);
  }
  if (path == PATH_TC && mode == TX_GEMM_3XTF32 && g.dtype == TX_F32) {
    G g3;
    void* rest;
    size_t rb;
    if ((rc = split3_prepare(g, ws, wsb, st, &g3, &rest, &rb))) return rc;
    return gemm_tc(g3, rest, rb, st);
  }
  switch (path) {
    case PATH_TC: return gemm_tc(g, ws, wsb, st);
    case PATH_SKINNY: return gemm_skinny(g, kind, ws, wsb, st);
    default: return gemm_simt(g, st);
  }
}

}  // extern "C"
