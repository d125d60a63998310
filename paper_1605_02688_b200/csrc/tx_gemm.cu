// tx_gemm: the Dot lowering entry point (reference ops/linalg.py:42-62).
// Chooses tcgen05 (large fp32), a memory-bound skinny kernel (one of M/N/K
// tiny), or the SIMT tile kernel (float64, or layouts TMA cannot address).
#include <cuda_runtime.h>

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
    TX_CHECK(epi->kind >= TX_EPI_BIAS && epi->kind <= TX_EPI_SGD, TX_E_ARG, "tx_gemm: unknown epilogue");
    int64_t s0 = 0, s1 = 0;
    if (epi->kind == TX_EPI_MUL_1MSQR || epi->kind == TX_EPI_MUL_AUX || epi->kind == TX_EPI_SGD) {
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

// path + skinny kind
void choose(const G& g, int mode, int* path, int* kind) {
  *kind = -1;
  if (mode == TX_GEMM_SIMT || g.dtype == TX_F64) { *path = PATH_SIMT; return; }
  if (mode == TX_GEMM_TC) { *path = PATH_TC; return; }
  if (g.K <= 16) { *path = PATH_SKINNY; *kind = SK_OUTER; return; }
  if (g.N <= 16 && g.sak == 1) { *path = PATH_SKINNY; *kind = SK_ROWDOT; return; }
  if (g.N <= 16 && g.sam == 1) { *path = PATH_SKINNY; *kind = SK_KRED; return; }
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
  return t;
}

}  // namespace

int gemm_with_colsum(const tx_tensor* A, const tx_tensor* B, tx_tensor* C, const tx_epilogue* epi, int mode,
                     float* partials, cudaStream_t st) {
  G g;
  int rc = build(A, B, C, epi, &g);
  if (rc) return rc;
  int path, kind;
  choose(g, mode, &path, &kind);
  if (path != PATH_TC || g.dtype != TX_F32 || g.M == 0 || g.N == 0 || g.K == 0) return TX_E_UNSUPPORTED;
  g.colsum = partials;
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
  if (*path == PATH_SIMT && g.M <= 16 && mode == TX_GEMM_AUTO && g.dtype == TX_F32) {
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
  if (path == PATH_SIMT && g.M <= 16 && mode == TX_GEMM_AUTO && g.dtype == TX_F32) {
    g = transposed(g);
    choose(g, mode, &path, &kind);
  }
  if (path == PATH_SKINNY && kind == SK_KRED) *bytes = (size_t)kred_splits(g.M, g.K) * g.M * g.N * 4 + 256;
  if (path == PATH_TC) *bytes = gemm_tc_workspace(g);
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
  if (path == PATH_SIMT && g.M <= 16 && mode == TX_GEMM_AUTO && g.dtype == TX_F32) {
    G t = transposed(g);
    int p2, k2;
    choose(t, mode, &p2, &k2);
    if (p2 == PATH_SKINNY) return gemm_skinny(t, k2, ws, wsb, st);
  }
  switch (path) {
    case PATH_TC: return gemm_tc(g, ws, wsb, st);
    case PATH_SKINNY: return gemm_skinny(g, kind, ws, wsb, st);
    default: return gemm_simt(g, st);
  }
}

}  // extern "C"
