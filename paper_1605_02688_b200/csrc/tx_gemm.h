// Internal GEMM problem description shared by the GEMM translation units.
#pragma once
#include <cuda_runtime.h>

#include "tx_common.h"

namespace tx {

// Fused epilogue, evaluated per output element with IEEE round-to-nearest
// intrinsics (no FMA contraction) so that it rounds exactly like the unfused
// elementwise nodes it replaces (add(b, dot) -> tanh, mul(dot, 1 - sqr(h))).
// apply() returns the primary output value; the DUAL kind also stores its
// second output as a side effect, so every GEMM path (tcgen05, skinny, SIMT)
// supports every epilogue through the same call.
template <class T>
struct Epi {
  int kind = TX_EPI_NONE;
  const T* aux = nullptr;
  int64_t s0 = 0, s1 = 0;  // aux strides (bias: s1 only; s0 after a transposition C^T = B^T A^T)
  T* out2 = nullptr;
  int64_t o0 = 0, o1 = 0;  // out2 strides
  T alpha = T(0);          // SGD learning rate
  const T* aux2 = nullptr; // ADD_AUX_BIAS: the bias row
  int64_t b0 = 0, b1 = 0;  // its strides (b1 along n; swapped with C^T = B^T A^T)
  __device__ __forceinline__ T apply(T acc, int64_t m, int64_t n) const;
};

template <>
__device__ __forceinline__ float Epi<float>::apply(float acc, int64_t m, int64_t n) const {
  switch (kind) {
    case TX_EPI_BIAS: return __fadd_rn(aux[m * s0 + n * s1], acc);
    case TX_EPI_BIAS_TANH: return tanhf(__fadd_rn(aux[m * s0 + n * s1], acc));
    case TX_EPI_MUL_1MSQR: {
      float h = aux[m * s0 + n * s1];
      return __fmul_rn(acc, __fsub_rn(1.0f, __fmul_rn(h, h)));
    }
    case TX_EPI_BIAS_TANH_DUAL: {
      const float h = tanhf(__fadd_rn(aux[m * s0 + n * s1], acc));
      out2[m * o0 + n * o1] = __fsub_rn(1.0f, __fmul_rn(h, h));
      return h;
    }
    case TX_EPI_MUL_AUX: return __fmul_rn(acc, aux[m * s0 + n * s1]);
    case TX_EPI_SGD: return __fsub_rn(aux[m * s0 + n * s1], __fmul_rn(alpha, acc));
    case TX_EPI_ADD_AUX_BIAS: return __fadd_rn(aux2[m * b0 + n * b1], __fadd_rn(aux[m * s0 + n * s1], acc));
  }
  return acc;
}

template <>
__device__ __forceinline__ double Epi<double>::apply(double acc, int64_t m, int64_t n) const {
  switch (kind) {
    case TX_EPI_BIAS: return __dadd_rn(aux[m * s0 + n * s1], acc);
    case TX_EPI_BIAS_TANH: return tanh(__dadd_rn(aux[m * s0 + n * s1], acc));
    case TX_EPI_MUL_1MSQR: {
      double h = aux[m * s0 + n * s1];
      return __dmul_rn(acc, __dsub_rn(1.0, __dmul_rn(h, h)));
    }
    case TX_EPI_BIAS_TANH_DUAL: {
      const double h = tanh(__dadd_rn(aux[m * s0 + n * s1], acc));
      out2[m * o0 + n * o1] = __dsub_rn(1.0, __dmul_rn(h, h));
      return h;
    }
    case TX_EPI_MUL_AUX: return __dmul_rn(acc, aux[m * s0 + n * s1]);
    case TX_EPI_SGD: return __dsub_rn(aux[m * s0 + n * s1], __dmul_rn(alpha, acc));
    case TX_EPI_ADD_AUX_BIAS: return __dadd_rn(aux2[m * b0 + n * b1], __dadd_rn(aux[m * s0 + n * s1], acc));
  }
  return acc;
}

struct G {
  int dtype;
  const void* A;
  const void* B;
  void* C;
  int64_t M, N, K;
  int64_t sam, sak, sbk, sbn, scm, scn;
  Epi<float> epi_f;
  Epi<double> epi_d;
  float* colsum = nullptr;  // tcgen05 path only: [ceil(M/32)][N] column sums of C per 32-row block
  int promo = 0;            // tcgen05 path only: k-blocks per accumulation-promotion chunk (0 = off) ...
  int promo_first = 0;      // ... after a first chunk of this many k-blocks
};

enum { PATH_SIMT = 0, PATH_SKINNY = 1, PATH_TC = 2 };
enum { SK_ROWDOT = 0, SK_OUTER = 1, SK_KRED = 2, SK_SMALLM = 3 };
// AUTO-mode products with M <= SMALLM_MAX_M and a B of at most SMALLM_MAX_NK
// elements take the SIMT small-M kernel (beyond that B streams from HBM and
// the tensor cores' FLOP headroom wins)
constexpr int SMALLM_MAX_M = 32;
constexpr int64_t SMALLM_MAX_NK = 1LL << 21;

int gemm_simt(const G& g, cudaStream_t st);
int gemm_skinny(const G& g, int kind, void* ws, size_t wsb, cudaStream_t st);
int kred_splits(int64_t M, int64_t K);
// tcgen05 path: returns TX_E_UNSUPPORTED if the layout is ineligible
int gemm_tc_eligible(const G& g);
int gemm_tc(const G& g, void* ws, size_t wsb, cudaStream_t st);
size_t gemm_tc_workspace(const G& g);
// implicit-GEMM stride-1 convolution (tx_conv_implicit)
int gemm_tc_conv(const float* xpad, int64_t N, int64_t Hp, int64_t Wp, int64_t C, const float* w, int64_t K, int kh,
                 int kw, float* out, int out_nchw, cudaStream_t st);
// C = A.B (+ epilogue) on the tcgen05 path with per-32-row-block column sums
// of C into `partials` ([ceil(M/32)][N] fp32); TX_E_UNSUPPORTED when the
// product does not take that path (caller reduces C separately)
int gemm_with_colsum(const tx_tensor* A, const tx_tensor* B, tx_tensor* C, const tx_epilogue* epi, int mode,
                     void* ws, size_t wsb, float* partials, cudaStream_t st);
void choose_tile(const G& g, int* cg, int* bn);
// C = epi(sum over splits of P[split][M][N]), fixed split order
int splitk_finalize(const float* P, const G& g, int splits, cudaStream_t st);
// stream-K fix-up: tiles whose k-range was split across clusters get
// C = epi(sum of their pieces in k order); whole tiles were stored directly
int streamk_fixup(const float* P, const G& g, int num_m, int num_n, int bm, int bn, int num_kb, int nclusters,
                  int group_m, cudaStream_t st = 0);

}  // namespace tx
