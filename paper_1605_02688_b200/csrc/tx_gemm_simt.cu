// CUDA-core GEMM kernels: the general SIMT tile kernel (float32 exact-FMA and
// float64) and the memory-bound skinny kernels used where one of M/N/K is tiny
// (the [B,10] softmax layer of every config: x.W, dz.W^T, x^T.dz).
//
// Replaces np.dot for those shapes (reference ops/linalg.py:42-62); the
// tensor-core path for large fp32 problems is tx_gemm_tc.cu.
#include <cuda_runtime.h>

#include "tx_common.h"
#include "tx_gemm.h"

namespace tx {
namespace {

// --------------------------------------------------------------- SIMT tiles
// 64x64 tile, 256 threads, 4x4 outputs per thread, BK = 16; arbitrary strides.
template <class T>
__global__ void __launch_bounds__(256) simt_gemm(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                                                int64_t M, int64_t N, int64_t K, int64_t sam, int64_t sak,
                                                int64_t sbk, int64_t sbn, int64_t scm, int64_t scn, Epi<T> epi) {
  __shared__ T As[16][64 + 1];
  __shared__ T Bs[16][64 + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    // load A tile 64x16 and B tile 16x64 (4 elements per thread each)
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      int r, c;
      if (sak == 1) { r = e / 16; c = e % 16; } else { r = e % 64; c = e / 64; }
      int64_t gm = m0 + r, gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? A[gm * sam + gk * sak] : T(0);
      int kr, nc;
      if (sbn == 1) { kr = e / 64; nc = e % 64; } else { kr = e % 16; nc = e / 16; }
      int64_t bk = k0 + kr, bn = n0 + nc;
      Bs[kr][nc] = (bk < K && bn < N) ? B[bk * sbk + bn * sbn] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t gn = n0 + tx * 4 + j;
      if (gn < N) C[gm * scm + gn * scn] = epi.apply(acc[i][j], gm, gn);
    }
  }
}

// ------------------------------------------------- N <= 16, A K-contiguous
// C[m, n] = sum_k A[m, k] B[k, n].  Block = 8 warps x 4 rows; B[kc:kc+256, :N]
// staged in shared memory and reused by all 32 rows of the block.
template <int NN>
__global__ void __launch_bounds__(256) rowdot_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                    float* __restrict__ C, int64_t M, int N, int64_t K, int64_t sam,
                                                    int64_t sbk, int64_t sbn, int64_t scm, int64_t scn, Epi<float> epi) {
  constexpr int KC = 256;
  __shared__ float Bs[KC][NN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * 32 + warp * 4;
  float acc[4][NN];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int n = 0; n < NN; ++n) acc[r][n] = 0.f;
  for (int64_t k0 = 0; k0 < K; k0 += KC) {
    __syncthreads();
    for (int e = threadIdx.x; e < KC * NN; e += 256) {
      int kk = e / NN, n = e % NN;
      int64_t gk = k0 + kk;
      Bs[kk][n] = (gk < K && n < N) ? B[gk * sbk + n * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t m = row0 + r;
      if (m >= M) break;
      const float* a = A + m * sam + k0;
#pragma unroll 4
      for (int j = 0; j < KC / 32; ++j) {
        const int kk = lane + 32 * j;
        const float av = (k0 + kk < K) ? __ldg(a + kk) : 0.f;
#pragma unroll
        for (int n = 0; n < NN; ++n) acc[r][n] += av * Bs[kk][n];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      float v = acc[r][n];
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      acc[r][n] = v;
    }
    const int64_t m = row0 + r;
    if (m < M && lane < N) {
      float v = 0.f;
#pragma unroll
      for (int n = 0; n < NN; ++n)
        if (n == lane) v = acc[r][n];
      C[m * scm + (int64_t)lane * scn] = epi.apply(v, m, lane);
    }
  }
}

// ------------------------------------------------ K <= 16 (outer-product-like)
// C[m, n] = sum_{k<K} A[m,k] B[k,n]; tile 32 rows x 256 cols; A and B tiles in smem.
template <int KK>
__global__ void __launch_bounds__(256) outer_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                   float* __restrict__ C, int64_t M, int64_t N, int K, int64_t sam,
                                                   int64_t sak, int64_t sbk, int64_t sbn, int64_t scm, int64_t scn,
                                                   Epi<float> epi) {
  __shared__ float As[32][KK];
  __shared__ float Bs[KK][256];
  const int64_t m0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 256;
  for (int e = threadIdx.x; e < 32 * KK; e += 256) {
    int r = e / KK, k = e % KK;
    As[r][k] = (m0 + r < M && k < K) ? A[(m0 + r) * sam + k * sak] : 0.f;
  }
  for (int e = threadIdx.x; e < KK * 256; e += 256) {
    int k, c;
    if (sbn == 1) { k = e / 256; c = e % 256; } else { k = e % KK; c = e / KK; }
    Bs[k][c] = (k < K && n0 + c < N) ? B[k * sbk + (n0 + c) * sbn] : 0.f;
  }
  __syncthreads();
  const int64_t n = n0 + threadIdx.x;
  if (n >= N) return;
  float b[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) b[k] = Bs[k][threadIdx.x];
  for (int r = 0; r < 32; ++r) {
    const int64_t m = m0 + r;
    if (m >= M) break;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < KK; ++k) acc += As[r][k] * b[k];
    C[m * scm + n * scn] = epi.apply(acc, m, n);
  }
}

// ------------------------------------- N <= 16, A M-contiguous (x^T . dz form)
// C[m, n] = sum_k A[k-th row][m] * B[k, n]: a column reduction over k.
// grid.x covers m (one column per thread), grid.y splits k; partials [S][M][N]
// are combined in order by kred_finalize (deterministic).
template <int NN>
__global__ void __launch_bounds__(256) kred_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                  float* __restrict__ P, int64_t M, int N, int64_t K, int64_t sak,
                                                  int64_t sbk, int64_t sbn, int splits) {
  constexpr int KC = 64;
  __shared__ float Bs[KC][NN];
  const int64_t m = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t chunk = (K + splits - 1) / splits;
  const int64_t klo = (int64_t)blockIdx.y * chunk, khi = min(K, klo + chunk);
  float acc[NN];
#pragma unroll
  for (int n = 0; n < NN; ++n) acc[n] = 0.f;
  for (int64_t k0 = klo; k0 < khi; k0 += KC) {
    __syncthreads();
    for (int e = threadIdx.x; e < KC * NN; e += 256) {
      int kk = e / NN, n = e % NN;
      Bs[kk][n] = (k0 + kk < khi && n < N) ? B[(k0 + kk) * sbk + n * sbn] : 0.f;
    }
    __syncthreads();
    if (m < M) {
      const int kend = (int)min((int64_t)KC, khi - k0);
      for (int kk = 0; kk < kend; ++kk) {
        const float av = __ldcs(A + (k0 + kk) * sak + m);
#pragma unroll
        for (int n = 0; n < NN; ++n) acc[n] += av * Bs[kk][n];
      }
    }
  }
  if (m < M) {
#pragma unroll
    for (int n = 0; n < NN; ++n)
      if (n < N) P[((int64_t)blockIdx.y * M + m) * N + n] = acc[n];
  }
}

__global__ void kred_finalize(const float* __restrict__ P, float* __restrict__ C, int64_t M, int N, int splits,
                              int64_t scm, int64_t scn, Epi<float> epi) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  int64_t m = e / N;
  int n = (int)(e - m * N);
  float v = 0.f;
  for (int s = 0; s < splits; ++s) v += P[((int64_t)s * M + m) * N + n];
  C[m * scm + n * scn] = epi.apply(v, m, n);
}

template <int NN>
static int launch_rowdot(const G& g, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.M + 31) / 32);
  rowdot_kernel<NN><<<blocks, 256, 0, st>>>((const float*)g.A, (const float*)g.B, (float*)g.C, g.M, (int)g.N, g.K,
                                            g.sam, g.sbk, g.sbn, g.scm, g.scn, g.epi_f);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

template <int KK>
static int launch_outer(const G& g, cudaStream_t st) {
  dim3 grid((unsigned)((g.N + 255) / 256), (unsigned)((g.M + 31) / 32));
  outer_kernel<KK><<<grid, 256, 0, st>>>((const float*)g.A, (const float*)g.B, (float*)g.C, g.M, g.N, (int)g.K, g.sam,
                                         g.sak, g.sbk, g.sbn, g.scm, g.scn, g.epi_f);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

template <int NN>
static int launch_kred(const G& g, void* ws, size_t wsb, cudaStream_t st) {
  int splits = kred_splits(g.M, g.K);
  TX_CHECK((size_t)splits * g.M * g.N * 4 <= wsb, TX_E_ARG, "tx_gemm: skinny workspace too small");
  dim3 grid((unsigned)((g.M + 255) / 256), (unsigned)splits);
  kred_kernel<NN><<<grid, 256, 0, st>>>((const float*)g.A, (const float*)g.B, (float*)ws, g.M, (int)g.N, g.K, g.sak,
                                        g.sbk, g.sbn, splits);
  int64_t tot = g.M * g.N;
  kred_finalize<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>((const float*)ws, (float*)g.C, g.M, (int)g.N, splits,
                                                              g.scm, g.scn, g.epi_f);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

}  // namespace

int kred_splits(int64_t M, int64_t K) {
  int64_t mblocks = (M + 255) / 256;
  int64_t want = (int64_t)sm_count() * 4;
  int64_t s = (want + mblocks - 1) / mblocks;
  int64_t maxs = K / 64;
  if (s > maxs) s = maxs;
  if (s > 1024) s = 1024;
  if (s < 1) s = 1;
  return (int)s;
}

int gemm_simt(const G& g, cudaStream_t st) {
  dim3 grid((unsigned)((g.N + 63) / 64), (unsigned)((g.M + 63) / 64));
  if (g.dtype == TX_F32)
    simt_gemm<float><<<grid, 256, 0, st>>>((const float*)g.A, (const float*)g.B, (float*)g.C, g.M, g.N, g.K, g.sam,
                                           g.sak, g.sbk, g.sbn, g.scm, g.scn, g.epi_f);
  else
    simt_gemm<double><<<grid, 256, 0, st>>>((const double*)g.A, (const double*)g.B, (double*)g.C, g.M, g.N, g.K,
                                            g.sam, g.sak, g.sbk, g.sbn, g.scm, g.scn, g.epi_d);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

int gemm_skinny(const G& g, int kind, void* ws, size_t wsb, cudaStream_t st) {
  if (kind == SK_OUTER) {
    if (g.K <= 4) return launch_outer<4>(g, st);
    if (g.K <= 8) return launch_outer<8>(g, st);
    return launch_outer<16>(g, st);
  }
  if (kind == SK_ROWDOT) {
    if (g.N <= 4) return launch_rowdot<4>(g, st);
    if (g.N <= 8) return launch_rowdot<8>(g, st);
    return launch_rowdot<16>(g, st);
  }
  if (g.N <= 4) return launch_kred<4>(g, ws, wsb, st);
  if (g.N <= 8) return launch_kred<8>(g, ws, wsb, st);
  return launch_kred<16>(g, ws, wsb, st);
}

}  // namespace tx
