// CUDA-core GEMM kernels: the general SIMT tile kernel (float32 exact-FMA and
// float64) and the memory-bound skinny kernels used where one of M/N/K is tiny
// (the [B,10] softmax layer of every config: x.W, dz.W^T, x^T.dz).
//
// Replaces np.dot for those shapes (reference ops/linalg.py:42-62); the
// tensor-core path for large fp32 problems is tx_gemm_tc.cu.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdlib>

#include "tx_common.h"
#include "tx_gemm.h"

namespace tx {
namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}

// --------------------------------------------------------------- SIMT tiles
// 64x64 tile, 256 threads, 4x4 outputs per thread, BK = 16; arbitrary strides.
template <class T>
__global__ void __launch_bounds__(256) simt_gemm(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                                                int64_t M, int64_t N, int64_t K, int64_t sam, int64_t sak,
                                                int64_t sbk, int64_t sbn, int64_t scm, int64_t scn, Epi<T> epi) {
  TX_GRID_WAIT();
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
// C[m, n] = sum_k A[m, k] B[k, n] (x.W3 / x.W in the softmax layers).  One
// warp owns R rows; B[k0:k0+KC, :N] is staged TRANSPOSED in shared memory
// (Bt[n][k]) so lanes read consecutive k (conflict-free 128-bit loads) and
// every row of the CTA reuses it.  A is streamed with 128-bit loads.
constexpr int RD_KC = 512;

template <int NN, int R>
__global__ void __launch_bounds__(256) rowdot_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                    float* __restrict__ C, int64_t M, int N, int64_t K, int64_t sam,
                                                    int64_t sbk, int64_t sbn, int64_t scm, int64_t scn, Epi<float> epi) {
  TX_GRID_WAIT();
  __shared__ __align__(16) float Bt[NN][RD_KC];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = ((int64_t)blockIdx.x * 8 + warp) * R;
  const bool vec = (sam % 4 == 0) && (((uintptr_t)A & 15) == 0);
  float acc[R][NN];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int n = 0; n < NN; ++n) acc[r][n] = 0.f;
  for (int64_t k0 = 0; k0 < K; k0 += RD_KC) {
    const int kc = (int)min((int64_t)RD_KC, K - k0);
    __syncthreads();
    if (sbn == 1) {
      for (int e = threadIdx.x; e < RD_KC * NN; e += 256) {
        const int kk = e / NN, n = e % NN;
        Bt[n][kk] = (kk < kc && n < N) ? B[(k0 + kk) * sbk + n] : 0.f;
      }
    } else {
      for (int e = threadIdx.x; e < RD_KC * NN; e += 256) {
        const int n = e / RD_KC, kk = e % RD_KC;
        Bt[n][kk] = (kk < kc && n < N) ? B[(k0 + kk) * sbk + n * sbn] : 0.f;
      }
    }
    __syncthreads();
    if (vec && kc == RD_KC) {
      // each B vector (NN float4 from smem) is reused by the warp's R rows:
      // R independent 128-bit A loads in flight, NN/R smem loads per A load
#pragma unroll
      for (int j = 0; j < RD_KC / 128; ++j) {
        const int kk = j * 128 + lane * 4;
        float4 bv[NN];
#pragma unroll
        for (int n = 0; n < NN; ++n) bv[n] = *reinterpret_cast<const float4*>(&Bt[n][kk]);
        float4 av[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
          av[r] = (row0 + r < M) ? __ldg(reinterpret_cast<const float4*>(A + (row0 + r) * sam + k0 + kk))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int n = 0; n < NN; ++n)
            acc[r][n] += av[r].x * bv[n].x + av[r].y * bv[n].y + av[r].z * bv[n].z + av[r].w * bv[n].w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t m = row0 + r;
        if (m >= M) break;
        const float* a = A + m * sam + k0;
        for (int kk = lane; kk < kc; kk += 32) {
          const float av = __ldg(a + kk);
#pragma unroll
          for (int n = 0; n < NN; ++n) acc[r][n] += av * Bt[n][kk];
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      float v = acc[r][n];
#pragma unroll
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

// Whole-K variant: B (K x NN fp32, its natural row-major layout) is staged
// ONCE per CTA in shared memory with cp.async (every thread issues all of its
// 16-byte copies back to back, so the staging is one latency, not one per
// element), and the CTA then walks row groups grid-stride (persistent): no
// per-chunk __syncthreads, each lane keeps R x 2 independent 128-bit A loads
// in flight.  Lane l handles k = 4l + 128j: the NN float4 at Bs[k*NN ..] are
// B rows k..k+3.  This is the HBM-bound form for h2.W3 ([8192,4096] x
// [4096,10]: 128 MB of A per call) and the logreg x.W.
constexpr int RDF_MAX_SMEM = 200 * 1024;


// TRANS: B is staged transposed, Bt[n][k] with the row pitch Kp = K rounded
// up to 32 plus 4 floats, so the per-lane 128-bit reads of 4 consecutive k of
// one column are bank-conflict free (the natural [k][n] layout puts lanes 160 B
// apart: two-way conflicts on every read); the staging reads B coalesced.
template <int NN, int R, bool TRANS = false>
__global__ void __launch_bounds__(R >= 8 ? 256 : 512) rowdot_full_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                         float* __restrict__ C, int64_t M, int N, int64_t K,
                                                         int64_t sam, int64_t sbk, int64_t sbn, int64_t scm,
                                                         int64_t scn, Epi<float> epi) {
  TX_GRID_WAIT();
  extern __shared__ __align__(16) float Bs[];  // [K][NN], or Bt [NN][Kp] when TRANS
  const int64_t total = K * NN;
  const int64_t Kp = ((K + 31) & ~(int64_t)31) + 4;
  if (TRANS) {
#pragma unroll 8
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int64_t k = e / NN;
      const int n = (int)(e - k * NN);
      Bs[n * Kp + k] = n < N ? B[k * sbk + (int64_t)n * sbn] : 0.f;
    }
  } else if (sbn == 1 && sbk == NN && N == NN && (((uintptr_t)B & 15) == 0) && total % 4 == 0) {
    for (int64_t e = threadIdx.x; e < total / 4; e += blockDim.x) cp_async16(Bs + 4 * e, B + 4 * e);
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
#pragma unroll 4
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int64_t k = e / NN;
      const int n = (int)(e - k * NN);
      Bs[e] = n < N ? B[k * sbk + (int64_t)n * sbn] : 0.f;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const bool vec = (sam % 4 == 0) && (K % 4 == 0) && (((uintptr_t)A & 15) == 0);
  for (int64_t g = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); g * R < M; g += (int64_t)gridDim.x * warps) {
    const int64_t row0 = g * R;
    float acc[R][NN];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int n = 0; n < NN; ++n) acc[r][n] = 0.f;
    if (vec) {
#pragma unroll 2
      for (int64_t kk = lane * 4; kk < K; kk += 128) {
        float4 av[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
          av[r] = (row0 + r < M) ? __ldcs(reinterpret_cast<const float4*>(A + (row0 + r) * sam + kk))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        if (TRANS) {
#pragma unroll
          for (int n = 0; n < NN; ++n) {
            const float4 bv = *reinterpret_cast<const float4*>(Bs + n * Kp + kk);
#pragma unroll
            for (int r = 0; r < R; ++r)
              acc[r][n] += av[r].x * bv.x + av[r].y * bv.y + av[r].z * bv.z + av[r].w * bv.w;
          }
        } else {
          // rows kk..kk+3 of B are NN float4 at a 16-byte aligned float4 index
          const float4* B4 = reinterpret_cast<const float4*>(Bs) + (kk >> 2) * NN;
          float b[4 * NN];
#pragma unroll
          for (int q = 0; q < NN; ++q) {
            const float4 t = B4[q];
            b[4 * q] = t.x; b[4 * q + 1] = t.y; b[4 * q + 2] = t.z; b[4 * q + 3] = t.w;
          }
          // four dependent FMAs straight into each accumulator (no separate
          // multiply + add per term): the loop is issue-bound, not memory-bound
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int n = 0; n < NN; ++n) {
              float a_ = acc[r][n];
              a_ = fmaf(av[r].x, b[n], a_);
              a_ = fmaf(av[r].y, b[NN + n], a_);
              a_ = fmaf(av[r].z, b[2 * NN + n], a_);
              acc[r][n] = fmaf(av[r].w, b[3 * NN + n], a_);
            }
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t m = row0 + r;
        if (m >= M) break;
        const float* a = A + m * sam;
        for (int64_t kk = lane; kk < K; kk += 32) {
          const float av = __ldg(a + kk);
#pragma unroll
          for (int n = 0; n < NN; ++n) acc[r][n] += av * (TRANS ? Bs[n * Kp + kk] : Bs[kk * NN + n]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        float v = acc[r][n];
#pragma unroll
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
}

// ------------------------------------------------ K <= 16 (outer-product-like)
// C[m, n] = sum_{k<K} A[m,k] B[k,n] (dz.W3^T).  CTA tile 32 rows x 1024 cols,
// 4 adjacent columns per thread held in registers, A tile broadcast from smem,
// 128-bit stores; writing C is the whole cost.
template <int KK>
__global__ void __launch_bounds__(256) outer_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                   float* __restrict__ C, int64_t M, int64_t N, int K, int64_t sam,
                                                   int64_t sak, int64_t sbk, int64_t sbn, int64_t scm, int64_t scn,
                                                   Epi<float> epi) {
  TX_GRID_WAIT();
  __shared__ float As[32][KK];
  const int64_t m0 = (int64_t)blockIdx.y * 32;
  const int64_t n0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
  for (int e = threadIdx.x; e < 32 * KK; e += 256) {
    const int r = e / KK, k = e % KK;
    As[r][k] = (m0 + r < M && k < K) ? A[(m0 + r) * sam + k * sak] : 0.f;
  }
  __syncthreads();
  if (n0 >= N) return;
  float b[KK][4];
#pragma unroll
  for (int k = 0; k < KK; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) b[k][j] = (k < K && n0 + j < N) ? __ldg(B + k * sbk + (n0 + j) * sbn) : 0.f;
  const bool vst = scn == 1 && (scm % 4 == 0) && (((uintptr_t)C & 15) == 0) && n0 + 4 <= N;
  const int rows = (int)min((int64_t)32, M - m0);
  // [M,N] epilogue operand read with 128-bit loads, 4 rows in flight (dH*g:
  // reading the aux tensor is half of this kernel's traffic)
  const bool vaux = vst && (epi.kind == TX_EPI_MUL_AUX || epi.kind == TX_EPI_MUL_1MSQR) && epi.s1 == 1 &&
                    (epi.s0 % 4 == 0) && (((uintptr_t)epi.aux & 15) == 0);
  if (vaux && rows == 32) {
#pragma unroll 1
    for (int r0 = 0; r0 < 32; r0 += 4) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldcs(reinterpret_cast<const float4*>(epi.aux + (m0 + r0 + u) * epi.s0 + n0));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u;
        float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < KK; ++k) {
          const float av = As[r][k];
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] += av * b[k][j];
        }
        float g[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float f = epi.kind == TX_EPI_MUL_AUX ? g[j] : __fsub_rn(1.0f, __fmul_rn(g[j], g[j]));
          o[j] = __fmul_rn(o[j], f);
        }
        __stcs(reinterpret_cast<float4*>(C + (m0 + r) * scm + n0), make_float4(o[0], o[1], o[2], o[3]));
      }
    }
    return;
  }
  for (int r = 0; r < rows; ++r) {
    const int64_t m = m0 + r;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      const float av = As[r][k];
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] += av * b[k][j];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (n0 + j < N) o[j] = epi.apply(o[j], m, n0 + j);
    if (vst) {
      *reinterpret_cast<float4*>(C + m * scm + n0) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
      for (int j = 0; j < 4 && n0 + j < N; ++j) C[m * scm + (n0 + j) * scn] = o[j];
    }
  }
}

// ------------------------------------- N <= 16, A M-contiguous (x^T . dz form)
// C[m, n] = sum_k A[k*sak + m] * B[k, n]: a column reduction over k.  Each
// thread owns 4 adjacent m (128-bit loads along the contiguous M axis) and
// keeps KR_U of them in flight; B rows are broadcast from smem; grid.y splits
// k and writes partials [S][M][N] that kred_finalize sums in fixed order
// (deterministic, no atomics).  128-thread CTAs (512 m per CTA) keep the
// partial volume S*M*N small for a given CTA count.
constexpr int KR_KC = 64;
constexpr int KR_THREADS = 128;
constexpr int KR_U = 8;

template <int NN>
__global__ void __launch_bounds__(KR_THREADS) kred_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                         float* __restrict__ P, int64_t M, int N, int64_t K,
                                                         int64_t sak, int64_t sbk, int64_t sbn, int splits) {
  TX_GRID_WAIT();
  __shared__ float Bs[KR_KC][NN];
  const int64_t m0 = ((int64_t)blockIdx.x * KR_THREADS + threadIdx.x) * 4;
  const int64_t chunk = (K + splits - 1) / splits;
  const int64_t klo = (int64_t)blockIdx.y * chunk, khi = min(K, klo + chunk);
  const bool vec = (sak % 4 == 0) && (((uintptr_t)A & 15) == 0) && m0 + 4 <= M;
  float acc[4][NN];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int n = 0; n < NN; ++n) acc[j][n] = 0.f;
  for (int64_t k0 = klo; k0 < khi; k0 += KR_KC) {
    __syncthreads();
    for (int e = threadIdx.x; e < KR_KC * NN; e += KR_THREADS) {
      const int kk = e / NN, n = e % NN;
      Bs[kk][n] = (k0 + kk < khi && n < N) ? B[(k0 + kk) * sbk + n * sbn] : 0.f;
    }
    __syncthreads();
    if (m0 < M) {
      const int kend = (int)min((int64_t)KR_KC, khi - k0);
      if (vec) {
        int kk = 0;
        for (; kk + KR_U <= kend; kk += KR_U) {
          float4 av[KR_U];
#pragma unroll
          for (int u = 0; u < KR_U; ++u) av[u] = __ldcs(reinterpret_cast<const float4*>(A + (k0 + kk + u) * sak + m0));
#pragma unroll
          for (int u = 0; u < KR_U; ++u)
#pragma unroll
            for (int n = 0; n < NN; ++n) {
              const float bv = Bs[kk + u][n];
              acc[0][n] += av[u].x * bv;
              acc[1][n] += av[u].y * bv;
              acc[2][n] += av[u].z * bv;
              acc[3][n] += av[u].w * bv;
            }
        }
        for (; kk < kend; ++kk) {
          const float4 av = __ldcs(reinterpret_cast<const float4*>(A + (k0 + kk) * sak + m0));
#pragma unroll
          for (int n = 0; n < NN; ++n) {
            const float bv = Bs[kk][n];
            acc[0][n] += av.x * bv;
            acc[1][n] += av.y * bv;
            acc[2][n] += av.z * bv;
            acc[3][n] += av.w * bv;
          }
        }
      } else {
        for (int kk = 0; kk < kend; ++kk) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (m0 + j >= M) break;
            const float av = A[(k0 + kk) * sak + m0 + j];
#pragma unroll
            for (int n = 0; n < NN; ++n) acc[j][n] += av * Bs[kk][n];
          }
        }
      }
    }
  }
  for (int j = 0; j < 4; ++j) {
    const int64_t m = m0 + j;
    if (m >= M) break;
#pragma unroll
    for (int n = 0; n < NN; ++n)
      if (n < N) P[((int64_t)blockIdx.y * M + m) * N + n] = acc[j][n];
  }
}

// Ring variant (M % 4 == 0, aligned, M-contiguous A): every thread streams its
// own 16-byte column slice of A rows through a KR_S-stage cp.async ring in
// shared memory (KR_S x KR_RU rows in flight per thread, independent of the
// register budget), and the CTA's slice of B (chunk x NN) is staged once.
// Only the issuing thread reads its ring slots, so there is no CTA barrier in
// the loop.
constexpr int KR_S = 4, KR_RU = 4;

template <int NN>
__global__ void __launch_bounds__(KR_THREADS) kred_ring_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                              float* __restrict__ P, int64_t M, int N, int64_t K,
                                                              int64_t sak, int64_t sbk, int64_t sbn, int splits) {
  TX_GRID_WAIT();
  extern __shared__ __align__(16) float4 kr_smem[];
  float4* ring = kr_smem;                                                  // [KR_S*KR_RU][KR_THREADS]
  float* Bs = reinterpret_cast<float*>(kr_smem + KR_S * KR_RU * KR_THREADS);  // [chunk][NN]
  const int tid = threadIdx.x;
  const int64_t m0 = ((int64_t)blockIdx.x * KR_THREADS + tid) * 4;
  const int64_t chunk = (K + splits - 1) / splits;
  const int64_t klo = (int64_t)blockIdx.y * chunk, khi = min(K, klo + chunk);
  const int nrows = (int)max((int64_t)0, khi - klo);
#pragma unroll 4
  for (int e = tid; e < nrows * NN; e += KR_THREADS) {
    const int k = e / NN, n = e - k * NN;
    Bs[e] = n < N ? B[(klo + k) * sbk + (int64_t)n * sbn] : 0.f;
  }
  __syncthreads();
  const bool active = m0 < M;
  const float* a0 = A + klo * sak + m0;
  auto issue = [&](int r0) {
#pragma unroll
    for (int u = 0; u < KR_RU; ++u) {
      const int r = r0 + u;
      if (active && r < nrows) cp_async16(&ring[(r % (KR_S * KR_RU)) * KR_THREADS + tid], a0 + (int64_t)r * sak);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int st = 0; st < KR_S; ++st) issue(st * KR_RU);
  float acc[4][NN];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int n = 0; n < NN; ++n) acc[j][n] = 0.f;
  for (int r0 = 0; r0 < nrows; r0 += KR_RU) {
    asm volatile("cp.async.wait_group %0;" ::"n"(KR_S - 1) : "memory");
#pragma unroll
    for (int u = 0; u < KR_RU; ++u) {
      const int r = r0 + u;
      if (r < nrows) {
        const float4 av = ring[(r % (KR_S * KR_RU)) * KR_THREADS + tid];
#pragma unroll
        for (int n = 0; n < NN; ++n) {
          const float bv = Bs[r * NN + n];
          acc[0][n] += av.x * bv;
          acc[1][n] += av.y * bv;
          acc[2][n] += av.z * bv;
          acc[3][n] += av.w * bv;
        }
      }
    }
    issue(r0 + KR_S * KR_RU);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (!active) return;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t m = m0 + j;
#pragma unroll
    for (int n = 0; n < NN; ++n)
      if (n < N) P[((int64_t)blockIdx.y * M + m) * N + n] = acc[j][n];
  }
}

// sums the S partials of each output in split order; 8 independent loads in
// flight per thread (the adds stay in order, so the result is deterministic)
__global__ void kred_finalize(const float* __restrict__ P, float* __restrict__ C, int64_t M, int N, int splits,
                              int64_t scm, int64_t scn, Epi<float> epi) {
  TX_GRID_WAIT();
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t MN = M * N;
  if (e >= MN) return;
  int64_t m = e / N;
  int n = (int)(e - m * N);
  float v = 0.f;
  int s = 0;
  for (; s + 8 <= splits; s += 8) {
    float q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = __ldcs(P + (int64_t)(s + u) * MN + e);
#pragma unroll
    for (int u = 0; u < 8; ++u) v += q[u];
  }
  for (; s < splits; ++s) v += P[(int64_t)s * MN + e];
  C[m * scm + n * scn] = epi.apply(v, m, n);
}

// Many splits (the skinny K reductions: up to 1024 partials of a few
// thousand outputs): 32 outputs per CTA, the splits interleaved over its 8
// warps, partials added in warp order (deterministic) -- 8x the loads in
// flight of one thread walking every split.
__global__ void __launch_bounds__(256) kred_finalize_wide(const float* __restrict__ P, float* __restrict__ C,
                                                          int64_t M, int N, int splits, int64_t scm, int64_t scn,
                                                          Epi<float> epi) {
  TX_GRID_WAIT();
  __shared__ float part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t MN = M * N;
  const int64_t e = blockIdx.x * 32LL + lane;
  float v = 0.f;
  if (e < MN) {
    int s = w;
    for (; s + 24 < splits; s += 32) {
      const float q0 = __ldcs(P + (int64_t)s * MN + e), q1 = __ldcs(P + (int64_t)(s + 8) * MN + e);
      const float q2 = __ldcs(P + (int64_t)(s + 16) * MN + e), q3 = __ldcs(P + (int64_t)(s + 24) * MN + e);
      v += q0; v += q1; v += q2; v += q3;
    }
    for (; s < splits; s += 8) v += P[(int64_t)s * MN + e];
  }
  part[w][lane] = v;
  __syncthreads();
  if (w != 0 || e >= MN) return;
  float t = part[0][lane];
#pragma unroll
  for (int u = 1; u < 8; ++u) t += part[u][lane];
  const int64_t m = e / N;
  const int n = (int)(e - m * N);
  C[m * scm + n * scn] = epi.apply(t, m, n);
}

template <int NN, int R, bool TRANS = false>
static int launch_rowdot_full(const G& g, int threads, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    TX_CUDA(cudaFuncSetAttribute(rowdot_full_kernel<NN, R, TRANS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 RDF_MAX_SMEM));
    attr = true;
  }
  if (TRANS) smem = (size_t)NN * (size_t)(((g.K + 31) & ~(int64_t)31) + 4) * 4;
  const int warps = threads / 32;
  int64_t groups = (g.M + R - 1) / R;
  int64_t blocks = (groups + warps - 1) / warps;
  const int per_sm = (int)(RDF_MAX_SMEM / (smem + 1024)) > 0 ? (int)(RDF_MAX_SMEM / (smem + 1024)) : 1;
  const int64_t cap = (int64_t)sm_count() * (per_sm < 4 ? per_sm : 4);
  if (blocks > cap) blocks = cap;
  ::tx::launch(rowdot_full_kernel<NN, R, TRANS>, dim3((unsigned)blocks), dim3(threads), smem, st, (const float*)g.A, (const float*)g.B, (float*)g.C,
                                                                     g.M, (int)g.N, g.K, g.sam, g.sbk, g.sbn, g.scm,
                                                                     g.scn, g.epi_f);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

template <int NN>
static int launch_rowdot(const G& g, cudaStream_t st) {
  const size_t smem = (size_t)NN * (size_t)g.K * 4;
  if (smem <= (size_t)RDF_MAX_SMEM) {
    // many rows: 16 warps x 4 rows per CTA, one CTA per SM; few rows (logreg):
    // 4-warp CTAs, one row per warp, to spread over the SMs
    if (g.M >= 4096) {
      const char* v = getenv("TX_RD_VARIANT");
      const int var = v ? atoi(v) : 0;
      if constexpr (NN <= 10) {
        if (var == 1) return launch_rowdot_full<NN, 8>(g, 256, smem, st);
        if (var == 2) return launch_rowdot_full<NN, 2>(g, 512, smem, st);
        if (var == 3) return launch_rowdot_full<NN, 4, true>(g, 512, smem, st);
        if (var == 4) return launch_rowdot_full<NN, 2, true>(g, 512, smem, st);
      }
      return launch_rowdot_full<NN, (NN <= 10 ? 4 : 2)>(g, 512, smem, st);
    }
    return launch_rowdot_full<NN, 1>(g, 128, smem, st);
  }
  if (g.M >= 4096) {
    unsigned blocks = (unsigned)((g.M + 31) / 32);
    ::tx::launch(rowdot_kernel<NN, 4>, dim3(blocks), dim3(256), 0, st, (const float*)g.A, (const float*)g.B, (float*)g.C, g.M, (int)g.N,
                                                 g.K, g.sam, g.sbk, g.sbn, g.scm, g.scn, g.epi_f);
  } else {
    unsigned blocks = (unsigned)((g.M + 7) / 8);
    ::tx::launch(rowdot_kernel<NN, 1>, dim3(blocks), dim3(256), 0, st, (const float*)g.A, (const float*)g.B, (float*)g.C, g.M, (int)g.N,
                                                 g.K, g.sam, g.sbk, g.sbn, g.scm, g.scn, g.epi_f);
  }
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

template <int KK>
static int launch_outer(const G& g, cudaStream_t st) {
  dim3 grid((unsigned)((g.N + 1023) / 1024), (unsigned)((g.M + 31) / 32));
  ::tx::launch(outer_kernel<KK>, dim3(grid), dim3(256), 0, st, (const float*)g.A, (const float*)g.B, (float*)g.C, g.M, g.N, (int)g.K, g.sam,
                                         g.sak, g.sbk, g.sbn, g.scm, g.scn, g.epi_f);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

template <int NN>
static int launch_kred(const G& g, void* ws, size_t wsb, cudaStream_t st) {
  int splits = kred_splits(g.M, g.K);
  TX_CHECK((size_t)splits * g.M * g.N * 4 <= wsb, TX_E_ARG, "tx_gemm: skinny workspace too small");
  dim3 grid((unsigned)((g.M + 4 * KR_THREADS - 1) / (4 * KR_THREADS)), (unsigned)splits);
  const int64_t chunk = (g.K + splits - 1) / splits;
  const size_t smem = (size_t)KR_S * KR_RU * KR_THREADS * 16 + (size_t)chunk * NN * 4;
  if (g.M % 4 == 0 && g.sak % 4 == 0 && ((uintptr_t)g.A & 15) == 0 && smem <= 48 * 1024) {
    ::tx::launch(kred_ring_kernel<NN>, dim3(grid), dim3(KR_THREADS), smem, st, (const float*)g.A, (const float*)g.B, (float*)ws, g.M,
                                                         (int)g.N, g.K, g.sak, g.sbk, g.sbn, splits);
  } else
  ::tx::launch(kred_kernel<NN>, dim3(grid), dim3(KR_THREADS), 0, st, (const float*)g.A, (const float*)g.B, (float*)ws, g.M, (int)g.N, g.K, g.sak,
                                        g.sbk, g.sbn, splits);
  int64_t tot = g.M * g.N;
  if (splits >= 32)
    ::tx::launch(kred_finalize_wide, dim3((unsigned)((tot + 31) / 32)), dim3(256), 0, st, (const float*)ws, (float*)g.C, g.M,
                 (int)g.N, splits, g.scm, g.scn, g.epi_f);
  else
  ::tx::launch(kred_finalize, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, (const float*)ws, (float*)g.C, g.M, (int)g.N, splits,
                                                              g.scm, g.scn, g.epi_f);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}


// ------------------------------------------------ M <= 32: few rows, any N, K
// The recurrent products of an unrolled scan (h.W_h, dz.W_h^T: M = the
// minibatch, 20 in the LSTM configs) are too thin for a 128-row tcgen05 tile:
// the tensor-core kernel's fixed cost (TMEM allocation, barrier set-up, one
// k-block pipeline fill, TMEM drain) was ~10 us per launch on [20 x 800 x 200].
// Here one CTA owns 32 output columns (one per lane) and a K range; its 8
// warps take interleaved groups of 8 k-rows.  A is staged per 256-row piece
// in shared memory as [m][k] rows (16-byte cp.async when A is K-contiguous),
// read back as broadcast float4s along k, so the accumulator count is M
// rounded up to 4 (no padding to a tile).  Every load of a piece (this
// warp's <= 4 B groups: 128-byte coalesced rows for N-major B, two 16-byte
// vectors per lane for K-major B) is issued before its first use.  The K
// range is split over a thread-block cluster (<= 8 CTAs); the column blocks'
// partials are summed by rank 0 through distributed shared memory in rank
// order and the fused epilogue is applied: one launch, deterministic, exact
// fp32 FMAs (tighter than the TF32 tensor-core path it replaces).
constexpr int SMM_THREADS = 256;
constexpr int SMM_KP = 128;       // k rows per staged A piece
constexpr int SMM_KPP = SMM_KP + 4;  // row pitch (16-byte aligned; spreads the transposing stage's banks)

__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, int bytes, int valid) {
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(valid) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(valid) : "memory");
}

// BMODE 0: N-major B (sbn == 1); 1: K-major B, 16-byte vectors; 2: generic strides.
// AK: A K-contiguous with 16-byte aligned rows (16-byte staging).
template <int MT, int BMODE, bool AK>
__global__ void __launch_bounds__(SMM_THREADS, 2) smallm_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                               float* __restrict__ C, int M, int N, int64_t K,
                                                               int64_t sam, int64_t sak, int64_t sbk, int64_t sbn,
                                                               int64_t scm, int64_t scn, Epi<float> epi, int64_t kchunk) {
  TX_GRID_WAIT();
  constexpr int STAGE = MT * SMM_KPP, RED = 8 * MT * 32;
  __shared__ __align__(16) float smem[STAGE > RED ? STAGE : RED];
  __shared__ float part[MT * 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.x * 32;
  const int n = n0 + lane;
  const bool nok = n < N;
  const int64_t klo = (int64_t)blockIdx.y * kchunk;
  const int64_t khi = klo + kchunk < K ? klo + kchunk : K;
  float acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m] = 0.f;
  auto load_b = [&](int64_t k, int avail, float (&b)[8]) {  // k rows [k, k + 8) of column n (zero past `avail`)
    if (BMODE == 1 && avail >= 8 && nok) {
      const float4* bp = reinterpret_cast<const float4*>(B + (int64_t)n * sbn + k);
      const float4 u = __ldg(bp), w = __ldg(bp + 1);
      b[0] = u.x; b[1] = u.y; b[2] = u.z; b[3] = u.w; b[4] = w.x; b[5] = w.y; b[6] = w.z; b[7] = w.w;
    } else {
      const float* bp = B + k * sbk + (BMODE == 0 ? (int64_t)n : (int64_t)n * sbn);
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = (i < avail && nok) ? __ldg(bp + i * sbk) : 0.f;
    }
  };
  const int g0 = warp * 8;
  for (int64_t p0 = klo; p0 < khi; p0 += SMM_KP) {
    const int rows = (int)(khi - p0 < SMM_KP ? khi - p0 : SMM_KP);
    const int rows8 = (rows + 7) & ~7;  // whole 8-row groups; k in [rows, rows8) stage as zeros
    float bq[SMM_KP / 64][8];
#pragma unroll
    for (int q = 0; q < SMM_KP / 64; ++q)
      if (g0 + 64 * q < rows) load_b(p0 + g0 + 64 * q, rows - g0 - 64 * q, bq[q]);
    __syncthreads();  // the previous piece is consumed
    if (AK) {  // 16-byte chunks of A rows: MT x SMM_KP / 4 chunks
#pragma unroll
      for (int u = 0; u < (MT * SMM_KP / 4 + SMM_THREADS - 1) / SMM_THREADS; ++u) {
        const int e = tid + u * SMM_THREADS;
        const int m = e / (SMM_KP / 4), c = (e % (SMM_KP / 4)) * 4;
        if (m < M && c < rows8) {
          const int valid = rows - c >= 4 ? 16 : (rows > c ? (rows - c) * 4 : 0);
          cp_async_zfill(smem + m * SMM_KPP + c, valid ? A + (int64_t)m * sam + p0 + c : A, 16, valid);
        }
      }
    } else {
#pragma unroll 4
      for (int u = 0; u < MT * SMM_KP / SMM_THREADS; ++u) {
        const int e = tid + u * SMM_THREADS;
        int r, m;
        if (sam == 1) { r = e / MT; m = e - r * MT; }  // A M-contiguous: m fastest
        else { m = e / SMM_KP; r = e % SMM_KP; }       // k fastest
        if (m < M && r < rows8) {
          const bool ok = r < rows;
          cp_async_zfill(smem + m * SMM_KPP + r, ok ? A + (int64_t)m * sam + (p0 + r) * sak : A, 4, ok ? 4 : 0);
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int q = 0; q < SMM_KP / 64; ++q) {
      const int g = g0 + 64 * q;
      if (g >= rows) break;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const float4* a4 = reinterpret_cast<const float4*>(smem + m * SMM_KPP + g);
        const float4 u = a4[0], w = a4[1];
        float a = acc[m];
        a = fmaf(u.x, bq[q][0], a); a = fmaf(u.y, bq[q][1], a); a = fmaf(u.z, bq[q][2], a); a = fmaf(u.w, bq[q][3], a);
        a = fmaf(w.x, bq[q][4], a); a = fmaf(w.y, bq[q][5], a); a = fmaf(w.z, bq[q][6], a); a = fmaf(w.w, bq[q][7], a);
        acc[m] = a;
      }
    }
  }
  // warps -> CTA partial (fixed warp order)
  __syncthreads();
#pragma unroll
  for (int m = 0; m < MT; ++m) smem[(warp * MT + m) * 32 + lane] = acc[m];
  __syncthreads();
  for (int e = tid; e < MT * 32; e += SMM_THREADS) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += smem[w * MT * 32 + e];
    part[e] = v;
  }
  namespace cg = cooperative_groups;
  const int cs = (int)gridDim.y;
  if (cs > 1) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if (cl.block_rank() == 0) {
#pragma unroll 1
      for (int e = tid; e < MT * 32; e += SMM_THREADS) {
        const int m = e >> 5, c = n0 + (e & 31);
        if (m >= M || c >= N) continue;
        float v = part[e];
        for (int r = 1; r < cs; ++r) v += cl.map_shared_rank(part, r)[e];
        C[(int64_t)m * scm + (int64_t)c * scn] = epi.kind != TX_EPI_NONE ? epi.apply(v, m, c) : v;
      }
    }
    cl.sync();  // the other ranks' partials stay resident until rank 0 has read them
    return;
  }
  __syncthreads();
#pragma unroll 1
  for (int e = tid; e < MT * 32; e += SMM_THREADS) {
    const int m = e >> 5, c = n0 + (e & 31);
    if (m >= M || c >= N) continue;
    const float v = part[e];
    C[(int64_t)m * scm + (int64_t)c * scn] = epi.kind != TX_EPI_NONE ? epi.apply(v, m, c) : v;
  }
}

template <int MT, int BMODE, bool AK>
static int launch_smallm_t(const G& g, int cs, int64_t kchunk, cudaStream_t st) {
  const unsigned strips = (unsigned)((g.N + 31) / 32);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(strips, (unsigned)cs, 1);
  cfg.blockDim = dim3(SMM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = (unsigned)cs;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  TX_CUDA(cudaLaunchKernelEx(&cfg, smallm_kernel<MT, BMODE, AK>, (const float*)g.A, (const float*)g.B, (float*)g.C,
                             (int)g.M, (int)g.N, g.K, g.sam, g.sak, g.sbk, g.sbn, g.scm, g.scn, g.epi_f, kchunk));
  return TX_OK;
}

template <int MT, int BMODE>
static int launch_smallm_b(const G& g, int cs, int64_t kchunk, cudaStream_t st) {
  const bool ak = g.sak == 1 && g.sam % 4 == 0 && ((uintptr_t)g.A & 15) == 0;
  return ak ? launch_smallm_t<MT, BMODE, true>(g, cs, kchunk, st) : launch_smallm_t<MT, BMODE, false>(g, cs, kchunk, st);
}

template <int MT>
static int launch_smallm_m(const G& g, int cs, int64_t kchunk, cudaStream_t st) {
  if (g.sbn == 1) return launch_smallm_b<MT, 0>(g, cs, kchunk, st);
  if (g.sbk == 1 && g.sbn % 4 == 0 && ((uintptr_t)g.B & 15) == 0) return launch_smallm_b<MT, 1>(g, cs, kchunk, st);
  return launch_smallm_b<MT, 2>(g, cs, kchunk, st);
}

static int launch_smallm(const G& g, cudaStream_t st) {
  // cluster split of K: about two CTAs per SM overall while every warp keeps
  // >= 32 k-rows (its fixed costs -- staging, reduction -- stay amortised)
  const int64_t strips = (g.N + 31) / 32;
  int64_t cs = (2 * (int64_t)sm_count() + strips - 1) / strips;
  if (cs > 8) cs = 8;
  if (cs > g.K / 256) cs = g.K / 256;
  // small products (B of <= 2^18 elements) are latency-bound: one staged
  // piece per CTA where the cluster allows, i.e. fewer serial load rounds
  // (LSTM small 797 -> 765 us per batch; the medium model's larger products
  // keep the rule above, 1816 vs 1937 us).  TX_SMALLM_CS=0/1/k+1 for A/B.
  static const int rule_env = getenv("TX_SMALLM_CS") ? atoi(getenv("TX_SMALLM_CS")) : -1;
  const int rule = rule_env >= 0 ? rule_env : (g.N * g.K <= (1 << 18) ? 1 : 0);
  if (rule == 1) {
    cs = (g.K + SMM_KP - 1) / SMM_KP;
    if (cs > 8) cs = 8;
    while (cs > 1 && strips * cs > 4 * (int64_t)sm_count()) --cs;
  } else if (rule > 1) {
    cs = rule - 1;
  }
  if (cs < 1) cs = 1;
  int64_t kchunk = (g.K + cs - 1) / cs;
  kchunk = (kchunk + 7) / 8 * 8;  // pieces start 32-byte aligned along k
  cs = (g.K + kchunk - 1) / kchunk;
  switch ((g.M + 3) / 4) {
    case 1: return launch_smallm_m<4>(g, (int)cs, kchunk, st);
    case 2: return launch_smallm_m<8>(g, (int)cs, kchunk, st);
    case 3: return launch_smallm_m<12>(g, (int)cs, kchunk, st);
    case 4: return launch_smallm_m<16>(g, (int)cs, kchunk, st);
    case 5: return launch_smallm_m<20>(g, (int)cs, kchunk, st);
    case 6: return launch_smallm_m<24>(g, (int)cs, kchunk, st);
    case 7: return launch_smallm_m<28>(g, (int)cs, kchunk, st);
    default: return launch_smallm_m<32>(g, (int)cs, kchunk, st);
  }
}

}  // namespace

int kred_splits(int64_t M, int64_t K) {
  int64_t mblocks = (M + 4 * KR_THREADS - 1) / (4 * KR_THREADS);
  int64_t want = (int64_t)sm_count() * 4;
  int64_t s = (want + mblocks - 1) / mblocks;
  int64_t maxs = K / 16;
  if (s > maxs) s = maxs;
  if (s > 1024) s = 1024;
  if (s < 1) s = 1;
  return (int)s;
}

namespace {
__device__ __forceinline__ int sk_owner_h(int64_t u, int64_t U, int NC) {
  int c = (int)((u * NC) / U);
  while (c + 1 < NC && ((int64_t)(c + 1) * U) / NC <= u) ++c;
  while (c > 0 && ((int64_t)c * U) / NC > u) --c;
  return c;
}

// grid (remainder tile, 16-row slab): owners computed once per CTA, then each
// thread sums 4 adjacent columns x 4 rows over the tile's pieces in k order
// and applies the epilogue (32-bit index math, coalesced accesses)
__global__ void __launch_bounds__(256) streamk_fixup_kernel(const float* __restrict__ P, float* __restrict__ C,
                                                           int64_t M, int64_t N, int64_t scm, int64_t scn,
                                                           Epi<float> epi, int num_m, int num_n, int bm, int bn,
                                                           int num_kb, int NC, int group_m, int base) {
  TX_GRID_WAIT();
  const int num_tiles = num_m * num_n;
  const int64_t U2 = (int64_t)(num_tiles - base) * num_kb;
  const int rt = blockIdx.x;
  const int c0 = sk_owner_h((int64_t)rt * num_kb, U2, NC), c1 = sk_owner_h((int64_t)rt * num_kb + num_kb - 1, U2, NC);
  if (c0 == c1) return;  // whole tile stored by its single owner
  const int t = base + rt;
  const int per_group = group_m * num_n;
  const int g = t / per_group, first = g * group_m;
  const int gsz = min(num_m - first, group_m);
  const int r = t - g * per_group;
  const int mb = first + r % gsz, nb = r / gsz;
  const int64_t n0 = (int64_t)nb * bn + (threadIdx.x & 63) * 4;
  const int64_t MN = M * N;
  const int npieces = c1 - c0 + 1;
  // 128-bit form: the 4 adjacent columns of a thread as one float4 per piece
  // (r01: the scalar form moved 36.8 MB in 28.7 us, 1.3 TB/s)
  const bool v4 = scn == 1 && (scm & 3) == 0 && (N & 3) == 0 && ((uintptr_t)C & 15) == 0 && ((uintptr_t)P & 15) == 0 &&
                  n0 + 4 <= N && n0 + 4 <= (int64_t)nb * bn + bn;
  if (v4) {
    float4 acc[4];
    int64_t rows[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      rows[i] = (int64_t)mb * bm + (int64_t)blockIdx.y * 16 + (threadIdx.x >> 6) + 4 * i;
      acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const bool slab_ok = (int64_t)blockIdx.y * 16 < bm;
    for (int q = 0; q < npieces; ++q) {  // pieces in k order; the 4 rows' loads are independent
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < M && slab_ok) {
          const float4 p = __ldcs(reinterpret_cast<const float4*>(P + q * MN + rows[i] * N + n0));
          acc[i].x += p.x; acc[i].y += p.y; acc[i].z += p.z; acc[i].w += p.w;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t m = rows[i];
      if (m >= M || !slab_ok) continue;
      float4 o;
      o.x = epi.apply(acc[i].x, m, n0);
      o.y = epi.apply(acc[i].y, m, n0 + 1);
      o.z = epi.apply(acc[i].z, m, n0 + 2);
      o.w = epi.apply(acc[i].w, m, n0 + 3);
      *reinterpret_cast<float4*>(C + m * scm + n0) = o;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = (int64_t)mb * bm + (int64_t)blockIdx.y * 16 + (threadIdx.x >> 6) + 4 * i;
    if (m >= M || (int64_t)blockIdx.y * 16 >= bm) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + j;
      if (n >= N || n >= (int64_t)nb * bn + bn) continue;
      float v = 0.f;
      for (int q = 0; q < npieces; ++q) v += P[q * MN + m * N + n];
      C[m * scm + n * scn] = epi.apply(v, m, n);
    }
  }
}
}  // namespace

int streamk_fixup(const float* P, const G& g, int num_m, int num_n, int bm, int bn, int num_kb, int nclusters,
                  int group_m, cudaStream_t st) {
  const int num_tiles = num_m * num_n;
  const int base = (num_tiles / nclusters) * nclusters;
  if (num_tiles == base) return TX_OK;
  TX_CHECK(bn <= 256, TX_E_ARG, "streamk_fixup: tile too wide");
  dim3 grid((unsigned)(num_tiles - base), (unsigned)((bm + 15) / 16));
  ::tx::launch(streamk_fixup_kernel, dim3(grid), dim3(256), 0, st, P, (float*)g.C, g.M, g.N, g.scm, g.scn, g.epi_f, num_m, num_n, bm, bn,
                                             num_kb, nclusters, group_m, base);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

int splitk_finalize(const float* P, const G& g, int splits, cudaStream_t st) {
  const int64_t tot = g.M * g.N;
  ::tx::launch(kred_finalize, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, P, (float*)g.C, g.M, (int)g.N, splits, g.scm, g.scn,
                                                              g.epi_f);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

int gemm_simt(const G& g, cudaStream_t st) {
  dim3 grid((unsigned)((g.N + 63) / 64), (unsigned)((g.M + 63) / 64));
  if (g.dtype == TX_F32)
    ::tx::launch(simt_gemm<float>, dim3(grid), dim3(256), 0, st, (const float*)g.A, (const float*)g.B, (float*)g.C, g.M, g.N, g.K, g.sam,
                                           g.sak, g.sbk, g.sbn, g.scm, g.scn, g.epi_f);
  else
    ::tx::launch(simt_gemm<double>, dim3(grid), dim3(256), 0, st, (const double*)g.A, (const double*)g.B, (double*)g.C, g.M, g.N, g.K,
                                            g.sam, g.sak, g.sbk, g.sbn, g.scm, g.scn, g.epi_d);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

#define TX_WIDTHS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

int gemm_skinny(const G& g, int kind, void* ws, size_t wsb, cudaStream_t st) {
  if (kind == SK_OUTER) {
    switch ((int)g.K) {
#define CASE(w) case w: return launch_outer<w>(g, st);
      TX_WIDTHS(CASE)
#undef CASE
    }
  } else if (kind == SK_ROWDOT) {
    switch ((int)g.N) {
#define CASE(w) case w: return launch_rowdot<w>(g, st);
      TX_WIDTHS(CASE)
#undef CASE
    }
  } else if (kind == SK_SMALLM) {
    return launch_smallm(g, st);
  } else {
    switch ((int)g.N) {
#define CASE(w) case w: return launch_kred<w>(g, ws, wsb, st);
      TX_WIDTHS(CASE)
#undef CASE
    }
  }
  return fail(TX_E_ARG, "tx_gemm: skinny width out of range");
}

}  // namespace tx
