// CAReduce on sm_100a: sum / max / first-max one-hot / first-max index over an
// arbitrary axis set of a strided tensor.
//
// Replaces np.add.reduce / np.maximum.reduce / np.argmax+put_along_axis in
// reference pkg/src/texpr/ops/reductions.py:91-101, :119-129, :166-179.
//
// The (kept dims) x (reduced dims) problem is collapsed to the cheapest form:
//   ROW    reduced elements contiguous per output ("axis 1" / all axes):
//          CTA-per-row (or per row-slice), 128-bit loads, warp-shuffle tree,
//          optional split of long rows across CTAs with a deterministic
//          second pass (no atomics: results are run-to-run identical).
//   COL    kept elements contiguous ("axis 0"): each thread owns 4 adjacent
//          columns (one 128-bit load per row), rows split across grid.y into
//          partials combined in fixed order by a finalize kernel.
//   COLTMA the COL case for 4-byte types when TMA can address the matrix:
//          [16 rows x 256 columns] tiles are streamed by one producer lane
//          with cp.async.bulk.tensor into a 4-stage shared-memory ring
//          (mbarrier transaction counts), 8 consumer warps reduce them
//          column-per-thread; up to 192 KB in flight per SM regardless of
//          the register budget.
//   GEN    anything else: one thread per output, div/mod addressing.
// max / argmax are bit-exact with NumPy: NaN propagates (and counts as the
// maximum for argmax), and the first maximal element wins ties.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <algorithm>
#include <type_traits>

#include "tx_common.h"

namespace tx {
namespace {

constexpr int kThreads = 256;

template <class T> __device__ __forceinline__ bool isnan_(T v) { return false; }
template <> __device__ __forceinline__ bool isnan_<float>(float v) { return v != v; }
template <> __device__ __forceinline__ bool isnan_<double>(double v) { return v != v; }

template <class T> __device__ __forceinline__ T lowest();
template <> __device__ __forceinline__ float lowest<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double lowest<double>() { return -INFINITY; }
template <> __device__ __forceinline__ int lowest<int>() { return INT_MIN; }
template <> __device__ __forceinline__ long long lowest<long long>() { return LLONG_MIN; }
template <> __device__ __forceinline__ unsigned char lowest<unsigned char>() { return 0; }

// Accumulator state for one reduction op.  idx is the flat index over the
// reduced dims (only meaningful for the argmax ops).
template <class T, int OP>
struct Acc {
  T v;
  long long i;
  __device__ __forceinline__ void init() {
    if (OP == TX_SUM) v = T(0); else v = lowest<T>();
    i = LLONG_MAX;
  }
  // Elements pushed by one thread arrive in increasing index order, so for
  // argmax a strict ">" keeps the first maximum and the first NaN sticks.
  __device__ __forceinline__ void push(T x, long long idx) {
    if (OP == TX_SUM) {
      v = v + x;
    } else if (OP == TX_MAX) {
      // NaN-propagating max (np.maximum semantics)
      if (isnan_<T>(v)) return;
      if (isnan_<T>(x) || x > v) v = x;
    } else {
      const bool take = (i == LLONG_MAX) | (x > v) | (isnan_<T>(x) & !isnan_<T>(v));
      if (take) { v = x; i = idx; }
    }
  }
  __device__ __forceinline__ void merge_pair(T x, long long idx) {
    bool xn = isnan_<T>(x), vn = isnan_<T>(v);
    bool take;
    if (vn && xn) take = idx < i;
    else if (vn) take = false;
    else if (xn) take = true;
    else if (x > v) take = true;
    else if (x < v) take = false;
    else take = idx < i;
    if (i == LLONG_MAX) take = true;
    if (take) { v = x; i = idx; }
  }
  __device__ __forceinline__ void merge(const Acc& o) {
    if (OP == TX_SUM) v = v + o.v;
    else if (OP == TX_MAX) push(o.v, 0);
    else if (o.i != LLONG_MAX) merge_pair(o.v, o.i);
  }
};

template <class T, int OP>
__device__ __forceinline__ Acc<T, OP> shfl_down(const Acc<T, OP>& a, int off) {
  Acc<T, OP> r;
  r.v = __shfl_down_sync(0xffffffffu, a.v, off);
  r.i = __shfl_down_sync(0xffffffffu, a.i, off);
  return r;
}

template <class T, int OP>
__device__ __forceinline__ Acc<T, OP> block_reduce(Acc<T, OP> a) {
  __shared__ T sv[kThreads / 32];
  __shared__ long long si[kThreads / 32];
  for (int off = 16; off > 0; off >>= 1) a.merge(shfl_down(a, off));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sv[warp] = a.v; si[warp] = a.i; }
  __syncthreads();
  if (warp == 0) {
    Acc<T, OP> b;
    b.init();
    if (lane < (int)(blockDim.x >> 5)) { b.v = sv[lane]; b.i = si[lane]; }
    for (int off = 16; off > 0; off >>= 1) b.merge(shfl_down(b, off));
    a = b;
  }
  return a;  // valid in thread 0
}

template <class T> struct Vec4 {};
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<int> { using type = int4; };

// Argmax over a thread's float4 stream (k = tid, tid + bd, ...): the
// NaN-aware maximum of each float4 and the index of the FIRST float4 that
// raised the running maximum (strict ">"; a NaN sticks); KEEP also keeps
// that float4.  The caller finds the element inside it.
template <bool KEEP>
__device__ __forceinline__ void argmax_scan(const float4* __restrict__ pv4, int64_t nv, int64_t bd, float& best,
                                            int64_t& bk, float4& bq) {
  auto chunk_max = [](const float4 q) {
    const bool nan4 = (q.x != q.x) | (q.y != q.y) | (q.z != q.z) | (q.w != q.w);
    const float m = fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w));
    return nan4 ? __int_as_float(0x7fc00000) : m;
  };
  auto take = [&](const float4 q, int64_t k) {
    const float m = chunk_max(q);
    if (bk < 0 || (best == best && (m != m || m > best))) {
      best = m;
      bk = k;
      if (KEEP) bq = q;
    }
  };
  int64_t k = threadIdx.x;
  for (; k + 3 * bd < nv; k += 4 * bd) {
    float4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = __ldcs(pv4 + k + u * bd);
#pragma unroll
    for (int u = 0; u < 4; ++u) take(q[u], k + u * bd);
  }
  for (; k < nv; k += bd) take(__ldcs(pv4 + k), k);
}

// ------------------------------------------------------------------ ROW
// rows x R, row r at x + r*rs, contiguous within the row.  grid = (splits, rows).
// splits == 1: write the final result; else write partials [rows][splits].
template <class T, int OP>
__global__ void __launch_bounds__(kThreads, (OP == TX_ARGMAX_INDEX || OP == TX_ARGMAX_ONEHOT) ? 8 : 1) row_kernel(const T* __restrict__ x, int64_t rows, int64_t R, int64_t rs,
                                                      int64_t es, int splits, T* __restrict__ out,
                                                      long long* __restrict__ out_idx, T* __restrict__ pv,
                                                      long long* __restrict__ pi) {
  TX_GRID_WAIT();
  const int64_t row = blockIdx.y + (int64_t)blockIdx.z * gridDim.y;
  if (row >= rows) return;
  // split chunks are a multiple of 4 elements so every split of an aligned
  // row starts 16-byte aligned (the 128-bit paths below)
  const int64_t chunk = splits == 1 ? R : (((R + splits - 1) / splits + 3) & ~(int64_t)3);
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(R, lo + chunk);
  const T* p = x + row * rs;
  Acc<T, OP> a;
  a.init();
  if (es != 1) {
    for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) a.push(p[k * es], k);
  } else if constexpr (sizeof(T) == 4 && (OP == TX_SUM || OP == TX_MAX) && !std::is_same<T, unsigned char>::value) {
    // 128-bit path when the slice start is 16 B aligned
    int64_t head = lo;
    const int64_t mis = ((uintptr_t)(p + lo) & 15) / sizeof(T);
    int64_t vstart = lo + (mis ? (4 - mis) : 0);
    if (vstart > hi) vstart = hi;
    for (int64_t k = lo + threadIdx.x; k < vstart; k += blockDim.x) a.push(p[k], k);
    const int64_t nv = (hi - vstart) / 4;
    using V = typename Vec4<T>::type;
    const V* pv4 = reinterpret_cast<const V*>(p + vstart);
    int64_t k = threadIdx.x;
    for (; k + 3 * (int64_t)blockDim.x < nv; k += 4 * (int64_t)blockDim.x) {
      V q0 = __ldcs(pv4 + k), q1 = __ldcs(pv4 + k + blockDim.x);
      V q2 = __ldcs(pv4 + k + 2 * blockDim.x), q3 = __ldcs(pv4 + k + 3 * blockDim.x);
      a.push(q0.x, 0); a.push(q0.y, 0); a.push(q0.z, 0); a.push(q0.w, 0);
      a.push(q1.x, 0); a.push(q1.y, 0); a.push(q1.z, 0); a.push(q1.w, 0);
      a.push(q2.x, 0); a.push(q2.y, 0); a.push(q2.z, 0); a.push(q2.w, 0);
      a.push(q3.x, 0); a.push(q3.y, 0); a.push(q3.z, 0); a.push(q3.w, 0);
    }
    for (; k < nv; k += blockDim.x) {
      V q = __ldcs(pv4 + k);
      a.push(q.x, 0); a.push(q.y, 0); a.push(q.z, 0); a.push(q.w, 0);
    }
    for (int64_t t = vstart + nv * 4 + threadIdx.x; t < hi; t += blockDim.x) a.push(p[t], t);
    (void)head;
  } else if constexpr (std::is_same<T, float>::value && (OP == TX_ARGMAX_INDEX || OP == TX_ARGMAX_ONEHOT)) {
    const bool al = (((uintptr_t)(p + lo)) & 15) == 0;
    if (al) {
      // Per float4: its NaN-aware maximum, kept with the index of the FIRST
      // float4 that raised the running maximum (argmax_scan).  The element is
      // found inside that float4 at the end: the first NaN in it, else the
      // first element equal to the maximum -- the same first-occurrence
      // answer as pushing every element, at ~3 instructions per element
      // instead of ~10 (64-bit index selects).
      const int64_t nv = (hi - lo) / 4;
      const float4* pv4 = reinterpret_cast<const float4*>(p + lo);
      const int64_t bd = blockDim.x;
      float best = -INFINITY;
      int64_t bk = -1;
      float4 bq = make_float4(0.f, 0.f, 0.f, 0.f);
      // short spans (one row per CTA: axis-1 argmax) keep the winning float4
      // in registers -- the end-of-span re-read is a full memory latency per
      // CTA; long spans (all-axes splits) re-read it once (measured faster)
      if (nv < 64 * bd) argmax_scan<true>(pv4, nv, bd, best, bk, bq);
      else argmax_scan<false>(pv4, nv, bd, best, bk, bq);
      if (bk >= 0) {
        if (nv >= 64 * bd) bq = pv4[bk];
        const float e[4] = {bq.x, bq.y, bq.z, bq.w};
        int j = 0;
        if (best != best) { while (e[j] == e[j]) ++j; }
        else { while (!(e[j] == best)) ++j; }
        a.push(e[j], lo + 4 * bk + j);
      }
      for (int64_t t = lo + nv * 4 + threadIdx.x; t < hi; t += blockDim.x) a.push(p[t], t);
    } else {
      for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) a.push(p[k * es], k);
    }
  } else if constexpr (sizeof(T) == 4 && (OP == TX_ARGMAX_INDEX || OP == TX_ARGMAX_ONEHOT)) {
    const bool al = (((uintptr_t)(p + lo)) & 15) == 0;
    if (al) {
      using V = typename Vec4<T>::type;
      const int64_t nv = (hi - lo) / 4;
      const V* pv4 = reinterpret_cast<const V*>(p + lo);
      int64_t k = threadIdx.x;
      const int64_t bd = blockDim.x;
      for (; k + 3 * bd < nv; k += 4 * bd) {
        V q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = __ldcs(pv4 + k + u * bd);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t b = lo + 4 * (k + u * bd);
          a.push(q[u].x, b); a.push(q[u].y, b + 1); a.push(q[u].z, b + 2); a.push(q[u].w, b + 3);
        }
      }
      for (; k < nv; k += bd) {
        V q = __ldcs(pv4 + k);
        int64_t b = lo + 4 * k;
        a.push(q.x, b); a.push(q.y, b + 1); a.push(q.z, b + 2); a.push(q.w, b + 3);
      }
      for (int64_t t = lo + nv * 4 + threadIdx.x; t < hi; t += blockDim.x) a.push(p[t], t);
    } else {
      for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) a.push(p[k * es], k);
    }
  } else {
    for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) a.push(p[k * es], k);
  }
  a = block_reduce<T, OP>(a);
  if (threadIdx.x == 0) {
    if (splits == 1) {
      if (OP == TX_SUM || OP == TX_MAX) out[row] = a.v; else out_idx[row] = a.i;
    } else {
      pv[row * splits + blockIdx.x] = a.v;
      pi[row * splits + blockIdx.x] = a.i;
    }
  }
}

// warp-per-row variant for short rows (softmax-sized [B, 10] tensors)
template <class T, int OP>
__global__ void __launch_bounds__(kThreads) row_warp_kernel(const T* __restrict__ x, int64_t rows, int64_t R, int64_t rs,
                                                           int64_t es, T* __restrict__ out, long long* __restrict__ out_idx) {
  TX_GRID_WAIT();
  const int64_t row = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const T* p = x + row * rs;
  Acc<T, OP> a;
  a.init();
  for (int64_t k = lane; k < R; k += 32) a.push(p[k * es], k);
  for (int off = 16; off > 0; off >>= 1) a.merge(shfl_down(a, off));
  if (lane == 0) {
    if (OP == TX_SUM || OP == TX_MAX) out[row] = a.v; else out_idx[row] = a.i;
  }
}

// one CTA per output merges that output's split partials (strided over the
// CTA, then the shuffle tree) — splits can be several hundred (the all-axes
// reduction of a 16384^2 matrix uses 592), too many for one serial thread.
template <class T, int OP>
__global__ void __launch_bounds__(kThreads) finalize_splits(int64_t rows, int splits, const T* __restrict__ pv,
                                                           const long long* __restrict__ pi, T* __restrict__ out,
                                                           long long* __restrict__ out_idx) {
  TX_GRID_WAIT();
  const int64_t row = blockIdx.x;
  Acc<T, OP> a;
  a.init();
  for (int s = threadIdx.x; s < splits; s += blockDim.x) {
    Acc<T, OP> b;
    b.v = pv[row * splits + s];
    b.i = pi[row * splits + s];
    a.merge(b);
  }
  a = block_reduce<T, OP>(a);
  if (threadIdx.x == 0) {
    if (OP == TX_SUM || OP == TX_MAX) out[row] = a.v; else out_idx[row] = a.i;
  }
}

// ------------------------------------------------------------------ COL
// R rows x K columns, element (r, c) at x + r*rs + c (kept dim contiguous).
// grid.x covers columns (4 per thread), grid.y splits rows.
template <class T, int OP>
__global__ void __launch_bounds__(kThreads) col_kernel(const T* __restrict__ x, int64_t R, int64_t K, int64_t rs,
                                                      int splits, bool vec, T* __restrict__ out,
                                                      long long* __restrict__ out_idx, T* __restrict__ pv,
                                                      long long* __restrict__ pi) {
  TX_GRID_WAIT();
  const int64_t c0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c0 >= K) return;
  const int64_t chunk = (R + splits - 1) / splits;
  const int64_t lo = (int64_t)blockIdx.y * chunk;
  const int64_t hi = min(R, lo + chunk);
  Acc<T, OP> a[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) a[j].init();
  const int nc = (int)min((int64_t)4, K - c0);
  if constexpr (sizeof(T) == 4 && !std::is_same<T, unsigned char>::value) {
    if (vec && nc == 4) {
      using V = typename Vec4<T>::type;
      int64_t r = lo;
      for (; r + 3 < hi; r += 4) {
        V q0 = __ldcs(reinterpret_cast<const V*>(x + r * rs + c0));
        V q1 = __ldcs(reinterpret_cast<const V*>(x + (r + 1) * rs + c0));
        V q2 = __ldcs(reinterpret_cast<const V*>(x + (r + 2) * rs + c0));
        V q3 = __ldcs(reinterpret_cast<const V*>(x + (r + 3) * rs + c0));
        a[0].push(q0.x, r); a[1].push(q0.y, r); a[2].push(q0.z, r); a[3].push(q0.w, r);
        a[0].push(q1.x, r + 1); a[1].push(q1.y, r + 1); a[2].push(q1.z, r + 1); a[3].push(q1.w, r + 1);
        a[0].push(q2.x, r + 2); a[1].push(q2.y, r + 2); a[2].push(q2.z, r + 2); a[3].push(q2.w, r + 2);
        a[0].push(q3.x, r + 3); a[1].push(q3.y, r + 3); a[2].push(q3.z, r + 3); a[3].push(q3.w, r + 3);
      }
      for (; r < hi; ++r) {
        V q = __ldcs(reinterpret_cast<const V*>(x + r * rs + c0));
        a[0].push(q.x, r); a[1].push(q.y, r); a[2].push(q.z, r); a[3].push(q.w, r);
      }
      goto done;
    }
  }
  for (int64_t r = lo; r < hi; ++r)
    for (int j = 0; j < nc; ++j) a[j].push(x[r * rs + c0 + j], r);
done:
  for (int j = 0; j < nc; ++j) {
    const int64_t c = c0 + j;
    if (splits == 1) {
      if (OP == TX_SUM || OP == TX_MAX) out[c] = a[j].v; else out_idx[c] = a[j].i;
    } else {
      pv[(int64_t)blockIdx.y * K + c] = a[j].v;
      if (OP == TX_ARGMAX_INDEX || OP == TX_ARGMAX_ONEHOT) pi[(int64_t)blockIdx.y * K + c] = a[j].i;
    }
  }
}

// ------------------------------------------------------------------ COLTMA
constexpr int CT_COLS = 256, CT_ROWS = 16, CT_STAGES = 4;
constexpr int CT_THREADS = CT_COLS + 32;  // 8 consumer warps + 1 producer warp
constexpr size_t CT_SMEM = (size_t)CT_STAGES * CT_ROWS * CT_COLS * 4 + 2 * CT_STAGES * 8 + 128;

__device__ __forceinline__ uint32_t sa32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <class T, int OP>
__global__ void __launch_bounds__(CT_THREADS) col_tma_kernel(const __grid_constant__ CUtensorMap map, int64_t R,
                                                            int64_t K, int splits, T* __restrict__ out,
                                                            long long* __restrict__ out_idx, T* __restrict__ pv,
                                                            long long* __restrict__ pi) {
  TX_GRID_WAIT();
  extern __shared__ __align__(128) uint8_t ct_smem[];
  T* tiles = reinterpret_cast<T*>(ct_smem);  // [STAGES][ROWS][COLS]
  uint64_t* full = reinterpret_cast<uint64_t*>(ct_smem + (size_t)CT_STAGES * CT_ROWS * CT_COLS * sizeof(T));
  uint64_t* empty = full + CT_STAGES;
  const int64_t c0 = (int64_t)blockIdx.x * CT_COLS;
  int64_t chunk = (R + splits - 1) / splits;
  chunk = (chunk + CT_ROWS - 1) / CT_ROWS * CT_ROWS;
  const int64_t lo = (int64_t)blockIdx.y * chunk, hi = min(R, lo + chunk);
  const int ntiles = hi > lo ? (int)((hi - lo + CT_ROWS - 1) / CT_ROWS) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CT_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa32(full + s)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(empty + s)), "r"(CT_COLS / 32) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [](uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(sa32(b)), "r"(parity) : "memory");
    } while (!done);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == CT_COLS / 32) {  // producer
    if (lane == 0) {
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % CT_STAGES;
        wait(empty + s, ((i / CT_STAGES) & 1) ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa32(full + s)),
                     "r"((uint32_t)(CT_ROWS * CT_COLS * sizeof(T))) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                sa32(tiles + (size_t)s * CT_ROWS * CT_COLS)),
            "l"((uint64_t)&map), "r"(sa32(full + s)), "r"((int)c0), "r"((int)(lo + (int64_t)i * CT_ROWS))
            : "memory");
      }
    }
    return;
  }
  const int t = threadIdx.x;
  Acc<T, OP> a;
  a.init();
  if constexpr (std::is_same<T, float>::value && (OP == TX_MAX || OP == TX_ARGMAX_INDEX || OP == TX_ARGMAX_ONEHOT)) {
    // float max / argmax: the per-element compare-select is the issue-bound
    // part of this kernel (sum: ~21% SM throughput, argmax: ~65%), so it is
    // cut to the minimum: one unordered compare (take unless x <= v, which is
    // also true for a NaN x) gated by v being a number (a NaN v is final), a
    // 32-bit split-local row and two selects.  Rows arrive in increasing
    // order: the first maximum and the first NaN win, exactly as the generic
    // Acc::push (np.argmax / np.maximum.reduce, signed zeros included).
    // v = -inf with row 0 as its index needs no "empty" sentinel: row 0 is
    // taken unless it is -inf, in which case the first maximum IS row 0
    // whenever nothing larger follows
    float v = -INFINITY;
    int vi = 0;
    auto step = [&](float x, int row) {
      const bool take = !(x <= v) & (v == v);
      v = take ? x : v;
      if constexpr (OP != TX_MAX) vi = take ? row : vi;
    };
    for (int i = 0; i < ntiles; ++i) {
      const int s = i % CT_STAGES;
      wait(full + s, (i / CT_STAGES) & 1);
      const float* tile = reinterpret_cast<const float*>(tiles) + (size_t)s * CT_ROWS * CT_COLS;
      const int rl = i * CT_ROWS;
      const int nr = (int)min((int64_t)CT_ROWS, hi - (lo + rl));
      if (nr == CT_ROWS) {
#pragma unroll
        for (int r = 0; r < CT_ROWS; ++r) step(tile[r * CT_COLS + t], rl + r);
      } else {
        for (int r = 0; r < nr; ++r) step(tile[r * CT_COLS + t], rl + r);
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa32(empty + s)) : "memory");
    }
    if (ntiles > 0) {
      a.v = v;
      if constexpr (OP != TX_MAX) a.i = lo + vi;
    }
  } else {
  for (int i = 0; i < ntiles; ++i) {
    const int s = i % CT_STAGES;
    wait(full + s, (i / CT_STAGES) & 1);
    const T* tile = tiles + (size_t)s * CT_ROWS * CT_COLS;
    const int64_t r0 = lo + (int64_t)i * CT_ROWS;
    const int nr = (int)min((int64_t)CT_ROWS, hi - r0);
    if (nr == CT_ROWS) {
#pragma unroll
      for (int r = 0; r < CT_ROWS; ++r) a.push(tile[r * CT_COLS + t], r0 + r);
    } else {
      for (int r = 0; r < nr; ++r) a.push(tile[r * CT_COLS + t], r0 + r);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa32(empty + s)) : "memory");
  }
  }
  const int64_t c = c0 + t;
  if (c >= K) return;
  if (splits == 1) {
    if (OP == TX_SUM || OP == TX_MAX) out[c] = a.v; else out_idx[c] = a.i;
  } else {
    pv[(int64_t)blockIdx.y * K + c] = a.v;
    if (OP == TX_ARGMAX_INDEX || OP == TX_ARGMAX_ONEHOT) pi[(int64_t)blockIdx.y * K + c] = a.i;
  }
}

// partials [splits][K]: a 32-column x 8-lane CTA, each lane merging every
// 8th split (coalesced across columns), then the 8 lanes merged in order.
template <class T, int OP>
__global__ void __launch_bounds__(256) finalize_cols(int64_t K, int splits, const T* __restrict__ pv,
                                                    const long long* __restrict__ pi, T* __restrict__ out,
                                                    long long* __restrict__ out_idx) {
  TX_GRID_WAIT();
  __shared__ T sv[8][32];
  __shared__ long long si[8][32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + tx;
  Acc<T, OP> a;
  a.init();
  if (c < K) {
    for (int s = ty; s < splits; s += 8) {
      Acc<T, OP> b;
      b.v = pv[(int64_t)s * K + c];
      b.i = (OP == TX_ARGMAX_INDEX || OP == TX_ARGMAX_ONEHOT) ? pi[(int64_t)s * K + c] : 0;
      a.merge(b);
    }
  }
  sv[ty][tx] = a.v;
  si[ty][tx] = a.i;
  __syncthreads();
  if (ty == 0 && c < K) {
    for (int j = 1; j < 8; ++j) {
      Acc<T, OP> b;
      b.v = sv[j][tx];
      b.i = si[j][tx];
      a.merge(b);
    }
    if (OP == TX_SUM || OP == TX_MAX) out[c] = a.v; else out_idx[c] = a.i;
  }
}

// ------------------------------------------------------------------ GEN
struct GenMeta {
  int nk, nr;
  int64_t kshape[TX_MAX_RANK], kstride[TX_MAX_RANK];
  int64_t rshape[TX_MAX_RANK], rstride[TX_MAX_RANK];
};

template <class T, int OP>
__global__ void gen_kernel(const T* __restrict__ x, int64_t K, int64_t R, GenMeta m, T* __restrict__ out,
                           long long* __restrict__ out_idx) {
  TX_GRID_WAIT();
  int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= K) return;
  int64_t base = 0, t = o;
  for (int d = m.nk - 1; d >= 0; --d) { base += (t % m.kshape[d]) * m.kstride[d]; t /= m.kshape[d]; }
  Acc<T, OP> a;
  a.init();
  for (int64_t r = 0; r < R; ++r) {
    int64_t off = 0, u = r;
    for (int d = m.nr - 1; d >= 0; --d) { off += (u % m.rshape[d]) * m.rstride[d]; u /= m.rshape[d]; }
    a.push(x[base + off], r);
  }
  if (OP == TX_SUM || OP == TX_MAX) out[o] = a.v; else out_idx[o] = a.i;
}

// max reductions: the sign of a zero maximum.  np.maximum.reduce keeps the
// LATER operand on ties (reference ops/reductions.py:126, NumPy's
// (a > b || isnan(a)) ? a : b), so a +0 / -0 tie resolves to the sign of the
// last zero in index order.  The reduction kernels compute the maximum value
// (any zero); this pass gives every zero result the sign of its range's last
// zero, scanning backwards -- work only for outputs that are zero.
template <class T>
__global__ void max_zero_sign(const T* __restrict__ x, int64_t K, int64_t R, GenMeta m, T* __restrict__ out) {
  TX_GRID_WAIT();
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= K || out[o] != T(0)) return;
  int64_t base = 0, t = o;
  for (int d = m.nk - 1; d >= 0; --d) { base += (t % m.kshape[d]) * m.kstride[d]; t /= m.kshape[d]; }
  for (int64_t r = R - 1; r >= 0; --r) {
    int64_t off = 0, u = r;
    for (int d = m.nr - 1; d >= 0; --d) { off += (u % m.rshape[d]) * m.rstride[d]; u /= m.rshape[d]; }
    const T e = x[base + off];
    if (e == T(0)) { out[o] = e; return; }
  }
}

// one-hot materialisation: y has x's shape; element is 1 where its flat
// reduced index equals idx[flat kept index].
template <class T>
__global__ void onehot_kernel(T* __restrict__ y, int64_t n, GenMeta m, const long long* __restrict__ idx) {
  TX_GRID_WAIT();
  // m.kshape/kstride hold y's FULL shape and a per-dim role: kstride[d] = 1 kept, 0 reduced
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e, ki = 0, ri = 0, kmul = 1, rmul = 1, off = 0;
    for (int d = m.nk - 1; d >= 0; --d) {
      int64_t c = t % m.kshape[d];
      t /= m.kshape[d];
      off += c * m.rstride[d];
      if (m.kstride[d]) { ki += c * kmul; kmul *= m.kshape[d]; }
      else { ri += c * rmul; rmul *= m.kshape[d]; }
    }
    y[off] = (ri == idx[ki]) ? T(1) : T(0);
  }
}

template <class T>
__global__ void onehot_rows(T* __restrict__ y, int64_t rows, int64_t R, const long long* __restrict__ idx) {
  TX_GRID_WAIT();
  // y contiguous [rows, R]
  const int64_t n = rows * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / R;
    __stcs(y + e, (e - r * R) == idx[r] ? T(1) : T(0));
  }
}

template <class T>
__global__ void onehot_cols(T* __restrict__ y, int64_t R, int64_t K, const long long* __restrict__ idx) {
  TX_GRID_WAIT();
  // y contiguous [R, K]; idx per column
  const int64_t n = R * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / K;
    __stcs(y + e, r == idx[e - r * K] ? T(1) : T(0));
  }
}

// ------------------------------------------------------------------ planning
enum Form { ROW, ROWWARP, COL, COLTMA, GEN };

struct Plan {
  Form form;
  int64_t K = 1, R = 1;   // outputs, reduced elements
  int64_t ks = 0, rs = 0; // collapsed single-dim strides (ROW: row stride; COL: row stride)
  int64_t es = 1;         // ROWWARP element stride
  int splits = 1;
  GenMeta gm;
  size_t ws_partial = 0, ws_idx = 0;
};

// merge a list of (extent, stride) dims in order when row-major compatible
static int merge_dims(int n, int64_t* sh, int64_t* st) {
  int o = 0;
  for (int i = 0; i < n; ++i) {
    if (sh[i] == 1) continue;
    if (o > 0 && st[o - 1] == st[i] * sh[i]) {
      sh[o - 1] *= sh[i];
      st[o - 1] = st[i];
      continue;
    }
    sh[o] = sh[i];
    st[o] = st[i];
    ++o;
  }
  return o;
}

static void make_plan(int op, const tx_tensor& x, uint32_t mask, int itemsz, Plan* p) {
  int64_t ksh[TX_MAX_RANK], kst[TX_MAX_RANK], rsh[TX_MAX_RANK], rst[TX_MAX_RANK];
  int nk = 0, nr = 0;
  for (int d = 0; d < x.ndim; ++d) {
    if (mask & (1u << d)) { rsh[nr] = x.shape[d]; rst[nr] = x.strides[d]; ++nr; }
    else { ksh[nk] = x.shape[d]; kst[nk] = x.strides[d]; ++nk; }
  }
  int64_t K = 1, R = 1;
  for (int i = 0; i < nk; ++i) K *= ksh[i];
  for (int i = 0; i < nr; ++i) R *= rsh[i];
  p->K = K;
  p->R = R;
  // keep an uncollapsed copy for GEN
  p->gm.nk = nk;
  p->gm.nr = nr;
  for (int i = 0; i < nk; ++i) { p->gm.kshape[i] = ksh[i]; p->gm.kstride[i] = kst[i]; }
  for (int i = 0; i < nr; ++i) { p->gm.rshape[i] = rsh[i]; p->gm.rstride[i] = rst[i]; }
  int mk = merge_dims(nk, ksh, kst);
  int mr = merge_dims(nr, rsh, rst);
  const int sms = sm_count();
  int col_splits_max = 1;
  if (mk <= 1 && mr <= 1) {
    const int64_t kstride = mk == 1 ? kst[0] : 0;
    const int64_t rstride = mr == 1 ? rst[0] : 1;
    if (kstride == 1 && K >= 512 && rstride != 1) {
      // COL: kept dim contiguous and wide enough for coalesced 128-bit rows
      p->form = COL;
      p->rs = rstride;
      int64_t colblocks = (K + 4 * kThreads - 1) / (4 * kThreads);
      int64_t want = (int64_t)sms * 4;
      int64_t splits = (want + colblocks - 1) / colblocks;
      int64_t maxs = R / 64;
      if (splits > maxs) splits = maxs;
      if (splits > 65535) splits = 65535;
      if (splits < 1) splits = 1;
      p->splits = (int)splits;
      // the workspace must fit either form (the query may see another pointer)
      col_splits_max = (int)splits;
      if (itemsz == 4 && ((uintptr_t)x.data & 15) == 0 && (rstride * 4) % 16 == 0 && rstride >= K &&
          R < (int64_t)INT32_MAX && K < (int64_t)INT32_MAX && tmap_encoder() && !getenv("TX_REDUCE_NO_TMA")) {
        // ~1.75 waves of 3 CTAs per SM (64 KB ring each): the second partial
        // wave fills SMs whose first CTAs finish early (r02 A/B at 16384^2:
        // 7 splits = 448 CTAs on 444 slots 190-194 us, 12 splits 174-179 us)
        p->form = COLTMA;
        const int64_t strips = (K + CT_COLS - 1) / CT_COLS;
        int64_t want = (int64_t)sms * 3 * 7 / 4;
        int64_t sp = want / strips;
        int64_t maxs = R / (4 * CT_ROWS);
        if (sp > maxs) sp = maxs;
        if (sp > 65535) sp = 65535;
        if (sp < 1) sp = 1;
        if (const char* e = getenv("TX_REDUCE_COL_SPLITS")) sp = atoi(e);  // experiments
        p->splits = (int)sp;
      }
      {
        const int64_t strips = (K + CT_COLS - 1) / CT_COLS;
        int64_t sp = std::max<int64_t>((int64_t)sms * 3 * 7 / 4 / strips, (int64_t)sms * 3 / strips + 1);
        int64_t maxs = R / (4 * CT_ROWS);
        if (sp > maxs) sp = maxs;
        if (sp > 65535) sp = 65535;
        if (const char* e = getenv("TX_REDUCE_COL_SPLITS")) sp = atoi(e);
        if (sp > col_splits_max) col_splits_max = (int)sp;
      }
    } else if (R <= 512 && K >= 8) {
      // one warp per output (softmax-sized rows, any element stride)
      p->form = ROWWARP;
      p->ks = kstride;
      p->es = rstride;
    } else {
      // one CTA (or a split of CTAs) per output, any element stride
      p->form = ROW;
      p->ks = kstride;
      p->es = rstride;
      int64_t want = (int64_t)sms * 4;
      int64_t splits = 1;
      if (K < want) {
        splits = (want + K - 1) / K;
        int64_t maxs = R / 4096;
        if (splits > maxs) splits = maxs;
        if (splits < 1) splits = 1;
      }
      p->splits = (int)splits;
    }
  } else {
    p->form = GEN;
  }
  if (col_splits_max > p->splits) p->ws_partial = (size_t)col_splits_max * (size_t)p->K * 16 + 64;
  else if (p->splits > 1) p->ws_partial = (size_t)p->splits * (size_t)p->K * 16 + 64;
  if (op == TX_ARGMAX_ONEHOT) p->ws_idx = (size_t)p->K * 8;
}

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

template <class T, int OP>
static int run(const tx_tensor& x, uint32_t mask, tx_tensor& y, char* ws, size_t ws_bytes, cudaStream_t st) {
  Plan p;
  make_plan(OP, x, mask, (int)sizeof(T), &p);
  TX_CHECK(align256(p.ws_partial) + p.ws_idx <= ws_bytes || (p.ws_partial == 0 && p.ws_idx == 0), TX_E_ARG,
           "tx_reduce: workspace too small");
  const int sms = sm_count();
  T* out = (T*)y.data;
  long long* out_idx = (long long*)y.data;
  long long* onehot_idx = nullptr;
  if (OP == TX_ARGMAX_ONEHOT) {
    onehot_idx = (long long*)(ws + align256(p.ws_partial));
    out_idx = onehot_idx;
  }
  // the output of SUM / MAX / ARGMAX_INDEX is written densely in kept-dim C order;
  // require y contiguous for those (the VM allocates it so).
  if (OP != TX_ARGMAX_ONEHOT) TX_CHECK(is_contiguous(y), TX_E_ARG, "tx_reduce: output must be contiguous");
  T* pv = (T*)ws;
  long long* pi = (long long*)(ws + (size_t)p.splits * p.K * sizeof(T));
  if (p.splits > 1) pi = (long long*)(ws + (((size_t)p.splits * p.K * sizeof(T) + 7) & ~(size_t)7));
  if (p.K == 0) return TX_OK;
  if (p.R == 0) {
    TX_CHECK(OP == TX_SUM, TX_E_ARG, "zero-size array to reduction operation maximum which has no identity");
    TX_CUDA(cudaMemsetAsync(y.data, 0, (size_t)p.K * sizeof(T), st));
    return TX_OK;
  }
  const T* xp = (const T*)x.data;
  switch (p.form) {
    case ROW: {
      int64_t rows = p.K;
      unsigned gy = (unsigned)(rows < 65535 ? rows : 65535);
      unsigned gz = (unsigned)((rows + gy - 1) / gy);
      dim3 grid((unsigned)p.splits, gy, gz);
      ::tx::launch(row_kernel<T, OP>, dim3(grid), dim3(kThreads), 0, st, xp, rows, p.R, p.ks, p.es, p.splits, out, out_idx, pv, pi);
      if (p.splits > 1)
        ::tx::launch(finalize_splits<T, OP>, dim3((unsigned)rows), dim3(kThreads), 0, st, rows, p.splits, pv, pi, out, out_idx);
      break;
    }
    case ROWWARP: {
      int64_t rows = p.K;
      unsigned blocks = (unsigned)((rows + (kThreads / 32) - 1) / (kThreads / 32));
      ::tx::launch(row_warp_kernel<T, OP>, dim3(blocks), dim3(kThreads), 0, st, xp, rows, p.R, p.ks, p.es, out, out_idx);
      break;
    }
    case COL: {
      bool vec = ((uintptr_t)xp & 15) == 0 && (p.rs % 4) == 0;
      unsigned gx = (unsigned)((p.K + 4 * kThreads - 1) / (4 * kThreads));
      dim3 grid(gx, (unsigned)p.splits);
      ::tx::launch(col_kernel<T, OP>, dim3(grid), dim3(kThreads), 0, st, xp, p.R, p.K, p.rs, p.splits, vec, out, out_idx, pv, pi);
      if (p.splits > 1)
        ::tx::launch(finalize_cols<T, OP>, dim3((unsigned)((p.K + 31) / 32)), dim3(256), 0, st, p.K, p.splits, pv, pi, out, out_idx);
      break;
    }
    case COLTMA: {
      typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
      Enc enc = (Enc)tmap_encoder();
      CUtensorMap map;
      cuuint64_t dims[2] = {(cuuint64_t)p.K, (cuuint64_t)p.R};
      cuuint64_t gstr[1] = {(cuuint64_t)(p.rs * 4)};
      cuuint32_t box[2] = {(cuuint32_t)CT_COLS, (cuuint32_t)CT_ROWS};
      cuuint32_t es[2] = {1, 1};
      CUtensorMapDataType dt = std::is_same<T, float>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32;
      CUresult r = enc(&map, dt, 2, (void*)xp, dims, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      TX_CHECK(r == CUDA_SUCCESS, TX_E_CUDA, "tx_reduce: cuTensorMapEncodeTiled failed");
      static bool attr = false;
      if (!attr) {
        TX_CUDA(cudaFuncSetAttribute(col_tma_kernel<T, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CT_SMEM));
        attr = true;
      }
      dim3 grid((unsigned)((p.K + CT_COLS - 1) / CT_COLS), (unsigned)p.splits);
      ::tx::launch(col_tma_kernel<T, OP>, dim3(grid), dim3(CT_THREADS), CT_SMEM, st, map, p.R, p.K, p.splits, out, out_idx, pv, pi);
      if (p.splits > 1)
        ::tx::launch(finalize_cols<T, OP>, dim3((unsigned)((p.K + 31) / 32)), dim3(256), 0, st, p.K, p.splits, pv, pi, out, out_idx);
      break;
    }
    case GEN: {
      ::tx::launch(gen_kernel<T, OP>, dim3((unsigned)((p.K + 127) / 128)), dim3(128), 0, st, xp, p.K, p.R, p.gm, out, out_idx);
      break;
    }
  }
  TX_CUDA(cudaGetLastError());
  if constexpr (OP == TX_MAX && (std::is_same<T, float>::value || std::is_same<T, double>::value)) {
    static const bool off = getenv("TX_NO_MAX_ZERO_SIGN") != nullptr;  // A/B diagnostics only
    if (p.K > 0 && p.R > 0 && !off) {
      ::tx::launch(max_zero_sign<T>, dim3((unsigned)((p.K + 127) / 128)), dim3(128), 0, st, xp, p.K, p.R, p.gm, out);
      TX_CUDA(cudaGetLastError());
    }
  }
  if (OP == TX_ARGMAX_ONEHOT) {
    T* yp = (T*)y.data;
    int64_t n = numel(y);
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    // fast forms when y is contiguous and the reduced dims are a trailing / leading block
    bool ycont = is_contiguous(y);
    int first_r = -1, last_r = -1, nred = 0;
    for (int d = 0; d < x.ndim; ++d)
      if (mask & (1u << d)) { if (first_r < 0) first_r = d; last_r = d; ++nred; }
    bool block_contig = nred > 0 && (last_r - first_r + 1) == nred;
    if (ycont && block_contig && last_r == x.ndim - 1) {
      ::tx::launch(onehot_rows<T>, dim3((unsigned)blocks), dim3(256), 0, st, yp, p.K, p.R, onehot_idx);
    } else if (ycont && block_contig && first_r == 0) {
      ::tx::launch(onehot_cols<T>, dim3((unsigned)blocks), dim3(256), 0, st, yp, p.R, p.K, onehot_idx);
    } else {
      GenMeta m;
      m.nk = y.ndim;
      for (int d = 0; d < y.ndim; ++d) {
        m.kshape[d] = y.shape[d];
        m.kstride[d] = (mask & (1u << d)) ? 0 : 1;
        m.rstride[d] = y.strides[d];
      }
      ::tx::launch(onehot_kernel<T>, dim3((unsigned)blocks), dim3(256), 0, st, yp, n, m, onehot_idx);
    }
    TX_CUDA(cudaGetLastError());
  }
  return TX_OK;
}

template <class T>
static int dispatch_op(int op, const tx_tensor& x, uint32_t mask, tx_tensor& y, char* ws, size_t wsb, cudaStream_t st) {
  switch (op) {
    case TX_SUM: return run<T, TX_SUM>(x, mask, y, ws, wsb, st);
    case TX_MAX: return run<T, TX_MAX>(x, mask, y, ws, wsb, st);
    case TX_ARGMAX_ONEHOT: return run<T, TX_ARGMAX_ONEHOT>(x, mask, y, ws, wsb, st);
    case TX_ARGMAX_INDEX: return run<T, TX_ARGMAX_INDEX>(x, mask, y, ws, wsb, st);
  }
  return fail(TX_E_ARG, "tx_reduce: unknown op");
}

}  // namespace

int reduce_launch(int op, const tx_tensor& x, uint32_t mask, tx_tensor& y, void* ws, size_t wsb, cudaStream_t st) {
  switch (x.dtype) {
    case TX_F32: return dispatch_op<float>(op, x, mask, y, (char*)ws, wsb, st);
    case TX_F64: return dispatch_op<double>(op, x, mask, y, (char*)ws, wsb, st);
    case TX_I32: return dispatch_op<int>(op, x, mask, y, (char*)ws, wsb, st);
    case TX_I64: return dispatch_op<long long>(op, x, mask, y, (char*)ws, wsb, st);
    case TX_BOOL:
      // numpy add.reduce into a bool buffer is logical OR == max over {0,1}
      return dispatch_op<unsigned char>(op == TX_SUM ? TX_MAX : op, x, mask, y, (char*)ws, wsb, st);
  }
  return fail(TX_E_UNSUPPORTED, "tx_reduce: dtype");
}

}  // namespace tx

using namespace tx;

extern "C" {

// Zero-size cases, before any planning (which divides by the extents):
// returns 1 when there is nothing to launch.
static int empty_case(int op, const tx_tensor& x, uint32_t mask, tx_tensor* y, cudaStream_t st, bool run, int* rc) {
  int64_t red = 1, keep = 1;
  for (int d = 0; d < x.ndim; ++d) ((mask >> d) & 1u ? red : keep) *= x.shape[d];
  if (op == TX_ARGMAX_ONEHOT) keep *= red;  // the one-hot output has the input's shape
  *rc = TX_OK;
  if (red == 0 && op != TX_SUM) {           // NumPy raises for max / argmax over an empty axis
    *rc = fail(TX_E_ARG, "zero-size reduction: max / argmax have no identity");  // (even for an empty result)
    return 1;
  }
  if (keep == 0) return 1;                  // empty result: nothing to compute
  if (red != 0) return 0;
  if (run) {                                // sum over an empty axis is 0
    if (!is_contiguous(*y)) {
      *rc = fail(TX_E_UNSUPPORTED, "tx_reduce: empty-axis sum into a strided output");
      return 1;
    }
    const cudaError_t e = cudaMemsetAsync(y->data, 0, (size_t)numel(*y) * itemsize(y->dtype), st);
    if (e != cudaSuccess) *rc = cuda_fail(e, "cudaMemsetAsync");
  }
  return 1;
}

int tx_reduce_workspace(int op, const tx_tensor* x, uint32_t mask, size_t* bytes) {
  TX_CHECK(x && bytes, TX_E_ARG, "tx_reduce_workspace: null argument");
  int erc;
  if (mask && empty_case(op, *x, mask, nullptr, 0, false, &erc)) {
    *bytes = 0;
    return TX_OK;
  }
  Plan p;
  int isz = itemsize(x->dtype);
  make_plan(op, *x, mask, isz < 4 ? 4 : isz, &p);
  *bytes = (p.ws_partial || p.ws_idx) ? align256(p.ws_partial) + p.ws_idx + 256 : 0;
  return TX_OK;
}

int tx_reduce(int op, const tx_tensor* x, uint32_t mask, tx_tensor* y, void* ws, size_t wsb, void* stream) {
  TX_CHECK(x && y, TX_E_ARG, "tx_reduce: null tensor");
  TX_CHECK(x->ndim <= TX_MAX_RANK, TX_E_ARG, "tx_reduce: rank");
  if (mask == 0) {  // empty axis tuple: identity copy (reference ops/reductions.py:94-95)
    if (op == TX_ARGMAX_ONEHOT) {
      TX_CHECK(false, TX_E_UNSUPPORTED, "argmax_onehot over no axes is lowered as a fill");
    }
    return tx_copy(x, y, stream);
  }
  int erc;
  if (empty_case(op, *x, mask, y, (cudaStream_t)stream, true, &erc)) return erc;
  return reduce_launch(op, *x, mask, *y, ws, wsb, (cudaStream_t)stream);
}

}  // extern "C"
