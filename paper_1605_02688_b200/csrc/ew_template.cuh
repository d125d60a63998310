// ew_template.cuh — hand-written template for fused elementwise kernels.
//
// The Python code generator (paper_1605_02688_b200/codegen.py) instantiates
// this file for one Composite program: it substitutes the @-markers below
// with per-operand pointer casts, vector loads/stores and the straight-line
// scalar body, then hands the translation unit to tx_ew_compile (NVRTC,
// sm_100a, -fmad=false, IEEE div/sqrt, no FTZ).  Three entry points:
//
//   tx_ew_flat    all operands share the output's contiguous layout and are
//                 16-byte aligned: grid-stride over 4-element vectors, 128-bit
//                 streaming loads/stores (ld/st.global.cs), scalar tail.
//   tx_ew_2d      rank <= 2 after dim collapsing (row/column broadcasts such as
//                 bias rows [1,N] and softmax columns [B,1]): 32-bit index
//                 math, threads along the contiguous dim.
//   tx_ew_nd      anything else: per-element div/mod over <= 8 dims.
//
// Scalar semantics reproduce NumPy's, which the reference calls
// (pkg/src/texpr/ops/elemwise.py:36-113): NaN-propagating maximum, the
// branch-stable sigmoid of :44-46, floor division (with a zero-division flag)
// for integer div (:49-55), bool results for comparisons.
#pragma once

typedef long long i64;
typedef unsigned char u8;

#define TX_MAXOPS 24
#define TX_MAXRANK 8

struct TxEwArgs {
  i64 n;
  int ndim;
  int vec_ok;
  i64 shape[TX_MAXRANK];
  void* ptr[TX_MAXOPS];
  i64 strides[TX_MAXOPS][TX_MAXRANK];
  int* err;
};

// ------------------------------------------------------------ scalar helpers
__device__ __forceinline__ float tx_exp(float x) { return expf(x); }
__device__ __forceinline__ double tx_exp(double x) { return exp(x); }
__device__ __forceinline__ float tx_log(float x) { return logf(x); }
__device__ __forceinline__ double tx_log(double x) { return log(x); }
__device__ __forceinline__ float tx_log1p(float x) { return log1pf(x); }
__device__ __forceinline__ double tx_log1p(double x) { return log1p(x); }
__device__ __forceinline__ float tx_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double tx_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float tx_tanh(float x) { return tanhf(x); }
__device__ __forceinline__ double tx_tanh(double x) { return tanh(x); }
__device__ __forceinline__ float tx_pow(float a, float b) { return powf(a, b); }
__device__ __forceinline__ double tx_pow(double a, double b) { return pow(a, b); }

// integer fallbacks: computed in double, truncated back to the declared type
template <class T> __device__ __forceinline__ T tx_exp(T x) { return (T)exp((double)x); }
template <class T> __device__ __forceinline__ T tx_log(T x) { return (T)log((double)x); }
template <class T> __device__ __forceinline__ T tx_log1p(T x) { return (T)log1p((double)x); }
template <class T> __device__ __forceinline__ T tx_sqrt(T x) { return (T)sqrt((double)x); }
template <class T> __device__ __forceinline__ T tx_tanh(T x) { return (T)tanh((double)x); }
template <class T> __device__ __forceinline__ T tx_pow(T a, T b) {
  if (b < 0) return (T)0;
  T r = 1;
  while (b) { if (b & 1) r *= a; a *= a; b >>= 1; }
  return r;
}

__device__ __forceinline__ float tx_sigmoid(float x) {
  float z = expf(-fabsf(x));
  return x >= 0.0f ? 1.0f / (1.0f + z) : z / (1.0f + z);
}
__device__ __forceinline__ double tx_sigmoid(double x) {
  double z = exp(-fabs(x));
  return x >= 0.0 ? 1.0 / (1.0 + z) : z / (1.0 + z);
}
template <class T> __device__ __forceinline__ T tx_sigmoid(T x) { return (T)tx_sigmoid((double)x); }

// np.maximum: NaN in either operand propagates (the first NaN if both); ties give the SECOND
// operand ((a > b || isnan(a)) ? a : b), which decides the sign of a +0 / -0 tie
__device__ __forceinline__ float tx_maximum(float a, float b) { return (a != a) ? a : (b != b) ? b : (a > b ? a : b); }
__device__ __forceinline__ double tx_maximum(double a, double b) { return (a != a) ? a : (b != b) ? b : (a > b ? a : b); }
template <class T> __device__ __forceinline__ T tx_maximum(T a, T b) { return a > b ? a : b; }

__device__ __forceinline__ float tx_div(float a, float b, int*) { return a / b; }
__device__ __forceinline__ double tx_div(double a, double b, int*) { return a / b; }
template <class T> __device__ __forceinline__ T tx_div(T a, T b, int* err) {
  if (b == 0) { if (err) atomicExch(err, 1); return (T)0; }
  T q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return q;
}

__device__ __forceinline__ u8 tx_isnan(float a) { return a != a; }
__device__ __forceinline__ u8 tx_isnan(double a) { return a != a; }
template <class T> __device__ __forceinline__ u8 tx_isnan(T) { return 0; }

// ------------------------------------------------------- vector load/store
// 4 consecutive elements per thread; 16 B per access for 4-byte types,
// two 16 B accesses for 8-byte types, one 4 B access for bool.
template <class T> struct V4 { T v[4]; };

__device__ __forceinline__ V4<float> tx_ld4(const float* p) {
  float4 t = __ldcs(reinterpret_cast<const float4*>(p));
  return V4<float>{{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ V4<int> tx_ld4(const int* p) {
  int4 t = __ldcs(reinterpret_cast<const int4*>(p));
  return V4<int>{{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ V4<double> tx_ld4(const double* p) {
  double2 a = __ldcs(reinterpret_cast<const double2*>(p));
  double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  return V4<double>{{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ V4<i64> tx_ld4(const i64* p) {
  longlong2 a = __ldcs(reinterpret_cast<const longlong2*>(p));
  longlong2 b = __ldcs(reinterpret_cast<const longlong2*>(p) + 1);
  return V4<i64>{{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ V4<u8> tx_ld4(const u8* p) {
  unsigned int t = __ldcs(reinterpret_cast<const unsigned int*>(p));
  return V4<u8>{{(u8)(t & 0xff), (u8)((t >> 8) & 0xff), (u8)((t >> 16) & 0xff), (u8)(t >> 24)}};
}

__device__ __forceinline__ void tx_st4(float* p, const V4<float>& x) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(x.v[0], x.v[1], x.v[2], x.v[3]));
}
__device__ __forceinline__ void tx_st4(int* p, const V4<int>& x) {
  __stcs(reinterpret_cast<int4*>(p), make_int4(x.v[0], x.v[1], x.v[2], x.v[3]));
}
__device__ __forceinline__ void tx_st4(double* p, const V4<double>& x) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(x.v[0], x.v[1]));
  __stcs(reinterpret_cast<double2*>(p) + 1, make_double2(x.v[2], x.v[3]));
}
__device__ __forceinline__ void tx_st4(i64* p, const V4<i64>& x) {
  __stcs(reinterpret_cast<longlong2*>(p), make_longlong2(x.v[0], x.v[1]));
  __stcs(reinterpret_cast<longlong2*>(p) + 1, make_longlong2(x.v[2], x.v[3]));
}
__device__ __forceinline__ void tx_st4(u8* p, const V4<u8>& x) {
  unsigned int t = (unsigned)x.v[0] | ((unsigned)x.v[1] << 8) | ((unsigned)x.v[2] << 16) | ((unsigned)x.v[3] << 24);
  __stcs(reinterpret_cast<unsigned int*>(p), t);
}


// plain (cached) vector loads, for operands re-read across rows (bias rows)
__device__ __forceinline__ V4<float> tx_ld4n(const float* p) {
  float4 t = *reinterpret_cast<const float4*>(p);
  return V4<float>{{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ V4<int> tx_ld4n(const int* p) {
  int4 t = *reinterpret_cast<const int4*>(p);
  return V4<int>{{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ V4<double> tx_ld4n(const double* p) {
  double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  return V4<double>{{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ V4<i64> tx_ld4n(const i64* p) {
  longlong2 a = reinterpret_cast<const longlong2*>(p)[0], b = reinterpret_cast<const longlong2*>(p)[1];
  return V4<i64>{{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ V4<u8> tx_ld4n(const u8* p) {
  unsigned int t = *reinterpret_cast<const unsigned int*>(p);
  return V4<u8>{{(u8)(t & 0xff), (u8)((t >> 8) & 0xff), (u8)((t >> 16) & 0xff), (u8)(t >> 24)}};
}
// 4 consecutive columns of one row: a vector load, or one value broadcast when
// the operand is constant along the row (column-broadcast [B,1] operands)
template <class T>
__device__ __forceinline__ V4<T> tx_ld4b(const T* p, i64 s1) {
  if (s1 == 0) {
    const T v = *p;
    return V4<T>{{v, v, v, v}};
  }
  return tx_ld4n(p);
}

// ------------------------------------------------------------ kernels
// The generator defines, before including the kernels below:
//   TX_PTRS            pointer declarations p<k> (inputs) and q<k> (outputs)
//   TX_BODY(IN, OUT)   the scalar program: IN(k) reads input k, OUT(k, v)
//                      writes output k
//   TX_VDECL / TX_VLOAD(off) / TX_VSTORE(off) for the flat kernel
//   TX_NOPS            number of operands (outputs first)
#ifdef TX_KERNELS

extern "C" __global__ void __launch_bounds__(256) tx_ew_flat(const TxEwArgs a) {
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");  // programmatic dependent launch (tx_common.h)
  TX_PTRS
  int* err = a.err;
  (void)err;
  const i64 n = a.n;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 t0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (a.vec_ok) {
    const i64 nvec = n >> 2;
    for (i64 v = t0; v < nvec; v += stride) {
      const i64 off = v << 2;
      TX_VDECL
      TX_VLOAD(off)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#define IN(k) vin##k.v[j]
#define OUT(k, val) vout##k.v[j] = (val)
        TX_BODY
#undef IN
#undef OUT
      }
      TX_VSTORE(off)
    }
    for (i64 i = (nvec << 2) + t0; i < n; i += stride) {
#define IN(k) p##k[i]
#define OUT(k, val) q##k[i] = (val)
      TX_BODY
#undef IN
#undef OUT
    }
  } else {
    for (i64 i = t0; i < n; i += stride) {
#define IN(k) p##k[i]
#define OUT(k, val) q##k[i] = (val)
      TX_BODY
#undef IN
#undef OUT
    }
  }
}

// Row-major forms: shape[1] columns (operand column stride strides[k][1]) by
// rows = e0 * e1 * e2, the row index split into up to three coordinates
// (c0 < e0 = shape[0], stride strides[k][0]; c1 < e1 = shape[2], strides[k][2];
// c2 < e2 = shape[3], strides[k][3]; ndim = 2, 3 or 4).  Rank-3/4 spaces
// that do not collapse to 2-D (a reversed-time view, a [T]-vector broadcast
// over [T, B, V]) keep the contiguous, vectorised column loop; the row
// coordinates cost two integer divisions per row, not per element as in
// tx_ew_nd.
#define TX_ROWS_DECL                                       \
  const int e0 = (int)a.shape[0];                          \
  const int e1 = a.ndim >= 3 ? (int)a.shape[2] : 1;        \
  const int e2 = a.ndim >= 4 ? (int)a.shape[3] : 1;        \
  const int rows = e0 * e1 * e2;
#define TX_ROW_COORDS                                      \
  int c0 = row, c1 = 0, c2 = 0;                            \
  if (a.ndim > 2) {                                        \
    c0 = row % e0;                                         \
    const int t_ = row / e0;                               \
    c1 = t_ % e1;                                          \
    c2 = t_ / e1;                                          \
  }
extern "C" __global__ void __launch_bounds__(256) tx_ew_2d(const TxEwArgs a) {
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");  // programmatic dependent launch (tx_common.h)
  TX_PTRS
  int* err = a.err;
  (void)err;
  TX_ROWS_DECL
  const int cols = (int)a.shape[1];
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= cols) return;
  for (int row = blockIdx.y; row < rows; row += gridDim.y) {
    TX_ROW_COORDS
#define OFF(k) ((i64)c0 * a.strides[k][0] + (i64)c1 * a.strides[k][2] + (i64)c2 * a.strides[k][3] + (i64)col * a.strides[k][1])
#define IN(k) p##k[OFF(TX_IN_SLOT(k))]
#define OUT(k, val) q##k[OFF(k)] = (val)
    TX_BODY
#undef IN
#undef OUT
#undef OFF
  }
}


// rank-2 with the contiguous dim vectorised: every operand has column stride
// 0 or 1 and 16 B-aligned rows; 4 columns per thread, one row per grid.y step.
extern "C" __global__ void __launch_bounds__(256) tx_ew_2dv(const TxEwArgs a) {
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");  // programmatic dependent launch (tx_common.h)
  TX_PTRS
  int* err = a.err;
  (void)err;
  TX_ROWS_DECL
  const int cols4 = (int)(a.shape[1] >> 2);
  const int c4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c4 >= cols4) return;
  const i64 col = (i64)c4 << 2;
  for (int row = blockIdx.y; row < rows; row += gridDim.y) {
    TX_ROW_COORDS
#define OFF(k) ((i64)c0 * a.strides[k][0] + (i64)c1 * a.strides[k][2] + (i64)c2 * a.strides[k][3] + col * a.strides[k][1])
    TX_VDECL
    TX_VLOAD2D
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#define IN(k) vin##k.v[j]
#define OUT(k, val) vout##k.v[j] = (val)
      TX_BODY
#undef IN
#undef OUT
    }
    TX_VSTORE2D
#undef OFF
  }
}

extern "C" __global__ void __launch_bounds__(256) tx_ew_nd(const TxEwArgs a) {
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");  // programmatic dependent launch (tx_common.h)
  TX_PTRS
  int* err = a.err;
  (void)err;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    i64 off[TX_NOPS];
#pragma unroll
    for (int k = 0; k < TX_NOPS; ++k) off[k] = 0;
    i64 r = i;
    for (int d = a.ndim - 1; d >= 0; --d) {
      const i64 e = a.shape[d];
      const i64 c = r % e;
      r /= e;
#pragma unroll
      for (int k = 0; k < TX_NOPS; ++k) off[k] += c * a.strides[k][d];
    }
#define IN(k) p##k[off[TX_IN_SLOT(k)]]
#define OUT(k, val) q##k[off[k]] = (val)
    TX_BODY
#undef IN
#undef OUT
  }
}

#endif  // TX_KERNELS
