// 2-d convolution data movement for the im2col -> tcgen05 GEMM lowering of
// the reference's conv2d trio (pkg/src/texpr/ops/conv.py:108-157):
//   tx_im2col  x[N,C,H,W] (any strides) -> cols[N*Ho*Wo, C*kh*kw] (row-major),
//              zero outside the padded input (ops/conv.py:108-119)
//   tx_col2im  dcols[N*Ho*Wo, C*kh*kw] -> dx[N,C,H,W]: the transpose, as a
//              gather per input element summing its (u, v) taps in ascending
//              order -- the same order as the reference's scatter loop
//              (ops/conv.py:142-155), so no atomics and a deterministic sum.
// The contractions themselves are tx_gemm calls (tensor cores for fp32).
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "tx_common.h"
#include "tx_gemm.h"

namespace tx {
namespace {

struct ConvGeom {
  int64_t N, C, H, W, Ho, Wo;
  int kh, kw, sh, sw, ph, pw;
  int64_t xs[4];  // input strides (elements)
};

template <class T>
__global__ void im2col_kernel(const T* __restrict__ x, T* __restrict__ cols, ConvGeom g, int64_t total) {
  TX_GRID_WAIT();
  const int64_t ckk = g.C * g.kh * g.kw;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / ckk, col = e - row * ckk;
    const int64_t n = row / (g.Ho * g.Wo), p = row - n * (g.Ho * g.Wo);
    const int64_t i = p / g.Wo, j = p - i * g.Wo;
    const int64_t c = col / (g.kh * g.kw), r = col - c * (g.kh * g.kw);
    const int u = (int)(r / g.kw), v = (int)(r - (int64_t)u * g.kw);
    const int64_t h = i * g.sh - g.ph + u, w = j * g.sw - g.pw + v;
    T val = T(0);
    if (h >= 0 && h < g.H && w >= 0 && w < g.W) val = x[n * g.xs[0] + c * g.xs[1] + h * g.xs[2] + w * g.xs[3]];
    cols[e] = val;
  }
}

// Row-block form (the default): a CTA owns RB consecutive rows of cols (output
// pixels, decoded once into shared memory) and its threads walk the
// C*kh*kw columns, so every store is a coalesced run along a row and no
// thread divides by more than the small window sizes; the input reads are
// gathers that hit L2 (and L1 across the block's neighbouring pixels).
// (The element-per-thread form above spent ~5 64-bit divisions per element:
// 465 us for the 231 MB patch matrix of a 32x64x56x56 3x3 layer; this form
// 91 us.  A [32 pixels x 64 columns] shared-tile transpose with lane =
// pixel for the gather measured slower, 150 us.)
constexpr int IM2COL_RB = 16;

template <class T>
__global__ void __launch_bounds__(256) im2col_rows(const T* __restrict__ x, T* __restrict__ cols, ConvGeom g,
                                                   int64_t rows) {
  TX_GRID_WAIT();
  __shared__ int64_t sbase[IM2COL_RB];
  __shared__ int sh0[IM2COL_RB], sw0[IM2COL_RB];
  const int64_t row0 = (int64_t)blockIdx.x * IM2COL_RB;
  if (threadIdx.x < IM2COL_RB) {
    const int64_t row = row0 + threadIdx.x;
    const int64_t n = row / (g.Ho * g.Wo), p = row - n * (g.Ho * g.Wo);
    const int64_t i = p / g.Wo, j = p - i * g.Wo;
    sbase[threadIdx.x] = n * g.xs[0];
    sh0[threadIdx.x] = (int)(i * g.sh - g.ph);
    sw0[threadIdx.x] = (int)(j * g.sw - g.pw);
  }
  __syncthreads();
  const int kk = g.kh * g.kw;
  const int ckk = (int)g.C * kk;
  const int nr = (int)min((int64_t)IM2COL_RB, rows - row0);
  for (int col = threadIdx.x; col < ckk; col += blockDim.x) {
    const int c = col / kk, r = col - c * kk;
    const int u = r / g.kw, v = r - u * g.kw;
    const T* xc = x + (int64_t)c * g.xs[1];
    T* out = cols + row0 * ckk + col;
#pragma unroll 4
    for (int rr = 0; rr < nr; ++rr) {
      const int h = sh0[rr] + u, w = sw0[rr] + v;
      T val = T(0);
      if (h >= 0 && h < g.H && w >= 0 && w < g.W) val = xc[sbase[rr] + (int64_t)h * g.xs[2] + (int64_t)w * g.xs[3]];
      out[(int64_t)rr * ckk] = val;
    }
  }
}

// (u, v, c) column order over a channel-contiguous input: thread t of the
// CTA handles VEC consecutive channels of one (u, v) for 16 output pixels,
// so loads and stores run along c (one 128-bit access per thread when VEC = 4).
template <class T, int VEC>
__global__ void __launch_bounds__(256) im2col_hwc_rows(const T* __restrict__ x, T* __restrict__ cols, ConvGeom g,
                                                       int64_t rows) {
  TX_GRID_WAIT();
  __shared__ int64_t sbase[IM2COL_RB];
  __shared__ int sh0[IM2COL_RB], sw0[IM2COL_RB];
  const int64_t row0 = (int64_t)blockIdx.x * IM2COL_RB;
  if (threadIdx.x < IM2COL_RB) {
    const int64_t row = row0 + threadIdx.x;
    const int64_t n = row / (g.Ho * g.Wo), p = row - n * (g.Ho * g.Wo);
    const int64_t i = p / g.Wo, j = p - i * g.Wo;
    sbase[threadIdx.x] = n * g.xs[0];
    sh0[threadIdx.x] = (int)(i * g.sh - g.ph);
    sw0[threadIdx.x] = (int)(j * g.sw - g.pw);
  }
  __syncthreads();
  const int C = (int)g.C;
  const int ckk = C * g.kh * g.kw;
  const int nr = (int)min((int64_t)IM2COL_RB, rows - row0);
  using V = typename std::conditional<VEC == 4 && sizeof(T) == 4, float4, T>::type;
  for (int col = threadIdx.x * VEC; col < ckk; col += blockDim.x * VEC) {
    const int uv = col / C, c = col - uv * C;
    const int u = uv / g.kw, v = uv - u * g.kw;
    const T* xc = x + c;  // channel stride 1
    T* out = cols + row0 * ckk + col;
#pragma unroll 4
    for (int rr = 0; rr < nr; ++rr) {
      const int h = sh0[rr] + u, w = sw0[rr] + v;
      const bool in = h >= 0 && h < g.H && w >= 0 && w < g.W;
      const T* src = xc + sbase[rr] + (int64_t)h * g.xs[2] + (int64_t)w * g.xs[3];
      if constexpr (VEC == 4 && sizeof(T) == 4) {
        const float4 val = in ? *reinterpret_cast<const float4*>(src) : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(out + (int64_t)rr * ckk) = val;
      } else {
        out[(int64_t)rr * ckk] = in ? *src : T(0);
      }
    }
  }
}

template <class T>
__global__ void col2im_kernel(const T* __restrict__ dcols, T* __restrict__ dx, ConvGeom g, int64_t total) {
  TX_GRID_WAIT();
  const int64_t ckk = g.C * g.kh * g.kw;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int64_t w = t % g.W; t /= g.W;
    const int64_t h = t % g.H; t /= g.H;
    const int64_t c = t % g.C;
    const int64_t n = t / g.C;
    T acc = T(0);
    for (int u = 0; u < g.kh; ++u) {
      const int64_t hi = h + g.ph - u;
      if (hi < 0 || hi % g.sh) continue;
      const int64_t i = hi / g.sh;
      if (i >= g.Ho) continue;
      for (int v = 0; v < g.kw; ++v) {
        const int64_t wi = w + g.pw - v;
        if (wi < 0 || wi % g.sw) continue;
        const int64_t j = wi / g.sw;
        if (j >= g.Wo) continue;
        acc += dcols[((n * g.Ho + i) * g.Wo + j) * ckk + (c * g.kh + u) * g.kw + v];
      }
    }
    dx[e] = acc;
  }
}

int geom(const tx_tensor* x4, const int* win, int64_t Ho, int64_t Wo, ConvGeom* g) {
  TX_CHECK(x4->ndim == 4, TX_E_ARG, "conv: rank-4 tensors expected");
  g->N = x4->shape[0]; g->C = x4->shape[1]; g->H = x4->shape[2]; g->W = x4->shape[3];
  g->kh = win[0]; g->kw = win[1]; g->sh = win[2]; g->sw = win[3]; g->ph = win[4]; g->pw = win[5];
  TX_CHECK(g->sh > 0 && g->sw > 0 && g->kh > 0 && g->kw > 0, TX_E_ARG, "conv: bad window");
  g->Ho = Ho; g->Wo = Wo;
  for (int i = 0; i < 4; ++i) g->xs[i] = x4->strides[i];
  return TX_OK;
}

// x[N, C, H, W] (any strides) -> y[N, Hp, Wp, C] contiguous with zero borders
// (the implicit GEMM's input).  One CTA per padded row (n, hp): the row's
// C x W interior goes through a shared tile in channel blocks of 32 (reads
// run along w, writes along c: both coalesced), border pixels and rows are
// written as zeros in the same pass (no separate memset).
constexpr int PAD_CB = 32;
template <class T>
__global__ void __launch_bounds__(256) pad_nhwc_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t N, int64_t C,
                                                       int64_t H, int64_t W, int ph, int pw, int64_t xs0, int64_t xs1,
                                                       int64_t xs2, int64_t xs3) {
  TX_GRID_WAIT();
  extern __shared__ __align__(16) unsigned char pad_smem[];
  T* tile = reinterpret_cast<T*>(pad_smem);  // [PAD_CB][W + 1]
  const int64_t Hp = H + 2 * ph, Wp = W + 2 * pw;
  const int64_t n = blockIdx.x / Hp, hp = blockIdx.x % Hp;
  const int64_t h = hp - ph;
  T* yrow = y + (n * Hp + hp) * Wp * C;
  if (h < 0 || h >= H) {
    for (int64_t e = threadIdx.x; e < Wp * C; e += blockDim.x) yrow[e] = T(0);
    return;
  }
  // lane along w (reads) / along c (writes), warp along the other axis: no
  // per-element division, 128-byte runs on both sides
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const T* xrow = x + n * xs0 + h * xs2;
  for (int64_t c0 = 0; c0 < C; c0 += PAD_CB) {
    const int cb = (int)(C - c0 < PAD_CB ? C - c0 : PAD_CB);
    __syncthreads();
    for (int c = wq; c < cb; c += nw)
      for (int64_t w = lane; w < W; w += 32) tile[c * (W + 1) + w] = xrow[(c0 + c) * xs1 + w * xs3];
    __syncthreads();
    if (lane < cb)
      for (int64_t wp = wq; wp < Wp; wp += nw) {
        const int64_t w = wp - pw;
        yrow[wp * C + c0 + lane] = (w >= 0 && w < W) ? tile[lane * (W + 1) + w] : T(0);
      }
  }
}

int64_t grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 16;
  return b < cap ? (b < 1 ? 1 : b) : cap;
}

}  // namespace
}  // namespace tx

using namespace tx;

extern "C" {

int tx_im2col(const tx_tensor* x, tx_tensor* cols, const int* win, void* stream) {
  TX_CHECK(x && cols && win && x->dtype == cols->dtype, TX_E_ARG, "tx_im2col: bad arguments");
  TX_CHECK(cols->ndim == 2 && is_contiguous(*cols), TX_E_ARG, "tx_im2col: cols must be contiguous [rows, C*kh*kw]");
  ConvGeom g;
  const int64_t Ho = (x->shape[2] + 2 * win[4] - win[0]) / win[2] + 1;
  const int64_t Wo = (x->shape[3] + 2 * win[5] - win[1]) / win[3] + 1;
  int rc = geom(x, win, Ho, Wo, &g);
  if (rc) return rc;
  TX_CHECK(cols->shape[0] == g.N * Ho * Wo && cols->shape[1] == g.C * g.kh * g.kw, TX_E_ARG, "tx_im2col: cols shape");
  const int64_t total = numel(*cols);
  if (total == 0) return TX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = cols->shape[0];
  const bool by_rows = g.C * g.kh * g.kw < (int64_t)INT32_MAX && !getenv("TX_IM2COL_FLAT");
  const unsigned rb = (unsigned)((rows + IM2COL_RB - 1) / IM2COL_RB);
  if (x->dtype == TX_F32 && by_rows)
    ::tx::launch(im2col_rows<float>, dim3(rb), dim3(256), 0, st, (const float*)x->data, (float*)cols->data, g, rows);
  else if (x->dtype == TX_F64 && by_rows)
    ::tx::launch(im2col_rows<double>, dim3(rb), dim3(256), 0, st, (const double*)x->data, (double*)cols->data, g, rows);
  else if (x->dtype == TX_F32)
    ::tx::launch(im2col_kernel<float>, dim3((unsigned)grid_for(total)), dim3(256), 0, st, (const float*)x->data, (float*)cols->data, g, total);
  else if (x->dtype == TX_F64)
    ::tx::launch(im2col_kernel<double>, dim3((unsigned)grid_for(total)), dim3(256), 0, st, (const double*)x->data, (double*)cols->data, g, total);
  else
    return fail(TX_E_UNSUPPORTED, "tx_im2col: float32/float64 only");
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

int tx_pad_nhwc(const tx_tensor* x, tx_tensor* y, const int* pad, void* stream) {
  TX_CHECK(x && y && pad && x->dtype == y->dtype && x->ndim == 4 && y->ndim == 4 && is_contiguous(*y), TX_E_ARG,
           "tx_pad_nhwc: x[N,C,H,W], contiguous y[N,H+2ph,W+2pw,C]");
  const int64_t N = x->shape[0], C = x->shape[1], H = x->shape[2], W = x->shape[3];
  const int ph = pad[0], pw = pad[1];
  TX_CHECK(ph >= 0 && pw >= 0 && y->shape[0] == N && y->shape[1] == H + 2 * ph && y->shape[2] == W + 2 * pw &&
               y->shape[3] == C,
           TX_E_ARG, "tx_pad_nhwc: output shape");
  const int64_t rows = N * (H + 2 * ph);
  if (rows == 0 || C == 0 || W == 0) return TX_OK;
  TX_CHECK(rows < (1LL << 31), TX_E_UNSUPPORTED, "tx_pad_nhwc: too many rows");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = (size_t)PAD_CB * (W + 1) * itemsize(x->dtype);
  TX_CHECK(smem <= 48 * 1024, TX_E_UNSUPPORTED, "tx_pad_nhwc: rows wider than the shared tile");
  if (x->dtype == TX_F32)
    TX_CUDA(::tx::launch(pad_nhwc_kernel<float>, dim3((unsigned)rows), dim3(256), smem, st, (const float*)x->data,
                         (float*)y->data, N, C, H, W, ph, pw, x->strides[0], x->strides[1], x->strides[2], x->strides[3]));
  else if (x->dtype == TX_F64)
    TX_CUDA(::tx::launch(pad_nhwc_kernel<double>, dim3((unsigned)rows), dim3(256), smem, st, (const double*)x->data,
                         (double*)y->data, N, C, H, W, ph, pw, x->strides[0], x->strides[1], x->strides[2],
                         x->strides[3]));
  else
    return fail(TX_E_UNSUPPORTED, "tx_pad_nhwc: float32/float64 only");
  return TX_OK;
}

int tx_im2col_hwc(const tx_tensor* x, tx_tensor* cols, const int* win, void* stream) {
  TX_CHECK(x && cols && win && x->dtype == cols->dtype, TX_E_ARG, "tx_im2col_hwc: bad arguments");
  TX_CHECK(cols->ndim == 2 && is_contiguous(*cols), TX_E_ARG, "tx_im2col_hwc: cols must be contiguous");
  TX_CHECK(x->ndim == 4 && x->strides[1] == 1, TX_E_ARG, "tx_im2col_hwc: the channel dim must be contiguous");
  ConvGeom g;
  const int64_t Ho = (x->shape[2] + 2 * win[4] - win[0]) / win[2] + 1;
  const int64_t Wo = (x->shape[3] + 2 * win[5] - win[1]) / win[3] + 1;
  int rc = geom(x, win, Ho, Wo, &g);
  if (rc) return rc;
  TX_CHECK(cols->shape[0] == g.N * Ho * Wo && cols->shape[1] == g.C * g.kh * g.kw, TX_E_ARG,
           "tx_im2col_hwc: cols shape");
  TX_CHECK(g.C * g.kh * g.kw < (int64_t)INT32_MAX, TX_E_ARG, "tx_im2col_hwc: too many columns");
  const int64_t rows = cols->shape[0];
  if (rows == 0 || g.C == 0) return TX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned rb = (unsigned)((rows + IM2COL_RB - 1) / IM2COL_RB);
  const bool v4 = x->dtype == TX_F32 && g.C % 4 == 0 && ((uintptr_t)x->data & 15) == 0 &&
                  ((uintptr_t)cols->data & 15) == 0 && g.xs[0] % 4 == 0 && g.xs[2] % 4 == 0 && g.xs[3] % 4 == 0;
  if (v4)
    ::tx::launch(im2col_hwc_rows<float, 4>, dim3(rb), dim3(256), 0, st, (const float*)x->data, (float*)cols->data, g, rows);
  else if (x->dtype == TX_F32)
    ::tx::launch(im2col_hwc_rows<float, 1>, dim3(rb), dim3(256), 0, st, (const float*)x->data, (float*)cols->data, g, rows);
  else if (x->dtype == TX_F64)
    ::tx::launch(im2col_hwc_rows<double, 1>, dim3(rb), dim3(256), 0, st, (const double*)x->data, (double*)cols->data, g, rows);
  else
    return fail(TX_E_UNSUPPORTED, "tx_im2col_hwc: float32/float64 only");
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

int tx_col2im(const tx_tensor* dcols, tx_tensor* dx, const int* win, int64_t Ho, int64_t Wo, void* stream) {
  TX_CHECK(dcols && dx && win && dx->dtype == dcols->dtype, TX_E_ARG, "tx_col2im: bad arguments");
  TX_CHECK(is_contiguous(*dx) && is_contiguous(*dcols), TX_E_ARG, "tx_col2im: contiguous operands expected");
  ConvGeom g;
  int rc = geom(dx, win, Ho, Wo, &g);
  if (rc) return rc;
  TX_CHECK(dcols->ndim == 2 && dcols->shape[0] == g.N * Ho * Wo && dcols->shape[1] == g.C * g.kh * g.kw, TX_E_ARG,
           "tx_col2im: dcols shape");
  const int64_t total = numel(*dx);
  if (total == 0) return TX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dx->dtype == TX_F32)
    ::tx::launch(col2im_kernel<float>, dim3((unsigned)grid_for(total)), dim3(256), 0, st, (const float*)dcols->data, (float*)dx->data, g, total);
  else if (dx->dtype == TX_F64)
    ::tx::launch(col2im_kernel<double>, dim3((unsigned)grid_for(total)), dim3(256), 0, st, (const double*)dcols->data, (double*)dx->data, g, total);
  else
    return fail(TX_E_UNSUPPORTED, "tx_col2im: float32/float64 only");
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

}  // extern "C"

extern "C" int tx_conv_implicit(const tx_tensor* xpad, const tx_tensor* w, tx_tensor* out, const int* win,
                                void* stream) {
  using namespace tx;
  TX_CHECK(xpad && w && out && win, TX_E_ARG, "tx_conv_implicit: bad arguments");
  TX_CHECK(xpad->dtype == TX_F32 && w->dtype == TX_F32 && out->dtype == TX_F32, TX_E_UNSUPPORTED,
           "tx_conv_implicit: float32 only");
  TX_CHECK(xpad->ndim == 4 && is_contiguous(*xpad) && w->ndim == 2 && is_contiguous(*w) &&
               (out->ndim == 2 || out->ndim == 4) && is_contiguous(*out),
           TX_E_ARG, "tx_conv_implicit: contiguous xpad[N,Hp,Wp,C], w[K,kh*kw*C], out[N*P*Q,K] or [N,K,P,Q]");
  const int kh = win[0], kw = win[1];
  const int64_t N = xpad->shape[0], Hp = xpad->shape[1], Wp = xpad->shape[2], C = xpad->shape[3];
  const int64_t K = w->shape[0];
  TX_CHECK(kh >= 1 && kw >= 1 && w->shape[1] == (int64_t)kh * kw * C, TX_E_ARG, "tx_conv_implicit: filter shape");
  const int64_t P = Hp - kh + 1, Q = Wp - kw + 1;
  const bool nchw = out->ndim == 4;
  TX_CHECK(nchw ? (out->shape[0] == N && out->shape[1] == K && out->shape[2] == P && out->shape[3] == Q)
                : (out->shape[0] == N * P * Q && out->shape[1] == K),
           TX_E_ARG, "tx_conv_implicit: output shape");
  if (N * P * Q == 0) return TX_OK;
  return gemm_tc_conv((const float*)xpad->data, N, Hp, Wp, C, (const float*)w->data, K, kh, kw, (float*)out->data,
                      nchw ? 1 : 0, (cudaStream_t)stream);
}
