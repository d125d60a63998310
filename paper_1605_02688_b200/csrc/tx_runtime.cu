// Runtime plumbing of libtexpr_b200: errors, device, streams, events, CUDA
// graph capture (the VM's replacement for the reference's per-node Python
// loop, runtime.py:428-446), async copies and a strided copy kernel.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>

#include <cstring>
#include <mutex>
#include <string>

#include "tx_common.h"

namespace tx {

static thread_local std::string g_last_error;
static int g_sm_count = 0;

void set_error(const std::string& msg) { g_last_error = msg; }

int sm_count() {
  if (g_sm_count == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  return g_sm_count;
}

bool pdl_enabled() {
  static const bool on = getenv("TX_NO_PDL") == nullptr;
  return on;
}

void collapse(int ndim, const int64_t* shape, int nops, const int64_t (*strides)[TX_MAX_RANK], Space* out) {
  // drop extent-1 dims
  int64_t sh[TX_MAX_RANK];
  int64_t st[32][TX_MAX_RANK];
  int nd = 0;
  for (int d = 0; d < ndim; ++d) {
    if (shape[d] == 1) continue;
    sh[nd] = shape[d];
    for (int k = 0; k < nops; ++k) st[k][nd] = strides[k][d];
    ++nd;
  }
  // merge dim d into d+1 (row-major) when every operand has stride[d] == stride[d+1]*shape[d+1]
  int od = 0;
  for (int d = 0; d < nd; ++d) {
    if (od > 0) {
      bool ok = true;
      for (int k = 0; k < nops; ++k)
        if (out->strides[k][od - 1] != st[k][d] * sh[d]) { ok = false; break; }
      if (ok) {
        out->shape[od - 1] *= sh[d];
        for (int k = 0; k < nops; ++k) out->strides[k][od - 1] = st[k][d];
        continue;
      }
    }
    out->shape[od] = sh[d];
    for (int k = 0; k < nops; ++k) out->strides[k][od] = st[k][d];
    ++od;
  }
  out->ndim = od;
}

// ---------------------------------------------------------------- copy kernel
struct CopyMeta {
  int64_t v[3 * TX_MAX_RANK];
};

template <typename T>
__global__ void strided_copy_kernel_p(const T* __restrict__ src, T* __restrict__ dst, int64_t n, int nd,
                                      CopyMeta m) {
  TX_GRID_WAIT();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i, so = 0, dof = 0;
    for (int d = nd - 1; d >= 0; --d) {
      int64_t e = m.v[d];
      int64_t c = r % e;
      r /= e;
      so += c * m.v[nd + d];
      dof += c * m.v[2 * nd + d];
    }
    dst[dof] = src[so];
  }
}

// Transposing copies (the conv lowering's NCHW <-> [pixels, channels]
// reorders, DimShuffle materialisations): dim p is unit-stride in the source,
// dim q in the destination.  32 x 32 tiles through shared memory make both the
// loads (along p) and the stores (along q) coalesced; the remaining dims are
// one batch index per blockIdx.z decoded once per block.  (The
// element-per-thread kernel above decodes every index with 64-bit divisions
// and scatters one side: 55 us for a 25.7 MB [100352 x 64] transpose.)
struct TileMeta {
  int64_t sp, sq;              // extents of p and q
  int64_t s_q, d_p;            // source stride of q, destination stride of p
  int nb;                      // number of batch dims
  int64_t bshape[TX_MAX_RANK], bs[TX_MAX_RANK], bd[TX_MAX_RANK];
};

template <typename T>
__global__ void __launch_bounds__(256) transpose_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, TileMeta m,
                                                             int64_t nbatch) {
  TX_GRID_WAIT();
  __shared__ T tile[32][33];
  const int64_t p0 = (int64_t)blockIdx.y * 32, q0 = (int64_t)blockIdx.x * 32;
  for (int64_t b = blockIdx.z; b < nbatch; b += gridDim.z) {
    int64_t r = b, so = 0, dof = 0;
    for (int d = m.nb - 1; d >= 0; --d) {
      const int64_t c = r % m.bshape[d];
      r /= m.bshape[d];
      so += c * m.bs[d];
      dof += c * m.bd[d];
    }
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int64_t p = p0 + threadIdx.x, q = q0 + threadIdx.y + j;
      if (p < m.sp && q < m.sq) tile[threadIdx.y + j][threadIdx.x] = src[so + p + q * m.s_q];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int64_t q = q0 + threadIdx.x, p = p0 + threadIdx.y + j;
      if (p < m.sp && q < m.sq) dst[dof + q + p * m.d_p] = tile[threadIdx.x][threadIdx.y + j];
    }
    __syncthreads();
  }
}

// Copies whose innermost dim is unit-stride on both sides (permutations of
// outer dims over contiguous rows: [K, N, P] <-> [N, K, P]): one row per
// block-iteration, the outer index decoded once per row.
template <typename T>
__global__ void __launch_bounds__(256) row_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, TileMeta m,
                                                       int64_t nrows) {
  TX_GRID_WAIT();
  // blockIdx.y: a 1024-element chunk of the row (4 independent copies per thread)
  const int64_t i0 = (int64_t)blockIdx.y * 1024 + threadIdx.x;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    int64_t r = row, so = 0, dof = 0;
    for (int d = m.nb - 1; d >= 0; --d) {
      const int64_t c = r % m.bshape[d];
      r /= m.bshape[d];
      so += c * m.bs[d];
      dof += c * m.bd[d];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = i0 + 256 * k;
      if (i < m.sp) dst[dof + i] = src[so + i];
    }
  }
}

template <typename T>
static int launch_copy(const tx_tensor* s, tx_tensor* d, cudaStream_t st) {
  int64_t strides[2][TX_MAX_RANK];
  int nd = d->ndim;
  for (int i = 0; i < nd; ++i) {
    int j = i - (nd - s->ndim);
    strides[0][i] = (j >= 0 && s->shape[j] != 1) ? s->strides[j] : 0;
    strides[1][i] = d->strides[i];
  }
  Space sp;
  collapse(nd, d->shape, 2, strides, &sp);
  int64_t n = numel(*d);
  if (n == 0) return TX_OK;
  CopyMeta m;
  for (int i = 0; i < sp.ndim; ++i) {
    m.v[i] = sp.shape[i];
    m.v[sp.ndim + i] = sp.strides[0][i];
    m.v[2 * sp.ndim + i] = sp.strides[1][i];
  }
  if (sp.ndim == 0) {  // scalar
    m.v[0] = 1; m.v[1] = 0; m.v[2] = 0; sp.ndim = 1;
  }
  static const bool generic_only = getenv("TX_COPY_GENERIC") != nullptr;  // A/B diagnostics
  // (small copies -- the LSTM's per-step reorders -- stay on the generic
  // kernel: its one-thread-per-element grid hides latency better there)
  if (sizeof(T) >= 4 && sp.ndim >= 2 && n >= (1 << 21) && !generic_only) {
    int p = -1, q = -1;
    for (int i = 0; i < sp.ndim; ++i) {
      if (sp.strides[0][i] == 1 && sp.shape[i] > 1) p = i;
      if (sp.strides[1][i] == 1 && sp.shape[i] > 1) q = i;
    }
    if (p >= 0 && q >= 0 && p != q && sp.shape[p] >= 8 && sp.shape[q] >= 8) {
      TileMeta t;
      t.sp = sp.shape[p];
      t.sq = sp.shape[q];
      t.s_q = sp.strides[0][q];
      t.d_p = sp.strides[1][p];
      t.nb = 0;
      int64_t nbatch = 1;
      for (int i = 0; i < sp.ndim; ++i) {
        if (i == p || i == q) continue;
        t.bshape[t.nb] = sp.shape[i];
        t.bs[t.nb] = sp.strides[0][i];
        t.bd[t.nb] = sp.strides[1][i];
        nbatch *= sp.shape[i];
        ++t.nb;
      }
      dim3 grid((unsigned)((t.sq + 31) / 32), (unsigned)((t.sp + 31) / 32),
                (unsigned)(nbatch < 65535 ? nbatch : 65535));
      if (grid.y <= 65535) {
        ::tx::launch(transpose_copy_kernel<T>, dim3(grid), dim3(dim3(32, 8)), 0, st, (const T*)s->data, (T*)d->data, t, nbatch);
        TX_CUDA(cudaGetLastError());
        return TX_OK;
      }
    }
    const int last = sp.ndim - 1;
    if (sp.strides[0][last] == 1 && sp.strides[1][last] == 1 && sp.shape[last] >= 64 &&
        (sp.shape[last] + 1023) / 1024 <= 65535) {
      TileMeta t;
      t.sp = sp.shape[last];
      t.nb = last;
      int64_t nrows = 1;
      for (int i = 0; i < last; ++i) {
        t.bshape[i] = sp.shape[i];
        t.bs[i] = sp.strides[0][i];
        t.bd[i] = sp.strides[1][i];
        nrows *= sp.shape[i];
      }
      const int64_t cap = (int64_t)sm_count() * 16;
      const int64_t gy = (t.sp + 1023) / 1024;
      const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(nrows, cap / std::max<int64_t>(gy, 1) + 1));
      ::tx::launch(row_copy_kernel<T>, dim3(dim3((unsigned)std::min<int64_t>(gx, 65535 * 16), (unsigned)std::min<int64_t>(gy, 65535))), dim3(256), 0, st, (const T*)s->data, (T*)d->data, t, nrows);
      TX_CUDA(cudaGetLastError());
      return TX_OK;
    }
  }
  int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  ::tx::launch(strided_copy_kernel_p<T>, dim3((unsigned)blocks), dim3(threads), 0, st, (const T*)s->data, (T*)d->data, n, sp.ndim, m);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

// ---------------------------------------------------------------- NaN guard
template <typename T>
__global__ void check_values_kernel(const T* __restrict__ x, int64_t n, int nd, CopyMeta m, uint32_t* flags,
                                    int slot, int mode, double big) {
  TX_GRID_WAIT();
  uint32_t bits = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i, off = 0;
    for (int d = nd - 1; d >= 0; --d) {
      const int64_t e = m.v[d];
      off += (r % e) * m.v[nd + d];
      r /= e;
    }
    const double v = (double)x[off];
    if (v != v) bits |= 1u;
    else if (v == INFINITY || v == -INFINITY) bits |= 2u;
    else if (v > big || v < -big) bits |= 4u;
  }
  bits &= (uint32_t)mode;
  bits = __reduce_or_sync(0xffffffffu, bits);
  if ((threadIdx.x & 31) == 0 && bits) atomicOr(flags + slot, bits);
}

}  // namespace tx

using namespace tx;

extern "C" {

int tx_version(void) { return TX_ABI_VERSION; }

const char* tx_last_error(void) { return g_last_error.c_str(); }

int tx_init(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(TX_E_NODEVICE, std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "count=0"));
  TX_CHECK(device >= 0 && device < n, TX_E_ARG, "device index out of range");
  TX_CUDA(cudaSetDevice(device));
  TX_CUDA(cudaFree(0));  // create the primary context
  g_sm_count = 0;
  sm_count();
  return TX_OK;
}

int tx_device_info(int* sms, int* major, int* minor, int64_t* total_mem) {
  int dev = 0;
  TX_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p;
  TX_CUDA(cudaGetDeviceProperties(&p, dev));
  if (sms) *sms = p.multiProcessorCount;
  if (major) *major = p.major;
  if (minor) *minor = p.minor;
  if (total_mem) *total_mem = (int64_t)p.totalGlobalMem;
  return TX_OK;
}

int tx_stream_create(void** s) {
  cudaStream_t st;
  TX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  *s = st;
  return TX_OK;
}
int tx_stream_destroy(void* s) { TX_CUDA(cudaStreamDestroy((cudaStream_t)s)); return TX_OK; }
int tx_stream_sync(void* s) { TX_CUDA(cudaStreamSynchronize((cudaStream_t)s)); return TX_OK; }
int tx_event_create(void** ev) {
  cudaEvent_t e;
  TX_CUDA(cudaEventCreate(&e));
  *ev = e;
  return TX_OK;
}
int tx_event_destroy(void* ev) { TX_CUDA(cudaEventDestroy((cudaEvent_t)ev)); return TX_OK; }
int tx_event_record(void* ev, void* s) { TX_CUDA(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)s)); return TX_OK; }
int tx_stream_wait_event(void* s, void* ev) {
  TX_CUDA(cudaStreamWaitEvent((cudaStream_t)s, (cudaEvent_t)ev, 0));
  return TX_OK;
}
int tx_event_sync(void* ev) { TX_CUDA(cudaEventSynchronize((cudaEvent_t)ev)); return TX_OK; }
int tx_event_elapsed_ms(void* a, void* b, float* ms) {
  TX_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)a, (cudaEvent_t)b));
  return TX_OK;
}
int tx_memcpy_async(void* dst, const void* src, size_t bytes, int kind, void* s) {
  cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (bytes == 0) return TX_OK;
  TX_CUDA(cudaMemcpyAsync(dst, src, bytes, k, (cudaStream_t)s));
  return TX_OK;
}
int tx_device_alloc(size_t bytes, void** ptr) {
  TX_CHECK(ptr, TX_E_ARG, "tx_device_alloc: null out pointer");
  *ptr = nullptr;
  TX_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
  return TX_OK;
}
int tx_device_free(void* ptr) {
  if (ptr) TX_CUDA(cudaFree(ptr));
  return TX_OK;
}
int tx_memset_async(void* dst, int value, size_t bytes, void* s) {
  if (bytes == 0) return TX_OK;
  TX_CUDA(cudaMemsetAsync(dst, value, bytes, (cudaStream_t)s));
  return TX_OK;
}
int tx_host_register(void* p, size_t bytes) {
  TX_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return TX_OK;
}
int tx_host_unregister(void* p) { TX_CUDA(cudaHostUnregister(p)); return TX_OK; }

int tx_graph_begin(void* s) {
  TX_CUDA(cudaStreamBeginCapture((cudaStream_t)s, cudaStreamCaptureModeThreadLocal));
  return TX_OK;
}
int tx_graph_end(void* s, void** exec) {
  cudaGraph_t g;
  TX_CUDA(cudaStreamEndCapture((cudaStream_t)s, &g));
  cudaGraphExec_t ge;
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  *exec = ge;
  return TX_OK;
}
int tx_graph_launch(void* exec, void* s) {
  TX_CUDA(cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)s));
  return TX_OK;
}
int tx_graph_destroy(void* exec) { TX_CUDA(cudaGraphExecDestroy((cudaGraphExec_t)exec)); return TX_OK; }

int tx_check_values(const tx_tensor* x, uint32_t* flags, int slot, int mode, double big, void* s) {
  TX_CHECK(x && flags, TX_E_ARG, "tx_check_values: null argument");
  TX_CHECK(x->dtype == TX_F32 || x->dtype == TX_F64, TX_E_ARG, "tx_check_values: float tensors only");
  const int64_t n = numel(*x);
  if (n == 0) return TX_OK;
  int64_t strides[1][TX_MAX_RANK];
  for (int i = 0; i < x->ndim; ++i) strides[0][i] = x->strides[i];
  Space sp;
  collapse(x->ndim, x->shape, 1, strides, &sp);
  CopyMeta m;
  int nd = sp.ndim;
  for (int i = 0; i < nd; ++i) {
    m.v[i] = sp.shape[i];
    m.v[nd + i] = sp.strides[0][i];
  }
  if (nd == 0) { m.v[0] = 1; m.v[1] = 0; nd = 1; }
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  cudaStream_t st = (cudaStream_t)s;
  if (x->dtype == TX_F32)
    ::tx::launch(check_values_kernel<float>, dim3((unsigned)blocks), dim3(256), 0, st, (const float*)x->data, n, nd, m, flags, slot, mode, big);
  else
    ::tx::launch(check_values_kernel<double>, dim3((unsigned)blocks), dim3(256), 0, st, (const double*)x->data, n, nd, m, flags, slot, mode, big);
  TX_CUDA(cudaGetLastError());
  return TX_OK;
}

int tx_copy(const tx_tensor* src, tx_tensor* dst, void* s) {
  TX_CHECK(src && dst && src->dtype == dst->dtype, TX_E_ARG, "tx_copy: dtype mismatch");
  TX_CHECK(src->ndim <= dst->ndim, TX_E_ARG, "tx_copy: source rank exceeds destination");
  cudaStream_t st = (cudaStream_t)s;
  switch (itemsize(dst->dtype)) {
    case 1: return launch_copy<uint8_t>(src, dst, st);
    case 4: return launch_copy<uint32_t>(src, dst, st);
    case 8: return launch_copy<uint64_t>(src, dst, st);
  }
  return fail(TX_E_UNSUPPORTED, "tx_copy: dtype");
}

}  // extern "C"
