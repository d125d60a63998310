/*
 * texpr_b200.h — C ABI of libtexpr_b200.so, the B200 (sm_100a) execution
 * library behind the compiled-graph hot path of the texpr expression compiler
 * (arXiv 1605.02688, "Theano").
 *
 * The reference has no native boundary: its VM calls op.perform() on NumPy
 * arrays (pkg/src/texpr/runtime.py:326-349 -> ops/*.py perform).  Each entry
 * point below replaces one of those perform() families; the Python VM
 * (paper_1605_02688_b200/vm.py) binds them with ctypes.
 *
 * Conventions
 *  - Every function returns int: 0 = TX_OK, otherwise a TX_E_* code; the
 *    message is read with tx_last_error() (thread-local).  Nothing aborts or
 *    throws across the ABI.
 *  - Device memory is owned by the caller (PyTorch allocations used as plain
 *    buffers).  The library owns only NVRTC modules, CUDA graphs, events,
 *    streams it created, and NCCL communicators; each has a *_destroy.
 *  - Tensors are passed as tx_tensor: data pointer, dtype code, rank, shape,
 *    strides in ELEMENTS (0 = broadcast).  Rank <= 8 (reference graph.py:23).
 *  - All launches take an explicit cudaStream_t (passed as void*).  A handle
 *    may be used by one host thread at a time (mirrors the per-function lock,
 *    reference runtime.py:301, :371-373).
 */
#ifndef TEXPR_B200_H
#define TEXPR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TX_MAX_RANK 8
#define TX_ABI_VERSION 1

/* dtype codes — the closed set of reference dtypes.py:16-21 */
enum { TX_F32 = 0, TX_F64 = 1, TX_I32 = 2, TX_I64 = 3, TX_BOOL = 4 };

/* status codes */
enum {
  TX_OK = 0,
  TX_E_ARG = 1,        /* bad argument / unsupported layout            */
  TX_E_CUDA = 2,       /* CUDA runtime or driver error                 */
  TX_E_NVRTC = 3,      /* NVRTC compilation failed (log in message)    */
  TX_E_NCCL = 4,       /* NCCL error                                   */
  TX_E_UNSUPPORTED = 5,/* dtype / shape combination not implemented    */
  TX_E_NODEVICE = 6,   /* no CUDA device / driver                      */
  TX_E_ZERODIV = 7     /* integer division by zero inside a kernel     */
};

typedef struct tx_tensor {
  void* data;
  int32_t dtype;
  int32_t ndim;
  int64_t shape[TX_MAX_RANK];
  int64_t strides[TX_MAX_RANK]; /* in elements */
} tx_tensor;

/* ---------------------------------------------------------------- runtime */
int tx_version(void);
const char* tx_last_error(void);
/* Select the device; fails with TX_E_NODEVICE when no driver/GPU exists. */
int tx_init(int device);
int tx_device_info(int* sm_count, int* cc_major, int* cc_minor, int64_t* total_mem);

int tx_stream_create(void** stream);
int tx_stream_destroy(void* stream);
int tx_stream_sync(void* stream);
int tx_event_create(void** ev);
int tx_event_destroy(void* ev);
int tx_event_record(void* ev, void* stream);
int tx_stream_wait_event(void* stream, void* ev);
int tx_event_elapsed_ms(void* start, void* stop, float* ms);
/* Block the calling host thread until the event has completed. */
int tx_event_sync(void* ev);
/* kind: 0 H2D, 1 D2H, 2 D2D (all async on stream) */
int tx_memcpy_async(void* dst, const void* src, size_t bytes, int kind, void* stream);
int tx_memset_async(void* dst, int value, size_t bytes, void* stream);
int tx_host_register(void* ptr, size_t bytes);
int tx_host_unregister(void* ptr);
/* Device memory for callers without their own allocator (a cgo / JNI /
 * ctypes binding of the reference; the Python package uses torch tensors).
 * 256-byte aligned; tx_device_free(NULL) is a no-op. */
int tx_device_alloc(size_t bytes, void** ptr);
int tx_device_free(void* ptr);

/* Capture every launch issued on `stream` between begin/end into one CUDA
 * graph (replaces the per-node Python walk, runtime.py:428-446). */
int tx_graph_begin(void* stream);
int tx_graph_end(void* stream, void** graph_exec);
int tx_graph_launch(void* graph_exec, void* stream);
int tx_graph_destroy(void* graph_exec);

/* Strided copy dst <- src (same dtype, broadcast src allowed).  Used for
 * update commits and outputs that alias storage. */
int tx_copy(const tx_tensor* src, tx_tensor* dst, void* stream);

/* ------------------------------------------- fused elementwise (NVRTC)
 * Replaces Elemwise.perform / CompositeElemwise._perform_chunked/_plain
 * (reference ops/elemwise.py:314-326, :538-597).
 * `source` is a complete CUDA translation unit produced by the Python code
 * generator from the hand-written template (csrc/ew_template.cuh); it must
 * define extern "C" kernels tx_ew_flat and tx_ew_strided.  Compiled for
 * sm_100a without fast-math (-fmad=false, IEEE div/sqrt, no FTZ).  Handles are
 * cached by the caller; tx_ew_destroy unloads. */
int tx_ew_compile(const char* source, const char* name, void** kernel);
/* Compile-only check (no device needed): returns the cubin size. */
int tx_ew_check(const char* source, const char* name, size_t* cubin_bytes);
/* ops: n_out outputs first, then n_in inputs.  Inputs broadcast to the
 * output shape (all outputs share one shape).  err_flag: optional device int
 * set to 1 on integer division by zero. */
int tx_ew_launch(void* kernel, int n_out, int n_in, const tx_tensor* ops, int* err_flag, void* stream);
int tx_ew_destroy(void* kernel);

/* Generated single-entry kernels (row-fused softmax / cross-entropy regions:
 * the composed graph of SURVEY Appendix B run as one warp-per-row kernel).
 * `entry` names the extern "C" kernel; it takes one by-value argument
 * struct, passed here by pointer. */
int tx_kernel_compile(const char* source, const char* name, const char* entry, void** kernel);
int tx_kernel_launch(void* kernel, unsigned grid, unsigned block, void* args, void* stream);
int tx_kernel_destroy(void* kernel);

/* ------------------------------------------------------------ reductions
 * Replaces Sum/Max/ArgmaxOnehot.perform (reference ops/reductions.py:87-188)
 * and adds an index argmax.  axes_mask bit i = reduce dim i. */
enum { TX_SUM = 0, TX_MAX = 1, TX_ARGMAX_ONEHOT = 2, TX_ARGMAX_INDEX = 3 };
/* 2-d convolution data movement (reference ops/conv.py:108-157); `win` =
 * {kh, kw, stride_h, stride_w, pad_h, pad_w}.  tx_im2col: x[N,C,H,W] (any
 * strides) -> cols[N*Ho*Wo, C*kh*kw] row-major, zero padding.  tx_col2im:
 * dcols -> dx[N,C,H,W] contiguous, each element the sum of its taps in
 * (u, v) order (deterministic).  The contractions are tx_gemm calls. */
int tx_im2col(const tx_tensor* x, tx_tensor* cols, const int* win, void* stream);
/* The same patch matrix with the columns in (u, v, c) order --
 * cols[N*Ho*Wo, kh*kw*C] -- for a channel-contiguous input (x given as the
 * [N,C,H,W] view of NHWC memory, channel stride 1): every gather and store
 * is a run along c (128-bit when C % 4 == 0). */
int tx_im2col_hwc(const tx_tensor* x, tx_tensor* cols, const int* win, void* stream);
int tx_col2im(const tx_tensor* dcols, tx_tensor* dx, const int* win, int64_t Ho, int64_t Wo, void* stream);
/* x[N,C,H,W] (any strides) -> y[N, H+2*pad[0], W+2*pad[1], C] contiguous,
 * zero borders: the implicit GEMM's input, in one pass. */
int tx_pad_nhwc(const tx_tensor* x, tx_tensor* y, const int* pad, void* stream);
/* Implicit-GEMM stride-1 convolution on the tensor cores (the reference's
 * im2col + np.dot of ops/conv.py:108-157 without the patch matrix):
 * out[(n,p,q), k] = sum_{u,v,c} xpad[n, p+u, q+v, c] * w[k, (u,v,c)], TF32.
 * xpad: zero-padded NHWC input [N, Hp, Wp, C] contiguous; w: [K, kh*kw*C]
 * contiguous in (u, v, c) order; out: [N*P*Q, K] (NHWC rows) or
 * [N, K, P, Q] (NCHW), contiguous, with P = Hp-kh+1, Q = Wp-kw+1.
 * `win` = {kh, kw}.  TX_E_UNSUPPORTED unless
 * float32, C % 32 == 0, Q <= 128 and 16-byte aligned operands. */
int tx_conv_implicit(const tx_tensor* xpad, const tx_tensor* w, tx_tensor* out, const int* win, void* stream);

/* NaN guard (reference diagnostics.py:52-88 nan_guard_check, hooked per node
 * at runtime.py:359-367): scan one float tensor and OR into flags[slot]
 * bit 1 if it holds a NaN, bit 2 an infinity, bit 4 a finite value with
 * |v| > big (checks enabled by `mode` bits 1/2/4).  Device-side only; the
 * host reads the flag words once per step. */
int tx_check_values(const tx_tensor* x, uint32_t* flags, int slot, int mode, double big, void* stream);

int tx_reduce_workspace(int op, const tx_tensor* x, uint32_t axes_mask, size_t* bytes);
int tx_reduce(int op, const tx_tensor* x, uint32_t axes_mask, tx_tensor* y,
              void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ GEMM
 * Replaces Dot.perform -> np.dot -> OpenBLAS sgemm (reference
 * ops/linalg.py:42-62).  C[M,N] = A[M,K] . B[K,N]; operand transposes are
 * expressed by strides.  fp32 uses tcgen05/TMEM TF32 tensor cores fed by TMA
 * when the layout allows; skinny or float64 problems use CUDA-core kernels. */
enum {
  TX_GEMM_AUTO = 0,    /* tcgen05 TF32 where eligible                    */
  TX_GEMM_SIMT = 1,    /* force CUDA-core fp32/fp64 (exact fp32 products) */
  TX_GEMM_TC = 2,      /* force tcgen05 (error if the layout is ineligible) */
  TX_GEMM_3XTF32 = 3   /* fp32-equivalent: as AUTO, but tcgen05 products run as
                          big/small TF32 splits (3 products into one fp32
                          accumulator, error ~2^-21 |A||B|) -- the reference's
                          sgemm precision; needs tx_gemm_workspace() bytes */
};
/* Optional fused epilogue applied to the accumulator before the store. */
/* Fused epilogues, applied per output element with IEEE round-to-nearest
 * (no FMA contraction) so they round exactly like the elementwise nodes they
 * replace (the compile-time rewrite fuse_gemm_epilogue matches them):
 *   BIAS            C = b[n] + acc                          add(b, dot)
 *   BIAS_TANH       C = tanh(b[n] + acc)
 *   MUL_1MSQR       C = acc * (1 - h^2)
 *   BIAS_TANH_DUAL  C = tanh(b[n] + acc), C2 = 1 - C^2       the MLP forward composite
 *   MUL_AUX         C = acc * g[m,n]                        mul(dot, g) in the backward
 *   SGD             C = w[m,n] - alpha * acc                sub(w, mul(lr, dot)): the SGD update of a
 *                                                           weight from its gradient GEMM (C may alias w) */
enum { TX_EPI_NONE = 0, TX_EPI_BIAS = 1, TX_EPI_BIAS_TANH = 2, TX_EPI_MUL_1MSQR = 3, TX_EPI_BIAS_TANH_DUAL = 4,
       TX_EPI_MUL_AUX = 5, TX_EPI_SGD = 6, TX_EPI_ADD_AUX_BIAS = 7 };
/*   ADD_AUX_BIAS    C = b[n] + (g[m,n] + acc)                  add(b, add(g, dot)): a recurrent layer's
 *                                                              pre-activation (input projection g) */
typedef struct tx_epilogue {
  int32_t kind;
  tx_tensor aux;  /* BIAS*: bias row [N]; MUL_* / SGD / ADD_AUX_BIAS: [M,N] operand */
  tx_tensor out2; /* BIAS_TANH_DUAL: second output [M,N] */
  double alpha;   /* SGD: the learning rate */
  tx_tensor aux2; /* ADD_AUX_BIAS: bias row [N] */
} tx_epilogue;
int tx_gemm_workspace(const tx_tensor* A, const tx_tensor* B, const tx_tensor* C, int mode,
                      size_t* bytes);
int tx_gemm(const tx_tensor* A, const tx_tensor* B, tx_tensor* C, const tx_epilogue* epi,
            int mode, void* workspace, size_t workspace_bytes, void* stream);
/* Which path tx_gemm would take (0 simt, 1 skinny, 2 tcgen05). */
int tx_gemm_path(const tx_tensor* A, const tx_tensor* B, const tx_tensor* C, int mode, int* path);

/* ------------------------------------------------------ fused layer grad
 * The backward of a tanh layer h feeding a narrow dense layer z = h.W + b
 * (k = z's width <= 16; the MLP's 10-class output), one pass over h.
 * Replaces, from the differentiated graph, Dot.grad's two products
 * (reference ops/linalg.py:68-70), the tanh-grad composite
 * (ops/elemwise.py:126-157) and the bias gradient Sum[0]
 * (ops/reductions.py:87-112 via ops/elemwise.py:411-442):
 *   dh = dot(dz, wt) * (1 - h^2)   dz [B,k], wt = W^T [k,H] (strides), h, dh [B,H]
 *   gW = epi(dot(h^T, dz))         [H,k]; epi NONE or SGD (aux = W, C may alias it)
 *   db = sum(dh, axis 0)           [H]; skipped when db is NULL or db->data is NULL
 * gW and db are summed in a fixed order (deterministic).  Layouts the fused
 * kernel does not take (float64, k > 16, unaligned rows) run the three ops
 * through tx_gemm / tx_reduce with the same workspace. */
int tx_narrow_grad_workspace(const tx_tensor* dz, const tx_tensor* wt, const tx_tensor* h, const tx_tensor* dh,
                             const tx_tensor* gw, const tx_tensor* db, int mode, size_t* bytes);
int tx_narrow_grad(const tx_tensor* dz, const tx_tensor* wt, const tx_tensor* h, tx_tensor* dh, tx_tensor* gw,
                   const tx_epilogue* gw_epi, tx_tensor* db, int mode, void* workspace, size_t workspace_bytes,
                   void* stream);

/* ------------------------------------------------------------------ NCCL
 * Gradient sync for data-parallel updates (new; Platoon-style synchronous
 * DP).  libnccl.so.2 is dlopen'ed (the one torch loaded). */
int tx_nccl_unique_id(char out[128]);
int tx_nccl_init(int nranks, int rank, const char uid[128], void** comm);
int tx_nccl_allreduce_sum(void* comm, void* buf, size_t count, int dtype, void* stream);
int tx_nccl_destroy(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* TEXPR_B200_H */
