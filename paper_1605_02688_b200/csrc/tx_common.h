// Internal helpers shared by the libtexpr_b200 translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/texpr_b200.h"

namespace tx {

void set_error(const std::string& msg);

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

inline int cuda_fail(cudaError_t e, const char* what) {
  return fail(TX_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define TX_CUDA(call)                                        \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return ::tx::cuda_fail(_e, #call); \
  } while (0)

#define TX_CHECK(cond, code, msg)                   \
  do {                                              \
    if (!(cond)) return ::tx::fail((code), (msg));  \
  } while (0)

inline int itemsize(int dtype) {
  switch (dtype) {
    case TX_F32: case TX_I32: return 4;
    case TX_F64: case TX_I64: return 8;
    case TX_BOOL: return 1;
  }
  return 0;
}

inline int64_t numel(const tx_tensor& t) {
  int64_t n = 1;
  for (int i = 0; i < t.ndim; ++i) n *= t.shape[i];
  return n;
}

inline bool is_contiguous(const tx_tensor& t) {
  int64_t s = 1;
  for (int i = t.ndim - 1; i >= 0; --i) {
    if (t.shape[i] != 1 && t.strides[i] != s) return false;
    s *= t.shape[i];
  }
  return true;
}

// A flattened iteration space: dims merged where every operand is
// stride-compatible, extent-1 dims removed.
struct Space {
  int ndim = 0;
  int64_t shape[TX_MAX_RANK];
  int64_t strides[32][TX_MAX_RANK];  // per operand
};

// Collapse `nops` operands broadcast against `shape` (rank `ndim`,
// per-operand strides already right-aligned to that rank).
void collapse(int ndim, const int64_t* shape, int nops, const int64_t (*strides)[TX_MAX_RANK], Space* out);

int sm_count();

// ---------------------------------------------- programmatic dependent launch
// Every kernel of the library starts with TX_GRID_WAIT() (griddepcontrol.wait:
// returns once the preceding kernel in the stream has completed and its
// writes are visible; immediately when there is none) and is launched with
// the programmatic-stream-serialization attribute; right after the wait it
// releases its own dependents (griddepcontrol.launch_dependents), so the next
// kernel's CTAs are launched and resident while this one runs and start the
// moment it completes -- inside captured CUDA graphs too.  The chains of small dependent kernels (an unrolled scan's
// bodies, the logistic-regression step) are launch-latency bound; this is
// the gap it closes.  TX_NO_PDL=1 launches plainly (A/B).
#define TX_GRID_WAIT() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
bool pdl_enabled();

template <class... KArgs, class... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// cuTensorMapEncodeTiled through the runtime's driver entry point (nullptr
// when no driver is present); shared by the GEMM and reduction TMA paths
void* tmap_encoder();
int reduce_launch(int op, const tx_tensor& x, uint32_t mask, tx_tensor& y, void* ws, size_t ws_bytes,
                  cudaStream_t st);

}  // namespace tx
