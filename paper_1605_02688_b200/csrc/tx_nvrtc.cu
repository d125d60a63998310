// NVRTC compilation and launch of generated fused-elementwise kernels.
//
// Replaces the reference's chunked NumPy evaluation of Composite nodes
// (pkg/src/texpr/ops/elemwise.py:538-597) and single Elemwise.perform
// (:314-326).  The driver API is reached through cudaGetDriverEntryPoint so
// the library loads on hosts without a GPU driver (CPU CI loads it to check
// exports) and links no libcuda.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tx_common.h"

namespace tx {

// ---------------------------------------------------------- driver entry points
struct Drv {
  CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*moduleUnload)(CUmodule) = nullptr;
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           CUstream, void**, void**) = nullptr;
  CUresult (*launchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;  // optional
  CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*getErrorString)(CUresult, const char**) = nullptr;
  bool ok = false;
};

static Drv g_drv;
static std::once_flag g_drv_once;

template <class F>
static bool entry(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

static const Drv& drv() {
  std::call_once(g_drv_once, [] {
    Drv d;
    d.ok = entry("cuModuleLoadData", &d.moduleLoadData) && entry("cuModuleUnload", &d.moduleUnload) &&
           entry("cuModuleGetFunction", &d.moduleGetFunction) && entry("cuLaunchKernel", &d.launchKernel) &&
           entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", &d.occupancy) &&
           entry("cuGetErrorString", &d.getErrorString);
    if (!entry("cuLaunchKernelEx", &d.launchKernelEx)) d.launchKernelEx = nullptr;
    g_drv = d;
  });
  return g_drv;
}

// cuLaunchKernel, as a programmatic dependent launch when the kernel opens
// with griddepcontrol.wait (every generated kernel of this library does;
// tx_common.h TX_GRID_WAIT)
static CUresult launch_drv(CUfunction fn, unsigned gx, unsigned gy, unsigned gz, unsigned bx, unsigned by, unsigned bz,
                           unsigned smem, CUstream st, void** params, bool waits) {
  const Drv& d = drv();
  if (!waits || !d.launchKernelEx || !pdl_enabled())
    return d.launchKernel(fn, gx, gy, gz, bx, by, bz, smem, st, params, nullptr);
  CUlaunchAttribute attr[1];
  attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  attr[0].value.programmaticStreamSerializationAllowed = 1;
  CUlaunchConfig cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDimX = gx; cfg.gridDimY = gy; cfg.gridDimZ = gz;
  cfg.blockDimX = bx; cfg.blockDimY = by; cfg.blockDimZ = bz;
  cfg.sharedMemBytes = smem;
  cfg.hStream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return d.launchKernelEx(&cfg, fn, params, nullptr);
}

static int drv_fail(CUresult r, const char* what) {
  const char* s = "unknown";
  if (drv().getErrorString) drv().getErrorString(r, &s);
  return fail(TX_E_CUDA, std::string(what) + ": " + s);
}

// --------------------------------------------------------------- compilation
static int nvrtc_compile(const char* source, const char* name, std::vector<char>* cubin) {
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, source, name, 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail(TX_E_NVRTC, std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false", "--prec-div=true",
                        "--prec-sqrt=true", "--ftz=false", 
                        "--extra-device-vectorization"};
  r = nvrtcCompileProgram(prog, sizeof(opts) / sizeof(opts[0]), opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return fail(TX_E_NVRTC, std::string("NVRTC compile of ") + name + " failed:\n" + log);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  return TX_OK;
}

struct EwKernel {
  CUmodule mod = nullptr;
  CUfunction flat = nullptr, k2d = nullptr, k2dv = nullptr, knd = nullptr;
  int occ_flat = 4, occ_nd = 4;
};

// Layout of the generated kernels' single by-value parameter
// (csrc/ew_template.cuh struct TxEwArgs).
struct TxEwArgs {
  int64_t n;
  int32_t ndim;
  int32_t vec_ok;
  int64_t shape[TX_MAX_RANK];
  void* ptr[24];
  int64_t strides[24][TX_MAX_RANK];
  int* err;
};

}  // namespace tx

using namespace tx;

extern "C" {

int tx_ew_check(const char* source, const char* name, size_t* cubin_bytes) {
  std::vector<char> cubin;
  int rc = nvrtc_compile(source, name, &cubin);
  if (rc) return rc;
  if (cubin_bytes) *cubin_bytes = cubin.size();
  return TX_OK;
}

int tx_ew_compile(const char* source, const char* name, void** out) {
  const Drv& d = drv();
  TX_CHECK(d.ok, TX_E_NODEVICE, "CUDA driver entry points unavailable");
  std::vector<char> cubin;
  int rc = nvrtc_compile(source, name, &cubin);
  if (rc) return rc;
  EwKernel* k = new EwKernel();
  CUresult r = d.moduleLoadData(&k->mod, cubin.data());
  if (r != CUDA_SUCCESS) { delete k; return drv_fail(r, "cuModuleLoadData"); }
  if ((r = d.moduleGetFunction(&k->flat, k->mod, "tx_ew_flat")) != CUDA_SUCCESS ||
      (r = d.moduleGetFunction(&k->k2d, k->mod, "tx_ew_2d")) != CUDA_SUCCESS ||
      (r = d.moduleGetFunction(&k->k2dv, k->mod, "tx_ew_2dv")) != CUDA_SUCCESS ||
      (r = d.moduleGetFunction(&k->knd, k->mod, "tx_ew_nd")) != CUDA_SUCCESS) {
    d.moduleUnload(k->mod);
    delete k;
    return drv_fail(r, "cuModuleGetFunction");
  }
  int occ = 0;
  if (d.occupancy(&occ, k->flat, 256, 0) == CUDA_SUCCESS && occ > 0) k->occ_flat = occ;
  if (d.occupancy(&occ, k->knd, 256, 0) == CUDA_SUCCESS && occ > 0) k->occ_nd = occ;
  *out = k;
  return TX_OK;
}

// Generic generated kernels (row-fused regions): one module, one named entry
// taking a single by-value argument struct.
struct GenKernel {
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  bool waits = false;  // the source opens with griddepcontrol.wait: launched as a programmatic dependent
};

int tx_kernel_compile(const char* source, const char* name, const char* entry, void** out) {
  const Drv& d = drv();
  TX_CHECK(d.ok, TX_E_NODEVICE, "CUDA driver entry points unavailable");
  std::vector<char> cubin;
  int rc = nvrtc_compile(source, name, &cubin);
  if (rc) return rc;
  GenKernel* k = new GenKernel();
  k->waits = strstr(source, "griddepcontrol.wait") != nullptr;
  CUresult r = d.moduleLoadData(&k->mod, cubin.data());
  if (r != CUDA_SUCCESS) { delete k; return drv_fail(r, "cuModuleLoadData"); }
  if ((r = d.moduleGetFunction(&k->fn, k->mod, entry)) != CUDA_SUCCESS) {
    d.moduleUnload(k->mod);
    delete k;
    return drv_fail(r, "cuModuleGetFunction");
  }
  *out = k;
  return TX_OK;
}

int tx_kernel_launch(void* h, unsigned grid, unsigned block, void* args, void* stream) {
  GenKernel* k = (GenKernel*)h;
  TX_CHECK(k && drv().ok, TX_E_ARG, "tx_kernel_launch: invalid handle");
  void* params[] = {args};
  CUresult r = launch_drv(k->fn, grid, 1, 1, block, 1, 1, 0, (cudaStream_t)stream, params, k->waits);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuLaunchKernel(generated)");
  return TX_OK;
}

int tx_kernel_destroy(void* h) {
  GenKernel* k = (GenKernel*)h;
  if (!k) return TX_OK;
  if (k->mod && drv().moduleUnload) drv().moduleUnload(k->mod);
  delete k;
  return TX_OK;
}

int tx_ew_destroy(void* h) {
  EwKernel* k = (EwKernel*)h;
  if (!k) return TX_OK;
  if (k->mod && drv().moduleUnload) drv().moduleUnload(k->mod);
  delete k;
  return TX_OK;
}

int tx_ew_launch(void* h, int n_out, int n_in, const tx_tensor* ops, int* err_flag, void* stream) {
  EwKernel* k = (EwKernel*)h;
  const Drv& d = drv();
  TX_CHECK(k && d.ok, TX_E_ARG, "tx_ew_launch: invalid kernel handle");
  const int nops = n_out + n_in;
  TX_CHECK(n_out >= 1 && nops <= 24, TX_E_ARG, "tx_ew_launch: operand count");
  const tx_tensor& o0 = ops[0];
  const int nd = o0.ndim;
  for (int i = 0; i < n_out; ++i) {
    TX_CHECK(ops[i].ndim == nd, TX_E_ARG, "tx_ew_launch: outputs must share one rank");
    for (int j = 0; j < nd; ++j) TX_CHECK(ops[i].shape[j] == o0.shape[j], TX_E_ARG, "tx_ew_launch: output shapes differ");
  }
  TxEwArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = numel(o0);
  a.err = err_flag;
  if (a.n == 0) return TX_OK;
  // right-align every operand against the output shape; broadcast dims get stride 0
  int64_t st[24][TX_MAX_RANK];
  bool flat = true;
  for (int op = 0; op < nops; ++op) {
    const tx_tensor& t = ops[op];
    TX_CHECK(t.ndim <= nd, TX_E_ARG, "tx_ew_launch: input rank exceeds output rank");
    for (int i = 0; i < nd; ++i) {
      int j = i - (nd - t.ndim);
      if (j < 0 || t.shape[j] == 1) {
        st[op][i] = 0;
        if (o0.shape[i] != 1) flat = false;
      } else {
        TX_CHECK(t.shape[j] == o0.shape[i], TX_E_ARG, "tx_ew_launch: operand does not broadcast to the output");
        st[op][i] = t.strides[j];
      }
    }
    a.ptr[op] = t.data;
  }
  Space sp;
  collapse(nd, o0.shape, nops, st, &sp);
  if (flat) {
    // flat only if every operand is the same dense row-major layout
    for (int op = 0; op < nops && flat; ++op) {
      int64_t expect = 1;
      for (int i = sp.ndim - 1; i >= 0; --i) {
        if (sp.strides[op][i] != expect) { flat = false; break; }
        expect *= sp.shape[i];
      }
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int sms = sm_count();
  CUresult r;
  void* params[] = {&a};
  if (flat) {
    bool vec = true;
    for (int op = 0; op < nops; ++op) {
      int isz = itemsize(ops[op].dtype);
      uintptr_t p = (uintptr_t)ops[op].data;
      if ((isz == 1 && (p & 3)) || (isz >= 4 && (p & 15))) vec = false;
    }
    a.vec_ok = vec ? 1 : 0;
    int64_t work = vec ? (a.n + 3) / 4 : a.n;
    int64_t blocks = (work + 255) / 256;
    int64_t cap = (int64_t)sms * k->occ_flat;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    r = launch_drv(k->flat, (unsigned)blocks, 1, 1, 256, 1, 1, 0, s, params, true);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuLaunchKernel(tx_ew_flat)");
    return TX_OK;
  }
  a.ndim = sp.ndim;
  for (int i = 0; i < sp.ndim; ++i) a.shape[i] = sp.shape[i];
  for (int op = 0; op < nops; ++op)
    for (int i = 0; i < sp.ndim; ++i) a.strides[op][i] = sp.strides[op][i];
  if (sp.ndim >= 3 && sp.ndim <= 4 && a.n < (int64_t)1 << 31 && !getenv("TX_EW_NO_ROWS")) {
    // row-major form (ew_template.cuh TX_ROW_COORDS): [0] inner row dim,
    // [1] columns, [2] / [3] outer row dims
    const int nd = sp.ndim;
    const int map[4] = {nd - 2, nd - 1, nd - 3, nd - 4};
    for (int i = 0; i < 4; ++i) a.shape[i] = i < nd ? sp.shape[map[i]] : 1;
    for (int op = 0; op < nops; ++op)
      for (int i = 0; i < 4; ++i) a.strides[op][i] = i < nd ? sp.strides[op][map[i]] : 0;
  }
  if (sp.ndim <= 4 && a.n < (int64_t)1 << 31 && (sp.ndim <= 2 || !getenv("TX_EW_NO_ROWS"))) {
    if (sp.ndim == 1) {  // treat as one row
      a.shape[1] = a.shape[0];
      a.shape[0] = 1;
      for (int op = 0; op < nops; ++op) { a.strides[op][1] = a.strides[op][0]; a.strides[op][0] = 0; }
    } else if (sp.ndim == 0) {
      a.shape[0] = a.shape[1] = 1;
    }
    int64_t rows = a.shape[0] * (sp.ndim >= 3 ? a.shape[2] : 1) * (sp.ndim >= 4 ? a.shape[3] : 1), cols = a.shape[1];
    // vectorised variant: column strides in {0,1}, outputs contiguous along
    // columns, rows 16 B aligned for every vector-loaded operand
    bool v2 = (cols % 4 == 0);
    for (int op = 0; op < nops && v2; ++op) {
      const int64_t s1 = a.strides[op][1];
      const int isz = itemsize(ops[op].dtype);
      const uintptr_t pa = (uintptr_t)ops[op].data;
      if (op < n_out && s1 != 1) v2 = false;
      if (s1 != 0 && s1 != 1) v2 = false;
      if (s1 == 1) {
        const int64_t need = isz == 1 ? 4 : 16;
        if ((pa % need) || ((a.strides[op][0] * isz) % need) || ((a.strides[op][2] * isz) % need) ||
            ((a.strides[op][3] * isz) % need))
          v2 = false;
      }
    }
    if (v2) {
      unsigned gx = (unsigned)((cols / 4 + 255) / 256);
      int64_t gy = rows < 65535 ? rows : 65535;
      r = launch_drv(k->k2dv, gx, (unsigned)gy, 1, 256, 1, 1, 0, s, params, true);
      if (r != CUDA_SUCCESS) return drv_fail(r, "cuLaunchKernel(tx_ew_2dv)");
      return TX_OK;
    }
    unsigned gx = (unsigned)((cols + 255) / 256);
    int64_t gy = rows;
    int64_t want = ((int64_t)sms * 8 + gx - 1) / gx;  // enough CTAs to fill the chip
    if (gy > want) gy = want;
    if (gy > 65535) gy = 65535;
    if (gy < 1) gy = 1;
    r = launch_drv(k->k2d, gx, (unsigned)gy, 1, 256, 1, 1, 0, s, params, true);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuLaunchKernel(tx_ew_2d)");
    return TX_OK;
  }
  static const bool trace = getenv("TX_EW_TRACE_ND") != nullptr;  // diagnostics: which launches take the N-d path
  if (trace) {
    fprintf(stderr, "tx_ew_nd: n=%lld ndim=%d shape", (long long)a.n, sp.ndim);
    for (int i = 0; i < sp.ndim; ++i) fprintf(stderr, " %lld", (long long)sp.shape[i]);
    for (int op = 0; op < nops; ++op) {
      fprintf(stderr, " | op%d", op);
      for (int i = 0; i < sp.ndim; ++i) fprintf(stderr, " %lld", (long long)sp.strides[op][i]);
    }
    fprintf(stderr, "\n");
  }
  int64_t blocks = (a.n + 255) / 256;
  int64_t cap = (int64_t)sms * k->occ_nd;
  if (blocks > cap) blocks = cap;
  r = launch_drv(k->knd, (unsigned)blocks, 1, 1, 256, 1, 1, 0, s, params, true);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuLaunchKernel(tx_ew_nd)");
  return TX_OK;
}

}  // extern "C"
