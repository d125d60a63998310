// NCCL gradient synchronisation for data-parallel training steps.
//
// New subsystem (the reference has no distribution; the paper's Platoon is
// described at PAPER.md:530-546).  libnccl.so.2 is dlopen'ed lazily so the
// library loads on CPU-only hosts and binds to the NCCL torch already loaded
// in the process (same soname -> same instance).  The allreduce is issued on
// the VM's stream, so it is captured into the step's CUDA graph with the
// kernels around it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "tx_common.h"

namespace tx {
namespace {

typedef struct { char internal[128]; } UniqueId;
typedef void* Comm;
typedef int (*GetUniqueIdFn)(UniqueId*);
typedef int (*CommInitRankFn)(Comm*, int, UniqueId, int);
typedef int (*AllReduceFn)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*CommDestroyFn)(Comm);
typedef const char* (*ErrStrFn)(int);

struct Nccl {
  void* h = nullptr;
  GetUniqueIdFn uid = nullptr;
  CommInitRankFn init = nullptr;
  AllReduceFn allreduce = nullptr;
  CommDestroyFn destroy = nullptr;
  ErrStrFn err = nullptr;
};
Nccl g_nccl;
std::once_flag g_once;

const Nccl& nccl() {
  std::call_once(g_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_nccl.h = h;
    g_nccl.uid = (GetUniqueIdFn)dlsym(h, "ncclGetUniqueId");
    g_nccl.init = (CommInitRankFn)dlsym(h, "ncclCommInitRank");
    g_nccl.allreduce = (AllReduceFn)dlsym(h, "ncclAllReduce");
    g_nccl.destroy = (CommDestroyFn)dlsym(h, "ncclCommDestroy");
    g_nccl.err = (ErrStrFn)dlsym(h, "ncclGetErrorString");
  });
  return g_nccl;
}

int nccl_fail(int r, const char* what) {
  const char* s = nccl().err ? nccl().err(r) : "unknown";
  return fail(TX_E_NCCL, std::string(what) + ": " + s);
}

// ncclDataType_t values
int nccl_dtype(int tx) {
  switch (tx) {
    case TX_F32: return 7;  // ncclFloat32
    case TX_F64: return 8;  // ncclFloat64
    case TX_I32: return 2;  // ncclInt32
    case TX_I64: return 4;  // ncclInt64
    case TX_BOOL: return 1; // ncclUint8
  }
  return -1;
}

}  // namespace
}  // namespace tx

using namespace tx;

extern "C" {

int tx_nccl_unique_id(char out[128]) {
  const Nccl& n = nccl();
  TX_CHECK(n.uid, TX_E_NCCL, "libnccl.so.2 not available");
  UniqueId id;
  int r = n.uid(&id);
  if (r) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
  return TX_OK;
}

int tx_nccl_init(int nranks, int rank, const char uid[128], void** comm) {
  const Nccl& n = nccl();
  TX_CHECK(n.init, TX_E_NCCL, "libnccl.so.2 not available");
  UniqueId id;
  std::memcpy(id.internal, uid, 128);
  Comm c = nullptr;
  int r = n.init(&c, nranks, id, rank);
  if (r) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return TX_OK;
}

int tx_nccl_allreduce_sum(void* comm, void* buf, size_t count, int dtype, void* stream) {
  const Nccl& n = nccl();
  TX_CHECK(n.allreduce && comm, TX_E_NCCL, "NCCL communicator not initialised");
  int dt = nccl_dtype(dtype);
  TX_CHECK(dt >= 0, TX_E_ARG, "tx_nccl_allreduce_sum: dtype");
  int r = n.allreduce(buf, buf, count, dt, /*ncclSum*/ 0, (Comm)comm, (cudaStream_t)stream);
  if (r) return nccl_fail(r, "ncclAllReduce");
  return TX_OK;
}

int tx_nccl_destroy(void* comm) {
  const Nccl& n = nccl();
  if (!comm || !n.destroy) return TX_OK;
  int r = n.destroy((Comm)comm);
  if (r) return nccl_fail(r, "ncclCommDestroy");
  return TX_OK;
}

}  // extern "C"
