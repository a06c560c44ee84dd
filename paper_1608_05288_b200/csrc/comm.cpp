// comm.cpp — built-in NCCL transport for the all-gather of row-sharded UTIL
// messages.  NCCL is loaded at run time (dlopen of
// libnccl.so.2, the copy torch ships or the system one), so libgbe has no
// link-time dependency on it and single-GPU use never touches it.  The
// collective runs on the solve stream over NVLink 5 / NVSwitch.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "common.h"
#include "executor.h"

namespace gbe {
namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.x)
typedef struct ncclComm *ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclUint8 = 1;

struct Nccl {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, void *) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl &nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
    n.AllGather = (decltype(n.AllGather))dlsym(n.h, "ncclAllGather");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
  });
  if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.AllGather || !n.CommDestroy)
    GBE_FAIL(GBE_E_COMM, "NCCL not available (dlopen libnccl.so.2 failed: %s)", dlerror() ? dlerror() : "?");
  return n;
}

ncclComm_t g_comm = nullptr;

int nccl_allgather(const void *send, void *recv, size_t bytes, void *stream, void *u) {
  (void)u;
  Nccl &n = nccl();
  return n.AllGather(send, recv, bytes, kNcclUint8, g_comm, stream) == 0 ? 0 : 1;
}

}  // namespace

void comm_nccl_id(void *id128) {
  Nccl &n = nccl();
  ncclUniqueId id;
  ncclResult_t r = n.GetUniqueId(&id);
  if (r != 0) GBE_FAIL(GBE_E_COMM, "ncclGetUniqueId: %s", n.GetErrorString ? n.GetErrorString(r) : "?");
  std::memcpy(id128, id.internal, 128);
}

void comm_nccl_init(const void *id128, int nranks, int rank, int device) {
  Nccl &n = nccl();
  if (nranks < 1 || rank < 0 || rank >= nranks) GBE_FAIL(GBE_E_INVALID, "bad nranks/rank");
  if (cudaSetDevice(device) != cudaSuccess) GBE_FAIL(GBE_E_CUDA, "cudaSetDevice(%d) failed", device);
  if (g_comm) {
    n.CommDestroy(g_comm);
    g_comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(id.internal, id128, 128);
  ncclResult_t r = n.CommInitRank(&g_comm, nranks, id, rank);
  if (r != 0) GBE_FAIL(GBE_E_COMM, "ncclCommInitRank: %s", n.GetErrorString ? n.GetErrorString(r) : "?");
  set_allgather_capturable(nccl_allgather, nullptr);
}

void comm_finalize() {
  if (g_comm) {
    nccl().CommDestroy(g_comm);
    g_comm = nullptr;
    set_allgather(nullptr, nullptr);
  }
}

}  // namespace gbe
