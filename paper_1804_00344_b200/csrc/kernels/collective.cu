// Data-parallel gradient exchange.  The reference combines worker gradients
// with a sequential host loop g = sum_i (tokens_i/total) g_i in worker order
// (trainSync train.cpp:254-269); here every rank pre-scales its gradient by
// tokens_r/total (through the loss seed) and the ranks sum with NCCL
// all-reduces over NVLink/NVSwitch.
//
// NCCL is bound at first use with dlopen: a process that already loaded
// libnccl.so.2 (e.g. PyTorch's bundled NCCL) reuses that copy, so the two
// never conflict; MTK_NCCL_LIB selects a specific library.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

using namespace mtkc;

namespace {

struct Nccl {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  bool ok = false;
  std::string err;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("MTK_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if(!h) {
      n.err = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
    n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
    n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
    n.allReduce = (decltype(n.allReduce))dlsym(h, "ncclAllReduce");
    n.errorString = (decltype(n.errorString))dlsym(h, "ncclGetErrorString");
    n.commCount = (decltype(n.commCount))dlsym(h, "ncclCommCount");
    n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.allReduce && n.errorString &&
           n.commCount;
    if(!n.ok)
      n.err = "NCCL library lacks required symbols";
  });
  return n;
}

int nccl_status(ncclResult_t r, const char* where) {
  if(r == ncclSuccess)
    return MTKC_OK;
  return fail(MTKC_CUDA, std::string(where) + ": " + nccl().errorString(r));
}

#define NCCL_READY()                                   \
  do {                                                 \
    if(!nccl().ok)                                     \
      return fail(MTKC_CUDA, nccl().err);              \
  } while(0)

}  // namespace

extern "C" {

int mtkc_nccl_unique_id(void* id_out_128) {
  NCCL_READY();
  ncclUniqueId id;
  int rc = nccl_status(nccl().getUniqueId(&id), "ncclGetUniqueId");
  if(rc)
    return rc;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id_out_128, &id, sizeof(id));
  return MTKC_OK;
}

int mtkc_nccl_comm_init(void** comm, int nranks, int rank, const void* id_128) {
  NCCL_READY();
  ncclUniqueId id;
  std::memcpy(&id, id_128, sizeof(id));
  ncclComm_t c;
  int rc = nccl_status(nccl().commInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  if(rc)
    return rc;
  *comm = (void*)c;
  return MTKC_OK;
}

int mtkc_nccl_comm_destroy(void* comm) {
  NCCL_READY();
  return nccl_status(nccl().commDestroy((ncclComm_t)comm), "ncclCommDestroy");
}

int mtkc_nccl_comm_count(void* comm, int* count) {
  NCCL_READY();
  return nccl_status(nccl().commCount((ncclComm_t)comm, count), "ncclCommCount");
}

int mtkc_allreduce_sum(void* comm, float* buf, int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  NCCL_READY();
  ProfScope prof(S(stream), "allreduce", 4.0 * n);
  return nccl_status(nccl().allReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum,
                                      (ncclComm_t)comm, S(stream)),
                     "ncclAllReduce");
}

}  // extern "C"
