// Data-parallel gradient exchange.  The reference combines worker gradients
// with a sequential host loop g = sum_i (tokens_i/total) g_i in worker order
// (trainSync train.cpp:254-269); here every rank pre-scales its gradient by
// tokens_r/total (through the loss seed) and the ranks sum with one NCCL
// all-reduce per gradient bucket over NVLink/NVSwitch.
#include <nccl.h>

#include <cstring>

#include "common.cuh"

using namespace mtkc;

namespace {
int nccl_status(ncclResult_t r, const char* where) {
  if(r == ncclSuccess)
    return MTKC_OK;
  return fail(MTKC_CUDA, std::string(where) + ": " + ncclGetErrorString(r));
}
}  // namespace

extern "C" {

int mtkc_nccl_unique_id(void* id_out_128) {
  ncclUniqueId id;
  int rc = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId");
  if(rc)
    return rc;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id_out_128, &id, sizeof(id));
  return MTKC_OK;
}

int mtkc_nccl_comm_init(void** comm, int nranks, int rank, const void* id_128) {
  ncclUniqueId id;
  std::memcpy(&id, id_128, sizeof(id));
  ncclComm_t c;
  int rc = nccl_status(ncclCommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  if(rc)
    return rc;
  *comm = (void*)c;
  return MTKC_OK;
}

int mtkc_nccl_comm_destroy(void* comm) {
  return nccl_status(ncclCommDestroy((ncclComm_t)comm), "ncclCommDestroy");
}

int mtkc_allreduce_sum(void* comm, float* buf, int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  return nccl_status(
      ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, (ncclComm_t)comm, S(stream)),
      "ncclAllReduce");
}

}  // extern "C"
