// Runtime half of the C-ABI: errors, device memory, streams, events.
// Replaces the reference's host-memory Arena backing store (tensor.cpp:30-59)
// with device memory; the host C++ arena carves graph workspaces out of one
// mtkc_malloc'd slab.
#include "common.cuh"

#include <cstdio>

namespace mtkc {

static thread_local std::string t_err;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if(e == cudaSuccess)
    return MTKC_OK;
  t_err = std::string(where) + ": " + cudaGetErrorString(e);
  return MTKC_CUDA;
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

}  // namespace mtkc

using namespace mtkc;

extern "C" {

const char* mtkc_last_error(void) { return t_err.c_str(); }

uint64_t mtkc_launch_count(void) { return g_launches.load(); }

int mtkc_init(int device) { return cuda_status(cudaSetDevice(device), "cudaSetDevice"); }

int mtkc_device_count(int* count) {
  return cuda_status(cudaGetDeviceCount(count), "cudaGetDeviceCount");
}

int mtkc_sm_count(int* count) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if(e != cudaSuccess)
    return cuda_status(e, "cudaGetDevice");
  return cuda_status(cudaDeviceGetAttribute(count, cudaDevAttrMultiProcessorCount, dev),
                     "cudaDeviceGetAttribute");
}

int mtkc_malloc(void** ptr, size_t bytes) {
  return cuda_status(cudaMalloc(ptr, bytes), "cudaMalloc");
}

int mtkc_free(void* ptr) { return cuda_status(cudaFree(ptr), "cudaFree"); }

int mtkc_host_alloc_pinned(void** ptr, size_t bytes) {
  return cuda_status(cudaMallocHost(ptr, bytes), "cudaMallocHost");
}

int mtkc_host_free_pinned(void* ptr) { return cuda_status(cudaFreeHost(ptr), "cudaFreeHost"); }

int mtkc_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(stream)),
                     "cudaMemcpyAsync(H2D)");
}

int mtkc_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S(stream)),
                     "cudaMemcpyAsync(D2H)");
}

int mtkc_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream)),
                     "cudaMemcpyAsync(D2D)");
}

int mtkc_memset(void* dst, int value, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  return cuda_status(cudaMemsetAsync(dst, value, bytes, S(stream)), "cudaMemsetAsync");
}

int mtkc_stream_create(void** stream) {
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  *stream = (void*)s;
  return cuda_status(e, "cudaStreamCreate");
}

int mtkc_stream_destroy(void* stream) {
  return cuda_status(cudaStreamDestroy(S(stream)), "cudaStreamDestroy");
}

int mtkc_stream_sync(void* stream) {
  return cuda_status(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize");
}

int mtkc_event_create(void** ev) {
  cudaEvent_t e;
  cudaError_t r = cudaEventCreate(&e);
  *ev = (void*)e;
  return cuda_status(r, "cudaEventCreate");
}

int mtkc_event_destroy(void* ev) {
  return cuda_status(cudaEventDestroy((cudaEvent_t)ev), "cudaEventDestroy");
}

int mtkc_event_record(void* ev, void* stream) {
  return cuda_status(cudaEventRecord((cudaEvent_t)ev, S(stream)), "cudaEventRecord");
}

int mtkc_stream_wait_event(void* stream, void* ev) {
  return cuda_status(cudaStreamWaitEvent(S(stream), (cudaEvent_t)ev, 0), "cudaStreamWaitEvent");
}

int mtkc_event_elapsed_ms(void* start, void* stop, float* ms) {
  return cuda_status(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop),
                     "cudaEventElapsedTime");
}

int mtkc_device_sync(void) { return cuda_status(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

}  // extern "C"
