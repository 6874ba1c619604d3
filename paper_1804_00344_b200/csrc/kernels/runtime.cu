// Runtime half of the C-ABI: errors, device memory, streams, events.
// Replaces the reference's host-memory Arena backing store (tensor.cpp:30-59)
// with device memory; the host C++ arena carves graph workspaces out of one
// mtkc_malloc'd slab.
#include "common.cuh"

#include <execinfo.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

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

bool pdl_enabled() {
  static const bool on = std::getenv("MTK_NO_PDL") == nullptr;
  return on;
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static std::atomic<uint64_t> g_h2d{0}, g_d2h{0};

namespace {
// dst[i] = src[i]; host (mapped pinned) sources are read into registers
// before the programmatic-dependency wait, device sources after it
constexpr int COPY_U = 4;
template <typename T>
__global__ void __launch_bounds__(256) copy_kernel(T* dst, const T* src, size_t n, int hostSrc) {
  if(hostSrc) {
    const size_t i0 = (size_t)blockIdx.x * 256 * COPY_U + threadIdx.x;
    T v[COPY_U];
#pragma unroll
    for(int u = 0; u < COPY_U; ++u)
      if(i0 + (size_t)u * 256 < n)
        v[u] = src[i0 + (size_t)u * 256];
    MTKC_PDL_ENTRY();
#pragma unroll
    for(int u = 0; u < COPY_U; ++u)
      if(i0 + (size_t)u * 256 < n)
        dst[i0 + (size_t)u * 256] = v[u];
    return;
  }
  MTKC_PDL_ENTRY();
  for(size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256)
    dst[i] = src[i];
}

template <typename T>
__global__ void __launch_bounds__(256) fill_kernel(T* dst, size_t n, T v) {
  MTKC_PDL_ENTRY();
  for(size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256)
    dst[i] = v;
}

// MTK_TRACE_BLOCK=<us>: report (with a host backtrace) every runtime call that
// blocked the host longer than <us> microseconds -- finds hidden syncs.
double trace_block_us() {
  static double us = [] {
    const char* e = std::getenv("MTK_TRACE_BLOCK");
    return e ? std::atof(e) : -1.0;
  }();
  return us;
}
struct BlockTimer {
  const char* what;
  std::chrono::steady_clock::time_point t0;
  explicit BlockTimer(const char* w) : what(w) {
    if(trace_block_us() >= 0)
      t0 = std::chrono::steady_clock::now();
  }
  ~BlockTimer() {
    double lim = trace_block_us();
    if(lim < 0)
      return;
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                    .count();
    if(us < lim)
      return;
    double now = std::chrono::duration<double>(
                     std::chrono::steady_clock::now().time_since_epoch()).count();
    std::fprintf(stderr, "[mtk block] %s %.0f us at %.6f\n", what, us, now);
    void* bt[12];
    int n = backtrace(bt, 12);
    backtrace_symbols_fd(bt + 1, n - 1, 2);
  }
};
}  // namespace

// ------------------------------------------------------------ profiling
namespace {
struct ProfRec {
  cudaEvent_t a, b;
  std::string cls;
  double work;
};
int g_prof = 0;
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_evpool;

cudaEvent_t take_event() {
  if(g_evpool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = g_evpool.back();
  g_evpool.pop_back();
  return e;
}
}  // namespace

bool prof_on() { return g_prof != 0; }
bool prof_detail() { return g_prof == 2; }

void prof_begin(cudaStream_t st, void** token) {
  cudaEvent_t e = take_event();
  cudaEventRecord(e, st);
  *token = (void*)e;
}

void prof_end(cudaStream_t st, void* token, const std::string& cls, double work) {
  cudaEvent_t e = take_event();
  cudaEventRecord(e, st);
  g_recs.push_back(ProfRec{(cudaEvent_t)token, e, cls, work});
}

}  // namespace mtkc

using namespace mtkc;

extern "C" {

const char* mtkc_last_error(void) { return t_err.c_str(); }

uint64_t mtkc_launch_count(void) { return g_launches.load(); }
uint64_t mtkc_h2d_bytes(void) { return g_h2d.load(); }
uint64_t mtkc_d2h_bytes(void) { return g_d2h.load(); }

__global__ void sleep_kernel(int64_t ns) {
  MTKC_PDL_ENTRY();
  int64_t t0 = (int64_t)clock64();
  (void)t0;
  uint64_t start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  for(;;) {
    uint64_t now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if((int64_t)(now - start) >= ns)
      break;
    __nanosleep(10000);
  }
}

int mtkc_gpu_sleep(int64_t us, void* stream) {
  ::mtkc::launch(sleep_kernel, 1, 1, 0, S(stream), us * 1000);
  return cuda_status(cudaGetLastError(), "sleep_kernel");
}

int mtkc_prof_enable(int on) {
  g_prof = on;
  return MTKC_OK;
}

int mtkc_prof_report(char* buf, size_t len) {
  cudaError_t e = cudaDeviceSynchronize();
  if(e != cudaSuccess)
    return cuda_status(e, "mtkc_prof_report");
  struct Acc {
    int64_t n = 0;
    double ms = 0, work = 0;
  };
  std::vector<std::pair<std::string, Acc>> acc;
  for(auto& r : g_recs) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto it = std::find_if(acc.begin(), acc.end(), [&](auto& p) { return p.first == r.cls; });
    if(it == acc.end()) {
      acc.push_back({r.cls, Acc{}});
      it = acc.end() - 1;
    }
    it->second.n += 1;
    it->second.ms += ms;
    it->second.work += r.work;
    g_evpool.push_back(r.a);
    g_evpool.push_back(r.b);
  }
  g_recs.clear();
  std::string out;
  char line[256];
  for(auto& [k, a] : acc) {
    snprintf(line, sizeof(line), "%s %lld %.6f %.6e\n", k.c_str(), (long long)a.n, a.ms, a.work);
    out += line;
  }
  if(buf && len) {
    size_t n = std::min(len - 1, out.size());
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return MTKC_OK;
}

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
  BlockTimer bt("cudaMalloc");
  return cuda_status(cudaMalloc(ptr, bytes), "cudaMalloc");
}

int mtkc_free(void* ptr) {
  BlockTimer bt("cudaFree");
  return cuda_status(cudaFree(ptr), "cudaFree");
}

int mtkc_host_alloc_pinned(void** ptr, size_t bytes) {
  return cuda_status(cudaMallocHost(ptr, bytes), "cudaMallocHost");
}

int mtkc_host_free_pinned(void* ptr) { return cuda_status(cudaFreeHost(ptr), "cudaFreeHost"); }

int mtkc_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  g_h2d.fetch_add(bytes, std::memory_order_relaxed);
  BlockTimer bt("memcpy_h2d");
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(stream)),
                     "cudaMemcpyAsync(H2D)");
}

int mtkc_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  g_d2h.fetch_add(bytes, std::memory_order_relaxed);
  BlockTimer bt("memcpy_d2h");
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S(stream)),
                     "cudaMemcpyAsync(D2H)");
}

// Copies and fills as kernels: a copy-engine operation in the stream ends
// the programmatic-dependent-launch chain (the DMA waits for the previous
// kernel to drain, the next kernel cannot start before the DMA is done), a
// few microseconds of idle device per copy; a kernel overlaps its neighbours
// like every other launch.  MTK_COPY_ENGINE=1 restores cudaMemcpyAsync /
// cudaMemsetAsync.
static bool copy_engine() {
  static const bool e = getenv("MTK_COPY_ENGINE") && getenv("MTK_COPY_ENGINE")[0] == '1';
  return e;
}

static int copy_kernel_launch(void* dst, const void* src, size_t bytes, bool hostSrc, cudaStream_t st) {
  const uintptr_t al = (uintptr_t)dst | (uintptr_t)src | (uintptr_t)bytes;
  const int vec = (al & 15) == 0 ? 16 : ((al & 3) == 0 ? 4 : 1);
  const size_t n = bytes / (size_t)vec;
  // host sources: every element in registers before the wait (one pass)
  const size_t perCta = 256 * (size_t)COPY_U;
  const unsigned grid = (unsigned)std::min<size_t>((n + perCta - 1) / perCta,
                                                   hostSrc ? 65535 : 148 * 8);
  cudaError_t e;
  if(vec == 16)
    e = launch(copy_kernel<uint4>, dim3(grid), dim3(256), 0, st, (uint4*)dst, (const uint4*)src,
               n, hostSrc ? 1 : 0);
  else if(vec == 4)
    e = launch(copy_kernel<uint32_t>, dim3(grid), dim3(256), 0, st, (uint32_t*)dst,
               (const uint32_t*)src, n, hostSrc ? 1 : 0);
  else
    e = launch(copy_kernel<uint8_t>, dim3(grid), dim3(256), 0, st, (uint8_t*)dst,
               (const uint8_t*)src, n, hostSrc ? 1 : 0);
  count_launch();
  return cuda_status(e, "copy_kernel");
}

int mtkc_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  if(copy_engine())
    return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream)),
                       "cudaMemcpyAsync(D2D)");
  return copy_kernel_launch(dst, src, bytes, false, S(stream));
}

int mtkc_upload_pinned(void* dst, const void* pinned_src, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  g_h2d.fetch_add(bytes, std::memory_order_relaxed);
  if(copy_engine() || bytes > ((size_t)64 << 20))
    return cuda_status(cudaMemcpyAsync(dst, pinned_src, bytes, cudaMemcpyHostToDevice, S(stream)),
                       "cudaMemcpyAsync(H2D)");
  return copy_kernel_launch(dst, pinned_src, bytes, true, S(stream));
}

int mtkc_memset(void* dst, int value, size_t bytes, void* stream) {
  if(!bytes)
    return MTKC_OK;
  if(copy_engine())
    return cuda_status(cudaMemsetAsync(dst, value, bytes, S(stream)), "cudaMemsetAsync");
  const uint32_t b = (uint32_t)value & 0xffu;
  const uint32_t w = b | (b << 8) | (b << 16) | (b << 24);
  const uintptr_t al = (uintptr_t)dst | (uintptr_t)bytes;
  const int vec = (al & 15) == 0 ? 16 : ((al & 3) == 0 ? 4 : 1);
  const size_t n = bytes / (size_t)vec;
  const unsigned grid = (unsigned)std::min<size_t>((n + 256 * 4 - 1) / (256 * 4), 148 * 8);
  cudaError_t e;
  if(vec == 16)
    e = launch(fill_kernel<uint4>, dim3(grid), dim3(256), 0, S(stream), (uint4*)dst, n,
               make_uint4(w, w, w, w));
  else if(vec == 4)
    e = launch(fill_kernel<uint32_t>, dim3(grid), dim3(256), 0, S(stream), (uint32_t*)dst, n, w);
  else
    e = launch(fill_kernel<uint8_t>, dim3(grid), dim3(256), 0, S(stream), (uint8_t*)dst, n,
               (uint8_t)b);
  count_launch();
  return cuda_status(e, "fill_kernel");
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
  BlockTimer bt("stream_sync");
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

int mtkc_event_sync(void* ev) {
  BlockTimer bt("event_sync");
  return cuda_status(cudaEventSynchronize((cudaEvent_t)ev), "cudaEventSynchronize");
}

int mtkc_event_elapsed_ms(void* start, void* stop, float* ms) {
  return cuda_status(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop),
                     "cudaEventElapsedTime");
}

int mtkc_device_sync(void) { return cuda_status(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

}  // extern "C"
