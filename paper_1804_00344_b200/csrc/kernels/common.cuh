// Shared helpers for the libmtkcuda.so kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "mtk_cuda.h"

namespace mtkc {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* where);
void count_launch(int n = 1);

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Event-bracketed profiling of one C-ABI call (mtkc_prof_enable).
bool prof_on();
bool prof_detail();  // mtkc_prof_enable(2): classes carry the call's shape
void prof_begin(cudaStream_t st, void** token);
void prof_end(cudaStream_t st, void* token, const std::string& cls, double work);
struct ProfScope {
  cudaStream_t st;
  void* tok = nullptr;
  const char* cls;
  double work;
  std::string detail;  // appended to the class name in detail mode
  ProfScope(cudaStream_t s, const char* c, double w) : st(s), cls(c), work(w) {
    if(prof_on())
      prof_begin(st, &tok);
  }
  ~ProfScope() {
    if(tok)
      prof_end(st, tok, detail.empty() ? std::string(cls) : std::string(cls) + ":" + detail,
               work);
  }
};

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every kernel is launched with
// programmatic stream serialisation, so its CTAs may be scheduled while the
// previous kernel on the stream is still draining (its launch latency and
// prologue overlap the predecessor's tail).  Correctness: every kernel
// executes MTKC_PDL_ENTRY() -- griddepcontrol.wait, which blocks until the
// preceding grid has completed and its memory is visible -- before touching
// any global memory, and only then lets its own dependents launch
// (griddepcontrol.launch_dependents), so at most one grid waits ahead.
// MTK_NO_PDL=1 launches without the attribute (plain stream order).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#define MTKC_PDL_ENTRY()     \
  do {                       \
    ::mtkc::pdl_wait();      \
    ::mtkc::pdl_trigger();   \
  } while(0)

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Same, as clusters of `cluster_x` CTAs along x (CTA pairs of the GEMM).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t st, unsigned cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Launch check used after every launch: counts the launch and converts a
// launch failure into MTKC_CUDA with the kernel name.
#define MTKC_POST_LAUNCH(name)                                  \
  do {                                                          \
    ::mtkc::count_launch();                                     \
    cudaError_t _e = cudaGetLastError();                        \
    if(_e != cudaSuccess) return ::mtkc::cuda_status(_e, name); \
  } while(0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline unsigned grid1d(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = cdiv(n, threads);
  if(g > cap)
    g = cap;
  if(g < 1)
    g = 1;
  return (unsigned)g;
}

// Right-aligned 4-d strides of a broadcast operand (tensor.cpp:120-130).
struct Bcast4 {
  int64_t s[4];
};

inline Bcast4 bcast_strides(const int64_t d[4]) {
  Bcast4 b;
  int64_t run = 1;
  for(int i = 3; i >= 0; --i) {
    b.s[i] = d[i] == 1 ? 0 : run;
    run *= d[i];
  }
  return b;
}

struct Dims4 {
  int64_t d[4];
};

inline Dims4 dims4(const int64_t d[4]) {
  Dims4 r;
  for(int i = 0; i < 4; ++i)
    r.d[i] = d[i];
  return r;
}

}  // namespace mtkc

// ---------------------------------------------------------------- device

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for(int o = 16; o > 0; o >>= 1)
    v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for(int o = 16; o > 0; o >>= 1)
    v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `red` must hold >= 32 floats. All threads get the result.
__device__ __forceinline__ float block_sum(float v, float* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if(lane == 0)
    red[w] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : 0.f;
  t = warp_sum(t);
  return t;
}

__device__ __forceinline__ float block_max(float v, float* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if(lane == 0)
    red[w] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : -INFINITY;
  t = warp_max(t);
  return t;
}

// Reference elementwise semantics (tensor.cpp:140-158).
__device__ __forceinline__ float apply_unary(int op, float x) {
  switch(op) {
    case MTKC_TANH: return tanhf(x);
    case MTKC_SIGMOID: return 1.f / (1.f + expf(-x));
    case MTKC_RELU: return x > 0.f ? x : 0.f;
    case MTKC_EXP: return expf(x);
    case MTKC_LOG: return logf(x);
    case MTKC_NEG: return -x;
    default: return x;
  }
}

__device__ __forceinline__ float apply_binary(int op, float x, float y) {
  switch(op) {
    case MTKC_ADD: return x + y;
    case MTKC_SUB: return x - y;
    case MTKC_MUL: return x * y;
    case MTKC_DIV: return x / y;
    default: return x;
  }
}
