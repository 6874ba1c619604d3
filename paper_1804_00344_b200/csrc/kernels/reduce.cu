// Reductions: reduceInto (tensor.cpp:322-368) and its graph backward
// (graph.cpp:488-521); deterministic column sums for bias/gain gradients;
// the allFinite scan (tensor.cpp:95-100) as a device flag.
#include "colred.cuh"
#include "common.cuh"

using namespace mtkc;

namespace {

__global__ void reduce_kernel(int op, float* out, const float* in, int64_t outer, int64_t n,
                              int64_t inner) {
  int64_t total = outer * inner;
  for(int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
      t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = t / inner, c = t % inner;
    const float* base = in + a * n * inner + c;
    float acc;
    if(op == MTKC_RSUM || op == MTKC_RMEAN) {
      acc = 0.f;
      for(int64_t i = 0; i < n; ++i)
        acc += base[i * inner];
      if(op == MTKC_RMEAN)
        acc /= (float)n;
    } else if(op == MTKC_RMAX) {
      acc = base[0];
      for(int64_t i = 1; i < n; ++i)
        acc = fmaxf(acc, base[i * inner]);
    } else {
      float best = base[0];
      int64_t arg = 0;
      for(int64_t i = 1; i < n; ++i)
        if(base[i * inner] > best) {  // strict: ties keep the lowest index (:357)
          best = base[i * inner];
          arg = i;
        }
      acc = (float)arg;
    }
    out[t] = acc;
  }
}

__global__ void reduce_bwd_kernel(int op, float* gin, const float* gout, const float* in,
                                  int64_t outer, int64_t n, int64_t inner) {
  int64_t total = outer * inner;
  for(int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
      t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = t / inner, c = t % inner;
    float go = gout[t];
    float* base = gin + a * n * inner + c;
    const float* xv = in + a * n * inner + c;
    if(op == MTKC_RSUM) {
      for(int64_t i = 0; i < n; ++i)
        base[i * inner] += go;
    } else if(op == MTKC_RMEAN) {
      float v = go / (float)n;
      for(int64_t i = 0; i < n; ++i)
        base[i * inner] += v;
    } else if(op == MTKC_RMAX) {
      int64_t best = 0;
      for(int64_t i = 1; i < n; ++i)
        if(xv[i * inner] > xv[best * inner])
          best = i;
      base[best * inner] += go;
    }
  }
}

constexpr int CS_ROWS = 128;  // below this many rows a single pass is used

// single-level variant (no workspace): one thread per column walks all rows
__global__ void colsum_direct_kernel(float* out, const float* in, int64_t rows, int64_t cols,
                                     int accumulate) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if(c >= cols)
    return;
  float s = 0.f;
  for(int64_t r = 0; r < rows; ++r)
    s += in[r * cols + c];
  out[c] = (accumulate ? out[c] : 0.f) + s;
}

__global__ void finite_kernel(const float* in, int64_t n, int* flags) {
  bool bad = false;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(in[i]);
  if(__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(flags, MTKC_FLAG_NONFINITE);
}

__global__ void finite4_kernel(const float4* in, int64_t n4, int* flags) {
  bool bad = false;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
      i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = in[i];
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
  }
  if(__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(flags, MTKC_FLAG_NONFINITE);
}

}  // namespace

extern "C" {

int mtkc_reduce(int op, float* out, const float* in, int64_t outer, int64_t n, int64_t inner,
                void* stream) {
  if(outer * inner <= 0 || n <= 0)
    return MTKC_OK;
  reduce_kernel<<<grid1d(outer * inner, 128), 128, 0, S(stream)>>>(op, out, in, outer, n, inner);
  MTKC_POST_LAUNCH("reduce_kernel");
  return MTKC_OK;
}

int mtkc_reduce_backward(int op, float* gin, const float* gout, const float* in,
                         int64_t outer, int64_t n, int64_t inner, void* stream) {
  if(op == MTKC_RARGMAX || outer * inner <= 0)
    return MTKC_OK;
  reduce_bwd_kernel<<<grid1d(outer * inner, 128), 128, 0, S(stream)>>>(op, gin, gout, in, outer,
                                                                       n, inner);
  MTKC_POST_LAUNCH("reduce_bwd_kernel");
  return MTKC_OK;
}

int mtkc_colsum(float* out, const float* in, int64_t rows, int64_t cols, int accumulate,
                float* workspace, size_t workspace_bytes, void* stream) {
  if(rows <= 0 || cols <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "colsum", 4.0 * rows * cols);
  if(rows <= CS_ROWS || !workspace || workspace_bytes < colred_workspace_bytes(1, rows, cols)) {
    colsum_direct_kernel<<<(unsigned)cdiv(cols, 128), 128, 0, S(stream)>>>(out, in, rows, cols,
                                                                          accumulate);
    MTKC_POST_LAUNCH("colsum_direct_kernel");
    return MTKC_OK;
  }
  int64_t nblk = cdiv(rows, CR_ROWS);
  colred_partial_kernel<1><<<dim3((unsigned)cdiv(cols, CR_COLS), (unsigned)nblk), 256, 0,
                             S(stream)>>>(workspace, in, nullptr, rows, cols);
  MTKC_POST_LAUNCH("colred_partial_kernel");
  colred_final_kernel<1><<<colred_final_grid(cols), 256, 0, S(stream)>>>(
      out, nullptr, workspace, nblk, cols, accumulate);
  MTKC_POST_LAUNCH("colred_final_kernel");
  return MTKC_OK;
}

int mtkc_check_finite(const float* in, int64_t n, int* flags, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  if(n % 4 == 0 && (uintptr_t)in % 16 == 0)
    finite4_kernel<<<grid1d(n / 4, 256, 148 * 8), 256, 0, S(stream)>>>((const float4*)in, n / 4,
                                                                      flags);
  else
    finite_kernel<<<grid1d(n, 256, 148 * 8), 256, 0, S(stream)>>>(in, n, flags);
  MTKC_POST_LAUNCH("finite_kernel");
  return MTKC_OK;
}

}  // extern "C"
