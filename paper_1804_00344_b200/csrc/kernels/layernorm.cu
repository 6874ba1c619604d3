// Layer normalisation over the last axis: layerNormInto / layerNormBackward
// (tensor.cpp:545-599), graph layerNorm (graph.cpp:563-591).
//
// Forward: one warp per row, the row held in registers (d <= 1024) or
// re-read from L1 (larger d).  Two-pass statistics exactly like the
// reference: mu = sum(x)/d, var = sum((x-mu)^2)/d, rs = 1/sqrt(var + eps);
// caches invStd [rows] and xhat [rows x d] for the backward.
// Backward: one warp per row for dx; dgain/dbias are reduced over rows in a
// fixed order (per-CTA partials, then a column pass) so results are bitwise
// reproducible run to run.
#include "common.cuh"

using namespace mtkc;

namespace {

constexpr int LN_WARPS = 8;
constexpr int LN_ROWS_PER_CTA = 64;

template <int V>
__global__ void __launch_bounds__(LN_WARPS * 32)
    ln_fwd_kernel(float* out, const float* x, const float* g, const float* b, float eps,
                  float* invStd, float* xhat, int64_t rows, int64_t d) {
  int64_t row = blockIdx.x * (int64_t)LN_WARPS + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if(row >= rows)
    return;
  const float* xr = x + row * d;
  float v[V > 0 ? V : 1];
  float s = 0.f;
  if constexpr(V > 0) {
#pragma unroll
    for(int k = 0; k < V; ++k) {
      int64_t j = lane + 32 * k;
      v[k] = j < d ? xr[j] : 0.f;
      s += v[k];
    }
  } else {
    for(int64_t j = lane; j < d; j += 32)
      s += xr[j];
  }
  s = warp_sum(s);
  float mu = s / (float)d;
  float q = 0.f;
  if constexpr(V > 0) {
#pragma unroll
    for(int k = 0; k < V; ++k) {
      int64_t j = lane + 32 * k;
      if(j < d) {
        float c = v[k] - mu;
        q += c * c;
      }
    }
  } else {
    for(int64_t j = lane; j < d; j += 32) {
      float c = xr[j] - mu;
      q += c * c;
    }
  }
  q = warp_sum(q);
  float var = q / (float)d;
  float rs = 1.f / sqrtf(var + eps);
  if(lane == 0)
    invStd[row] = rs;
  float* xh = xhat + row * d;
  float* o = out + row * d;
  if constexpr(V > 0) {
#pragma unroll
    for(int k = 0; k < V; ++k) {
      int64_t j = lane + 32 * k;
      if(j < d) {
        float h = (v[k] - mu) * rs;
        xh[j] = h;
        o[j] = g[j] * h + b[j];
      }
    }
  } else {
    for(int64_t j = lane; j < d; j += 32) {
      float h = (xr[j] - mu) * rs;
      xh[j] = h;
      o[j] = g[j] * h + b[j];
    }
  }
}

// dx (+)= rs*(dxh - mean(dxh) - xhat*mean(dxh*xhat)), dxh = dy*g.
// Per-CTA column partials of dy*xhat and dy go to part[blockIdx][2][d].
__global__ void __launch_bounds__(LN_WARPS * 32)
    ln_bwd_kernel(const float* dy, const float* g, const float* invStd, const float* xhat,
                  float* dx, float* part, int64_t rows, int64_t d, int accDx) {
  extern __shared__ float sm[];  // [LN_WARPS][2][d] when part != nullptr
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t r0 = (int64_t)blockIdx.x * LN_ROWS_PER_CTA;
  int64_t r1 = min(rows, r0 + LN_ROWS_PER_CTA);
  float* myG = part ? sm + (size_t)w * 2 * d : nullptr;
  float* myB = part ? myG + d : nullptr;
  if(part)
    for(int64_t j = lane; j < d; j += 32) {
      myG[j] = 0.f;
      myB[j] = 0.f;
    }
  for(int64_t row = r0 + w; row < r1; row += LN_WARPS) {
    const float* dyr = dy + row * d;
    const float* xr = xhat + row * d;
    float s1 = 0.f, s2 = 0.f;
    for(int64_t j = lane; j < d; j += 32) {
      float h = dyr[j] * g[j];
      s1 += h;
      s2 += h * xr[j];
      if(part) {
        myG[j] += dyr[j] * xr[j];
        myB[j] += dyr[j];
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    float m1 = s1 / (float)d, m2 = s2 / (float)d;
    float rs = invStd[row];
    float* dxr = dx + row * d;
    for(int64_t j = lane; j < d; j += 32) {
      float h = dyr[j] * g[j];
      float val = rs * (h - m1 - xr[j] * m2);
      dxr[j] = accDx ? dxr[j] + val : val;
    }
  }
  if(!part)
    return;
  __syncthreads();
  float* dst = part + (int64_t)blockIdx.x * 2 * d;
  for(int64_t j = threadIdx.x; j < 2 * d; j += blockDim.x) {
    float acc = 0.f;
    for(int k = 0; k < LN_WARPS; ++k)
      acc += sm[(size_t)k * 2 * d + j];
    dst[j] = acc;
  }
}

__global__ void ln_param_final_kernel(float* dgain, float* dbias, const float* part,
                                      int64_t nparts, int64_t d, int acc) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if(j >= d)
    return;
  float sg = 0.f, sb = 0.f;
  for(int64_t p = 0; p < nparts; ++p) {
    sg += part[p * 2 * d + j];
    sb += part[p * 2 * d + d + j];
  }
  dgain[j] = (acc ? dgain[j] : 0.f) + sg;
  dbias[j] = (acc ? dbias[j] : 0.f) + sb;
}

// no-workspace fallback: one thread per column over all rows
__global__ void ln_param_direct_kernel(const float* dy, const float* xhat, float* dgain,
                                       float* dbias, int64_t rows, int64_t d, int acc) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if(j >= d)
    return;
  float sg = 0.f, sb = 0.f;
  for(int64_t r = 0; r < rows; ++r) {
    sg += dy[r * d + j] * xhat[r * d + j];
    sb += dy[r * d + j];
  }
  dgain[j] = (acc ? dgain[j] : 0.f) + sg;
  dbias[j] = (acc ? dbias[j] : 0.f) + sb;
}

}  // namespace

extern "C" {

int mtkc_layernorm(float* out, const float* x, const float* gain, const float* bias,
                   float eps, float* inv_std, float* xhat, int64_t rows, int64_t d,
                   void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  if(d < 2)
    return fail(MTKC_DIMENSION, "layer norm needs last extent >= 2");
  unsigned grid = (unsigned)cdiv(rows, LN_WARPS);
  cudaStream_t st = S(stream);
  ProfScope prof(st, "layernorm", 8.0 * rows * d);  // read x, write y
  int v = (int)cdiv(d, 32);
  if(v <= 1)
    ln_fwd_kernel<1><<<grid, LN_WARPS * 32, 0, st>>>(out, x, gain, bias, eps, inv_std, xhat, rows, d);
  else if(v <= 2)
    ln_fwd_kernel<2><<<grid, LN_WARPS * 32, 0, st>>>(out, x, gain, bias, eps, inv_std, xhat, rows, d);
  else if(v <= 4)
    ln_fwd_kernel<4><<<grid, LN_WARPS * 32, 0, st>>>(out, x, gain, bias, eps, inv_std, xhat, rows, d);
  else if(v <= 8)
    ln_fwd_kernel<8><<<grid, LN_WARPS * 32, 0, st>>>(out, x, gain, bias, eps, inv_std, xhat, rows, d);
  else if(v <= 16)
    ln_fwd_kernel<16><<<grid, LN_WARPS * 32, 0, st>>>(out, x, gain, bias, eps, inv_std, xhat, rows, d);
  else if(v <= 32)
    ln_fwd_kernel<32><<<grid, LN_WARPS * 32, 0, st>>>(out, x, gain, bias, eps, inv_std, xhat, rows, d);
  else
    ln_fwd_kernel<0><<<grid, LN_WARPS * 32, 0, st>>>(out, x, gain, bias, eps, inv_std, xhat, rows, d);
  MTKC_POST_LAUNCH("ln_fwd_kernel");
  return MTKC_OK;
}

int mtkc_layernorm_backward(const float* dy, const float* gain, const float* inv_std,
                            const float* xhat, float* dx, float* dgain, float* dbias,
                            int64_t rows, int64_t d, int accumulate_dx, int accumulate_params,
                            float* workspace, size_t workspace_bytes, void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  cudaStream_t st = S(stream);
  ProfScope prof(st, "layernorm", 12.0 * rows * d);  // read dy, xhat; write dx
  int64_t nparts = cdiv(rows, LN_ROWS_PER_CTA);
  size_t smem = (size_t)LN_WARPS * 2 * (size_t)d * sizeof(float);
  bool usePart = dgain && workspace &&
                 workspace_bytes >= (size_t)nparts * 2 * (size_t)d * sizeof(float) &&
                 smem <= 200 * 1024;
  if(usePart && smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ln_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if(e != cudaSuccess)
      return cuda_status(e, "ln_bwd_kernel smem attribute");
  }
  ln_bwd_kernel<<<(unsigned)nparts, LN_WARPS * 32, usePart ? smem : 0, st>>>(
      dy, gain, inv_std, xhat, dx, usePart ? workspace : nullptr, rows, d, accumulate_dx);
  MTKC_POST_LAUNCH("ln_bwd_kernel");
  if(!dgain)
    return MTKC_OK;
  if(usePart) {
    ln_param_final_kernel<<<(unsigned)cdiv(d, 128), 128, 0, st>>>(dgain, dbias, workspace, nparts,
                                                                  d, accumulate_params);
    MTKC_POST_LAUNCH("ln_param_final_kernel");
  } else {
    ln_param_direct_kernel<<<(unsigned)cdiv(d, 128), 128, 0, st>>>(dy, xhat, dgain, dbias, rows,
                                                                   d, accumulate_params);
    MTKC_POST_LAUNCH("ln_param_direct_kernel");
  }
  return MTKC_OK;
}

}  // extern "C"
