// Layer normalisation over the last axis: layerNormInto / layerNormBackward
// (tensor.cpp:545-599), graph layerNorm (graph.cpp:563-591).
//
// Forward: one warp per row, the row held in registers (d <= 1024) or
// re-read from L1 (larger d).  Two-pass statistics exactly like the
// reference: mu = sum(x)/d, var = sum((x-mu)^2)/d, rs = 1/sqrt(var + eps);
// caches invStd [rows] and xhat [rows x d] for the backward.
// Backward: one warp per row for dx (row in registers, one read of dy and
// xhat); dgain/dbias are column reductions over rows in a fixed order
// (colred.cuh) so results are bitwise reproducible run to run.
#include "colred.cuh"
#include "common.cuh"

using namespace mtkc;

namespace {

constexpr int LN_WARPS = 8;

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

// dx (+)= rs*(dxh - mean(dxh) - xhat*mean(dxh*xhat)), dxh = dy*g
template <int V>
__global__ void __launch_bounds__(LN_WARPS * 32)
    ln_bwd_dx_kernel(const float* dy, const float* g, const float* invStd, const float* xhat,
                     float* dx, int64_t rows, int64_t d, int accDx) {
  int64_t row = blockIdx.x * (int64_t)LN_WARPS + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if(row >= rows)
    return;
  const float* dyr = dy + row * d;
  const float* xr = xhat + row * d;
  float* dxr = dx + row * d;
  float s1 = 0.f, s2 = 0.f;
  if constexpr(V > 0) {
    float h[V], xv[V];
#pragma unroll
    for(int k = 0; k < V; ++k) {
      int64_t j = lane + 32 * k;
      h[k] = j < d ? dyr[j] * g[j] : 0.f;
      xv[k] = j < d ? xr[j] : 0.f;
      s1 += h[k];
      s2 += h[k] * xv[k];
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    float m1 = s1 / (float)d, m2 = s2 / (float)d;
    float rs = invStd[row];
#pragma unroll
    for(int k = 0; k < V; ++k) {
      int64_t j = lane + 32 * k;
      if(j < d) {
        float val = rs * (h[k] - m1 - xv[k] * m2);
        dxr[j] = accDx ? dxr[j] + val : val;
      }
    }
  } else {
    for(int64_t j = lane; j < d; j += 32) {
      float h = dyr[j] * g[j];
      s1 += h;
      s2 += h * xr[j];
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    float m1 = s1 / (float)d, m2 = s2 / (float)d;
    float rs = invStd[row];
    for(int64_t j = lane; j < d; j += 32) {
      float h = dyr[j] * g[j];
      float val = rs * (h - m1 - xr[j] * m2);
      dxr[j] = accDx ? dxr[j] + val : val;
    }
  }
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

template <template <int> class K, typename... Args>
void launch_v(int64_t d, dim3 grid, cudaStream_t st, Args... args);

#define LN_DISPATCH(KERNEL, ...)                                             \
  do {                                                                       \
    int v_ = (int)cdiv(d, 32);                                               \
    if(v_ <= 1)                                                              \
      KERNEL<1><<<grid, LN_WARPS * 32, 0, st>>>(__VA_ARGS__);                \
    else if(v_ <= 2)                                                         \
      KERNEL<2><<<grid, LN_WARPS * 32, 0, st>>>(__VA_ARGS__);                \
    else if(v_ <= 4)                                                         \
      KERNEL<4><<<grid, LN_WARPS * 32, 0, st>>>(__VA_ARGS__);                \
    else if(v_ <= 8)                                                         \
      KERNEL<8><<<grid, LN_WARPS * 32, 0, st>>>(__VA_ARGS__);                \
    else if(v_ <= 16)                                                        \
      KERNEL<16><<<grid, LN_WARPS * 32, 0, st>>>(__VA_ARGS__);               \
    else if(v_ <= 32)                                                        \
      KERNEL<32><<<grid, LN_WARPS * 32, 0, st>>>(__VA_ARGS__);               \
    else                                                                     \
      KERNEL<0><<<grid, LN_WARPS * 32, 0, st>>>(__VA_ARGS__);                \
  } while(0)

}  // namespace

extern "C" {

int mtkc_layernorm(float* out, const float* x, const float* gain, const float* bias,
                   float eps, float* inv_std, float* xhat, int64_t rows, int64_t d,
                   void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  if(d < 2)
    return fail(MTKC_DIMENSION, "layer norm needs last extent >= 2");
  dim3 grid((unsigned)cdiv(rows, LN_WARPS));
  cudaStream_t st = S(stream);
  ProfScope prof(st, "layernorm", 8.0 * rows * d);  // read x, write y
  LN_DISPATCH(ln_fwd_kernel, out, x, gain, bias, eps, inv_std, xhat, rows, d);
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
  dim3 grid((unsigned)cdiv(rows, LN_WARPS));
  LN_DISPATCH(ln_bwd_dx_kernel, dy, gain, inv_std, xhat, dx, rows, d, accumulate_dx);
  MTKC_POST_LAUNCH("ln_bwd_dx_kernel");
  if(!dgain)
    return MTKC_OK;
  if(workspace && workspace_bytes >= colred_workspace_bytes(2, rows, d)) {
    int64_t nblk = cdiv(rows, CR_ROWS);
    colred_partial_kernel<2><<<dim3((unsigned)cdiv(d, CR_COLS), (unsigned)nblk), 256, 0, st>>>(
        workspace, dy, xhat, rows, d);
    MTKC_POST_LAUNCH("colred_partial_kernel");
    colred_final_kernel<2><<<colred_final_grid(d), 256, 0, st>>>(dgain, dbias, workspace, nblk,
                                                                  d, accumulate_params);
    MTKC_POST_LAUNCH("colred_final_kernel");
  } else {
    ln_param_direct_kernel<<<(unsigned)cdiv(d, 128), 128, 0, st>>>(dy, xhat, dgain, dbias, rows,
                                                                   d, accumulate_params);
    MTKC_POST_LAUNCH("ln_param_direct_kernel");
  }
  return MTKC_OK;
}

}  // extern "C"
