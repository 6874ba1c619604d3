// Fused LSTM cell pointwise kernels (BASELINE.json north_star: "the fused
// GRU/LSTM cell ops").  The reference has no LSTM; the
// cell is pinned against the reference's own primitives composed in the
// same order (tests/test_lstm_gpu.py: dot, add, slice, sigmoid, tanh, mul,
// concat on the reference ExpressionGraph), like the reference pins its
// fused GRU against an unfused composition (tests/gradsuite.h:304-320).
//
//   pre = h*U, then + x*W (GEMMs, gruPre's order graph.cpp:636-644), + b
//   [i | f | o | g] = [sig | sig | sig | tanh](pre)   (gate blocks of d)
//   c' = f*c + i*g ;  h' = o*tanh(c')               out = [h' | c']
// One warp-strided thread per (row, column); the row's 4 gates and the
// cell state stay in registers; the backward recomputes nothing but
// tanh(c') from the cache.
#include "common.cuh"

using namespace mtkc;

namespace {

__device__ __forceinline__ float sigm(float a) { return 1.f / (1.f + expf(-a)); }

__global__ void lstm_fwd_kernel(const float* __restrict__ pre, const float* __restrict__ bias,
                                const float* __restrict__ c, float* __restrict__ out,
                                float* __restrict__ cache, int64_t b, int64_t d) {
  MTKC_PDL_ENTRY();
  const int64_t n = b * d;
  for(int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
      idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / d, j = idx - r * d;
    const float* p = pre + r * 4 * d;
    const float i = sigm(p[j] + bias[j]);
    const float f = sigm(p[d + j] + bias[d + j]);
    const float o = sigm(p[2 * d + j] + bias[2 * d + j]);
    const float g = tanhf(p[3 * d + j] + bias[3 * d + j]);
    const float cn = f * c[idx] + i * g;
    const float tc = tanhf(cn);
    out[r * 2 * d + j] = o * tc;
    out[r * 2 * d + d + j] = cn;
    float* k = cache + r * 5 * d;
    k[j] = i;
    k[d + j] = f;
    k[2 * d + j] = o;
    k[3 * d + j] = g;
    k[4 * d + j] = tc;
  }
}

// gout = [dh' | dc'] ; dpre (written) ; dc (+)= dc'_total * f
__global__ void lstm_bwd_kernel(const float* __restrict__ gout, const float* __restrict__ cache,
                                const float* __restrict__ c, float* __restrict__ dpre,
                                float* __restrict__ dc, int accC, int64_t b, int64_t d) {
  MTKC_PDL_ENTRY();
  const int64_t n = b * d;
  for(int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
      idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / d, j = idx - r * d;
    const float* k = cache + r * 5 * d;
    const float i = k[j], f = k[d + j], o = k[2 * d + j], g = k[3 * d + j], tc = k[4 * d + j];
    const float dh = gout[r * 2 * d + j];
    const float dcn = gout[r * 2 * d + d + j] + dh * o * (1.f - tc * tc);
    const float dO = dh * tc;
    const float dI = dcn * g, dF = dcn * c[idx], dG = dcn * i;
    float* q = dpre + r * 4 * d;
    q[j] = dI * i * (1.f - i);
    q[d + j] = dF * f * (1.f - f);
    q[2 * d + j] = dO * o * (1.f - o);
    q[3 * d + j] = dG * (1.f - g * g);
    if(dc) {
      const float v = dcn * f;
      dc[idx] = accC ? dc[idx] + v : v;
    }
  }
}

}  // namespace

extern "C" {

int mtkc_lstm_forward(const float* pre, const float* bias, const float* c, float* out,
                      float* cache, int64_t b, int64_t d, void* stream) {
  if(b * d <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "lstm", 4.0 * b * d * 12);
  ::mtkc::launch(lstm_fwd_kernel, grid1d(b * d, 256), 256, 0, S(stream), pre, bias, c, out,
                 cache, b, d);
  MTKC_POST_LAUNCH("lstm_fwd_kernel");
  return MTKC_OK;
}

int mtkc_lstm_backward(const float* gout, const float* cache, const float* c, float* dpre,
                       float* dc, int accumulate_c, int64_t b, int64_t d, void* stream) {
  if(b * d <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "lstm", 4.0 * b * d * 14);
  ::mtkc::launch(lstm_bwd_kernel, grid1d(b * d, 256), 256, 0, S(stream), gout, cache, c, dpre,
                 dc, accumulate_c, b, d);
  MTKC_POST_LAUNCH("lstm_bwd_kernel");
  return MTKC_OK;
}

}  // extern "C"
