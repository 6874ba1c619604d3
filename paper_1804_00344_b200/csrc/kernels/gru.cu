// Fused GRU block pointwise kernels (gruCell graph.cpp:648-813).  One CTA
// per batch row; the row's three gates (and their optional layer norms, with
// block-wide two-pass statistics like layerNormInto) stay in registers.
// The h*U / x*W products are tcgen05 GEMMs issued by the host op.
#include "common.cuh"

using namespace mtkc;

namespace {

constexpr int GT = 256;  // threads per row
constexpr int GV = 8;    // max elements per thread (d <= 2048)

// block-wide sums of NQ values (all threads receive the totals)
template <int NQ>
__device__ __forceinline__ void block_sums(float (&v)[NQ], float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for(int q = 0; q < NQ; ++q)
    v[q] = warp_sum(v[q]);
  __syncthreads();
  if(lane == 0)
#pragma unroll
    for(int q = 0; q < NQ; ++q)
      red[q * 32 + w] = v[q];
  __syncthreads();
#pragma unroll
  for(int q = 0; q < NQ; ++q) {
    float t = lane < nw ? red[q * 32 + lane] : 0.f;
    v[q] = warp_sum(t);
  }
}

__device__ __forceinline__ float sigm(float a) { return 1.f / (1.f + expf(-a)); }

__global__ void __launch_bounds__(GT) gru_fwd_kernel(mtkc_gru_args p) {
  MTKC_PDL_ENTRY();
  __shared__ float red[6 * 32];
  const int64_t r = blockIdx.x, d = p.d;
  const bool hasX = p.xw != nullptr, ln = p.lnGz != nullptr;
  const float* hu = p.hu + r * 3 * d;
  const float* xw = hasX ? p.xw + r * 3 * d : nullptr;
  float az[GV], ar[GV], ax[GV];
#pragma unroll
  for(int n = 0; n < GV; ++n)
    az[n] = ar[n] = ax[n] = 0.f;
#pragma unroll
  for(int n = 0; n < GV; ++n) {
    const int64_t j = threadIdx.x + (int64_t)n * GT;
    if(j >= d)
      break;
    // gruPre: h*U, then + x*W, then + b (graph.cpp:636-644)
    float z = hu[j], rr = hu[d + j];
    if(hasX) {
      z = z + xw[j];
      rr = rr + xw[d + j];
    }
    az[n] = z + p.bz[j];
    ar[n] = rr + p.br[j];
    ax[n] = hasX ? xw[2 * d + j] : 0.f;
  }
  float rsz = 0.f, rsr = 0.f, rsx = 0.f;
  if(ln) {  // two-pass statistics per gate (tensor.cpp:545-572)
    float s[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for(int k = 0; k < GV; ++k) {  // entries past d are 0
      s[0] += az[k];
      s[1] += ar[k];
      s[2] += ax[k];
    }
    block_sums<3>(s, red);
    float mz = s[0] / (float)d, mr = s[1] / (float)d, mx = s[2] / (float)d;
    float q[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for(int k = 0; k < GV; ++k) {
      if(threadIdx.x + (int64_t)k * GT >= d)
        break;
      float cz = az[k] - mz, cr = ar[k] - mr, cx = ax[k] - mx;
      q[0] += cz * cz;
      q[1] += cr * cr;
      q[2] += cx * cx;
    }
    block_sums<3>(q, red);
    rsz = 1.f / sqrtf(q[0] / (float)d + p.eps);
    rsr = 1.f / sqrtf(q[1] / (float)d + p.eps);
    rsx = 1.f / sqrtf(q[2] / (float)d + p.eps);
    if(threadIdx.x == 0) {
      p.lnrs[r * 3] = rsz;
      p.lnrs[r * 3 + 1] = rsr;
      p.lnrs[r * 3 + 2] = rsx;
    }
    float* xh = p.lnc + r * 3 * d;
    #pragma unroll
    for(int k = 0; k < GV; ++k) {
      const int64_t j = threadIdx.x + (int64_t)k * GT;
      if(j >= d)
        break;
      float hz = (az[k] - mz) * rsz, hr = (ar[k] - mr) * rsr;
      xh[j] = hz;
      xh[d + j] = hr;
      az[k] = p.lnGz[j] * hz + p.lnBz[j];
      ar[k] = p.lnGr[j] * hr + p.lnBr[j];
      if(hasX) {
        float hx = (ax[k] - mx) * rsx;
        xh[2 * d + j] = hx;
        ax[k] = p.lnGx[j] * hx + p.lnBx[j];
      }
    }
  }
  float* cache = p.cache + r * 3 * d;
  const float* h = p.h + r * d;
  float* ho = p.hout + r * d;
  const bool blend = p.blend_mask != nullptr;
  const float m = blend ? p.blend_mask[r] : 1.f, notm = 1.f - m;
  const float* prev = blend ? p.blend_prev + r * d : nullptr;
  #pragma unroll
  for(int k = 0; k < GV; ++k) {
    const int64_t j = threadIdx.x + (int64_t)k * GT;
    if(j >= d)
      break;
    float z = sigm(az[k]), rr = sigm(ar[k]);
    float ac = ax[k] + (rr * hu[2 * d + j] + p.bh[j]);  // graph.cpp:737-738
    float ht = tanhf(ac);
    cache[j] = z;
    cache[d + j] = rr;
    cache[2 * d + j] = ht;
    float hn = (1.f - z) * ht + z * h[j];
    ho[j] = blend ? hn * m + prev[j] * notm : hn;  // a*m + b*(1-m)
  }
}

// LN backward of one row (tensor.cpp:574-599) given the block sums
__device__ __forceinline__ float ln_dx(float dy, float g, float xh, float rs, float m1,
                                       float m2) {
  return rs * (dy * g - m1 - xh * m2);
}

__global__ void __launch_bounds__(GT) gru_bwd_kernel(mtkc_gru_args p) {
  MTKC_PDL_ENTRY();
  __shared__ float red[6 * 32];
  const int64_t r = blockIdx.x, d = p.d;
  const bool hasX = p.xw != nullptr, ln = p.lnGz != nullptr;
  const float* cache = p.cache + r * 3 * d;
  const float* hu = p.hu + r * 3 * d;
  const float* h = p.h + r * d;
  const float* go = p.go + r * d;
  const bool blend = p.blend_mask != nullptr;
  const float m = blend ? p.blend_mask[r] : 1.f, notm = 1.f - m;
  const bool prevIsH = blend && p.gprev == p.gh;
  float daz[GV], dar[GV], dacv[GV];
#pragma unroll
  for(int n = 0; n < GV; ++n)
    daz[n] = dar[n] = dacv[n] = 0.f;
#pragma unroll
  for(int n = 0; n < GV; ++n) {  // graph.cpp:755-770
    const int64_t j = threadIdx.x + (int64_t)n * GT;
    if(j >= d)
      break;
    float g0 = go[j];
    float g = blend ? g0 * m : g0;  // maskBlend backward (mul by m / 1-m)
    float z = cache[j], rr = cache[d + j], ht = cache[2 * d + j];
    float dz = g * (h[j] - ht);
    float dht = g * (1.f - z);
    float ghv = g * z;
    if(prevIsH) {
      float t = p.accumulate_h ? p.gh[r * d + j] + ghv : ghv;
      p.gh[r * d + j] = t + g0 * notm;
    } else {
      p.gh[r * d + j] = p.accumulate_h ? p.gh[r * d + j] + ghv : ghv;
      if(blend && p.gprev) {
        float gp = g0 * notm;
        p.gprev[r * d + j] = p.accumulate_prev ? p.gprev[r * d + j] + gp : gp;
      }
    }
    float dac = dht * (1.f - ht * ht);
    float dr = dac * hu[2 * d + j];
    p.duh[r * d + j] = dac * rr;
    p.dac[r * d + j] = dac;
    dacv[n] = dac;
    daz[n] = dz * z * (1.f - z);   // graph.cpp:790-792
    dar[n] = dr * rr * (1.f - rr);
  }
  if(!ln) {
    #pragma unroll
    for(int k = 0; k < GV; ++k) {
      const int64_t j = threadIdx.x + (int64_t)k * GT;
      if(j >= d)
        break;
      p.dpz[r * d + j] = daz[k];
      p.dpr[r * d + j] = dar[k];
      if(hasX && p.dax != p.dac)
        p.dax[r * d + j] = dacv[k];
    }
    return;
  }
  const float* xh = p.lnc + r * 3 * d;
  const float rsz = p.lnrs[r * 3], rsr = p.lnrs[r * 3 + 1], rsx = p.lnrs[r * 3 + 2];
  float s[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  #pragma unroll
  for(int k = 0; k < GV; ++k) {
    const int64_t j = threadIdx.x + (int64_t)k * GT;
    if(j >= d)
      break;
    float hz = daz[k] * p.lnGz[j], hr = dar[k] * p.lnGr[j];
    s[0] += hz;
    s[1] += hz * xh[j];
    s[2] += hr;
    s[3] += hr * xh[d + j];
    if(hasX) {
      float hx = dacv[k] * p.lnGx[j];
      s[4] += hx;
      s[5] += hx * xh[2 * d + j];
    }
  }
  block_sums<6>(s, red);
  const float fd = (float)d;
  float* lp = p.lnparts + r * 6 * d;
  #pragma unroll
  for(int k = 0; k < GV; ++k) {
    const int64_t j = threadIdx.x + (int64_t)k * GT;
    if(j >= d)
      break;
    p.dpz[r * d + j] = ln_dx(daz[k], p.lnGz[j], xh[j], rsz, s[0] / fd, s[1] / fd);
    p.dpr[r * d + j] = ln_dx(dar[k], p.lnGr[j], xh[d + j], rsr, s[2] / fd, s[3] / fd);
    lp[j] = daz[k] * xh[j];
    lp[d + j] = daz[k];
    lp[2 * d + j] = dar[k] * xh[d + j];
    lp[3 * d + j] = dar[k];
    if(hasX) {
      p.dax[r * d + j] = ln_dx(dacv[k], p.lnGx[j], xh[2 * d + j], rsx, s[4] / fd, s[5] / fd);
      lp[4 * d + j] = dacv[k] * xh[2 * d + j];
      lp[5 * d + j] = dacv[k];
    }
  }
}

}  // namespace

extern "C" {

int mtkc_gru_forward(const mtkc_gru_args* a, void* stream) {
  if(a->b <= 0)
    return MTKC_OK;
  if(a->d > (int64_t)GT * GV)
    return fail(MTKC_DIMENSION, "gru: state dim above 2048");
  ProfScope prof(S(stream), "gru", 4.0 * a->b * a->d * 10);
  ::mtkc::launch(gru_fwd_kernel, (unsigned)a->b, GT, 0, S(stream), *a);
  MTKC_POST_LAUNCH("gru_fwd_kernel");
  return MTKC_OK;
}

int mtkc_gru_backward(const mtkc_gru_args* a, void* stream) {
  if(a->b <= 0)
    return MTKC_OK;
  if(a->d > (int64_t)GT * GV)
    return fail(MTKC_DIMENSION, "gru: state dim above 2048");
  ProfScope prof(S(stream), "gru", 4.0 * a->b * a->d * 14);
  ::mtkc::launch(gru_bwd_kernel, (unsigned)a->b, GT, 0, S(stream), *a);
  MTKC_POST_LAUNCH("gru_bwd_kernel");
  return MTKC_OK;
}

}  // extern "C"
