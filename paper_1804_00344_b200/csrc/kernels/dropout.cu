// Device (counter-based) dropout for throughput mode.
//
// Reference: ExpressionGraph::dropoutMask / dropout (graph.cpp:817-846) draw
// an inverted-dropout mask on the host from the graph's mt19937_64 stream
// (keep = 1/(1-p) where u >= p) and multiply it in as a constant node.  The
// host path (bit-exact with the reference) stays in csrc/host/graph.cpp;
// this file is the B200 throughput path: the mask element for mask index i
// is a pure function of (key, i) -- Philox4x32-10, the 24 high bits of one
// 32-bit word compared with ceil(p * 2^24) -- so it is never stored: the
// forward and the backward recompute the same bits.  The key is one 64-bit
// draw from the same per-(update, worker) graph RNG (train.cpp:170-176), so
// runs are reproducible and workers decorrelated exactly as in the reference.
//
// Mask index of element idx (variational dropout, graph.cpp:838-843: one
// mask broadcast along axis `a`): idx = (o * axisLen + t) * inner + j  ->
// mi = o * inner + j.  axisLen == 1 is the plain (full-shape) mask.
#include <cmath>

#include "common.cuh"

using namespace mtkc;

namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for(int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += W0;
    k.y += W1;
  }
  return c;
}

struct DropP {
  uint2 key;
  uint32_t thr;  // keep iff (word >> 8) >= thr
  float keep;    // 1/(1-p), rounded as the reference does (Real arithmetic)
  int64_t n, inner, axisLen;
};

__device__ __forceinline__ float mask4(const uint4& w, int lane, const DropP& p) {
  const uint32_t v = lane == 0 ? w.x : lane == 1 ? w.y : lane == 2 ? w.z : w.w;
  return (v >> 8) >= p.thr ? p.keep : 0.f;
}

__device__ __forceinline__ int64_t mask_index(int64_t idx, const DropP& p) {
  if(p.axisLen == 1)
    return idx;
  const int64_t j = idx % p.inner;
  const int64_t o = idx / (p.inner * p.axisLen);
  return o * p.inner + j;
}

__device__ __forceinline__ float mask_at(int64_t mi, const DropP& p) {
  const uint64_t g = (uint64_t)mi >> 2;
  const uint4 w = philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0u, 0u), p.key);
  return mask4(w, (int)(mi & 3), p);
}

// four consecutive elements whose mask indices are 4-aligned and consecutive
__device__ __forceinline__ float4 mask_vec(int64_t idx, const DropP& p) {
  const int64_t mi = mask_index(idx, p);
  const uint64_t g = (uint64_t)mi >> 2;
  const uint4 w = philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0u, 0u), p.key);
  return make_float4(mask4(w, 0, p), mask4(w, 1, p), mask4(w, 2, p), mask4(w, 3, p));
}

// out = (addend ? addend : 0) + x * m   (dropout, or the fused residual
// x + dropout(f) of a pre-norm sublayer, layers.cpp:135: add(x, dropout(f)))
template <bool VEC>
__global__ void dropout_kernel(float* __restrict__ out, const float* __restrict__ x,
                               const float* __restrict__ addend, DropP p) {
  MTKC_PDL_ENTRY();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if(VEC) {
    const int64_t n4 = p.n >> 2;
    for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 m = mask_vec(i * 4, p);
      const float4 v = reinterpret_cast<const float4*>(x)[i];
      float4 y = make_float4(v.x * m.x, v.y * m.y, v.z * m.z, v.w * m.w);
      if(addend) {
        const float4 r = reinterpret_cast<const float4*>(addend)[i];
        y = make_float4(r.x + y.x, r.y + y.y, r.z + y.z, r.w + y.w);
      }
      reinterpret_cast<float4*>(out)[i] = y;
    }
  } else {
    for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += stride) {
      float y = x[i] * mask_at(mask_index(i, p), p);
      if(addend)
        y = addend[i] + y;
      out[i] = y;
    }
  }
}

// gx (+)= go * m
template <bool VEC>
__global__ void dropout_bwd_kernel(float* __restrict__ gx, const float* __restrict__ go, DropP p,
                                   int accumulate) {
  MTKC_PDL_ENTRY();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if(VEC) {
    const int64_t n4 = p.n >> 2;
    for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 m = mask_vec(i * 4, p);
      const float4 g = reinterpret_cast<const float4*>(go)[i];
      float4 y = make_float4(g.x * m.x, g.y * m.y, g.z * m.z, g.w * m.w);
      if(accumulate) {
        const float4 o = reinterpret_cast<const float4*>(gx)[i];
        y = make_float4(o.x + y.x, o.y + y.y, o.z + y.z, o.w + y.w);
      }
      reinterpret_cast<float4*>(gx)[i] = y;
    }
  } else {
    for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += stride) {
      const float y = go[i] * mask_at(mask_index(i, p), p);
      gx[i] = accumulate ? gx[i] + y : y;
    }
  }
}

__global__ void dropout_mask_kernel(float* __restrict__ out, DropP p) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n;
      i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mask_at(i, p);
}

int make_params(DropP* p, int64_t n, int64_t inner, int64_t axis_len, float prob, uint64_t seed) {
  if(n < 0 || inner < 1 || axis_len < 1 || (axis_len > 1 && n % (inner * axis_len) != 0))
    return fail(MTKC_DIMENSION, "dropout: bad shape");
  if(!(prob >= 0.f && prob < 1.f))
    return fail(MTKC_CONTRACT, "dropout probability must be in [0, 1)");
  p->key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const double t = std::ceil((double)prob * 16777216.0);
  p->thr = (uint32_t)t;
  p->keep = 1.f / (1.f - prob);
  p->n = n;
  p->inner = inner;
  p->axisLen = axis_len;
  return MTKC_OK;
}

bool vec_ok(const DropP& p, const void* a, const void* b, const void* c) {
  auto al = [](const void* q) { return ((uintptr_t)q & 15u) == 0; };
  return p.n % 4 == 0 && (p.axisLen == 1 || p.inner % 4 == 0) && al(a) && al(b) && al(c);
}

}  // namespace

extern "C" {

int mtkc_dropout(float* out, const float* x, const float* addend, int64_t n, int64_t inner,
                 int64_t axis_len, float p, uint64_t seed, void* stream) {
  DropP q;
  if(int e = make_params(&q, n, inner, axis_len, p, seed))
    return e;
  if(n == 0)
    return MTKC_OK;
  ProfScope ps(S(stream), "dropout", (addend ? 12.0 : 8.0) * (double)n);
  if(vec_ok(q, out, x, addend))
    ::mtkc::launch(dropout_kernel<true>, grid1d(n / 4, 256), 256, 0, S(stream), out, x, addend, q);
  else
    ::mtkc::launch(dropout_kernel<false>, grid1d(n, 256), 256, 0, S(stream), out, x, addend, q);
  MTKC_POST_LAUNCH("dropout_kernel");
  return MTKC_OK;
}

int mtkc_dropout_backward(float* gx, const float* go, int64_t n, int64_t inner, int64_t axis_len,
                          float p, uint64_t seed, int accumulate, void* stream) {
  DropP q;
  if(int e = make_params(&q, n, inner, axis_len, p, seed))
    return e;
  if(n == 0)
    return MTKC_OK;
  ProfScope ps(S(stream), "dropout", (accumulate ? 12.0 : 8.0) * (double)n);
  if(vec_ok(q, gx, go, nullptr))
    ::mtkc::launch(dropout_bwd_kernel<true>, grid1d(n / 4, 256), 256, 0, S(stream), gx, go, q,
                   accumulate);
  else
    ::mtkc::launch(dropout_bwd_kernel<false>, grid1d(n, 256), 256, 0, S(stream), gx, go, q,
                   accumulate);
  MTKC_POST_LAUNCH("dropout_bwd_kernel");
  return MTKC_OK;
}

int mtkc_dropout_mask(float* out, int64_t n, float p, uint64_t seed, void* stream) {
  DropP q;
  if(int e = make_params(&q, n, 1, 1, p, seed))
    return e;
  if(n == 0)
    return MTKC_OK;
  ::mtkc::launch(dropout_mask_kernel, grid1d(n, 256), 256, 0, S(stream), out, q);
  MTKC_POST_LAUNCH("dropout_mask_kernel");
  return MTKC_OK;
}

}  // extern "C"
