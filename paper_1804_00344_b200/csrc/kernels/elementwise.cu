// Elementwise, broadcast and reverse-broadcast kernels.
// Reference: ewiseBinaryInto / ewiseUnaryInto / accumulateReduced / axpy
// (tensor.cpp:111-237) and the graph's unary/binary/scale/addScalar backward
// rules (graph.cpp:139-268).  Grid-stride, 4-d right-aligned indexing.
#include "common.cuh"

using namespace mtkc;

namespace {

struct BinP {
  int op;
  float* out;
  const float* a;
  const float* b;
  int64_t od[4];
  int64_t sa[4], sb[4];
  int64_t n;
  int* flags;
};

__global__ void binary_kernel(BinP p) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n;
      i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    int64_t i3 = r % p.od[3];
    r /= p.od[3];
    int64_t i2 = r % p.od[2];
    r /= p.od[2];
    int64_t i1 = r % p.od[1];
    int64_t i0 = r / p.od[1];
    float x = p.a[i0 * p.sa[0] + i1 * p.sa[1] + i2 * p.sa[2] + i3 * p.sa[3]];
    float y = p.b[i0 * p.sb[0] + i1 * p.sb[1] + i2 * p.sb[2] + i3 * p.sb[3]];
    if(p.op == MTKC_DIV && y == 0.f && p.flags)
      atomicOr(p.flags, MTKC_FLAG_DIV_ZERO);
    p.out[i] = apply_binary(p.op, x, y);
  }
}

// same-shape operands: contiguous, 16-byte vectors
__global__ void binary_same4_kernel(int op, float4* out, const float4* a, const float4* b,
                                    int64_t n4, int* flags) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
      i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = a[i], y = b[i];
    if(op == MTKC_DIV && flags && (y.x == 0.f || y.y == 0.f || y.z == 0.f || y.w == 0.f))
      atomicOr(flags, MTKC_FLAG_DIV_ZERO);
    out[i] = make_float4(apply_binary(op, x.x, y.x), apply_binary(op, x.y, y.y),
                         apply_binary(op, x.z, y.z), apply_binary(op, x.w, y.w));
  }
}

__global__ void unary_kernel(int op, float* out, const float* a, int64_t n) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x)
    out[i] = apply_unary(op, a[i]);
}

// graph.cpp:200-218
__global__ void unary_bwd_kernel(int op, float* gx, const float* go, const float* y,
                                 const float* x, int64_t n) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    float g = go[i];
    switch(op) {
      case MTKC_TANH: gx[i] += g * (1.f - y[i] * y[i]); break;
      case MTKC_SIGMOID: gx[i] += g * y[i] * (1.f - y[i]); break;
      case MTKC_RELU: gx[i] += x[i] > 0.f ? g : 0.f; break;
      case MTKC_EXP: gx[i] += g * y[i]; break;
      case MTKC_LOG: gx[i] += g / x[i]; break;
      case MTKC_NEG: gx[i] -= g; break;
      default: break;
    }
  }
}

// Per-element gradient contribution of one binary operand (graph.cpp:153-179).
__device__ __forceinline__ float binary_grad(int op, int which, float g, float xa, float xb,
                                             float y) {
  switch(op) {
    case MTKC_ADD: return g;
    case MTKC_SUB: return which == 0 ? g : -g;
    case MTKC_MUL: return which == 0 ? g * xb : g * xa;
    case MTKC_DIV: return which == 0 ? g / xb : -((g * y) / xb);
    default: return 0.f;
  }
}

struct BinBwdP {
  int op, which;
  float* gt;
  const float* go;
  const float* a;
  const float* b;
  const float* y;
  int64_t od[4];
  int64_t sa[4], sb[4];
  int64_t td[4];   // target dims (padded)
  int64_t st[4];   // target strides over od (0 on broadcast dims)
  int64_t tn;      // target element count
  int64_t bcount;  // broadcast positions per target element
  int64_t bd[4];   // extents of broadcast dims (1 elsewhere)
};

// One thread per target element; sums its broadcast positions in output
// row-major order, the order accumulateReduced visits them (tensor.cpp:214-222).
__global__ void binary_bwd_kernel(BinBwdP p) {
  MTKC_PDL_ENTRY();
  for(int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < p.tn;
      t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t;
    int64_t tc[4];
    for(int d = 3; d >= 0; --d) {
      tc[d] = r % p.td[d];
      r /= p.td[d];
    }
    float acc = p.gt[t];
    for(int64_t k = 0; k < p.bcount; ++k) {
      int64_t kk = k;
      int64_t oc[4];
      for(int d = 3; d >= 0; --d) {
        int64_t bi = kk % p.bd[d];
        kk /= p.bd[d];
        oc[d] = p.bd[d] > 1 ? bi : tc[d];
      }
      int64_t oi = ((oc[0] * p.od[1] + oc[1]) * p.od[2] + oc[2]) * p.od[3] + oc[3];
      float xa = p.a ? p.a[oc[0] * p.sa[0] + oc[1] * p.sa[1] + oc[2] * p.sa[2] + oc[3] * p.sa[3]]
                     : 0.f;
      float xb = p.b ? p.b[oc[0] * p.sb[0] + oc[1] * p.sb[1] + oc[2] * p.sb[2] + oc[3] * p.sb[3]]
                     : 0.f;
      acc += binary_grad(p.op, p.which, p.go[oi], xa, xb, p.y ? p.y[oi] : 0.f);
    }
    p.gt[t] = acc;
  }
}

__global__ void scale_shift_kernel(float* out, const float* a, float s, float c, int64_t n) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    float v = a[i];
    if(s != 1.f)
      v = s * v;
    if(c != 0.f)
      v = v + c;
    out[i] = v;
  }
}

__global__ void axpy_kernel(float* out, const float* a, float alpha, int64_t n) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x)
    out[i] += alpha == 1.f ? a[i] : alpha * a[i];
}

__global__ void axpy4_kernel(float4* out, const float4* a, float alpha, int64_t n4) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
      i += (int64_t)gridDim.x * blockDim.x) {
    float4 o = out[i], x = a[i];
    if(alpha != 1.f) {
      x.x *= alpha;
      x.y *= alpha;
      x.z *= alpha;
      x.w *= alpha;
    }
    o.x += x.x;
    o.y += x.y;
    o.z += x.z;
    o.w += x.w;
    out[i] = o;
  }
}

__global__ void fill_kernel(float* out, float v, int64_t n) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

// h = hn*m + h*(1-m) with m [rows] (models.cpp:170-172): reference computes
// notM = addScalar(neg(m), 1) then add(mul(hn, m), mul(h, notM)).
__global__ void mask_blend_kernel(float* out, const float* a, const float* b, const float* m,
                                  int64_t rows, int64_t cols) {
  MTKC_PDL_ENTRY();
  int64_t n = rows * cols;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    float mm = m[i / cols];
    float nm = -mm + 1.f;
    out[i] = a[i] * mm + b[i] * nm;
  }
}

__global__ void mask_blend_bwd_kernel(float* ga, float* gb, const float* go, const float* m,
                                      int64_t rows, int64_t cols, int acc_a, int acc_b) {
  MTKC_PDL_ENTRY();
  int64_t n = rows * cols;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    float mm = m[i / cols];
    float nm = -mm + 1.f;
    float g = go[i];
    if(ga)
      ga[i] = (acc_a ? ga[i] : 0.f) + g * mm;
    if(gb)
      gb[i] = (acc_b ? gb[i] : 0.f) + g * nm;
  }
}

__global__ void scale_add_periodic_kernel(float* out, const float* x, float s, const float* c,
                                          int64_t n, int64_t period) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    float v = x[i];
    if(s != 1.f)
      v = s * v;
    out[i] = v + c[i % period];
  }
}

__global__ void relu_mask_kernel(float* gx, const float* gate, int64_t n) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x)
    if(!(gate[i] > 0.f))
      gx[i] = 0.f;
}

int64_t prod4(const int64_t d[4]) { return d[0] * d[1] * d[2] * d[3]; }

}  // namespace

extern "C" {

int mtkc_ewise_binary(int op, float* out, const int64_t od[4], const float* a,
                      const int64_t ad[4], const float* b, const int64_t bd[4], int* flags,
                      void* stream) {
  BinP p;
  p.op = op;
  p.out = out;
  p.a = a;
  p.b = b;
  p.n = prod4(od);
  p.flags = flags;
  Bcast4 sa = bcast_strides(ad), sb = bcast_strides(bd);
  for(int i = 0; i < 4; ++i) {
    p.od[i] = od[i];
    p.sa[i] = sa.s[i];
    p.sb[i] = sb.s[i];
  }
  if(p.n == 0)
    return MTKC_OK;
  bool same = true;
  for(int i = 0; i < 4; ++i)
    same &= ad[i] == od[i] && bd[i] == od[i];
  if(same && p.n % 4 == 0 && ((uintptr_t)out | (uintptr_t)a | (uintptr_t)b) % 16 == 0) {
    ::mtkc::launch(binary_same4_kernel, grid1d(p.n / 4, 256), 256, 0, S(stream), 
        op, (float4*)out, (const float4*)a, (const float4*)b, p.n / 4, flags);
    MTKC_POST_LAUNCH("binary_same4_kernel");
    return MTKC_OK;
  }
  ::mtkc::launch(binary_kernel, grid1d(p.n, 256), 256, 0, S(stream), p);
  MTKC_POST_LAUNCH("binary_kernel");
  return MTKC_OK;
}

int mtkc_ewise_unary(int op, float* out, const float* a, int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  ::mtkc::launch(unary_kernel, grid1d(n, 256), 256, 0, S(stream), op, out, a, n);
  MTKC_POST_LAUNCH("unary_kernel");
  return MTKC_OK;
}

int mtkc_unary_backward(int op, float* gx, const float* go, const float* y, const float* x,
                        int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  ::mtkc::launch(unary_bwd_kernel, grid1d(n, 256), 256, 0, S(stream), op, gx, go, y, x, n);
  MTKC_POST_LAUNCH("unary_bwd_kernel");
  return MTKC_OK;
}

int mtkc_binary_backward(int op, int which, float* gtarget, const int64_t td[4],
                         const float* go, const int64_t od[4], const float* a,
                         const int64_t ad[4], const float* b, const int64_t bd[4],
                         const float* y, void* stream) {
  BinBwdP p;
  p.op = op;
  p.which = which;
  p.gt = gtarget;
  p.go = go;
  p.a = a;
  p.b = b;
  p.y = y;
  Bcast4 sa = bcast_strides(ad), sb = bcast_strides(bd);
  p.bcount = 1;
  for(int i = 0; i < 4; ++i) {
    p.od[i] = od[i];
    p.sa[i] = sa.s[i];
    p.sb[i] = sb.s[i];
    p.td[i] = td[i];
    if(td[i] != od[i] && td[i] != 1)
      return fail(MTKC_DIMENSION, "binary_backward: target not broadcast-compatible");
    p.bd[i] = td[i] == od[i] ? 1 : od[i];
    p.bcount *= p.bd[i];
  }
  p.tn = prod4(td);
  if(p.tn == 0)
    return MTKC_OK;
  ::mtkc::launch(binary_bwd_kernel, grid1d(p.tn, 128), 128, 0, S(stream), p);
  MTKC_POST_LAUNCH("binary_bwd_kernel");
  return MTKC_OK;
}

int mtkc_scale_shift(float* out, const float* a, float s, float c, int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  ::mtkc::launch(scale_shift_kernel, grid1d(n, 256), 256, 0, S(stream), out, a, s, c, n);
  MTKC_POST_LAUNCH("scale_shift_kernel");
  return MTKC_OK;
}

int mtkc_axpy(float* out, const float* a, float alpha, int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  if(n % 4 == 0 && ((uintptr_t)out % 16 == 0) && ((uintptr_t)a % 16 == 0)) {
    ::mtkc::launch(axpy4_kernel, grid1d(n / 4, 256), 256, 0, S(stream), (float4*)out, (const float4*)a,
                                                            alpha, n / 4);
  } else {
    ::mtkc::launch(axpy_kernel, grid1d(n, 256), 256, 0, S(stream), out, a, alpha, n);
  }
  MTKC_POST_LAUNCH("axpy_kernel");
  return MTKC_OK;
}

int mtkc_accumulate_reduced(float* out, const int64_t od[4], const float* src,
                            const int64_t sd[4], void* stream) {
  // out += reduce(src): the Add rule of binary_backward with go = src.
  return mtkc_binary_backward(MTKC_ADD, 0, out, od, src, sd, nullptr, sd, nullptr, sd, nullptr,
                              stream);
}

int mtkc_fill(float* out, float v, int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  ::mtkc::launch(fill_kernel, grid1d(n, 256), 256, 0, S(stream), out, v, n);
  MTKC_POST_LAUNCH("fill_kernel");
  return MTKC_OK;
}

int mtkc_scale_add_periodic(float* out, const float* x, float s, const float* c, int64_t n,
                            int64_t period, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  ::mtkc::launch(scale_add_periodic_kernel, grid1d(n, 256), 256, 0, S(stream), out, x, s, c, n, period);
  MTKC_POST_LAUNCH("scale_add_periodic_kernel");
  return MTKC_OK;
}

int mtkc_relu_mask(float* gx, const float* gate, int64_t n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  ::mtkc::launch(relu_mask_kernel, grid1d(n, 256), 256, 0, S(stream), gx, gate, n);
  MTKC_POST_LAUNCH("relu_mask_kernel");
  return MTKC_OK;
}

int mtkc_mask_blend(float* out, const float* a, const float* b, const float* m, int64_t rows,
                    int64_t cols, void* stream) {
  if(rows * cols <= 0)
    return MTKC_OK;
  ::mtkc::launch(mask_blend_kernel, grid1d(rows * cols, 256), 256, 0, S(stream), out, a, b, m, rows, cols);
  MTKC_POST_LAUNCH("mask_blend_kernel");
  return MTKC_OK;
}

int mtkc_mask_blend_backward(float* ga, float* gb, const float* go, const float* m,
                             int64_t rows, int64_t cols, int accumulate_a, int accumulate_b,
                             void* stream) {
  if(rows * cols <= 0)
    return MTKC_OK;
  ::mtkc::launch(mask_blend_bwd_kernel, grid1d(rows * cols, 256), 256, 0, S(stream), 
      ga, gb, go, m, rows, cols, accumulate_a, accumulate_b);
  MTKC_POST_LAUNCH("mask_blend_bwd_kernel");
  return MTKC_OK;
}

}  // extern "C"
