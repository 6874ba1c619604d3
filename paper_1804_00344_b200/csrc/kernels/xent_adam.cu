// Fused softmax + cross-entropy over the vocabulary (crossEntropy
// graph.cpp:859-924) and the fused Adam + EMA + grad-zero update
// (Adam::updateTensor train.cpp:30-47, Adam::update :49-59,
// AveragedParameters::update :69-79).
//
// Cross-entropy never materialises probabilities: the forward keeps only the
// per-row max and sum of exp(x - max) (8 bytes per row instead of the
// reference's [N x V] probs cache, graph.cpp:882-897); the backward
// recomputes p = exp(x - max)/sum in the same order as the reference and
// writes the logits gradient in one pass: 2*4*N*V bytes of HBM per step.
#include "common.cuh"
#include "tc_ptx.cuh"

using namespace mtkc;

namespace {

constexpr int XT = 512;

// stats[r] = {max, sum}; row_loss[r] = m*(max + log(sum) - x[y]) or 0
__global__ void __launch_bounds__(XT) xent_fwd_kernel(const float* logits, const int32_t* tg,
                                                      const float* mask, int64_t V,
                                                      float* stats, float* rowLoss) {
  MTKC_PDL_ENTRY();
  __shared__ float red[32];
  int64_t r = blockIdx.x;
  const float* x = logits + r * V;
  float mx = -INFINITY;
  if(V % 4 == 0 && ((uintptr_t)x % 16 == 0)) {
    const float4* x4 = (const float4*)x;
    for(int64_t j = threadIdx.x; j < V / 4; j += XT) {
      float4 v = x4[j];
      mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
  } else {
    for(int64_t j = threadIdx.x; j < V; j += XT)
      mx = fmaxf(mx, x[j]);
  }
  mx = block_max(mx, red);
  float s = 0.f;
  if(V % 4 == 0 && ((uintptr_t)x % 16 == 0)) {
    const float4* x4 = (const float4*)x;
    for(int64_t j = threadIdx.x; j < V / 4; j += XT) {
      float4 v = x4[j];
      s += expf(v.x - mx) + expf(v.y - mx) + expf(v.z - mx) + expf(v.w - mx);
    }
  } else {
    for(int64_t j = threadIdx.x; j < V; j += XT)
      s += expf(x[j] - mx);
  }
  s = block_sum(s, red);
  if(threadIdx.x == 0) {
    stats[2 * r] = mx;
    stats[2 * r + 1] = s;
    float m = mask ? mask[r] : 1.f;
    float l = 0.f;
    if(m != 0.f) {
      float lse = mx + logf(s);
      l = m * (lse - x[tg[r]]);
    }
    rowLoss[r] = l;
  }
}

// FP32 parity mode: the reference's summation order (graph.cpp:887-898) --
// per row, sum += exp(x_j - max) for j = 0..V-1 one after the other.  The
// row max (order-free) comes from xent_fwd_kernel.  One warp owns 32 rows:
// each 32-column chunk of those rows is staged through shared memory with
// coalesced loads (one 128-B row segment per load instruction), then every
// lane adds its own row's 32 terms in column order.  Also writes row_loss.
__global__ void __launch_bounds__(32) xent_sum_seq_kernel(const float* logits, const int32_t* tg,
                                                          const float* mask, int64_t rows,
                                                          int64_t V, float* stats,
                                                          float* rowLoss) {
  MTKC_PDL_ENTRY();
  __shared__ float tile[32][33];
  const int lane = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * 32, me = r0 + lane;
  const float mx = me < rows ? stats[2 * me] : 0.f;
  float s = 0.f;
  for(int64_t c = 0; c < V; c += 32) {
#pragma unroll 8
    for(int i = 0; i < 32; ++i) {
      int64_t r = r0 + i, j = c + lane;
      tile[i][lane] = (r < rows && j < V) ? logits[r * V + j] : 0.f;
    }
    __syncwarp();
    const int n = V - c < 32 ? (int)(V - c) : 32;
    for(int j = 0; j < n; ++j)
      s = s + expf(tile[lane][j] - mx);
    __syncwarp();
  }
  if(me < rows) {
    stats[2 * me + 1] = s;
    float m = mask ? mask[me] : 1.f;
    float l = 0.f;
    if(m != 0.f) {
      float lse = mx + logf(s);
      l = m * (lse - logits[me * V + tg[me]]);
    }
    rowLoss[me] = l;
  }
}

// FP32 parity mode: lossSum over rows in row order, then / count
// (graph.cpp:899-906); masked rows contribute an exact 0
__global__ void loss_seq_kernel(const float* rowLoss, int64_t rows, float count, float* loss) {
  MTKC_PDL_ENTRY();
  if(threadIdx.x != 0)
    return;
  float s = 0.f;
  for(int64_t r = 0; r < rows; ++r)
    s = s + rowLoss[r];
  loss[0] = s / count;
}

// loss = sum(row_loss)/count, fixed-order block reduction
__global__ void __launch_bounds__(1024) loss_sum_kernel(const float* rowLoss, int64_t rows,
                                                        float count, float* loss) {
  MTKC_PDL_ENTRY();
  __shared__ float red[32];
  float s = 0.f;
  for(int64_t r = threadIdx.x; r < rows; r += blockDim.x)
    s += rowLoss[r];
  s = block_sum(s, red);
  if(threadIdx.x == 0)
    loss[0] = s / count;
}

// g[r,j] (+)= (go*m)*p_j, then g[r,y] -= go*m  (graph.cpp:909-922)
__global__ void __launch_bounds__(256) xent_bwd_kernel(float* g, const float* logits,
                                                       const float* stats, const int32_t* tg,
                                                       const float* mask, const float* gloss,
                                                       int64_t rows, int64_t V, float count,
                                                       int acc) {
  MTKC_PDL_ENTRY();
  int64_t r = blockIdx.y;
  float go = gloss[0] / count;
  float m = mask ? mask[r] : 1.f;
  float gm = go * m;
  float mx = stats[2 * r], sum = stats[2 * r + 1];
  int32_t y = tg[r];
  const float* x = logits + r * V;
  float* gr = g + r * V;
  int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  bool vec = V % 4 == 0 && ((uintptr_t)x % 16 == 0) && ((uintptr_t)gr % 16 == 0);
  for(int64_t j = j0; j < V; j += stride) {
    if(vec) {
      float4 xv = *(const float4*)(x + j);
      float4 o = acc ? *(float4*)(gr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      float xs[4] = {xv.x, xv.y, xv.z, xv.w};
      float os[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for(int u = 0; u < 4; ++u) {
        if(m != 0.f) {
          float p = expf(xs[u] - mx) / sum;
          float t = os[u] + gm * p;
          if(j + u == y)
            t = t - gm;
          os[u] = t;
        }
      }
      *(float4*)(gr + j) = make_float4(os[0], os[1], os[2], os[3]);
    } else {
      for(int u = 0; u < 4 && j + u < V; ++u) {
        float t = acc ? gr[j + u] : 0.f;
        if(m != 0.f) {
          float p = expf(x[j + u] - mx) / sum;
          t = t + gm * p;
          if(j + u == y)
            t = t - gm;
        }
        gr[j + u] = t;
      }
    }
  }
}

// TF32-mode variants (mtkc_xent_forward_fast / _backward_fast): the same
// stats / loss / gradient from ONE pass over each row -- running max and
// rescaled sum (online softmax), exp as ex2.approx (__expf, rel. err ~2^-21)
// and a reciprocal instead of a division per element.
__global__ void __launch_bounds__(XT) xent_fwd_fast_kernel(const float* logits,
                                                           const int32_t* tg, const float* mask,
                                                           int64_t V, float* stats,
                                                           float* rowLoss) {
  MTKC_PDL_ENTRY();
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  const float* x = logits + r * V;
  float mx = -INFINITY, s = 0.f;
  auto add4 = [&](float a, float b, float c, float d) {
    const float m4 = fmaxf(fmaxf(a, b), fmaxf(c, d));
    if(m4 > mx) {
      s = mx == -INFINITY ? 0.f : s * __expf(mx - m4);
      mx = m4;
    }
    s += (__expf(a - mx) + __expf(b - mx)) + (__expf(c - mx) + __expf(d - mx));
  };
  if(V % 4 == 0 && ((uintptr_t)x % 16 == 0)) {
    const float4* x4 = (const float4*)x;
    int64_t j = threadIdx.x;
    for(; j + XT < V / 4; j += 2 * XT) {  // two loads in flight
      const float4 u = __ldcs(x4 + j), v = __ldcs(x4 + j + XT);
      add4(u.x, u.y, u.z, u.w);
      add4(v.x, v.y, v.z, v.w);
    }
    if(j < V / 4) {
      const float4 u = __ldcs(x4 + j);
      add4(u.x, u.y, u.z, u.w);
    }
  } else {
    for(int64_t j = threadIdx.x; j < V; j += XT)
      add4(x[j], -INFINITY, -INFINITY, -INFINITY);
  }
  // combine (max, sum) pairs across the block in a fixed order
  const float M = block_max(mx, red);
  float sc = mx == -INFINITY ? 0.f : s * __expf(mx - M);
  sc = block_sum(sc, red);
  if(threadIdx.x == 0) {
    stats[2 * r] = M;
    stats[2 * r + 1] = sc;
    float m = mask ? mask[r] : 1.f;
    float l = 0.f;
    if(m != 0.f)
      l = m * (M + logf(sc) - x[tg[r]]);
    rowLoss[r] = l;
  }
}

__global__ void __launch_bounds__(256) xent_bwd_fast_kernel(float* g, const float* logits,
                                                            const float* stats,
                                                            const int32_t* tg, const float* mask,
                                                            const float* gloss, int64_t V,
                                                            float count, int acc) {
  MTKC_PDL_ENTRY();
  const int64_t r = blockIdx.y;
  const float m = mask ? mask[r] : 1.f;
  const float gm = (gloss[0] / count) * m;
  const float mx = stats[2 * r], scale = m != 0.f ? gm / stats[2 * r + 1] : 0.f;
  const int32_t y = tg[r];
  const float4* x4 = reinterpret_cast<const float4*>(logits + r * V);
  float4* g4 = reinterpret_cast<float4*>(g + r * V);
  for(int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < V / 4;
      j += (int64_t)gridDim.x * blockDim.x) {
    const float4 xv = __ldcs(x4 + j);
    float4 o = acc ? g4[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    o.x += scale * __expf(xv.x - mx);
    o.y += scale * __expf(xv.y - mx);
    o.z += scale * __expf(xv.z - mx);
    o.w += scale * __expf(xv.w - mx);
    const int64_t d = (int64_t)y - 4 * j;
    if(m != 0.f && d >= 0 && d < 4) {
      if(d == 0) o.x -= gm;
      if(d == 1) o.y -= gm;
      if(d == 2) o.z -= gm;
      if(d == 3) o.w -= gm;
    }
    g4[j] = o;
  }
}

// Fused cross-entropy forward + backward (TF32 training path): one CTA of
// 1024 threads per row keeps the whole row in registers (V <= 4096*NV), so
// the logits are read from HBM once: row max, sum of exp (two-pass, the
// reference's order of operations, graph.cpp:880-922), the row loss, and
// the gradient d = (exp(x - max)/sum - onehot) * m * scale / count written
// IN PLACE over the logits (their only consumer is this loss; `scale` is
// the loss seed the backward would receive).
constexpr int XF = 1024;
template <int NV>
__global__ void __launch_bounds__(XF, 1) xent_fused_kernel(float* logits, const int32_t* tg,
                                                           const float* mask, int64_t V,
                                                           float scale, float count,
                                                           float* rowLoss) {
  MTKC_PDL_ENTRY();
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  float4* x4 = reinterpret_cast<float4*>(logits + r * V);
  const int64_t V4 = V / 4;
  float4 v[NV];
  float mx = -INFINITY;
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t j = threadIdx.x + (int64_t)k * XF;
    v[k] = j < V4 ? __ldcs(x4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    mx = fmaxf(mx, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
  }
  mx = block_max(mx, red);
  float s = 0.f;
#pragma unroll
  for(int k = 0; k < NV; ++k)
    if(threadIdx.x + (int64_t)k * XF < V4)
      s += (__expf(v[k].x - mx) + __expf(v[k].y - mx)) + (__expf(v[k].z - mx) + __expf(v[k].w - mx));
  s = block_sum(s, red);
  const float m = mask ? mask[r] : 1.f;
  const int32_t y = tg[r];
  if(threadIdx.x == 0) {
    // x[y] is read before any thread overwrites the row: block_sum ends in a barrier
    rowLoss[r] = m != 0.f ? m * (mx + logf(s) - logits[r * V + y]) : 0.f;
  }
  __syncthreads();
  const float gm = (scale / count) * m;
  const float sc = m != 0.f ? gm / s : 0.f;
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t j = threadIdx.x + (int64_t)k * XF;
    if(j >= V4)
      break;
    float4 o;
    o.x = sc * __expf(v[k].x - mx);
    o.y = sc * __expf(v[k].y - mx);
    o.z = sc * __expf(v[k].z - mx);
    o.w = sc * __expf(v[k].w - mx);
    const int64_t dd = (int64_t)y - 4 * j;
    if(m != 0.f && dd >= 0 && dd < 4) {
      if(dd == 0) o.x -= gm;
      if(dd == 1) o.y -= gm;
      if(dd == 2) o.z -= gm;
      if(dd == 3) o.w -= gm;
    }
    __stcs(x4 + j, o);
  }
}

// Persistent form of xent_fused_kernel: one CTA per SM walks rows
// r, r + grid, ...; while row r is reduced and its gradient stored from
// registers, row r + grid already streams into shared memory (one bulk
// copy), so every SM keeps a row of reads in flight through the whole
// kernel (the one-row-per-CTA form idles HBM during its reductions).
// Same arithmetic, same order as xent_fused_kernel.
template <int NV>
__global__ void __launch_bounds__(XF, 1) xent_fused_persist_kernel(float* logits,
                                                                   const int32_t* tg,
                                                                   const float* mask, int64_t rows,
                                                                   int64_t V, float scale,
                                                                   float count, float* rowLoss) {
  extern __shared__ __align__(16) float srow[];  // [V]
  __shared__ float red[32];
  __shared__ __align__(8) uint64_t bar;
  const int64_t V4 = V / 4;
  const uint32_t bytes = (uint32_t)(V * 4);
  if(threadIdx.x == 0) {
    mtkc::tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  MTKC_PDL_ENTRY();
  if(threadIdx.x == 0 && (int64_t)blockIdx.x < rows) {
    mtkc::tc::mbar_expect_tx(&bar, bytes);
    mtkc::tc::bulk_load_1d(srow, logits + (int64_t)blockIdx.x * V, bytes, &bar);
  }
  uint32_t phase = 0;
  const float4* s4 = reinterpret_cast<const float4*>(srow);
  for(int64_t r = blockIdx.x; r < rows; r += gridDim.x, phase ^= 1) {
    mtkc::tc::mbar_wait(&bar, phase);
    float4 v[NV];
    float mx = -INFINITY;
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t j = threadIdx.x + (int64_t)k * XF;
      v[k] = j < V4 ? s4[j] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      mx = fmaxf(mx, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
    }
    const int32_t y = tg[r];
    const float xy = srow[y];
    __syncthreads();  // the row buffer is free: stream in the next row
    if(threadIdx.x == 0 && r + gridDim.x < rows) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mtkc::tc::mbar_expect_tx(&bar, bytes);
      mtkc::tc::bulk_load_1d(srow, logits + (r + gridDim.x) * V, bytes, &bar);
    }
    mx = block_max(mx, red);
    float s = 0.f;
#pragma unroll
    for(int k = 0; k < NV; ++k)
      if(threadIdx.x + (int64_t)k * XF < V4)
        s += (__expf(v[k].x - mx) + __expf(v[k].y - mx)) + (__expf(v[k].z - mx) + __expf(v[k].w - mx));
    s = block_sum(s, red);
    const float m = mask ? mask[r] : 1.f;
    if(threadIdx.x == 0)
      rowLoss[r] = m != 0.f ? m * (mx + logf(s) - xy) : 0.f;
    const float gm = (scale / count) * m;
    const float sc = m != 0.f ? gm / s : 0.f;
    float4* x4 = reinterpret_cast<float4*>(logits + r * V);
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t j = threadIdx.x + (int64_t)k * XF;
      if(j >= V4)
        break;
      float4 o;
      o.x = sc * __expf(v[k].x - mx);
      o.y = sc * __expf(v[k].y - mx);
      o.z = sc * __expf(v[k].z - mx);
      o.w = sc * __expf(v[k].w - mx);
      const int64_t dd = (int64_t)y - 4 * j;
      if(m != 0.f && dd >= 0 && dd < 4) {
        if(dd == 0) o.x -= gm;
        if(dd == 1) o.y -= gm;
        if(dd == 2) o.z -= gm;
        if(dd == 3) o.w -= gm;
      }
      __stcs(x4 + j, o);
    }
  }
}

// One element of the reference's Adam + EMA, with separately rounded ops
// (kernels are compiled with -fmad=false) in the reference's order.
__device__ __forceinline__ void adam_one(float& th, float& g, float& m, float& v, float& a,
                                         float lr, float b1, float b2, float eps, float c1,
                                         float c2, float ab, int doAvg, int zg) {
  float gv = g;
  m = b1 * m + (1.f - b1) * gv;
  v = b2 * v + (1.f - b2) * gv * gv;
  float mh = m / c1;
  float vh = v / c2;
  th = th - lr * mh / (sqrtf(vh) + eps);
  if(doAvg)
    a = ab * a + (1.f - ab) * th;
  if(zg)
    g = 0.f;
}

__global__ void adam_ema_kernel(float* th, float* g, float* m, float* v, float* a, int64_t n,
                                float lr, float b1, float b2, float eps, float c1, float c2,
                                float ab, int doAvg, int zg, const int* flags) {
  MTKC_PDL_ENTRY();
  if(flags && *flags)
    return;  // all-or-nothing (train.cpp:51-53); also skipped after a device error
  int64_t n4 = n / 4;
  float4* th4 = (float4*)th;
  float4* g4 = (float4*)g;
  float4* m4 = (float4*)m;
  float4* v4 = (float4*)v;
  float4* a4 = (float4*)a;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
      i += (int64_t)gridDim.x * blockDim.x) {
    float4 T = th4[i], G = g4[i], M = m4[i], Vv = v4[i];
    float4 A = doAvg ? a4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    adam_one(T.x, G.x, M.x, Vv.x, A.x, lr, b1, b2, eps, c1, c2, ab, doAvg, zg);
    adam_one(T.y, G.y, M.y, Vv.y, A.y, lr, b1, b2, eps, c1, c2, ab, doAvg, zg);
    adam_one(T.z, G.z, M.z, Vv.z, A.z, lr, b1, b2, eps, c1, c2, ab, doAvg, zg);
    adam_one(T.w, G.w, M.w, Vv.w, A.w, lr, b1, b2, eps, c1, c2, ab, doAvg, zg);
    th4[i] = T;
    m4[i] = M;
    v4[i] = Vv;
    if(zg)
      g4[i] = G;
    if(doAvg)
      a4[i] = A;
  }
  for(int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    float dummy = 0.f;
    adam_one(th[i], g[i], m[i], v[i], doAvg ? a[i] : dummy, lr, b1, b2, eps, c1, c2, ab, doAvg,
             zg);
  }
}

__global__ void ema_kernel(float* a, const float* th, int64_t n, float b) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x)
    a[i] = b * a[i] + (1.f - b) * th[i];
}

}  // namespace

extern "C" {

int mtkc_ema(float* avg, const float* theta, int64_t n, float beta, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  ::mtkc::launch(ema_kernel, grid1d(n, 256), 256, 0, S(stream), avg, theta, n, beta);
  MTKC_POST_LAUNCH("ema_kernel");
  return MTKC_OK;
}

int mtkc_xent_forward(const float* logits, const int32_t* targets, const float* mask,
                      int64_t rows, int64_t vocab, float* lse, float* row_loss, float* loss,
                      float count, void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "xent", 4.0 * rows * vocab);  // read logits
  ::mtkc::launch(xent_fwd_kernel, (unsigned)rows, XT, 0, S(stream), logits, targets, mask, vocab, lse,
                                                       row_loss);
  MTKC_POST_LAUNCH("xent_fwd_kernel");
  // the row sums and the loss again, in the reference's order (the block
  // reduction above is ~sqrt(V) times more accurate than the reference's
  // running sum, which differs from it by up to ~1e-4 relative at V = 50k)
  ::mtkc::launch(xent_sum_seq_kernel, (unsigned)cdiv(rows, 32), 32, 0, S(stream), logits, targets, mask,
                 rows, vocab, lse, row_loss);
  MTKC_POST_LAUNCH("xent_sum_seq_kernel");
  ::mtkc::launch(loss_seq_kernel, 1, 32, 0, S(stream), row_loss, rows, count, loss);
  MTKC_POST_LAUNCH("loss_seq_kernel");
  return MTKC_OK;
}

int mtkc_xent_backward(float* glogits, const float* logits, const float* lse,
                       const int32_t* targets, const float* mask, const float* gloss,
                       int64_t rows, int64_t vocab, float count, int accumulate,
                       void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "xent", (accumulate ? 12.0 : 8.0) * rows * vocab);
  int64_t per = cdiv(vocab, 4);
  unsigned gx = (unsigned)std::min<int64_t>(cdiv(per, 256), 8);
  dim3 grid(gx, (unsigned)rows);
  ::mtkc::launch(xent_bwd_kernel, grid, 256, 0, S(stream), glogits, logits, lse, targets, mask, gloss, rows,
                                              vocab, count, accumulate);
  MTKC_POST_LAUNCH("xent_bwd_kernel");
  return MTKC_OK;
}

int mtkc_xent_forward_fast(const float* logits, const int32_t* targets, const float* mask,
                           int64_t rows, int64_t vocab, float* lse, float* row_loss, float* loss,
                           float count, void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "xent", 4.0 * rows * vocab);  // read logits once
  ::mtkc::launch(xent_fwd_fast_kernel, (unsigned)rows, XT, 0, S(stream), logits, targets, mask,
                 vocab, lse, row_loss);
  MTKC_POST_LAUNCH("xent_fwd_fast_kernel");
  ::mtkc::launch(loss_sum_kernel, 1, 1024, 0, S(stream), row_loss, rows, count, loss);
  MTKC_POST_LAUNCH("loss_sum_kernel");
  return MTKC_OK;
}

int mtkc_xent_fused_supported(int64_t vocab) { return vocab % 4 == 0 && vocab <= 4 * XF * 8; }

int mtkc_xent_fused(float* logits, const int32_t* targets, const float* mask, int64_t rows,
                    int64_t vocab, float scale, float* row_loss, float* loss, float count,
                    void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  if(!mtkc_xent_fused_supported(vocab) || (uintptr_t)logits % 16)
    return fail(MTKC_DIMENSION, "fused cross entropy needs vocab % 4 == 0, vocab <= 32768");
  ProfScope prof(S(stream), "xent", 8.0 * rows * vocab);  // read logits, write dlogits
  const int nv = (int)cdiv(vocab / 4, XF);
  static const bool persist = getenv("MTK_XENT_ROWS") == nullptr;  // A/B switch
  if(persist) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<int64_t>(rows, sms);
    const size_t smem = (size_t)vocab * sizeof(float);
#define XF_LAUNCH(NVV)                                                                        \
  if(nv <= NVV) {                                                                             \
    static bool attr = false;                                                                 \
    if(!attr) {                                                                               \
      cudaFuncSetAttribute(xent_fused_persist_kernel<NVV>,                                    \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);           \
      attr = true;                                                                            \
    }                                                                                         \
    ::mtkc::launch(xent_fused_persist_kernel<NVV>, grid, XF, smem, S(stream), logits, targets, \
                   mask, rows, vocab, scale, count, row_loss);                                \
  } else
    XF_LAUNCH(1) XF_LAUNCH(2) XF_LAUNCH(4) XF_LAUNCH(8) {}
#undef XF_LAUNCH
  } else {
#define XF_LAUNCH(NVV)                                                                       \
  if(nv <= NVV) {                                                                            \
    ::mtkc::launch(xent_fused_kernel<NVV>, (unsigned)rows, XF, 0, S(stream), logits, targets, \
                   mask, vocab, scale, count, row_loss);                                     \
  } else
    XF_LAUNCH(1) XF_LAUNCH(2) XF_LAUNCH(4) XF_LAUNCH(8) {}
#undef XF_LAUNCH
  }
  MTKC_POST_LAUNCH("xent_fused_kernel");
  ::mtkc::launch(loss_sum_kernel, 1, 1024, 0, S(stream), row_loss, rows, count, loss);
  MTKC_POST_LAUNCH("loss_sum_kernel");
  return MTKC_OK;
}

int mtkc_xent_backward_fast(float* glogits, const float* logits, const float* lse,
                            const int32_t* targets, const float* mask, const float* gloss,
                            int64_t rows, int64_t vocab, float count, int accumulate,
                            void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  if(vocab % 4 || ((uintptr_t)logits | (uintptr_t)glogits) % 16)
    return mtkc_xent_backward(glogits, logits, lse, targets, mask, gloss, rows, vocab, count,
                              accumulate, stream);
  ProfScope prof(S(stream), "xent", (accumulate ? 12.0 : 8.0) * rows * vocab);
  const unsigned gx = (unsigned)std::min<int64_t>(cdiv(vocab / 4, 256), 8);
  ::mtkc::launch(xent_bwd_fast_kernel, dim3(gx, (unsigned)rows), 256, 0, S(stream), glogits,
                 logits, lse, targets, mask, gloss, vocab, count, accumulate);
  MTKC_POST_LAUNCH("xent_bwd_fast_kernel");
  return MTKC_OK;
}

int mtkc_adam_ema(float* theta, float* grad, float* m, float* v, float* avg, int64_t n,
                  float lr, float beta1, float beta2, float eps, float corr1, float corr2,
                  float avg_beta, int do_avg, int zero_grad, const int* flags, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  if(((uintptr_t)theta | (uintptr_t)grad | (uintptr_t)m | (uintptr_t)v |
      (do_avg ? (uintptr_t)avg : 0)) % 16)
    return fail(MTKC_CONTRACT, "adam: buffers must be 16-byte aligned");
  ProfScope prof(S(stream), "adam_ema", (do_avg ? 36.0 : 28.0) * n);
  ::mtkc::launch(adam_ema_kernel, grid1d(cdiv(n, 4), 256, 148 * 16), 256, 0, S(stream), 
      theta, grad, m, v, avg, n, lr, beta1, beta2, eps, corr1, corr2, avg_beta, do_avg,
      zero_grad, flags);
  MTKC_POST_LAUNCH("adam_ema_kernel");
  return MTKC_OK;
}

}  // extern "C"
