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
#include <algorithm>

#include "colred.cuh"
#include "common.cuh"

using namespace mtkc;

namespace {

constexpr int LN_WARPS = 8;

template <int V>
__global__ void __launch_bounds__(LN_WARPS * 32)
    ln_fwd_kernel(float* out, const float* x, const float* g, const float* b, float eps,
                  float* invStd, float* xhat, int64_t rows, int64_t d) {
  MTKC_PDL_ENTRY();
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
  MTKC_PDL_ENTRY();
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
  MTKC_PDL_ENTRY();
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

// ---------------------------------------------------------------------------
// Vectorised path (d % 4 == 0, d <= 128*NV): no xhat tensor.  The forward
// caches only (mean, invStd) per row; the backward recomputes
// xhat = (x - mean) * invStd from the layer input (same float expression as
// the forward, so the same bits) and fuses the gain/bias column reductions
// into the dx pass: each CTA owns a block of rows, accumulates
// sum(dy*xhat) / sum(dy) per column in registers, combines its 8 warps in a
// fixed order and writes one partial row pair; colred_final_kernel<2> sums
// the partials in a fixed order.  HBM per element: forward 8 B (read x,
// write y), backward 12 B (read dy, x; write dx) instead of 12 B + 20 B.

template <int NV>
__global__ void __launch_bounds__(LN_WARPS * 32)
    ln_fwd4_kernel(float* out, const float* x, const float* g, const float* b, float eps,
                   float* mean, float* invStd, int64_t rows, int64_t d) {
  MTKC_PDL_ENTRY();
  const int64_t row = blockIdx.x * (int64_t)LN_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if(row >= rows)
    return;
  const float* xr = x + row * d;
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t c = 128 * k + 4 * lane;
    v[k] = c < d ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  s = warp_sum(s);
  const float mu = s / (float)d;
  float q = 0.f;
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t c = 128 * k + 4 * lane;
    if(c < d) {
      const float a = v[k].x - mu, bb = v[k].y - mu, cc = v[k].z - mu, dd = v[k].w - mu;
      q += (a * a + bb * bb) + (cc * cc + dd * dd);
    }
  }
  q = warp_sum(q);
  const float rs = 1.f / sqrtf(q / (float)d + eps);
  if(lane == 0) {
    mean[row] = mu;
    invStd[row] = rs;
  }
  float* o = out + row * d;
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t c = 128 * k + 4 * lane;
    if(c < d) {
      const float4 g4 = __ldg(reinterpret_cast<const float4*>(g + c));
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(b + c));
      float4 y;
      y.x = g4.x * ((v[k].x - mu) * rs) + b4.x;
      y.y = g4.y * ((v[k].y - mu) * rs) + b4.y;
      y.z = g4.z * ((v[k].z - mu) * rs) + b4.z;
      y.w = g4.w * ((v[k].w - mu) * rs) + b4.w;
      *reinterpret_cast<float4*>(o + c) = y;
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(LN_WARPS * 32)
    ln_bwd4_kernel(const float* dy, const float* x, const float* g, const float* mean,
                   const float* invStd, float* dx, float* part, int64_t rows, int64_t d,
                   int64_t rowsPerCta, int accDx) {
  MTKC_PDL_ENTRY();
  extern __shared__ float4 red4[];  // [LN_WARPS][2][d/4] (param partials only)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4 gg[NV], sg[NV], sb[NV];
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t c = 128 * k + 4 * lane;
    gg[k] = c < d ? __ldg(reinterpret_cast<const float4*>(g + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    sg[k] = sb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int64_t r0 = blockIdx.x * rowsPerCta, r1 = min(rows, r0 + rowsPerCta);
  // one row per warp iteration; every load of the row (dy, x, and the dx
  // being accumulated into) is issued before the first reduction, so a row
  // costs one memory round trip
  for(int64_t row = r0 + w; row < r1; row += LN_WARPS) {
    float4 dy4[NV], xh[NV], prev[NV];
    const float mu = mean[row], rs = invStd[row];
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t c = 128 * k + 4 * lane;
      dy4[k] = xh[k] = prev[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if(c < d) {
        dy4[k] = *reinterpret_cast<const float4*>(dy + row * d + c);
        xh[k] = *reinterpret_cast<const float4*>(x + row * d + c);
        if(accDx)
          prev[k] = *reinterpret_cast<const float4*>(dx + row * d + c);
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t c = 128 * k + 4 * lane;
      if(c < d) {
        const float4 x4 = xh[k];
        xh[k] = make_float4((x4.x - mu) * rs, (x4.y - mu) * rs, (x4.z - mu) * rs, (x4.w - mu) * rs);
      }
      const float4 d4v = dy4[k];
      const float4 h = make_float4(d4v.x * gg[k].x, d4v.y * gg[k].y, d4v.z * gg[k].z,
                                   d4v.w * gg[k].w);
      s1 += (h.x + h.y) + (h.z + h.w);
      s2 += (h.x * xh[k].x + h.y * xh[k].y) + (h.z * xh[k].z + h.w * xh[k].w);
      sg[k].x += d4v.x * xh[k].x;
      sg[k].y += d4v.y * xh[k].y;
      sg[k].z += d4v.z * xh[k].z;
      sg[k].w += d4v.w * xh[k].w;
      f4add(sb[k], d4v);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const float m1 = s1 / (float)d, m2 = s2 / (float)d;
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t c = 128 * k + 4 * lane;
      if(c < d) {
        const float4 d4v = dy4[k];
        float4 o;
        o.x = rs * (d4v.x * gg[k].x - m1 - xh[k].x * m2);
        o.y = rs * (d4v.y * gg[k].y - m1 - xh[k].y * m2);
        o.z = rs * (d4v.z * gg[k].z - m1 - xh[k].z * m2);
        o.w = rs * (d4v.w * gg[k].w - m1 - xh[k].w * m2);
        if(accDx)
          f4add(o, prev[k]);
        *reinterpret_cast<float4*>(dx + row * d + c) = o;
      }
    }
  }
  if(!part)
    return;
  const int64_t d4 = d / 4;
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t c4 = 32 * k + lane;
    if(c4 < d4) {
      red4[(w * 2 + 0) * d4 + c4] = sg[k];
      red4[(w * 2 + 1) * d4 + c4] = sb[k];
    }
  }
  __syncthreads();
  for(int64_t e = threadIdx.x; e < 2 * d4; e += LN_WARPS * 32) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for(int ww = 0; ww < LN_WARPS; ++ww)
      f4add(t, red4[ww * 2 * d4 + e]);
    reinterpret_cast<float4*>(part)[blockIdx.x * 2 * d4 + e] = t;  // [blk][q][d]
  }
}

// Same backward, rows staged through shared memory with cp.async: each warp
// keeps row i+1's dy / x / dx in flight (LNS stages) while it reduces row i,
// so the rows in flight per SM are not bounded by the register file.  Each
// lane copies and later reads back only its own 16-byte chunks (no warp
// barrier needed); arithmetic identical to ln_bwd4_kernel.
constexpr int LNS = 2;
template <int NV>
__global__ void __launch_bounds__(LN_WARPS * 32)
    ln_bwd4_async_kernel(const float* dy, const float* x, const float* g, const float* mean,
                         const float* invStd, float* dx, float* part, int64_t rows, int64_t d,
                         int64_t rowsPerCta, int accDx) {
  MTKC_PDL_ENTRY();
  extern __shared__ float4 sm4[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // [LN_WARPS][LNS][3][NV*32] float4 row stages; after the row loop the
  // same space holds the partials [LN_WARPS][2][d/4]
  float4* stg = sm4 + (size_t)w * LNS * 3 * NV * 32;
  float4* red4 = sm4;
  float4 gg[NV], sg[NV], sb[NV];
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t c = 128 * k + 4 * lane;
    gg[k] = c < d ? __ldg(reinterpret_cast<const float4*>(g + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    sg[k] = sb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int64_t r0 = blockIdx.x * rowsPerCta, r1 = min(rows, r0 + rowsPerCta);
  auto issue = [&](int64_t row, int st) {
    float4* b = stg + st * 3 * NV * 32;
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t c = 128 * k + 4 * lane;
      if(c < d) {
        const uint32_t o = (uint32_t)__cvta_generic_to_shared(b + k * 32 + lane);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(o), "l"(dy + row * d + c)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(o + NV * 32 * 16),
                     "l"(x + row * d + c)
                     : "memory");
        if(accDx)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(o + 2 * NV * 32 * 16),
                       "l"(dx + row * d + c)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int it = 0;
  // the row statistics travel one row ahead with the staged rows (a load at
  // use would put an L2 round trip in front of every row)
  float muN = 0.f, rsN = 0.f;
  if(r0 + w < r1) {
    issue(r0 + w, 0);
    muN = __ldg(mean + r0 + w);
    rsN = __ldg(invStd + r0 + w);
  }
  for(int64_t row = r0 + w; row < r1; row += LN_WARPS, ++it) {
    const int st = it % LNS;
    const float mu = muN, rs = rsN;
    if(row + LN_WARPS < r1) {
      issue(row + LN_WARPS, (it + 1) % LNS);
      muN = __ldg(mean + row + LN_WARPS);
      rsN = __ldg(invStd + row + LN_WARPS);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    const float4* b = stg + st * 3 * NV * 32;
    float4 dy4[NV], xh[NV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t c = 128 * k + 4 * lane;
      dy4[k] = xh[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if(c < d) {
        dy4[k] = b[k * 32 + lane];
        const float4 x4 = b[NV * 32 + k * 32 + lane];
        xh[k] = make_float4((x4.x - mu) * rs, (x4.y - mu) * rs, (x4.z - mu) * rs, (x4.w - mu) * rs);
      }
      const float4 d4v = dy4[k];
      const float4 h = make_float4(d4v.x * gg[k].x, d4v.y * gg[k].y, d4v.z * gg[k].z,
                                   d4v.w * gg[k].w);
      s1 += (h.x + h.y) + (h.z + h.w);
      s2 += (h.x * xh[k].x + h.y * xh[k].y) + (h.z * xh[k].z + h.w * xh[k].w);
      sg[k].x += d4v.x * xh[k].x;
      sg[k].y += d4v.y * xh[k].y;
      sg[k].z += d4v.z * xh[k].z;
      sg[k].w += d4v.w * xh[k].w;
      f4add(sb[k], d4v);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const float m1 = s1 / (float)d, m2 = s2 / (float)d;
#pragma unroll
    for(int k = 0; k < NV; ++k) {
      const int64_t c = 128 * k + 4 * lane;
      if(c < d) {
        const float4 d4v = dy4[k];
        float4 o;
        o.x = rs * (d4v.x * gg[k].x - m1 - xh[k].x * m2);
        o.y = rs * (d4v.y * gg[k].y - m1 - xh[k].y * m2);
        o.z = rs * (d4v.z * gg[k].z - m1 - xh[k].z * m2);
        o.w = rs * (d4v.w * gg[k].w - m1 - xh[k].w * m2);
        if(accDx)
          f4add(o, b[2 * NV * 32 + k * 32 + lane]);
        *reinterpret_cast<float4*>(dx + row * d + c) = o;
      }
    }
  }
  if(!part)
    return;
  __syncthreads();  // every warp is done with its stages
  const int64_t d4 = d / 4;
#pragma unroll
  for(int k = 0; k < NV; ++k) {
    const int64_t c4 = 32 * k + lane;
    if(c4 < d4) {
      red4[(w * 2 + 0) * d4 + c4] = sg[k];
      red4[(w * 2 + 1) * d4 + c4] = sb[k];
    }
  }
  __syncthreads();
  for(int64_t e = threadIdx.x; e < 2 * d4; e += LN_WARPS * 32) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for(int ww = 0; ww < LN_WARPS; ++ww)
      f4add(t, red4[ww * 2 * d4 + e]);
    reinterpret_cast<float4*>(part)[blockIdx.x * 2 * d4 + e] = t;  // [blk][q][d]
  }
}

// Several independent two-quantity reductions in one launch: blockIdx.y picks
// the job, each job summed exactly as colred_final_kernel<2> would (same
// lane split, same order), so the deferred result is bit-identical.
struct ColredJob2 {
  float* out0;
  float* out1;
  const float* part;
  int64_t nblk, cols;
  int acc;
};
constexpr int COLRED_MAX_JOBS = 32;
struct ColredJobs2 {
  ColredJob2 j[COLRED_MAX_JOBS];
};

__global__ void __launch_bounds__(256) colred_final_many_kernel(const __grid_constant__ ColredJobs2 jobs) {
  MTKC_PDL_ENTRY();
  const ColredJob2& jb = jobs.j[blockIdx.y];
  __shared__ float red[8][2][32];
  const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + cx;
  if((int64_t)blockIdx.x * 32 >= jb.cols)
    return;  // whole block past this job's columns (uniform)
  float s[2] = {0.f, 0.f};
  if(c < jb.cols) {
    for(int64_t rb = ry; rb < jb.nblk; rb += 64) {
      float v[8][2];
#pragma unroll
      for(int u = 0; u < 8; ++u)
#pragma unroll
        for(int q = 0; q < 2; ++q)
          v[u][q] = rb + 8 * u < jb.nblk ? __ldcg(jb.part + ((rb + 8 * u) * 2 + q) * jb.cols + c)
                                         : 0.f;
#pragma unroll
      for(int u = 0; u < 8; ++u)
#pragma unroll
        for(int q = 0; q < 2; ++q)
          s[q] += v[u][q];
    }
  }
#pragma unroll
  for(int q = 0; q < 2; ++q)
    red[ry][q][cx] = s[q];
  __syncthreads();
  if(ry == 0 && c < jb.cols) {
    float t[2];
#pragma unroll
    for(int q = 0; q < 2; ++q) {
      t[q] = 0.f;
#pragma unroll
      for(int k = 0; k < 8; ++k)
        t[q] += red[k][q][cx];
    }
    jb.out0[c] = (jb.acc ? jb.out0[c] : 0.f) + t[0];
    jb.out1[c] = (jb.acc ? jb.out1[c] : 0.f) + t[1];
  }
}

template <template <int> class K, typename... Args>
void launch_v(int64_t d, dim3 grid, cudaStream_t st, Args... args);

#define LN_DISPATCH(KERNEL, ...)                                             \
  do {                                                                       \
    int v_ = (int)cdiv(d, 32);                                               \
    if(v_ <= 1)                                                              \
      ::mtkc::launch(KERNEL<1>, grid, LN_WARPS * 32, 0, st, __VA_ARGS__);                \
    else if(v_ <= 2)                                                         \
      ::mtkc::launch(KERNEL<2>, grid, LN_WARPS * 32, 0, st, __VA_ARGS__);                \
    else if(v_ <= 4)                                                         \
      ::mtkc::launch(KERNEL<4>, grid, LN_WARPS * 32, 0, st, __VA_ARGS__);                \
    else if(v_ <= 8)                                                         \
      ::mtkc::launch(KERNEL<8>, grid, LN_WARPS * 32, 0, st, __VA_ARGS__);                \
    else if(v_ <= 16)                                                        \
      ::mtkc::launch(KERNEL<16>, grid, LN_WARPS * 32, 0, st, __VA_ARGS__);               \
    else if(v_ <= 32)                                                        \
      ::mtkc::launch(KERNEL<32>, grid, LN_WARPS * 32, 0, st, __VA_ARGS__);               \
    else                                                                     \
      ::mtkc::launch(KERNEL<0>, grid, LN_WARPS * 32, 0, st, __VA_ARGS__);                \
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
    ::mtkc::launch(colred_partial_kernel<2>, dim3((unsigned)cdiv(d, CR_COLS), (unsigned)nblk), 256, 0, st, 
        workspace, dy, xhat, rows, d);
    MTKC_POST_LAUNCH("colred_partial_kernel");
    ::mtkc::launch(colred_final_kernel<2>, colred_final_grid(d), 256, 0, st, dgain, dbias, workspace, nblk,
                                                                  d, accumulate_params);
    MTKC_POST_LAUNCH("colred_final_kernel");
  } else {
    ::mtkc::launch(ln_param_direct_kernel, (unsigned)cdiv(d, 128), 128, 0, st, dy, xhat, dgain, dbias, rows,
                                                                   d, accumulate_params);
    MTKC_POST_LAUNCH("ln_param_direct_kernel");
  }
  return MTKC_OK;
}

int mtkc_layernorm_fast_supported(int64_t d) { return d >= 4 && d % 4 == 0 && d <= 1024; }

int mtkc_layernorm_stats(float* out, const float* x, const float* gain, const float* bias,
                         float eps, float* mean, float* inv_std, int64_t rows, int64_t d,
                         void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  if(!mtkc_layernorm_fast_supported(d) || ((uintptr_t)x | (uintptr_t)out | (uintptr_t)gain |
                                           (uintptr_t)bias) % 16)
    return fail(MTKC_DIMENSION, "mtkc_layernorm_stats needs d % 4 == 0, d <= 1024, aligned rows");
  cudaStream_t st = S(stream);
  ProfScope prof(st, "layernorm", 8.0 * rows * d);  // read x, write y
  if(prof_detail())
    prof.detail = "fwd4_r" + std::to_string(rows) + "_d" + std::to_string(d);
  dim3 grid((unsigned)cdiv(rows, LN_WARPS));
  const int nv = (int)cdiv(d, 128);
#define LN4_FWD(NVV)                                                                   \
  if(nv <= NVV) {                                                                      \
    ::mtkc::launch(ln_fwd4_kernel<NVV>, grid, LN_WARPS * 32, 0, st, out, x, gain, bias, eps, mean, \
                                                        inv_std, rows, d);              \
  } else
  LN4_FWD(1) LN4_FWD(2) LN4_FWD(4) LN4_FWD(8) {}
#undef LN4_FWD
  MTKC_POST_LAUNCH("ln_fwd4_kernel");
  return MTKC_OK;
}

size_t mtkc_layernorm_stats_workspace_bytes(int64_t rows, int64_t d) {
  int64_t rpc = std::max<int64_t>(LN_WARPS, cdiv(cdiv(rows, 2 * 148), LN_WARPS) * LN_WARPS);
  return (size_t)cdiv(rows, rpc) * 2 * (size_t)d * sizeof(float);
}

int mtkc_layernorm_stats_backward(const float* dy, const float* x, const float* gain,
                                  const float* mean, const float* inv_std, float* dx,
                                  float* dgain, float* dbias, int64_t rows, int64_t d,
                                  int accumulate_dx, int accumulate_params, float* workspace,
                                  size_t workspace_bytes, void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  if(!mtkc_layernorm_fast_supported(d) ||
     ((uintptr_t)x | (uintptr_t)dy | (uintptr_t)dx | (uintptr_t)gain) % 16)
    return fail(MTKC_DIMENSION, "mtkc_layernorm_stats_backward needs d % 4 == 0, d <= 1024");
  cudaStream_t st = S(stream);
  ProfScope prof(st, "layernorm", 12.0 * rows * d);  // read dy, x; write dx
  if(prof_detail())
    prof.detail = "bwd4_r" + std::to_string(rows) + "_d" + std::to_string(d);
  // about two CTAs per SM, rows per CTA a multiple of the warp count
  const int64_t rpc = std::max<int64_t>(LN_WARPS, cdiv(cdiv(rows, 2 * 148), LN_WARPS) * LN_WARPS);
  const int64_t nblk = cdiv(rows, rpc);
  float* part = nullptr;
  if(dgain) {
    if(!workspace || workspace_bytes < (size_t)nblk * 2 * (size_t)d * sizeof(float))
      return fail(MTKC_CONTRACT, "layer norm backward workspace too small");
    part = workspace;
  }
  const size_t smem = part ? (size_t)LN_WARPS * 2 * (size_t)d * sizeof(float) : 0;
  const int nv = (int)cdiv(d, 128);
#define LN4_BWD(NVV)                                                                         \
  if(nv <= NVV) {                                                                            \
    if(smem > 48 * 1024)                                                                     \
      cudaFuncSetAttribute(ln_bwd4_kernel<NVV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                       \
    ::mtkc::launch(ln_bwd4_kernel<NVV>, (unsigned)nblk, LN_WARPS * 32, smem, st,                         \
        dy, x, gain, mean, inv_std, dx, part, rows, d, rpc, accumulate_dx);                  \
  } else
  static const bool async = !getenv("MTK_LN_SYNC");
  if(async && nv <= 4) {
    const size_t smemA = 0;
#define LN4_BWDA(NVV)                                                                         \
  if(nv <= NVV) {                                                                             \
    const size_t sm = std::max((size_t)LN_WARPS * LNS * 3 * NVV * 32 * 16,                     \
                               part ? (size_t)LN_WARPS * 2 * d * 4 : (size_t)0);              \
    if(sm > 48 * 1024)                                                                        \
      cudaFuncSetAttribute(ln_bwd4_async_kernel<NVV>,                                         \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);             \
    ::mtkc::launch(ln_bwd4_async_kernel<NVV>, (unsigned)nblk, LN_WARPS * 32, sm, st, dy, x,     \
                   gain, mean, inv_std, dx, part, rows, d, rpc, accumulate_dx);               \
  } else
    LN4_BWDA(1) LN4_BWDA(2) LN4_BWDA(4) {}
#undef LN4_BWDA
    (void)smemA;
  } else
  LN4_BWD(1) LN4_BWD(2) LN4_BWD(4) LN4_BWD(8) {}
#undef LN4_BWD
  MTKC_POST_LAUNCH("ln_bwd4_kernel");
  if(part && !(accumulate_params & MTKC_LN_DEFER_PARAMS)) {
    ::mtkc::launch(colred_final_kernel<2>, colred_final_grid(d), 256, 0, st, dgain, dbias, part, nblk, d,
                                                                  accumulate_params);
    MTKC_POST_LAUNCH("colred_final_kernel");
  }
  return MTKC_OK;
}

int64_t mtkc_layernorm_stats_partial_blocks(int64_t rows) {
  if(rows <= 0)
    return 0;
  const int64_t rpc = std::max<int64_t>(LN_WARPS, cdiv(cdiv(rows, 2 * 148), LN_WARPS) * LN_WARPS);
  return cdiv(rows, rpc);
}

int mtkc_layernorm_param_reduce_many(const mtkc_ln_param_job* jobs, int n_jobs, void* stream) {
  if(n_jobs <= 0)
    return MTKC_OK;
  if(n_jobs > COLRED_MAX_JOBS)
    return fail(MTKC_CONTRACT, "mtkc_layernorm_param_reduce_many: at most 32 jobs per call");
  ColredJobs2 js{};
  int64_t maxCols = 0;
  for(int i = 0; i < n_jobs; ++i) {
    const mtkc_ln_param_job& j = jobs[i];
    if(!j.dgain || !j.dbias || !j.partials || j.d <= 0 || j.blocks <= 0)
      return fail(MTKC_CONTRACT, "mtkc_layernorm_param_reduce_many: empty job");
    js.j[i] = ColredJob2{j.dgain, j.dbias, j.partials, j.blocks, j.d, j.accumulate ? 1 : 0};
    maxCols = std::max(maxCols, j.d);
  }
  cudaStream_t st = S(stream);
  ::mtkc::launch(colred_final_many_kernel, dim3(colred_final_grid(maxCols), (unsigned)n_jobs), 256,
                 0, st, js);
  MTKC_POST_LAUNCH("colred_final_many_kernel");
  return MTKC_OK;
}

}  // extern "C"
