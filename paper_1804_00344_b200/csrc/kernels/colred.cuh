// Deterministic column reductions over a row-major [rows x cols] matrix:
//   out[c] (+)= sum_r f(r, c)
// Stage 1: CTAs tile (128-column chunk) x (CR_ROWS-row block); warp w owns
// rows r0 + w + 8i (i < CR_ROWS/8) and issues all of its float4 loads
// before summing them in row order (memory-level parallelism: ~8 loads in
// flight per thread, enough CTAs to cover all SMs several times); the 8
// warps then combine in a fixed order in shared memory -> partial[rb][c].
// Stage 2: 8 threads per column sum interleaved row-block partials in
// order, combined in a fixed order -> the result is bitwise run-to-run
// stable for a given shape.
// Used for bias gradients (colsum) and layer-norm gain/bias gradients.
#pragma once

#include "common.cuh"

namespace mtkc {

constexpr int CR_ROWS = 64;   // rows per stage-1 block
constexpr int CR_COLS = 128;  // columns per stage-1 block (32 lanes x float4)
constexpr int CR_RPW = CR_ROWS / 8;  // rows per warp

__device__ __forceinline__ void f4add(float4& s, const float4& x) {
  s.x += x.x;
  s.y += x.y;
  s.z += x.z;
  s.w += x.w;
}

// NQ quantities per column: Q=1 sum(a), Q=2 {sum(a*b), sum(a)}
template <int NQ>
__global__ void __launch_bounds__(256) colred_partial_kernel(float* part, const float* a,
                                                             const float* b, int64_t rows,
                                                             int64_t cols) {
  MTKC_PDL_ENTRY();
  __shared__ float4 red[8][NQ][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * CR_COLS + lane * 4;
  const int64_t r0 = (int64_t)blockIdx.y * CR_ROWS + w;
  float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
  if(c < cols) {
    const bool vec = (cols % 4 == 0) && c + 3 < cols;
    if(vec) {
      float4 xa[CR_RPW], xb[CR_RPW];
#pragma unroll
      for(int i = 0; i < CR_RPW; ++i) {
        const int64_t r = r0 + 8 * i;
        xa[i] = r < rows ? __ldg(reinterpret_cast<const float4*>(a + r * cols + c))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        if(NQ == 2)
          xb[i] = r < rows ? __ldg(reinterpret_cast<const float4*>(b + r * cols + c))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for(int i = 0; i < CR_RPW; ++i) {
        if(NQ == 2) {
          s0.x += xa[i].x * xb[i].x;
          s0.y += xa[i].y * xb[i].y;
          s0.z += xa[i].z * xb[i].z;
          s0.w += xa[i].w * xb[i].w;
          f4add(s1, xa[i]);
        } else {
          f4add(s0, xa[i]);
        }
      }
    } else {
      for(int i = 0; i < CR_RPW; ++i) {
        const int64_t r = r0 + 8 * i;
        if(r >= rows)
          break;
        float xs[4] = {0.f, 0.f, 0.f, 0.f}, ys[4] = {0.f, 0.f, 0.f, 0.f};
        for(int u = 0; u < 4; ++u)
          if(c + u < cols) {
            xs[u] = a[r * cols + c + u];
            if(NQ == 2)
              ys[u] = b[r * cols + c + u];
          }
        if(NQ == 2) {
          s0.x += xs[0] * ys[0];
          s0.y += xs[1] * ys[1];
          s0.z += xs[2] * ys[2];
          s0.w += xs[3] * ys[3];
          f4add(s1, make_float4(xs[0], xs[1], xs[2], xs[3]));
        } else {
          f4add(s0, make_float4(xs[0], xs[1], xs[2], xs[3]));
        }
      }
    }
  }
  red[w][0][lane] = s0;
  if(NQ == 2)
    red[w][NQ - 1][lane] = s1;
  __syncthreads();
  if(w < NQ && c < cols) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for(int k = 0; k < 8; ++k)
      f4add(t, red[k][w][lane]);
    float* dst = part + ((int64_t)blockIdx.y * NQ + w) * cols;
    if((cols % 4 == 0) && c + 3 < cols) {
      *reinterpret_cast<float4*>(dst + c) = t;
    } else {
      float tv[4] = {t.x, t.y, t.z, t.w};
      for(int u = 0; u < 4; ++u)
        if(c + u < cols)
          dst[c + u] = tv[u];
    }
  }
}

// out_q[c] (+)= sum_rb part[rb][q][c]; block = 32 columns x 8 row-block lanes.
// Lane ry sums row blocks ry, ry+8, ... in order, eight loads per quantity in
// flight per batch (the kernel is latency-bound: few CTAs, short rows).
template <int NQ>
__global__ void __launch_bounds__(256) colred_final_kernel(float* out0, float* out1,
                                                           const float* part, int64_t nblk,
                                                           int64_t cols, int acc) {
  MTKC_PDL_ENTRY();
  __shared__ float red[8][NQ][32];
  const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + cx;
  float s[NQ];
#pragma unroll
  for(int q = 0; q < NQ; ++q)
    s[q] = 0.f;
  if(c < cols) {
    for(int64_t rb = ry; rb < nblk; rb += 64) {
      float v[8][NQ];
#pragma unroll
      for(int u = 0; u < 8; ++u)
#pragma unroll
        for(int q = 0; q < NQ; ++q)
          v[u][q] = rb + 8 * u < nblk ? __ldcg(part + ((rb + 8 * u) * NQ + q) * cols + c) : 0.f;
#pragma unroll
      for(int u = 0; u < 8; ++u)
#pragma unroll
        for(int q = 0; q < NQ; ++q)
          s[q] += v[u][q];
    }
  }
#pragma unroll
  for(int q = 0; q < NQ; ++q)
    red[ry][q][cx] = s[q];
  __syncthreads();
  if(ry == 0 && c < cols) {
    float t[NQ];
#pragma unroll
    for(int q = 0; q < NQ; ++q) {
      t[q] = 0.f;
#pragma unroll
      for(int k = 0; k < 8; ++k)
        t[q] += red[k][q][cx];
    }
    out0[c] = (acc ? out0[c] : 0.f) + t[0];
    if(NQ == 2)
      out1[c] = (acc ? out1[c] : 0.f) + t[NQ - 1];
  }
}

inline size_t colred_workspace_bytes(int nq, int64_t rows, int64_t cols) {
  return (size_t)cdiv(rows, CR_ROWS) * (size_t)nq * (size_t)cols * sizeof(float);
}

inline unsigned colred_final_grid(int64_t cols) { return (unsigned)cdiv(cols, 32); }

}  // namespace mtkc
