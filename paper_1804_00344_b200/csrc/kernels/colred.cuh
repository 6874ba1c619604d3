// Deterministic column reductions over a row-major [rows x cols] matrix:
//   out[c] (+)= sum_r f(r, c)
// Stage 1: CTAs tile (128-column chunk) x (CR_ROWS-row block); each of the
// 8 warps walks every 8th row of the block with float4 loads, then the
// warps combine in a fixed order in shared memory -> partial[rb][c].
// Stage 2: one thread per column sums the row-block partials in order.
// Used for bias gradients (colsum) and layer-norm gain/bias gradients.
#pragma once

#include "common.cuh"

namespace mtkc {

constexpr int CR_ROWS = 256;  // rows per stage-1 block
constexpr int CR_COLS = 128;  // columns per stage-1 block (32 lanes x float4)

// NQ quantities per column: Q=1 sum(a), Q=2 {sum(a*b), sum(a)}
template <int NQ>
__global__ void __launch_bounds__(256) colred_partial_kernel(float* part, const float* a,
                                                             const float* b, int64_t rows,
                                                             int64_t cols) {
  __shared__ float4 red[8][NQ][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * CR_COLS + lane * 4;
  const int64_t r0 = (int64_t)blockIdx.y * CR_ROWS;
  const int64_t r1 = min(rows, r0 + CR_ROWS);
  float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
  if(c < cols) {
    const bool vec = (cols % 4 == 0) && c + 3 < cols;
    for(int64_t r = r0 + w; r < r1; r += 8) {
      if(vec) {
        float4 x = *reinterpret_cast<const float4*>(a + r * cols + c);
        if(NQ == 2) {
          float4 y = *reinterpret_cast<const float4*>(b + r * cols + c);
          s0.x += x.x * y.x;
          s0.y += x.y * y.y;
          s0.z += x.z * y.z;
          s0.w += x.w * y.w;
          s1.x += x.x;
          s1.y += x.y;
          s1.z += x.z;
          s1.w += x.w;
        } else {
          s0.x += x.x;
          s0.y += x.y;
          s0.z += x.z;
          s0.w += x.w;
        }
      } else {
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
          s1.x += xs[0];
          s1.y += xs[1];
          s1.z += xs[2];
          s1.w += xs[3];
        } else {
          s0.x += xs[0];
          s0.y += xs[1];
          s0.z += xs[2];
          s0.w += xs[3];
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
    for(int k = 0; k < 8; ++k) {
      float4 v = red[k][w][lane];
      t.x += v.x;
      t.y += v.y;
      t.z += v.z;
      t.w += v.w;
    }
    float* dst = part + ((int64_t)blockIdx.y * NQ + w) * cols;
    float tv[4] = {t.x, t.y, t.z, t.w};
    for(int u = 0; u < 4; ++u)
      if(c + u < cols)
        dst[c + u] = tv[u];
  }
}

// out_q[c] (+)= sum_rb part[rb][q][c]
template <int NQ>
__global__ void colred_final_kernel(float* out0, float* out1, const float* part, int64_t nblk,
                                    int64_t cols, int acc) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if(c >= cols)
    return;
  float s[NQ];
  for(int q = 0; q < NQ; ++q)
    s[q] = 0.f;
  for(int64_t rb = 0; rb < nblk; ++rb)
    for(int q = 0; q < NQ; ++q)
      s[q] += part[(rb * NQ + q) * cols + c];
  out0[c] = (acc ? out0[c] : 0.f) + s[0];
  if(NQ == 2)
    out1[c] = (acc ? out1[c] : 0.f) + s[NQ - 1];
}

inline size_t colred_workspace_bytes(int nq, int64_t rows, int64_t cols) {
  return (size_t)cdiv(rows, CR_ROWS) * (size_t)nq * (size_t)cols * sizeof(float);
}

}  // namespace mtkc
