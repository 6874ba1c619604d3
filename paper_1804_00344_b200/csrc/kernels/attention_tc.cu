// Tensor-core (mma.sync tf32) scaled dot-product attention for the short
// sentences of every BASELINE config (tq, tk <= 64, head dim 64): the TF32
// counterpart of the FP32 padded-tile kernels in attention.cu, selected by
// the host in TF32 precision mode (the same mode that runs the projections on
// tcgen05 kind::tf32).  Same node semantics as MultiHeadAttention::apply
// (layers.cpp:89-126): scores = scale * q k^T per head, masked softmax over
// keys (key mask [b, tk] + causal rule j > tk - tq + i, layers.cpp:115-116),
// context = P v; probabilities P are saved for the backward pass
// (softmax backward graph.cpp:538-553 fused with the two dot backwards).
//
// One CTA per (head, batch row), TT/16 warps.  Operands are staged into
// padded shared-memory tiles with cp.async (zero-filled past tq/tk) and every
// product is a chain of m16n8k8 tf32 MMAs with fp32 accumulation; softmax row
// reductions stay inside the 4-lane quads of the accumulator layout.  The
// kernels are HBM-bound: per (row, head) the forward reads q, k, v and writes
// context + P, the backward reads q, k, v, dO, P and writes dq, dk, dv.
#include "common.cuh"

using namespace mtkc;

namespace {

constexpr int DKT = 64;  // head dim handled here

// fp32 -> tf32, round to nearest (ties away) on the 13 dropped mantissa bits:
// two integer ops instead of the multi-instruction cvt.rna.tf32 sequence.
// Operands here are finite (masked scores never enter an MMA).
__device__ __forceinline__ uint32_t tf32(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
}

// D = A(16x8, row) * B(8x8, col) + D, tf32 in / fp32 accumulate.
// Fragments (g = lane/4, t = lane%4): a0 (g,t) a1 (g+8,t) a2 (g,t+4)
// a3 (g+8,t+4); b0 (k=t,n=g) b1 (k=t+4,n=g); c0 (g,2t) c1 (g,2t+1)
// c2 (g+8,2t) c3 (g+8,2t+1).
__device__ __forceinline__ void mma8(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                     uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  int n = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// rows x 64 floats (row stride ld) -> smem [TT][LD], rows >= rows zero-filled;
// NTH threads (2*TT or 4*TT) move 16*TT 16-byte chunks: 16*TT/NTH per thread
template <int TT, int LD, int NTH = 2 * TT>
__device__ __forceinline__ void stage(float* dst, const float* src, int64_t ld, int rows) {
  const int c4 = threadIdx.x & 15, rb = threadIdx.x >> 4;
#pragma unroll
  for(int i = 0; i < 16 * TT / NTH; ++i) {
    const int r = rb + i * (NTH / 16);
    const float* s = src + (int64_t)(r < rows ? r : 0) * ld + c4 * 4;
    cp_async16(dst + r * LD + c4 * 4, s, r < rows);
  }
}

struct TcAttP {
  float* out;
  int64_t ldo;
  float* probs;
  const float* q;
  int64_t ldq;
  const float* k;
  const float* v;
  int64_t ldk;
  const float* mask;
  int tq, tk, heads;
  float scale;
  int causal;
  int* flags;
  // varlen (packed rows): sentence bi's queries are rows qoff[bi] ..
  // qoff[bi+1]-1, its keys koff[bi] .. koff[bi+1]-1; tq / tk are the maxima
  // (the probability tensor keeps the padded [b, heads, tq, tk] layout)
  const int* qoff;
  const int* koff;
  const int* sid;  // sentence of CTA row blockIdx.y (length-bucketed launches), or NULL
};

struct TcAttBP {
  const float* gout;
  int64_t ldo;
  const float* probs;
  const float* q;
  int64_t ldq;
  const float* k;
  const float* v;
  int64_t ldk;
  float* gq;
  float* gk;
  float* gv;
  int tq, tk, heads;
  float scale;
  int accQ, accK, accV;
  float* colpart;  // optional [3][b][heads*64]: column sums of this CTA's dq/dk/dv
  const int* qoff;  // varlen, as in TcAttP
  const int* koff;
  const int* sid;
};

// strides (floats): L4 = 4*odd mod 32 for row-fragment reads (g*L + t),
// L8 = 8*odd mod 32 for transposed reads (t*L + g)
constexpr int L4 = DKT + 4;  // 68
constexpr int L8 = DKT + 8;  // 72
template <int TT>
struct PStride {
  static constexpr int v = TT + 8;  // 24, 40, 56, 72: 8*odd mod 32
};

template <int TT>
constexpr size_t fwd_smem() {
  return sizeof(float) * ((size_t)TT * L4 * 2 + (size_t)TT * L8 + 5 * TT);
}
// backward: V's region is reused for dS once phase 1 is done
template <int TT>
constexpr int bwd_vs() {
  return TT * L4 > TT * PStride<TT>::v ? TT * L4 : TT * PStride<TT>::v;
}
template <int TT>
constexpr size_t bwd_smem() {
  return sizeof(float) * ((size_t)TT * L8 * 2 + (size_t)bwd_vs<TT>() + (size_t)TT * L4 +
                          (size_t)TT * PStride<TT>::v + 2 * TT + 3 * (TT / 16) * DKT);
}

// column sums of a warp's 16 x 8*NJ accumulator tile: sum rows (g, g+8) of
// each lane, then across the 8 lanes sharing t; lanes with g == 0 hold the
// totals of columns jd*8 + 2t + {0,1}
template <int NJ>
__device__ __forceinline__ void tile_colsum(const float (&o)[NJ][4], float* dst, int g, int t) {
#pragma unroll
  for(int jd = 0; jd < NJ; ++jd)
#pragma unroll
    for(int e = 0; e < 2; ++e) {
      float v = o[jd][e] + o[jd][2 + e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if(g == 0)
        dst[jd * 8 + 2 * t + e] = v;
    }
}

// Two warps per 16-row block (4*TT threads): the pair splits the keys of
// S = Q K^T (row max / sum exchanged through shared memory) and the 64
// output columns of O = P V.
template <int TT>
__global__ void __launch_bounds__(TT * 4) attn_tc_fwd_kernel(TcAttP p) {
  MTKC_PDL_ENTRY();
  constexpr int NT = TT / 8, NH = NT / 2, NTH = TT * 4, NWB = TT / 16, NJ = DKT / 16;
  extern __shared__ float4 smem4[];
  float* Q = reinterpret_cast<float*>(smem4);  // [TT][L4], later P
  float* K = Q + TT * L4;                       // [TT][L4]
  float* V = K + TT * L4;                       // [TT][L8]
  float* mk = V + TT * L8;                      // [TT] key usable (mask)
  float* xch = mk + TT;                         // [2][2][TT] row max / row sum per key half
  const int h = blockIdx.x, bi = p.sid ? p.sid[blockIdx.y] : (int)blockIdx.y;
  int tq = p.tq, tk = p.tk;
  int64_t qb = (int64_t)bi * tq, kb = (int64_t)bi * tk;  // first query / key row
  if(p.qoff) {
    qb = p.qoff[bi];
    tq = p.qoff[bi + 1] - (int)qb;
    kb = p.koff[bi];
    tk = p.koff[bi + 1] - (int)kb;
  }
  const int hoff = h * DKT;
  stage<TT, L4, NTH>(Q, p.q + qb * p.ldq + hoff, p.ldq, tq);
  stage<TT, L4, NTH>(K, p.k + kb * p.ldk + hoff, p.ldk, tk);
  stage<TT, L8, NTH>(V, p.v + kb * p.ldk + hoff, p.ldk, tk);
  for(int j = threadIdx.x; j < TT; j += NTH)
    mk[j] = (j < tk && (!p.mask || p.mask[(int64_t)bi * tk + j] != 0.f)) ? 1.f : 0.f;
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rbk = warp % NWB, half = warp / NWB;
  const int m0 = rbk * 16;
  const bool live = m0 < tq;  // uniform per row block (both warps of the pair)

  // S = Q K^T over this warp's key half (16 x 8*NH)
  float s[NH][4];
#pragma unroll
  for(int j = 0; j < NH; ++j)
    s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
  const float* Qr0 = Q + (m0 + g) * L4;
  const float* Qr1 = Qr0 + 8 * L4;
  if(live) {
#pragma unroll
    for(int kk = 0; kk < DKT / 8; ++kk) {
      const int c = kk * 8 + t;
      uint32_t a0 = tf32(Qr0[c]), a1 = tf32(Qr1[c]), a2 = tf32(Qr0[c + 4]),
               a3 = tf32(Qr1[c + 4]);
#pragma unroll
      for(int j = 0; j < NH; ++j) {  // padded keys are zero rows: no guards
        const float* Kr = K + ((half * NH + j) * 8 + g) * L4 + c;
        mma8(s[j], a0, a1, a2, a3, tf32(Kr[0]), tf32(Kr[4]));
      }
    }
  }

  // masked softmax over each query row (rows r0 = m0+g, r1 = m0+g+8)
  const int r0 = m0 + g, r1 = r0 + 8;
  const int lim0 = p.causal ? tk - tq + r0 : tk - 1;  // last usable key
  const int lim1 = p.causal ? tk - tq + r1 : tk - 1;
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for(int j = 0; j < NH; ++j) {
#pragma unroll
    for(int e = 0; e < 2; ++e) {
      const int c = (half * NH + j) * 8 + 2 * t + e;
      const bool ok = mk[c] != 0.f;  // 0 past tk
      s[j][e] = (ok && c <= lim0) ? p.scale * s[j][e] : -INFINITY;
      s[j][2 + e] = (ok && c <= lim1) ? p.scale * s[j][2 + e] : -INFINITY;
      mx0 = fmaxf(mx0, s[j][e]);
      mx1 = fmaxf(mx1, s[j][2 + e]);
    }
  }
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  if(t == 0) {
    xch[half * TT + r0] = mx0;
    xch[half * TT + r1] = mx1;
  }
  __syncthreads();
  mx0 = fmaxf(xch[r0], xch[TT + r0]);
  mx1 = fmaxf(xch[r1], xch[TT + r1]);
  float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
  for(int j = 0; j < NH; ++j)
#pragma unroll
    for(int e = 0; e < 2; ++e) {
      s[j][e] = s[j][e] == -INFINITY ? 0.f : __expf(s[j][e] - mx0);
      s[j][2 + e] = s[j][2 + e] == -INFINITY ? 0.f : __expf(s[j][2 + e] - mx1);
      sum0 += s[j][e];
      sum1 += s[j][2 + e];
    }
  sum0 += __shfl_xor_sync(0xffffffffu, sum0, 1);
  sum0 += __shfl_xor_sync(0xffffffffu, sum0, 2);
  sum1 += __shfl_xor_sync(0xffffffffu, sum1, 1);
  sum1 += __shfl_xor_sync(0xffffffffu, sum1, 2);
  if(t == 0) {
    xch[2 * TT + half * TT + r0] = sum0;
    xch[2 * TT + half * TT + r1] = sum1;
  }
  __syncthreads();  // also: every read of Q is done, P may overwrite it
  sum0 = xch[2 * TT + r0] + xch[3 * TT + r0];
  sum1 = xch[2 * TT + r1] + xch[3 * TT + r1];
  const bool any0 = mx0 != -INFINITY, any1 = mx1 != -INFINITY;
  if(live && half == 0 && t == 0 && p.flags && ((r0 < tq && !any0) || (r1 < tq && !any1)))
    atomicOr(p.flags, MTKC_FLAG_MASKED_ROW);

  const float inv0 = any0 ? 1.f / sum0 : 0.f, inv1 = any1 ? 1.f / sum1 : 0.f;
  float* P0 = Q + r0 * L4;
  float* P1 = Q + r1 * L4;
#pragma unroll
  for(int j = 0; j < NH; ++j) {
    const int c = (half * NH + j) * 8 + 2 * t;
    *reinterpret_cast<float2*>(P0 + c) = make_float2(s[j][0] * inv0, s[j][1] * inv0);
    *reinterpret_cast<float2*>(P1 + c) = make_float2(s[j][2] * inv1, s[j][3] * inv1);
  }
  __syncthreads();
  if(!live)
    return;
  // probabilities to HBM: this warp's 8 rows of the block's [16 x tk] slice
  {
    const int rows = min(8, tq - m0 - half * 8);
    float* gP = p.probs + (((int64_t)bi * p.heads + h) * p.tq + m0 + half * 8) * p.tk;
    const float* Ps = Q + (m0 + half * 8) * L4;
#pragma unroll
    for(int r = 0; r < 8; ++r)
      if(r < rows) {
#pragma unroll
        for(int c = lane; c < TT; c += 32)
          if(c < tk)
            gP[r * p.tk + c] = Ps[r * L4 + c];
      }
  }
  // O = P V over this warp's 32 columns: keys outer, 4 output tiles inner
  float o[NJ][4];
#pragma unroll
  for(int jd = 0; jd < NJ; ++jd)
    o[jd][0] = o[jd][1] = o[jd][2] = o[jd][3] = 0.f;
#pragma unroll
  for(int kk = 0; kk < NT; ++kk) {
    const int c = kk * 8 + t;
    const uint32_t a0 = tf32(P0[c]), a1 = tf32(P1[c]), a2 = tf32(P0[c + 4]), a3 = tf32(P1[c + 4]);
    const float* Vr = V + c * L8 + half * 32 + g;
#pragma unroll
    for(int jd = 0; jd < NJ; ++jd)
      mma8(o[jd], a0, a1, a2, a3, tf32(Vr[jd * 8]), tf32(Vr[jd * 8 + 4 * L8]));
  }
  float* out = p.out + qb * p.ldo + hoff + half * 32;
#pragma unroll
  for(int jd = 0; jd < NJ; ++jd) {
    const int col = jd * 8 + 2 * t;
    if(r0 < tq)
      *reinterpret_cast<float2*>(out + (int64_t)r0 * p.ldo + col) = make_float2(o[jd][0], o[jd][1]);
    if(r1 < tq)
      *reinterpret_cast<float2*>(out + (int64_t)r1 * p.ldo + col) = make_float2(o[jd][2], o[jd][3]);
  }
}

__device__ __forceinline__ void store2(float* d, float a, float b, int acc) {
  float2* p2 = reinterpret_cast<float2*>(d);
  if(acc) {
    float2 o = *p2;
    a += o.x;
    b += o.y;
  }
  *p2 = make_float2(a, b);
}

// Two warps per 16-row block (4*TT threads): the warp pair splits the keys
// of dP = dO V^T (exchanging the row sums D through shared memory) and the
// 64 output columns of dQ / dK / dV, so a CTA keeps twice the warps busy
// and V's smem is recycled for dS -- ~3x the resident warps per SM.
template <int TT>
__global__ void __launch_bounds__(TT * 4) attn_tc_bwd_kernel(TcAttBP p) {
  MTKC_PDL_ENTRY();
  constexpr int NT = TT / 8, NH = NT / 2, LP = PStride<TT>::v, NTH = TT * 4;
  constexpr int NWB = TT / 16, NJ = DKT / 16;  // row blocks; 8-col tiles per half
  extern __shared__ float4 smem4[];
  float* Q = reinterpret_cast<float*>(smem4);  // [TT][L8]
  float* K = Q + TT * L8;                       // [TT][L8]
  float* V = K + TT * L8;                       // [TT][L4], then dS [TT][LP]
  float* dS = V;
  float* dO = V + bwd_vs<TT>();                 // [TT][L4]
  float* P = dO + TT * L4;                      // [TT][LP]
  float* Dp = P + TT * LP;                      // [2][TT] row sums of dP*P per key half
  float* csum = Dp + 2 * TT;                    // [3][NWB][64] per-row-block column sums
  const int h = blockIdx.x, bi = p.sid ? p.sid[blockIdx.y] : (int)blockIdx.y;
  int tq = p.tq, tk = p.tk;
  int64_t qb = (int64_t)bi * tq, kb = (int64_t)bi * tk;
  if(p.qoff) {
    qb = p.qoff[bi];
    tq = p.qoff[bi + 1] - (int)qb;
    kb = p.koff[bi];
    tk = p.koff[bi + 1] - (int)kb;
  }
  const int hoff = h * DKT;
  stage<TT, L8, NTH>(Q, p.q + qb * p.ldq + hoff, p.ldq, tq);
  stage<TT, L8, NTH>(K, p.k + kb * p.ldk + hoff, p.ldk, tk);
  stage<TT, L4, NTH>(V, p.v + kb * p.ldk + hoff, p.ldk, tk);
  stage<TT, L4, NTH>(dO, p.gout + qb * p.ldo + hoff, p.ldo, tq);
  {
    const float* gP = p.probs + ((int64_t)bi * p.heads + h) * p.tq * p.tk;
    // thread covers column c = tid % TT of rows tid / TT + 4i
    const int c = threadIdx.x % TT, rb = threadIdx.x / TT;
#pragma unroll
    for(int i = 0; i < TT / 4; ++i) {
      const int r = rb + 4 * i;
      const bool ok = r < tq && c < tk;
      cp_async4(P + r * LP + c, gP + (ok ? r * p.tk + c : 0), ok);
    }
  }
  if(p.colpart)
    for(int e = threadIdx.x; e < 3 * NWB * DKT; e += NTH)
      csum[e] = 0.f;
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rbk = warp % NWB, half = warp / NWB;
  const int m0 = rbk * 16;
  const int r0 = m0 + g, r1 = r0 + 8;

  // phase 1 (query rows m0..m0+15, this warp's half of the keys):
  // dP = dO V^T, D = rowsum(dP*P) over both halves,
  // dS = scale * P * (dP - D)   (graph.cpp:539-552 with the MHA scale)
  float dp[NH][4];
#pragma unroll
  for(int j = 0; j < NH; ++j)
    dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
  if(m0 < tq) {
    const float* A0 = dO + r0 * L4;
    const float* A1 = A0 + 8 * L4;
#pragma unroll
    for(int kk = 0; kk < DKT / 8; ++kk) {
      const int c = kk * 8 + t;
      uint32_t a0 = tf32(A0[c]), a1 = tf32(A1[c]), a2 = tf32(A0[c + 4]), a3 = tf32(A1[c + 4]);
#pragma unroll
      for(int j = 0; j < NH; ++j) {
        const float* Vr = V + ((half * NH + j) * 8 + g) * L4 + c;
        mma8(dp[j], a0, a1, a2, a3, tf32(Vr[0]), tf32(Vr[4]));
      }
    }
  }
  {
    float D0 = 0.f, D1 = 0.f;
#pragma unroll
    for(int j = 0; j < NH; ++j) {
      const int c = (half * NH + j) * 8 + 2 * t;
      D0 += dp[j][0] * P[r0 * LP + c] + dp[j][1] * P[r0 * LP + c + 1];
      D1 += dp[j][2] * P[r1 * LP + c] + dp[j][3] * P[r1 * LP + c + 1];
    }
    D0 += __shfl_xor_sync(0xffffffffu, D0, 1);
    D0 += __shfl_xor_sync(0xffffffffu, D0, 2);
    D1 += __shfl_xor_sync(0xffffffffu, D1, 1);
    D1 += __shfl_xor_sync(0xffffffffu, D1, 2);
    if(t == 0) {
      Dp[half * TT + r0] = D0;
      Dp[half * TT + r1] = D1;
    }
  }
  __syncthreads();  // D halves exchanged; every read of V is done (dS reuses it)
  {
    const float D0 = Dp[r0] + Dp[TT + r0], D1 = Dp[r1] + Dp[TT + r1];
#pragma unroll
    for(int j = 0; j < NH; ++j) {
      const int c = (half * NH + j) * 8 + 2 * t;
#pragma unroll
      for(int e = 0; e < 2; ++e) {
        dS[r0 * LP + c + e] = p.scale * (P[r0 * LP + c + e] * (dp[j][e] - D0));
        dS[r1 * LP + c + e] = p.scale * (P[r1 * LP + c + e] * (dp[j][2 + e] - D1));
      }
    }
  }
  __syncthreads();

  // phase 2 (query rows, this warp's 32 columns): dQ = dS K
  if(m0 < tq) {
    const float* A0 = dS + r0 * LP;
    const float* A1 = A0 + 8 * LP;
    float o[NJ][4];
#pragma unroll
    for(int jd = 0; jd < NJ; ++jd)
      o[jd][0] = o[jd][1] = o[jd][2] = o[jd][3] = 0.f;
#pragma unroll
    for(int kk = 0; kk < NT; ++kk) {
      const int c = kk * 8 + t;
      const uint32_t a0 = tf32(A0[c]), a1 = tf32(A1[c]), a2 = tf32(A0[c + 4]),
                     a3 = tf32(A1[c + 4]);
      const float* Kr = K + c * L8 + half * 32 + g;
#pragma unroll
      for(int jd = 0; jd < NJ; ++jd)
        mma8(o[jd], a0, a1, a2, a3, tf32(Kr[jd * 8]), tf32(Kr[jd * 8 + 4 * L8]));
    }
    float* gq = p.gq + qb * p.ldq + hoff + half * 32;
#pragma unroll
    for(int jd = 0; jd < NJ; ++jd) {
      const int col = jd * 8 + 2 * t;
      if(r0 < tq)
        store2(gq + (int64_t)r0 * p.ldq + col, o[jd][0], o[jd][1], p.accQ);
      if(r1 < tq)
        store2(gq + (int64_t)r1 * p.ldq + col, o[jd][2], o[jd][3], p.accQ);
    }
    if(p.colpart)  // padded rows contribute exact zeros
      tile_colsum<NJ>(o, csum + (0 * NWB + rbk) * DKT + half * 32, g, t);
  }
  // phase 3 (key rows m0..m0+15, this warp's 32 columns): dK = dS^T Q, dV = P^T dO
  if(m0 < tk) {
    float ok[NJ][4], ov[NJ][4];
#pragma unroll
    for(int jd = 0; jd < NJ; ++jd) {
      ok[jd][0] = ok[jd][1] = ok[jd][2] = ok[jd][3] = 0.f;
      ov[jd][0] = ov[jd][1] = ov[jd][2] = ov[jd][3] = 0.f;
    }
#pragma unroll
    for(int kk = 0; kk < NT; ++kk) {
      const int q0 = kk * 8 + t;  // query index of a0/a1 (a2/a3: +4)
      const float* S0 = dS + q0 * LP + r0;
      const float* P0 = P + q0 * LP + r0;
      const uint32_t s0 = tf32(S0[0]), s1 = tf32(S0[8]), s2 = tf32(S0[4 * LP]),
                     s3 = tf32(S0[4 * LP + 8]);
      const uint32_t p0 = tf32(P0[0]), p1 = tf32(P0[8]), p2 = tf32(P0[4 * LP]),
                     p3 = tf32(P0[4 * LP + 8]);
      const float* Qr = Q + q0 * L8 + half * 32 + g;
      const float* Or = dO + q0 * L4 + half * 32 + g;
#pragma unroll
      for(int jd = 0; jd < NJ; ++jd) {
        mma8(ok[jd], s0, s1, s2, s3, tf32(Qr[jd * 8]), tf32(Qr[jd * 8 + 4 * L8]));
        mma8(ov[jd], p0, p1, p2, p3, tf32(Or[jd * 8]), tf32(Or[jd * 8 + 4 * L4]));
      }
    }
    float* gk = p.gk + kb * p.ldk + hoff + half * 32;
    float* gv = p.gv + kb * p.ldk + hoff + half * 32;
#pragma unroll
    for(int jd = 0; jd < NJ; ++jd) {
      const int col = jd * 8 + 2 * t;
      if(r0 < tk) {
        store2(gk + (int64_t)r0 * p.ldk + col, ok[jd][0], ok[jd][1], p.accK);
        store2(gv + (int64_t)r0 * p.ldk + col, ov[jd][0], ov[jd][1], p.accV);
      }
      if(r1 < tk) {
        store2(gk + (int64_t)r1 * p.ldk + col, ok[jd][2], ok[jd][3], p.accK);
        store2(gv + (int64_t)r1 * p.ldk + col, ov[jd][2], ov[jd][3], p.accV);
      }
    }
    if(p.colpart) {
      tile_colsum<NJ>(ok, csum + (1 * NWB + rbk) * DKT + half * 32, g, t);
      tile_colsum<NJ>(ov, csum + (2 * NWB + rbk) * DKT + half * 32, g, t);
    }
  }
  if(p.colpart) {  // this CTA's column sums, row blocks combined in fixed order
    __syncthreads();
    const int64_t hd = (int64_t)p.heads * DKT, B = gridDim.y;
    for(int e = threadIdx.x; e < 3 * DKT; e += NTH) {
      const int which = e / DKT, c = e % DKT;
      float v = 0.f;
#pragma unroll
      for(int w = 0; w < NWB; ++w)
        v += csum[(which * NWB + w) * DKT + c];
      p.colpart[((int64_t)which * B + bi) * hd + hoff + c] = v;
    }
  }
}

int tc_tile(int64_t tq, int64_t tk, int64_t dk, int64_t ldq, int64_t ldk, int64_t ldo,
            std::initializer_list<const void*> ptrs) {
  if(dk != DKT || (ldq | ldk | ldo) % 4)
    return 0;
  for(const void* q : ptrs)
    if(q && ((uintptr_t)q & 15))
      return 0;
  int64_t t = std::max(tq, tk);
  return t <= 16 ? 16 : t <= 32 ? 32 : t <= 48 ? 48 : t <= 64 ? 64 : 0;
}

int set_smem_attr(const void* fn, size_t bytes) {
  if(bytes <= 48 * 1024)
    return MTKC_OK;
  return cuda_status(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
      "cudaFuncSetAttribute(attention_tc)");
}

// varlen offsets of the current call (set by the _varlen entry points);
// with g_sid the launch covers g_nsent sentences whose longest sequence is
// g_tile (the tile size), not all b sentences
thread_local const int* g_qoff = nullptr;
thread_local const int* g_koff = nullptr;
thread_local const int* g_sid = nullptr;
thread_local int64_t g_nsent = 0, g_tile = 0;

}  // namespace

extern "C" {

int mtkc_attention_tc_supported(int64_t tq, int64_t tk, int64_t dk) {
  return tc_tile(tq, tk, dk, 4, 4, 4, {}) != 0;
}

int mtkc_attention_tc(float* out, int64_t ldo, float* probs, const float* q, int64_t ldq,
                      const float* k, const float* v, int64_t ldk, const float* key_mask,
                      int64_t b, int64_t tq, int64_t tk, int heads, int64_t dk, float scale,
                      int causal, int* flags, void* stream) {
  if(b <= 0 || tq <= 0 || tk <= 0)
    return MTKC_OK;
  int tt = g_sid ? tc_tile(g_tile, g_tile, dk, ldq, ldk, ldo, {out, q, k, v})
                 : tc_tile(tq, tk, dk, ldq, ldk, ldo, {out, q, k, v});
  if(!tt)
    return fail(MTKC_DIMENSION,
                "tensor-core attention needs head dim 64, tq/tk <= 64, 16-byte aligned rows");
  ProfScope prof(S(stream), "attention", 4.0 * b * heads * tq * tk * dk);
  if(prof_detail())
    prof.detail = "tcfwd_b" + std::to_string(b) + "_tq" + std::to_string(tq) + "_tk" +
                  std::to_string(tk);
  TcAttP p{out, ldo, probs, q, ldq, k, v, ldk, key_mask, (int)tq, (int)tk, heads, scale, causal,
           flags, g_qoff, g_koff, g_sid};
  dim3 grid((unsigned)heads, (unsigned)(g_sid ? g_nsent : b));
#define MTKC_TC_FWD(TTV)                                                          \
  if(tt == TTV) {                                                                 \
    size_t smem = fwd_smem<TTV>();                                                \
    if(int rc = set_smem_attr((const void*)attn_tc_fwd_kernel<TTV>, smem))        \
      return rc;                                                                  \
    ::mtkc::launch(attn_tc_fwd_kernel<TTV>, grid, TTV * 4, smem, S(stream), p);               \
  }
  MTKC_TC_FWD(16) MTKC_TC_FWD(32) MTKC_TC_FWD(48) MTKC_TC_FWD(64)
#undef MTKC_TC_FWD
  MTKC_POST_LAUNCH("attn_tc_fwd_kernel");
  return MTKC_OK;
}

int mtkc_attention_tc_backward(const float* gout, int64_t ldo, const float* probs,
                               const float* q, int64_t ldq, const float* k, const float* v,
                               int64_t ldk, float* gq, float* gk, float* gv, int64_t b,
                               int64_t tq, int64_t tk, int heads, int64_t dk, float scale,
                               int accumulate_q, int accumulate_k, int accumulate_v,
                               float* colpart, void* stream) {
  if(b <= 0 || tq <= 0 || tk <= 0)
    return MTKC_OK;
  int tt = g_sid ? tc_tile(g_tile, g_tile, dk, ldq, ldk, ldo, {gout, q, k, v, gq, gk, gv})
                 : tc_tile(tq, tk, dk, ldq, ldk, ldo, {gout, q, k, v, gq, gk, gv});
  if(!tt)
    return fail(MTKC_DIMENSION,
                "tensor-core attention needs head dim 64, tq/tk <= 64, 16-byte aligned rows");
  ProfScope prof(S(stream), "attention", 8.0 * b * heads * tq * tk * dk);
  if(prof_detail())
    prof.detail = "tcbwd_b" + std::to_string(b) + "_tq" + std::to_string(tq) + "_tk" +
                  std::to_string(tk);
  TcAttBP p{gout, ldo, probs, q, ldq, k, v, ldk, gq, gk, gv, (int)tq, (int)tk, heads, scale,
            accumulate_q, accumulate_k, accumulate_v, colpart, g_qoff, g_koff, g_sid};
  dim3 grid((unsigned)heads, (unsigned)(g_sid ? g_nsent : b));
#define MTKC_TC_BWD(TTV)                                                          \
  if(tt == TTV) {                                                                 \
    size_t smem = bwd_smem<TTV>();                                                \
    if(int rc = set_smem_attr((const void*)attn_tc_bwd_kernel<TTV>, smem))        \
      return rc;                                                                  \
    ::mtkc::launch(attn_tc_bwd_kernel<TTV>, grid, TTV * 4, smem, S(stream), p);               \
  }
  MTKC_TC_BWD(16) MTKC_TC_BWD(32) MTKC_TC_BWD(48) MTKC_TC_BWD(64)
#undef MTKC_TC_BWD
  MTKC_POST_LAUNCH("attn_tc_bwd_kernel");
  return MTKC_OK;
}

int mtkc_attention_tc_varlen(float* out, int64_t ldo, float* probs, const float* q, int64_t ldq,
                             const float* k, const float* v, int64_t ldk, const int32_t* qoff,
                             const int32_t* koff, int64_t b, int64_t tq_max, int64_t tk_max,
                             int heads, int64_t dk, float scale, int causal, int* flags,
                             void* stream) {
  g_qoff = qoff;
  g_koff = koff;
  int rc = mtkc_attention_tc(out, ldo, probs, q, ldq, k, v, ldk, nullptr, b, tq_max, tk_max,
                             heads, dk, scale, causal, flags, stream);
  g_qoff = g_koff = nullptr;
  return rc;
}

int mtkc_attention_tc_varlen_backward(const float* gout, int64_t ldo, const float* probs,
                                      const float* q, int64_t ldq, const float* k,
                                      const float* v, int64_t ldk, float* gq, float* gk,
                                      float* gv, const int32_t* qoff, const int32_t* koff,
                                      int64_t b, int64_t tq_max, int64_t tk_max, int heads,
                                      int64_t dk, float scale, int accumulate_q,
                                      int accumulate_k, int accumulate_v, void* stream) {
  g_qoff = qoff;
  g_koff = koff;
  int rc = mtkc_attention_tc_backward(gout, ldo, probs, q, ldq, k, v, ldk, gq, gk, gv, b,
                                      tq_max, tk_max, heads, dk, scale, accumulate_q,
                                      accumulate_k, accumulate_v, nullptr, stream);
  g_qoff = g_koff = nullptr;
  return rc;
}

int mtkc_attention_tc_varlen_ids(float* out, int64_t ldo, float* probs, const float* q,
                                 int64_t ldq, const float* k, const float* v, int64_t ldk,
                                 const int32_t* qoff, const int32_t* koff,
                                 const int32_t* sent_ids, int64_t n_sent, int64_t tile_len,
                                 int64_t b, int64_t tq_max, int64_t tk_max, int heads, int64_t dk,
                                 float scale, int causal, int* flags, void* stream) {
  g_sid = sent_ids;
  g_nsent = n_sent;
  g_tile = tile_len;
  int rc = n_sent > 0 ? mtkc_attention_tc_varlen(out, ldo, probs, q, ldq, k, v, ldk, qoff, koff,
                                                 b, tq_max, tk_max, heads, dk, scale, causal,
                                                 flags, stream)
                      : MTKC_OK;
  g_sid = nullptr;
  g_nsent = g_tile = 0;
  return rc;
}

int mtkc_attention_tc_varlen_ids_backward(
    const float* gout, int64_t ldo, const float* probs, const float* q, int64_t ldq,
    const float* k, const float* v, int64_t ldk, float* gq, float* gk, float* gv,
    const int32_t* qoff, const int32_t* koff, const int32_t* sent_ids, int64_t n_sent,
    int64_t tile_len, int64_t b, int64_t tq_max, int64_t tk_max, int heads, int64_t dk,
    float scale, int accumulate_q, int accumulate_k, int accumulate_v, void* stream) {
  g_sid = sent_ids;
  g_nsent = n_sent;
  g_tile = tile_len;
  int rc = n_sent > 0 ? mtkc_attention_tc_varlen_backward(
                            gout, ldo, probs, q, ldq, k, v, ldk, gq, gk, gv, qoff, koff, b,
                            tq_max, tk_max, heads, dk, scale, accumulate_q, accumulate_k,
                            accumulate_v, stream)
                      : MTKC_OK;
  g_sid = nullptr;
  g_nsent = g_tile = 0;
  return rc;
}

}  // extern "C"
