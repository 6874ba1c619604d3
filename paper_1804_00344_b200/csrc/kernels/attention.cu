// Fused scaled dot-product multi-head attention core.
//
// Replaces the reference's node chain in MultiHeadAttention::apply
// (layers.cpp:89-126): splitHeads (reshape/transpose/reshape copies),
// dot(q, k^T), scale(1/sqrt(dk)), softmax with a host-built dense
// [b*h, tq, tk] mask (:108-118), dot(weights, v) and the merge transpose.
// Here heads are column slices of the projection outputs (no transposes),
// the mask is the [b, tk] key mask plus a causal flag, and probabilities are
// saved once for the backward pass.  Products are summed over the head dim
// and over keys in ascending order with separately rounded multiply/add
// (the reference's GEMM order, tensor.cpp:289-303), so scores and context
// match the unfused reference up to the softmax's exp/sum rounding.
#include "common.cuh"

using namespace mtkc;

namespace {

constexpr int QB = 32;      // query rows per CTA
constexpr int KC = 64;      // keys per staged chunk
constexpr int ATT_T = 128;  // threads
constexpr int MAX_TK = 512;
constexpr int MAX_DK = 128;

struct AttP {
  float* out;
  int64_t ldo;
  float* probs;
  const float* q;
  int64_t ldq;
  const float* k;
  const float* v;
  int64_t ldk;
  const float* mask;
  int64_t b, tq, tk;
  int heads;
  int64_t dk;
  float scale;
  int causal;
  int* flags;
};

__device__ __forceinline__ bool key_ok(const AttP& p, int64_t bi, int64_t i, int64_t j) {
  if(p.mask && p.mask[bi * p.tk + j] == 0.f)
    return false;
  if(p.causal && j > p.tk - p.tq + i)  // layers.cpp:115-116
    return false;
  return true;
}

__global__ void __launch_bounds__(ATT_T) attn_fwd_kernel(AttP p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float sm[];
  const int64_t dk = p.dk, ldS = p.tk + 1;
  float* Qs = sm;                       // [QB][dk+1]
  float* KVs = Qs + QB * (dk + 1);      // [KC][dk+1]
  float* Ss = KVs + KC * (dk + 1);      // [QB][tk+1]
  const int64_t q0 = (int64_t)blockIdx.x * QB;
  const int h = blockIdx.y;
  const int64_t bi = blockIdx.z;
  const int nq = (int)min((int64_t)QB, p.tq - q0);
  const int tid = threadIdx.x;
  const int64_t hoff = (int64_t)h * dk;

  for(int e = tid; e < QB * dk; e += ATT_T) {
    int i = e / (int)dk, c = e % (int)dk;
    Qs[i * (dk + 1) + c] = i < nq ? p.q[(bi * p.tq + q0 + i) * p.ldq + hoff + c] : 0.f;
  }
  // scores
  for(int64_t k0 = 0; k0 < p.tk; k0 += KC) {
    int nk = (int)min((int64_t)KC, p.tk - k0);
    __syncthreads();
    for(int e = tid; e < KC * dk; e += ATT_T) {
      int j = e / (int)dk, c = e % (int)dk;
      KVs[j * (dk + 1) + c] = j < nk ? p.k[(bi * p.tk + k0 + j) * p.ldk + hoff + c] : 0.f;
    }
    __syncthreads();
    for(int e = tid; e < QB * KC; e += ATT_T) {
      int i = e / KC, j = e % KC;
      if(i >= nq || j >= nk)
        continue;
      const float* qr = Qs + i * (dk + 1);
      const float* kr = KVs + j * (dk + 1);
      float acc = 0.f;
      for(int c = 0; c < dk; ++c)
        if(qr[c] != 0.f)
          acc = __fadd_rn(acc, __fmul_rn(qr[c], kr[c]));
      Ss[i * ldS + k0 + j] = __fmul_rn(p.scale, acc);
    }
  }
  __syncthreads();
  // masked softmax, one warp per row
  const int w = tid >> 5, lane = tid & 31;
  for(int i = w; i < nq; i += ATT_T / 32) {
    int64_t gi = q0 + i;
    float* sr = Ss + i * ldS;
    float mx = -INFINITY;
    int any = 0;
    for(int64_t j = lane; j < p.tk; j += 32)
      if(key_ok(p, bi, gi, j)) {
        any = 1;
        mx = fmaxf(mx, sr[j]);
      }
    mx = warp_max(mx);
    any = __any_sync(0xffffffffu, any);
    if(!any && lane == 0 && p.flags)
      atomicOr(p.flags, MTKC_FLAG_MASKED_ROW);
    float s = 0.f;
    for(int64_t j = lane; j < p.tk; j += 32)
      if(key_ok(p, bi, gi, j))
        s += expf(sr[j] - mx);
    s = warp_sum(s);
    float* pr = p.probs + (((bi * p.heads + h) * p.tq) + gi) * p.tk;
    for(int64_t j = lane; j < p.tk; j += 32) {
      float y = (any && key_ok(p, bi, gi, j)) ? expf(sr[j] - mx) / s : 0.f;
      sr[j] = y;
      pr[j] = y;
    }
  }
  // context = P V
  const int CPT = (int)((QB * dk + ATT_T - 1) / ATT_T);  // outputs per thread (<= 32)
  float acc[32];
#pragma unroll
  for(int u = 0; u < 32; ++u)
    acc[u] = 0.f;
  for(int64_t k0 = 0; k0 < p.tk; k0 += KC) {
    int nk = (int)min((int64_t)KC, p.tk - k0);
    __syncthreads();
    for(int e = tid; e < KC * dk; e += ATT_T) {
      int j = e / (int)dk, c = e % (int)dk;
      KVs[j * (dk + 1) + c] = j < nk ? p.v[(bi * p.tk + k0 + j) * p.ldk + hoff + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for(int u = 0; u < 32; ++u) {
      if(u >= CPT)
        break;
      int e = tid + u * ATT_T;
      int i = e / (int)dk, c = e % (int)dk;
      if(i >= nq)
        continue;
      const float* pr = Ss + i * ldS + k0;
      float a = acc[u];
      for(int j = 0; j < nk; ++j) {
        float pv = pr[j];
        if(pv != 0.f)
          a = __fadd_rn(a, __fmul_rn(pv, KVs[j * (dk + 1) + c]));
      }
      acc[u] = a;
    }
  }
#pragma unroll
  for(int u = 0; u < 32; ++u) {
    if(u >= CPT)
      break;
    int e = tid + u * ATT_T;
    int i = e / (int)dk, c = e % (int)dk;
    if(i < nq)
      p.out[(bi * p.tq + q0 + i) * p.ldo + hoff + c] = acc[u];
  }
}

struct AttBP {
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
  float* ds;
  int64_t b, tq, tk;
  int heads;
  int64_t dk;
  float scale;
  int accQ, accK, accV;
};

// Pass A, per (query block, head, batch row):
//   dP = dO V^T ; D = rowsum(dP*P) ; G = scale * P*(dP - D) -> ds ; dQ (+)= G K
__global__ void __launch_bounds__(ATT_T) attn_bwd_q_kernel(AttBP p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float sm[];
  const int64_t dk = p.dk, ldS = p.tk + 1;
  float* Os = sm;                   // dO block [QB][dk+1]
  float* KVs = Os + QB * (dk + 1);  // [KC][dk+1]
  float* Ss = KVs + KC * (dk + 1);  // dP then G [QB][tk+1]
  const int64_t q0 = (int64_t)blockIdx.x * QB;
  const int h = blockIdx.y;
  const int64_t bi = blockIdx.z;
  const int nq = (int)min((int64_t)QB, p.tq - q0);
  const int tid = threadIdx.x;
  const int64_t hoff = (int64_t)h * dk;
  const float* P = p.probs + ((bi * p.heads + h) * p.tq) * p.tk;

  for(int e = tid; e < QB * dk; e += ATT_T) {
    int i = e / (int)dk, c = e % (int)dk;
    Os[i * (dk + 1) + c] = i < nq ? p.gout[(bi * p.tq + q0 + i) * p.ldo + hoff + c] : 0.f;
  }
  for(int64_t k0 = 0; k0 < p.tk; k0 += KC) {
    int nk = (int)min((int64_t)KC, p.tk - k0);
    __syncthreads();
    for(int e = tid; e < KC * dk; e += ATT_T) {
      int j = e / (int)dk, c = e % (int)dk;
      KVs[j * (dk + 1) + c] = j < nk ? p.v[(bi * p.tk + k0 + j) * p.ldk + hoff + c] : 0.f;
    }
    __syncthreads();
    for(int e = tid; e < QB * KC; e += ATT_T) {
      int i = e / KC, j = e % KC;
      if(i >= nq || j >= nk)
        continue;
      const float* orow = Os + i * (dk + 1);
      const float* vr = KVs + j * (dk + 1);
      float acc = 0.f;
      for(int c = 0; c < dk; ++c)
        acc = __fadd_rn(acc, __fmul_rn(orow[c], vr[c]));
      Ss[i * ldS + k0 + j] = acc;
    }
  }
  __syncthreads();
  const int w = tid >> 5, lane = tid & 31;
  for(int i = w; i < nq; i += ATT_T / 32) {
    const float* pr = P + (q0 + i) * p.tk;
    float* sr = Ss + i * ldS;
    float d = 0.f;
    for(int64_t j = lane; j < p.tk; j += 32)
      d += sr[j] * pr[j];
    d = warp_sum(d);
    float* dsr = p.ds + ((bi * p.heads + h) * p.tq + q0 + i) * p.tk;
    for(int64_t j = lane; j < p.tk; j += 32) {
      float gval = p.scale * (pr[j] * (sr[j] - d));
      sr[j] = gval;
      dsr[j] = gval;
    }
  }
  // dQ = G K
  const int CPT = (int)((QB * dk + ATT_T - 1) / ATT_T);
  float acc[32];
#pragma unroll
  for(int u = 0; u < 32; ++u)
    acc[u] = 0.f;
  for(int64_t k0 = 0; k0 < p.tk; k0 += KC) {
    int nk = (int)min((int64_t)KC, p.tk - k0);
    __syncthreads();
    for(int e = tid; e < KC * dk; e += ATT_T) {
      int j = e / (int)dk, c = e % (int)dk;
      KVs[j * (dk + 1) + c] = j < nk ? p.k[(bi * p.tk + k0 + j) * p.ldk + hoff + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for(int u = 0; u < 32; ++u) {
      if(u >= CPT)
        break;
      int e = tid + u * ATT_T;
      int i = e / (int)dk, c = e % (int)dk;
      if(i >= nq)
        continue;
      const float* gr = Ss + i * ldS + k0;
      float a = acc[u];
      for(int j = 0; j < nk; ++j)
        a = __fadd_rn(a, __fmul_rn(gr[j], KVs[j * (dk + 1) + c]));
      acc[u] = a;
    }
  }
#pragma unroll
  for(int u = 0; u < 32; ++u) {
    if(u >= CPT)
      break;
    int e = tid + u * ATT_T;
    int i = e / (int)dk, c = e % (int)dk;
    if(i < nq) {
      float* dst = p.gq + (bi * p.tq + q0 + i) * p.ldq + hoff + c;
      *dst = p.accQ ? *dst + acc[u] : acc[u];
    }
  }
}

// Pass B, per (key chunk, head, batch row): dK (+)= G^T Q, dV (+)= P^T dO,
// summing over queries in ascending order.
__global__ void __launch_bounds__(ATT_T) attn_bwd_kv_kernel(AttBP p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float sm[];
  const int64_t dk = p.dk;
  float* Qs = sm;                     // [QB][dk+1] query chunk (Q then dO)
  float* Gs = Qs + QB * (dk + 1);     // [QB][KC+1] G chunk
  float* Ps = Gs + QB * (KC + 1);     // [QB][KC+1] P chunk
  float* Os = Ps + QB * (KC + 1);     // [QB][dk+1] dO chunk
  const int64_t k0 = (int64_t)blockIdx.x * KC;
  const int h = blockIdx.y;
  const int64_t bi = blockIdx.z;
  const int nk = (int)min((int64_t)KC, p.tk - k0);
  const int tid = threadIdx.x;
  const int64_t hoff = (int64_t)h * dk;
  const float* P = p.probs + ((bi * p.heads + h) * p.tq) * p.tk;
  const float* G = p.ds + ((bi * p.heads + h) * p.tq) * p.tk;
  const int CPT = (int)((KC * dk + ATT_T - 1) / ATT_T);  // <= 64
  float ak[64], av[64];
#pragma unroll
  for(int u = 0; u < 64; ++u) {
    ak[u] = 0.f;
    av[u] = 0.f;
  }
  for(int64_t i0 = 0; i0 < p.tq; i0 += QB) {
    int nq = (int)min((int64_t)QB, p.tq - i0);
    __syncthreads();
    for(int e = tid; e < QB * dk; e += ATT_T) {
      int i = e / (int)dk, c = e % (int)dk;
      bool ok = i < nq;
      Qs[i * (dk + 1) + c] = ok ? p.q[(bi * p.tq + i0 + i) * p.ldq + hoff + c] : 0.f;
      Os[i * (dk + 1) + c] = ok ? p.gout[(bi * p.tq + i0 + i) * p.ldo + hoff + c] : 0.f;
    }
    for(int e = tid; e < QB * KC; e += ATT_T) {
      int i = e / KC, j = e % KC;
      bool ok = i < nq && j < nk;
      Gs[i * (KC + 1) + j] = ok ? G[(i0 + i) * p.tk + k0 + j] : 0.f;
      Ps[i * (KC + 1) + j] = ok ? P[(i0 + i) * p.tk + k0 + j] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for(int u = 0; u < 64; ++u) {
      if(u >= CPT)
        break;
      int e = tid + u * ATT_T;
      int j = e / (int)dk, c = e % (int)dk;
      if(j >= nk)
        continue;
      float a1 = ak[u], a2 = av[u];
      for(int i = 0; i < nq; ++i) {
        a1 = __fadd_rn(a1, __fmul_rn(Gs[i * (KC + 1) + j], Qs[i * (dk + 1) + c]));
        a2 = __fadd_rn(a2, __fmul_rn(Ps[i * (KC + 1) + j], Os[i * (dk + 1) + c]));
      }
      ak[u] = a1;
      av[u] = a2;
    }
  }
#pragma unroll
  for(int u = 0; u < 64; ++u) {
    if(u >= CPT)
      break;
    int e = tid + u * ATT_T;
    int j = e / (int)dk, c = e % (int)dk;
    if(j >= nk)
      continue;
    int64_t off = (bi * p.tk + k0 + j) * p.ldk + hoff + c;
    p.gk[off] = p.accK ? p.gk[off] + ak[u] : ak[u];
    p.gv[off] = p.accV ? p.gv[off] + av[u] : av[u];
  }
}

int set_smem(const void* fn, size_t bytes) {
  if(bytes <= 48 * 1024)
    return MTKC_OK;
  return cuda_status(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
      "attention smem attribute");
}

// ---------------------------------------------------------------------------
// Single-tile fast path: tq, tk <= 64 and dk <= 64 (every BASELINE config:
// sentences of 17..33 tokens, d_k = 64).  One CTA of 256 threads owns one
// (batch row, head); all operands sit in shared memory and every product is
// a 64x64 register-tiled micro-GEMM (each thread a 4x4 block, float4 smem
// reads, FMA).  Row reductions of the softmax stay inside a 16-lane group.
constexpr int T64 = 64;
constexpr int TILE = T64 * T64;  // floats per staged 64x64 operand

// acc[4][4] += sum_k At[k][m] * Bt[k][n] for this thread's rows m = 4ty..,
// columns n = 4tx..
__device__ __forceinline__ void mm64(const float* At, const float* Bt, int K, float acc[4][4],
                                     int ty, int tx) {
#pragma unroll 4
  for(int k = 0; k < K; ++k) {
    float4 a = *reinterpret_cast<const float4*>(At + k * T64 + ty * 4);
    float4 b = *reinterpret_cast<const float4*>(Bt + k * T64 + tx * 4);
    float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for(int i = 0; i < 4; ++i)
#pragma unroll
      for(int j = 0; j < 4; ++j)
        acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
  }
}

// dst[r][c] = src[(row0 + r) * ld + col0 + c] (natural) or dst[c][r]
// (transposed), zero outside [rows x cols].
__device__ __forceinline__ void stage(float* dst, const float* src, int64_t ld, int rows,
                                      int cols, bool transpose) {
  for(int e = threadIdx.x; e < TILE; e += blockDim.x) {
    int r = e / T64, c = e % T64;
    float v = (r < rows && c < cols) ? src[(int64_t)r * ld + c] : 0.f;
    if(transpose)
      dst[c * T64 + r] = v;
    else
      dst[r * T64 + c] = v;
  }
}

__device__ __forceinline__ float grp_max(float v) {
#pragma unroll
  for(int o = 8; o > 0; o >>= 1)
    v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float grp_sum(float v) {
#pragma unroll
  for(int o = 8; o > 0; o >>= 1)
    v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) attn_fwd_tile_kernel(AttP p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  float* Qt = sm;             // [dk][i]
  float* Kt = Qt + TILE;      // [dk][j]
  float* V = Kt + TILE;       // [j][c]
  float* Pt = V + TILE;       // [j][i]
  const int h = blockIdx.x;
  const int64_t bi = blockIdx.y;
  const int tq = (int)p.tq, tk = (int)p.tk, dk = (int)p.dk;
  const int64_t hoff = (int64_t)h * dk;
  stage(Qt, p.q + bi * p.tq * p.ldq + hoff, p.ldq, tq, dk, true);
  stage(Kt, p.k + bi * p.tk * p.ldk + hoff, p.ldk, tk, dk, true);
  stage(V, p.v + bi * p.tk * p.ldk + hoff, p.ldk, tk, dk, false);
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float s[4][4] = {};
  mm64(Qt, Kt, dk, s, ty, tx);
  float* P = p.probs + ((bi * p.heads + h) * p.tq) * p.tk;
#pragma unroll
  for(int a = 0; a < 4; ++a) {
    int i = ty * 4 + a;
    bool ok[4];
    float mx = -INFINITY;
#pragma unroll
    for(int c = 0; c < 4; ++c) {
      int j = tx * 4 + c;
      ok[c] = i < tq && j < tk && key_ok(p, bi, i, j);
      s[a][c] = p.scale * s[a][c];
      if(ok[c])
        mx = fmaxf(mx, s[a][c]);
    }
    mx = grp_max(mx);
    bool any = mx != -INFINITY;
    float e[4], sum = 0.f;
#pragma unroll
    for(int c = 0; c < 4; ++c) {
      e[c] = ok[c] ? expf(s[a][c] - mx) : 0.f;
      sum += e[c];
    }
    sum = grp_sum(sum);
    if(i < tq && !any && tx == 0 && p.flags)
      atomicOr(p.flags, MTKC_FLAG_MASKED_ROW);
#pragma unroll
    for(int c = 0; c < 4; ++c) {
      int j = tx * 4 + c;
      float y = any ? e[c] / sum : 0.f;
      Pt[j * T64 + i] = y;
      if(i < tq && j < tk)
        P[(int64_t)i * tk + j] = y;
    }
  }
  __syncthreads();
  float o[4][4] = {};
  mm64(Pt, V, tk, o, ty, tx);
#pragma unroll
  for(int a = 0; a < 4; ++a) {
    int i = ty * 4 + a;
    if(i >= tq)
      continue;
    float* dst = p.out + (bi * p.tq + i) * p.ldo + hoff;
#pragma unroll
    for(int c = 0; c < 4; ++c) {
      int col = tx * 4 + c;
      if(col < dk)
        dst[col] = o[a][c];
    }
  }
}

__global__ void __launch_bounds__(256) attn_bwd_tile_kernel(AttBP p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  float* dO = sm;            // [i][c]
  float* B1 = dO + TILE;     // dOt [c][i], then Q [i][c]
  float* B2 = B1 + TILE;     // Vt [c][j], then K [j][c]
  float* Pn = B2 + TILE;     // P [i][j]
  float* dS = Pn + TILE;     // [i][j]
  float* dSt = dS + TILE;    // [j][i]
  const int h = blockIdx.x;
  const int64_t bi = blockIdx.y;
  const int tq = (int)p.tq, tk = (int)p.tk, dk = (int)p.dk;
  const int64_t hoff = (int64_t)h * dk;
  const float* go = p.gout + bi * p.tq * p.ldo + hoff;
  stage(dO, go, p.ldo, tq, dk, false);
  stage(B1, go, p.ldo, tq, dk, true);
  stage(B2, p.v + bi * p.tk * p.ldk + hoff, p.ldk, tk, dk, true);
  stage(Pn, p.probs + ((bi * p.heads + h) * p.tq) * p.tk, p.tk, tq, tk, false);
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float dp[4][4] = {};
  mm64(B1, B2, dk, dp, ty, tx);  // dP = dO V^T
  float* G = p.ds + ((bi * p.heads + h) * p.tq) * p.tk;
#pragma unroll
  for(int a = 0; a < 4; ++a) {
    int i = ty * 4 + a;
    float pv[4], d = 0.f;
#pragma unroll
    for(int c = 0; c < 4; ++c) {
      pv[c] = Pn[i * T64 + tx * 4 + c];
      d += dp[a][c] * pv[c];
    }
    d = grp_sum(d);
#pragma unroll
    for(int c = 0; c < 4; ++c) {
      int j = tx * 4 + c;
      float gval = p.scale * (pv[c] * (dp[a][c] - d));
      dS[i * T64 + j] = gval;
      dSt[j * T64 + i] = gval;
      if(i < tq && j < tk)
        G[(int64_t)i * tk + j] = gval;
    }
  }
  __syncthreads();
  stage(B1, p.q + bi * p.tq * p.ldq + hoff, p.ldq, tq, dk, false);
  stage(B2, p.k + bi * p.tk * p.ldk + hoff, p.ldk, tk, dk, false);
  __syncthreads();
  float acc[4][4];
  auto store = [&](float* base, int64_t ld, int rows, int acc_mode) {
#pragma unroll
    for(int a = 0; a < 4; ++a) {
      int r = ty * 4 + a;
      if(r >= rows)
        continue;
#pragma unroll
      for(int c = 0; c < 4; ++c) {
        int col = tx * 4 + c;
        if(col < dk) {
          float* dst = base + (int64_t)r * ld + col;
          *dst = acc_mode ? *dst + acc[a][c] : acc[a][c];
        }
      }
    }
  };
  // dQ = dS K
  for(auto& r : acc)
    for(float& x : r)
      x = 0.f;
  mm64(dSt, B2, tk, acc, ty, tx);
  store(p.gq + bi * p.tq * p.ldq + hoff, p.ldq, tq, p.accQ);
  // dK = dS^T Q
  for(auto& r : acc)
    for(float& x : r)
      x = 0.f;
  mm64(dS, B1, tq, acc, ty, tx);
  store(p.gk + bi * p.tk * p.ldk + hoff, p.ldk, tk, p.accK);
  // dV = P^T dO
  for(auto& r : acc)
    for(float& x : r)
      x = 0.f;
  mm64(Pn, dO, tq, acc, ty, tx);
  store(p.gv + bi * p.tk * p.ldk + hoff, p.ldk, tk, p.accV);
}

// ---------------------------------------------------------------------------
// Padded-tile path for head dim 64 and tq, tk <= TT (TT = 32, 48 or 64): all
// operands row-major in shared memory with a padded leading dimension of
// 4*odd floats, so the strided float4 reads of the micro-GEMMs below are
// bank-conflict free; 256 threads, each a 4x4 register tile.
constexpr int DK = 64;
constexpr int LDK = DK + 4;  // 68 = 4*17

template <int TT>
struct Pad {
  static constexpr int LDP = TT + 4;  // 36, 52, 68: 4 * odd
};

// C[i][j] = sum_k A[i][k] * B[j][k]   (A: M x K, B: N x K, both row-major)
// thread tile: rows i = ti + a*(M/4), cols j = tj + b*(N/4)
template <int M, int N>
__device__ __forceinline__ void mm_nt(const float* A, int lda, const float* B, int ldb, int K,
                                      float* C, int ldc, float scale) {
  constexpr int TI = M / 4, TJ = N / 4;
  for(int t = threadIdx.x; t < TI * TJ; t += blockDim.x) {
    const int ti = t % TI, tj = t / TI;
    float acc[4][4] = {};
    for(int k = 0; k < K; k += 4) {
      float4 a[4], b[4];
#pragma unroll
      for(int u = 0; u < 4; ++u) {
        a[u] = *reinterpret_cast<const float4*>(A + (ti + u * TI) * lda + k);
        b[u] = *reinterpret_cast<const float4*>(B + (tj + u * TJ) * ldb + k);
      }
#pragma unroll
      for(int u = 0; u < 4; ++u)
#pragma unroll
        for(int v = 0; v < 4; ++v) {
          acc[u][v] = __fmaf_rn(a[u].x, b[v].x, acc[u][v]);
          acc[u][v] = __fmaf_rn(a[u].y, b[v].y, acc[u][v]);
          acc[u][v] = __fmaf_rn(a[u].z, b[v].z, acc[u][v]);
          acc[u][v] = __fmaf_rn(a[u].w, b[v].w, acc[u][v]);
        }
    }
#pragma unroll
    for(int u = 0; u < 4; ++u)
#pragma unroll
      for(int v = 0; v < 4; ++v)
        C[(ti + u * TI) * ldc + tj + v * TJ] = scale * acc[u][v];
  }
}

// acc = sum_k A[i][k] * B[k][c] for rows i = ti + a*(M/4), cols c = 4tj..4tj+3
// (A: M x K row-major, B: K x N row-major); calls store(i, c, value)
template <int M, int N, typename Store>
__device__ __forceinline__ void mm_nn(const float* A, int lda, const float* B, int ldb, int K,
                                      Store store) {
  constexpr int TI = M / 4, TJ = N / 4;
  for(int t = threadIdx.x; t < TI * TJ; t += blockDim.x) {
    const int ti = t % TI, tj = t / TI;
    float acc[4][4] = {};
    for(int k = 0; k < K; k += 4) {
      float4 a[4], b[4];
#pragma unroll
      for(int u = 0; u < 4; ++u) {
        a[u] = *reinterpret_cast<const float4*>(A + (ti + u * TI) * lda + k);
        b[u] = *reinterpret_cast<const float4*>(B + (k + u) * ldb + tj * 4);
      }
#pragma unroll
      for(int u = 0; u < 4; ++u) {
        const float av[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
        for(int kk = 0; kk < 4; ++kk) {
          acc[u][0] = __fmaf_rn(av[kk], (&b[kk].x)[0], acc[u][0]);
          acc[u][1] = __fmaf_rn(av[kk], (&b[kk].x)[1], acc[u][1]);
          acc[u][2] = __fmaf_rn(av[kk], (&b[kk].x)[2], acc[u][2]);
          acc[u][3] = __fmaf_rn(av[kk], (&b[kk].x)[3], acc[u][3]);
        }
      }
    }
#pragma unroll
    for(int u = 0; u < 4; ++u)
#pragma unroll
      for(int v = 0; v < 4; ++v)
        store(ti + u * TI, tj * 4 + v, acc[u][v]);
  }
}

// stage rows x 64 floats of a head slice (row stride ld) into [TT][LDK],
// zero-filling rows >= rows; float4 loads, consecutive threads on a row
template <int TT>
__device__ __forceinline__ void stage64(float* dst, const float* src, int64_t ld, int rows) {
  for(int e = threadIdx.x; e < TT * (DK / 4); e += blockDim.x) {
    const int r = e / (DK / 4), c4 = e % (DK / 4);
    float4 v = r < rows ? *reinterpret_cast<const float4*>(src + (int64_t)r * ld + c4 * 4)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(dst + r * LDK + c4 * 4) = v;
  }
}

template <int TT>
__global__ void __launch_bounds__(256) attn_fwd_pad_kernel(AttP p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float4 smem4[];
  constexpr int LDP = Pad<TT>::LDP;
  float* sm = reinterpret_cast<float*>(smem4);
  float* Q = sm;                 // [TT][LDK]
  float* K = Q + TT * LDK;
  float* V = K + TT * LDK;
  float* S = V + TT * LDK;       // [TT][LDP] scores, then P
  const int h = blockIdx.x;
  const int64_t bi = blockIdx.y;
  const int tq = (int)p.tq, tk = (int)p.tk;
  const int64_t hoff = (int64_t)h * DK;
  stage64<TT>(Q, p.q + bi * p.tq * p.ldq + hoff, p.ldq, tq);
  stage64<TT>(K, p.k + bi * p.tk * p.ldk + hoff, p.ldk, tk);
  stage64<TT>(V, p.v + bi * p.tk * p.ldk + hoff, p.ldk, tk);
  __syncthreads();
  mm_nt<TT, TT>(Q, LDK, K, LDK, DK, S, LDP, p.scale);
  __syncthreads();
  // masked softmax: one warp per query row, two keys per lane (tk <= 64)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* P = p.probs + ((bi * p.heads + h) * p.tq) * p.tk;
  for(int i = warp; i < TT; i += blockDim.x / 32) {
    float* sr = S + i * LDP;
    float x0 = -INFINITY, x1 = -INFINITY;
    bool o0 = false, o1 = false;
    if(i < tq) {
      o0 = lane < tk && key_ok(p, bi, i, lane);
      o1 = lane + 32 < tk && key_ok(p, bi, i, lane + 32);
      if(o0)
        x0 = sr[lane];
      if(o1 && lane + 32 < TT)
        x1 = sr[lane + 32];
    }
    float mx = warp_max(fmaxf(x0, x1));
    bool any = mx != -INFINITY;
    float e0 = o0 ? expf(x0 - mx) : 0.f, e1 = o1 ? expf(x1 - mx) : 0.f;
    float s = warp_sum(e0 + e1);
    if(i < tq && !any && lane == 0 && p.flags)
      atomicOr(p.flags, MTKC_FLAG_MASKED_ROW);
    float y0 = any ? e0 / s : 0.f, y1 = any ? e1 / s : 0.f;
    if(lane < TT)
      sr[lane] = y0;
    if(lane + 32 < TT)
      sr[lane + 32] = y1;
    if(i < tq) {
      if(lane < tk)
        P[(int64_t)i * tk + lane] = y0;
      if(lane + 32 < tk)
        P[(int64_t)i * tk + lane + 32] = y1;
    }
  }
  __syncthreads();
  float* out = p.out + bi * p.tq * p.ldo + hoff;
  mm_nn<TT, DK>(S, LDP, V, LDK, TT, [&](int i, int c, float v) {
    if(i < tq)
      out[(int64_t)i * p.ldo + c] = v;
  });
}

template <int TT>
__global__ void __launch_bounds__(256) attn_bwd_pad_kernel(AttBP p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float4 smem4[];
  constexpr int LDP = Pad<TT>::LDP;
  float* sm = reinterpret_cast<float*>(smem4);
  float* Q = sm;                  // [TT][LDK]
  float* K = Q + TT * LDK;
  float* V = K + TT * LDK;
  float* dO = V + TT * LDK;
  float* P = dO + TT * LDK;       // [TT][LDP]
  float* dP = P + TT * LDP;       // [TT][LDP] dP, then dS
  float* dSt = dP + TT * LDP;     // [TT][LDP] dS^T
  float* Pt = dSt + TT * LDP;     // [TT][LDP] P^T
  const int h = blockIdx.x;
  const int64_t bi = blockIdx.y;
  const int tq = (int)p.tq, tk = (int)p.tk;
  const int64_t hoff = (int64_t)h * DK;
  stage64<TT>(Q, p.q + bi * p.tq * p.ldq + hoff, p.ldq, tq);
  stage64<TT>(K, p.k + bi * p.tk * p.ldk + hoff, p.ldk, tk);
  stage64<TT>(V, p.v + bi * p.tk * p.ldk + hoff, p.ldk, tk);
  stage64<TT>(dO, p.gout + bi * p.tq * p.ldo + hoff, p.ldo, tq);
  const float* Pg = p.probs + ((bi * p.heads + h) * p.tq) * p.tk;
  for(int e = threadIdx.x; e < TT * TT; e += blockDim.x) {
    const int i = e / TT, j = e % TT;
    float v = (i < tq && j < tk) ? Pg[(int64_t)i * tk + j] : 0.f;
    P[i * LDP + j] = v;
    Pt[j * LDP + i] = v;
  }
  __syncthreads();
  mm_nt<TT, TT>(dO, LDK, V, LDK, DK, dP, LDP, 1.f);  // dP = dO V^T
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* G = p.ds + ((bi * p.heads + h) * p.tq) * p.tk;
  for(int i = warp; i < TT; i += blockDim.x / 32) {
    const float p0 = lane < TT ? P[i * LDP + lane] : 0.f;
    const float p1 = lane + 32 < TT ? P[i * LDP + lane + 32] : 0.f;
    const float d0 = lane < TT ? dP[i * LDP + lane] : 0.f;
    const float d1 = lane + 32 < TT ? dP[i * LDP + lane + 32] : 0.f;
    const float D = warp_sum(d0 * p0 + d1 * p1);
    const float g0 = p.scale * (p0 * (d0 - D)), g1 = p.scale * (p1 * (d1 - D));
    if(lane < TT) {
      dP[i * LDP + lane] = g0;
      dSt[lane * LDP + i] = g0;
    }
    if(lane + 32 < TT) {
      dP[i * LDP + lane + 32] = g1;
      dSt[(lane + 32) * LDP + i] = g1;
    }
    if(i < tq) {
      if(lane < tk)
        G[(int64_t)i * tk + lane] = g0;
      if(lane + 32 < tk)
        G[(int64_t)i * tk + lane + 32] = g1;
    }
  }
  __syncthreads();
  float* gq = p.gq + bi * p.tq * p.ldq + hoff;
  float* gk = p.gk + bi * p.tk * p.ldk + hoff;
  float* gv = p.gv + bi * p.tk * p.ldk + hoff;
  mm_nn<TT, DK>(dP, LDP, K, LDK, TT, [&](int i, int c, float v) {  // dQ = dS K
    if(i < tq) {
      float* d = gq + (int64_t)i * p.ldq + c;
      *d = p.accQ ? *d + v : v;
    }
  });
  mm_nn<TT, DK>(dSt, LDP, Q, LDK, TT, [&](int j, int c, float v) {  // dK = dS^T Q
    if(j < tk) {
      float* d = gk + (int64_t)j * p.ldk + c;
      *d = p.accK ? *d + v : v;
    }
  });
  mm_nn<TT, DK>(Pt, LDP, dO, LDK, TT, [&](int j, int c, float v) {  // dV = P^T dO
    if(j < tk) {
      float* d = gv + (int64_t)j * p.ldk + c;
      *d = p.accV ? *d + v : v;
    }
  });
}

int pad_tile(int64_t tq, int64_t tk, int64_t dk, int64_t ldq, int64_t ldk, int64_t ldo) {
  if(dk != DK || (ldq | ldk | ldo) % 4 || getenv("MTK_ATTN_TILE64"))
    return 0;
  int64_t t = std::max(tq, tk);
  return t <= 32 ? 32 : t <= 48 ? 48 : t <= 64 ? 64 : 0;
}

template <int TT>
size_t pad_smem(bool bwd) {
  return sizeof(float) * (bwd ? (4 * TT * LDK + 4 * TT * Pad<TT>::LDP)
                              : (3 * TT * LDK + TT * Pad<TT>::LDP));
}

bool tile_path(int64_t tq, int64_t tk, int64_t dk, int64_t ldq, int64_t ldk, int64_t ldo) {
  (void)ldq;
  (void)ldk;
  (void)ldo;
  return tq <= T64 && tk <= T64 && dk <= T64 && dk % 4 == 0 && !getenv("MTK_ATTN_GENERIC");
}

}  // namespace

extern "C" {

int mtkc_attention(float* out, int64_t ldo, float* probs, const float* q, int64_t ldq,
                   const float* k, const float* v, int64_t ldk, const float* key_mask,
                   int64_t b, int64_t tq, int64_t tk, int heads, int64_t dk, float scale,
                   int causal, int* flags, void* stream) {
  if(b <= 0 || tq <= 0 || tk <= 0)
    return MTKC_OK;
  if(tk > MAX_TK || dk > MAX_DK || dk <= 0)
    return fail(MTKC_DIMENSION, "fused attention supports tk <= 512 and head dim <= 128");
  ProfScope prof(S(stream), "attention", 4.0 * b * heads * tq * tk * dk);
  if(prof_detail())
    prof.detail = "fwd_b" + std::to_string(b) + "_tq" + std::to_string(tq) + "_tk" + std::to_string(tk);
  AttP p{out, ldo, probs, q, ldq, k, v, ldk, key_mask, b, tq, tk, heads, dk, scale, causal, flags};
  if(int tt = pad_tile(tq, tk, dk, ldq, ldk, ldo)) {
    dim3 grid((unsigned)heads, (unsigned)b);
    int rc = MTKC_OK;
#define MTKC_ATT_FWD(TTV)                                                         \
  if(tt == TTV) {                                                                 \
    size_t smem = pad_smem<TTV>(false);                                           \
    rc = set_smem((const void*)attn_fwd_pad_kernel<TTV>, smem);                   \
    if(rc)                                                                        \
      return rc;                                                                  \
    ::mtkc::launch(attn_fwd_pad_kernel<TTV>, grid, 256, smem, S(stream), p);                  \
  }
    MTKC_ATT_FWD(32) MTKC_ATT_FWD(48) MTKC_ATT_FWD(64)
#undef MTKC_ATT_FWD
    MTKC_POST_LAUNCH("attn_fwd_pad_kernel");
    return MTKC_OK;
  }
  if(tile_path(tq, tk, dk, ldq, ldk, ldo)) {
    size_t smem = 4 * TILE * sizeof(float);
    int rc = set_smem((const void*)attn_fwd_tile_kernel, smem);
    if(rc)
      return rc;
    ::mtkc::launch(attn_fwd_tile_kernel, dim3((unsigned)heads, (unsigned)b), 256, smem, S(stream), p);
    MTKC_POST_LAUNCH("attn_fwd_tile_kernel");
    return MTKC_OK;
  }
  size_t smem = sizeof(float) * ((size_t)QB * (dk + 1) + (size_t)KC * (dk + 1) +
                                 (size_t)QB * (tk + 1));
  int rc = set_smem((const void*)attn_fwd_kernel, smem);
  if(rc)
    return rc;
  dim3 grid((unsigned)cdiv(tq, QB), (unsigned)heads, (unsigned)b);
  ::mtkc::launch(attn_fwd_kernel, grid, ATT_T, smem, S(stream), p);
  MTKC_POST_LAUNCH("attn_fwd_kernel");
  return MTKC_OK;
}

int mtkc_attention_backward(const float* gout, int64_t ldo, const float* probs,
                            const float* q, int64_t ldq, const float* k, const float* v,
                            int64_t ldk, float* gq, float* gk, float* gv, float* dsbuf,
                            int64_t b, int64_t tq, int64_t tk, int heads, int64_t dk,
                            float scale, int accumulate_q, int accumulate_k, int accumulate_v,
                            void* stream) {
  if(b <= 0 || tq <= 0 || tk <= 0)
    return MTKC_OK;
  if(tk > MAX_TK || dk > MAX_DK || dk <= 0)
    return fail(MTKC_DIMENSION, "fused attention supports tk <= 512 and head dim <= 128");
  ProfScope prof(S(stream), "attention", 8.0 * b * heads * tq * tk * dk);
  if(prof_detail())
    prof.detail = "bwd_b" + std::to_string(b) + "_tq" + std::to_string(tq) + "_tk" + std::to_string(tk);
  AttBP p{gout, ldo, probs, q, ldq, k, v, ldk, gq, gk, gv, dsbuf, b, tq, tk, heads, dk, scale,
          accumulate_q, accumulate_k, accumulate_v};
  if(int tt = pad_tile(tq, tk, dk, ldq, ldk, ldo)) {
    dim3 grid((unsigned)heads, (unsigned)b);
    int rc = MTKC_OK;
#define MTKC_ATT_BWD(TTV)                                                         \
  if(tt == TTV) {                                                                 \
    size_t smem = pad_smem<TTV>(true);                                            \
    rc = set_smem((const void*)attn_bwd_pad_kernel<TTV>, smem);                   \
    if(rc)                                                                        \
      return rc;                                                                  \
    ::mtkc::launch(attn_bwd_pad_kernel<TTV>, grid, 256, smem, S(stream), p);                  \
  }
    MTKC_ATT_BWD(32) MTKC_ATT_BWD(48) MTKC_ATT_BWD(64)
#undef MTKC_ATT_BWD
    MTKC_POST_LAUNCH("attn_bwd_pad_kernel");
    return MTKC_OK;
  }
  if(tile_path(tq, tk, dk, ldq, ldk, ldo)) {
    size_t smem = 6 * TILE * sizeof(float);
    int rc = set_smem((const void*)attn_bwd_tile_kernel, smem);
    if(rc)
      return rc;
    ::mtkc::launch(attn_bwd_tile_kernel, dim3((unsigned)heads, (unsigned)b), 256, smem, S(stream), p);
    MTKC_POST_LAUNCH("attn_bwd_tile_kernel");
    return MTKC_OK;
  }
  size_t smemA = sizeof(float) * ((size_t)QB * (dk + 1) + (size_t)KC * (dk + 1) +
                                  (size_t)QB * (tk + 1));
  int rc = set_smem((const void*)attn_bwd_q_kernel, smemA);
  if(rc)
    return rc;
  dim3 gA((unsigned)cdiv(tq, QB), (unsigned)heads, (unsigned)b);
  ::mtkc::launch(attn_bwd_q_kernel, gA, ATT_T, smemA, S(stream), p);
  MTKC_POST_LAUNCH("attn_bwd_q_kernel");
  size_t smemB = sizeof(float) * (2 * (size_t)QB * (dk + 1) + 2 * (size_t)QB * (KC + 1));
  rc = set_smem((const void*)attn_bwd_kv_kernel, smemB);
  if(rc)
    return rc;
  dim3 gB((unsigned)cdiv(tk, KC), (unsigned)heads, (unsigned)b);
  ::mtkc::launch(attn_bwd_kv_kernel, gB, ATT_T, smemB, S(stream), p);
  MTKC_POST_LAUNCH("attn_bwd_kv_kernel");
  return MTKC_OK;
}

}  // extern "C"
