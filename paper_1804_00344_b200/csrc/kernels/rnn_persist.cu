// Persistent GRU scan: the whole time loop of a deep-transition GRU stack
// (RnnEncoder::build / RnnDecoder::step, reference models.cpp:146-187 and
// 312-382; DeepTransitionCell layers.cpp:183-244; gruCell graph.cpp:633-745;
// BahdanauAttention::apply layers.cpp:59-79) in ONE cooperative launch.
//
// Why: per step and block the recurrence is a skinny product
// [b x d] x [d x 3d] (b = 60..128 rows) followed by a row-wise pointwise
// pass.  As separate launches that is ~4 kernels per block-step (GEMM,
// split-K reduce, GRU pointwise, ...) -- thousands per training step, more
// host submission time than GPU time.  Here every SM stays resident for the
// whole sequence and the phases are separated by grid barriers:
//
//   PROD  the recurrent product as K-split units (m-tile 128 rows x n-tile
//         96 gate columns x k-slice) over all CTAs of the direction:
//         warp 0 issues TMA loads (6-stage ring, 128-byte swizzle), warp 1
//         issues tcgen05.mma kind::tf32 into a TMEM accumulator, warps 4-7
//         read it back (tcgen05.ld) and store fp32 partials;
//   PW    one CTA per batch row: sum the partials in a fixed order (k-slice
//         0, 1, ...), then bias + per-gate layer norm + sigmoid/tanh gates +
//         interpolation (+ padding blend), exactly the arithmetic of
//         gru_fwd_kernel (kernels/gru.cu);
//   ATT   (decoder, after block 1) the query product s1*W is a PROD phase;
//         then one CTA per row computes the scores, masked softmax and the
//         context (the arithmetic of bahdanau_score/ctx_kernel).
//
// The weight operands are fed K-major: the host transposes U / W / attW
// once per forward into the workspace (weights are constant within a step).
// Both directions of the bidirectional encoder run in one launch on
// disjoint halves of the grid (separate barriers).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>
#include <cstdio>

#include "common.cuh"
#include "tc_ptx.cuh"

using namespace mtkc;
using namespace mtkc::tc;

namespace {

constexpr int RT = 256;        // threads: warp 0 TMA, warp 1 MMA, warps 4..7 epilogue
constexpr int RST = 6;         // smem ring stages
constexpr int NTH = 96;        // n-tile of the gate products (3d is a multiple of 96)
constexpr uint32_t A_STAGE = 128 * 32 * 4;  // 16 KB: 128 rows x 32 fp32
constexpr uint32_t B_STAGE = NTH * 32 * 4;  // 12 KB
constexpr int TMEM_COLS = 256;  // two 128-column accumulators (units alternate)
constexpr int MAXA = 2048;  // attention width cap (row-phase smem)
constexpr int MAXS = 1024;  // source positions cap

struct Maps {
  CUtensorMap hh[2];    // A: state slots [(T+1)*b x d]
  CUtensorMap sout[2];  // A: intermediate block outputs [(K-1)*T*b x d]
  CUtensorMap ut[2];    // B: [U_z|U_r|U_h]^T per block, [K*3d x d]
  CUtensorMap ctx;      // A: contexts [T*b x kd]
  CUtensorMap w2t;      // B: [W_z|W_r|W_x]^T of block 2, [3d x kd]
  CUtensorMap watt;     // B: attention W^T [a x d]
};

struct KP {
  mtkc_rnn_scan_args a;
  float* partHu[2];  // [KCh][b][3d] per direction
  float* partX;      // [KCx][b][3d]
  float* partQ;      // [KCq][b][a]
  unsigned* ctr;     // [2] grid-barrier counters (zeroed before launch)
  unsigned long long* prof;  // MTK_RNN_PROF: CTA 0's phase timestamps, or NULL
  // attention row teams: `team` CTAs per batch row (positions / columns
  // split between them), synchronised per row through teamCtr[r]; scratch
  // teamBuf [b x S] exchanges the scores
  int team;
  unsigned* teamCtr;
  float* teamBuf;
  int KCh, KCx, KCq, NTq;
};

struct Prod {
  const CUtensorMap* ma;
  const CUtensorMap* mb;
  int aRow0, bRow0, N, NT, KS, KC, nT, mT;
  float* part;
  __device__ int units() const { return mT * nT * KC; }
};

struct Smem {
  uint8_t* sA;
  uint8_t* sB;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t tmem;
};

// ------------------------------------------------------------ grid barrier

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// the `team` CTAs working on one batch row: release-add, acquire-spin
__device__ __forceinline__ void team_bar(unsigned* ctr, unsigned n, unsigned& epoch) {
  __syncthreads();
  if(threadIdx.x == 0) {
    epoch += n;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    while(ld_acquire(ctr) < epoch)
      ;
  }
  __syncthreads();
}

// all CTAs of one direction group; counter is monotonic (epoch = phases * n)
// (bar.sync orders the CTA's writes before thread 0's release; the release
// reduction is cumulative at gpu scope, the acquire load pairs with it)
__device__ __forceinline__ void grid_bar(unsigned* ctr, unsigned n, unsigned& epoch) {
  __syncthreads();
  if(threadIdx.x == 0) {
    epoch += n;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    while(ld_acquire(ctr) < epoch)
      ;
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// CTA 0 records (phase kind, start time) pairs
__device__ __forceinline__ void mark(unsigned long long* prof, int& np, int kind) {
  if(prof && blockIdx.x == 0 && threadIdx.x == 0 && np < 8190) {
    prof[2 * np] = (unsigned long long)kind;
    prof[2 * np + 1] = gtimer();
    ++np;
  }
}

// ------------------------------------------------------------ PROD phase

__device__ void run_prods(const Prod* P, int np, int gi, int gs, const Smem& sm, uint32_t& ring,
                          uint32_t& ucnt, int64_t b) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tot = 0;
  for(int q = 0; q < np; ++q)
    tot += P[q].units();
  auto decode = [&](int u, int& q, int& mt, int& nt, int& kc) {
    q = 0;
    while(u >= P[q].units()) {
      u -= P[q].units();
      ++q;
    }
    mt = u % P[q].mT;
    u /= P[q].mT;
    nt = u % P[q].nT;
    kc = u / P[q].nT;
  };
  if(warp == 0) {
    if(lane == 0) {
      // the operands were written by generic-proxy stores of other CTAs
      asm volatile("fence.proxy.async.global;" ::: "memory");
      for(int u = gi; u < tot; u += gs) {
        int q, mt, nt, kc;
        decode(u, q, mt, nt, kc);
        const Prod& pr = P[q];
        const int nkb = pr.KS / 32;
        for(int kb = 0; kb < nkb; ++kb, ++ring) {
          const int s = ring % RST;
          if(ring >= RST)
            mbar_wait(&sm.empty[s], ((ring / RST) - 1) & 1);
          mbar_expect_tx(&sm.full[s], A_STAGE + (uint32_t)pr.NT * 128u);
          const int k0 = kc * pr.KS + kb * 32;
          tma_load_2d(sm.sA + s * A_STAGE, pr.ma, &sm.full[s], k0, pr.aRow0 + mt * 128);
          tma_load_2d(sm.sB + s * B_STAGE, pr.mb, &sm.full[s], k0, pr.bRow0 + nt * pr.NT);
        }
      }
    }
  } else if(warp == 1) {
    for(int u = gi; u < tot; u += gs) {
      int q, mt, nt, kc;
      decode(u, q, mt, nt, kc);
      const Prod& pr = P[q];
      // accumulator ucnt & 1: wait until the epilogue drained its previous use
      const int acc = (int)(ucnt & 1);
      if(ucnt >= 2)
        mbar_wait(&sm.tempty[acc], ((ucnt >> 1) - 1) & 1);
      tc_fence_after();
      // D=f32, A=B=tf32, both K-major, N>>3, M>>4
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(pr.NT >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const int nkb = pr.KS / 32;
      for(int kb = 0; kb < nkb; ++kb, ++ring) {
        const int s = ring % RST;
        mbar_wait(&sm.full[s], (ring / RST) & 1);
        tc_fence_after();
        if(lane == 0) {
          const uint32_t aBase = smem_u32(sm.sA + s * A_STAGE);
          const uint32_t bBase = smem_u32(sm.sB + s * B_STAGE);
#pragma unroll
          for(int kk = 0; kk < 4; ++kk)
            mma_tf32(sm.tmem + (uint32_t)acc * 128u, umma_desc(aBase + kk * 32, 16, 1024, 2),
                     umma_desc(bBase + kk * 32, 16, 1024, 2), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&sm.empty[s]);
        }
        __syncwarp();
      }
      if(lane == 0)
        mma_commit(&sm.tfull[acc]);
      __syncwarp();
      ++ucnt;
    }
  } else if(warp >= 4) {
    const int qd = warp & 3;  // TMEM lane quarter this warp may read
    for(int u = gi; u < tot; u += gs) {
      int q, mt, nt, kc;
      decode(u, q, mt, nt, kc);
      const Prod& pr = P[q];
      const int acc = (int)(ucnt & 1);
      mbar_wait(&sm.tfull[acc], (ucnt >> 1) & 1);
      tc_fence_after();
      const int64_t row = (int64_t)mt * 128 + qd * 32 + lane;
      for(int c0 = 0; c0 < pr.NT; c0 += 32) {
        float v[32];
        tmem_ld32(sm.tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)acc * 128u + (uint32_t)c0, v);
        if(row < b) {
          float4* dst = reinterpret_cast<float4*>(pr.part + ((int64_t)kc * b + row) * pr.N +
                                                  (int64_t)nt * pr.NT + c0);
#pragma unroll
          for(int j = 0; j < 8; ++j)
            dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if(lane == 0)
        mbar_arrive(&sm.tempty[acc]);
      ++ucnt;
    }
  }
}

// ------------------------------------------------------------ row phases

template <int NQ>
__device__ __forceinline__ void block_sums(float (&v)[NQ], float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
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
    float t = lane < RT / 32 ? red[q * 32 + lane] : 0.f;
    v[q] = warp_sum(t);
  }
}

__device__ __forceinline__ float sigm(float a) { return 1.f / (1.f + expf(-a)); }

__device__ __forceinline__ float4 ldcg4(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 ld4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void st4(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void add4(float (&acc)[4], const float4& v) {
  acc[0] += v.x;
  acc[1] += v.y;
  acc[2] += v.z;
  acc[3] += v.w;
}
__device__ __forceinline__ void set4(float (&acc)[4], const float4& v) {
  acc[0] = v.x;
  acc[1] = v.y;
  acc[2] = v.z;
  acc[3] = v.w;
}

constexpr int GQ = 2;  // float4 groups per thread in the GRU row phase (d <= 2048)

// One GRU block for batch row r at step t (gru_fwd_kernel's arithmetic).
// hin: the block's state input row; partials summed in k-slice order.  Each
// thread owns GQ groups of 4 consecutive columns; every global load of the
// row is issued before the arithmetic (the phase is latency-bound).
__device__ void gru_row(const KP& p, const mtkc_rnn_dir& D, int k, int64_t t, int64_t r,
                        const float* hin, const float* partHu, int KCh, const float* partX,
                        int KCx, const float* xwHoist, float* out, const float* prevRow,
                        float blendM, bool blend, float* red) {
  const int64_t b = p.a.b, d = p.a.d, d3 = 3 * d, d4 = d / 4;
  const mtkc_rnn_block& B = D.blk[k];
  const bool ln = B.ln[0] != nullptr;
  const bool hasX = xwHoist != nullptr || partX != nullptr;
  const int64_t tr = t * b + r;  // time-major row
  float hz[GQ][4], hr[GQ][4], hh[GQ][4], xz[GQ][4], xr[GQ][4], xx[GQ][4], hv[GQ][4];
#pragma unroll
  for(int q = 0; q < GQ; ++q) {
    const int64_t g = threadIdx.x + (int64_t)q * RT;
#pragma unroll
    for(int i = 0; i < 4; ++i)
      hz[q][i] = hr[q][i] = hh[q][i] = xz[q][i] = xr[q][i] = xx[q][i] = hv[q][i] = 0.f;
    if(g >= d4)
      continue;
    const int64_t j = 4 * g;
    for(int kc = 0; kc < KCh; ++kc) {
      const float* pp = partHu + ((int64_t)kc * b + r) * d3 + j;
      const float4 a0 = ldcg4(pp), a1 = ldcg4(pp + d), a2 = ldcg4(pp + 2 * d);
      add4(hz[q], a0);
      add4(hr[q], a1);
      add4(hh[q], a2);
    }
    if(xwHoist) {
      const float* xw = xwHoist + tr * d3 + j;
      set4(xz[q], ld4(xw));
      set4(xr[q], ld4(xw + d));
      set4(xx[q], ld4(xw + 2 * d));
    } else if(partX) {
      for(int kc = 0; kc < KCx; ++kc) {
        const float* pp = partX + ((int64_t)kc * b + r) * d3 + j;
        const float4 a0 = ldcg4(pp), a1 = ldcg4(pp + d), a2 = ldcg4(pp + 2 * d);
        add4(xz[q], a0);
        add4(xr[q], a1);
        add4(xx[q], a2);
      }
    }
    set4(hv[q], ldcg4(hin + j));
  }
  float az[GQ][4], ar[GQ][4], ax[GQ][4];
#pragma unroll
  for(int q = 0; q < GQ; ++q) {
    const int64_t g = threadIdx.x + (int64_t)q * RT;
#pragma unroll
    for(int i = 0; i < 4; ++i)
      az[q][i] = ar[q][i] = ax[q][i] = 0.f;
    if(g >= d4)
      continue;
    const int64_t j = 4 * g;
    float* huOut = B.hu + tr * d3 + j;
    if(!p.a.lean_cache) {  // the persistent backward reads only the h-gate third
      st4(huOut, hz[q]);
      st4(huOut + d, hr[q]);
    }
    st4(huOut + 2 * d, hh[q]);
    if(partX && !p.a.lean_cache) {
      float* xo = D.xw2 + tr * d3 + j;
      st4(xo, xz[q]);
      st4(xo + d, xr[q]);
      st4(xo + 2 * d, xx[q]);
    }
    const float4 bz = ld4(B.bias[0] + j), br = ld4(B.bias[1] + j);
    const float bzv[4] = {bz.x, bz.y, bz.z, bz.w}, brv[4] = {br.x, br.y, br.z, br.w};
#pragma unroll
    for(int i = 0; i < 4; ++i) {
      // gruPre: h*U, then + x*W, then + b (graph.cpp:636-644)
      float z = hz[q][i], rr = hr[q][i];
      if(hasX) {
        z = z + xz[q][i];
        rr = rr + xr[q][i];
      }
      az[q][i] = z + bzv[i];
      ar[q][i] = rr + brv[i];
      ax[q][i] = hasX ? xx[q][i] : 0.f;
    }
  }
  if(ln) {  // two-pass statistics per gate (tensor.cpp:545-572)
    float s[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for(int q = 0; q < GQ; ++q)
#pragma unroll
      for(int i = 0; i < 4; ++i) {
        s[0] += az[q][i];
        s[1] += ar[q][i];
        s[2] += ax[q][i];
      }
    block_sums<3>(s, red);
    const float mz = s[0] / (float)d, mr = s[1] / (float)d, mx = s[2] / (float)d;
    float qv[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for(int q = 0; q < GQ; ++q) {
      if(threadIdx.x + (int64_t)q * RT >= d4)
        continue;
#pragma unroll
      for(int i = 0; i < 4; ++i) {
        const float cz = az[q][i] - mz, cr = ar[q][i] - mr, cx = ax[q][i] - mx;
        qv[0] += cz * cz;
        qv[1] += cr * cr;
        qv[2] += cx * cx;
      }
    }
    block_sums<3>(qv, red);
    const float rsz = 1.f / sqrtf(qv[0] / (float)d + p.a.eps);
    const float rsr = 1.f / sqrtf(qv[1] / (float)d + p.a.eps);
    const float rsx = 1.f / sqrtf(qv[2] / (float)d + p.a.eps);
    if(threadIdx.x == 0) {
      B.lnrs[tr * 3] = rsz;
      B.lnrs[tr * 3 + 1] = rsr;
      B.lnrs[tr * 3 + 2] = rsx;
    }
#pragma unroll
    for(int q = 0; q < GQ; ++q) {
      const int64_t g = threadIdx.x + (int64_t)q * RT;
      if(g >= d4)
        continue;
      const int64_t j = 4 * g;
      float* xh = B.lnc + tr * d3 + j;
      const float4 gz = ld4(B.ln[0] + j), bz = ld4(B.ln[1] + j);
      const float4 gr = ld4(B.ln[2] + j), br = ld4(B.ln[3] + j);
      const float gzv[4] = {gz.x, gz.y, gz.z, gz.w}, bzv[4] = {bz.x, bz.y, bz.z, bz.w};
      const float grv[4] = {gr.x, gr.y, gr.z, gr.w}, brv[4] = {br.x, br.y, br.z, br.w};
      float xhz[4], xhr[4], xhx[4];
#pragma unroll
      for(int i = 0; i < 4; ++i) {
        xhz[i] = (az[q][i] - mz) * rsz;
        xhr[i] = (ar[q][i] - mr) * rsr;
        az[q][i] = gzv[i] * xhz[i] + bzv[i];
        ar[q][i] = grv[i] * xhr[i] + brv[i];
      }
      st4(xh, xhz);
      st4(xh + d, xhr);
      if(hasX) {
        const float4 gx = ld4(B.ln[4] + j), bx = ld4(B.ln[5] + j);
        const float gxv[4] = {gx.x, gx.y, gx.z, gx.w}, bxv[4] = {bx.x, bx.y, bx.z, bx.w};
#pragma unroll
        for(int i = 0; i < 4; ++i) {
          xhx[i] = (ax[q][i] - mx) * rsx;
          ax[q][i] = gxv[i] * xhx[i] + bxv[i];
        }
        st4(xh + 2 * d, xhx);
      }
    }
  }
  const float notm = 1.f - blendM;
#pragma unroll
  for(int q = 0; q < GQ; ++q) {
    const int64_t g = threadIdx.x + (int64_t)q * RT;
    if(g >= d4)
      continue;
    const int64_t j = 4 * g;
    const float4 bh = ld4(B.bias[2] + j);
    const float bhv[4] = {bh.x, bh.y, bh.z, bh.w};
    float pv[4] = {0.f, 0.f, 0.f, 0.f};
    if(blend)
      set4(pv, ldcg4(prevRow + j));
    float zc[4], rc[4], hc[4], o[4];
#pragma unroll
    for(int i = 0; i < 4; ++i) {
      const float z = sigm(az[q][i]), rr = sigm(ar[q][i]);
      const float ac = ax[q][i] + (rr * hh[q][i] + bhv[i]);  // graph.cpp:737-738
      const float ht = tanhf(ac);
      zc[i] = z;
      rc[i] = rr;
      hc[i] = ht;
      const float hn = (1.f - z) * ht + z * hv[q][i];
      o[i] = blend ? hn * blendM + pv[i] * notm : hn;  // a*m + b*(1-m)
    }
    float* cache = B.cache + tr * d3 + j;
    st4(cache, zc);
    st4(cache + d, rc);
    st4(cache + 2 * d, hc);
    st4(out + j, o);
  }
}

// Bahdanau attention for batch row r at step t (bahdanau_score_kernel +
// bahdanau_ctx_kernel arithmetic): wq from the partials, scores per
// position (one warp each, float4 lanes, the position's loads in flight
// together), masked softmax, context (float4 columns, positions unrolled).
constexpr int AQ = MAXA / 128;  // float4 groups per lane over the attention width
constexpr int CU = 12;          // positions per batch of loads in the context sums
constexpr int BU = 8;           // positions per batch of loads in the attention backward columns

// Team member `m` of `P` (P CTAs per row, P = 1 without teams): scores of
// the positions j = m, m+P, ... then (P > 1) a team barrier, then the
// context columns of its 1/P share.
__device__ void att_row(const KP& p, int64_t t, int64_t r, int m, int P, unsigned& tepoch,
                        float* sW, float* sE, float* sP, int& np_) {
  mark(p.prof, np_, 8);
  const mtkc_rnn_scan_args& a = p.a;
  const int64_t b = a.b, A = a.a, S = a.S, KD = a.kd, A4 = A / 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tr = t * b + r;
  for(int64_t c4 = threadIdx.x; c4 < A4; c4 += RT) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    for(int kc = 0; kc < p.KCq; ++kc)
      add4(v, ldcg4(p.partQ + ((int64_t)kc * b + r) * A + 4 * c4));
    st4(sW + 4 * c4, v);
    if(m == 0)
      st4(a.wq + tr * A + 4 * c4, v);
  }
  __syncthreads();
  mark(p.prof, np_, 9);
  const bool ln = a.attLnG != nullptr;
  const int nq = (int)((A4 + 31) / 32);  // groups per lane (<= AQ)
  for(int64_t j = m + (int64_t)warp * P; j < S; j += (int64_t)(RT / 32) * P) {
    const int64_t rj = r * S + j;    // row of uk / keys
    const int64_t trj = tr * S + j;  // row of the per-step caches
    const float* uk = a.uk + rj * A;
    float x[AQ][4];
#pragma unroll
    for(int q = 0; q < AQ; ++q) {
      const int64_t c4 = lane + 32 * q;
      if(q < nq && c4 < A4) {
        const float4 u = ld4(uk + 4 * c4);
        const float4 w = *reinterpret_cast<const float4*>(sW + 4 * c4);
        x[q][0] = w.x + u.x;
        x[q][1] = w.y + u.y;
        x[q][2] = w.z + u.z;
        x[q][3] = w.w + u.w;
      } else {
        x[q][0] = x[q][1] = x[q][2] = x[q][3] = 0.f;
      }
    }
    float mu = 0.f, rs = 0.f;
    if(ln) {
      float s1 = 0.f;
#pragma unroll
      for(int q = 0; q < AQ; ++q)
        s1 += (x[q][0] + x[q][1]) + (x[q][2] + x[q][3]);
      mu = warp_sum(s1) / (float)A;
      float s2 = 0.f;
#pragma unroll
      for(int q = 0; q < AQ; ++q) {
        const int64_t c4 = lane + 32 * q;
        if(q < nq && c4 < A4)
#pragma unroll
          for(int i = 0; i < 4; ++i) {
            const float dd = x[q][i] - mu;
            s2 += dd * dd;
          }
      }
      rs = 1.f / sqrtf(warp_sum(s2) / (float)A + a.eps);
      if(lane == 0)
        a.attLnrs[trj] = rs;
    }
    float acc = 0.f;
#pragma unroll
    for(int q = 0; q < AQ; ++q) {
      const int64_t c4 = lane + 32 * q;
      if(q >= nq || c4 >= A4)
        continue;
      const int64_t c = 4 * c4;
      if(ln) {
        float xh[4];
        const float4 g = ld4(a.attLnG + c), bb = ld4(a.attLnB + c);
        const float gv[4] = {g.x, g.y, g.z, g.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for(int i = 0; i < 4; ++i) {
          xh[i] = (x[q][i] - mu) * rs;
          x[q][i] = gv[i] * xh[i] + bv[i];
        }
        st4(a.attLnx + trj * A + c, xh);
      }
      const float4 vv = ld4(a.attV + c);
      const float vvv[4] = {vv.x, vv.y, vv.z, vv.w};
      float th[4];
#pragma unroll
      for(int i = 0; i < 4; ++i) {
        th[i] = tanhf(x[q][i]);
        acc += th[i] * vvv[i];
      }
      st4(a.attT + trj * A + c, th);
    }
    acc = warp_sum(acc);
    if(lane == 0) {
      sE[j] = acc;
      if(P > 1)
        p.teamBuf[r * S + j] = acc;
    }
  }
  if(P > 1) {  // every member needs all scores
    team_bar(p.teamCtr + r, (unsigned)P, tepoch);
    for(int64_t j = threadIdx.x; j < S; j += RT)
      sE[j] = __ldcg(p.teamBuf + r * S + j);
  }
  __syncthreads();
  mark(p.prof, np_, 11);
  if(warp == 0) {  // masked softmax over positions (tensor.cpp:393-440)
    const float* mk = a.attMask ? a.attMask + r * S : nullptr;
    float mx = -INFINITY;
    int any = 0;
    for(int64_t j = lane; j < S; j += 32)
      if(!mk || mk[j] != 0.f) {
        mx = fmaxf(mx, sE[j]);
        any = 1;
      }
    mx = warp_max(mx);
    any = __any_sync(0xffffffffu, any);
    if(!any && lane == 0 && a.flags && m == 0)
      atomicOr(a.flags, MTKC_FLAG_MASKED_ROW);
    float sum = 0.f;
    for(int64_t j = lane; j < S; j += 32)
      if(!mk || mk[j] != 0.f)
        sum += expf(sE[j] - mx);
    sum = warp_sum(sum);
    for(int64_t j = lane; j < S; j += 32) {
      const float y = (any && (!mk || mk[j] != 0.f)) ? expf(sE[j] - mx) / sum : 0.f;
      sP[j] = y;
      if(m == 0)
        a.attWts[tr * S + j] = y;
    }
  }
  __syncthreads();
  mark(p.prof, np_, 12);
  // context: sum over positions in ascending order, 4 positions' loads in
  // flight; this member's share of the columns
  const float* keys = a.keys + r * S * KD;
  const int64_t K4 = KD / 4, kb = K4 * m / P, ke = K4 * (m + 1) / P;
  // (CU positions' loads in flight per thread: the loop is L2-latency bound)
  for(int64_t k4 = kb + threadIdx.x; k4 < ke; k4 += RT) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for(int64_t j = 0; j < S; j += CU) {
      float4 kv[CU];
#pragma unroll
      for(int u = 0; u < CU; ++u)
        kv[u] = j + u < S ? ld4(keys + (j + u) * KD + 4 * k4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for(int u = 0; u < CU; ++u) {
        if(j + u >= S)
          break;
        const float w = sP[j + u];
        acc[0] += w * kv[u].x;
        acc[1] += w * kv[u].y;
        acc[2] += w * kv[u].z;
        acc[3] += w * kv[u].w;
      }
    }
    st4(a.ctx + tr * KD + 4 * k4, acc);
  }
  __syncthreads();  // sW / sE / sP are reused by the next row
}

// ------------------------------------------------------------ kernel

constexpr size_t SMEM_BYTES = 1024 + RST * (size_t)(A_STAGE + B_STAGE) +
                              (MAXA + 2 * MAXS + 6 * 32) * sizeof(float) + 256;
constexpr size_t SMEM_BYTES_B = SMEM_BYTES + MAXS * sizeof(float) + 64;

__global__ void __launch_bounds__(RT, 1)
    rnn_scan_fwd_kernel(const __grid_constant__ Maps maps, const __grid_constant__ KP p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Smem sm;
  sm.sA = base;
  sm.sB = base + RST * A_STAGE;
  float* sW = (float*)(sm.sB + RST * B_STAGE);
  float* sE = sW + MAXA;
  float* sP = sE + MAXS;
  float* red = sP + MAXS;
  uint64_t* bars = (uint64_t*)(red + 6 * 32);
  sm.full = bars;
  sm.empty = bars + RST;
  sm.tfull = bars + 2 * RST;
  sm.tempty = bars + 2 * RST + 2;
  uint32_t* tmemSlot = (uint32_t*)(bars + 2 * RST + 4);
  const int warp = threadIdx.x >> 5;
  const mtkc_rnn_scan_args& a = p.a;

  if(threadIdx.x == 0) {
    for(int s = 0; s < RST; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for(int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for(int q = 0; q < a.ndir; ++q) {
      prefetch_tmap(&maps.hh[q]);
      prefetch_tmap(&maps.sout[q]);
      prefetch_tmap(&maps.ut[q]);
    }
    if(a.has_att) {
      prefetch_tmap(&maps.ctx);
      prefetch_tmap(&maps.w2t);
      prefetch_tmap(&maps.watt);
    }
  }
  if(warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmemSlot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  sm.tmem = *tmemSlot;

  const int gs = gridDim.x / a.ndir;
  const int dir = blockIdx.x / gs, gi = blockIdx.x % gs;
  const mtkc_rnn_dir& D = a.dir[dir];
  unsigned* ctr = p.ctr + dir;
  unsigned epoch = 0;
  uint32_t ring = 0, ucnt = 0;
  unsigned tepoch = 0;  // team barriers passed (every row of this CTA, in order)
  int npf = 0;
  const int64_t b = a.b, T = a.T, d = a.d, d3 = 3 * d;
  const int K = D.nblocks;
  const int mT = (int)((b + 127) / 128);

  if(p.prof) {  // barrier microbenchmark: 200 back-to-back barriers
    mark(p.prof, npf, 7);
    for(int q = 0; q < 200; ++q)
      grid_bar(ctr, gs, epoch);
    mark(p.prof, npf, 5);
  }
  for(int64_t i = 0; i < T; ++i) {
    const int64_t t = D.reverse ? T - 1 - i : i;
    const int64_t hp = D.reverse ? t + 1 : t, hs = D.reverse ? t : t + 1;
    for(int k = 0; k < K; ++k) {
      const bool attIn = a.has_att && k == 1;
      Prod P[2];
      int np = 1;
      P[0].ma = k == 0 ? &maps.hh[dir] : &maps.sout[dir];
      P[0].mb = &maps.ut[dir];
      P[0].aRow0 = (int)(k == 0 ? hp * b : (int64_t)(k - 1) * T * b + t * b);
      P[0].bRow0 = (int)(k * d3);
      P[0].N = (int)d3;
      P[0].NT = NTH;
      P[0].KC = p.KCh;
      P[0].KS = (int)(d / p.KCh);
      P[0].nT = (int)(d3 / NTH);
      P[0].mT = mT;
      P[0].part = p.partHu[dir];
      if(attIn) {
        P[1].ma = &maps.ctx;
        P[1].mb = &maps.w2t;
        P[1].aRow0 = (int)(t * b);
        P[1].bRow0 = 0;
        P[1].N = (int)d3;
        P[1].NT = NTH;
        P[1].KC = p.KCx;
        P[1].KS = (int)(a.kd / p.KCx);
        P[1].nT = (int)(d3 / NTH);
        P[1].mT = mT;
        P[1].part = p.partX;
        np = 2;
      }
      mark(p.prof, npf, attIn ? 4 : 0);
      run_prods(P, np, gi, gs, sm, ring, ucnt, b);
      mark(p.prof, npf, 5);
      grid_bar(ctr, gs, epoch);
      mark(p.prof, npf, 1);
      const bool last = k == K - 1;
      for(int64_t r = gi; r < b; r += gs) {
        const float* hin = k == 0 ? D.HH + (hp * b + r) * d : D.sout + (((int64_t)(k - 1) * T + t) * b + r) * d;
        float* out = last ? D.HH + (hs * b + r) * d : D.sout + (((int64_t)k * T + t) * b + r) * d;
        const bool blend = last && a.maskT != nullptr;
        const float m = blend ? a.maskT[t * b + r] : 1.f;
        gru_row(p, D, k, t, r, hin, p.partHu[dir], p.KCh, attIn ? p.partX : nullptr, p.KCx,
                k == 0 ? D.xw1 : nullptr, out, D.HH + (hp * b + r) * d, m, blend, red);
      }
      mark(p.prof, npf, 5);
      grid_bar(ctr, gs, epoch);
      if(a.has_att && k == 0) {
        Prod Q;
        Q.ma = &maps.sout[dir];
        Q.mb = &maps.watt;
        Q.aRow0 = (int)(t * b);  // block 1's output (sout block 0)
        Q.bRow0 = 0;
        Q.N = (int)a.a;
        Q.NT = p.NTq;
        Q.KC = p.KCq;
        Q.KS = (int)(d / p.KCq);
        Q.nT = (int)(a.a / p.NTq);
        Q.mT = mT;
        Q.part = p.partQ;
        mark(p.prof, npf, 2);
        run_prods(&Q, 1, gi, gs, sm, ring, ucnt, b);
        mark(p.prof, npf, 5);
        grid_bar(ctr, gs, epoch);
        mark(p.prof, npf, 3);
        for(int64_t u = gi; u < b * p.team; u += gs)  // team member u % team of row u / team
          att_row(p, t, u / p.team, (int)(u % p.team), p.team, tepoch, sW, sE, sP, npf);
        mark(p.prof, npf, 5);
        grid_bar(ctr, gs, epoch);
      }
    }
  }
  mark(p.prof, npf, 6);
  tc_fence_before();
  __syncthreads();
  if(warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem),
                 "r"(TMEM_COLS));
}

// ------------------------------------------------------------ backward
//
// Reverse sweep, per step and block k = K-1 .. 0 (backwardStep in
// csrc/host/rnn_scan.cpp; gru_bwd_kernel / bahdanau_*_kernel arithmetic):
//   PWB    one CTA per row: the block's output gradient = direct term
//          (go*z of the block above, or the state slot) + the K-split
//          partials of the product phase that fed it; GRU (+LN) backward;
//          writes dG = [dpz|dpr|duh] (the next product's A operand), dGx,
//          dac, LN partials and the direct part of the input gradient;
//   PRODB  d(input) = dG * [Uz|Ur|Uh]^T (K = 3d) as K-split partials, plus
//          (block 2 of the decoder) d(ctx) = dGx * [Wz|Wr|Wx]^T;
//   ATTB   (decoder) one CTA per row: d(ctx) sum, d(weights) against the
//          keys, softmax backward, LN backward, d(uk) (accumulated over
//          steps), d(wq) and the v / LN partials; then PRODQ: the query
//          projection's input gradient dwq * W^T feeding block 1.

struct BMaps {
  CUtensorMap dg[2];  // A: [K*T*b x 3d] per direction
  CUtensorMap uh[2];  // B: [K*d x 3d] per direction ([Uz|Ur|Uh] side by side)
  CUtensorMap dgx;    // A: block-2 [dpz|dpr|dax] [T*b x 3d]
  CUtensorMap w2c;    // B: [kd x 3d] ([Wz|Wr|Wx] side by side)
  CUtensorMap dwq;    // A: [T*b x a]
  CUtensorMap watt;   // B: attention W as stored [d x a]
};

struct BKP {
  mtkc_rnn_scan_args a;
  float* partB[2];  // [KCb][b][d] per direction
  float* partC;     // [KCc][b][kd]
  float* partQ;     // [KCq][b][d]
  float* dsd[2];    // [K-1][b][d] per direction: direct term go*z into the block below
  unsigned* ctr;
  unsigned long long* prof;
  int KCb, KCc, KCq, NTb, NTc;
  int team;           // CTAs per batch row in the attention phase (see KP)
  unsigned* teamCtr;  // [b]
  float* teamBuf;     // [b x S x 2]
};

__device__ void gru_bwd_row(const BKP& p, const mtkc_rnn_dir& D, int dir, int k, int64_t t,
                            int64_t r, int64_t hp, const float* base, const float* partIn,
                            const float* partQ2, bool blend, float blendM, float* red) {
  const mtkc_rnn_scan_args& a = p.a;
  const int64_t b = a.b, T = a.T, d = a.d, d3 = 3 * d, d4 = d / 4;
  const int K = D.nblocks;
  const mtkc_rnn_block& B = D.blk[k];
  const bool ln = B.ln[0] != nullptr;
  const bool hasX = (k == 0 && D.xw1 != nullptr) || (k == 1 && a.has_att);
  const int64_t tr = t * b + r;
  const float* sIn = k == 0 ? D.HH + (hp * b + r) * d : D.sout + (((int64_t)(k - 1) * T + t) * b + r) * d;
  float* ghp = D.GH + (hp * b + r) * d;
  const float notm = 1.f - blendM;
  float g0[GQ][4], z[GQ][4], rr[GQ][4], ht[GQ][4], uh[GQ][4], hv[GQ][4];
#pragma unroll
  for(int q = 0; q < GQ; ++q) {
    const int64_t g = threadIdx.x + (int64_t)q * RT;
#pragma unroll
    for(int i = 0; i < 4; ++i)
      g0[q][i] = z[q][i] = rr[q][i] = ht[q][i] = uh[q][i] = hv[q][i] = 0.f;
    if(g >= d4)
      continue;
    const int64_t j = 4 * g;
    set4(g0[q], ldcg4(base + j));
    if(partIn)
      for(int kc = 0; kc < p.KCb; ++kc)
        add4(g0[q], ldcg4(partIn + ((int64_t)kc * b + r) * d + j));
    if(partQ2)
      for(int kc = 0; kc < p.KCq; ++kc)
        add4(g0[q], ldcg4(partQ2 + ((int64_t)kc * b + r) * d + j));
    const float* cache = B.cache + tr * d3 + j;
    set4(z[q], ld4(cache));
    set4(rr[q], ld4(cache + d));
    set4(ht[q], ld4(cache + 2 * d));
    set4(uh[q], ld4(B.hu + tr * d3 + 2 * d + j));
    set4(hv[q], ldcg4(sIn + j));
  }
  float daz[GQ][4], dar[GQ][4], dac[GQ][4], duh[GQ][4];
#pragma unroll
  for(int q = 0; q < GQ; ++q) {  // graph.cpp:755-792
    const int64_t g = threadIdx.x + (int64_t)q * RT;
#pragma unroll
    for(int i = 0; i < 4; ++i)
      daz[q][i] = dar[q][i] = dac[q][i] = duh[q][i] = 0.f;
    if(g >= d4)
      continue;
    const int64_t j = 4 * g;
    float ghv[4], gp[4];
#pragma unroll
    for(int i = 0; i < 4; ++i) {
      const float gg = blend ? g0[q][i] * blendM : g0[q][i];  // maskBlend backward
      const float dz = gg * (hv[q][i] - ht[q][i]);
      const float dht = gg * (1.f - z[q][i]);
      ghv[i] = gg * z[q][i];
      gp[i] = g0[q][i] * notm;
      const float c = dht * (1.f - ht[q][i] * ht[q][i]);
      const float dr = c * uh[q][i];
      duh[q][i] = c * rr[q][i];
      dac[q][i] = c;
      daz[q][i] = dz * z[q][i] * (1.f - z[q][i]);
      dar[q][i] = dr * rr[q][i] * (1.f - rr[q][i]);
    }
    if(k == 0) {  // input = the previous state slot (accumulating)
      float o[4];
      set4(o, ldcg4(ghp + j));
#pragma unroll
      for(int i = 0; i < 4; ++i)
        o[i] = (blend && K == 1) ? (o[i] + ghv[i]) + gp[i] : o[i] + ghv[i];
      st4(ghp + j, o);
    } else {
      st4(p.dsd[dir] + ((int64_t)(k - 1) * b + r) * d + j, ghv);
      if(blend) {  // last block: gprev (+)= go*(1-m)
        float o[4];
        set4(o, ldcg4(ghp + j));
#pragma unroll
        for(int i = 0; i < 4; ++i)
          o[i] += gp[i];
        st4(ghp + j, o);
      }
    }
  }
  float dpz[GQ][4], dpr[GQ][4], dax[GQ][4];
#pragma unroll
  for(int q = 0; q < GQ; ++q)
#pragma unroll
    for(int i = 0; i < 4; ++i) {
      dpz[q][i] = daz[q][i];
      dpr[q][i] = dar[q][i];
      dax[q][i] = dac[q][i];
    }
  const float fd = (float)d;
  if(ln) {
    const float rsz = B.lnrs[tr * 3], rsr = B.lnrs[tr * 3 + 1], rsx = B.lnrs[tr * 3 + 2];
    float xz[GQ][4], xr[GQ][4], xx[GQ][4], gz[GQ][4], gr[GQ][4], gx[GQ][4];
    float s[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for(int q = 0; q < GQ; ++q) {
      const int64_t g = threadIdx.x + (int64_t)q * RT;
#pragma unroll
      for(int i = 0; i < 4; ++i)
        xz[q][i] = xr[q][i] = xx[q][i] = gz[q][i] = gr[q][i] = gx[q][i] = 0.f;
      if(g >= d4)
        continue;
      const int64_t j = 4 * g;
      const float* xh = B.lnc + tr * d3 + j;
      set4(xz[q], ld4(xh));
      set4(xr[q], ld4(xh + d));
      set4(gz[q], ld4(B.ln[0] + j));
      set4(gr[q], ld4(B.ln[2] + j));
      if(hasX) {
        set4(xx[q], ld4(xh + 2 * d));
        set4(gx[q], ld4(B.ln[4] + j));
      }
#pragma unroll
      for(int i = 0; i < 4; ++i) {
        const float hz = daz[q][i] * gz[q][i], hr = dar[q][i] * gr[q][i];
        s[0] += hz;
        s[1] += hz * xz[q][i];
        s[2] += hr;
        s[3] += hr * xr[q][i];
        if(hasX) {
          const float hx = dac[q][i] * gx[q][i];
          s[4] += hx;
          s[5] += hx * xx[q][i];
        }
      }
    }
    block_sums<6>(s, red);
#pragma unroll
    for(int q = 0; q < GQ; ++q) {
      const int64_t g = threadIdx.x + (int64_t)q * RT;
      if(g >= d4)
        continue;
      const int64_t j = 4 * g;
      float l0[4], l1[4], l2[4], l3[4], l4[4], l5[4];
#pragma unroll
      for(int i = 0; i < 4; ++i) {
        dpz[q][i] = rsz * (daz[q][i] * gz[q][i] - s[0] / fd - xz[q][i] * (s[1] / fd));
        dpr[q][i] = rsr * (dar[q][i] * gr[q][i] - s[2] / fd - xr[q][i] * (s[3] / fd));
        l0[i] = daz[q][i] * xz[q][i];
        l1[i] = daz[q][i];
        l2[i] = dar[q][i] * xr[q][i];
        l3[i] = dar[q][i];
        if(hasX) {
          dax[q][i] = rsx * (dac[q][i] * gx[q][i] - s[4] / fd - xx[q][i] * (s[5] / fd));
          l4[i] = dac[q][i] * xx[q][i];
          l5[i] = dac[q][i];
        }
      }
      float* lp = B.lnp + tr * 6 * d + j;
      st4(lp, l0);
      st4(lp + d, l1);
      st4(lp + 2 * d, l2);
      st4(lp + 3 * d, l3);
      if(hasX) {
        st4(lp + 4 * d, l4);
        st4(lp + 5 * d, l5);
      }
    }
  }
#pragma unroll
  for(int q = 0; q < GQ; ++q) {
    const int64_t g = threadIdx.x + (int64_t)q * RT;
    if(g >= d4)
      continue;
    const int64_t j = 4 * g;
    float* dg = D.dG + (((int64_t)k * T + t) * b + r) * d3 + j;
    st4(dg, dpz[q]);
    st4(dg + d, dpr[q]);
    st4(dg + 2 * d, duh[q]);
    if(B.dGx) {
      float* dx = B.dGx + tr * d3 + j;
      st4(dx, dpz[q]);
      st4(dx + d, dpr[q]);
      st4(dx + 2 * d, dax[q]);
    }
    st4(B.dac + tr * d + j, dac[q]);
  }
}

__device__ void att_bwd_row(const BKP& p, int64_t ii, int64_t t, int64_t r, int m, int P,
                            unsigned& tepoch, float* sC, float* sE, float* sP, float* sQ,
                            float* scratch, int& np_) {
  mark(p.prof, np_, 8);
  const mtkc_rnn_scan_args& a = p.a;
  const int64_t b = a.b, T = a.T, A = a.a, S = a.S, KD = a.kd, A4 = A / 4, K4 = KD / 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tr = t * b + r, TB = T * b;
  for(int64_t k4 = threadIdx.x; k4 < K4; k4 += RT) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if(a.ctxGrad)
      set4(v, ld4(a.ctxGrad + tr * KD + 4 * k4));
    for(int kc = 0; kc < p.KCc; ++kc)
      add4(v, ldcg4(p.partC + ((int64_t)kc * b + r) * KD + 4 * k4));
    st4(sC + 4 * k4, v);
    if(m == 0)
      st4(a.dctx + tr * KD + 4 * k4, v);
  }
  __syncthreads();
  mark(p.prof, np_, 9);
  // d(weights)_j = dctx . keys_j  (bahdanau_dw_kernel; the key gradient
  // sum_t w_tj dctx_t is one batched product after the sweep); positions
  // j = m, m+P, ... of this team member
  for(int64_t j = m + (int64_t)warp * P; j < S; j += (int64_t)(RT / 32) * P) {
    const float* keys = a.keys + (r * S + j) * KD;
    float acc = 0.f;
    // every key load of the lane issued before the sums (K4 <= MAXA / 4):
    // same (chunk, u) summation order as a 4-wide loop over c4 = lane + 128 i
    float4 kv[MAXA / 128];
#pragma unroll
    for(int q = 0; q < MAXA / 128; ++q) {
      const int64_t cc = lane + 32 * q;
      kv[q] = cc < K4 ? ld4(keys + 4 * cc) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for(int q = 0; q < MAXA / 128; ++q) {
      const int64_t cc = lane + 32 * q;
      if(cc < K4) {
        const float4 cv = *reinterpret_cast<const float4*>(sC + 4 * cc);
        acc += cv.x * kv[q].x + cv.y * kv[q].y + cv.z * kv[q].z + cv.w * kv[q].w;
      }
    }
    acc = warp_sum(acc);
    if(lane == 0) {
      sE[j] = acc;
      if(P > 1)
        p.teamBuf[(r * S + j) * 2] = acc;
    }
  }
  if(P > 1) {
    team_bar(p.teamCtr + r, (unsigned)P, tepoch);
    for(int64_t j = threadIdx.x; j < S; j += RT)
      sE[j] = __ldcg(p.teamBuf + (r * S + j) * 2);
  }
  __syncthreads();
  mark(p.prof, np_, 11);
  if(warp == 0) {  // softmax backward: de_j = w_j (dw_j - sum_l w_l dw_l)
    float s = 0.f;
    for(int64_t j = lane; j < S; j += 32)
      s += a.attWts[tr * S + j] * sE[j];
    s = warp_sum(s);
    __syncwarp();
    for(int64_t j = lane; j < S; j += 32)
      sE[j] = a.attWts[tr * S + j] * (sE[j] - s);
  }
  __syncthreads();
  mark(p.prof, np_, 12);
  const bool ln = a.attLnG != nullptr;
  if(ln) {  // LN backward row statistics per position (bahdanau_de_kernel)
    for(int64_t j = m + (int64_t)warp * P; j < S; j += (int64_t)(RT / 32) * P) {
      const int64_t trj = tr * S + j;
      const float dej = sE[j];
      float s1 = 0.f, s2 = 0.f;
      for(int64_t c4 = lane; c4 < A4; c4 += 32) {
        const float4 tv = ld4(a.attT + trj * A + 4 * c4), xh = ld4(a.attLnx + trj * A + 4 * c4);
        const float4 vv = ld4(a.attV + 4 * c4), gg = ld4(a.attLnG + 4 * c4);
        const float tt[4] = {tv.x, tv.y, tv.z, tv.w}, xx[4] = {xh.x, xh.y, xh.z, xh.w};
        const float v4[4] = {vv.x, vv.y, vv.z, vv.w}, g4[4] = {gg.x, gg.y, gg.z, gg.w};
#pragma unroll
        for(int i = 0; i < 4; ++i) {
          const float h = ((dej * v4[i]) * (1.f - tt[i] * tt[i])) * g4[i];
          s1 += h;
          s2 += h * xx[i];
        }
      }
      s1 = warp_sum(s1) / (float)A;
      s2 = warp_sum(s2) / (float)A;
      if(lane == 0) {
        sP[j] = s1;
        sQ[j] = s2;
        if(P > 1) {
          p.teamBuf[(r * S + j) * 2] = s1;
          p.teamBuf[(r * S + j) * 2 + 1] = s2;
        }
      }
    }
    if(P > 1) {
      team_bar(p.teamCtr + r, (unsigned)P, tepoch);
      for(int64_t j = threadIdx.x; j < S; j += RT) {
        sP[j] = __ldcg(p.teamBuf + (r * S + j) * 2);
        sQ[j] = __ldcg(p.teamBuf + (r * S + j) * 2 + 1);
      }
    }
    __syncthreads();
  }
  mark(p.prof, np_, 13);
  // per column (bahdanau_cols_kernel): d(uk), d(wq), v / LN partials;
  // four positions' loads in flight
  const bool acc = ii > 0 || a.acc_uk;
  const int64_t cb = A4 * m / P, ce = A4 * (m + 1) / P;  // this member's columns
  // fewer column groups than threads: `sp` thread groups split the positions
  // of each column (j = part, part + sp, ...), combined in part order below
  const int64_t Cn = ce - cb;
  const int sp = Cn >= RT ? 1 : (int)std::min<int64_t>(4, RT / std::max<int64_t>(Cn, 1));
  const int part = sp > 1 ? (int)(threadIdx.x / Cn) : 0;
  const int64_t cfirst = sp > 1 ? cb + threadIdx.x % Cn : cb + threadIdx.x;
  const int64_t cstep = sp > 1 ? ce : RT;  // one column per thread when split
  for(int64_t c4 = cfirst; part < sp && c4 < ce; c4 += cstep) {
    const int64_t c = 4 * c4;
    const float4 vv = ld4(a.attV + c);
    const float vc[4] = {vv.x, vv.y, vv.z, vv.w};
    float gc[4] = {0.f, 0.f, 0.f, 0.f};
    if(ln)
      set4(gc, ld4(a.attLnG + c));
    float awq[4] = {0.f, 0.f, 0.f, 0.f}, av[4] = {0.f, 0.f, 0.f, 0.f};
    float ag[4] = {0.f, 0.f, 0.f, 0.f}, ab[4] = {0.f, 0.f, 0.f, 0.f};
    for(int64_t j0 = part; j0 < S; j0 += BU * sp) {
      float4 tv[BU], xv[BU], gv[BU];
#pragma unroll
      for(int u = 0; u < BU; ++u) {
        const int64_t j = j0 + u * sp;
        if(j < S) {
          tv[u] = ld4(a.attT + (tr * S + j) * A + c);
          xv[u] = ln ? ld4(a.attLnx + (tr * S + j) * A + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          gv[u] = acc ? ldcg4(a.guk + (r * S + j) * A + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for(int u = 0; u < BU; ++u) {
        const int64_t j = j0 + u * sp;
        if(j >= S)
          break;
        const float dej = sE[j];
        const float tt[4] = {tv[u].x, tv[u].y, tv[u].z, tv[u].w};
        const float xx[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
        float gu[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
        const float rs = ln ? a.attLnrs[tr * S + j] : 0.f;
#pragma unroll
        for(int i = 0; i < 4; ++i) {
          av[i] += tt[i] * dej;
          const float dln = (dej * vc[i]) * (1.f - tt[i] * tt[i]);
          float ds = dln;
          if(ln) {
            ag[i] += dln * xx[i];
            ab[i] += dln;
            ds = rs * (dln * gc[i] - sP[j] - xx[i] * sQ[j]);
          }
          gu[i] = acc ? gu[i] + ds : ds;
          awq[i] += ds;
        }
        st4(a.guk + (r * S + j) * A + c, gu);
      }
    }
    if(sp > 1) {  // partial sums of this part -> scratch [sp][Cn][16]
      float* dst = scratch + ((int64_t)part * Cn + (c4 - cb)) * 16;
      st4(dst, awq);
      st4(dst + 4, av);
      st4(dst + 8, ag);
      st4(dst + 12, ab);
      continue;
    }
    st4(a.dwq + tr * A + c, awq);
    st4(a.vpart + tr * A + c, av);
    if(ln) {
      st4(a.vpart + TB * A + tr * A + c, ag);
      st4(a.vpart + 2 * TB * A + tr * A + c, ab);
    }
  }
  if(sp > 1) {
    __syncthreads();
    for(int64_t k = threadIdx.x; k < Cn; k += RT) {
      float q[16];
      for(int i = 0; i < 16; ++i)
        q[i] = 0.f;
      for(int pp = 0; pp < sp; ++pp) {  // fixed part order
        const float* src = scratch + ((int64_t)pp * Cn + k) * 16;
        for(int i = 0; i < 16; ++i)
          q[i] += src[i];
      }
      const int64_t c = 4 * (cb + k);
      const float awq[4] = {q[0], q[1], q[2], q[3]}, av[4] = {q[4], q[5], q[6], q[7]};
      const float ag[4] = {q[8], q[9], q[10], q[11]}, ab[4] = {q[12], q[13], q[14], q[15]};
      st4(a.dwq + tr * A + c, awq);
      st4(a.vpart + tr * A + c, av);
      if(ln) {
        st4(a.vpart + TB * A + tr * A + c, ag);
        st4(a.vpart + 2 * TB * A + tr * A + c, ab);
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(RT, 1)
    rnn_scan_bwd_kernel(const __grid_constant__ BMaps maps, const __grid_constant__ BKP p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Smem sm;
  sm.sA = base;
  sm.sB = base + RST * A_STAGE;
  float* sC = (float*)(sm.sB + RST * B_STAGE);
  float* sE = sC + MAXA;
  float* sP = sE + MAXS;
  float* red = sP + MAXS;
  uint64_t* bars = (uint64_t*)(red + 6 * 32);
  sm.full = bars;
  sm.empty = bars + RST;
  sm.tfull = bars + 2 * RST;
  sm.tempty = bars + 2 * RST + 2;
  uint32_t* tmemSlot = (uint32_t*)(bars + 2 * RST + 4);
  float* sQ = (float*)(tmemSlot + 4);
  const int warp = threadIdx.x >> 5;
  const mtkc_rnn_scan_args& a = p.a;
  if(threadIdx.x == 0) {
    for(int s = 0; s < RST; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for(int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for(int q = 0; q < a.ndir; ++q) {
      prefetch_tmap(&maps.dg[q]);
      prefetch_tmap(&maps.uh[q]);
    }
    if(a.has_att) {
      prefetch_tmap(&maps.dgx);
      prefetch_tmap(&maps.w2c);
      prefetch_tmap(&maps.dwq);
      prefetch_tmap(&maps.watt);
    }
  }
  if(warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmemSlot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  sm.tmem = *tmemSlot;

  const int gs = gridDim.x / a.ndir;
  const int dir = blockIdx.x / gs, gi = blockIdx.x % gs;
  const mtkc_rnn_dir& D = a.dir[dir];
  unsigned* ctr = p.ctr + dir;
  unsigned epoch = 0;
  uint32_t ring = 0, ucnt = 0;
  unsigned tepoch = 0;
  int npf = 0;
  const int64_t b = a.b, T = a.T, d = a.d, d3 = 3 * d;
  const int K = D.nblocks;
  const int mT = (int)((b + 127) / 128);

  for(int64_t ii = 0; ii < T; ++ii) {
    const int64_t t = D.reverse ? ii : T - 1 - ii;
    const int64_t hp = D.reverse ? t + 1 : t, hs = D.reverse ? t : t + 1;
    for(int k = K - 1; k >= 0; --k) {
      const bool att1 = a.has_att && k == 1;
      const bool last = k == K - 1;
      mark(p.prof, npf, 1);
      for(int64_t r = gi; r < b; r += gs) {
        const float* baseRow = last ? D.GH + (hs * b + r) * d : p.dsd[dir] + ((int64_t)k * b + r) * d;
        const float* partIn = (!last || ii > 0) ? p.partB[dir] : nullptr;
        const float* partQ2 = (k == 0 && a.has_att) ? p.partQ : nullptr;
        const bool blend = last && a.maskT != nullptr;
        const float m = blend ? a.maskT[t * b + r] : 1.f;
        gru_bwd_row(p, D, dir, k, t, r, hp, baseRow, partIn, partQ2, blend, m, red);
      }
      mark(p.prof, npf, 5);
      grid_bar(ctr, gs, epoch);
      Prod P[2];
      int np = 1;
      P[0].ma = &maps.dg[dir];
      P[0].mb = &maps.uh[dir];
      P[0].aRow0 = (int)(((int64_t)k * T + t) * b);
      P[0].bRow0 = (int)(k * d);
      P[0].N = (int)d;
      P[0].NT = p.NTb;
      P[0].KC = p.KCb;
      P[0].KS = (int)(d3 / p.KCb);
      P[0].nT = (int)(d / p.NTb);
      P[0].mT = mT;
      P[0].part = p.partB[dir];
      if(att1) {
        P[1].ma = &maps.dgx;
        P[1].mb = &maps.w2c;
        P[1].aRow0 = (int)(t * b);
        P[1].bRow0 = 0;
        P[1].N = (int)a.kd;
        P[1].NT = p.NTc;
        P[1].KC = p.KCc;
        P[1].KS = (int)(d3 / p.KCc);
        P[1].nT = (int)(a.kd / p.NTc);
        P[1].mT = mT;
        P[1].part = p.partC;
        np = 2;
      }
      mark(p.prof, npf, att1 ? 4 : 0);
      run_prods(P, np, gi, gs, sm, ring, ucnt, b);
      mark(p.prof, npf, 5);
      grid_bar(ctr, gs, epoch);
      if(att1) {
        mark(p.prof, npf, 3);
        for(int64_t u = gi; u < b * p.team; u += gs)
          att_bwd_row(p, ii, t, u / p.team, (int)(u % p.team), p.team, tepoch, sC, sE, sP, sQ,
                      (float*)sm.sA, npf);
        mark(p.prof, npf, 5);
        grid_bar(ctr, gs, epoch);
        Prod Q;
        Q.ma = &maps.dwq;
        Q.mb = &maps.watt;
        Q.aRow0 = (int)(t * b);
        Q.bRow0 = 0;
        Q.N = (int)d;
        Q.NT = p.NTb;
        Q.KC = p.KCq;
        Q.KS = (int)(a.a / p.KCq);
        Q.nT = (int)(d / p.NTb);
        Q.mT = mT;
        Q.part = p.partQ;
        mark(p.prof, npf, 2);
        run_prods(&Q, 1, gi, gs, sm, ring, ucnt, b);
        mark(p.prof, npf, 5);
        grid_bar(ctr, gs, epoch);
      }
    }
  }
  // the last block-1 product feeds the initial-state slot
  const int64_t h0 = D.reverse ? T : 0;
  for(int64_t r = gi; r < b; r += gs)
    for(int64_t j4 = threadIdx.x; j4 < d / 4; j4 += RT) {
      float v[4];
      set4(v, ldcg4(D.GH + (h0 * b + r) * d + 4 * j4));
      for(int kc = 0; kc < p.KCb; ++kc)
        add4(v, ldcg4(p.partB[dir] + ((int64_t)kc * b + r) * d + 4 * j4));
      st4(D.GH + (h0 * b + r) * d + 4 * j4, v);
    }
  mark(p.prof, npf, 6);
  tc_fence_before();
  __syncthreads();
  if(warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem),
                 "r"(TMEM_COLS));
}

// strided copies into the workspace: dst[r * ldd + c] = src[r * lds + c]
struct CJob {
  const float* src;
  float* dst;
  int rows, cols, lds, ldd;
};
struct CJobs {
  CJob j[2 * 3 * MTKC_RNN_MAX_BLOCKS + 4];
  int n;
};

__global__ void copy_jobs_kernel(const __grid_constant__ CJobs jobs) {
  MTKC_PDL_ENTRY();
  const CJob& J = jobs.j[blockIdx.y];
  const int64_t n4 = (int64_t)J.rows * (J.cols / 4);
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
      i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (J.cols / 4), c = (i % (J.cols / 4)) * 4;
    *reinterpret_cast<float4*>(J.dst + r * J.ldd + c) =
        *reinterpret_cast<const float4*>(J.src + r * J.lds + c);
  }
}

// weight transposes into the workspace: dst[c * rows + r] = src[r * cols + c]
struct TJob {
  const float* src;
  float* dst;
  int rows, cols;
};
constexpr int MAXJOBS = 2 * 3 * MTKC_RNN_MAX_BLOCKS + 4;
struct TJobs {
  TJob j[MAXJOBS];
  int n;
};

__global__ void transpose_jobs_kernel(const __grid_constant__ TJobs jobs) {
  MTKC_PDL_ENTRY();
  __shared__ float tile[32][33];
  const TJob& J = jobs.j[blockIdx.z];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  if(r0 >= J.rows || c0 >= J.cols)
    return;
  for(int y = threadIdx.y; y < 32; y += 8) {
    const int r = r0 + y, c = c0 + threadIdx.x;
    if(r < J.rows && c < J.cols)
      tile[y][threadIdx.x] = J.src[(int64_t)r * J.cols + c];
  }
  __syncthreads();
  for(int y = threadIdx.y; y < 32; y += 8) {
    const int c = c0 + y, r = r0 + threadIdx.x;
    if(r < J.rows && c < J.cols)
      J.dst[(int64_t)c * J.rows + r] = tile[threadIdx.x][y];
  }
}

// ------------------------------------------------------------ host side

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) ==
           cudaSuccess &&
       r == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)q;
  });
  return fn;
}

bool tf32_round() {
  const char* e = getenv("MTK_TMA_TF32");
  return !(e && e[0] == '0');
}

// K-major operand [rows x K] (row-major, ld = K), box 32 x boxRows, SWIZZLE_128B
bool kmap(CUtensorMap* m, const float* p, int64_t K, int64_t rows, uint32_t boxRows) {
  EncodeFn fn = encode_fn();
  if(!fn)
    return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {32, boxRows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, tf32_round() ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
            2, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// largest divisor kc of nkb (k-blocks) with kc <= target
int pick_kc(int nkb, int target) {
  target = std::max(1, std::min(target, nkb));
  for(int kc = target; kc >= 1; --kc)
    if(nkb % kc == 0)
      return kc;
  return 1;
}

struct Plan {
  int G, gs, KCh, KCx, KCq, NTq, team;
  size_t offUT[2], offW2T, offWattT, offPH[2], offPX, offPQ, offTeamBuf, offCtr, total;
};

int grid_size() {
  static int sms = 0;
  if(!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if(sms <= 0)
      sms = 148;
  }
  return sms;
}

Plan make_plan(const mtkc_rnn_scan_args* a) {
  Plan P{};
  const int64_t b = a->b, d = a->d, d3 = 3 * d;
  P.G = grid_size();
  P.G -= P.G % a->ndir;
  P.gs = P.G / a->ndir;
  const int mT = (int)((b + 127) / 128);
  const int nTh = (int)(d3 / NTH);
  P.KCh = pick_kc((int)(d / 32), P.gs / std::max(1, nTh * mT));
  if(const char* e = getenv("MTK_RNN_KCH"))  // tuning override
    P.KCh = pick_kc((int)(d / 32), atoi(e));
  P.KCx = a->has_att ? pick_kc((int)(a->kd / 32), P.gs / std::max(1, nTh * mT)) : 1;
  if(const char* e = getenv("MTK_RNN_KCX"))  // tuning override
    P.KCx = a->has_att ? pick_kc((int)(a->kd / 32), atoi(e)) : 1;
  P.NTq = a->has_att ? (a->a % 64 == 0 ? 64 : 32) : 32;
  P.KCq = a->has_att ? pick_kc((int)(d / 32), P.gs / std::max<int>(1, (int)(a->a / P.NTq) * mT))
                     : 1;
  size_t off = 0;
  auto take = [&](size_t floats) {
    size_t o = off;
    off += (floats * sizeof(float) + 255) / 256 * 256;
    return o;
  };
  for(int q = 0; q < a->ndir; ++q)
    P.offUT[q] = take((size_t)a->dir[q].nblocks * d3 * d);
  if(a->has_att) {
    P.offW2T = take((size_t)d3 * a->kd);
    P.offWattT = take((size_t)a->a * d);
    P.offPX = take((size_t)P.KCx * b * d3);
    P.offPQ = take((size_t)P.KCq * b * a->a);
  }
  for(int q = 0; q < a->ndir; ++q)
    P.offPH[q] = take((size_t)P.KCh * b * d3);
  P.team = a->has_att ? std::max(1, P.gs / (int)b) : 1;
  if(getenv("MTK_RNN_TEAM"))
    P.team = std::max(1, std::min(P.team, atoi(getenv("MTK_RNN_TEAM"))));
  P.offTeamBuf = take((size_t)b * std::max<int64_t>(a->S, 1) * 2);
  P.offCtr = take(64 + (size_t)b);  // grid counters, then one team counter per row
  P.total = off;
  return P;
}

bool supported(const mtkc_rnn_scan_args* a) {
  if(a->b <= 0 || a->T <= 0 || a->d <= 0 || a->d % 32 || a->d > 2048)
    return false;
  if(a->ndir < 1 || a->ndir > 2 || (a->ndir == 2 && a->has_att))
    return false;
  for(int q = 0; q < a->ndir; ++q) {
    const mtkc_rnn_dir& D = a->dir[q];
    if(D.nblocks < 1 || D.nblocks > MTKC_RNN_MAX_BLOCKS)
      return false;
    if(D.nblocks > 1 && !D.sout)
      return false;
  }
  if(a->has_att) {
    if(a->dir[0].nblocks < 2 || a->kd % 32 || a->a % 32 || a->a > MAXA || a->S > MAXS ||
       a->S < 1)
      return false;
  }
  // rows of the A boxes are addressed with 32-bit coordinates
  if((a->T + 1) * a->b * (int64_t)MTKC_RNN_MAX_BLOCKS > (1ll << 31))
    return false;
  return true;
}


struct BPlan {
  int G, gs, KCb, KCc, KCq, NTb, NTc, team;
  size_t offUH[2], offW2C, offPB[2], offPC, offPQ, offDSD[2], offTeamBuf, offCtr, total;
};

BPlan make_bplan(const mtkc_rnn_scan_args* a) {
  BPlan P{};
  const int64_t b = a->b, d = a->d, d3 = 3 * d;
  P.G = grid_size();
  P.G -= P.G % a->ndir;
  P.gs = P.G / a->ndir;
  const int mT = (int)((b + 127) / 128);
  P.NTb = d % 64 == 0 ? 64 : 32;
  P.NTc = a->has_att ? (a->kd % 64 == 0 ? 64 : 32) : 32;
  P.KCb = pick_kc((int)(d3 / 32), P.gs / std::max<int>(1, (int)(d / P.NTb) * mT));
  if(const char* e = getenv("MTK_RNN_KCB"))  // tuning override
    P.KCb = pick_kc((int)(d3 / 32), atoi(e));
  P.KCc = a->has_att ? pick_kc((int)(d3 / 32), P.gs / std::max<int>(1, (int)(a->kd / P.NTc) * mT)) : 1;
  if(const char* e = getenv("MTK_RNN_KCC"))  // tuning override
    P.KCc = a->has_att ? pick_kc((int)(d3 / 32), atoi(e)) : 1;
  P.KCq = a->has_att ? pick_kc((int)(a->a / 32), P.gs / std::max<int>(1, (int)(d / P.NTb) * mT)) : 1;
  size_t off = 0;
  auto take = [&](size_t floats) {
    size_t o = off;
    off += (floats * sizeof(float) + 255) / 256 * 256;
    return o;
  };
  for(int q = 0; q < a->ndir; ++q) {
    P.offUH[q] = take((size_t)a->dir[q].nblocks * d * d3);
    P.offPB[q] = take((size_t)P.KCb * b * d);
    P.offDSD[q] = take((size_t)std::max(1, a->dir[q].nblocks - 1) * b * d);
  }
  if(a->has_att) {
    P.offW2C = take((size_t)a->kd * d3);
    P.offPC = take((size_t)P.KCc * b * a->kd);
    P.offPQ = take((size_t)P.KCq * b * d);
  }
  P.team = a->has_att ? std::max(1, P.gs / (int)b) : 1;
  if(getenv("MTK_RNN_TEAM"))
    P.team = std::max(1, std::min(P.team, atoi(getenv("MTK_RNN_TEAM"))));
  P.offTeamBuf = take((size_t)b * std::max<int64_t>(a->S, 1) * 2);
  P.offCtr = take(64 + (size_t)b);
  P.total = off;
  return P;
}

bool bwd_supported(const mtkc_rnn_scan_args* a) {
  if(!supported(a))
    return false;
  for(int q = 0; q < a->ndir; ++q) {
    const mtkc_rnn_dir& D = a->dir[q];
    if(!D.GH || !D.dG)
      return false;
    for(int k = 0; k < D.nblocks; ++k)
      if(!D.blk[k].dac || (D.blk[k].ln[0] && !D.blk[k].lnp))
        return false;
  }
  if(a->has_att && (a->kd > MAXA || !a->dctx || !a->dwq || !a->guk || !a->vpart ||
                    !a->dir[0].blk[1].dGx))
    return false;
  return true;
}
}  // namespace

// Executed tensor-op FLOPs of one scan launch over the padded b x T grid
// (the roofline basis of bench.py's rnn classes, scaled there to real
// tokens): recurrent products h*U of every block and direction, plus with
// attention ctx*W2 (kd x 3d), the query s1*W (d x a) and the score /
// context contractions (S x a, S x kd per row and step).  The backward
// computes the same products transposed (input gradients; the weight
// gradients are hoisted GEMMs) and the attention backward's two
// contractions again.
static double scan_flops(const mtkc_rnn_scan_args* a, bool bwd) {
  const double bt = (double)a->b * (double)a->T, d = (double)a->d;
  double f = 0.0;
  for(int q = 0; q < a->ndir; ++q)
    f += 2.0 * bt * d * 3.0 * d * a->dir[q].nblocks;
  if(a->has_att) {
    const double S = (double)a->S, A = (double)a->a, kd = (double)a->kd;
    f += 2.0 * bt * (kd * 3.0 * d + d * A) + 2.0 * bt * S * (A + kd) * (bwd ? 2.0 : 1.0);
  }
  return f;
}

extern "C" {

int mtkc_rnn_scan_supported(const mtkc_rnn_scan_args* a) { return supported(a) ? 1 : 0; }

size_t mtkc_rnn_scan_workspace(const mtkc_rnn_scan_args* a) {
  if(!supported(a))
    return 0;
  return make_plan(a).total;
}

int mtkc_rnn_scan_forward(const mtkc_rnn_scan_args* a, void* stream) {
  if(!supported(a))
    return fail(MTKC_CONTRACT, "rnn scan: dimensions not supported by the persistent path");
  const Plan P = make_plan(a);
  if(!a->workspace || a->workspace_bytes < P.total)
    return fail(MTKC_CONTRACT, "rnn scan: workspace too small");
  cudaStream_t st = S(stream);
  uint8_t* ws = (uint8_t*)a->workspace;
  const int64_t b = a->b, T = a->T, d = a->d, d3 = 3 * d;
  ProfScope prof(st, "rnn_scan", scan_flops(a, false));

  // K-major weight copies (weights are constant within the step)
  TJobs jobs{};
  for(int q = 0; q < a->ndir; ++q) {
    const mtkc_rnn_dir& D = a->dir[q];
    float* ut = (float*)(ws + P.offUT[q]);
    for(int k = 0; k < D.nblocks; ++k)
      for(int g = 0; g < 3; ++g)
        jobs.j[jobs.n++] = TJob{D.blk[k].U[g], ut + ((int64_t)k * d3 + g * d) * d, (int)d, (int)d};
  }
  if(a->has_att) {
    float* w2t = (float*)(ws + P.offW2T);
    for(int g = 0; g < 3; ++g)
      jobs.j[jobs.n++] = TJob{a->dir[0].blk[1].W[g], w2t + (int64_t)g * d * a->kd, (int)a->kd, (int)d};
    jobs.j[jobs.n++] = TJob{a->attW, (float*)(ws + P.offWattT), (int)d, (int)a->a};
  }
  {
    const int mx = (int)std::max<int64_t>(std::max<int64_t>(d, a->has_att ? a->kd : 0),
                                          a->has_att ? a->a : 0);
    dim3 grid((unsigned)((mx + 31) / 32), (unsigned)((mx + 31) / 32), (unsigned)jobs.n);
    ::mtkc::launch(transpose_jobs_kernel, grid, dim3(32, 8), 0, st, jobs);
    MTKC_POST_LAUNCH("transpose_jobs_kernel");
  }
  if(cudaError_t e = cudaMemsetAsync(ws + P.offCtr, 0, (64 + (size_t)b) * sizeof(float), st))
    return cuda_status(e, "rnn scan counters");

  Maps maps;
  memset(&maps, 0, sizeof(maps));
  bool ok = true;
  for(int q = 0; q < a->ndir; ++q) {
    const mtkc_rnn_dir& D = a->dir[q];
    ok = ok && kmap(&maps.hh[q], D.HH, d, (T + 1) * b, 128);
    ok = ok && kmap(&maps.sout[q], D.nblocks > 1 ? D.sout : D.HH, d,
                    D.nblocks > 1 ? (int64_t)(D.nblocks - 1) * T * b : (T + 1) * b, 128);
    ok = ok && kmap(&maps.ut[q], (const float*)(ws + P.offUT[q]), d, (int64_t)D.nblocks * d3, NTH);
  }
  if(a->has_att) {
    ok = ok && kmap(&maps.ctx, a->ctx, a->kd, T * b, 128);
    ok = ok && kmap(&maps.w2t, (const float*)(ws + P.offW2T), a->kd, d3, NTH);
    ok = ok && kmap(&maps.watt, (const float*)(ws + P.offWattT), d, a->a, (uint32_t)P.NTq);
  }
  if(!ok)
    return fail(MTKC_CUDA, "rnn scan: tensor map encoding failed");

  KP kp;
  memset(&kp, 0, sizeof(kp));
  kp.a = *a;
  for(int q = 0; q < a->ndir; ++q)
    kp.partHu[q] = (float*)(ws + P.offPH[q]);
  kp.partX = a->has_att ? (float*)(ws + P.offPX) : nullptr;
  kp.partQ = a->has_att ? (float*)(ws + P.offPQ) : nullptr;
  kp.ctr = (unsigned*)(ws + P.offCtr);
  kp.KCh = P.KCh;
  kp.KCx = P.KCx;
  kp.KCq = P.KCq;
  kp.NTq = P.NTq;
  kp.team = P.team;
  kp.teamCtr = (unsigned*)(ws + P.offCtr) + 64;
  kp.teamBuf = (float*)(ws + P.offTeamBuf);

  static bool attr = false;
  if(!attr) {
    cudaError_t e = cudaFuncSetAttribute(rnn_scan_fwd_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if(e != cudaSuccess)
      return cuda_status(e, "rnn scan smem attribute");
    attr = true;
  }
  // cooperative launch: every CTA resident (the grid barriers need it); no
  // programmatic serialisation, so no dependent grid can take SMs first
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P.G);
  cfg.blockDim = dim3(RT);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  static unsigned long long* profBuf = nullptr;
  const bool profOn = getenv("MTK_RNN_PROF") != nullptr;
  if(profOn) {
    if(!profBuf)
      cudaMalloc(&profBuf, 8192 * 2 * sizeof(unsigned long long));
    cudaMemsetAsync(profBuf, 0, 8192 * 2 * sizeof(unsigned long long), st);
    kp.prof = profBuf;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, rnn_scan_fwd_kernel, maps, kp);
  if(e != cudaSuccess)
    return cuda_status(e, "rnn_scan_fwd_kernel");
  count_launch();
  if(profOn) {  // phase durations of CTA 0 (kind: 0 PROD h*U, 4 PROD h*U + ctx*W, 1 PW,
              // 2 PROD query, 3 ATT, 5 barrier)
    std::vector<unsigned long long> h(8192 * 2);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), profBuf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double sum[16] = {0}, cnt[16] = {0};
    for(int i = 0; i + 1 < 8192 && h[2 * i + 3]; ++i) {
      int k = (int)h[2 * i];
      sum[k] += (double)(h[2 * i + 3] - h[2 * i + 1]);
      cnt[k] += 1;
    }
    const char* nm[16] = {"prod-hU", "pw", "prod-q", "att", "prod-hU+ctxW", "barrier", "end",
                          "200bars", "att:wq", "att:scores", "-", "att:softmax", "att:context",
                          "-", "-", "-"};
    fprintf(stderr, "[rnn prof] ndir %d b %lld T %lld:", a->ndir, (long long)b, (long long)T);
    for(int k = 0; k < 16; ++k)
      if(cnt[k] > 0)
        fprintf(stderr, " %s %.0f x %.2f us", nm[k], cnt[k], sum[k] / cnt[k] / 1e3);
    fprintf(stderr, "\n");
  }
  return MTKC_OK;
}

size_t mtkc_rnn_scan_bwd_workspace(const mtkc_rnn_scan_args* a) {
  if(!bwd_supported(a))
    return 0;
  return make_bplan(a).total;
}

int mtkc_rnn_scan_backward(const mtkc_rnn_scan_args* a, void* stream) {
  if(!bwd_supported(a))
    return fail(MTKC_CONTRACT, "rnn scan backward: arguments not supported by the persistent path");
  const BPlan P = make_bplan(a);
  if(!a->workspace || a->workspace_bytes < P.total)
    return fail(MTKC_CONTRACT, "rnn scan backward: workspace too small");
  cudaStream_t st = S(stream);
  uint8_t* ws = (uint8_t*)a->workspace;
  const int64_t b = a->b, T = a->T, d = a->d, d3 = 3 * d;
  ProfScope prof(st, "rnn_scan_bwd", scan_flops(a, true));
  // [Uz|Ur|Uh] and [Wz|Wr|Wx] side by side (K-major B operands of the
  // input-gradient products)
  CJobs jobs{};
  for(int q = 0; q < a->ndir; ++q) {
    const mtkc_rnn_dir& D = a->dir[q];
    float* uh = (float*)(ws + P.offUH[q]);
    for(int k = 0; k < D.nblocks; ++k)
      for(int g = 0; g < 3; ++g)
        jobs.j[jobs.n++] = CJob{D.blk[k].U[g], uh + (int64_t)k * d * d3 + g * d, (int)d, (int)d,
                                (int)d, (int)d3};
  }
  if(a->has_att) {
    float* w2c = (float*)(ws + P.offW2C);
    for(int g = 0; g < 3; ++g)
      jobs.j[jobs.n++] = CJob{a->dir[0].blk[1].W[g], w2c + g * d, (int)a->kd, (int)d, (int)d,
                              (int)d3};
  }
  ::mtkc::launch(copy_jobs_kernel, dim3(148, (unsigned)jobs.n), 256, 0, st, jobs);
  MTKC_POST_LAUNCH("copy_jobs_kernel");
  if(cudaError_t e = cudaMemsetAsync(ws + P.offCtr, 0, (64 + (size_t)b) * sizeof(float), st))
    return cuda_status(e, "rnn scan counters");

  BMaps maps;
  memset(&maps, 0, sizeof(maps));
  bool ok = true;
  for(int q = 0; q < a->ndir; ++q) {
    const mtkc_rnn_dir& D = a->dir[q];
    ok = ok && kmap(&maps.dg[q], D.dG, d3, (int64_t)D.nblocks * T * b, 128);
    ok = ok && kmap(&maps.uh[q], (const float*)(ws + P.offUH[q]), d3, (int64_t)D.nblocks * d,
                    (uint32_t)P.NTb);
  }
  if(a->has_att) {
    ok = ok && kmap(&maps.dgx, a->dir[0].blk[1].dGx, d3, T * b, 128);
    ok = ok && kmap(&maps.w2c, (const float*)(ws + P.offW2C), d3, a->kd, (uint32_t)P.NTc);
    ok = ok && kmap(&maps.dwq, a->dwq, a->a, T * b, 128);
    ok = ok && kmap(&maps.watt, a->attW, a->a, d, (uint32_t)P.NTb);
  }
  if(!ok)
    return fail(MTKC_CUDA, "rnn scan backward: tensor map encoding failed");
  BKP kp;
  memset(&kp, 0, sizeof(kp));
  kp.a = *a;
  for(int q = 0; q < a->ndir; ++q) {
    kp.partB[q] = (float*)(ws + P.offPB[q]);
    kp.dsd[q] = (float*)(ws + P.offDSD[q]);
  }
  kp.partC = a->has_att ? (float*)(ws + P.offPC) : nullptr;
  kp.partQ = a->has_att ? (float*)(ws + P.offPQ) : nullptr;
  kp.ctr = (unsigned*)(ws + P.offCtr);
  kp.KCb = P.KCb;
  kp.KCc = P.KCc;
  kp.KCq = P.KCq;
  kp.NTb = P.NTb;
  kp.NTc = P.NTc;
  kp.team = P.team;
  kp.teamCtr = (unsigned*)(ws + P.offCtr) + 64;
  kp.teamBuf = (float*)(ws + P.offTeamBuf);
  static bool attr = false;
  if(!attr) {
    cudaError_t e = cudaFuncSetAttribute(rnn_scan_bwd_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES_B);
    if(e != cudaSuccess)
      return cuda_status(e, "rnn scan bwd smem attribute");
    attr = true;
  }
  static unsigned long long* profBuf = nullptr;
  const bool profOn = getenv("MTK_RNN_PROF") != nullptr;
  if(profOn) {
    if(!profBuf)
      cudaMalloc(&profBuf, 8192 * 2 * sizeof(unsigned long long));
    cudaMemsetAsync(profBuf, 0, 8192 * 2 * sizeof(unsigned long long), st);
    kp.prof = profBuf;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P.G);
  cfg.blockDim = dim3(RT);
  cfg.dynamicSmemBytes = SMEM_BYTES_B;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, rnn_scan_bwd_kernel, maps, kp);
  if(e != cudaSuccess)
    return cuda_status(e, "rnn_scan_bwd_kernel");
  count_launch();
  if(profOn) {  // kinds: 1 PWB, 0 PRODB, 4 PRODB + ctx, 3 ATTB, 2 PRODQ, 5 barrier
    std::vector<unsigned long long> h(8192 * 2);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), profBuf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double sum[16] = {0}, cnt[16] = {0};
    for(int i = 0; i + 1 < 8192 && h[2 * i + 3]; ++i) {
      int k = (int)h[2 * i];
      sum[k] += (double)(h[2 * i + 3] - h[2 * i + 1]);
      cnt[k] += 1;
    }
    const char* nm[16] = {"prodB", "pwB", "prodQ", "attB", "prodB+ctx", "barrier", "end", "-",
                          "attB:dctx", "attB:dw", "-", "attB:softmax", "attB:lnstats",
                          "attB:cols", "-", "-"};
    fprintf(stderr, "[rnn prof bwd] ndir %d b %lld T %lld:", a->ndir, (long long)b, (long long)T);
    for(int k = 0; k < 16; ++k)
      if(cnt[k] > 0 && k != 6)
        fprintf(stderr, " %s %.0f x %.2f us", nm[k], cnt[k], sum[k] / cnt[k] / 1e3);
    fprintf(stderr, "\n");
  }
  return MTKC_OK;
}

}  // extern "C"


// ------------------------------------------------------------ key gradient
// d(keys)[r, s, :] (+)= sum_t w[t, r, s] * dctx[t, r, :] (the context's key
// gradient, bahdanau_dw_kernel's gk term summed over the decoder steps):
// one CTA per (row r, 256-column chunk); the row's weights and the chunk of
// every step's context gradient are staged in shared memory, sums in step
// order.
namespace {
constexpr int KG_COLS = 256;
__global__ void __launch_bounds__(256) rnn_key_grad_kernel(float* gkeys, const float* attW,
                                                           const float* dctx, int64_t b,
                                                           int64_t T, int64_t S, int64_t kd,
                                                           int acc) {
  MTKC_PDL_ENTRY();
  extern __shared__ float ks[];  // [T][KG_COLS] dctx chunk, then [T][S] weights
  const int64_t r = blockIdx.y, c0 = (int64_t)blockIdx.x * KG_COLS;
  const int64_t nc = min((int64_t)KG_COLS, kd - c0);
  float* sd = ks;
  float* sw = ks + T * KG_COLS;
  for(int64_t i = threadIdx.x; i < T * KG_COLS; i += blockDim.x) {
    const int64_t t = i / KG_COLS, c = i % KG_COLS;
    sd[i] = c < nc ? dctx[(t * b + r) * kd + c0 + c] : 0.f;
  }
  for(int64_t i = threadIdx.x; i < T * S; i += blockDim.x) {
    const int64_t t = i / S, s = i % S;
    sw[i] = attW[(t * b + r) * S + s];
  }
  __syncthreads();
  const int64_t c = threadIdx.x;
  if(c >= nc)
    return;
  for(int64_t s = 0; s < S; ++s) {
    float v = 0.f;
    for(int64_t t = 0; t < T; ++t)
      v += sw[t * S + s] * sd[t * KG_COLS + c];
    float* o = gkeys + (r * S + s) * kd + c0 + c;
    *o = acc ? *o + v : v;
  }
}
}  // namespace

extern "C" int mtkc_rnn_key_grad(float* gkeys, const float* attW, const float* dctx, int64_t b,
                                 int64_t T, int64_t nS, int64_t kd, int accumulate, void* stream) {
  if(b <= 0 || T <= 0 || nS <= 0 || kd <= 0)
    return MTKC_OK;
  const size_t smem = (size_t)T * (KG_COLS + nS) * sizeof(float);
  if(smem > 200 * 1024)
    return fail(MTKC_DIMENSION, "rnn key gradient: T x (256 + S) floats exceed shared memory");
  static size_t attr = 0;
  if(smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(rnn_key_grad_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if(e != cudaSuccess)
      return cuda_status(e, "rnn key gradient smem attribute");
    attr = smem;
  }
  ProfScope prof(S(stream), "rnn_scan_bwd", 4.0 * (double)(b * nS * kd + T * b * kd));
  ::mtkc::launch(rnn_key_grad_kernel, dim3((unsigned)cdiv(kd, KG_COLS), (unsigned)b), 256, smem,
                 S(stream), gkeys, attW, dctx, b, T, nS, kd, accumulate);
  MTKC_POST_LAUNCH("rnn_key_grad_kernel");
  return MTKC_OK;
}
