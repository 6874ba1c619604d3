// Fused Bahdanau MLP attention core (BahdanauAttention::apply,
// layers.cpp:59-79): one CTA per batch row.  Replaces the reference's chain
// of broadcast add, layer norm, tanh, [b,s,a]x[a,1] product, reshape,
// masked softmax and [b,1,s]x[b,s,k] product (five of them batched GEMMs with
// tiny inner dimensions) by two kernels; the projections wq = query*W and
// uk = keys*U stay tensor-core GEMMs (uk once per batch, not per step).
#include "common.cuh"

using namespace mtkc;

namespace {

constexpr int BT = 256;  // threads
constexpr int BW = BT / 32;

__global__ void __launch_bounds__(BT) bahdanau_fwd_kernel(mtkc_bahdanau_args p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float sm[];
  float* e = sm;             // [s]
  float* wsh = e + p.s;      // [s]
  const int64_t r = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t A = p.a, S = p.s;
  const float* wq = p.wq + r * A;
  const bool ln = p.lnG != nullptr;
  for(int64_t j = warp; j < S; j += BW) {
    const float* uk = p.uk + (r * S + j) * A;
    float* t = p.t + (r * S + j) * A;
    float mu = 0.f, rs = 0.f;
    if(ln) {  // two-pass LN statistics over a (tensor.cpp:545-572)
      float s1 = 0.f;
      for(int64_t c = lane; c < A; c += 32)
        s1 += wq[c] + uk[c];
      mu = warp_sum(s1) / (float)A;
      float s2 = 0.f;
      for(int64_t c = lane; c < A; c += 32) {
        float d = (wq[c] + uk[c]) - mu;
        s2 += d * d;
      }
      rs = 1.f / sqrtf(warp_sum(s2) / (float)A + p.eps);
      if(lane == 0)
        p.lnrs[r * S + j] = rs;
    }
    float acc = 0.f;
    for(int64_t c = lane; c < A; c += 32) {
      float x = wq[c] + uk[c];
      if(ln) {
        float xh = (x - mu) * rs;
        p.lnxh[(r * S + j) * A + c] = xh;
        x = p.lnG[c] * xh + p.lnB[c];
      }
      float tv = tanhf(x);
      t[c] = tv;
      acc += tv * p.v[c];
    }
    acc = warp_sum(acc);
    if(lane == 0)
      e[j] = acc;
  }
  __syncthreads();
  if(warp == 0) {  // masked softmax over source positions (tensor.cpp:393-440)
    const float* m = p.mask ? p.mask + r * S : nullptr;
    float mx = -INFINITY;
    int any = 0;
    for(int64_t j = lane; j < S; j += 32)
      if(!m || m[j] != 0.f) {
        mx = fmaxf(mx, e[j]);
        any = 1;
      }
    mx = warp_max(mx);
    any = __any_sync(0xffffffffu, any);
    if(!any && lane == 0 && p.flags)
      atomicOr(p.flags, MTKC_FLAG_MASKED_ROW);
    float sum = 0.f;
    for(int64_t j = lane; j < S; j += 32)
      if(!m || m[j] != 0.f)
        sum += expf(e[j] - mx);
    sum = warp_sum(sum);
    for(int64_t j = lane; j < S; j += 32) {
      float y = (any && (!m || m[j] != 0.f)) ? expf(e[j] - mx) / sum : 0.f;
      wsh[j] = y;
      p.w[r * S + j] = y;
    }
  }
  __syncthreads();
  const float* keys = p.keys + r * S * p.kd;
  for(int64_t k = threadIdx.x; k < p.kd; k += BT) {
    float acc = 0.f;
    for(int64_t j = 0; j < S; ++j)
      acc += wsh[j] * keys[j * p.kd + k];
    p.ctx[r * p.kd + k] = acc;
  }
}

__global__ void __launch_bounds__(BT) bahdanau_bwd_kernel(mtkc_bahdanau_args p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float sm[];
  const int64_t A = p.a, S = p.s, KD = p.kd;
  float* dw = sm;                // [s]
  float* de = dw + S;            // [s]
  float* pwq = de + S;           // [BW][A] partial d(wq)
  float* pv = pwq + BW * A;      // [BW][A] partial d(v)
  float* pg = pv + BW * A;       // [BW][A] partial d(lnG)  (LN only)
  float* pb = pg + BW * A;       // [BW][A] partial d(lnB)  (LN only)
  const int64_t r = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool ln = p.lnG != nullptr;
  const float* gctx = p.gctx + r * KD;
  const float* keys = p.keys + r * S * KD;
  const float* w = p.w + r * S;
  // d(weights)_j = gctx . keys_j ; d(keys)_j (+)= w_j * gctx
  for(int64_t j = warp; j < S; j += BW) {
    float acc = 0.f;
    float wj = w[j];
    float* gk = p.gkeys + (r * S + j) * KD;
    for(int64_t k = lane; k < KD; k += 32) {
      float g = gctx[k];
      acc += g * keys[j * KD + k];
      float add = wj * g;
      gk[k] = p.acc_keys ? gk[k] + add : add;
    }
    acc = warp_sum(acc);
    if(lane == 0)
      dw[j] = acc;
  }
  for(int64_t c = threadIdx.x; c < BW * A; c += BT) {
    pwq[c] = 0.f;
    pv[c] = 0.f;
    if(ln) {
      pg[c] = 0.f;
      pb[c] = 0.f;
    }
  }
  __syncthreads();
  if(warp == 0) {  // softmax backward: de = w (dw - sum(w dw))  (graph.cpp:539-552)
    float s = 0.f;
    for(int64_t j = lane; j < S; j += 32)
      s += w[j] * dw[j];
    s = warp_sum(s);
    for(int64_t j = lane; j < S; j += 32)
      de[j] = w[j] * (dw[j] - s);
  }
  __syncthreads();
  for(int64_t j = warp; j < S; j += BW) {
    const float dej = de[j];
    const float* t = p.t + (r * S + j) * A;
    float* guk = p.guk + (r * S + j) * A;
    float* mywq = pwq + warp * A;
    float* myv = pv + warp * A;
    if(!ln) {
      for(int64_t c = lane; c < A; c += 32) {
        float tv = t[c];
        myv[c] += tv * dej;
        float ds = (dej * p.v[c]) * (1.f - tv * tv);
        guk[c] = p.acc_uk ? guk[c] + ds : ds;
        mywq[c] += ds;
      }
      continue;
    }
    const float* xh = p.lnxh + (r * S + j) * A;
    const float rs = p.lnrs[r * S + j];
    float s1 = 0.f, s2 = 0.f;
    for(int64_t c = lane; c < A; c += 32) {
      float tv = t[c];
      float dln = (dej * p.v[c]) * (1.f - tv * tv);
      float h = dln * p.lnG[c];
      s1 += h;
      s2 += h * xh[c];
    }
    s1 = warp_sum(s1) / (float)A;
    s2 = warp_sum(s2) / (float)A;
    float* myg = pg + warp * A;
    float* myb = pb + warp * A;
    for(int64_t c = lane; c < A; c += 32) {
      float tv = t[c];
      myv[c] += tv * dej;
      float dln = (dej * p.v[c]) * (1.f - tv * tv);
      myg[c] += dln * xh[c];
      myb[c] += dln;
      float ds = rs * (dln * p.lnG[c] - s1 - xh[c] * s2);
      guk[c] = p.acc_uk ? guk[c] + ds : ds;
      mywq[c] += ds;
    }
  }
  __syncthreads();
  for(int64_t c = threadIdx.x; c < A; c += BT) {
    float a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f;
    for(int k = 0; k < BW; ++k) {
      a1 += pwq[k * A + c];
      a2 += pv[k * A + c];
      if(ln) {
        a3 += pg[k * A + c];
        a4 += pb[k * A + c];
      }
    }
    float* gwq = p.gwq + r * A + c;
    *gwq = p.acc_wq ? *gwq + a1 : a1;
    p.gv_part[r * A + c] = a2;
    if(ln) {
      p.glnG_part[r * A + c] = a3;
      p.glnB_part[r * A + c] = a4;
    }
  }
}

int set_smem(const void* fn, size_t bytes) {
  if(bytes <= 48 * 1024)
    return MTKC_OK;
  return cuda_status(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
      "bahdanau smem attribute");
}

}  // namespace

extern "C" {

int mtkc_bahdanau_forward(const mtkc_bahdanau_args* a, void* stream) {
  if(a->b <= 0 || a->s <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "bahdanau", 4.0 * a->b * a->s * (3.0 * a->a + a->kd));
  size_t smem = 2 * (size_t)a->s * sizeof(float);
  int rc = set_smem((const void*)bahdanau_fwd_kernel, smem);
  if(rc)
    return rc;
  ::mtkc::launch(bahdanau_fwd_kernel, (unsigned)a->b, BT, smem, S(stream), *a);
  MTKC_POST_LAUNCH("bahdanau_fwd_kernel");
  return MTKC_OK;
}

int mtkc_bahdanau_backward(const mtkc_bahdanau_args* a, void* stream) {
  if(a->b <= 0 || a->s <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "bahdanau", 4.0 * a->b * a->s * (4.0 * a->a + 3.0 * a->kd));
  size_t smem = (2 * (size_t)a->s + (a->lnG ? 4 : 2) * (size_t)BW * a->a) * sizeof(float);
  if(smem > 220 * 1024)
    return fail(MTKC_DIMENSION, "bahdanau: attention dim too large for the fused kernel");
  int rc = set_smem((const void*)bahdanau_bwd_kernel, smem);
  if(rc)
    return rc;
  ::mtkc::launch(bahdanau_bwd_kernel, (unsigned)a->b, BT, smem, S(stream), *a);
  MTKC_POST_LAUNCH("bahdanau_bwd_kernel");
  return MTKC_OK;
}

}  // extern "C"
