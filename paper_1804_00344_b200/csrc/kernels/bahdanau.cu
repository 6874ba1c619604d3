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

// Work is spread over (row, source position) warps and (row, column-chunk)
// CTAs instead of one CTA per batch row (85-120 rows would leave most SMs
// idle): forward = scores kernel + softmax/context kernel, backward =
// d(weights)/d(keys) kernel + softmax-backward/LN-statistics kernel +
// column kernel.  Per (row, position) sums keep the lane-strided order of
// the single-kernel version; sums over positions run in ascending order.

// e[r,j] = v . tanh(LN(wq[r] + uk[r,j]));  warp per (r, j)
__global__ void __launch_bounds__(BT) bahdanau_score_kernel(mtkc_bahdanau_args p) {
  MTKC_PDL_ENTRY();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rj = (int64_t)blockIdx.x * BW + warp;
  const int64_t A = p.a, S = p.s;
  if(rj >= p.b * S)
    return;
  const int64_t r = rj / S;
  const float* wq = p.wq + r * A;
  const bool ln = p.lnG != nullptr;
  const float* uk = p.uk + rj * A;
  float* t = p.t + rj * A;
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
      p.lnrs[rj] = rs;
  }
  float acc = 0.f;
  for(int64_t c = lane; c < A; c += 32) {
    float x = wq[c] + uk[c];
    if(ln) {
      float xh = (x - mu) * rs;
      p.lnxh[rj * A + c] = xh;
      x = p.lnG[c] * xh + p.lnB[c];
    }
    float tv = tanhf(x);
    t[c] = tv;
    acc += tv * p.v[c];
  }
  acc = warp_sum(acc);
  if(lane == 0)
    p.scratch[rj] = acc;
}

// masked softmax over positions (tensor.cpp:393-440) + context for one
// 256-column chunk of row r; chunk 0 also stores the weights
__global__ void __launch_bounds__(BT) bahdanau_ctx_kernel(mtkc_bahdanau_args p) {
  MTKC_PDL_ENTRY();
  extern __shared__ float wsh[];  // [s]
  const int64_t r = blockIdx.x, S = p.s;
  const int lane = threadIdx.x & 31;
  if(threadIdx.x < 32) {
    const float* e = p.scratch + r * S;
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
    if(!any && lane == 0 && p.flags && blockIdx.y == 0)
      atomicOr(p.flags, MTKC_FLAG_MASKED_ROW);
    float sum = 0.f;
    for(int64_t j = lane; j < S; j += 32)
      if(!m || m[j] != 0.f)
        sum += expf(e[j] - mx);
    sum = warp_sum(sum);
    for(int64_t j = lane; j < S; j += 32) {
      float y = (any && (!m || m[j] != 0.f)) ? expf(e[j] - mx) / sum : 0.f;
      wsh[j] = y;
      if(blockIdx.y == 0)
        p.w[r * S + j] = y;
    }
  }
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.y * BT + threadIdx.x;
  if(k >= p.kd)
    return;
  const float* keys = p.keys + r * S * p.kd;
  float acc = 0.f;
  for(int64_t j = 0; j < S; ++j)
    acc += wsh[j] * keys[j * p.kd + k];
  p.ctx[r * p.kd + k] = acc;
}

// d(weights)_j = gctx . keys_j ; d(keys)_j (+)= w_j * gctx;  warp per (r, j)
__global__ void __launch_bounds__(BT) bahdanau_dw_kernel(mtkc_bahdanau_args p) {
  MTKC_PDL_ENTRY();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rj = (int64_t)blockIdx.x * BW + warp;
  const int64_t S = p.s, KD = p.kd;
  if(rj >= p.b * S)
    return;
  const int64_t r = rj / S;
  const float* gctx = p.gctx + r * KD;
  const float* keys = p.keys + rj * KD;
  float* gk = p.gkeys + rj * KD;
  const float wj = p.w[rj];
  float acc = 0.f;
  for(int64_t k = lane; k < KD; k += 32) {
    float g = gctx[k];
    acc += g * keys[k];
    float add = wj * g;
    gk[k] = p.acc_keys ? gk[k] + add : add;
  }
  acc = warp_sum(acc);
  if(lane == 0)
    p.scratch[rj] = acc;
}

// de_j = w_j (dw_j - sum_l w_l dw_l)  (softmax backward graph.cpp:539-552),
// and with layer norm the row statistics of its backward; warp per (r, j)
__global__ void __launch_bounds__(BT) bahdanau_de_kernel(mtkc_bahdanau_args p) {
  MTKC_PDL_ENTRY();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rj = (int64_t)blockIdx.x * BW + warp;
  const int64_t A = p.a, S = p.s, BS = p.b * S;
  if(rj >= BS)
    return;
  const int64_t r = rj / S;
  const float* w = p.w + r * S;
  const float* dw = p.scratch + r * S;
  float s = 0.f;
  for(int64_t j = lane; j < S; j += 32)
    s += w[j] * dw[j];
  s = warp_sum(s);
  const float dej = p.w[rj] * (p.scratch[rj] - s);
  if(p.lnG) {
    const float* t = p.t + rj * A;
    const float* xh = p.lnxh + rj * A;
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
    if(lane == 0) {
      p.scratch[2 * BS + rj] = s1;
      p.scratch[3 * BS + rj] = s2;
    }
  }
  if(lane == 0)
    p.scratch[BS + rj] = dej;
}

// per (row r, 256-column chunk): d(uk)[r,j,c], and the sums over positions
// d(wq)[r,c], v / LN-gain / LN-bias partials [r,c]
__global__ void __launch_bounds__(BT) bahdanau_cols_kernel(mtkc_bahdanau_args p) {
  MTKC_PDL_ENTRY();
  const int64_t r = blockIdx.x, A = p.a, S = p.s, BS = p.b * S;
  const int64_t c = (int64_t)blockIdx.y * BT + threadIdx.x;
  if(c >= A)
    return;
  const bool ln = p.lnG != nullptr;
  const float vc = p.v[c];
  const float gc = ln ? p.lnG[c] : 0.f;
  float awq = 0.f, av = 0.f, ag = 0.f, ab = 0.f;
  for(int64_t j = 0; j < S; ++j) {
    const int64_t rj = r * S + j;
    const float dej = p.scratch[BS + rj];
    const float tv = p.t[rj * A + c];
    av += tv * dej;
    const float dln = (dej * vc) * (1.f - tv * tv);
    float ds = dln;
    if(ln) {
      const float xh = p.lnxh[rj * A + c];
      ag += dln * xh;
      ab += dln;
      ds = p.lnrs[rj] * (dln * gc - p.scratch[2 * BS + rj] - xh * p.scratch[3 * BS + rj]);
    }
    float* gu = p.guk + rj * A + c;
    *gu = p.acc_uk ? *gu + ds : ds;
    awq += ds;
  }
  float* gwq = p.gwq + r * A + c;
  *gwq = p.acc_wq ? *gwq + awq : awq;
  p.gv_part[r * A + c] = av;
  if(ln) {
    p.glnG_part[r * A + c] = ag;
    p.glnB_part[r * A + c] = ab;
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
  if(!a->scratch)
    return fail(MTKC_CONTRACT, "bahdanau: scratch [b x s x 4] required");
  ProfScope prof(S(stream), "bahdanau", 4.0 * a->b * a->s * (3.0 * a->a + a->kd));
  const int64_t bs = a->b * a->s;
  ::mtkc::launch(bahdanau_score_kernel, (unsigned)cdiv(bs, BW), BT, 0, S(stream), *a);
  MTKC_POST_LAUNCH("bahdanau_score_kernel");
  size_t smem = (size_t)a->s * sizeof(float);
  int rc = set_smem((const void*)bahdanau_ctx_kernel, smem);
  if(rc)
    return rc;
  ::mtkc::launch(bahdanau_ctx_kernel, dim3((unsigned)a->b, (unsigned)cdiv(a->kd, BT)), BT, smem,
                 S(stream), *a);
  MTKC_POST_LAUNCH("bahdanau_ctx_kernel");
  return MTKC_OK;
}

int mtkc_bahdanau_backward(const mtkc_bahdanau_args* a, void* stream) {
  if(a->b <= 0 || a->s <= 0)
    return MTKC_OK;
  if(!a->scratch)
    return fail(MTKC_CONTRACT, "bahdanau: scratch [b x s x 4] required");
  ProfScope prof(S(stream), "bahdanau", 4.0 * a->b * a->s * (4.0 * a->a + 3.0 * a->kd));
  const int64_t bs = a->b * a->s;
  ::mtkc::launch(bahdanau_dw_kernel, (unsigned)cdiv(bs, BW), BT, 0, S(stream), *a);
  MTKC_POST_LAUNCH("bahdanau_dw_kernel");
  ::mtkc::launch(bahdanau_de_kernel, (unsigned)cdiv(bs, BW), BT, 0, S(stream), *a);
  MTKC_POST_LAUNCH("bahdanau_de_kernel");
  ::mtkc::launch(bahdanau_cols_kernel, dim3((unsigned)a->b, (unsigned)cdiv(a->a, BT)), BT, 0,
                 S(stream), *a);
  MTKC_POST_LAUNCH("bahdanau_cols_kernel");
  return MTKC_OK;
}

}  // extern "C"
