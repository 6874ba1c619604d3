// GEMM entry point (matmulInto tensor.cpp:258-306, matmulAccumInto
// graph.cpp:273-291, affine graph.cpp:334-336) and its CUDA-core FP32 path.
//
// The FP32 path reproduces the reference's arithmetic exactly: every output
// element starts from beta*C (or 0), then adds round(round(alpha*a)*b) for
// k = 0..K-1 in ascending order, skipping alpha*a == 0 (tensor.cpp:282-303),
// with separately rounded multiplies and adds (the reference is compiled
// without FMA contraction).  It is the parity-mode GEMM and the fallback for
// shapes the tensor-core path does not take (unaligned strides, tiny or
// batched-broadcast products).  The tensor-core path lives in gemm_tc.cu.
#include "common.cuh"

namespace mtkc {
bool tc_gemm(const mtkc_gemm_args& a, cudaStream_t st, int* rc, bool* csFused);  // gemm_tc.cu
bool tc_gemm_group(const mtkc_gemm_args* probs, int nprob, int kconcat, cudaStream_t st,
                   int* rc, bool* csFused);
}

using namespace mtkc;

namespace {

thread_local int t_last_path = 0;

// relu_mask_out after a CUDA-core product: one warp per 32-column word
__global__ void relu_mask_pack_kernel(const float* C, int64_t ldc, int64_t M, int64_t N,
                                      uint32_t* mask) {
  MTKC_PDL_ENTRY();
  const int64_t mw = (N + 31) / 32, words = M * mw;
  const int lane = threadIdx.x & 31;
  for(int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < words;
      w += (int64_t)gridDim.x * blockDim.x / 32) {
    const int64_t r = w / mw, c = (w - r * mw) * 32 + lane;
    const uint32_t bits = __ballot_sync(0xffffffffu, c < N && C[r * ldc + c] > 0.f);
    if(lane == 0)
      mask[w] = bits;
  }
}

// The operand sums of mtkc_gemm_args.colsum as a separate pass (FP32
// precision, or a tensor-core launch that could not fuse them): column sums
// of the stored MN-major operand with mtkc_colsum's summation order.
int colsum_after(const mtkc_gemm_args& a, void* stream) {
  if(!a.colsum)
    return MTKC_OK;
  if(a.batch != 1)
    return fail(MTKC_CONTRACT, "mtkc_gemm: colsum needs batch == 1");
  if(a.colsum_of == MTKC_COLSUM_B && !a.transB && a.ldb == a.N)
    return mtkc_colsum(a.colsum, a.B, a.K, a.N, a.colsum_accumulate, a.workspace,
                       a.workspace_bytes, stream);
  if(a.colsum_of == MTKC_COLSUM_A && a.transA && a.lda == a.M)
    return mtkc_colsum(a.colsum, a.A, a.K, a.M, a.colsum_accumulate, a.workspace,
                       a.workspace_bytes, stream);
  return fail(MTKC_CONTRACT,
              "mtkc_gemm: colsum needs a densely stored MN-major operand (B untransposed with "
              "ldb == N, or A transposed with lda == M)");
}

constexpr int TM = 64, TN = 64, TK = 16;

struct GemmP {
  int64_t M, N, K, batch;
  const float* A;
  int64_t lda, sA;
  int tA;
  const float* B;
  int64_t ldb, sB;
  int tB;
  float* C;
  const float* Cin;  // source of the beta term: C, or the addend
  int64_t ldc, sC;
  float alpha, beta;
  const float* bias;
  int epi;
  const float* gate;
  const uint32_t* gateMask;  // bit mask form of the gate (batch 1), words per row mw
  int64_t mw;
  int foldBatch;  // sum over batch into one C
};

__global__ void __launch_bounds__(256) gemm_fp32_kernel(GemmP p) {
  MTKC_PDL_ENTRY();
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = (int64_t)blockIdx.y * TM, col0 = (int64_t)blockIdx.x * TN;
  const int64_t zb = p.foldBatch ? 0 : blockIdx.z;
  float* C = p.C + zb * p.sC;
  const float* Cin = p.Cin + zb * p.sC;
  float acc[4][4];
  const bool gated = p.gate != nullptr || p.gateMask != nullptr;
#pragma unroll
  for(int i = 0; i < 4; ++i)
#pragma unroll
    for(int j = 0; j < 4; ++j) {
      int64_t r = row0 + ty * 4 + i, c = col0 + tx * 4 + j;
      float v = 0.f;
      if(!gated && p.beta != 0.f && r < p.M && c < p.N) {
        v = Cin[r * p.ldc + c];
        if(p.beta != 1.f)
          v = __fmul_rn(v, p.beta);
      }
      acc[i][j] = v;
    }
  const int64_t nb = p.foldBatch ? p.batch : 1;
  for(int64_t bb = 0; bb < nb; ++bb) {
    const int64_t b = p.foldBatch ? bb : zb;
    const float* A = p.A + b * p.sA;
    const float* B = p.B + b * p.sB;
    for(int64_t k0 = 0; k0 < p.K; k0 += TK) {
      // cooperative tile loads (4 elements per thread per operand)
      for(int e = threadIdx.x; e < TK * TM; e += 256) {
        int kk = e / TM, mm = e % TM;
        int64_t gi = row0 + mm, gk = k0 + kk;
        float v = 0.f;
        if(gi < p.M && gk < p.K)
          v = p.tA ? A[gk * p.lda + gi] : A[gi * p.lda + gk];
        As[kk][mm] = p.alpha == 1.f ? v : __fmul_rn(p.alpha, v);
      }
      for(int e = threadIdx.x; e < TK * TN; e += 256) {
        int kk = e / TN, nn = e % TN;
        int64_t gj = col0 + nn, gk = k0 + kk;
        float v = 0.f;
        if(gj < p.N && gk < p.K)
          v = p.tB ? B[gj * p.ldb + gk] : B[gk * p.ldb + gj];
        Bs[kk][nn] = v;
      }
      __syncthreads();
      const int kmax = (int)min((int64_t)TK, p.K - k0);
      for(int kk = 0; kk < kmax; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for(int i = 0; i < 4; ++i)
          av[i] = As[kk][ty * 4 + i];
#pragma unroll
        for(int j = 0; j < 4; ++j)
          bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for(int i = 0; i < 4; ++i) {
          if(av[i] == 0.f)
            continue;  // tensor.cpp:293-294
#pragma unroll
          for(int j = 0; j < 4; ++j)
            acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
        }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for(int i = 0; i < 4; ++i)
#pragma unroll
    for(int j = 0; j < 4; ++j) {
      int64_t r = row0 + ty * 4 + i, c = col0 + tx * 4 + j;
      if(r >= p.M || c >= p.N)
        continue;
      float v = acc[i][j];
      if(p.bias)
        v = __fadd_rn(v, p.bias[c]);
      if(p.epi == MTKC_EPI_RELU)
        v = v > 0.f ? v : 0.f;
      float* dst = C + r * p.ldc + c;
      if(gated) {
        const bool on = p.gateMask ? ((p.gateMask[r * p.mw + (c >> 5)] >> (c & 31)) & 1u) != 0
                                   : p.gate[zb * p.sC + r * p.ldc + c] > 0.f;
        v = on ? v : 0.f;
        if(p.beta != 0.f)
          v = __fadd_rn(p.beta == 1.f ? Cin[r * p.ldc + c] : __fmul_rn(p.beta, Cin[r * p.ldc + c]),
                        v);
      }
      *dst = v;
    }
}

}  // namespace

extern "C" {

int mtkc_gemm_last_path(void) { return t_last_path; }

int mtkc_gemm(const mtkc_gemm_args* a, void* stream) {
  if(!a)
    return fail(MTKC_CONTRACT, "mtkc_gemm: null args");
  if(a->M <= 0 || a->N <= 0 || a->K <= 0 || a->batch <= 0)
    return fail(MTKC_DIMENSION, "mtkc_gemm: non-positive extent");
  if(!a->A || !a->B || !a->C)
    return fail(MTKC_CONTRACT, "mtkc_gemm: null operand");
  int rc = MTKC_OK;
  ProfScope prof(S(stream), "gemm_tc", 2.0 * a->M * a->N * a->K * a->batch);
  if(prof_detail()) {
    char d[128];
    snprintf(d, sizeof(d), "M%lld_N%lld_K%lld_b%lld_tA%d_tB%d_e%d%s%s",
             (long long)a->M, (long long)a->N, (long long)a->K, (long long)a->batch, a->transA,
             a->transB, a->epilogue, a->beta != 0.f ? "_acc" : "", a->bias ? "_bias" : "");
    prof.detail = d;
  }
  bool csFused = false;
  if(a->precision == MTKC_GEMM_TF32 && tc_gemm(*a, S(stream), &rc, &csFused)) {
    t_last_path = 1;
    if(rc == MTKC_OK && !csFused)
      rc = colsum_after(*a, stream);
    return rc;
  }
  prof.cls = "gemm_simt";
  t_last_path = 0;
  GemmP p;
  p.M = a->M;
  p.N = a->N;
  p.K = a->K;
  p.batch = a->batch;
  p.A = a->A;
  p.lda = a->lda;
  p.sA = a->strideA;
  p.tA = a->transA;
  p.B = a->B;
  p.ldb = a->ldb;
  p.sB = a->strideB;
  p.tB = a->transB;
  p.C = a->C;
  p.Cin = a->addend ? a->addend : a->C;
  p.ldc = a->ldc;
  p.sC = a->strideC;
  p.alpha = a->alpha;
  p.beta = a->beta;
  p.bias = a->bias;
  p.epi = a->epilogue;
  p.gate = a->gate;
  p.gateMask = a->gate_mask;
  p.mw = (a->N + 31) / 32;
  if((a->gate_mask || a->relu_mask_out) && a->batch != 1)
    return fail(MTKC_CONTRACT, "mtkc_gemm: relu masks need batch == 1");
  p.foldBatch = (a->batch > 1 && a->strideC == 0) ? 1 : 0;
  dim3 grid((unsigned)cdiv(a->N, TN), (unsigned)cdiv(a->M, TM),
            p.foldBatch ? 1u : (unsigned)a->batch);
  ::mtkc::launch(gemm_fp32_kernel, grid, 256, 0, S(stream), p);
  MTKC_POST_LAUNCH("gemm_fp32_kernel");
  if(a->relu_mask_out) {
    ::mtkc::launch(relu_mask_pack_kernel, grid1d(a->M * ((a->N + 31) / 32) * 32, 256, 148 * 16),
                   256, 0, S(stream), (const float*)a->C, a->ldc, a->M, a->N, a->relu_mask_out);
    MTKC_POST_LAUNCH("relu_mask_pack_kernel");
  }
  return colsum_after(*a, stream);
}

int mtkc_gemm_group(const mtkc_gemm_args* probs, int nprob, int kconcat, void* stream) {
  if(!probs || nprob < 1)
    return fail(MTKC_CONTRACT, "mtkc_gemm_group: no problems");
  const mtkc_gemm_args& a = probs[0];
  if(a.precision == MTKC_GEMM_TF32 && nprob <= 3) {
    int rc = MTKC_OK;
    ProfScope prof(S(stream), "gemm_tc", 2.0 * a.M * a.N * a.K * nprob);
    if(prof_detail()) {
      char d[128];
      snprintf(d, sizeof(d), "group%d%s_M%lld_N%lld_K%lld_tA%d_tB%d%s%s", nprob,
               kconcat ? "k" : "", (long long)a.M, (long long)a.N, (long long)a.K, a.transA,
               a.transB, a.beta != 0.f ? "_acc" : "", a.bias ? "_bias" : "");
      prof.detail = d;
    }
    bool csFused = false;
    if(tc_gemm_group(probs, nprob, kconcat, S(stream), &rc, &csFused)) {
      t_last_path = 1;
      for(int q = 0; q < nprob && rc == MTKC_OK && !csFused; ++q)
        rc = colsum_after(probs[q], stream);
      return rc;
    }
  }
  // same semantics, one product at a time
  for(int q = 0; q < nprob; ++q) {
    mtkc_gemm_args b = probs[q];
    if(kconcat && q > 0) {
      b.C = a.C;
      b.ldc = a.ldc;
      b.beta = 1.f;
      b.bias = nullptr;
    }
    if(int rc = mtkc_gemm(&b, stream))
      return rc;
  }
  return MTKC_OK;
}

}  // extern "C"
