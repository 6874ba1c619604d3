// Blackwell tensor-core GEMM for the graph's dot/affine nodes
// (matmulInto tensor.cpp:258-306 and the transposed products of the dot
// backward, graph.cpp:319-330).
//
// Data stays fp32 in HBM (the reference's storage type); operands are fed
// to tcgen05.mma kind::tf32 straight from TMA-staged shared memory and
// accumulate in fp32 in TMEM.  Every transpose case is a descriptor choice,
// not a copy: op(A)/op(B) are loaded K-major or MN-major with 128-byte
// swizzle, so dW = X^T dY and dX = dY W^T read the forward activations in
// place.
//
// Structure (one CTA per 128 x BN output tile, optionally split over K):
//   warp 0      TMA producer   (one elected lane, ST-stage mbarrier ring)
//   warp 1      MMA issuer     (one elected lane; owns the TMEM allocation)
//   warps 2..5  epilogue       (tcgen05.ld 32x32b -> alpha/beta/bias/relu/
//                               gate -> st.global, or split-K partials)
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace mtkc {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int ST = 4;   // pipeline stages
constexpr int TC_THREADS = 192;

// ---------------------------------------------------------------- PTX

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

// layout: 2 = SWIZZLE_128B (K-major operands), 1 = SWIZZLE_128B_BASE32B
// (the only MN-major layout tcgen05 accepts for 32-bit tf32 operands)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for(int i = 0; i < 32; ++i)
    v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- kernel

struct TcP {
  int64_t M, N, K;
  float* C;
  int64_t ldc;
  float alpha, beta;
  const float* bias;
  int epi;
  const float* gate;
  float* part;  // split-K partials [splits][M][N] (ld = N), or nullptr
  int kbPerSplit;
  int numKb;
};

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tf32_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                        const __grid_constant__ CUtensorMap mapB, TcP p) {
  constexpr uint32_t A_BYTES = BM * BK * 4;
  constexpr uint32_t B_BYTES = BN * BK * 4;
  constexpr uint32_t TMEM_COLS = BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * A_BYTES;
  uint64_t* full = (uint64_t*)(sB + ST * B_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tmemFull = empty + ST;
  uint32_t* tmemSlot = (uint32_t*)(tmemFull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb0 = blockIdx.z * p.kbPerSplit;
  const int kb1 = min(p.numKb, kb0 + p.kbPerSplit);
  const int nkb = kb1 - kb0;

  if(warp == 0 && lane == 0) {
    prefetch_tmap(&mapA);
    prefetch_tmap(&mapB);
    for(int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmemFull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  const uint32_t tmem = *tmemSlot;

  if(warp == 0) {
    if(lane == 0) {
      for(int i = 0; i < nkb; ++i) {
        int s = i % ST;
        if(i >= ST)
          mbar_wait(&empty[s], ((i / ST) - 1) & 1);
        mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
        int k0 = (kb0 + i) * BK;
        uint8_t* a = sA + s * A_BYTES;
        uint8_t* b = sB + s * B_BYTES;
        if(A_MN) {
#pragma unroll
          for(int j = 0; j < BM / 32; ++j)
            tma_load_2d(a + j * (BK * 128), &mapA, &full[s], m0 + j * 32, k0);
        } else {
          tma_load_2d(a, &mapA, &full[s], k0, m0);
        }
        if(B_MN) {
#pragma unroll
          for(int j = 0; j < BN / 32; ++j)
            tma_load_2d(b + j * (BK * 128), &mapB, &full[s], n0 + j * 32, k0);
        } else {
          tma_load_2d(b, &mapB, &full[s], k0, n0);
        }
      }
    }
  } else if(warp == 1) {
    // instruction descriptor: D=f32, A=B=tf32, majors, N>>3, M>>4
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) |
                           ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    for(int i = 0; i < nkb; ++i) {
      int s = i % ST;
      mbar_wait(&full[s], (i / ST) & 1);
      tc_fence_after();
      if(lane == 0) {
        uint32_t aBase = smem_u32(sA + s * A_BYTES);
        uint32_t bBase = smem_u32(sB + s * B_BYTES);
#pragma unroll
        for(int kk = 0; kk < BK / 8; ++kk) {
          // K-major (SW128): advance 8 tf32 = 32 B inside the swizzled row;
          //   8-row atoms are 1024 B apart (SBO).
          // MN-major (SW128 with 32 B atomicity): 128 B of M/N per K-row,
          //   4-row atoms 512 B apart (SBO), 32-element M/N chunks one TMA
          //   box (BK rows) apart (LBO); advance 8 K-rows = 1024 B.
          uint64_t ad = A_MN ? umma_desc(aBase + kk * 1024, BK * 128, 512, 1)
                             : umma_desc(aBase + kk * 32, 16, 1024, 2);
          uint64_t bd = B_MN ? umma_desc(bBase + kk * 1024, BK * 128, 512, 1)
                             : umma_desc(bBase + kk * 32, 16, 1024, 2);
          mma_tf32(tmem, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if(lane == 0) {
      if(nkb > 0)
        mma_commit(tmemFull);
    }
    __syncwarp();
  } else {
    // epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
    const int64_t row = m0 + q * 32 + lane;
    if(nkb > 0) {
      mbar_wait(tmemFull, 0);
      tc_fence_after();
    }
    const bool rowOk = row < p.M;
#pragma unroll 1
    for(int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      if(nkb > 0) {
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
      } else {
#pragma unroll
        for(int i = 0; i < 32; ++i)
          v[i] = 0.f;
      }
      if(!rowOk || n0 + c0 >= p.N)
        continue;
      const int64_t col0 = n0 + c0;
      if(p.part) {
        float* dst = p.part + ((int64_t)blockIdx.z * p.M + row) * p.N + col0;
#pragma unroll
        for(int i = 0; i < 32; ++i)
          if(col0 + i < p.N)
            dst[i] = v[i];
        continue;
      }
      float* dst = p.C + row * p.ldc + col0;
      const float* gt = p.gate ? p.gate + row * p.ldc + col0 : nullptr;
#pragma unroll
      for(int i = 0; i < 32; ++i) {
        if(col0 + i >= p.N)
          break;
        float x = p.alpha == 1.f ? v[i] : p.alpha * v[i];
        if(p.bias)
          x = x + p.bias[col0 + i];
        if(p.epi == MTKC_EPI_RELU)
          x = x > 0.f ? x : 0.f;
        if(gt)
          x = gt[i] > 0.f ? x : 0.f;
        if(p.beta != 0.f)
          x = (p.beta == 1.f ? dst[i] : p.beta * dst[i]) + x;
        dst[i] = x;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if(warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// C = alpha*sum_s part[s] (+bias, relu, gate) + beta*C  (fixed split order)
__global__ void splitk_reduce_kernel(const float* part, int splits, int64_t M, int64_t N,
                                     float* C, int64_t ldc, float alpha, float beta,
                                     const float* bias, int epi, const float* gate) {
  int64_t total = M * N;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
      i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / N, c = i % N;
    float acc = 0.f;
    for(int s = 0; s < splits; ++s)
      acc += part[(int64_t)s * total + i];
    float x = alpha == 1.f ? acc : alpha * acc;
    if(bias)
      x = x + bias[c];
    if(epi == MTKC_EPI_RELU)
      x = x > 0.f ? x : 0.f;
    float* dst = C + r * ldc + c;
    if(gate)
      x = gate[r * ldc + c] > 0.f ? x : 0.f;
    if(beta != 0.f)
      x = (beta == 1.f ? *dst : beta * *dst) + x;
    *dst = x;
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
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
           cudaSuccess &&
       q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  });
  return fn;
}

int g_tf32_round = -1;  // MTK_TMA_TF32: 1 = TMA converts fp32->tf32 (round), 0 = raw fp32

bool tma_tf32_round() {
  if(g_tf32_round < 0) {
    const char* e = getenv("MTK_TMA_TF32");
    g_tf32_round = (e && e[0] == '0') ? 0 : 1;
  }
  return g_tf32_round == 1;
}

// 2-d map over a row-major matrix [rows x cols] with leading dim ld (elements)
bool make_map(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld,
              uint32_t boxInner, uint32_t boxOuter, bool mnMajor) {
  EncodeFn fn = encode_fn();
  if(!fn)
    return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {boxInner, boxOuter};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, tma_tf32_round() ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                  2, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mnMajor ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const TcP& p, dim3 grid,
              cudaStream_t st) {
  constexpr size_t smem = 1024 + ST * (size_t)(BM * BK * 4 + BN * BK * 4) + 256;
  auto kern = gemm_tf32_tc_kernel<BN, A_MN, B_MN>;
  static bool attr = false;
  if(!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if(e != cudaSuccess)
      return cuda_status(e, "gemm_tf32_tc smem attribute");
    attr = true;
  }
  kern<<<grid, TC_THREADS, smem, st>>>(ma, mb, p);
  MTKC_POST_LAUNCH("gemm_tf32_tc_kernel");
  return MTKC_OK;
}

template <int BN>
int dispatch_majors(bool aMN, bool bMN, const CUtensorMap& ma, const CUtensorMap& mb,
                    const TcP& p, dim3 grid, cudaStream_t st) {
  if(!aMN && !bMN)
    return launch_tc<BN, false, false>(ma, mb, p, grid, st);
  if(!aMN && bMN)
    return launch_tc<BN, false, true>(ma, mb, p, grid, st);
  if(aMN && !bMN)
    return launch_tc<BN, true, false>(ma, mb, p, grid, st);
  return launch_tc<BN, true, true>(ma, mb, p, grid, st);
}

int g_sms = 0;

}  // namespace

// Returns false when the tensor-core path does not apply (caller falls back).
bool tc_gemm(const mtkc_gemm_args& a, cudaStream_t st, int* rc) {
  if(getenv("MTK_DISABLE_TC"))
    return false;
  if(a.batch != 1)
    return false;
  if(a.M < 64 || a.N < 32 || a.K < 8)
    return false;
  if(a.lda % 4 || a.ldb % 4 || ((uintptr_t)a.A % 16) || ((uintptr_t)a.B % 16))
    return false;
  if(a.gate && (a.ldc != a.N && a.gate == nullptr))
    return false;
  // operand majors: op(A) is K-major iff stored untransposed
  const bool aMN = a.transA != 0, bMN = a.transB == 0;
  if(!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if(g_sms <= 0)
      g_sms = 148;
  }
  const int64_t mt = cdiv(a.M, BM);
  int BN = 256;
  if(mt * cdiv(a.N, 256) < g_sms || a.N <= 128)
    BN = 128;
  const int64_t nt = cdiv(a.N, BN);
  const int numKb = (int)cdiv(a.K, BK);
  // split K when the tile grid leaves SMs idle and K is long
  int splits = 1;
  const int64_t tiles = mt * nt;
  if(tiles < g_sms && numKb >= 8 && a.workspace) {
    splits = (int)std::min<int64_t>(std::max<int64_t>(1, (g_sms + tiles - 1) / tiles),
                                    numKb / 4);
    size_t need = (size_t)splits * (size_t)a.M * (size_t)a.N * sizeof(float);
    while(splits > 1 && need > a.workspace_bytes) {
      --splits;
      need = (size_t)splits * (size_t)a.M * (size_t)a.N * sizeof(float);
    }
  }
  const int kbPer = (int)cdiv(numKb, splits);
  splits = (int)cdiv(numKb, kbPer);

  CUtensorMap ma, mb;
  bool ok;
  if(aMN)  // storage [K x M], M contiguous
    ok = make_map(&ma, a.A, a.M, a.K, a.lda, 32, BK, true);
  else     // storage [M x K]
    ok = make_map(&ma, a.A, a.K, a.M, a.lda, BK, BM, false);
  if(!ok)
    return false;
  if(bMN)  // storage [K x N]
    ok = make_map(&mb, a.B, a.N, a.K, a.ldb, 32, BK, true);
  else     // storage [N x K]
    ok = make_map(&mb, a.B, a.K, a.N, a.ldb, BK, (uint32_t)BN, false);
  if(!ok)
    return false;

  TcP p;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.C = a.C;
  p.ldc = a.ldc;
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.bias = a.bias;
  p.epi = a.epilogue;
  p.gate = a.gate;
  p.part = splits > 1 ? a.workspace : nullptr;
  p.kbPerSplit = kbPer;
  p.numKb = numKb;
  dim3 grid((unsigned)nt, (unsigned)mt, (unsigned)splits);
  *rc = BN == 256 ? dispatch_majors<256>(aMN, bMN, ma, mb, p, grid, st)
                  : dispatch_majors<128>(aMN, bMN, ma, mb, p, grid, st);
  if(*rc == MTKC_OK && splits > 1) {
    splitk_reduce_kernel<<<grid1d(a.M * a.N, 256), 256, 0, st>>>(
        a.workspace, splits, a.M, a.N, a.C, a.ldc, a.alpha, a.beta, a.bias, a.epilogue, a.gate);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if(e != cudaSuccess)
      *rc = cuda_status(e, "splitk_reduce_kernel");
  }
  return true;
}

}  // namespace mtkc
