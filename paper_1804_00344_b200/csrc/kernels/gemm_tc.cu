// Blackwell tensor-core GEMM for the graph's dot/affine nodes
// (matmulInto tensor.cpp:258-306 and the transposed products of the dot
// backward, graph.cpp:319-330).
//
// Data stays fp32 in HBM (the reference's storage type); operands are fed
// to tcgen05.mma kind::tf32 straight from TMA-staged shared memory and
// accumulate in fp32 in TMEM.  Every transpose case is a descriptor choice,
// not a copy: op(A)/op(B) are loaded K-major (128-byte swizzle) or MN-major
// (128-byte swizzle with 32-byte atoms, the tf32 MN-major layout), so
// dW = X^T dY and dX = dY W^T read the forward activations in place.
//
// Persistent, warp-specialised kernel (one CTA per SM):
//   warp 0      TMA producer   (one lane; ST-stage smem ring, mbarriers)
//   warp 1      MMA issuer     (one lane; owns a double-buffered TMEM
//                               accumulator, 2 x BN fp32 columns)
//   warps 2..5  epilogue       (tcgen05.ld 32x32b -> per-warp smem transpose
//                               -> alpha/bias/ReLU/gate/beta*C -> coalesced
//                               128-byte row stores, or split-K partials)
//   warp 6      operand sums   (optional: sums over k of the MN-major operand
//                               straight from the staged tiles -- the bias
//                               gradient colsum(dY) of a dW product)
// The epilogue of tile i overlaps the main loop of tile i+1.
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace mtkc {

namespace {

constexpr int BM = 128;
#ifndef MTK_BK
#define MTK_BK 32
#endif
// K extent of one pipeline stage: 32 fp32 = one 128-byte swizzle row, or 64
// (two atom columns per stage: half the barrier round trips per K)
constexpr int BK = MTK_BK;
constexpr int KA = BK / 32;  // 128-byte atom columns per K-major stage
#ifndef MTK_EPI_WARPS
#define MTK_EPI_WARPS 4
#endif
constexpr int EPI_WARPS = MTK_EPI_WARPS;  // 4 (one per TMEM lane quarter) or 8 (two)
constexpr int CS_WARP = 2 + EPI_WARPS;          // operand-sum warp
constexpr int TC_THREADS = 96 + 32 * EPI_WARPS;  // producer, MMA, epilogue, operand-sum warps
constexpr int EPI_STRIDE = 33;  // padded 32x32 transpose tile

using namespace ::mtkc::tc;

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
  int mt, nt, splits;
  int numTiles;
  int tmaStore;  // 1: epilogue writes C (or 3-d partials) through a TMA store map
  // problem groups (mtkc_gemm_group): nprob products of one shape in one
  // launch.  kconcat = 0: independent outputs C_p = op(A_p) op(B_p) (+bias_p);
  // kconcat = 1: one output C = sum_p op(A_p) op(B_p) (the K dimensions
  // concatenated: k-block kb of the sweep is block kb % nkbProb of problem
  // kb / nkbProb).  Problem 0 is the plain single GEMM.
  int nprob, kconcat, nkbProb;
  int hasAddend;  // beta term read through maps.r (fused residual), C write-only
  int a3d, b3d;   // MN-major operand loaded as one 3-d box (all 32-column atoms)
  int ak3d, bk3d; // K-major operand with KA > 1: one 3-d box over the atom columns
  const float* addend;
  const float* biasP[3];
  float* CP[3];
  // fused operand sums (mtkc_gemm_args.colsum): csOp 1 = A (rows of op(A),
  // length M), 2 = B (columns of op(B), length N).  The R = nt (A) or mt (B)
  // tiles sharing an operand block split its k-blocks round-robin (tile i
  // sums k-blocks kb % R == i), so no CTA carries all the extra smem reads;
  // with csSlots = splits * R > 1 the partials go to
  // csPart[nOut][csSlots][csLen] (slot split * R + i), summed by the reduce
  int csOp, csAcc, csSlots, csR;
  // ReLU gate as a bit mask: maskOut written by a ReLU producer, gateMask
  // read by the consumer's dX product; maskW words per row
  uint32_t* maskOut;
  const uint32_t* gateMask;
  int64_t maskW;
  int64_t csLen;
  float* csOut[3];
  float* csPart;
  int dbg;  // profiling switches (MTK_GEMM_DEBUG): 1 = no epilogue stores, 2 = no MMAs,
            // 4 = C / addend / gate through TMA boxes instead of per-lane prefetch
};

struct TcMaps {
  CUtensorMap a[3], b[3], c[3], g, r;  // r: addend (source of the beta term)
};

// staging buffers (32x32 fp32, 4 KB) per epilogue warp: two for the TMA
// store double buffer; a ring of four in the LOADS instantiation, where each
// buffer takes a TMA-loaded residual / C box, the result in place and the
// store, three chunks ahead of the one being drained
template <bool LOADS>
constexpr int epi_bufs() {
  return LOADS ? 4 : 2;
}

template <int BN, bool PAIR = false, bool LOADS = false>
struct TcSmem {
  static constexpr uint32_t A_BYTES = BM * BK * 4;
  // a CTA pair (cta_group::2) stages half of the tile's B columns per CTA
  static constexpr uint32_t B_BYTES = (PAIR ? BN / 2 : BN) * BK * 4;
  // per epilogue warp (8): two 32x32 fp32 staging tiles (128B-swizzled, TMA store)
  static constexpr size_t EPI_BYTES = EPI_WARPS * epi_bufs<LOADS>() * 32 * 32 * sizeof(float);
  // pipeline depth: as many stages as fit next to the epilogue staging
  // (227 KB): 6 x 32 KB for BN=128, 4 x 48 KB for BN=256; a CTA pair's
  // half-B stages give 6 x 32 KB (BN=256) / 8 x 24 KB (BN=128).  fp32
  // operands make a k-block short in FLOPs, so depth is what covers latency.
  static constexpr int ST_FIT = (int)((232448 - 1024 - EPI_BYTES - 512) / (A_BYTES + B_BYTES));
  static constexpr int ST_LEGACY = KA == 2 ? (BN == 256 ? 2 : 3)
                                 : (EPI_WARPS == 8 ? (BN == 256 ? 3 : 5) : (BN == 256 ? 4 : 6));
  static constexpr int ST = PAIR ? (ST_FIT < 8 ? ST_FIT : 8)
                                 : (ST_FIT < ST_LEGACY ? ST_FIT : ST_LEGACY);
  static constexpr size_t BYTES = 1024 + ST * (size_t)(A_BYTES + B_BYTES) + EPI_BYTES + 512;
};

// LOADS: the epilogue reads beta*C and/or a ReLU gate (TMA-loaded boxes);
// a separate instantiation so the common bias/ReLU epilogue stays lean.
// PAIR: a cluster of two CTAs on neighbouring SMs computes one 256 x BN tile
// with tcgen05.mma.cta_group::2 issued by the even CTA.  Each CTA stages its
// own 128 rows of A and half of the tile's B columns, so every SM receives
// 2/3 of the operand bytes of a single-CTA 128 x BN tile (the L2 -> SM
// traffic is what bounds these fp32-operand GEMMs); each CTA's TMEM holds
// its 128 rows of the accumulator and its own epilogue drains them.
template <int BN, bool A_MN, bool B_MN, bool LOADS, bool PAIR>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tf32_tc_kernel(const __grid_constant__ TcMaps maps, TcP p) {
  using L = TcSmem<BN, PAIR, LOADS>;
  constexpr int NB = epi_bufs<LOADS>();
  constexpr int BNL = PAIR ? BN / 2 : BN;  // B columns staged by this CTA
  constexpr int MT = PAIR ? 2 * BM : BM;    // output rows per tile
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const int unit0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int units = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  constexpr int ST = L::ST;
  constexpr uint32_t A_BYTES = L::A_BYTES, B_BYTES = L::B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered accumulator
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align to 1024 B without leaving the shared address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * A_BYTES;
  float* sEpi = (float*)(sB + ST * B_BYTES);
  uint64_t* full = (uint64_t*)((uint8_t*)sEpi + L::EPI_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;   // [2] MMA -> epilogue
  uint64_t* tempty = tfull + 2;   // [2] epilogue -> MMA
  uint64_t* ldbar = tempty + 2;   // [EPI_WARPS * NB] TMA loads of C / gate boxes
  uint32_t* tmemSlot = (uint32_t*)(ldbar + EPI_WARPS * NB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if(warp == 0 && lane == 0) {
    for(int q = 0; q < p.nprob; ++q) {
      prefetch_tmap(&maps.a[q]);
      prefetch_tmap(&maps.b[q]);
      if(p.tmaStore && (q == 0 || !p.kconcat))
        prefetch_tmap(&maps.c[q]);
    }
    if(p.gate && p.tmaStore)
      prefetch_tmap(&maps.g);
    if(p.hasAddend && p.tmaStore)
      prefetch_tmap(&maps.r);
    for(int w = 0; w < EPI_WARPS * NB; ++w)
      mbar_init(&ldbar[w], 1);
    for(int s = 0; s < ST; ++s) {
      // pair with operand sums: the odd CTA's operand-sum warp relays its
      // stage's arrival to the even CTA (see the producer)
      mbar_init(&full[s], (PAIR && p.csOp && rank == 0) ? 2 : 1);
      mbar_init(&empty[s], p.csOp ? 2 : 1);  // MMA commit (+ operand-sum warp)
    }
    for(int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS * (PAIR ? 2 : 1));  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if(warp == 1) {
    if(PAIR) {  // both CTAs of the pair allocate together (same column base)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmemSlot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmemSlot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if(PAIR)
    cluster_sync_all();  // the peer's barriers are initialised before any remote signal
  else
    __syncthreads();
  tc_fence_after();
  // PDL: barrier init, TMEM allocation and descriptor prefetch above overlap
  // the previous kernel's tail; wait for it before any operand is read
  MTKC_PDL_ENTRY();
  const uint32_t tmem = *tmemSlot;
  const int tilesPerSplit = p.mt * p.nt;
  const int tilesPerProb = tilesPerSplit * p.splits;
  const int nOut = p.kconcat ? 1 : p.nprob;  // output problems

  // tile t -> (output problem, split, m0, n0, k-block range); with kconcat
  // the k range runs over the concatenated k-blocks of all problems
  int tprob = 0;
  auto tileCoords = [&](int t, int& m0, int& n0, int& kb0, int& nkb, int& split) {
    tprob = p.kconcat ? 0 : t / tilesPerProb;
    t -= tprob * tilesPerProb;
    split = t / tilesPerSplit;
    int rem = t - split * tilesPerSplit;
    m0 = (rem % p.mt) * MT + (int)rank * BM;
    n0 = (rem / p.mt) * BN;
    kb0 = split * p.kbPerSplit;
    nkb = min(p.numKb, kb0 + p.kbPerSplit) - kb0;
  };

  if(warp == 0) {
    if(lane == 0) {
      int i = 0;  // global k-block counter (ring position)
      for(int t = unit0; t < p.numTiles; t += units) {
        int m0, n0, kb0, nkb, split;
        tileCoords(t, m0, n0, kb0, nkb, split);
        const int nB = n0 + (int)rank * BNL;  // this CTA's B columns
        for(int kb = 0; kb < nkb; ++kb, ++i) {
          int s = i % ST;
          if(i >= ST)
            mbar_wait(&empty[s], ((i / ST) - 1) & 1);
          // pair: both CTAs' bytes complete on the even CTA's barrier -- or,
          // when the odd CTA's operand-sum warp must see its own stage, on
          // each CTA's own barrier, the odd one relayed by that warp
          const bool relay = PAIR && p.csOp;
          if(!PAIR || rank == 0 || relay)
            mbar_expect_tx(&full[s], (A_BYTES + B_BYTES) * ((PAIR && !relay) ? 2u : 1u));
          const uint32_t fb = PAIR ? mapa_shared(smem_u32(&full[s]), relay ? rank : 0u) : 0u;
          auto ld2 = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if(PAIR)
              tma_load_2d_cg2(dst, m, fb, c0, c1);
            else
              tma_load_2d(dst, m, &full[s], c0, c1);
          };
          auto ld3 = [&](void* dst, const CUtensorMap* m, int c0, int c1, int c2) {
            if(PAIR)
              tma_load_3d_cg2(dst, m, fb, c0, c1, c2);
            else
              tma_load_3d(dst, m, &full[s], c0, c1, c2);
          };
          const int kbg = kb0 + kb;
          const int pk = p.kconcat ? kbg / p.nkbProb : tprob;  // problem of this k-block
          const int k0 = (p.kconcat ? kbg - pk * p.nkbProb : kbg) * BK;
          const CUtensorMap* mapA = &maps.a[pk];
          const CUtensorMap* mapB = &maps.b[pk];
          uint8_t* a = sA + s * A_BYTES;
          uint8_t* b = sB + s * B_BYTES;
          if(A_MN) {
            if(p.a3d)
              ld3(a, mapA, 0, k0, m0 / 32);
            else
              for(int j = 0; j < BM / 32; ++j)
                ld2(a + j * (BK * 128), mapA, m0 + j * 32, k0);
          } else if(KA == 1) {
            ld2(a, mapA, k0, m0);
          } else if(p.ak3d) {  // [KA][BM][32]
            ld3(a, mapA, 0, m0, k0 / 32);
          } else {
            for(int c = 0; c < KA; ++c)
              ld2(a + c * (BM * 128), mapA, k0 + c * 32, m0);
          }
          if(B_MN) {
            if(p.b3d)
              ld3(b, mapB, 0, k0, nB / 32);
            else
              for(int j = 0; j < BNL / 32; ++j)
                ld2(b + j * (BK * 128), mapB, nB + j * 32, k0);
          } else if(KA == 1) {
            ld2(b, mapB, k0, nB);
          } else if(p.bk3d) {  // [KA][BNL][32]
            ld3(b, mapB, 0, nB, k0 / 32);
          } else {
            for(int c = 0; c < KA; ++c)
              ld2(b + c * (BNL * 128), mapB, k0 + c * 32, nB);
          }
        }
      }
    }
  } else if(warp == 1) {
    if(!PAIR || rank == 0) {  // the even CTA issues the pair's MMAs
    // instruction descriptor: D=f32, A=B=tf32, majors, N>>3, M>>4
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) |
                           ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(MT >> 4) << 24);
    int i = 0, lt = 0;
    for(int t = unit0; t < p.numTiles; t += units, ++lt) {
      int m0, n0, kb0, nkb, split;
      tileCoords(t, m0, n0, kb0, nkb, split);
      const int acc = lt & 1;
      if(lt >= 2)
        mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t tacc = tmem + (uint32_t)(acc * BN);
      for(int kb = 0; kb < nkb; ++kb, ++i) {
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
            // K-major with KA > 1: atom column kk / 4 is a full [rows][32]
            //   block (rows * 128 B) after the previous one.
            uint64_t ad = A_MN ? umma_desc(aBase + kk * 1024, BK * 128, 512, 1)
                               : umma_desc(aBase + (kk >> 2) * (BM * 128) + (kk & 3) * 32, 16,
                                           1024, 2);
            uint64_t bd = B_MN ? umma_desc(bBase + kk * 1024, BK * 128, 512, 1)
                               : umma_desc(bBase + (kk >> 2) * (BNL * 128) + (kk & 3) * 32, 16,
                                           1024, 2);
            if(!(p.dbg & 2)) {
              if(PAIR)
                mma_tf32_cg2(tacc, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
              else
                mma_tf32(tacc, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            }
          }
          if(PAIR)
            mma_commit_cg2(&empty[s], 3);  // frees the stage in both CTAs
          else
            mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if(lane == 0) {
        if(PAIR)
          mma_commit_cg2(&tfull[acc], 3);  // both CTAs' epilogues
        else
          mma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
    } else if(PAIR && p.csOp) {
      // odd CTA with operand sums: its stages complete on its own barriers
      // (the operand-sum warp reads them); this otherwise idle warp relays
      // each arrival to the even CTA's MMA issuer
      int i = 0;
      for(int t = unit0; t < p.numTiles; t += units) {
        int m0, n0, kb0, nkb, split;
        tileCoords(t, m0, n0, kb0, nkb, split);
        for(int kb = 0; kb < nkb; ++kb, ++i) {
          const int s = i % ST;
          mbar_wait(&full[s], (i / ST) & 1);
          if(lane == 0)
            mbar_arrive_cluster(mapa_shared(smem_u32(&full[s]), 0));
          __syncwarp();
        }
      }
    }
  } else if(warp < CS_WARP) {
    // epilogue warps 2..9: TMEM lane quarter q = warp % 4 (the quarter a
    // warp may access), column half h = (warp - 2) / 4 of the tile
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;
    const int cBeg = h * (BN * 4 / EPI_WARPS), cEnd = cBeg + BN * 4 / EPI_WARPS;
    // two swizzled 32x32 staging tiles per warp (TMA-store mode); the
    // fallback path reuses the first one as a padded transpose buffer
    float* stage0 = sEpi + ew * NB * 1024;
    int chunk = 0;  // chunks handed to the TMA engine by this warp
    uint32_t ldPhase = 0;  // TMA C / gate box loads completed by this warp
    // beta*C / addend without a gate (the fused residual): a ring of NB
    // staging buffers per warp; chunk j's box is TMA-loaded NB - 1 chunks
    // ahead into buffer j % NB, the result overwrites it in place and is
    // TMA-stored from there (the load latency hides behind NB - 1 chunks)
    const bool ring = LOADS && NB > 2 && !p.part && p.tmaStore && !(p.dbg & 4) &&
                      p.beta != 0.f && p.gate == nullptr;
    constexpr int CPT = BN * 4 / EPI_WARPS / 32;  // chunks per tile and warp
    int jr = 0;                                   // ring position (every chunk)
    // box origin of this warp's rows in tile tt (cached: chunks arrive in order)
    int rcT = -1, rcRow = 0, rcCol = 0, rcPr = 0;
    auto ringTile = [&](int tt) {
      if(tt == rcT)
        return;
      rcT = tt;
      rcPr = p.kconcat ? 0 : tt / tilesPerProb;
      const int r2 = (tt - rcPr * tilesPerProb) % tilesPerSplit;
      const int mi = r2 % p.mt;
      rcRow = mi * MT + (int)rank * BM + q * 32;
      rcCol = ((r2 - mi) / p.mt) * BN + cBeg;
    };
    auto ringIssue = [&](int jj) {  // lane 0: the box of this warp's chunk jj
      const int ti = jj / CPT, tt = unit0 + ti * units;
      if(tt >= p.numTiles)
        return;
      uint64_t* bar = &ldbar[ew * NB + jj % NB];
      ringTile(tt);
      const int col = rcCol + 32 * (jj - ti * CPT);
      if(rcRow >= p.M || col >= p.N) {  // nothing to load: complete the phase
        mbar_arrive(bar);
        return;
      }
      mbar_expect_tx(bar, 4096u);
      tma_load_2d(stage0 + (jj % NB) * 1024, p.hasAddend ? &maps.r : &maps.c[rcPr], bar, col,
                  rcRow);
    };
    if(ring && lane == 0)
      for(int jj = 0; jj < NB - 1; ++jj)
        ringIssue(jj);
    // LOADS with one extra source otherwise (the ReLU gate, or beta*C when
    // the ring is off): each lane prefetches its row's 32 values of the NEXT
    // chunk into registers while the current chunk is processed; both sources
    // together use TMA boxes.
    const bool pf = LOADS && !ring && !p.part && p.tmaStore && !(p.dbg & 4) &&
                    ((p.beta != 0.f) != (p.gate != nullptr));
    float nx[32];
    auto loadChunk = [&](int tt, int cc) {
      const int pr = p.kconcat ? 0 : tt / tilesPerProb;
      const int r2 = (tt - pr * tilesPerProb) % tilesPerSplit;
      const int64_t row = (int64_t)(r2 % p.mt) * MT + rank * BM + q * 32 + lane;
      const int64_t col = (int64_t)(r2 / p.mt) * BN + cc;
      const float* src = p.gate ? p.gate : (p.hasAddend ? p.addend : p.CP[pr]);
      src += row * p.ldc + col;
      if(row < p.M && col + 32 <= p.N && ((uintptr_t)src & 15) == 0) {
#pragma unroll
        for(int j = 0; j < 8; ++j) {
          const float4 x4 = *reinterpret_cast<const float4*>(src + 4 * j);
          nx[4 * j] = x4.x;
          nx[4 * j + 1] = x4.y;
          nx[4 * j + 2] = x4.z;
          nx[4 * j + 3] = x4.w;
        }
      } else {
#pragma unroll
        for(int i = 0; i < 32; ++i)
          nx[i] = (row < p.M && col + i < p.N) ? src[i] : 0.f;
      }
    };
    if(pf && unit0 < p.numTiles)
      loadChunk(unit0, cBeg);
    int lt = 0;
    for(int t = unit0; t < p.numTiles; t += units, ++lt) {
      int m0, n0, kb0, nkb, split;
      tileCoords(t, m0, n0, kb0, nkb, split);
      const int acc = lt & 1;
      const int64_t rowBase = m0 + q * 32;
      // the epilogue's extra sources (residual / beta*C, ReLU gate) of this
      // warp's rows into L2 while the tile's main loop still runs -- for the
      // ring, one tile ahead (its loads run a few chunks into the next tile)
      if(LOADS && p.tmaStore && !p.part && lane == 0) {
        for(int tp = (ring && lt == 0) ? t : (ring ? t + units : t);
            tp <= (ring ? t + units : t) && tp < p.numTiles; tp += units) {
          int pm0, pn0, pkb0, pnkb, psplit;
          tileCoords(tp, pm0, pn0, pkb0, pnkb, psplit);
          const int prow = pm0 + q * 32;
          if(prow >= p.M)
            continue;
          const int pr = p.kconcat ? 0 : tp / tilesPerProb;
          const CUtensorMap* src0 =
              p.beta != 0.f ? (p.hasAddend ? &maps.r : &maps.c[pr]) : nullptr;
          const CUtensorMap* src1 = p.gate ? &maps.g : nullptr;
          for(int c0 = cBeg; c0 < cEnd && pn0 + c0 < p.N; c0 += 32) {
            if(src0)
              tma_prefetch_2d(src0, pn0 + c0, prow);
            if(src1)
              tma_prefetch_2d(src1, pn0 + c0, prow);
          }
        }
        tprob = p.kconcat ? 0 : t / tilesPerProb;  // tileCoords above moved it
      }
      const float* biasT = p.biasP[tprob];
      // this warp's bias columns, lane l holding column cBeg + 32 j + l of
      // chunk j: loaded before the accumulator wait, so the latency hides
      // behind the main loop (broadcast to the row-owning lanes by shuffles)
      constexpr int NCH = BN * 4 / EPI_WARPS / 32;
      float bw[NCH];
#pragma unroll
      for(int j = 0; j < NCH; ++j) {
        const int64_t c = (int64_t)n0 + cBeg + 32 * j + lane;
        bw[j] = (biasT && !p.part && c < p.N) ? __ldg(biasT + c) : 0.f;
      }
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const CUtensorMap* mapC = &maps.c[p.part ? 0 : tprob];
      float* CT = p.CP[tprob];
      const int zpart = split * nOut + tprob;  // partial plane of this tile
      // relu_mask_out words of this lane's row, stored once per tile (a full
      // 16/32-byte run per row instead of one 4-byte store per chunk)
      constexpr int MWN = BN * 4 / EPI_WARPS / 32;
      uint32_t mwords[MWN];
#pragma unroll
      for(int j = 0; j < MWN; ++j)
        mwords[j] = 0;
#pragma unroll 1
      for(int c0 = cBeg; c0 < cEnd; c0 += 32) {
        float cur[32];
        if(pf) {
#pragma unroll
          for(int i = 0; i < 32; ++i)
            cur[i] = nx[i];
          const int tn = c0 + 32 < cEnd ? t : t + units;
          if(tn < p.numTiles)
            loadChunk(tn, c0 + 32 < cEnd ? c0 + 32 : cBeg);
        }
        float v[32];
        uint32_t gm = 0;  // gate-mask word of this lane's row and chunk (issued early)
        if(p.gateMask && !p.part && rowBase + lane < p.M && n0 + c0 < p.N)
          gm = __ldg(p.gateMask + (rowBase + lane) * p.maskW + (n0 + c0) / 32);
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), v);
        if(c0 + 32 >= cEnd) {  // our share read: hand it back to the MMA warp
          tc_fence_before();
          if(lane == 0) {
            if(PAIR)
              mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
            else
              mbar_arrive(&tempty[acc]);
          }
        }
        if(ring) {  // this chunk's box, whether or not the chunk is stored
          mbar_wait(&ldbar[ew * NB + jr % NB], (jr / NB) & 1);
        }
        if(n0 + c0 >= p.N || rowBase >= p.M || (p.dbg & 1)) {
          if(ring) {  // keep the ring moving: the buffer of chunk jr - 1 is free
            if(lane == 0) {
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              ringIssue(jr + NB - 1);
            }
            __syncwarp();
            ++jr;
          }
          continue;
        }
        const int64_t col0 = n0 + c0;
        if(p.tmaStore) {
          float* stage = ring ? stage0 + (jr % NB) * 1024 : stage0 + (chunk & 1) * 1024;
          // the TMA engine must have finished reading this buffer (chunk - 2)
          // before it is refilled: early when a C / gate box lands in it,
          // otherwise as late as possible (after the arithmetic)
          // boxes land in the staging buffer (LOADS without prefetch): wait early
          const bool loads = LOADS && !pf && !ring;
          if(chunk >= 2 && loads) {
            if(lane == 0)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
          }
          // 16-byte chunk j of row `lane` sits at j ^ (lane % 8) (SWIZZLE_128B),
          // both for the TMA-loaded C / gate boxes and for the store staging
          float* srow = stage + lane * 32;
          const int sw = lane & 7;
          if(!p.part) {
            const bool needC = LOADS && p.beta != 0.f, needG = LOADS && p.gate != nullptr;
            float* grow = stage;  // gate box buffer
            if((needC || needG) && !pf && !ring) {
              // C and/or the ReLU gate arrive as swizzled 32x32 boxes by TMA
              // (coalesced, async) instead of per-lane strided row reads
              if(needC && needG) {
                grow = stage0 + ((chunk + 1) & 1) * 1024;
                if(lane == 0)
                  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
              }
              if(lane == 0) {
                mbar_expect_tx(&ldbar[ew], (needC ? 4096u : 0u) + (needG ? 4096u : 0u));
                if(needC)
                  tma_load_2d(stage, p.hasAddend ? &maps.r : mapC, &ldbar[ew], (int)col0,
                              (int)rowBase);
                if(needG)
                  tma_load_2d(grow, &maps.g, &ldbar[ew], (int)col0, (int)rowBase);
              }
              mbar_wait(&ldbar[ew], ldPhase & 1);
              ++ldPhase;
            }
            grow += lane * 32;
            // alpha, bias, ReLU.  Full aligned chunks read the 32 bias values
            // as 8 same-address float4 loads (one broadcast transaction each);
            // ragged chunks use one load per lane broadcast by shuffles.
            if(p.alpha != 1.f) {
#pragma unroll
              for(int i = 0; i < 32; ++i)
                v[i] = p.alpha * v[i];
            }
            if(biasT) {
              const int jc = (c0 - cBeg) >> 5;
              float bl = bw[0];
#pragma unroll
              for(int j = 1; j < NCH; ++j)
                bl = j == jc ? bw[j] : bl;
#pragma unroll
              for(int i = 0; i < 32; ++i)
                v[i] = v[i] + __shfl_sync(0xffffffffu, bl, i);
            }
            if(p.epi == MTKC_EPI_RELU) {
#pragma unroll
              for(int i = 0; i < 32; ++i)
                v[i] = v[i] > 0.f ? v[i] : 0.f;
            }
            if(p.gateMask) {
#pragma unroll
              for(int i = 0; i < 32; ++i)
                v[i] = ((gm >> i) & 1u) ? v[i] : 0.f;
            }
            // ReLU gate, then beta*C, from the TMA-loaded boxes (straight-line
            // loops under uniform branches)
            if(pf) {
              if(needG) {
#pragma unroll
                for(int i = 0; i < 32; ++i)
                  v[i] = cur[i] > 0.f ? v[i] : 0.f;
              } else {
                const float beta = p.beta;
#pragma unroll
                for(int i = 0; i < 32; ++i)
                  v[i] = (beta == 1.f ? cur[i] : beta * cur[i]) + v[i];
              }
            } else if(needG) {
#pragma unroll
              for(int j = 0; j < 8; ++j) {
                const float4 g4 = *reinterpret_cast<const float4*>(grow + ((j ^ sw) * 4));
                v[4 * j] = g4.x > 0.f ? v[4 * j] : 0.f;
                v[4 * j + 1] = g4.y > 0.f ? v[4 * j + 1] : 0.f;
                v[4 * j + 2] = g4.z > 0.f ? v[4 * j + 2] : 0.f;
                v[4 * j + 3] = g4.w > 0.f ? v[4 * j + 3] : 0.f;
              }
            }
            if(needC && !pf) {
              const float beta = p.beta;
#pragma unroll
              for(int j = 0; j < 8; ++j) {
                const float4 c4 = *reinterpret_cast<const float4*>(srow + ((j ^ sw) * 4));
                if(beta == 1.f) {
                  v[4 * j] = c4.x + v[4 * j];
                  v[4 * j + 1] = c4.y + v[4 * j + 1];
                  v[4 * j + 2] = c4.z + v[4 * j + 2];
                  v[4 * j + 3] = c4.w + v[4 * j + 3];
                } else {
                  v[4 * j] = beta * c4.x + v[4 * j];
                  v[4 * j + 1] = beta * c4.y + v[4 * j + 1];
                  v[4 * j + 2] = beta * c4.z + v[4 * j + 2];
                  v[4 * j + 3] = beta * c4.w + v[4 * j + 3];
                }
              }
            }
            if(p.maskOut) {  // after beta*C: bits of the stored C, written per tile
              uint32_t w = 0;
#pragma unroll
              for(int i = 0; i < 32; ++i)
                w |= (v[i] > 0.f && col0 + i < p.N) ? (1u << i) : 0u;
              mwords[(c0 - cBeg) >> 5] = w;
            }
            __syncwarp();  // every lane has read its C / gate row before the overwrite
          }
          if(chunk >= 2 && !loads && !ring) {
            if(lane == 0)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
          }
#pragma unroll
          for(int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(srow + ((j ^ sw) * 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if(lane == 0) {
            if(p.part)
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                  ::"l"((uint64_t)mapC), "r"(smem_u32(stage)), "r"((int)col0), "r"((int)rowBase),
                  "r"(zpart)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                  ::"l"((uint64_t)mapC), "r"(smem_u32(stage)), "r"((int)col0), "r"((int)rowBase)
                  : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if(ring) {  // all but this store have read their buffers: refill one
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              ringIssue(jr + NB - 1);
            }
          }
          if(ring) {
            __syncwarp();
            ++jr;
          }
          ++chunk;
          continue;
        }
        // fallback: padded transpose through shared memory, coalesced row stores
        float* st = stage0;
#pragma unroll
        for(int i2 = 0; i2 < 32; ++i2)
          st[lane * EPI_STRIDE + i2] = v[i2];
        __syncwarp();
        const int64_t col = col0 + lane;
        const bool colOk = col < p.N;
        const float bcol = (biasT && colOk && !p.part) ? biasT[col] : 0.f;
        const int rows = (int)min((int64_t)32, p.M - rowBase);
        for(int r = 0; r < rows; ++r) {
          float x = st[r * EPI_STRIDE + lane];
          const int64_t rr = rowBase + r;
          if(p.maskOut && !p.part) {  // bits of the final value (lanes = columns)
            float y = p.alpha == 1.f ? x : p.alpha * x;
            if(biasT)
              y = y + bcol;
            if(p.epi == MTKC_EPI_RELU)
              y = y > 0.f ? y : 0.f;
            if(p.gate)
              y = (colOk && p.gate[rr * p.ldc + col] > 0.f) ? y : 0.f;
            if(p.gateMask)
              y = (colOk && ((p.gateMask[rr * p.maskW + col0 / 32] >> lane) & 1u)) ? y : 0.f;
            if(p.beta != 0.f && colOk) {
              const float cv = p.addend ? p.addend[rr * p.ldc + col] : CT[rr * p.ldc + col];
              y = (p.beta == 1.f ? cv : p.beta * cv) + y;
            }
            const uint32_t bits = __ballot_sync(0xffffffffu, colOk && y > 0.f);
            if(lane == 0)
              p.maskOut[rr * p.maskW + col0 / 32] = bits;
          }
          if(!colOk)
            continue;
          if(p.part) {
            p.part[((int64_t)zpart * p.M + rr) * p.N + col] = x;
            continue;
          }
          float* dst = CT + rr * p.ldc + col;
          x = p.alpha == 1.f ? x : p.alpha * x;
          if(biasT)
            x = x + bcol;
          if(p.epi == MTKC_EPI_RELU)
            x = x > 0.f ? x : 0.f;
          if(p.gate)
            x = p.gate[rr * p.ldc + col] > 0.f ? x : 0.f;
          if(p.gateMask)
            x = ((p.gateMask[rr * p.maskW + col0 / 32] >> lane) & 1u) ? x : 0.f;
          if(p.beta != 0.f) {
            const float cv = p.addend ? p.addend[rr * p.ldc + col] : *dst;
            x = (p.beta == 1.f ? cv : p.beta * cv) + x;
          }
          *dst = x;
        }
        __syncwarp();
      }
      if(p.maskOut && p.tmaStore && !p.part && rowBase + lane < p.M && n0 + cBeg < p.N) {
        uint32_t* dst = p.maskOut + (rowBase + lane) * p.maskW + (n0 + cBeg) / 32;
        const int nw = (int)min((int64_t)MWN, p.maskW - (n0 + cBeg) / 32);
        if(nw == MWN && ((uintptr_t)dst & 15) == 0) {
#pragma unroll
          for(int j = 0; j < MWN; j += 4)
            *reinterpret_cast<uint4*>(dst + j) =
                make_uint4(mwords[j], mwords[j + 1], mwords[j + 2], mwords[j + 3]);
        } else {
          for(int j = 0; j < nw; ++j)
            dst[j] = mwords[j];
        }
      }
    }
    if(lane == 0)
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  } else if(p.csOp) {
    // operand sums over k, read from the MN-major stages the MMA consumes.
    // A stage holds 32-column atoms of BK rows x 128 B (atom j at j*BK*128),
    // 128-byte swizzled in 32-byte units: unit u of row k sits at u ^ (k & 3)
    // (Swizzle<2,5,2>).  Lane 8r + c reads 16-byte chunk c of rows k = r
    // (mod 4), whose logical columns 8*((c>>1) ^ r) + 4*(c&1) + 0..3 are the
    // same for every such k; lanes l, l^10, l^20, l^30 hold the same columns.
    constexpr int CH = (BN > BM ? BN : BM) / 32;
    const bool sumB = p.csOp == 2;
    const int nch = sumB ? BNL / 32 : BM / 32;
    const uint32_t sBytes = sumB ? B_BYTES : A_BYTES;
    const uint8_t* sOp = (sumB ? sB : sA) + (lane >> 3) * 128 + (lane & 7) * 16;
    int i = 0;
    for(int t = unit0; t < p.numTiles; t += units) {
      int m0, n0, kb0, nkb, split;
      tileCoords(t, m0, n0, kb0, nkb, split);
      // the first csR tiles of the operand block take its k-blocks in turn
      const int R = p.csR, ri = sumB ? (m0 - (int)rank * BM) / MT : n0 / BN;
      const bool on = (sumB ? B_MN : A_MN) && ri < R;
      float4 acc[CH];
#pragma unroll
      for(int c = 0; c < CH; ++c)
        acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      for(int kb = 0; kb < nkb; ++kb, ++i) {
        const int s = i % ST;
        mbar_wait(&full[s], (i / ST) & 1);
        if(on && (kb0 + kb) % R == ri) {
          const uint8_t* base = sOp + s * sBytes;
#pragma unroll
          for(int c = 0; c < CH; ++c)
            if(c < nch) {
#pragma unroll
              for(int kr = 0; kr < BK / 4; ++kr) {
                const float4 x = *reinterpret_cast<const float4*>(base + c * (BK * 128) + kr * 512);
                acc[c].x += x.x;
                acc[c].y += x.y;
                acc[c].z += x.z;
                acc[c].w += x.w;
              }
            }
        }
        __syncwarp();
        if(lane == 0)
          mbar_arrive(&empty[s]);
      }
      if(!on)
        continue;
      const int64_t len = p.csLen, base0 = sumB ? n0 + (int)rank * BNL : m0;
      float* dst = p.csSlots > 1
                       ? p.csPart + ((int64_t)tprob * p.csSlots + split * R + ri) * len
                       : p.csOut[tprob];
      const bool add = p.csSlots == 1 && p.csAcc;
#pragma unroll
      for(int c = 0; c < CH; ++c)
        if(c < nch) {
          float v[4] = {acc[c].x, acc[c].y, acc[c].z, acc[c].w};
#pragma unroll
          for(int e = 0; e < 4; ++e) {
            v[e] += __shfl_xor_sync(0xffffffffu, v[e], 10);
            v[e] += __shfl_xor_sync(0xffffffffu, v[e], 20);
          }
          const int64_t col = base0 + c * 32 + lane * 4;  // lanes 0..7: r = 0
          if(lane < 8)
#pragma unroll
            for(int e = 0; e < 4; ++e)
              if(col + e < len)
                dst[col + e] = add ? dst[col + e] + v[e] : v[e];
        }
    }
  }
  tc_fence_before();
  if(PAIR)
    cluster_sync_all();  // no CTA leaves while its peer may still signal it
  else
    __syncthreads();
  if(warp == 1) {
    tc_fence_after();
    if(PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
  }
}

// C = alpha*sum_s part[s] (+bias, relu, gate) + beta*C  (fixed split order).
// Grid-stride over (row, 4-column group); float4 when N and ldc allow.
// per output problem (blockIdx.y): destination, bias and beta source
struct ReduceOut {
  float* C[3];
  const float* bias[3];
  const float* Cin[3];
  // fused operand sums: partials [nOut][csSlots][csLen] -> cs[q] (+=, csAcc)
  float* cs[3];
  const float* csPart;
  int64_t csLen;
  int csAcc, csSlots;
};

template <bool VEC>
__global__ void splitk_reduce_kernel(const float* part, int splits, int64_t plane, int64_t M,
                                     int64_t N, ReduceOut outs, int64_t ldc, float alpha,
                                     float beta, int epi, const float* gate,
                                     const uint32_t* gateMask) {
  MTKC_PDL_ENTRY();
  // problem q's partials start at part + q*M*N; splits are `plane` apart
  const int q = blockIdx.y;
  part += (int64_t)q * M * N;
  float* C = outs.C[q];
  const float* bias = outs.bias[q];
  const float* Cin = outs.Cin[q];
  const int64_t groups = (N + 3) / 4, total = M * groups;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
      i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / groups, c = (i - r * groups) * 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if(VEC) {
      // eight partial loads in flight, summed in split order
      for(int s0 = 0; s0 < splits; s0 += 8) {
        float4 x[8];
#pragma unroll
        for(int u = 0; u < 8; ++u)
          x[u] = s0 + u < splits ? __ldcs(reinterpret_cast<const float4*>(part + (s0 + u) * plane +
                                                                           r * N + c))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for(int u = 0; u < 8; ++u) {
          acc[0] += x[u].x;
          acc[1] += x[u].y;
          acc[2] += x[u].z;
          acc[3] += x[u].w;
        }
      }
    } else {
      for(int s = 0; s < splits; ++s)
        for(int u = 0; u < 4; ++u)
          if(c + u < N)
            acc[u] += part[s * plane + r * N + c + u];
    }
    float out[4];
    float* dst = C + r * ldc + c;
    const float* src = Cin + r * ldc + c;
    for(int u = 0; u < 4; ++u) {
      if(!VEC && c + u >= N)
        break;
      float x = alpha == 1.f ? acc[u] : alpha * acc[u];
      if(bias)
        x = x + bias[c + u];
      if(epi == MTKC_EPI_RELU)
        x = x > 0.f ? x : 0.f;
      if(gate)
        x = gate[r * ldc + c + u] > 0.f ? x : 0.f;
      if(gateMask)
        x = ((gateMask[r * ((N + 31) / 32) + (c + u) / 32] >> ((c + u) & 31)) & 1u) ? x : 0.f;
      if(beta != 0.f)
        x = (beta == 1.f ? src[u] : beta * src[u]) + x;
      out[u] = x;
    }
    if(VEC) {
      *reinterpret_cast<float4*>(dst) = make_float4(out[0], out[1], out[2], out[3]);
    } else {
      for(int u = 0; u < 4 && c + u < N; ++u)
        dst[u] = out[u];
    }
  }
  if(outs.csPart) {  // operand sums: splits added in order
    const float* cp = outs.csPart + (int64_t)q * outs.csSlots * outs.csLen;
    float* cs = outs.cs[q];
    for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < outs.csLen;
        i += (int64_t)gridDim.x * blockDim.x) {
      float x = 0.f;
      for(int s0 = 0; s0 < outs.csSlots; s0 += 8) {  // eight loads in flight
        float y[8];
#pragma unroll
        for(int u = 0; u < 8; ++u)
          y[u] = s0 + u < outs.csSlots ? cp[(s0 + u) * outs.csLen + i] : 0.f;
#pragma unroll
        for(int u = 0; u < 8; ++u)
          if(s0 + u < outs.csSlots)
            x += y[u];
      }
      cs[i] = outs.csAcc ? cs[i] + x : x;
    }
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
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// MN-major operand [rows x cols] (cols contiguous, cols % 32 == 0) as a 3-d
// tensor (32, rows, cols/32): one box of nbox 32-column atoms x boxRows rows
// lands exactly like nbox separate 2-d boxes (atom j at j * boxRows * 128 B)
bool make_map3(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld,
               uint32_t boxRows, uint32_t nbox) {
  EncodeFn fn = encode_fn();
  if(!fn || cols % 32)
    return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(cols / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, 128};
  cuuint32_t box[3] = {32, boxRows, nbox};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, tma_tf32_round() ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                  3, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// K-major operand [rows x K] (K contiguous, K % 32 == 0) as a 3-d tensor
// (32, rows, K/32): one box of KA atom columns x boxRows rows lands as
// [KA][boxRows][32] (atom column c at c * boxRows * 128 B)
bool make_mapk3(CUtensorMap* m, const float* base, int64_t K, int64_t rows, int64_t ld,
                uint32_t boxRows) {
  EncodeFn fn = encode_fn();
  if(!fn || K % 32)
    return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(K / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, 128};
  cuuint32_t box[3] = {32, boxRows, (cuuint32_t)KA};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, tma_tf32_round() ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                  3, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// store map over C [rows x cols] (ld elements), or over split-K partials
// [depth][rows][cols]; 32x32 boxes, 128-byte swizzle (matches the staging tile)
bool make_store_map(CUtensorMap* m, float* base, int64_t cols, int64_t rows, int64_t ld,
                    int64_t depth) {
  EncodeFn fn = encode_fn();
  if(!fn)
    return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)depth};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(ld * rows) * 4};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, depth > 1 ? 3 : 2, (void*)base, dims,
                  strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_sms = 0;
int g_sm_limit = 0;  // 0 = every SM; else the persistent grid's cap (SMs left to NCCL)
inline int gemm_sms() { return g_sm_limit > 0 && g_sm_limit < g_sms ? g_sm_limit : g_sms; }

// CTA pairs resident at once (clusters of two; a TPC's two SMs), 0 = unknown
int g_pair_units = 0;
bool g_pair_enabled = getenv("MTK_GEMM_NO_PAIR") == nullptr;
// pairs also for products with fused operand sums (the odd CTA relays its
// stage arrivals to the even CTA); MTK_GEMM_PAIR_NO_CS=1 keeps them single
bool g_pair_colsum = getenv("MTK_GEMM_PAIR_NO_CS") == nullptr;

template <int BN, bool A_MN, bool B_MN, bool LOADS, bool PAIR>
int launch_tc(const TcMaps& maps, const TcP& p, cudaStream_t st) {
  constexpr size_t smem = TcSmem<BN, PAIR, LOADS>::BYTES;
  auto kern = gemm_tf32_tc_kernel<BN, A_MN, B_MN, LOADS, PAIR>;
  static int units = 0;  // persistent grid cap (pairs for PAIR)
  if(!units) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if(e != cudaSuccess)
      return cuda_status(e, "gemm_tf32_tc smem attribute");
    units = g_sms;
    if(PAIR) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * (unsigned)(g_sms / 2));
      cfg.blockDim = dim3(TC_THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      e = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
      if(e != cudaSuccess || nc <= 0) {
        cudaGetLastError();
        nc = g_sms / 2;
      }
      units = std::min(nc, g_sms / 2);
      g_pair_units = units;
    }
  }
  const int cap = PAIR ? std::min(units, gemm_sms() / 2) : gemm_sms();
  const int grid = std::min(p.numTiles, std::max(1, cap));
  if(PAIR)
    ::mtkc::launch_cluster(kern, dim3(2 * grid), TC_THREADS, smem, st, 2, maps, p);
  else
    ::mtkc::launch(kern, grid, TC_THREADS, smem, st, maps, p);
  MTKC_POST_LAUNCH("gemm_tf32_tc_kernel");
  return MTKC_OK;
}

template <int BN, bool LOADS, bool PAIR>
int dispatch_majors(bool aMN, bool bMN, const TcMaps& maps, const TcP& p, cudaStream_t st) {
  if(!aMN && !bMN)
    return launch_tc<BN, false, false, LOADS, PAIR>(maps, p, st);
  if(!aMN && bMN)
    return launch_tc<BN, false, true, LOADS, PAIR>(maps, p, st);
  if(aMN && !bMN)
    return launch_tc<BN, true, false, LOADS, PAIR>(maps, p, st);
  return launch_tc<BN, true, true, LOADS, PAIR>(maps, p, st);
}

template <bool PAIR>
int dispatch_tc(int BN, bool loads, bool aMN, bool bMN, const TcMaps& maps, const TcP& p,
                cudaStream_t st) {
  if(loads)
    return BN == 256 ? dispatch_majors<256, true, PAIR>(aMN, bMN, maps, p, st)
                     : dispatch_majors<128, true, PAIR>(aMN, bMN, maps, p, st);
  return BN == 256 ? dispatch_majors<256, false, PAIR>(aMN, bMN, maps, p, st)
                   : dispatch_majors<128, false, PAIR>(aMN, bMN, maps, p, st);
}

}  // namespace

// Returns false when the tensor-core path does not apply (caller falls back).
// probs[0..nprob): one shape (M, N, K, strides, transposes, alpha, beta,
// epilogue) with per-problem A, B, C, bias.  kconcat: C = sum_p op(A_p)op(B_p)
// into probs[0].C (bias from probs[0]).  *csFused: the operand sums the
// problems ask for (colsum) were produced by this launch; when false the
// caller runs them separately.
bool tc_gemm_group(const mtkc_gemm_args* probs, int nprob, int kconcat, cudaStream_t st,
                   int* rc, bool* csFused) {
  *csFused = false;
  const mtkc_gemm_args& a = probs[0];
  if(getenv("MTK_DISABLE_TC"))
    return false;
  if(nprob < 1 || nprob > 3)
    return false;
  for(int q = 0; q < nprob; ++q) {
    const mtkc_gemm_args& b = probs[q];
    if(b.batch != 1 || b.M != a.M || b.N != a.N || b.K != a.K || b.lda != a.lda ||
       b.ldb != a.ldb || b.ldc != a.ldc || b.transA != a.transA || b.transB != a.transB)
      return false;
    if(((uintptr_t)b.A % 16) || ((uintptr_t)b.B % 16))
      return false;
  }
  if(nprob > 1 && (a.gate || a.addend || a.gate_mask || a.relu_mask_out))
    return false;
  if(a.M < 1 || a.N < 8 || a.K < 8)
    return false;
  if(a.lda % 4 || a.ldb % 4)
    return false;
  // operand majors: op(A) is K-major iff stored untransposed
  const bool aMN = a.transA != 0, bMN = a.transB == 0;
  // fused operand sums: every problem asks for the same MN-major operand
  int csOp = 0;
  if(a.colsum && !kconcat && !getenv("MTK_NO_FUSED_COLSUM")) {
    csOp = (a.colsum_of == MTKC_COLSUM_B && bMN) ? 2 : (a.colsum_of == MTKC_COLSUM_A && aMN) ? 1 : 0;
    for(int q = 1; q < nprob; ++q)
      if(!probs[q].colsum || probs[q].colsum_of != a.colsum_of ||
         probs[q].colsum_accumulate != a.colsum_accumulate)
        csOp = 0;
  }
  const int64_t csLen = csOp == 2 ? a.N : a.M;
  if(!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if(g_sms <= 0)
      g_sms = 148;
  }
  const int nOut = kconcat ? 1 : nprob;
  // CTA pairs (256-row tiles over two SMs; the fused operand sums are taken
  // by each CTA over its own staged half).  Measured (tools/epi_var.py,
  // gemm_bench.py MTK_BENCH_AB=1): pairs win
  // once the single-CTA tiles fill more than one wave or the k loop is long
  // (operand traffic dominates); a single short wave (M x 512 x 512) and the
  // small-M weight-gradient products stay single-CTA
  const int64_t tiles1 = cdiv(a.M, BM) * cdiv(a.N, a.N >= 256 ? 256 : 128) * nOut;
  // (M = 512 with N >= 2048 -- the d x 4d weight gradients: pairs measured
  // 35.3 -> 33.1 us at K = 6530; M x 512 stays single-CTA)
  static const int64_t pairMinM =
      getenv("MTK_GEMM_PAIR_MINM") ? atoll(getenv("MTK_GEMM_PAIR_MINM")) : 1024;
  const bool pairM = a.M >= pairMinM || (a.M >= 512 && a.N >= 2048);
  const bool pair = g_pair_enabled && pairM && (csOp == 0 || g_pair_colsum) &&
                    (tiles1 > gemm_sms() || cdiv(a.K, BK) * (kconcat ? nprob : 1) >= 32);
  // scheduling units: CTAs, or CTA pairs
  const int sms = pair ? std::max(1, (g_pair_units ? std::min(g_pair_units, gemm_sms() / 2)
                                                   : gemm_sms() / 2))
                       : gemm_sms();
  const int64_t mt = cdiv(a.M, pair ? 2 * BM : BM);
  // wide tiles halve the re-reads of A (the L2->SM operand traffic that
  // bounds fp32-storage GEMMs) -- worth a partly idle wave; narrow tiles only
  // when there are so few wide tiles that split-K would have to fill the GPU
  int BN = (a.N >= 256 && mt * cdiv(a.N, 256) * nOut >= (pair ? 16 : 32)) ? 256 : 128;
  if(const char* e = getenv("MTK_GEMM_BN"))  // tuning override (tools/gemm_bench.py)
    BN = (atoi(e) == 256 && a.N >= 256) ? 256 : 128;
  const int64_t nt = cdiv(a.N, BN);
  // tiles sharing the summed operand's k-blocks (MTK_CS_DIST=0: one tile);
  // capped so the reduce sums at most ~32 partial slots per column
  static const bool csDist = !getenv("MTK_CS_DIST") || getenv("MTK_CS_DIST")[0] != '0';
  const int64_t csTiles = csOp == 2 ? mt : nt;
  const int nkbProb = (int)cdiv(a.K, BK);
  const int numKb = kconcat ? nkbProb * nprob : nkbProb;
  // Split K to fill the machine: pick the split count that maximises the
  // wave efficiency of the persistent grid, tiles*s / (SMs*ceil(tiles*s/SMs));
  // ties go to fewer splits.  Skinny products (RNN time steps: M = batch
  // rows, a handful of tiles) split down to 4 k-blocks per CTA; otherwise
  // keep >= 24 per split.
  int splits = 1;
  const int64_t tiles = mt * nt * nOut;
  const int minKb = tiles * 4 <= sms ? 4 : 24;
  if(a.workspace && numKb >= 2 * minKb && !a.relu_mask_out) {  // masks: no split
    double best = (double)tiles / (double)(sms * cdiv(tiles, sms));
    static const int maxSplit = getenv("MTK_GEMM_MAXSPLIT") ? atoi(getenv("MTK_GEMM_MAXSPLIT")) : 8;
    for(int s = 2; s <= maxSplit && numKb / s >= minKb; ++s) {
      size_t need = (size_t)s * nOut * ((size_t)a.M * (size_t)a.N + (csOp ? csLen * csTiles : 0)) *
                    sizeof(float);
      if(need > a.workspace_bytes)
        break;
      double eff = (double)(tiles * s) / (double)(sms * cdiv(tiles * s, sms));
      // partial sums cost an extra write+read of M*N per split: demand a real gain
      if(eff > best * 1.08) {
        best = eff;
        splits = s;
      }
    }
  }
  const int kbPer = (int)cdiv(numKb, splits);
  splits = (int)cdiv(numKb, kbPer);
  const int64_t csR = csDist ? std::max<int64_t>(1, std::min<int64_t>(csTiles, 32 / splits)) : 1;

  TcMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  const bool no3d = getenv("MTK_GEMM_NO_3D") != nullptr;
  const bool a3d = aMN && a.M % 32 == 0 && !no3d, b3d = bMN && a.N % 32 == 0 && !no3d;
  const bool ak3d = KA > 1 && !aMN && a.K % 32 == 0 && !no3d;
  const bool bk3d = KA > 1 && !bMN && a.K % 32 == 0 && !no3d;
  for(int q = 0; q < nprob; ++q) {
    const mtkc_gemm_args& b = probs[q];
    bool ok;
    if(aMN && a3d)
      ok = make_map3(&maps.a[q], b.A, a.M, a.K, a.lda, BK, BM / 32);
    else if(aMN)  // storage [K x M], M contiguous
      ok = make_map(&maps.a[q], b.A, a.M, a.K, a.lda, 32, BK, true);
    else if(ak3d)  // storage [M x K], KA atom columns per stage in one box
      ok = make_mapk3(&maps.a[q], b.A, a.K, a.M, a.lda, BM);
    else     // storage [M x K]
      ok = make_map(&maps.a[q], b.A, a.K, a.M, a.lda, 32, BM, false);
    if(!ok)
      return false;
    const uint32_t bnl = pair ? (uint32_t)BN / 2 : (uint32_t)BN;  // B columns per CTA
    if(bMN && b3d)
      ok = make_map3(&maps.b[q], b.B, a.N, a.K, a.ldb, BK, bnl / 32);
    else if(bMN)  // storage [K x N]
      ok = make_map(&maps.b[q], b.B, a.N, a.K, a.ldb, 32, BK, true);
    else if(bk3d)
      ok = make_mapk3(&maps.b[q], b.B, a.K, a.N, a.ldb, bnl);
    else     // storage [N x K]
      ok = make_map(&maps.b[q], b.B, a.K, a.N, a.ldb, 32, bnl, false);
    if(!ok)
      return false;
  }

  TcP p;
  std::memset(&p, 0, sizeof(p));
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
  p.nprob = nprob;
  p.a3d = a3d;
  p.b3d = b3d;
  p.ak3d = ak3d;
  p.bk3d = bk3d;
  p.addend = a.addend;
  p.hasAddend = a.addend != nullptr;
  p.kconcat = kconcat;
  p.nkbProb = nkbProb;
  for(int q = 0; q < nOut; ++q) {
    p.biasP[q] = probs[q].bias;
    p.CP[q] = probs[q].C;
    p.csOut[q] = csOp ? probs[q].colsum : nullptr;
  }
  p.part = splits > 1 ? a.workspace : nullptr;
  p.csOp = csOp;
  p.csAcc = a.colsum_accumulate;
  p.csLen = csLen;
  p.maskOut = a.relu_mask_out;
  p.gateMask = a.gate_mask;
  p.maskW = (a.N + 31) / 32;
  p.csSlots = csOp ? (int)(splits * csR) : 0;
  p.csR = (int)csR;
  p.csPart = nullptr;
  if(p.csSlots > 1) {
    const size_t off = splits > 1 ? (size_t)splits * nOut * a.M * a.N : 0;
    const size_t need = (off + (size_t)nOut * p.csSlots * csLen) * sizeof(float);
    if(!a.workspace || need > a.workspace_bytes) {
      p.csOp = 0;  // no room for the partials: the caller sums separately
      p.csSlots = 0;
      csOp = 0;
    } else {
      p.csPart = a.workspace + off;
    }
  }
  p.kbPerSplit = kbPer;
  p.numKb = numKb;
  p.mt = (int)mt;
  p.nt = (int)nt;
  p.splits = splits;
  p.numTiles = (int)(mt * nt * splits * nOut);
  {
    const char* e = getenv("MTK_GEMM_DEBUG");
    p.dbg = e ? atoi(e) : 0;
  }
  bool store = true;
  if(p.part) {
    store = (a.N % 4 == 0) && ((uintptr_t)a.workspace % 16 == 0) &&
            make_store_map(&maps.c[0], a.workspace, a.N, a.M, a.N, (int64_t)splits * nOut);
  } else {
    for(int q = 0; q < nOut && store; ++q)
      store = (a.ldc % 4 == 0) && ((uintptr_t)probs[q].C % 16 == 0) &&
              make_store_map(&maps.c[q], probs[q].C, a.N, a.M, a.ldc, 1);
  }
  // the ReLU gate is read as TMA boxes too (same geometry as C)
  if(store && !p.part && a.gate)
    store = ((uintptr_t)a.gate % 16 == 0) &&
            make_store_map(&maps.g, const_cast<float*>(a.gate), a.N, a.M, a.ldc, 1);
  if(store && !p.part && a.addend)
    store = ((uintptr_t)a.addend % 16 == 0) &&
            make_store_map(&maps.r, const_cast<float*>(a.addend), a.N, a.M, a.ldc, 1);
  p.tmaStore = store ? 1 : 0;
  if(getenv("MTK_GEMM_NO_TMA_STORE"))
    p.tmaStore = 0;
  const bool loads = p.tmaStore && !p.part && (a.beta != 0.f || a.gate != nullptr);
  *rc = pair ? dispatch_tc<true>(BN, loads, aMN, bMN, maps, p, st)
             : dispatch_tc<false>(BN, loads, aMN, bMN, maps, p, st);
  if(*rc == MTKC_OK && splits > 1) {  // one launch for every output problem
    ReduceOut outs{};
    bool vec = a.N % 4 == 0 && a.ldc % 4 == 0 && (uintptr_t)a.workspace % 16 == 0;
    for(int q = 0; q < nOut; ++q) {
      outs.C[q] = probs[q].C;
      outs.bias[q] = probs[q].bias;
      outs.Cin[q] = a.addend ? a.addend : probs[q].C;
      outs.cs[q] = p.csOut[q];
      vec = vec && (uintptr_t)probs[q].C % 16 == 0;
    }
    outs.csPart = p.csPart;
    outs.csLen = csLen;
    outs.csAcc = a.colsum_accumulate;
    outs.csSlots = p.csSlots;
    const int64_t sstride = (int64_t)nOut * a.M * a.N;  // between splits
    const dim3 grid(grid1d(a.M * cdiv(a.N, 4), 256, 148 * 32 / std::max(1, nOut)),
                    (unsigned)nOut);
    if(vec)
      ::mtkc::launch(splitk_reduce_kernel<true>, grid, 256, 0, st, a.workspace, splits, sstride,
                     a.M, a.N, outs, a.ldc, a.alpha, a.beta, a.epilogue, a.gate, a.gate_mask);
    else
      ::mtkc::launch(splitk_reduce_kernel<false>, grid, 256, 0, st, a.workspace, splits,
                     sstride, a.M, a.N, outs, a.ldc, a.alpha, a.beta, a.epilogue, a.gate,
                     a.gate_mask);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if(e != cudaSuccess)
      *rc = cuda_status(e, "splitk_reduce_kernel");
  }
  if(*rc == MTKC_OK && splits == 1 && p.csPart) {  // operand-sum partials only
    ReduceOut outs{};
    for(int q = 0; q < nOut; ++q)
      outs.cs[q] = p.csOut[q];
    outs.csPart = p.csPart;
    outs.csLen = csLen;
    outs.csAcc = a.colsum_accumulate;
    outs.csSlots = p.csSlots;
    const dim3 grid(grid1d(csLen, 256, 148), (unsigned)nOut);
    ::mtkc::launch(splitk_reduce_kernel<false>, grid, 256, 0, st, (const float*)nullptr, 1,
                   (int64_t)0, (int64_t)0, a.N, outs, a.ldc, a.alpha, a.beta, a.epilogue,
                   (const float*)nullptr, (const uint32_t*)nullptr);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if(e != cudaSuccess)
      *rc = cuda_status(e, "splitk_reduce_kernel");
  }
  *csFused = csOp != 0;
  return true;
}

bool tc_gemm(const mtkc_gemm_args& a, cudaStream_t st, int* rc, bool* csFused) {
  return tc_gemm_group(&a, 1, 0, st, rc, csFused);
}

}  // namespace mtkc

namespace mtkc {
void gemm_set_sm_limit(int sms) { g_sm_limit = sms > 0 ? sms : 0; }
}  // namespace mtkc

extern "C" int mtkc_gemm_set_pair(int enable) {
  mtkc::g_pair_enabled = enable != 0;
  mtkc::g_pair_colsum = enable != 3;
  return MTKC_OK;
}

extern "C" int mtkc_gemm_set_sm_limit(int sms) {
  mtkc::gemm_set_sm_limit(sms);
  return MTKC_OK;
}
