// Sequence-level GRU recurrences: the whole time loop of a deep-transition
// GRU stack (RnnEncoder::build, RnnDecoder::step, reference models.cpp:
// 140-193 and 264-391; DeepTransitionCell layers.cpp:183-244) as ONE graph
// node instead of one gruCell/bahdanau/maskBlend node per block and step.
//
// The arithmetic per block and step is the reference's (the gru_* and
// bahdanau_* kernels that back gruCell / the attention node), but the work
// is re-scheduled for the B200:
//   * the input products x*[Wz|Wr|Wx] of block 1 are one GEMM over all
//     b*T rows (time-major), not T skinny per-step products;
//   * every weight gradient (dU, dW, the attention W) and every bias / layer-
//     norm / attention-v gradient is ONE GEMM / column sum over all b*T rows
//     after the reverse sweep, instead of T per-step products and sums --
//     the per-step gate gradients are kept time-major for that;
//   * the padding blend (maskBlend) is folded into the last block's
//     pointwise kernel (forward and backward);
//   * the two directions of the bidirectional encoder run concurrently on
//     two streams (their per-step GEMMs fill different SMs).
// What stays sequential is what the recurrence forces: per step and block
// one h*U product (grouped z|r|h launch) and one pointwise kernel forward,
// one pointwise kernel and one K-concatenated (dz|dr|dh)*U^T product
// backward, plus the attention between blocks 1 and 2 of the decoder.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "mtk/device.h"
#include "mtk/graph.h"

namespace mtk {

namespace {

// GEMM launch context: stream + its own slice of the device scratch (the
// side stream must not share split-K partials with the compute stream)
struct Ctx {
  void* st;
  float* ws;
  size_t wsBytes;
  float* cs;  // column-sum workspace
  size_t csBytes;
};

Ctx ctxFor(int lane) {
  Device& d = Device::get();
  const size_t total = (size_t)1 << 30;
  float* base = d.scratch(total);
  const size_t q = total / 4;
  float* p = base + (size_t)lane * 2 * (q / sizeof(float));
  void* st = lane == 0 ? d.stream() : d.sideStream();
  return Ctx{st, p, q, p + q / sizeof(float), q};
}

void gemm1(const Ctx& c, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, bool tA,
           const float* B, int64_t ldb, bool tB, float* C, int64_t ldc, float beta) {
  mtkc_gemm_args g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch = 1;
  g.A = A;
  g.lda = lda;
  g.transA = tA;
  g.B = B;
  g.ldb = ldb;
  g.transB = tB;
  g.C = C;
  g.ldc = ldc;
  g.alpha = 1.f;
  g.beta = beta;
  g.precision = (int)Device::get().precision();
  g.workspace = c.ws;
  g.workspace_bytes = c.wsBytes;
  MTKC(mtkc_gemm(&g, c.st));
}

// n = 3 products of one shape: independent outputs, or C[0] += sum_k
// A[k] op(B[k]) (kconcat).  Mixed accumulate flags fall back to singles.
void gemm3(const Ctx& c, bool kconcat, int64_t M, int64_t N, int64_t K, const float* const* A,
           int64_t lda, bool tA, const float* const* B, int64_t ldb, bool tB, float* const* C,
           int64_t ldc, const float* beta) {
  if(!kconcat && !(beta[0] == beta[1] && beta[1] == beta[2])) {
    for(int k = 0; k < 3; ++k)
      gemm1(c, M, N, K, A[k], lda, tA, B[k], ldb, tB, C[k], ldc, beta[k]);
    return;
  }
  mtkc_gemm_args g[3];
  for(int k = 0; k < 3; ++k) {
    g[k] = mtkc_gemm_args{};
    g[k].M = M;
    g[k].N = N;
    g[k].K = K;
    g[k].batch = 1;
    g[k].A = A[k];
    g[k].lda = lda;
    g[k].transA = tA;
    g[k].B = B[k];
    g[k].ldb = ldb;
    g[k].transB = tB;
    g[k].C = C[kconcat ? 0 : k];
    g[k].ldc = ldc;
    g[k].alpha = 1.f;
    g[k].beta = beta[kconcat ? 0 : k];
    g[k].precision = (int)Device::get().precision();
    g[k].workspace = c.ws;
    g[k].workspace_bytes = c.wsBytes;
  }
  MTKC(mtkc_gemm_group(g, 3, kconcat ? 1 : 0, c.st));
}

void colsum(const Ctx& c, ExpressionGraph::GradDst dst, const float* in, int64_t rows,
            int64_t cols) {
  MTKC(mtkc_colsum(dst.ptr, in, rows, cols, dst.accumulate, c.cs, c.csBytes, c.st));
}

// slots (positions in Node::inputs) of one block's parameters
struct BlockSlots {
  int U[3], b[3], W[3] = {-1, -1, -1}, ln[6] = {-1, -1, -1, -1, -1, -1};
  int64_t in = 0;  // block input dim (0: transition-only)
};

BlockSlots addBlock(ExpressionGraph::Node& n, const GruParams& p, bool ln, int64_t in) {
  BlockSlots s;
  auto push = [&](const NodeRef& r) {
    n.inputs.push_back(r.index);
    return (int)n.inputs.size() - 1;
  };
  s.U[0] = push(p.Uz);
  s.b[0] = push(p.bz);
  s.U[1] = push(p.Ur);
  s.b[1] = push(p.br);
  s.U[2] = push(p.Uh);
  s.b[2] = push(p.bh);
  s.in = in;
  if(in > 0) {
    s.W[0] = push(p.Wz);
    s.W[1] = push(p.Wr);
    s.W[2] = push(p.Wx);
  }
  if(ln) {
    s.ln[0] = push(p.lnGz);
    s.ln[1] = push(p.lnBz);
    s.ln[2] = push(p.lnGr);
    s.ln[3] = push(p.lnBr);
    if(in > 0) {
      s.ln[4] = push(p.lnGx);
      s.ln[5] = push(p.lnBx);
    }
  }
  return s;
}

struct AttSlots {
  int W = -1, v = -1, lnG = -1, lnB = -1, keys = -1, uk = -1;
  int64_t S = 0, a = 0, kd = 0;
  Tensor mask;  // [b x S] host/device
  bool hasMask = false;
};

// One direction of a scan: parameters, and the buffers the forward keeps for
// the backward (all time-major: row t*b + r).
struct Dir {
  std::vector<BlockSlots> blocks;
  bool reverse = false;
  // forward state
  Tensor HH;  // [(T+1)*b x d]: h0 and every blended state H_t
  std::vector<Tensor> hu, cache, lnc, lnrs;  // per block ([T*b x d] / [T*b x 3d] / [T*b x 3])
  Tensor soutAll;  // outputs of blocks 1..K-1, block k at k*T*b rows ([(K-1)*T*b x d])
  int64_t soutStride = 0;  // T*b*d
  float* sout(int64_t k) const { return soutAll.dev() + k * soutStride; }
  Tensor xw1, xw2, ctx, wq, attT, attW, attLnx, attLnrs, attScratch;
  // backward
  Tensor GH;  // [(T+1)*b x d] gradient of HH
  struct Grads {
    Tensor dpz, dpr, duh, dac, dax, lnp;
    Tensor dGx;  // persistent layout: [dpz | dpr | dax] rows (blocks with an input)
  };
  // persistent backward layout: [dpz | dpr | duh] rows of every block in one
  // buffer (block k at k*T*b rows), the A operand of the in-kernel products
  bool inter = false;
  Tensor dGall;
  std::vector<Grads> G;       // per block, time-major gate gradients
  std::vector<Tensor> ds;     // gradients of the intermediate block outputs of a step
  Tensor dctx, dwq, vpart;
  ExpressionGraph::GradDst guk{}, gkeys{};
  const float* ctxGrad = nullptr;
};

struct ScanAux {
  int64_t b = 0, T = 0, d = 0, e = 0;
  bool ln = false;
  int xSlot = -1, h0Slot = -1;
  Dir dir[2];
  int ndir = 1;
  bool att = false;
  AttSlots A;
  Tensor maskT;  // time-major [T x b] padding mask, or empty
  int ctxView = -1, lastView = -1;
  Tensor xt;     // time-major input [T*b x e]
};

inline int64_t hprevSlot(const Dir& D, int64_t t) { return D.reverse ? t + 1 : t; }
inline int64_t hSlot(const Dir& D, int64_t t) { return D.reverse ? t : t + 1; }

void forwardBegin(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X, Dir& D, const Ctx& c,
                  const float* h0) {
  const int64_t b = X.b, T = X.T, d = X.d, d3 = 3 * d, K = (int64_t)D.blocks.size();
  D.HH = g.allocTensor(Shape({(T + 1) * b, d}));
  float* HH = D.HH.dev();
  const int64_t h0slot = D.reverse ? T : 0;
  if(h0)
    MTKC(mtkc_memcpy_d2d(HH + h0slot * b * d, h0, (size_t)(b * d) * sizeof(float), c.st));
  else
    MTKC(mtkc_memset(HH + h0slot * b * d, 0, (size_t)(b * d) * sizeof(float), c.st));
  if(K > 1)
    D.soutAll = g.allocTensor(Shape({(K - 1) * T * b, d}));
  D.soutStride = T * b * d;
  D.hu.assign((size_t)K, Tensor());
  D.cache.assign((size_t)K, Tensor());
  D.lnc.assign((size_t)K, Tensor());
  D.lnrs.assign((size_t)K, Tensor());
  for(int64_t k = 0; k < K; ++k) {
    D.hu[(size_t)k] = g.allocTensor(Shape({T * b, d3}));
    D.cache[(size_t)k] = g.allocTensor(Shape({T * b, d3}));
    if(X.ln) {
      D.lnc[(size_t)k] = g.allocTensor(Shape({T * b, d3}));
      D.lnrs[(size_t)k] = g.allocTensor(Shape({T * b, 3}));
    }
  }
  const BlockSlots& B0 = D.blocks[0];
  if(B0.in > 0) {  // hoisted input products of block 1: one GEMM over b*T rows
    D.xw1 = g.allocTensor(Shape({T * b, d3}));
    float* xw = D.xw1.dev();
    const float* A[3] = {X.xt.devc(), X.xt.devc(), X.xt.devc()};
    const float* Bw[3] = {g.valPtr(n.inputs[(size_t)B0.W[0]]), g.valPtr(n.inputs[(size_t)B0.W[1]]),
                          g.valPtr(n.inputs[(size_t)B0.W[2]])};
    float* C[3] = {xw, xw + d, xw + 2 * d};
    const float beta[3] = {0.f, 0.f, 0.f};
    gemm3(c, false, T * b, d, X.e, A, X.e, false, Bw, d, false, C, d3, beta);
  }
  const AttSlots& A = X.A;
  if(X.att) {
    D.xw2 = g.allocTensor(Shape({T * b, d3}));
    D.ctx = g.allocTensor(Shape({T * b, A.kd}));
    D.wq = g.allocTensor(Shape({T * b, A.a}));
    D.attT = g.allocTensor(Shape({T * b * A.S, A.a}));
    D.attW = g.allocTensor(Shape({T * b, A.S}));
    if(A.lnG >= 0) {
      D.attLnx = g.allocTensor(Shape({T * b * A.S, A.a}));
      D.attLnrs = g.allocTensor(Shape({T * b, A.S}));
    }
  }
  if(X.att)
    D.attScratch = g.allocTensor(Shape({4, b, A.S}));
}

// step i of the recurrence (t = i, or T-1-i for the reverse direction)
void forwardStep(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X, Dir& D, const Ctx& c,
                 int64_t i) {
  const int64_t b = X.b, T = X.T, d = X.d, d3 = 3 * d, K = (int64_t)D.blocks.size();
  float* HH = D.HH.dev();
  const AttSlots& A = X.A;
  const float* maskT = X.maskT.empty() ? nullptr : X.maskT.devc();
  {
    const int64_t t = D.reverse ? T - 1 - i : i;
    const float* hprev = HH + hprevSlot(D, t) * b * d;
    const float* s = hprev;
    for(int64_t k = 0; k < K; ++k) {
      const BlockSlots& Bk = D.blocks[(size_t)k];
      float* hu = D.hu[(size_t)k].dev() + t * b * d3;
      {
        const float* Ah[3] = {s, s, s};
        const float* Bu[3] = {g.valPtr(n.inputs[(size_t)Bk.U[0]]),
                              g.valPtr(n.inputs[(size_t)Bk.U[1]]),
                              g.valPtr(n.inputs[(size_t)Bk.U[2]])};
        float* C[3] = {hu, hu + d, hu + 2 * d};
        const float beta[3] = {0.f, 0.f, 0.f};
        gemm3(c, false, b, d, d, Ah, d, false, Bu, d, false, C, d3, beta);
      }
      const float* xw = nullptr;
      if(k == 0 && Bk.in > 0)
        xw = D.xw1.devc() + t * b * d3;
      if(k == 1 && X.att) {  // block 2 reads the attention context of block 1's state
        float* x2 = D.xw2.dev() + t * b * d3;
        const float* cx = D.ctx.devc() + t * b * A.kd;
        const float* Ac[3] = {cx, cx, cx};
        const float* Bw[3] = {g.valPtr(n.inputs[(size_t)Bk.W[0]]),
                              g.valPtr(n.inputs[(size_t)Bk.W[1]]),
                              g.valPtr(n.inputs[(size_t)Bk.W[2]])};
        float* C[3] = {x2, x2 + d, x2 + 2 * d};
        const float beta[3] = {0.f, 0.f, 0.f};
        gemm3(c, false, b, d, A.kd, Ac, A.kd, false, Bw, d, false, C, d3, beta);
        xw = x2;
      }
      mtkc_gru_args a{};
      a.b = b;
      a.d = d;
      a.h = s;
      a.hu = hu;
      a.xw = xw;
      a.bz = g.valPtr(n.inputs[(size_t)Bk.b[0]]);
      a.br = g.valPtr(n.inputs[(size_t)Bk.b[1]]);
      a.bh = g.valPtr(n.inputs[(size_t)Bk.b[2]]);
      if(X.ln) {
        a.lnGz = g.valPtr(n.inputs[(size_t)Bk.ln[0]]);
        a.lnBz = g.valPtr(n.inputs[(size_t)Bk.ln[1]]);
        a.lnGr = g.valPtr(n.inputs[(size_t)Bk.ln[2]]);
        a.lnBr = g.valPtr(n.inputs[(size_t)Bk.ln[3]]);
        if(xw) {
          a.lnGx = g.valPtr(n.inputs[(size_t)Bk.ln[4]]);
          a.lnBx = g.valPtr(n.inputs[(size_t)Bk.ln[5]]);
        }
        a.lnc = D.lnc[(size_t)k].dev() + t * b * d3;
        a.lnrs = D.lnrs[(size_t)k].dev() + t * b * 3;
      }
      a.eps = 1e-9f;  // graph.cpp:690
      a.cache = D.cache[(size_t)k].dev() + t * b * d3;
      float* out = k == K - 1 ? HH + hSlot(D, t) * b * d : D.sout(k) + t * b * d;
      a.hout = out;
      if(k == K - 1 && maskT) {  // keep the old state at padded positions
        a.blend_mask = maskT + t * b;
        a.blend_prev = hprev;
      }
      MTKC(mtkc_gru_forward(&a, c.st));
      s = out;
      if(k == 0 && X.att) {  // Bahdanau attention on block 1's state
        float* wq = D.wq.dev() + t * b * A.a;
        gemm1(c, b, A.a, d, s, d, false, g.valPtr(n.inputs[(size_t)A.W]), A.a, false, wq, A.a,
              0.f);
        mtkc_bahdanau_args p{};
        p.b = b;
        p.s = A.S;
        p.a = A.a;
        p.kd = A.kd;
        p.wq = wq;
        p.uk = g.valPtr(n.inputs[(size_t)A.uk]);
        p.v = g.valPtr(n.inputs[(size_t)A.v]);
        p.keys = g.valPtr(n.inputs[(size_t)A.keys]);
        p.mask = A.hasMask ? A.mask.devc() : nullptr;
        if(A.lnG >= 0) {
          p.lnG = g.valPtr(n.inputs[(size_t)A.lnG]);
          p.lnB = g.valPtr(n.inputs[(size_t)A.lnB]);
          p.lnxh = D.attLnx.dev() + t * b * A.S * A.a;
          p.lnrs = D.attLnrs.dev() + t * b * A.S;
        }
        p.eps = 1e-9f;
        p.t = D.attT.dev() + t * b * A.S * A.a;
        p.w = D.attW.dev() + t * b * A.S;
        p.ctx = D.ctx.dev() + t * b * A.kd;
        p.flags = Device::get().flags();
        p.scratch = D.attScratch.dev();
        MTKC(mtkc_bahdanau_forward(&p, c.st));
      }
    }
  }
}

// ---------------------------------------------------------- persistent path

// TF32 mode runs the whole forward recurrence as one cooperative kernel
// (kernels/rnn_persist.cu) when its dimension constraints hold;
// MTK_RNN_PERSIST=0 selects the per-step launches (forwardStep) instead.
bool persistEnabled() {
  const char* e = std::getenv("MTK_RNN_PERSIST");
  return !(e && e[0] == '0') && Device::get().precision() == Precision::TF32;
}

void fillDir(ExpressionGraph& g, ExpressionGraph::Node& n, const ScanAux& X, Dir& D,
             mtkc_rnn_dir& o) {
  const int64_t K = (int64_t)D.blocks.size();
  o.reverse = D.reverse ? 1 : 0;
  o.nblocks = (int)K;
  for(int64_t k = 0; k < K; ++k) {
    const BlockSlots& Bk = D.blocks[(size_t)k];
    mtkc_rnn_block& B = o.blk[k];
    for(int j = 0; j < 3; ++j) {
      B.U[j] = g.valPtr(n.inputs[(size_t)Bk.U[j]]);
      B.bias[j] = g.valPtr(n.inputs[(size_t)Bk.b[j]]);
      B.W[j] = (k == 1 && X.att) ? g.valPtr(n.inputs[(size_t)Bk.W[j]]) : nullptr;
    }
    for(int j = 0; j < 6; ++j)
      B.ln[j] = (X.ln && Bk.ln[j] >= 0) ? g.valPtr(n.inputs[(size_t)Bk.ln[j]]) : nullptr;
    B.hu = D.hu[(size_t)k].dev();
    B.cache = D.cache[(size_t)k].dev();
    B.lnc = X.ln ? D.lnc[(size_t)k].dev() : nullptr;
    B.lnrs = X.ln ? D.lnrs[(size_t)k].dev() : nullptr;
  }
  o.HH = D.HH.dev();
  o.sout = K > 1 ? D.soutAll.dev() : nullptr;
  o.xw1 = D.xw1.empty() ? nullptr : D.xw1.devc();
  o.xw2 = X.att ? D.xw2.dev() : nullptr;
}

mtkc_rnn_scan_args scanArgs(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X) {
  mtkc_rnn_scan_args a{};
  a.b = X.b;
  a.T = X.T;
  a.d = X.d;
  a.ndir = X.ndir;
  a.eps = 1e-9f;  // graph.cpp:690
  a.maskT = X.maskT.empty() ? nullptr : X.maskT.devc();
  for(int q = 0; q < X.ndir; ++q)
    fillDir(g, n, X, X.dir[q], a.dir[q]);
  a.flags = Device::get().flags();
  if(X.att) {
    const AttSlots& A = X.A;
    Dir& D = X.dir[0];
    a.has_att = 1;
    a.S = A.S;
    a.a = A.a;
    a.kd = A.kd;
    a.attW = g.valPtr(n.inputs[(size_t)A.W]);
    a.attV = g.valPtr(n.inputs[(size_t)A.v]);
    a.attLnG = A.lnG >= 0 ? g.valPtr(n.inputs[(size_t)A.lnG]) : nullptr;
    a.attLnB = A.lnB >= 0 ? g.valPtr(n.inputs[(size_t)A.lnB]) : nullptr;
    a.keys = g.valPtr(n.inputs[(size_t)A.keys]);
    a.uk = g.valPtr(n.inputs[(size_t)A.uk]);
    a.attMask = A.hasMask ? A.mask.devc() : nullptr;
    a.wq = D.wq.dev();
    a.attT = D.attT.dev();
    a.attWts = D.attW.dev();
    a.attLnx = A.lnG >= 0 ? D.attLnx.dev() : nullptr;
    a.attLnrs = A.lnG >= 0 ? D.attLnrs.dev() : nullptr;
    a.ctx = D.ctx.dev();
  }
  return a;
}

// true when the persistent kernel ran the recurrence (all T steps)
bool forwardPersistent(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X) {
  if(!persistEnabled())
    return false;
  mtkc_rnn_scan_args a = scanArgs(g, n, X);
  // the backward will be persistent too (same conditions): skip the caches
  // only the per-step backward reads
  a.lean_cache = !(X.att && X.A.kd > 2048) ? 1 : 0;
  const bool ok = mtkc_rnn_scan_supported(&a) != 0;
  Device& dev = Device::get();
  const size_t need = ok ? mtkc_rnn_scan_workspace(&a) : 0;
  if(std::getenv("MTK_RNN_DEBUG"))
    std::fprintf(stderr, "[rnn scan] ndir %d b %lld T %lld d %lld blocks %d att %d: %s, %zu B\n",
                 a.ndir, (long long)a.b, (long long)a.T, (long long)a.d, a.dir[0].nblocks,
                 a.has_att, ok ? "persistent" : "per-step", need);
  if(!ok)
    return false;
  // the upper half of the device scratch (ctxFor(1)'s slice; the side
  // stream is idle while the persistent kernel runs on the compute stream)
  const size_t total = (size_t)1 << 30;
  if(need > total / 2)
    return false;
  float* base = dev.scratch(total);
  a.workspace = base + (total / 2) / sizeof(float);
  a.workspace_bytes = total / 2;
  MTKC(mtkc_rnn_scan_forward(&a, dev.stream()));
  return true;
}

// the persistent backward applies to this scan (checked before the
// gradient buffers are laid out for it)
bool persistBwdEligible(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X) {
  if(!persistEnabled() || (X.att && X.A.kd > 2048))
    return false;
  mtkc_rnn_scan_args a = scanArgs(g, n, X);
  return mtkc_rnn_scan_supported(&a) != 0;
}

void backwardPersistent(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X) {
  mtkc_rnn_scan_args a = scanArgs(g, n, X);
  for(int q = 0; q < X.ndir; ++q) {
    Dir& D = X.dir[q];
    mtkc_rnn_dir& o = a.dir[q];
    o.GH = D.GH.dev();
    o.dG = D.dGall.dev();
    for(size_t k = 0; k < D.blocks.size(); ++k) {
      Dir::Grads& gq = D.G[k];
      o.blk[k].dGx = gq.dGx.empty() ? nullptr : gq.dGx.dev();
      o.blk[k].dac = gq.dac.dev();
      o.blk[k].lnp = gq.lnp.empty() ? nullptr : gq.lnp.dev();
    }
  }
  if(X.att) {
    Dir& D = X.dir[0];
    a.ctxGrad = D.ctxGrad;
    a.dctx = D.dctx.dev();
    a.dwq = D.dwq.dev();
    a.guk = D.guk.ptr;
    a.acc_uk = D.guk.accumulate;
    a.vpart = D.vpart.dev();
  }
  Device& dev = Device::get();
  const size_t need = mtkc_rnn_scan_bwd_workspace(&a);
  const size_t total = (size_t)1 << 30;
  if(need == 0 || need > total / 2)
    throw ContractError("rnn scan: persistent backward not applicable (workspace " +
                        std::to_string(need) + " B)");
  float* base = dev.scratch(total);
  a.workspace = base + (total / 2) / sizeof(float);
  a.workspace_bytes = total / 2;
  MTKC(mtkc_rnn_scan_backward(&a, dev.stream()));
}

void backwardBegin(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X, Dir& D,
                   const float* ctxGrad, bool inter = false) {
  const int64_t b = X.b, T = X.T, d = X.d, K = (int64_t)D.blocks.size();
  const int64_t TB = T * b;
  D.G.assign((size_t)K, Dir::Grads());
  D.inter = inter;
  if(inter) {  // persistent kernel layout (mtkc_rnn_scan_backward)
    D.dGall = g.allocTensor(Shape({K * TB, 3 * d}));
    for(int64_t k = 0; k < K; ++k) {
      Dir::Grads& q = D.G[(size_t)k];
      const bool hasX = D.blocks[(size_t)k].in > 0;
      q.dac = g.allocTensor(Shape({TB, d}));
      if(hasX)
        q.dGx = g.allocTensor(Shape({TB, 3 * d}));
      if(X.ln)
        q.lnp = g.allocTensor(Shape({TB, 6 * d}));
    }
    D.ctxGrad = ctxGrad;
    if(X.att) {
      const AttSlots& A = X.A;
      D.dctx = g.allocTensor(Shape({TB, A.kd}));
      D.dwq = g.allocTensor(Shape({TB, A.a}));
      D.vpart = g.allocTensor(Shape({A.lnG >= 0 ? 3 : 1, TB, A.a}));
      D.guk = g.gradDst(n.inputs[(size_t)A.uk]);
      D.gkeys = g.gradDst(n.inputs[(size_t)A.keys]);
    }
    return;
  }
  for(int64_t k = 0; k < K; ++k) {
    const BlockSlots& Bk = D.blocks[(size_t)k];
    const bool hasX = Bk.in > 0;
    Dir::Grads& q = D.G[(size_t)k];
    q.dpz = g.allocTensor(Shape({TB, d}));
    q.dpr = g.allocTensor(Shape({TB, d}));
    q.duh = g.allocTensor(Shape({TB, d}));
    q.dac = g.allocTensor(Shape({TB, d}));
    q.dax = (hasX && X.ln) ? g.allocTensor(Shape({TB, d})) : q.dac;
    if(X.ln)
      q.lnp = g.allocTensor(Shape({TB, 6 * d}));
  }
  D.ds.assign((size_t)std::max<int64_t>(K - 1, 0), Tensor());
  for(auto& t : D.ds)
    t = g.allocTensor(Shape({b, d}));
  const AttSlots& A = X.A;
  D.ctxGrad = ctxGrad;
  if(X.att) {
    D.dctx = g.allocTensor(Shape({b, A.kd}));
    D.dwq = g.allocTensor(Shape({TB, A.a}));
    D.vpart = g.allocTensor(Shape({A.lnG >= 0 ? 3 : 1, TB, A.a}));
    D.guk = g.gradDst(n.inputs[(size_t)A.uk]);
    D.gkeys = g.gradDst(n.inputs[(size_t)A.keys]);
  }
}

// reverse-sweep step for i = T-1 .. 0
void backwardStep(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X, Dir& D, const Ctx& c,
                  int64_t i) {
  const int64_t b = X.b, T = X.T, d = X.d, d3 = 3 * d, K = (int64_t)D.blocks.size();
  const int64_t TB = T * b;
  const float* HH = D.HH.devc();
  float* GH = D.GH.dev();
  const float* maskT = X.maskT.empty() ? nullptr : X.maskT.devc();
  const AttSlots& A = X.A;
  const float* ctxGrad = D.ctxGrad;
  auto& G = D.G;
  auto& ds = D.ds;
  Tensor& dctx = D.dctx;
  Tensor& dwq = D.dwq;
  Tensor& vpart = D.vpart;
  ExpressionGraph::GradDst& guk = D.guk;
  ExpressionGraph::GradDst& gkeys = D.gkeys;
  Tensor& attScratch = D.attScratch;
  {
    const int64_t t = D.reverse ? T - 1 - i : i;
    const int64_t hp = hprevSlot(D, t);
    const float* hprev = HH + hp * b * d;
    float* ghprev = GH + hp * b * d;  // pre-filled (output grads / zeros): accumulate
    for(int64_t k = K - 1; k >= 0; --k) {
      const BlockSlots& Bk = D.blocks[(size_t)k];
      Dir::Grads& q = G[(size_t)k];
      const float* go = k == K - 1 ? GH + hSlot(D, t) * b * d : ds[(size_t)k].devc();
      const float* sIn = k == 0 ? hprev : D.sout(k - 1) + t * b * d;
      float* gIn = k == 0 ? ghprev : ds[(size_t)k - 1].dev();
      const int accIn = k == 0 ? 1 : 0;
      const float* xw = nullptr;
      if(k == 0 && Bk.in > 0)
        xw = D.xw1.devc() + t * b * d3;
      if(k == 1 && X.att)
        xw = D.xw2.devc() + t * b * d3;
      mtkc_gru_args a{};
      a.b = b;
      a.d = d;
      a.h = sIn;
      a.hu = D.hu[(size_t)k].devc() + t * b * d3;
      a.xw = xw;
      a.cache = D.cache[(size_t)k].dev() + t * b * d3;
      if(X.ln) {
        a.lnGz = g.valPtr(n.inputs[(size_t)Bk.ln[0]]);
        a.lnGr = g.valPtr(n.inputs[(size_t)Bk.ln[2]]);
        if(xw)
          a.lnGx = g.valPtr(n.inputs[(size_t)Bk.ln[4]]);
        a.lnc = D.lnc[(size_t)k].dev() + t * b * d3;
        a.lnrs = D.lnrs[(size_t)k].dev() + t * b * 3;
        a.lnparts = q.lnp.dev() + t * b * 6 * d;
      }
      a.go = go;
      a.gh = gIn;
      a.accumulate_h = accIn;
      a.dpz = q.dpz.dev() + t * b * d;
      a.dpr = q.dpr.dev() + t * b * d;
      a.duh = q.duh.dev() + t * b * d;
      a.dac = q.dac.dev() + t * b * d;
      a.dax = q.dax.dev() + t * b * d;
      if(k == K - 1 && maskT) {
        a.blend_mask = maskT + t * b;
        a.blend_prev = hprev;
        a.gprev = ghprev;
        a.accumulate_prev = 1;
      }
      MTKC(mtkc_gru_backward(&a, c.st));
      {  // gIn += dz Uz^T + dr Ur^T + duh Uh^T (graph.cpp:772, 802)
        const float* Ag[3] = {a.dpz, a.dpr, a.duh};
        const float* Bu[3] = {g.valPtr(n.inputs[(size_t)Bk.U[0]]),
                              g.valPtr(n.inputs[(size_t)Bk.U[1]]),
                              g.valPtr(n.inputs[(size_t)Bk.U[2]])};
        float* C[1] = {gIn};
        const float beta[1] = {1.f};
        gemm3(c, true, b, d, d, Ag, d, false, Bu, d, true, C, d, beta);
      }
      if(k == 1 && X.att) {
        // d(context of step t) = readout's gradient + [dz|dr|dx] W2^T
        float* gc = dctx.dev();
        if(ctxGrad)
          MTKC(mtkc_memcpy_d2d(gc, ctxGrad + t * b * A.kd, (size_t)(b * A.kd) * sizeof(float),
                               c.st));
        const float* Ag[3] = {a.dpz, a.dpr, a.dax};
        const float* Bw[3] = {g.valPtr(n.inputs[(size_t)Bk.W[0]]),
                              g.valPtr(n.inputs[(size_t)Bk.W[1]]),
                              g.valPtr(n.inputs[(size_t)Bk.W[2]])};
        float* C[1] = {gc};
        const float beta[1] = {ctxGrad ? 1.f : 0.f};
        gemm3(c, true, b, A.kd, d, Ag, d, false, Bw, d, true, C, A.kd, beta);
        mtkc_bahdanau_args p{};
        p.b = b;
        p.s = A.S;
        p.a = A.a;
        p.kd = A.kd;
        p.wq = D.wq.devc() + t * b * A.a;
        p.uk = g.valPtr(n.inputs[(size_t)A.uk]);
        p.v = g.valPtr(n.inputs[(size_t)A.v]);
        p.keys = g.valPtr(n.inputs[(size_t)A.keys]);
        p.t = D.attT.dev() + t * b * A.S * A.a;
        p.w = D.attW.dev() + t * b * A.S;
        p.gctx = gc;
        p.gkeys = gkeys.ptr;
        p.acc_keys = (gkeys.accumulate || i < T - 1) ? 1 : 0;
        p.gwq = dwq.dev() + t * b * A.a;
        p.acc_wq = 0;
        p.guk = guk.ptr;
        p.acc_uk = (guk.accumulate || i < T - 1) ? 1 : 0;
        p.gv_part = vpart.dev() + t * b * A.a;
        if(A.lnG >= 0) {
          p.lnG = g.valPtr(n.inputs[(size_t)A.lnG]);
          p.lnB = g.valPtr(n.inputs[(size_t)A.lnB]);
          p.lnxh = D.attLnx.dev() + t * b * A.S * A.a;
          p.lnrs = D.attLnrs.dev() + t * b * A.S;
          p.glnG_part = vpart.dev() + TB * A.a + t * b * A.a;
          p.glnB_part = vpart.dev() + 2 * TB * A.a + t * b * A.a;
        }
        p.scratch = attScratch.dev();
        MTKC(mtkc_bahdanau_backward(&p, c.st));
        // block 1's state also fed the query projection: ds1 += dwq W^T
        gemm1(c, b, d, A.a, p.gwq, A.a, false, g.valPtr(n.inputs[(size_t)A.W]), A.a, true,
              ds[0].dev(), d, 1.f);
      }
    }
  }
}

// weight / bias / layer-norm gradients: one product or sum over b*T rows
void backwardEnd(ExpressionGraph& g, ExpressionGraph::Node& n, ScanAux& X, Dir& D, const Ctx& c,
                 float* dXt, int accX) {
  const int64_t b = X.b, T = X.T, d = X.d, K = (int64_t)D.blocks.size();
  const int64_t TB = T * b;
  const float* HH = D.HH.devc();
  const AttSlots& A = X.A;
  for(int64_t k = 0; k < K; ++k) {
    const BlockSlots& Bk = D.blocks[(size_t)k];
    Dir::Grads& q = D.G[(size_t)k];
    const float* sIn = k == 0 ? HH + (D.reverse ? b * d : 0) : D.sout(k - 1);
    const bool inter = D.inter;
    const int64_t ld = inter ? 3 * d : d;  // row stride of the gate gradients
    const float* dGk = inter ? D.dGall.devc() + k * TB * 3 * d : nullptr;
    const float* dp[3] = {inter ? dGk : q.dpz.devc(), inter ? dGk + d : q.dpr.devc(),
                          inter ? dGk + 2 * d : q.duh.devc()};
    {  // dU += S_in^T [dz|dr|duh]  (graph.cpp:773, 803)
      const float* As[3] = {sIn, sIn, sIn};
      float* C[3];
      float beta[3];
      for(int j = 0; j < 3; ++j) {
        auto dst = g.gradDst(n.inputs[(size_t)Bk.U[j]]);
        C[j] = dst.ptr;
        beta[j] = dst.accumulate ? 1.f : 0.f;
      }
      gemm3(c, false, d, d, TB, As, d, true, dp, ld, false, C, d, beta);
    }
    // biases (graph.cpp:771, 801) and the per-gate LN gains/biases: one
    // launch of column sums straight into the gradient slots (bz, br from
    // the dpz | dpr columns, bh from dac; LN from the lnp partials)
    mtkc_colsum_job jobs[MTKC_COLSUM_MAX_JOBS];
    int nj = 0;
    auto job = [&](const float* in, int64_t ldIn, int64_t cols) -> mtkc_colsum_job& {
      mtkc_colsum_job& J = jobs[nj++];
      J = mtkc_colsum_job{};
      J.in = in;
      J.ld = ldIn;
      J.cols = cols;
      J.seg = d;
      J.nseg = (int)(cols / d);
      return J;
    };
    auto slot = [&](mtkc_colsum_job& J, int s, int paramSlot) {
      auto dst = g.gradDst(n.inputs[(size_t)paramSlot]);
      J.out[s] = dst.ptr;
      J.acc[s] = dst.accumulate;
    };
    if(!inter) {
      slot(job(q.dpz.devc(), d, d), 0, Bk.b[0]);
      slot(job(q.dpr.devc(), d, d), 0, Bk.b[1]);
    } else {
      mtkc_colsum_job& J = job(dGk, 3 * d, 2 * d);  // dpz | dpr columns of [dpz|dpr|duh]
      slot(J, 0, Bk.b[0]);
      slot(J, 1, Bk.b[1]);
    }
    slot(job(q.dac.devc(), d, d), 0, Bk.b[2]);
    if(X.ln) {  // per-gate LN gain/bias partials [TB x 6d]
      const int nln = Bk.in > 0 ? 6 : 4;
      mtkc_colsum_job& J = job(q.lnp.devc(), 6 * d, (int64_t)nln * d);
      for(int j = 0; j < nln; ++j)
        slot(J, j, Bk.ln[j]);
    }
    MTKC(mtkc_colsum_multi(jobs, nj, TB, c.cs, c.csBytes, c.st));
    const float* dGxk = inter && !q.dGx.empty() ? q.dGx.devc() : nullptr;
    const float* dx[3] = {inter ? dGxk : q.dpz.devc(), inter ? dGxk + d : q.dpr.devc(),
                          inter ? dGxk + 2 * d : q.dax.devc()};
    const float* xin = nullptr;
    int64_t inDim = 0;
    if(k == 0 && Bk.in > 0) {
      xin = X.xt.devc();
      inDim = X.e;
    } else if(k == 1 && X.att) {
      xin = D.ctx.devc();
      inDim = A.kd;
    }
    if(xin) {  // dW += X^T [dz|dr|dx]
      const float* Ax[3] = {xin, xin, xin};
      float* C[3];
      float beta[3];
      for(int j = 0; j < 3; ++j) {
        auto dst = g.gradDst(n.inputs[(size_t)Bk.W[j]]);
        C[j] = dst.ptr;
        beta[j] = dst.accumulate ? 1.f : 0.f;
      }
      gemm3(c, false, inDim, d, TB, Ax, inDim, true, dx, ld, false, C, d, beta);
      if(k == 0 && dXt) {  // dX (+)= sum_k [dz|dr|dx]_k W_k^T
        const float* Bw[3] = {g.valPtr(n.inputs[(size_t)Bk.W[0]]),
                              g.valPtr(n.inputs[(size_t)Bk.W[1]]),
                              g.valPtr(n.inputs[(size_t)Bk.W[2]])};
        float* C1[1] = {dXt};
        const float b1[1] = {accX ? 1.f : 0.f};
        gemm3(c, true, TB, X.e, d, dx, ld, false, Bw, d, true, C1, X.e, b1);
      }
    }
  }
  if(X.att) {
    {  // attention query projection: dW += S1^T dwq over b*T rows
      auto dst = g.gradDst(n.inputs[(size_t)A.W]);
      gemm1(c, d, A.a, TB, D.sout(0), d, true, D.dwq.devc(), A.a, false, dst.ptr, A.a,
            dst.accumulate ? 1.f : 0.f);
    }
    const int np = A.lnG >= 0 ? 3 : 1;
    const int slots[3] = {A.v, A.lnG, A.lnB};
    for(int j = 0; j < np; ++j)
      colsum(c, g.gradDst(n.inputs[(size_t)slots[j]]), D.vpart.devc() + j * TB * A.a, TB, A.a);
    if(D.inter) {  // keys: d(keys)[r] (+)= sum_t w_t[r]^T dctx_t[r]
      MTKC(mtkc_rnn_key_grad(D.gkeys.ptr, D.attW.devc(), D.dctx.devc(), b, T, A.S, A.kd,
                             D.gkeys.accumulate, c.st));
    }
    if(false) {  // (batched-GEMM form of the same sum)
      mtkc_gemm_args q{};
      q.M = A.S;
      q.N = A.kd;
      q.K = T;
      q.batch = b;
      q.A = D.attW.devc();
      q.lda = b * A.S;
      q.strideA = A.S;
      q.transA = 1;
      q.B = D.dctx.devc();
      q.ldb = b * A.kd;
      q.strideB = A.kd;
      q.C = D.gkeys.ptr;
      q.ldc = A.kd;
      q.strideC = A.S * A.kd;
      q.alpha = 1.f;
      q.beta = D.gkeys.accumulate ? 1.f : 0.f;
      q.precision = (int)Device::get().precision();
      q.workspace = c.ws;
      q.workspace_bytes = c.wsBytes;
      MTKC(mtkc_gemm(&q, c.st));
    }
  }
}

}  // namespace

// ------------------------------------------------------------ encoder

NodeRef ExpressionGraph::rnnEncoderScan(NodeRef x, const std::vector<GruParams>& fwd,
                                        const std::vector<GruParams>& bwd, const Tensor& mask,
                                        bool layerNorm) {
  checkRef(x);
  if(x.shape.rank() != 3)
    throw DimensionError("rnnEncoderScan: x must be [b x s x e], got " + x.shape.str());
  if(fwd.empty() || fwd.size() != bwd.size())
    throw ContractError("rnnEncoderScan: both directions need the same number of blocks");
  const int64_t b = x.shape[0], T = x.shape[1], e = x.shape[2];
  const int64_t d = fwd[0].Uz.shape[0];
  auto X = std::make_shared<ScanAux>();
  X->b = b;
  X->T = T;
  X->d = d;
  X->e = e;
  X->ln = layerNorm;
  X->ndir = 2;
  Node n;
  n.op = "rnnEncoderScan";
  n.shape = Shape({b, T, 2 * d});
  n.inputs = {x.index};
  X->xSlot = 0;
  for(int q = 0; q < 2; ++q) {
    const auto& ps = q == 0 ? fwd : bwd;
    X->dir[q].reverse = q == 1;
    for(size_t k = 0; k < ps.size(); ++k)
      X->dir[q].blocks.push_back(addBlock(n, ps[k], layerNorm, k == 0 ? e : 0));
  }
  if(!mask.empty()) {  // time-major copy of the padding mask (models.cpp:170-172)
    const Real* m = mask.data();
    std::vector<Real> mt((size_t)(T * b));
    for(int64_t r = 0; r < b; ++r)
      for(int64_t t = 0; t < T; ++t)
        mt[(size_t)(t * b + r)] = m[r * T + t];
    X->maskT = Tensor(Shape({T, b}), std::move(mt));
  }
  n.aux = X;
  n.fwd = [X](ExpressionGraph& g, Node& n) {
    const int64_t b = X->b, T = X->T, d = X->d, e = X->e;
    Device& dev = Device::get();
    X->xt = g.allocTensor(Shape({T * b, e}));
    {
      const int64_t sd[4] = {1, b, T, e};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(X->xt.dev(), g.valPtr(n.inputs[0]), sd, perm, 0, dev.stream()));
    }
    if(!X->maskT.empty())
      X->maskT.devc();  // uploaded on the compute stream before the fork
    if(persistEnabled()) {  // both directions in one cooperative launch
      const Ctx c0 = ctxFor(0);
      forwardBegin(g, n, *X, X->dir[0], c0, nullptr);
      forwardBegin(g, n, *X, X->dir[1], c0, nullptr);
      if(!forwardPersistent(g, n, *X))
        for(int64_t i = 0; i < T; ++i) {
          forwardStep(g, n, *X, X->dir[0], c0, i);
          forwardStep(g, n, *X, X->dir[1], c0, i);
        }
    } else {
      dev.forkSide();
      const Ctx c0 = ctxFor(0), c1 = ctxFor(1);
      forwardBegin(g, n, *X, X->dir[0], c0, nullptr);
      forwardBegin(g, n, *X, X->dir[1], c1, nullptr);
      for(int64_t i = 0; i < T; ++i) {  // the two directions' steps interleaved
        forwardStep(g, n, *X, X->dir[0], c0, i);
        forwardStep(g, n, *X, X->dir[1], c1, i);
      }
      dev.joinSide();
    }
    // context [b x s x 2d] = [H_fwd | H_bwd] per position
    Tensor tmp = g.allocTensor(Shape({b, T, d}));
    for(int q = 0; q < 2; ++q) {
      const Dir& D = X->dir[q];
      const float* H = D.HH.devc() + (D.reverse ? 0 : b * d);
      const int64_t sd[4] = {1, T, b, d};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(tmp.dev(), H, sd, perm, 0, dev.stream()));
      MTKC(mtkc_copy_blocks(n.value.dev(), 2 * d, q * d, tmp.devc(), d, 0, b * T, d, 0,
                            dev.stream()));
    }
  };
  n.bwd = [X](ExpressionGraph& g, Node& n) {
    const int64_t b = X->b, T = X->T, d = X->d, e = X->e;
    Device& dev = Device::get();
    const float* go = g.gradSrc(n);  // [b x s x 2d]
    Tensor tmp = g.allocTensor(Shape({b, T, d}));
    for(int q = 0; q < 2; ++q) {  // unpack into the time-major state gradients
      Dir& D = X->dir[q];
      D.GH = g.allocTensor(Shape({(T + 1) * b, d}));
      float* GH = D.GH.dev();
      MTKC(mtkc_copy_blocks(tmp.dev(), d, 0, go, 2 * d, q * d, b * T, d, 0, dev.stream()));
      const int64_t sd[4] = {1, b, T, d};
      const int perm[4] = {0, 2, 1, 3};
      float* Hg = GH + (D.reverse ? 0 : b * d);
      MTKC(mtkc_transpose(Hg, tmp.devc(), sd, perm, 0, dev.stream()));
      const int64_t h0slot = D.reverse ? T : 0;
      MTKC(mtkc_memset(GH + h0slot * b * d, 0, (size_t)(b * d) * sizeof(float), dev.stream()));
    }
    const bool needX = g.node(g.resolve(n.inputs[0])).needsGrad;
    Tensor dxt[2];
    if(needX)
      for(auto& t : dxt)
        t = g.allocTensor(Shape({T * b, e}));
    // parameter gradient destinations are resolved before the fork (gradDst
    // is host bookkeeping; a lazily-zero buffer is only written, never read)
    const Ctx c0 = ctxFor(0), c1 = ctxFor(1);
    if(persistBwdEligible(g, n, *X)) {  // both directions in one cooperative launch
      backwardBegin(g, n, *X, X->dir[0], nullptr, true);
      backwardBegin(g, n, *X, X->dir[1], nullptr, true);
      backwardPersistent(g, n, *X);
    } else {
      backwardBegin(g, n, *X, X->dir[0], nullptr);
      backwardBegin(g, n, *X, X->dir[1], nullptr);
      dev.forkSide();
      for(int64_t i = T - 1; i >= 0; --i) {
        backwardStep(g, n, *X, X->dir[0], c0, i);
        backwardStep(g, n, *X, X->dir[1], c1, i);
      }
      dev.joinSide();
    }
    // the batched weight / bias sums run on the compute stream (each fills
    // the GPU on its own; the column sums' last-CTA tickets are global)
    backwardEnd(g, n, *X, X->dir[0], c0, needX ? dxt[0].dev() : nullptr, 0);
    backwardEnd(g, n, *X, X->dir[1], c0, needX ? dxt[1].dev() : nullptr, 0);
    if(needX) {  // dx [b x s x e] (+)= transpose(dX_fwd + dX_bwd)
      MTKC(mtkc_axpy(dxt[0].dev(), dxt[1].devc(), 1.f, T * b * e, dev.stream()));
      auto dst = g.gradDst(n.inputs[0]);
      const int64_t sd[4] = {1, T, b, e};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(dst.ptr, dxt[0].devc(), sd, perm, dst.accumulate, dev.stream()));
    }
  };
  return addNode(std::move(n));
}

// ------------------------------------------------------------ decoder

ExpressionGraph::RnnScanOut ExpressionGraph::rnnDecoderScan(
    NodeRef x, NodeRef h0, const std::vector<GruParams>& blocks, const RnnScanAttention* att,
    const Tensor& tokenMask, bool layerNorm) {
  checkRef(x);
  checkRef(h0);
  if(x.shape.rank() != 3 || h0.shape.rank() != 2)
    throw DimensionError("rnnDecoderScan: x [b x t x e], h0 [b x d]");
  if(blocks.size() < 1 || (att && blocks.size() < 2))
    throw ContractError("rnnDecoderScan: attention needs at least two blocks");
  const int64_t b = x.shape[0], T = x.shape[1], e = x.shape[2], d = h0.shape[1];
  if(h0.shape[0] != b)
    throw DimensionError("rnnDecoderScan: state rows " + h0.shape.str() + " vs " + x.shape.str());
  auto X = std::make_shared<ScanAux>();
  X->b = b;
  X->T = T;
  X->d = d;
  X->e = e;
  X->ln = layerNorm;
  X->ndir = 1;
  Node n;
  n.op = "rnnDecoderScan";
  n.shape = Shape({b, T, d});
  n.inputs = {x.index, h0.index};
  X->xSlot = 0;
  X->h0Slot = 1;
  X->att = att != nullptr;
  for(size_t k = 0; k < blocks.size(); ++k) {
    int64_t in = k == 0 ? e : (k == 1 && att ? att->keys.shape[2] : 0);
    X->dir[0].blocks.push_back(addBlock(n, blocks[k], layerNorm, in));
  }
  if(att) {
    AttSlots& A = X->A;
    auto push = [&](const NodeRef& r) {
      checkRef(r);
      n.inputs.push_back(r.index);
      return (int)n.inputs.size() - 1;
    };
    A.W = push(att->W);
    A.v = push(att->v);
    if(att->lnG.valid()) {
      A.lnG = push(att->lnG);
      A.lnB = push(att->lnB);
    }
    A.keys = push(att->keys);
    A.uk = push(att->uk);
    A.S = att->keys.shape[1];
    A.kd = att->keys.shape[2];
    A.a = att->W.shape[1];
    if(att->uk.shape != Shape({b, A.S, A.a}) || att->keys.shape[0] != b)
      throw DimensionError("rnnDecoderScan: attention shapes " + att->keys.shape.str() + " " +
                           att->uk.shape.str());
    if(!att->mask.empty()) {
      const Real* m = att->mask.data();
      for(int64_t r = 0; r < b; ++r) {  // tensor.cpp:424-425
        bool any = false;
        for(int64_t j = 0; j < A.S && !any; ++j)
          any = m[r * A.S + j] != 0;
        if(!any)
          throw NumericError("softmax over a fully-masked row");
      }
      A.mask = att->mask;
      A.hasMask = true;
    }
  }
  if(!tokenMask.empty()) {
    const Real* m = tokenMask.data();
    std::vector<Real> mt((size_t)(T * b));
    for(int64_t r = 0; r < b; ++r)
      for(int64_t t = 0; t < T; ++t)
        mt[(size_t)(t * b + r)] = m[r * T + t];
    X->maskT = Tensor(Shape({T, b}), std::move(mt));
  }
  n.aux = X;
  n.fwd = [X](ExpressionGraph& g, Node& n) {
    const int64_t b = X->b, T = X->T, d = X->d, e = X->e;
    Device& dev = Device::get();
    X->xt = g.allocTensor(Shape({T * b, e}));
    {
      const int64_t sd[4] = {1, b, T, e};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(X->xt.dev(), g.valPtr(n.inputs[0]), sd, perm, 0, dev.stream()));
    }
    Dir& D = X->dir[0];
    const Ctx c0 = ctxFor(0);
    forwardBegin(g, n, *X, D, c0, g.valPtr(n.inputs[1]));
    if(!forwardPersistent(g, n, *X))
      for(int64_t i = 0; i < T; ++i)
        forwardStep(g, n, *X, D, c0, i);
    {  // states [b x t x d]
      const int64_t sd[4] = {1, T, b, d};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(n.value.dev(), D.HH.devc() + b * d, sd, perm, 0, dev.stream()));
    }
    if(X->att && X->ctxView >= 0) {  // contexts [b x t x kd]
      Node& cv = g.node(X->ctxView);
      cv.value = g.allocTensor(cv.shape);
      const int64_t sd[4] = {1, T, b, X->A.kd};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(cv.value.dev(), D.ctx.devc(), sd, perm, 0, dev.stream()));
    }
    if(X->lastView >= 0) {  // final state (a copy of the last slot)
      Node& lv = g.node(X->lastView);
      lv.value = g.allocTensor(lv.shape);
      MTKC(mtkc_memcpy_d2d(lv.value.dev(), D.HH.devc() + T * b * d,
                           (size_t)(b * d) * sizeof(float), dev.stream()));
    }
  };
  n.bwd = [X](ExpressionGraph& g, Node& n) {
    const int64_t b = X->b, T = X->T, d = X->d, e = X->e;
    Device& dev = Device::get();
    Dir& D = X->dir[0];
    D.GH = g.allocTensor(Shape({(T + 1) * b, d}));
    float* GH = D.GH.dev();
    MTKC(mtkc_memset(GH, 0, (size_t)(b * d) * sizeof(float), dev.stream()));
    {
      const float* go = g.gradSrc(n);  // [b x t x d] -> slots 1..T
      const int64_t sd[4] = {1, b, T, d};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(GH + b * d, go, sd, perm, 0, dev.stream()));
    }
    if(X->lastView >= 0) {
      Node& lv = g.node(X->lastView);
      if(lv.gradLive)
        MTKC(mtkc_axpy(GH + T * b * d, lv.grad.devc(), 1.f, b * d, dev.stream()));
    }
    Tensor ctxg;
    if(X->att && X->ctxView >= 0) {
      Node& cv = g.node(X->ctxView);
      if(cv.gradLive) {
        ctxg = g.allocTensor(Shape({T * b, X->A.kd}));
        const int64_t sd[4] = {1, b, T, X->A.kd};
        const int perm[4] = {0, 2, 1, 3};
        MTKC(mtkc_transpose(ctxg.dev(), cv.grad.devc(), sd, perm, 0, dev.stream()));
      }
    }
    const bool needX = g.node(g.resolve(n.inputs[0])).needsGrad;
    Tensor dxt = needX ? g.allocTensor(Shape({T * b, e})) : Tensor();
    const Ctx c0 = ctxFor(0);
    if(persistBwdEligible(g, n, *X)) {
      backwardBegin(g, n, *X, D, ctxg.empty() ? nullptr : ctxg.devc(), true);
      backwardPersistent(g, n, *X);
    } else {
      backwardBegin(g, n, *X, D, ctxg.empty() ? nullptr : ctxg.devc());
      for(int64_t i = T - 1; i >= 0; --i)
        backwardStep(g, n, *X, D, c0, i);
    }
    backwardEnd(g, n, *X, D, c0, needX ? dxt.dev() : nullptr, 0);
    if(needX) {
      auto dst = g.gradDst(n.inputs[0]);
      const int64_t sd[4] = {1, T, b, e};
      const int perm[4] = {0, 2, 1, 3};
      MTKC(mtkc_transpose(dst.ptr, dxt.devc(), sd, perm, dst.accumulate, dev.stream()));
    }
    if(g.node(g.resolve(n.inputs[1])).needsGrad) {  // initial state (decoder initW/initB)
      auto dst = g.gradDst(n.inputs[1]);
      if(dst.accumulate)
        MTKC(mtkc_axpy(dst.ptr, GH, 1.f, b * d, dev.stream()));
      else
        MTKC(mtkc_memcpy_d2d(dst.ptr, GH, (size_t)(b * d) * sizeof(float), dev.stream()));
    }
  };
  NodeRef states = addNode(std::move(n));
  RnnScanOut out;
  out.states = states;
  auto view = [&](const char* op, Shape s) {
    Node v;
    v.op = op;
    v.shape = std::move(s);
    v.inputs = {states.index};
    // a gradient arriving here must reach the scan node's backward
    v.bwd = [](ExpressionGraph& g, Node& v) {
      auto d = g.gradDst(v.inputs[0]);
      if(!d.accumulate)
        MTKC(mtkc_memset(d.ptr, 0, (size_t)g.node(v.inputs[0]).shape.size() * sizeof(float),
                         Device::get().stream()));
    };
    return addNode(std::move(v));
  };
  if(att) {
    out.contexts = view("rnnScanContexts", Shape({b, T, X->A.kd}));
    X->ctxView = out.contexts.index;
  }
  out.last = view("rnnScanLast", Shape({b, d}));
  X->lastView = out.last.index;
  return out;
}

}  // namespace mtk
