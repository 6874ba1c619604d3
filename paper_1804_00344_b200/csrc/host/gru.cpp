// Fused GRU block (gruCell, reference graph.cpp:648-813).
//
// Forward: h*[Uz|Ur|Uh] and x*[Wz|Wr|Wx] as tcgen05 GEMMs into [b x 3d]
// buffers, then one pointwise kernel per row (bias, optional per-gate layer
// norm, sigmoid/tanh, state interpolation).  Backward: one pointwise kernel
// producing the gate pre-activation gradients, then the transposed GEMMs
// for dh, dU, dx, dW, column sums for the biases and layer-norm parameters.
#include "mtk/device.h"
#include "mtk/graph.h"

namespace mtk {

namespace {

void* stream() { return Device::get().stream(); }

void gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, bool tA, const float* B,
          int64_t ldb, bool tB, float* C, int64_t ldc, float beta) {
  Device& d = Device::get();
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
  g.precision = (int)d.precision();
  g.workspace = d.scratch(64 << 20);
  g.workspace_bytes = d.scratchBytes();
  MTKC(mtkc_gemm(&g, d.stream()));
}

// n <= 3 products of one shape in one launch (mtkc_gemm_group): independent
// outputs C[k] (kconcat = false) or C[0] += sum_k A[k] op(B[k]) (kconcat)
void gemmGroup(int n, bool kconcat, int64_t M, int64_t N, int64_t K, const float* const* A,
               int64_t lda, bool tA, const float* const* B, int64_t ldb, bool tB,
               float* const* C, int64_t ldc, const float* beta) {
  Device& d = Device::get();
  mtkc_gemm_args g[3];
  for(int k = 0; k < n; ++k) {
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
    g[k].precision = (int)d.precision();
    g[k].workspace = d.scratch(64 << 20);
    g[k].workspace_bytes = d.scratchBytes();
  }
  MTKC(mtkc_gemm_group(g, n, kconcat ? 1 : 0, d.stream()));
}

void colsumInto(ExpressionGraph::GradDst dst, const float* in, int64_t rows, int64_t cols) {
  Device& dev = Device::get();
  size_t ws = (size_t)((rows + 63) / 64) * (size_t)cols * sizeof(float) * 2;
  float* w = dev.scratch(ws);
  MTKC(mtkc_colsum(dst.ptr, in, rows, cols, dst.accumulate, w, dev.scratchBytes(), dev.stream()));
}

struct GruAux {
  Tensor hu, xw, cache, lnc, lnrs;
};

}  // namespace

NodeRef ExpressionGraph::gruCell(NodeRef state, NodeRef input, const GruParams& p,
                                 bool layerNorm) {
  checkRef(state);
  bool hasInput = input.valid();
  if(hasInput)
    checkRef(input);
  if(state.shape.rank() != 2)
    throw DimensionError("gru state must be rank 2 [batch x d], got " + state.shape.str());
  int64_t b = state.shape[0], d = state.shape.back();
  if(hasInput && input.shape[0] != b)
    throw DimensionError("gru input batch mismatch: " + input.shape.str() + " vs " +
                         state.shape.str());
  int64_t e = hasInput ? input.shape.back() : 0;
  Node n;
  n.op = "gruCell";
  n.shape = state.shape;
  // input slots follow the reference (graph.cpp:665-687)
  n.inputs = {state.index, p.Uz.index, p.bz.index, p.Ur.index, p.br.index, p.Uh.index,
              p.bh.index};
  int xSlot = -1, wSlot = -1, lnSlot = -1;
  if(hasInput) {
    xSlot = (int)n.inputs.size();
    n.inputs.push_back(input.index);
    wSlot = (int)n.inputs.size();
    n.inputs.push_back(p.Wz.index);
    n.inputs.push_back(p.Wr.index);
    n.inputs.push_back(p.Wx.index);
  }
  if(layerNorm) {
    lnSlot = (int)n.inputs.size();
    n.inputs.push_back(p.lnGz.index);
    n.inputs.push_back(p.lnBz.index);
    n.inputs.push_back(p.lnGr.index);
    n.inputs.push_back(p.lnBr.index);
    if(hasInput) {
      n.inputs.push_back(p.lnGx.index);
      n.inputs.push_back(p.lnBx.index);
    }
  }
  auto aux = std::make_shared<GruAux>();
  n.aux = aux;

  n.fwd = [=](ExpressionGraph& g, Node& n) {
    aux->hu = g.allocTensor(Shape({b, 3 * d}));
    aux->cache = g.allocTensor(Shape({b, 3 * d}));
    const float* h = g.valPtr(n.inputs[0]);
    float* hu = aux->hu.dev();
    {  // h [Uz|Ur|Uh]: one grouped launch
      const float* A[3] = {h, h, h};
      const float* B[3] = {g.valPtr(n.inputs[1]), g.valPtr(n.inputs[3]), g.valPtr(n.inputs[5])};
      float* C[3] = {hu, hu + d, hu + 2 * d};
      const float beta[3] = {0.f, 0.f, 0.f};
      gemmGroup(3, false, b, d, d, A, d, false, B, d, false, C, 3 * d, beta);
    }
    mtkc_gru_args a{};
    a.b = b;
    a.d = d;
    a.h = h;
    a.hu = hu;
    if(hasInput) {
      aux->xw = g.allocTensor(Shape({b, 3 * d}));
      float* xw = aux->xw.dev();
      const float* x = g.valPtr(n.inputs[xSlot]);
      const float* A[3] = {x, x, x};
      const float* B[3] = {g.valPtr(n.inputs[wSlot]), g.valPtr(n.inputs[wSlot + 1]),
                           g.valPtr(n.inputs[wSlot + 2])};
      float* C[3] = {xw, xw + d, xw + 2 * d};
      const float beta[3] = {0.f, 0.f, 0.f};
      gemmGroup(3, false, b, d, e, A, e, false, B, d, false, C, 3 * d, beta);
      a.xw = xw;
    }
    a.bz = g.valPtr(n.inputs[2]);
    a.br = g.valPtr(n.inputs[4]);
    a.bh = g.valPtr(n.inputs[6]);
    if(layerNorm) {
      aux->lnc = g.allocTensor(Shape({b, 3 * d}));
      aux->lnrs = g.allocTensor(Shape({b, 3}));
      a.lnGz = g.valPtr(n.inputs[lnSlot]);
      a.lnBz = g.valPtr(n.inputs[lnSlot + 1]);
      a.lnGr = g.valPtr(n.inputs[lnSlot + 2]);
      a.lnBr = g.valPtr(n.inputs[lnSlot + 3]);
      if(hasInput) {
        a.lnGx = g.valPtr(n.inputs[lnSlot + 4]);
        a.lnBx = g.valPtr(n.inputs[lnSlot + 5]);
      }
      a.lnc = aux->lnc.dev();
      a.lnrs = aux->lnrs.dev();
    }
    a.eps = 1e-9f;  // graph.cpp:690
    a.hout = n.value.dev();
    a.cache = aux->cache.dev();
    MTKC(mtkc_gru_forward(&a, stream()));
  };

  n.bwd = [=](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    Tensor dpz = g.allocTensor(Shape({b, d})), dpr = g.allocTensor(Shape({b, d}));
    Tensor duh = g.allocTensor(Shape({b, d})), dac = g.allocTensor(Shape({b, d}));
    Tensor dax = (hasInput && layerNorm) ? g.allocTensor(Shape({b, d})) : dac;
    Tensor lnparts;
    mtkc_gru_args a{};
    a.b = b;
    a.d = d;
    a.h = g.valPtr(n.inputs[0]);
    a.hu = aux->hu.devc();
    a.xw = hasInput ? aux->xw.devc() : nullptr;
    a.cache = aux->cache.dev();
    if(layerNorm) {
      lnparts = g.allocTensor(Shape({b, 6 * d}));
      a.lnGz = g.valPtr(n.inputs[lnSlot]);
      a.lnGr = g.valPtr(n.inputs[lnSlot + 2]);
      if(hasInput)
        a.lnGx = g.valPtr(n.inputs[lnSlot + 4]);
      a.lnc = aux->lnc.dev();
      a.lnrs = aux->lnrs.dev();
      a.lnparts = lnparts.dev();
    }
    a.go = go;
    auto gh = g.gradDst(n.inputs[0]);
    a.gh = gh.ptr;
    a.accumulate_h = gh.accumulate;
    a.dpz = dpz.dev();
    a.dpr = dpr.dev();
    a.duh = duh.dev();
    a.dac = dac.dev();
    a.dax = dax.dev();
    MTKC(mtkc_gru_backward(&a, stream()));
    const float* h = a.h;
    // dh += dpz Uz^T + dpr Ur^T + duh Uh^T   (graph.cpp:772, 802)
    const float* gsrc[3] = {a.dpz, a.dpr, a.duh};
    const float* Us[3] = {g.valPtr(n.inputs[1]), g.valPtr(n.inputs[3]), g.valPtr(n.inputs[5])};
    {  // one K-concatenated launch; FP32 mode falls back to z, r, h in order
      float* C[1] = {gh.ptr};
      const float beta[1] = {1.f};
      gemmGroup(3, true, b, d, d, gsrc, d, false, Us, d, true, C, d, beta);
    }
    // dU += h^T dpre   (graph.cpp:773, 803)
    {
      const float* hs[3] = {h, h, h};
      float* C[3];
      float beta[3];
      for(int k = 0; k < 3; ++k) {
        auto dU = g.gradDst(n.inputs[1 + 2 * k]);
        C[k] = dU.ptr;
        beta[k] = dU.accumulate ? 1.f : 0.f;
      }
      if(beta[0] == beta[1] && beta[1] == beta[2]) {
        gemmGroup(3, false, d, d, b, hs, d, true, gsrc, d, false, C, d, beta);
      } else {
        for(int k = 0; k < 3; ++k)
          gemm(d, d, b, h, d, true, gsrc[k], d, false, C[k], d, beta[k]);
      }
    }
    // biases (graph.cpp:771, 801)
    {  // the three gate biases in one launch
      auto gz = g.gradDst(n.inputs[2]), gr = g.gradDst(n.inputs[4]), gb = g.gradDst(n.inputs[6]);
      float* outs[3] = {gz.ptr, gr.ptr, gb.ptr};
      const float* ins[3] = {a.dpz, a.dpr, a.dac};
      const int acc[3] = {gz.accumulate, gr.accumulate, gb.accumulate};
      Device& dev = Device::get();
      float* w = dev.scratch((size_t)3 * ((b + 63) / 64) * (size_t)d * sizeof(float));
      MTKC(mtkc_colsum_group(outs, ins, acc, 3, b, d, w, dev.scratchBytes(), dev.stream()));
    }
    if(hasInput) {
      const float* x = g.valPtr(n.inputs[xSlot]);
      const float* wsrc[3] = {a.dpz, a.dpr, a.dax};
      auto dx = g.gradDst(n.inputs[xSlot]);
      const float* Ws[3] = {g.valPtr(n.inputs[wSlot]), g.valPtr(n.inputs[wSlot + 1]),
                            g.valPtr(n.inputs[wSlot + 2])};
      {
        float* C[1] = {dx.ptr};
        const float beta[1] = {dx.accumulate ? 1.f : 0.f};
        gemmGroup(3, true, b, e, d, wsrc, d, false, Ws, d, true, C, e, beta);
      }
      const float* xs[3] = {x, x, x};
      float* C[3];
      float beta[3];
      for(int k = 0; k < 3; ++k) {
        auto dW = g.gradDst(n.inputs[wSlot + k]);
        C[k] = dW.ptr;
        beta[k] = dW.accumulate ? 1.f : 0.f;
      }
      if(beta[0] == beta[1] && beta[1] == beta[2]) {
        gemmGroup(3, false, e, d, b, xs, e, true, wsrc, d, false, C, d, beta);
      } else {
        for(int k = 0; k < 3; ++k)
          gemm(e, d, b, x, e, true, wsrc[k], d, false, C[k], d, beta[k]);
      }
    }
    if(layerNorm) {  // per-gate LN gain/bias grads: one column sum, then slices
      int nln = hasInput ? 6 : 4;
      Tensor sums = g.allocTensor(Shape({6 * d}));
      colsumInto(ExpressionGraph::GradDst{sums.dev(), 0, nullptr}, lnparts.devc(), b, 6 * d);
      for(int k = 0; k < nln; ++k) {
        auto dst = g.gradDst(n.inputs[lnSlot + k]);
        if(dst.accumulate)
          MTKC(mtkc_axpy(dst.ptr, sums.devc() + k * d, 1.f, d, stream()));
        else
          MTKC(mtkc_memcpy_d2d(dst.ptr, sums.devc() + k * d, (size_t)d * sizeof(float),
                               stream()));
      }
    }
  };
  return addNode(std::move(n));
}

}  // namespace mtk
