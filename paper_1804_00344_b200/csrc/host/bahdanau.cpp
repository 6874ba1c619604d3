// Fused Bahdanau attention node (reference: BahdanauAttention::apply,
// layers.cpp:59-79, built there from add/layerNorm/tanh/dot/softmax nodes).
#include "mtk/device.h"
#include "mtk/graph.h"

namespace mtk {

namespace {
struct BahAux {
  Tensor t, lnxh, lnrs, w, mask;
  bool hasMask = false;
  int weightsNode = -1;
};
void* stream() { return Device::get().stream(); }
}  // namespace

std::pair<NodeRef, NodeRef> ExpressionGraph::bahdanau(NodeRef wq, NodeRef uk, NodeRef v,
                                                      NodeRef keys, const Tensor& mask,
                                                      NodeRef lnG, NodeRef lnB) {
  checkRef(wq);
  checkRef(uk);
  checkRef(v);
  checkRef(keys);
  bool ln = lnG.valid();
  if(ln) {
    checkRef(lnG);
    checkRef(lnB);
  }
  if(wq.shape.rank() != 2 || uk.shape.rank() != 3 || keys.shape.rank() != 3)
    throw DimensionError("bahdanau expects wq [b,a], uk [b,s,a], keys [b,s,k]");
  int64_t b = wq.shape[0], a = wq.shape[1], s = uk.shape[1], kd = keys.shape[2];
  if(uk.shape[0] != b || uk.shape[2] != a || keys.shape[0] != b || keys.shape[1] != s ||
     v.shape.size() != a)
    throw DimensionError("bahdanau shapes disagree: " + wq.shape.str() + " " + uk.shape.str() +
                         " " + keys.shape.str());
  if(!mask.empty()) {
    if(mask.size() != b * s)
      throw DimensionError("bahdanau mask must be [b x s]");
    const Real* m = mask.data();
    for(int64_t r = 0; r < b; ++r) {  // tensor.cpp:424-425
      bool any = false;
      for(int64_t j = 0; j < s && !any; ++j)
        any = m[r * s + j] != 0;
      if(!any)
        throw NumericError("softmax over a fully-masked row");
    }
  }
  auto aux = std::make_shared<BahAux>();
  if(!mask.empty()) {
    aux->mask = mask;  // shared device copy
    aux->hasMask = true;
  }
  Node n;
  n.op = "bahdanau";
  n.shape = Shape({b, kd});
  n.inputs = {wq.index, uk.index, v.index, keys.index};
  if(ln) {
    n.inputs.push_back(lnG.index);
    n.inputs.push_back(lnB.index);
  }
  n.aux = aux;
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    aux->t = g.allocTensor(Shape({b, s, a}));
    aux->w = g.allocTensor(Shape({b, s}));
    mtkc_bahdanau_args p{};
    p.b = b;
    p.s = s;
    p.a = a;
    p.kd = kd;
    p.wq = g.valPtr(n.inputs[0]);
    p.uk = g.valPtr(n.inputs[1]);
    p.v = g.valPtr(n.inputs[2]);
    p.keys = g.valPtr(n.inputs[3]);
    p.mask = aux->hasMask ? aux->mask.devc() : nullptr;
    if(ln) {
      aux->lnxh = g.allocTensor(Shape({b, s, a}));
      aux->lnrs = g.allocTensor(Shape({b, s}));
      p.lnG = g.valPtr(n.inputs[4]);
      p.lnB = g.valPtr(n.inputs[5]);
      p.lnxh = aux->lnxh.dev();
      p.lnrs = aux->lnrs.dev();
    }
    p.eps = 1e-9f;  // graph.h:103 default
    p.t = aux->t.dev();
    p.w = aux->w.dev();
    p.ctx = n.value.dev();
    p.flags = Device::get().flags();
    Tensor scratch = g.allocTensor(Shape({4, b, s}));
    p.scratch = scratch.dev();
    MTKC(mtkc_bahdanau_forward(&p, stream()));
    if(aux->weightsNode >= 0)
      g.node(aux->weightsNode).value = aux->w;
  };
  n.bwd = [=](ExpressionGraph& g, Node& n) {
    mtkc_bahdanau_args p{};
    p.b = b;
    p.s = s;
    p.a = a;
    p.kd = kd;
    p.wq = g.valPtr(n.inputs[0]);
    p.uk = g.valPtr(n.inputs[1]);
    p.v = g.valPtr(n.inputs[2]);
    p.keys = g.valPtr(n.inputs[3]);
    p.t = aux->t.dev();
    p.w = aux->w.dev();
    p.gctx = g.gradSrc(n);
    auto gk = g.gradDst(n.inputs[3]);
    auto gw = g.gradDst(n.inputs[0]);
    auto gu = g.gradDst(n.inputs[1]);
    p.gkeys = gk.ptr;
    p.acc_keys = gk.accumulate;
    p.gwq = gw.ptr;
    p.acc_wq = gw.accumulate;
    p.guk = gu.ptr;
    p.acc_uk = gu.accumulate;
    Tensor parts = g.allocTensor(Shape({ln ? 3 : 1, b, a}));
    p.gv_part = parts.dev();
    if(ln) {
      p.lnG = g.valPtr(n.inputs[4]);
      p.lnB = g.valPtr(n.inputs[5]);
      p.lnxh = aux->lnxh.dev();
      p.lnrs = aux->lnrs.dev();
      p.glnG_part = p.gv_part + b * a;
      p.glnB_part = p.gv_part + 2 * b * a;
    }
    Tensor scratch = g.allocTensor(Shape({4, b, s}));
    p.scratch = scratch.dev();
    MTKC(mtkc_bahdanau_backward(&p, stream()));
    Device& dev = Device::get();
    size_t ws = (size_t)((b + 63) / 64 + 1) * (size_t)a * sizeof(float) * 2;
    float* w = dev.scratch(ws);
    int nparam = ln ? 3 : 1;
    const int pidx[3] = {2, 4, 5};
    for(int k = 0; k < nparam; ++k) {
      auto dst = g.gradDst(n.inputs[(size_t)pidx[k]]);
      MTKC(mtkc_colsum(dst.ptr, p.gv_part + k * b * a, b, a, dst.accumulate, w,
                       dev.scratchBytes(), dev.stream()));
    }
  };
  NodeRef ctx = addNode(std::move(n));
  Node wn;
  wn.op = "attWeights";
  wn.shape = Shape({b, s});
  wn.inputs = {ctx.index};
  NodeRef weights = addNode(std::move(wn));
  aux->weightsNode = weights.index;
  return {ctx, weights};
}

}  // namespace mtk
