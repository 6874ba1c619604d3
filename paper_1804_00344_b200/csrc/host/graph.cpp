// Expression graph over device tensors (reference: src/graph.cpp).  Every
// op's forward/backward closure launches kernels from libmtkcuda.so on the
// device stream; see mtk/graph.h for the B200-specific execution model.
#include "mtk/graph.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "mtk/device.h"

namespace mtk {

// ----------------------------------------------------------------- refs

Tensor& NodeRef::val() const {
  if(!graph)
    throw ContractError("empty node reference");
  return graph->nodeValue(index, gen);
}

Tensor& NodeRef::grad() const {
  if(!graph)
    throw ContractError("empty node reference");
  return graph->nodeGrad(index, gen);
}

// ---------------------------------------------------------------- inits
// Host-side, bit-identical to the reference (graph.cpp:23-63): same RNG
// stream per parameter, same distribution calls.

namespace inits {

ParamInit zeros() {
  return [](Tensor& t, Rng&) { t.setZero(); };
}

ParamInit ones() {
  return [](Tensor& t, Rng&) { t.fill(1); };
}

ParamInit constant(Real v) {
  return [v](Tensor& t, Rng&) { t.fill(v); };
}

ParamInit glorotUniform() {
  return [](Tensor& t, Rng& rng) {
    int rank = t.shape().rank();
    Real fanIn = (Real)t.shape()[rank - 1];
    Real fanOut = rank >= 2 ? (Real)t.shape()[rank - 2] : fanIn;
    Real limit = std::sqrt(Real(6) / (fanIn + fanOut));
    std::uniform_real_distribution<double> d(-(double)limit, (double)limit);
    Real* p = t.data();
    for(int64_t i = 0; i < t.size(); ++i)
      p[i] = (Real)d(rng);
  };
}

ParamInit uniform(Real lo, Real hi) {
  return [lo, hi](Tensor& t, Rng& rng) {
    std::uniform_real_distribution<double> d((double)lo, (double)hi);
    Real* p = t.data();
    for(int64_t i = 0; i < t.size(); ++i)
      p[i] = (Real)d(rng);
  };
}

ParamInit fromVector(std::vector<Real> v) {
  return [v = std::move(v)](Tensor& t, Rng&) {
    if((int64_t)v.size() != t.size())
      throw DimensionError("init vector length mismatch");
    std::copy(v.begin(), v.end(), t.data());
  };
}

}  // namespace inits

// ------------------------------------------------------------ ParamPool

ParamPool::ParamPool() = default;

void ParamPool::grow(int64_t need) {
  int64_t cap = values_ ? (int64_t)values_->elems : 0;
  if(need <= cap)
    return;
  int64_t ncap = std::max<int64_t>(need, std::max<int64_t>(cap * 2, 1 << 20));
  Device& d = Device::get();
  auto swapIn = [&](std::shared_ptr<DeviceBuffer>& buf) {
    DeviceBuffer fresh((size_t)ncap);
    MTKC(mtkc_memset(fresh.ptr, 0, (size_t)ncap * sizeof(float), d.stream()));
    if(buf && used_ > 0)
      MTKC(mtkc_memcpy_d2d(fresh.ptr, buf->ptr, (size_t)used_ * sizeof(float), d.stream()));
    d.sync();
    if(!buf) {
      buf = std::make_shared<DeviceBuffer>();
      buf->owned = true;
    } else if(buf->ptr) {
      mtkc_free(buf->ptr);
    }
    // move the allocation into the long-lived buffer object so every view follows
    buf->ptr = fresh.ptr;
    buf->elems = (size_t)ncap;
    fresh.ptr = nullptr;
  };
  swapIn(values_);
  swapIn(grads_);
}

int64_t ParamPool::reserve(int64_t elems) {
  int64_t off = used_;
  int64_t n = (elems + 63) & ~(int64_t)63;
  grow(used_ + n);
  used_ += n;
  return off;
}

// ------------------------------------------------------------ the graph

ExpressionGraph::ExpressionGraph(uint64_t seed, bool inference)
    : arena_(defaultArenaBytes()), rng_(seed), seed_(seed), inference_(inference) {
  const char* e = std::getenv("MTK_CHECK_FINITE");
  checkFinite_ = e && e[0] == '1';
}

// The reference's 8 GiB host default (tensor.h:45) is far below one
// Transformer-base step's working set on a GPU with 180 GB of HBM3e; the
// device arena defaults to 96 GiB (MTK_ARENA_GB overrides).
size_t ExpressionGraph::defaultArenaBytes() {
  const char* e = std::getenv("MTK_ARENA_GB");
  double gb = e ? std::atof(e) : 96.0;
  return (size_t)(gb * (double)(1ull << 30));
}

void ExpressionGraph::checkRef(const NodeRef& r) const {
  if(r.graph != this)
    throw ContractError("node reference belongs to a different graph");
  if(r.gen != generation_)
    throw ContractError("stale node reference (graph was cleared)");
  if(r.index < 0 || (size_t)r.index >= nodes_.size())
    throw ContractError("node index out of range");
}

int ExpressionGraph::resolve(int i) const {
  while(nodes_[(size_t)i].alias >= 0)
    i = nodes_[(size_t)i].alias;
  return i;
}

Tensor& ExpressionGraph::nodeValue(int index, uint64_t gen) {
  if(gen != generation_)
    throw ContractError("stale node reference (graph was cleared)");
  Tensor& v = nodes_[(size_t)index].value;
  if(v.empty())
    throw ContractError("node value not computed; call forward() first");
  return v;
}

Tensor& ExpressionGraph::nodeGrad(int index, uint64_t gen) {
  if(gen != generation_)
    throw ContractError("stale node reference (graph was cleared)");
  Node& n = nodes_[(size_t)index];
  int r = resolve(index);
  Node& root = nodes_[(size_t)r];
  if(root.isParam) {
    Param& p = paramOf(root);
    if(!p.gradLive) {
      p.grad.setZero();
      p.gradLive = true;
    }
    if(r != index)
      n.grad = p.grad.reshaped(n.shape);
    else
      n.grad = p.grad;
    return n.grad;
  }
  if(root.grad.empty())
    throw ContractError("node gradient not available; call backward() first");
  if(!root.gradLive) {
    root.grad.setZero();
    root.gradLive = true;
  }
  gradSrc(root);  // apply a pending ReLU mask
  if(r != index)
    n.grad = root.grad.reshaped(n.shape);
  return n.grad;
}

NodeRef ExpressionGraph::addNode(Node n) {
  // gradients flow only toward parameters: constants and anything built
  // from constants alone are skipped by the backward sweep, and ops skip
  // the input gradients nobody needs (e.g. dot(mask, context))
  if(!n.isParam) {
    bool any = false;
    for(int in : n.inputs)
      any = any || nodes_[(size_t)resolve(in)].needsGrad;
    n.needsGrad = any;
  }
  nodes_.push_back(std::move(n));
  return NodeRef{this, (int)nodes_.size() - 1, generation_, nodes_.back().shape};
}

Tensor ExpressionGraph::allocTensor(const Shape& s) {
  auto [buf, off] = arena_.alloc(s.size());
  return Tensor(s, buf, off);
}

ExpressionGraph::Param& ExpressionGraph::paramOf(Node& n) { return params_.at(n.paramName); }

ExpressionGraph::GradDst ExpressionGraph::gradDst(int nodeIndex, bool supportsGate) {
  int r = resolve(nodeIndex);
  Node& n = nodes_[(size_t)r];
  if(n.isParam) {
    Param& p = paramOf(n);
    if(!lnPending_.empty()) {  // a later writer must see the deferred sum first
      const float* gp = p.grad.devc();
      for(const auto& j : lnPending_)
        if(gp == j.dgain || gp == j.dbias) {
          flushLnParams();
          break;
        }
    }
    int acc = p.gradLive ? 1 : 0;
    p.gradLive = true;
    return {p.grad.dev(), acc, nullptr, nullptr};
  }
  if(n.grad.empty())
    n.grad = allocTensor(n.shape);
  int acc = n.gradLive ? 1 : 0;
  n.gradLive = true;
  if(n.gate && !supportsGate)
    n.gradGated = false;
  return {n.grad.dev(), acc, supportsGate ? n.gate : nullptr,
          supportsGate ? n.gateMask : nullptr};
}

const float* ExpressionGraph::gradSrc(Node& n) {
  if(n.gate && !n.gradGated) {
    MTKC(mtkc_relu_mask(n.grad.dev(), n.gate, n.grad.size(), Device::get().stream()));
    n.gradGated = true;
  }
  return n.grad.devc();
}

namespace {

void* stream() { return Device::get().stream(); }

// destination pointer with "+=" semantics: zero-fills a fresh buffer
float* accPtr(ExpressionGraph& g, int idx, int64_t elems) {
  auto d = g.gradDst(idx);
  if(!d.accumulate)
    MTKC(mtkc_memset(d.ptr, 0, (size_t)elems * sizeof(float), stream()));
  return d.ptr;
}

void gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, bool tA, const float* B,
          int64_t ldb, bool tB, float* C, int64_t ldc, float beta, const float* bias = nullptr,
          int epi = MTKC_EPI_NONE, const float* gate = nullptr, int64_t batch = 1,
          int64_t sA = 0, int64_t sB = 0, int64_t sC = 0, float* colsum = nullptr,
          int colsumOf = 0, int colsumAcc = 0, const uint32_t* gateMask = nullptr,
          uint32_t* maskOut = nullptr) {
  Device& d = Device::get();
  mtkc_gemm_args g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch = batch;
  g.A = A;
  g.lda = lda;
  g.strideA = sA;
  g.transA = tA;
  g.B = B;
  g.ldb = ldb;
  g.strideB = sB;
  g.transB = tB;
  g.C = C;
  g.ldc = ldc;
  g.strideC = sC;
  g.alpha = 1.f;
  g.beta = beta;
  g.bias = bias;
  g.epilogue = epi;
  g.gate = gate;
  g.precision = (int)d.precision();
  g.workspace = d.scratch(64 << 20);
  g.workspace_bytes = d.scratchBytes();
  g.colsum = colsum;
  g.colsum_of = colsumOf;
  g.colsum_accumulate = colsumAcc;
  if(gateMask) {  // the bit form replaces the float gate
    g.gate = nullptr;
    g.gate_mask = gateMask;
  }
  g.relu_mask_out = maskOut;
  MTKC(mtkc_gemm(&g, d.stream()));
}

std::shared_ptr<DeviceBuffer> uploadIntsTo(ExpressionGraph& g, const std::vector<int32_t>& v,
                                           int64_t* off) {
  auto [buf, o] = g.arena().alloc(std::max<int64_t>((int64_t)v.size(), 1));
  Device::get().upload(buf->ptr + o, v.data(), v.size() * sizeof(int32_t));
  *off = o;
  return buf;
}

// device copy of a host tensor in the arena
Tensor uploadTensor(ExpressionGraph& g, const Tensor& t) {
  Tensor d = g.allocTensor(t.shape());
  if(t.onDevice())
    MTKC(mtkc_memcpy_d2d(d.dev(), t.devc(), (size_t)t.size() * sizeof(float), stream()));
  else
    Device::get().upload(d.dev(), t.data(), (size_t)t.size() * sizeof(float));
  return d;
}

// A read-only device view of a host constant (mask, position table): the
// tensor's own device copy, shared by every node and every copy of it, so a
// batch mask used by 18 attention nodes is uploaded once.
std::shared_ptr<Tensor> sharedConst(const Tensor& t) { return std::make_shared<Tensor>(t); }

// Deterministic scatter plan: positions stably sorted by id (counting
// sort), each id's segment split into chunks of at most kChunk positions.
struct ScatterPlan {
  std::shared_ptr<DeviceBuffer> buf;
  int64_t permOff = 0, cstartOff = 0, crowOff = 0, cslotOff = 0, mfirstOff = 0, mrowOff = 0;
  int64_t nChunks = 0, nMulti = 0, nSlots = 0;
};

constexpr int32_t kChunk = 32;

ScatterPlan makeScatterPlan(ExpressionGraph& g, const std::vector<int32_t>& ids) {
  int32_t maxId = 0;
  for(int32_t v : ids)
    maxId = std::max(maxId, v);
  std::vector<int32_t> cnt((size_t)maxId + 2, 0);
  for(int32_t v : ids)
    ++cnt[(size_t)v + 1];
  for(size_t i = 1; i < cnt.size(); ++i)
    cnt[i] += cnt[i - 1];
  std::vector<int32_t> perm(ids.size());
  {
    std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
    for(size_t i = 0; i < ids.size(); ++i)
      perm[(size_t)pos[(size_t)ids[i]]++] = (int32_t)i;
  }
  std::vector<int32_t> cstart, crow, cslot, mfirst, mrow;
  int32_t slots = 0;
  for(int32_t id = 0; id <= maxId; ++id) {
    int32_t s0 = cnt[(size_t)id], s1 = cnt[(size_t)id + 1];
    if(s0 == s1)
      continue;
    int32_t len = s1 - s0;
    if(len <= kChunk) {
      cstart.push_back(s0);
      crow.push_back(id);
      cslot.push_back(-1);
      continue;
    }
    mfirst.push_back(slots);
    mrow.push_back(id);
    for(int32_t k = s0; k < s1; k += kChunk) {
      cstart.push_back(k);
      crow.push_back(id);
      cslot.push_back(slots++);
    }
  }
  ScatterPlan p;
  p.nChunks = (int64_t)crow.size();
  p.nMulti = (int64_t)mrow.size();
  p.nSlots = slots;
  cstart.push_back((int32_t)perm.size());
  mfirst.push_back(slots);
  std::vector<int32_t> all;
  auto put = [&](const std::vector<int32_t>& v) {
    int64_t o = (int64_t)all.size();
    all.insert(all.end(), v.begin(), v.end());
    return o;
  };
  p.permOff = put(perm);
  p.cstartOff = put(cstart);
  p.crowOff = put(crow);
  p.cslotOff = put(cslot);
  p.mfirstOff = put(mfirst);
  p.mrowOff = put(mrow);
  int64_t off = 0;
  p.buf = uploadIntsTo(g, all, &off);
  for(int64_t* o : {&p.permOff, &p.cstartOff, &p.crowOff, &p.cslotOff, &p.mfirstOff, &p.mrowOff})
    *o += off;
  return p;
}

void scatterPlanAdd(ExpressionGraph& g, const ScatterPlan& p, float* out, const float* src,
                    int64_t cols, float s) {
  const int32_t* base = (const int32_t*)p.buf->ptr;
  float* partial = nullptr;
  if(p.nSlots > 0) {
    auto [buf, off] = g.arena().alloc(p.nSlots * cols);
    partial = buf->ptr + off;
  }
  MTKC(mtkc_scatter_add_rows_chunked(out, src, base + p.permOff, base + p.cstartOff,
                                     base + p.crowOff, base + p.cslotOff, p.nChunks,
                                     base + p.mfirstOff, base + p.mrowOff, p.nMulti, partial,
                                     cols, s, stream()));
}

void pad4(const Shape& s, int64_t out[4]) { s.pad4(out); }

}  // namespace

// ---------------------------------------------------------------- leaves

NodeRef ExpressionGraph::param(const std::string& name, const Shape& shape,
                               const ParamInit& init) {
  auto it = params_.find(name);
  if(it == params_.end()) {
    Param p;
    p.offset = pool_.reserve(shape.size());
    p.value = Tensor(shape, pool_.values(), p.offset);
    p.grad = Tensor(shape, pool_.grads(), p.offset);
    Tensor host(shape);
    Rng prng(hash64(name) ^ seed_);
    init(host, prng);
    MTKC(mtkc_memcpy_h2d(p.value.dev(), host.data(), (size_t)shape.size() * sizeof(float),
                         stream()));
    Device::get().sync();  // host staging vector goes out of scope
    it = params_.emplace(name, std::move(p)).first;
    paramOrder_.push_back(name);
  } else if(it->second.value.shape() != shape) {
    throw ContractError("parameter " + name + " redefined with shape " + shape.str() + " (was " +
                        it->second.value.shape().str() + ")");
  }
  // One node per parameter per graph generation: layers re-reference their
  // weights every time step (layers.cpp:216-224); sharing the node lets the
  // product cache below see repeated products of the same operands.
  auto pn = paramNode_.find(name);
  if(pn != paramNode_.end())
    return NodeRef{this, pn->second, generation_, shape};
  Node n;
  n.op = "param";
  n.shape = shape;
  n.isParam = true;
  n.paramName = name;
  n.value = it->second.value;
  NodeRef r = addNode(std::move(n));
  paramNode_[name] = r.index;
  return r;
}

NodeRef ExpressionGraph::constant(const Tensor& t) {
  Node n;
  n.op = "const";
  n.shape = t.shape();
  n.value = uploadTensor(*this, t);
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::constant(Shape shape, std::vector<Real> values) {
  return constant(Tensor(std::move(shape), std::move(values)));
}

// ----------------------------------------------------------- elementwise

NodeRef ExpressionGraph::binary(const std::string& name, EwiseOp op, NodeRef a, NodeRef b) {
  checkRef(a);
  checkRef(b);
  Node n;
  n.op = name;
  n.shape = broadcastShape(a.shape, b.shape);
  n.inputs = {a.index, b.index};
  n.fwd = [op](ExpressionGraph& g, Node& n) {
    int64_t od[4], ad[4], bd[4];
    pad4(n.shape, od);
    pad4(g.node(n.inputs[0]).shape, ad);
    pad4(g.node(n.inputs[1]).shape, bd);
    MTKC(mtkc_ewise_binary((int)op, n.value.dev(), od, g.valPtr(n.inputs[0]), ad,
                           g.valPtr(n.inputs[1]), bd, Device::get().flags(), stream()));
  };
  n.bwd = [op](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    int64_t od[4], ad[4], bd[4];
    Shape sa = g.node(n.inputs[0]).shape, sb = g.node(n.inputs[1]).shape;
    pad4(n.shape, od);
    pad4(sa, ad);
    pad4(sb, bd);
    bool aliased = false;
    int aliasedNode = -1;  // resolved operand that took over n.grad in this sweep
    for(int which = 0; which < 2; ++which) {
      const Shape& st = which == 0 ? sa : sb;
      int idx = n.inputs[(size_t)which];
      if(!g.node(g.resolve(idx)).needsGrad)
        continue;  // constant operand (mask, scale table)
      bool same = st == n.shape;
      if(op == EwiseOp::Add && same) {
        // residual adds: the first operand whose gradient buffer does not
        // exist yet shares this node's gradient buffer instead of receiving
        // a copy (only this node reads its own gradient, so later
        // contributions to the operand may update the shared buffer)
        Node& in = g.node(g.resolve(idx));
        if(!aliased && !in.isParam && !in.gate && !in.gradLive && in.grad.empty() &&
           in.alias < 0 && in.shape == n.shape) {
          in.grad = n.grad;
          in.gradLive = true;
          aliased = true;
          aliasedNode = g.resolve(idx);
          continue;
        }
        auto d = g.gradDst(idx);
        if(d.ptr == go) {
          // add(h, h) / add(h, reshape(h)): operand 0 took over this buffer
          // just now, so operand 1's contribution doubles it in place;
          // otherwise an earlier sweep aliased it and it already holds go
          if(g.resolve(idx) == aliasedNode)
            MTKC(mtkc_axpy(d.ptr, go, 1.f, st.size(), stream()));
          continue;
        }
        if(d.accumulate)
          MTKC(mtkc_axpy(d.ptr, go, 1.f, st.size(), stream()));
        else
          MTKC(mtkc_memcpy_d2d(d.ptr, go, (size_t)st.size() * sizeof(float), stream()));
        continue;
      }
      float* dst = accPtr(g, idx, st.size());
      MTKC(mtkc_binary_backward((int)op, which, dst, which == 0 ? ad : bd, go, od,
                                g.valPtr(n.inputs[0]), ad, g.valPtr(n.inputs[1]), bd,
                                n.value.devc(), stream()));
    }
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::unary(const std::string& name, EwiseOp op, NodeRef a) {
  checkRef(a);
  Node n;
  n.op = name;
  n.shape = a.shape;
  n.inputs = {a.index};
  n.fwd = [op](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_ewise_unary((int)op, n.value.dev(), g.valPtr(n.inputs[0]), n.value.size(),
                          stream()));
  };
  n.bwd = [op](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    float* dst = accPtr(g, n.inputs[0], n.shape.size());
    MTKC(mtkc_unary_backward((int)op, dst, go, n.value.devc(), g.valPtr(n.inputs[0]),
                             n.shape.size(), stream()));
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::add(NodeRef a, NodeRef b) { return binary("add", EwiseOp::Add, a, b); }
NodeRef ExpressionGraph::sub(NodeRef a, NodeRef b) { return binary("sub", EwiseOp::Sub, a, b); }
NodeRef ExpressionGraph::mul(NodeRef a, NodeRef b) { return binary("mul", EwiseOp::Mul, a, b); }
NodeRef ExpressionGraph::div(NodeRef a, NodeRef b) { return binary("div", EwiseOp::Div, a, b); }
NodeRef ExpressionGraph::tanh(NodeRef a) { return unary("tanh", EwiseOp::Tanh, a); }
NodeRef ExpressionGraph::sigmoid(NodeRef a) { return unary("sigmoid", EwiseOp::Sigmoid, a); }
NodeRef ExpressionGraph::relu(NodeRef a) { return unary("relu", EwiseOp::Relu, a); }
NodeRef ExpressionGraph::exp(NodeRef a) { return unary("exp", EwiseOp::Exp, a); }
NodeRef ExpressionGraph::log(NodeRef a) { return unary("log", EwiseOp::Log, a); }
NodeRef ExpressionGraph::neg(NodeRef a) { return unary("neg", EwiseOp::Neg, a); }

static NodeRef scaleShift(ExpressionGraph& g, const char* name, NodeRef a, Real s, Real c) {
  g.checkRef(a);
  ExpressionGraph::Node n;
  n.op = name;
  n.shape = a.shape;
  n.inputs = {a.index};
  n.fwd = [s, c](ExpressionGraph& g, ExpressionGraph::Node& n) {
    MTKC(mtkc_scale_shift(n.value.dev(), g.valPtr(n.inputs[0]), s, c, n.value.size(), stream()));
  };
  n.bwd = [s](ExpressionGraph& g, ExpressionGraph::Node& n) {
    const float* go = g.gradSrc(n);
    auto d = g.gradDst(n.inputs[0]);
    if(d.accumulate)
      MTKC(mtkc_axpy(d.ptr, go, s, n.shape.size(), stream()));
    else
      MTKC(mtkc_scale_shift(d.ptr, go, s, 0.f, n.shape.size(), stream()));
  };
  return g.addNode(std::move(n));
}

NodeRef ExpressionGraph::scale(NodeRef a, Real s) { return scaleShift(*this, "scale", a, s, 0); }
NodeRef ExpressionGraph::addScalar(NodeRef a, Real s) {
  return scaleShift(*this, "addScalar", a, 1, s);
}

// -------------------------------------------------------- linear algebra

namespace {
struct MV {
  int64_t batch, rows, cols, bstride, ld;
};
MV mview(const Shape& s, bool t) {
  if(s.rank() == 2)
    return {1, t ? s[1] : s[0], t ? s[0] : s[1], 0, s[1]};
  return {s[0], t ? s[2] : s[1], t ? s[1] : s[2], s[1] * s[2], s[2]};
}

// dst (+)= op(x) op(y) with the reference's batching rules (graph.cpp:273-291):
// a batched product accumulated into a rank-2 destination sums the batch.
void gemmAccum(float* dst, int acc, const Shape& ds, const float* x, const Shape& xs, bool tx,
               const float* y, const Shape& ys, bool ty) {
  MV vx = mview(xs, tx), vy = mview(ys, ty);
  int64_t M = vx.rows, K = vx.cols, N = vy.cols;
  int64_t batch = std::max(vx.batch, vy.batch);
  bool sumBatch = batch > 1 && ds.rank() == 2;
  if(sumBatch && xs.rank() == 3 && ys.rank() == 3 && tx && !ty) {
    // sum_b x_b^T y_b == X^T Y with the batch stacked along K
    gemm(M, N, K * batch, x, xs[2], true, y, ys[2], false, dst, N, acc ? 1.f : 0.f);
    return;
  }
  if(!sumBatch && ds.rank() == 3 && xs.rank() == 3 && ys.rank() == 2 && !tx) {
    // [B,T,K] x op(y) into [B,T,N]: one GEMM over B*T rows
    gemm(M * batch, N, K, x, vx.ld, false, y, vy.ld, ty, dst, N, acc ? 1.f : 0.f);
    return;
  }
  gemm(M, N, K, x, vx.ld, tx, y, vy.ld, ty, dst, N, acc ? 1.f : 0.f, nullptr, MTKC_EPI_NONE,
       nullptr, batch, vx.batch == 1 ? 0 : vx.bstride, vy.batch == 1 ? 0 : vy.bstride,
       sumBatch ? 0 : M * N);
}
}  // namespace

NodeRef ExpressionGraph::dot(NodeRef a, NodeRef b, bool transA, bool transB) {
  checkRef(a);
  checkRef(b);
  // Identical products are computed once per generation (e.g. the Bahdanau
  // key projection keys*U, which the decoder re-requests at every target
  // position, layers.cpp:68); every use accumulates into the one node's
  // gradient, exactly the sum the reference forms over its copies.
  auto key = std::make_tuple(a.index, b.index, transA, transB);
  auto cached = dotCache_.find(key);
  if(cached != dotCache_.end())
    return NodeRef{this, cached->second, generation_, nodes_[(size_t)cached->second].shape};
  NodeRef r = dotImpl(a, b, transA, transB);
  dotCache_[key] = r.index;
  return r;
}

NodeRef ExpressionGraph::dotImpl(NodeRef a, NodeRef b, bool transA, bool transB) {
  auto opRows = [](const Shape& s, bool t) { return t ? s.back() : s[s.rank() - 2]; };
  auto opCols = [](const Shape& s, bool t) { return t ? s[s.rank() - 2] : s.back(); };
  if(a.shape.rank() < 2 || b.shape.rank() < 2)
    throw DimensionError("matmul needs rank >= 2 operands: " + a.shape.str() + " x " +
                         b.shape.str());
  if(a.shape.rank() > 3 || b.shape.rank() > 3)
    throw DimensionError("matmul operands must be rank 2 or 3, got " + a.shape.str() + " x " +
                         b.shape.str());
  if(opCols(a.shape, transA) != opRows(b.shape, transB))
    throw DimensionError("matmul inner dims disagree: " + a.shape.str() + " x " +
                         b.shape.str());
  int64_t batchA = a.shape.rank() == 3 ? a.shape[0] : 1;
  int64_t batchB = b.shape.rank() == 3 ? b.shape[0] : 1;
  if(batchA != batchB && batchA != 1 && batchB != 1)
    throw DimensionError("matmul batch dims disagree: " + a.shape.str() + " x " +
                         b.shape.str());
  Node n;
  n.op = "matmul";
  int64_t m = opRows(a.shape, transA), c = opCols(b.shape, transB);
  n.shape = (a.shape.rank() == 3 || b.shape.rank() == 3)
                ? Shape({std::max(batchA, batchB), m, c})
                : Shape({m, c});
  n.inputs = {a.index, b.index};
  n.fwd = [transA, transB](ExpressionGraph& g, Node& n) {
    const Shape& sa = g.node(n.inputs[0]).shape;
    const Shape& sb = g.node(n.inputs[1]).shape;
    MV va = mview(sa, transA), vb = mview(sb, transB);
    int64_t batch = std::max(va.batch, vb.batch);
    if(batch == 1 || (sa.rank() == 3 && sb.rank() == 2 && !transA)) {
      // [B,T,K] x [K,N]: one GEMM over B*T rows
      int64_t rows = va.rows * va.batch;
      gemm(rows, vb.cols, va.cols, g.valPtr(n.inputs[0]), va.ld, transA, g.valPtr(n.inputs[1]),
           vb.ld, transB, n.value.dev(), vb.cols, 0.f);
      return;
    }
    gemm(va.rows, vb.cols, va.cols, g.valPtr(n.inputs[0]), va.ld, transA,
         g.valPtr(n.inputs[1]), vb.ld, transB, n.value.dev(), vb.cols, 0.f, nullptr,
         MTKC_EPI_NONE, nullptr, batch, va.batch == 1 ? 0 : va.bstride,
         vb.batch == 1 ? 0 : vb.bstride, va.rows * vb.cols);
  };
  n.bwd = [transA, transB](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    Node& na = g.node(n.inputs[0]);
    Node& nb = g.node(n.inputs[1]);
    Shape sa = na.shape, sb = nb.shape, so = n.shape;
    // graph.cpp:322-330
    if(na.needsGrad) {
      auto d = g.gradDst(n.inputs[0]);
      if(!transA)
        gemmAccum(d.ptr, d.accumulate, sa, go, so, false, g.valPtr(n.inputs[1]), sb, !transB);
      else
        gemmAccum(d.ptr, d.accumulate, sa, g.valPtr(n.inputs[1]), sb, transB, go, so, true);
    }
    if(nb.needsGrad) {
      auto d = g.gradDst(n.inputs[1]);
      if(!transB)
        gemmAccum(d.ptr, d.accumulate, sb, g.valPtr(n.inputs[0]), sa, !transA, go, so, false);
      else
        gemmAccum(d.ptr, d.accumulate, sb, go, so, true, g.valPtr(n.inputs[0]), sa, transA);
    }
  };
  return addNode(std::move(n));
}

// Fused affine: out = x op(W) + b in one GEMM with a bias (and optional
// ReLU) epilogue.  Backward: dX = dY op(W)^T (ReLU-gated epilogue into a
// gated producer), dW = X^T dY or dY^T X, db = colsum(dY).
static NodeRef affineImpl(ExpressionGraph& g, NodeRef x, NodeRef w, NodeRef b, bool transW,
                          bool relu) {
  g.checkRef(x);
  g.checkRef(w);
  g.checkRef(b);
  if(x.shape.rank() < 2 || w.shape.rank() != 2)
    throw DimensionError("matmul needs rank >= 2 operands: " + x.shape.str() + " x " +
                         w.shape.str());
  int64_t K = x.shape.back();
  int64_t wr = transW ? w.shape[1] : w.shape[0];
  int64_t N = transW ? w.shape[0] : w.shape[1];
  if(K != wr)
    throw DimensionError("matmul inner dims disagree: " + x.shape.str() + " x " +
                         w.shape.str());
  if(b.shape.size() != N)
    throw DimensionError("shapes not broadcastable: bias " + b.shape.str() + " vs output width " +
                         std::to_string(N));
  std::vector<int64_t> dims = x.shape.dims();
  dims.back() = N;
  ExpressionGraph::Node n;
  n.op = relu ? "affineRelu" : (transW ? "affineT" : "affine");
  n.shape = Shape(dims);
  n.inputs = {x.index, w.index, b.index};
  int64_t rows = x.shape.size() / K;
  n.fwd = [rows, K, N, transW, relu](ExpressionGraph& g, ExpressionGraph::Node& n) {
    // TF32: the ReLU also leaves its gate as a bit mask for the consumer's dX
    uint32_t* bits = nullptr;
    if(relu && Device::get().precision() == Precision::TF32) {
      n.gateBits = g.allocTensor(Shape({rows, (N + 31) / 32}));
      bits = reinterpret_cast<uint32_t*>(n.gateBits.dev());
    }
    gemm(rows, N, K, g.valPtr(n.inputs[0]), K, false, g.valPtr(n.inputs[1]), transW ? K : N,
         transW, n.value.dev(), N, 0.f, g.valPtr(n.inputs[2]),
         relu ? MTKC_EPI_RELU : MTKC_EPI_NONE, nullptr, 1, 0, 0, 0, nullptr, 0, 0, nullptr, bits);
    if(relu) {
      n.gate = n.value.devc();
      n.gateMask = bits;
    }
  };
  n.bwd = [rows, K, N, transW](ExpressionGraph& g, ExpressionGraph::Node& n) {
    const float* go = g.gradSrc(n);
    {  // dX = dY op(W)^T
      auto d = g.gradDst(n.inputs[0], true);
      gemm(rows, K, N, go, N, false, g.valPtr(n.inputs[1]), transW ? K : N, !transW, d.ptr, K,
           d.accumulate ? 1.f : 0.f, nullptr, MTKC_EPI_NONE, d.gate, 1, 0, 0, 0, nullptr, 0, 0,
           d.gateMask);
    }
    {  // dW, with db = colsum(dY) summed from the dY tiles the product stages
      auto d = g.gradDst(n.inputs[1]);
      auto db = g.gradDst(n.inputs[2]);
      if(!transW)
        gemm(K, N, rows, g.valPtr(n.inputs[0]), K, true, go, N, false, d.ptr, N,
             d.accumulate ? 1.f : 0.f, nullptr, MTKC_EPI_NONE, nullptr, 1, 0, 0, 0, db.ptr,
             MTKC_COLSUM_B, db.accumulate);
      else
        gemm(N, K, rows, go, N, true, g.valPtr(n.inputs[0]), K, false, d.ptr, K,
             d.accumulate ? 1.f : 0.f, nullptr, MTKC_EPI_NONE, nullptr, 1, 0, 0, 0, db.ptr,
             MTKC_COLSUM_A, db.accumulate);
    }
  };
  return g.addNode(std::move(n));
}

namespace {
// Siblings of an affineGroup: the q/k/v projections of one attention input.
struct AffineGroup {
  std::vector<int> members;  // affine node indices, ascending
  std::vector<ExpressionGraph::Fn> fwd0, bwd0;  // the members' own fwd/bwd
  int x = -1;
  std::vector<int> W, b;  // parameter node indices per member
  int64_t rows = 0, K = 0, N = 0;
  bool fwdDone = false;
  uint64_t bwdDone = ~0ull;  // backward sweep that already ran the group
};

mtkc_gemm_args groupArgs(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, bool tA,
                         const float* B, int64_t ldb, bool tB, float* C, int64_t ldc, float beta,
                         const float* bias) {
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
  g.bias = bias;
  g.epilogue = MTKC_EPI_NONE;
  g.precision = (int)d.precision();
  g.workspace = d.scratch(64 << 20);
  g.workspace_bytes = d.scratchBytes();
  return g;
}
}  // namespace

std::vector<NodeRef> ExpressionGraph::affineGroup(NodeRef x, const std::vector<NodeRef>& Ws,
                                                  const std::vector<NodeRef>& bs) {
  if(Ws.size() != bs.size() || Ws.empty() || Ws.size() > 3)
    throw ContractError("affineGroup takes 1..3 (W, b) pairs");
  std::vector<NodeRef> out;
  for(size_t i = 0; i < Ws.size(); ++i)
    out.push_back(affine(x, Ws[i], bs[i]));
  if(out.size() < 2)
    return out;
  for(auto& w : Ws)
    if(w.shape != Ws[0].shape)
      return out;  // unequal shapes: separate launches
  auto grp = std::make_shared<AffineGroup>();
  grp->x = x.index;
  grp->K = x.shape.back();
  grp->N = Ws[0].shape[1];
  grp->rows = x.shape.size() / grp->K;
  for(size_t i = 0; i < out.size(); ++i) {
    Node& n = nodes_[(size_t)out[i].index];
    grp->members.push_back(out[i].index);
    grp->fwd0.push_back(n.fwd);
    grp->bwd0.push_back(n.bwd);
    grp->W.push_back(Ws[i].index);
    grp->b.push_back(bs[i].index);
    n.group = grp;
  }
  const size_t G = out.size();
  // forward: the first member computes every member's output in one launch
  for(size_t i = 0; i < G; ++i) {
    nodes_[(size_t)out[i].index].fwd = [grp, G](ExpressionGraph& g, Node&) {
      if(grp->fwdDone)
        return;
      grp->fwdDone = true;
      mtkc_gemm_args probs[3];
      for(size_t j = 0; j < G; ++j) {
        Node& m = g.node(grp->members[j]);
        if(m.value.empty())
          m.value = g.allocTensor(m.shape);
        probs[j] = groupArgs(grp->rows, grp->N, grp->K, g.valPtr(grp->x), grp->K, false,
                             g.valPtr(grp->W[j]), grp->N, false, m.value.dev(), grp->N, 0.f,
                             g.valPtr(grp->b[j]));
      }
      MTKC(mtkc_gemm_group(probs, (int)G, 0, Device::get().stream()));
    };
  }
  // backward: the first live member reached by the sweep (highest index)
  // does dX, dW and db for every live member
  for(size_t i = 0; i < G; ++i) {
    nodes_[(size_t)out[i].index].bwd = [grp, G, i](ExpressionGraph& g, Node& n) {
      if(grp->bwdDone == g.backwardCount_)
        return;
      std::vector<size_t> live;
      for(size_t j = G; j-- > 0;)
        if(g.node(grp->members[j]).gradLive)
          live.push_back(j);
      if(live.size() < 2) {
        grp->bwd0[i](g, n);
        return;
      }
      grp->bwdDone = g.backwardCount_;
      const int64_t rows = grp->rows, K = grp->K, N = grp->N;
      Device& dev = Device::get();
      const float* dY[3];
      for(size_t q = 0; q < live.size(); ++q)
        dY[q] = g.gradSrc(g.node(grp->members[live[q]]));
      {  // dX (+)= sum_j dY_j W_j^T: one K-concatenated product
        auto d = g.gradDst(grp->x, true);
        if(d.gate) {  // ReLU-gated producer: per-member products keep the gate epilogue
          for(size_t q = 0; q < live.size(); ++q) {
            auto dq = q == 0 ? d : g.gradDst(grp->x, true);
            gemm(rows, K, N, dY[q], N, false, g.valPtr(grp->W[live[q]]), N, true, dq.ptr, K,
                 dq.accumulate ? 1.f : 0.f, nullptr, MTKC_EPI_NONE, dq.gate, 1, 0, 0, 0, nullptr, 0,
                 0, dq.gateMask);
          }
        } else {
          mtkc_gemm_args probs[3];
          for(size_t q = 0; q < live.size(); ++q)
            probs[q] = groupArgs(rows, K, N, dY[q], N, false, g.valPtr(grp->W[live[q]]), N, true,
                                 d.ptr, K, d.accumulate ? 1.f : 0.f, nullptr);
          MTKC(mtkc_gemm_group(probs, (int)live.size(), 1, dev.stream()));
        }
      }
      {  // dW_j (+)= X^T dY_j and db_j (+)= colsum(dY_j): one grouped launch
         // when the accumulate flags agree
        ExpressionGraph::GradDst dw[3], db[3];
        bool same = true;
        for(size_t q = 0; q < live.size(); ++q) {
          dw[q] = g.gradDst(grp->W[live[q]]);
          db[q] = g.gradDst(grp->b[live[q]]);
          same = same && dw[q].accumulate == dw[0].accumulate &&
                 db[q].accumulate == db[0].accumulate;
        }
        if(same) {
          mtkc_gemm_args probs[3];
          for(size_t q = 0; q < live.size(); ++q) {
            probs[q] = groupArgs(K, N, rows, g.valPtr(grp->x), K, true, dY[q], N, false,
                                 dw[q].ptr, N, dw[q].accumulate ? 1.f : 0.f, nullptr);
            probs[q].colsum = db[q].ptr;
            probs[q].colsum_of = MTKC_COLSUM_B;
            probs[q].colsum_accumulate = db[q].accumulate;
          }
          MTKC(mtkc_gemm_group(probs, (int)live.size(), 0, dev.stream()));
        } else {
          for(size_t q = 0; q < live.size(); ++q)
            gemm(K, N, rows, g.valPtr(grp->x), K, true, dY[q], N, false, dw[q].ptr, N,
                 dw[q].accumulate ? 1.f : 0.f, nullptr, MTKC_EPI_NONE, nullptr, 1, 0, 0, 0,
                 db[q].ptr, MTKC_COLSUM_B, db[q].accumulate);
        }
      }
    };
  }
  return out;
}

// device dropout node state (dropout / dropoutResidual)
namespace {
struct DropoutAux {
  uint64_t key;
  float p;
  int64_t inner, axisLen;
};
}  // namespace

NodeRef ExpressionGraph::residualAdd(NodeRef r, NodeRef z) {
  checkRef(r);
  checkRef(z);
  Node& zn = nodes_[(size_t)z.index];
  if(zn.op == "dropout" && z.index == (int)nodes_.size() - 1 && zn.shape == r.shape &&
     resolve(r.index) != resolve(zn.inputs[0]) && r.index != z.index &&
     (size_t)z.index >= computed_) {
    // r + dropout(f) (layers.cpp:135) as one pass: out = r + f * m
    // forward; d(r) = d(out) (shared buffer, as add's backward), d(f) = d(out) * m
    zn.op = "dropoutResidual";
    zn.inputs.push_back(r.index);
    zn.fwd = [](ExpressionGraph& g, Node& n) {
      auto* a = static_cast<DropoutAux*>(n.aux.get());
      MTKC(mtkc_dropout(n.value.dev(), g.valPtr(n.inputs[0]), g.valPtr(n.inputs[1]),
                        n.value.size(), a->inner, a->axisLen, a->p, a->key, stream()));
    };
    zn.bwd = [](ExpressionGraph& g, Node& n) {
      auto* a = static_cast<DropoutAux*>(n.aux.get());
      const float* go = g.gradSrc(n);
      if(g.node(g.resolve(n.inputs[0])).needsGrad) {
        auto d = g.gradDst(n.inputs[0]);
        MTKC(mtkc_dropout_backward(d.ptr, go, n.shape.size(), a->inner, a->axisLen, a->p, a->key,
                                   d.accumulate, stream()));
      }
      Node& in = g.node(g.resolve(n.inputs[1]));
      if(!in.needsGrad)
        return;
      if(!in.isParam && !in.gate && !in.gradLive && in.grad.empty() && in.alias < 0 &&
         in.shape == n.shape) {
        in.grad = n.grad;
        in.gradLive = true;
      } else {
        auto d = g.gradDst(n.inputs[1]);
        if(d.ptr != go) {
          if(d.accumulate)
            MTKC(mtkc_axpy(d.ptr, go, 1.f, n.shape.size(), stream()));
          else
            MTKC(mtkc_memcpy_d2d(d.ptr, go, (size_t)n.shape.size() * sizeof(float), stream()));
        }
      }
    };
    zn.needsGrad = zn.needsGrad || nodes_[(size_t)resolve(r.index)].needsGrad;
    return z;
  }
  const bool fusable = Device::get().precision() == Precision::TF32 &&
                       z.index == (int)nodes_.size() - 1 && zn.op == "affine" && !zn.group &&
                       zn.alias < 0 && zn.shape == r.shape && r.index != z.index &&
                       resolve(r.index) != resolve(zn.inputs[0]) &&
                       (size_t)z.index >= computed_;
  if(!fusable)
    return add(r, z);
  // z = x op(W) + b  ->  z = x op(W) + b + r : the affine forward with beta = 1
  // and the addend r (graph.cpp:139-176 add semantics, fused)
  zn.op = "affineResidual";
  zn.inputs.push_back(r.index);
  auto fwd0 = zn.fwd;
  auto bwd0 = zn.bwd;
  const int64_t K = nodes_[(size_t)zn.inputs[0]].shape.back();
  (void)fwd0;
  const int64_t N = zn.shape.back();
  const bool transW = false;  // only op "affine" (x W, not x W^T) is folded
  const int64_t rows = zn.shape.size() / N;
  zn.fwd = [rows, K, N, transW](ExpressionGraph& g, Node& n) {
    Device& d = Device::get();
    mtkc_gemm_args a{};
    a.M = rows;
    a.N = N;
    a.K = K;
    a.batch = 1;
    a.A = g.valPtr(n.inputs[0]);
    a.lda = K;
    a.B = g.valPtr(n.inputs[1]);
    a.ldb = transW ? K : N;
    a.transB = transW;
    a.C = n.value.dev();
    a.ldc = N;
    a.alpha = 1.f;
    a.beta = 1.f;
    a.bias = g.valPtr(n.inputs[2]);
    a.addend = g.valPtr(n.inputs[3]);
    a.precision = (int)d.precision();
    a.workspace = d.scratch(64 << 20);
    a.workspace_bytes = d.scratchBytes();
    MTKC(mtkc_gemm(&a, d.stream()));
  };
  zn.bwd = [bwd0](ExpressionGraph& g, Node& n) {
    // d(residual) = d(out): share the gradient buffer when the residual
    // operand has none yet (as the add backward does), else add into it
    const float* go = g.gradSrc(n);
    Node& in = g.node(g.resolve(n.inputs[3]));
    if(!in.isParam && !in.gate && !in.gradLive && in.grad.empty() && in.alias < 0 &&
       in.shape == n.shape) {
      in.grad = n.grad;
      in.gradLive = true;
    } else {
      auto d = g.gradDst(n.inputs[3]);
      if(d.ptr != go) {
        if(d.accumulate)
          MTKC(mtkc_axpy(d.ptr, go, 1.f, n.shape.size(), stream()));
        else
          MTKC(mtkc_memcpy_d2d(d.ptr, go, (size_t)n.shape.size() * sizeof(float), stream()));
      }
    }
    bwd0(g, n);  // dX, dW, db of the affine part (inputs 0..2)
  };
  return z;
}

NodeRef ExpressionGraph::affine(NodeRef x, NodeRef w, NodeRef b, bool transW) {
  return affineImpl(*this, x, w, b, transW, false);
}

NodeRef ExpressionGraph::affineRelu(NodeRef x, NodeRef w, NodeRef b) {
  return affineImpl(*this, x, w, b, false, true);
}

NodeRef ExpressionGraph::reshape(NodeRef a, Shape shape) {
  checkRef(a);
  if(shape.size() != a.shape.size())
    throw DimensionError("reshape element count mismatch: " + a.shape.str() + " -> " +
                         shape.str());
  Node n;
  n.op = "reshape";
  n.shape = shape;
  n.inputs = {a.index};
  n.alias = a.index;  // value and gradient are views of the input
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::transpose(NodeRef a, std::vector<int> perm) {
  checkRef(a);
  if((int)perm.size() != a.shape.rank())
    throw DimensionError("transpose perm rank mismatch");
  std::vector<int64_t> dims;
  for(int p : perm)
    dims.push_back(a.shape[p]);
  std::vector<int> inv((size_t)a.shape.rank());
  for(int i = 0; i < (int)perm.size(); ++i)
    inv[(size_t)perm[(size_t)i]] = i;
  Node n;
  n.op = "transpose";
  n.shape = Shape(dims);
  n.inputs = {a.index};
  auto p4 = [](const Shape& s, const std::vector<int>& p, int out[4]) {
    int off = 4 - s.rank();
    for(int i = 0; i < 4; ++i)
      out[i] = i;
    for(int i = 0; i < s.rank(); ++i)
      out[off + i] = off + p[(size_t)i];
  };
  n.fwd = [perm, p4](ExpressionGraph& g, Node& n) {
    const Shape& s = g.node(n.inputs[0]).shape;
    int64_t sd[4];
    int pp[4];
    pad4(s, sd);
    p4(s, perm, pp);
    MTKC(mtkc_transpose(n.value.dev(), g.valPtr(n.inputs[0]), sd, pp, 0, stream()));
  };
  n.bwd = [inv, p4](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    int64_t sd[4];
    int pp[4];
    pad4(n.shape, sd);
    p4(n.shape, inv, pp);
    auto d = g.gradDst(n.inputs[0]);
    MTKC(mtkc_transpose(d.ptr, go, sd, pp, d.accumulate, stream()));
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::concat(const std::vector<NodeRef>& parts, int axis) {
  if(parts.empty())
    throw ContractError("concat of zero parts");
  for(auto& p : parts)
    checkRef(p);
  std::vector<int64_t> dims = parts[0].shape.dims();
  for(size_t i = 1; i < parts.size(); ++i) {
    for(int d = 0; d < (int)dims.size(); ++d)
      if(d != axis && parts[i].shape[d] != dims[(size_t)d])
        throw DimensionError("concat shape mismatch on non-concat axis");
    dims[(size_t)axis] += parts[i].shape[axis];
  }
  Node n;
  n.op = "concat";
  n.shape = Shape(dims);
  for(auto& p : parts)
    n.inputs.push_back(p.index);
  int64_t outer = 1, inner = 1;
  for(int i = 0; i < axis; ++i)
    outer *= n.shape[i];
  for(int i = axis + 1; i < n.shape.rank(); ++i)
    inner *= n.shape[i];
  int64_t total = n.shape[axis];
  n.fwd = [axis, outer, inner, total](ExpressionGraph& g, Node& n) {
    int64_t off = 0;
    float* o = n.value.dev();
    for(int i : n.inputs) {
      int64_t pa = g.node(i).shape[axis];
      MTKC(mtkc_copy_blocks(o, total * inner, off * inner, g.valPtr(i), pa * inner, 0, outer,
                            pa * inner, 0, stream()));
      off += pa;
    }
  };
  n.bwd = [axis, outer, inner, total](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    int64_t off = 0;
    for(int i : n.inputs) {
      int64_t pa = g.node(i).shape[axis];
      auto d = g.gradDst(i);
      MTKC(mtkc_copy_blocks(d.ptr, pa * inner, 0, go, total * inner, off * inner, outer,
                            pa * inner, d.accumulate, stream()));
      off += pa;
    }
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::slice(NodeRef a, int axis, int64_t start, int64_t len) {
  checkRef(a);
  if(axis < 0 || axis >= a.shape.rank() || start < 0 || len < 1 || start + len > a.shape[axis])
    throw DimensionError("slice out of range for " + a.shape.str());
  std::vector<int64_t> dims = a.shape.dims();
  dims[(size_t)axis] = len;
  Node n;
  n.op = "slice";
  n.shape = Shape(dims);
  n.inputs = {a.index};
  int64_t outer = 1, inner = 1;
  for(int i = 0; i < axis; ++i)
    outer *= a.shape[i];
  for(int i = axis + 1; i < a.shape.rank(); ++i)
    inner *= a.shape[i];
  int64_t full = a.shape[axis];
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_copy_blocks(n.value.dev(), len * inner, 0, g.valPtr(n.inputs[0]), full * inner,
                          start * inner, outer, len * inner, 0, stream()));
  };
  n.bwd = [=](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    float* dst = accPtr(g, n.inputs[0], outer * full * inner);
    MTKC(mtkc_copy_blocks(dst, full * inner, start * inner, go, len * inner, 0, outer,
                          len * inner, 1, stream()));
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::gatherRows(NodeRef a, std::vector<int64_t> rows) {
  checkRef(a);
  std::vector<int64_t> dims = a.shape.dims();
  dims[0] = (int64_t)rows.size();
  std::vector<int32_t> r32(rows.size());
  for(size_t i = 0; i < rows.size(); ++i) {
    if(rows[i] < 0 || rows[i] >= a.shape[0])
      throw ContractError("row index " + std::to_string(rows[i]) + " out of range 0.." +
                          std::to_string(a.shape[0] - 1));
    r32[i] = (int32_t)rows[i];
  }
  Node n;
  n.op = "gatherRows";
  n.shape = Shape(dims);
  n.inputs = {a.index};
  int64_t cols = a.shape.size() / a.shape[0];
  int64_t srcRows = a.shape[0];
  int64_t off = 0;
  auto ids = uploadIntsTo(*this, r32, &off);
  auto plan = std::make_shared<ScatterPlan>(makeScatterPlan(*this, r32));
  n.aux = plan;
  int64_t nr = (int64_t)rows.size();
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_gather_rows(n.value.dev(), g.valPtr(n.inputs[0]), (const int32_t*)ids->ptr + off,
                          nr, cols, srcRows, Device::get().flags(), stream()));
  };
  n.bwd = [=](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    float* dst = accPtr(g, n.inputs[0], srcRows * cols);
    scatterPlanAdd(g, *plan, dst, go, cols, 1.f);
  };
  return addNode(std::move(n));
}

// -------------------------------------------- reductions / normalisation

NodeRef ExpressionGraph::reduce(ReduceOp op, NodeRef a, int axis, bool keepAxis) {
  checkRef(a);
  if(axis < 0 || axis >= a.shape.rank())
    throw DimensionError("reduce axis " + std::to_string(axis) + " out of range for " +
                         a.shape.str());
  std::vector<int64_t> dims;
  for(int i = 0; i < a.shape.rank(); ++i) {
    if(i == axis) {
      if(keepAxis)
        dims.push_back(1);
    } else {
      dims.push_back(a.shape[i]);
    }
  }
  if(dims.empty())
    dims.push_back(1);
  Node n;
  n.op = op == ReduceOp::Sum ? "sum" : op == ReduceOp::Mean ? "mean"
                                     : op == ReduceOp::Max  ? "max"
                                                            : "argmax";
  n.shape = Shape(dims);
  n.inputs = {a.index};
  int64_t outer = 1, inner = 1, cnt = a.shape[axis];
  for(int i = 0; i < axis; ++i)
    outer *= a.shape[i];
  for(int i = axis + 1; i < a.shape.rank(); ++i)
    inner *= a.shape[i];
  int64_t total = a.shape.size();
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_reduce((int)op, n.value.dev(), g.valPtr(n.inputs[0]), outer, cnt, inner,
                     stream()));
  };
  if(op != ReduceOp::Argmax) {
    n.bwd = [=](ExpressionGraph& g, Node& n) {
      const float* go = g.gradSrc(n);
      float* dst = accPtr(g, n.inputs[0], total);
      MTKC(mtkc_reduce_backward((int)op, dst, go, g.valPtr(n.inputs[0]), outer, cnt, inner,
                                stream()));
    };
  }
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::softmax(NodeRef a, Tensor mask) {
  checkRef(a);
  Node n;
  n.op = "softmax";
  n.shape = a.shape;
  n.inputs = {a.index};
  Tensor dmask;
  int64_t md[4] = {1, 1, 1, 1};
  if(!mask.empty()) {
    int64_t xd[4];
    a.shape.pad4(xd);
    mask.shape().pad4(md);
    for(int i = 0; i < 4; ++i)
      if(md[i] != 1 && md[i] != xd[i])
        throw DimensionError("operand shape " + mask.shape().str() +
                             " incompatible with broadcast result");
    dmask = mask;  // shared device copy, uploaded on first use
  }
  auto keep = std::make_shared<Tensor>(dmask);
  n.aux = keep;
  std::vector<int64_t> mdv(md, md + 4);
  n.fwd = [keep, mdv](ExpressionGraph& g, Node& n) {
    int64_t xd[4];
    pad4(n.shape, xd);
    Device& d = Device::get();
    MTKC(mtkc_softmax(n.value.dev(), g.valPtr(n.inputs[0]), xd,
                      keep->empty() ? nullptr : keep->devc(), mdv.data(), 0, d.flags(),
                      d.stream()));
  };
  n.bwd = [](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    int64_t cols = n.shape.back(), rows = n.shape.size() / cols;
    float* dst = accPtr(g, n.inputs[0], n.shape.size());
    MTKC(mtkc_softmax_backward(dst, n.value.devc(), go, rows, cols, stream()));
  };
  return addNode(std::move(n));
}

namespace {
struct LnCache {
  Tensor invStd, xhat, mean;
  bool fast = false;  // mean/invStd cache, xhat recomputed (mtkc_layernorm_stats)
};
}  // namespace

NodeRef ExpressionGraph::layerNorm(NodeRef x, NodeRef gain, NodeRef bias, Real eps) {
  checkRef(x);
  checkRef(gain);
  checkRef(bias);
  int64_t d = x.shape.back();
  if(d < 2)
    throw DimensionError("layer norm needs last extent >= 2, got " + x.shape.str());
  if(gain.shape.size() != d || bias.shape.size() != d)
    throw DimensionError("layer norm gain/bias must have length " + std::to_string(d));
  Node n;
  n.op = "layerNorm";
  n.shape = x.shape;
  n.inputs = {x.index, gain.index, bias.index};
  auto cache = std::make_shared<LnCache>();
  n.aux = cache;
  int64_t rows = x.shape.size() / d;
  n.fwd = [cache, eps, d, rows](ExpressionGraph& g, Node& n) {
    const float* xin = g.valPtr(n.inputs[0]);
    const float* gp = g.valPtr(n.inputs[1]);
    const float* bp = g.valPtr(n.inputs[2]);
    cache->invStd = g.allocTensor(Shape({rows}));
    cache->fast = mtkc_layernorm_fast_supported(d) &&
                  (((uintptr_t)xin | (uintptr_t)gp | (uintptr_t)bp) % 16) == 0;
    if(cache->fast) {
      cache->mean = g.allocTensor(Shape({rows}));
      MTKC(mtkc_layernorm_stats(n.value.dev(), xin, gp, bp, eps, cache->mean.dev(),
                                cache->invStd.dev(), rows, d, stream()));
      return;
    }
    cache->xhat = g.allocTensor(n.shape);
    MTKC(mtkc_layernorm(n.value.dev(), xin, gp, bp, eps, cache->invStd.dev(), cache->xhat.dev(),
                        rows, d, stream()));
  };
  n.bwd = [cache, d, rows](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    auto dx = g.gradDst(n.inputs[0]);
    auto dg = g.gradDst(n.inputs[1]);
    auto db = g.gradDst(n.inputs[2]);
    if(dg.accumulate != db.accumulate) {  // one flag for both parameter grads
      MTKC(mtkc_memset(dg.accumulate ? db.ptr : dg.ptr, 0, (size_t)d * sizeof(float), stream()));
      dg.accumulate = db.accumulate = 1;
    }
    Device& dev = Device::get();
    if(cache->fast && (((uintptr_t)go | (uintptr_t)dx.ptr) % 16) == 0) {
      if(g.lnDeferActive()) {
        const int64_t blocks = mtkc_layernorm_stats_partial_blocks(rows);
        Tensor part = g.allocTensor(Shape({blocks, 2, d}));
        MTKC(mtkc_layernorm_stats_backward(
            go, g.valPtr(n.inputs[0]), g.valPtr(n.inputs[1]), cache->mean.devc(),
            cache->invStd.devc(), dx.ptr, dg.ptr, db.ptr, rows, d, dx.accumulate,
            dg.accumulate | MTKC_LN_DEFER_PARAMS, part.dev(), (size_t)part.size() * sizeof(float),
            dev.stream()));
        g.deferLnParams(dg.ptr, db.ptr, part.devc(), blocks, d, dg.accumulate);
        return;
      }
      float* w = dev.scratch(mtkc_layernorm_stats_workspace_bytes(rows, d));
      MTKC(mtkc_layernorm_stats_backward(go, g.valPtr(n.inputs[0]), g.valPtr(n.inputs[1]),
                                         cache->mean.devc(), cache->invStd.devc(), dx.ptr, dg.ptr,
                                         db.ptr, rows, d, dx.accumulate, dg.accumulate, w,
                                         dev.scratchBytes(), dev.stream()));
      return;
    }
    if(cache->fast) {  // misaligned gradient buffers: materialise xhat for the generic kernel
      throw ContractError("layer norm backward: gradient rows not 16-byte aligned");
    }
    size_t ws = (size_t)((rows + 63) / 64) * 2 * (size_t)d * sizeof(float);
    float* w = dev.scratch(ws);
    MTKC(mtkc_layernorm_backward(go, g.valPtr(n.inputs[1]), cache->invStd.devc(),
                                 cache->xhat.devc(), dx.ptr, dg.ptr, db.ptr, rows, d,
                                 dx.accumulate, dg.accumulate, w, dev.scratchBytes(),
                                 dev.stream()));
  };
  return addNode(std::move(n));
}

// ---------------------------------------------------------------- embed

namespace {
struct EmbedAux {
  std::shared_ptr<DeviceBuffer> ids;
  int64_t off = 0;
  ScatterPlan plan;
  // folded positional encoding (scaleAddConst on a fresh embedding):
  // out = E[id] * scale + pe[pos], gradient scattered as scale * go
  float scale = 1.f;
  std::shared_ptr<Tensor> pe;
  int64_t t = 1;
};
}  // namespace

NodeRef ExpressionGraph::embed(NodeRef table, const IntMat& ids) {
  checkRef(table);
  if(table.shape.rank() != 2)
    throw DimensionError("embedding table must be rank 2, got " + table.shape.str());
  int64_t vocab = table.shape[0], e = table.shape[1];
  for(int32_t id : ids.data)
    if(id < 0 || id >= vocab)
      throw DataError("token id " + std::to_string(id) + " out of vocabulary of size " +
                      std::to_string(vocab));
  Node n;
  n.op = "embed";
  n.shape = Shape({ids.rows, ids.cols, e});
  n.inputs = {table.index};
  auto aux = std::make_shared<EmbedAux>();
  aux->ids = uploadIntsTo(*this, ids.data, &aux->off);
  if(!inference_)
    aux->plan = makeScatterPlan(*this, ids.data);
  n.aux = aux;
  int64_t cnt = ids.size();
  n.fwd = [aux, cnt, e, vocab](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_embed(n.value.dev(), g.valPtr(n.inputs[0]), (const int32_t*)aux->ids->ptr + aux->off,
                    cnt, e, vocab, aux->scale, aux->pe ? aux->pe->devc() : nullptr, aux->t,
                    Device::get().flags(), stream()));
  };
  n.bwd = [aux, e, vocab](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    float* dst = accPtr(g, n.inputs[0], vocab * e);
    scatterPlanAdd(g, aux->plan, dst, go, e, aux->scale);
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::embedPositions(NodeRef table, const std::vector<int32_t>& ids,
                                        const std::vector<int32_t>& pos, Real s,
                                        const Tensor& pe) {
  checkRef(table);
  if(table.shape.rank() != 2 || ids.size() != pos.size() || pe.shape().rank() != 2 ||
     pe.shape()[1] != table.shape[1])
    throw DimensionError("embedPositions shapes");
  const int64_t vocab = table.shape[0], e = table.shape[1], cnt = (int64_t)ids.size();
  for(size_t i = 0; i < ids.size(); ++i) {
    if(ids[i] < 0 || ids[i] >= vocab)
      throw DataError("token id " + std::to_string(ids[i]) + " out of vocabulary of size " +
                      std::to_string(vocab));
    if(pos[i] < 0 || pos[i] >= pe.shape()[0])
      throw ContractError("embedPositions: position out of the table");
  }
  Node n;
  n.op = "embedPositions";
  n.shape = Shape({cnt, e});
  n.inputs = {table.index};
  auto aux = std::make_shared<EmbedAux>();
  aux->ids = uploadIntsTo(*this, ids, &aux->off);
  int64_t posOff = 0;
  auto posBuf = uploadIntsTo(*this, pos, &posOff);
  if(!inference_)
    aux->plan = makeScatterPlan(*this, ids);
  aux->scale = s;
  aux->pe = sharedConst(pe);
  n.aux = aux;
  n.fwd = [aux, posBuf, posOff, cnt, e, vocab](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_embed_pos(n.value.dev(), g.valPtr(n.inputs[0]), (const int32_t*)aux->ids->ptr + aux->off,
                        (const int32_t*)posBuf->ptr + posOff, cnt, e, vocab, aux->scale,
                        aux->pe->devc(), Device::get().flags(), stream()));
  };
  n.bwd = [aux, e, vocab](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    float* dst = accPtr(g, n.inputs[0], vocab * e);
    scatterPlanAdd(g, aux->plan, dst, go, e, aux->scale);
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::scaleAddConst(NodeRef x, Real s, const Tensor& pe) {
  checkRef(x);
  if(x.shape.size() % pe.size() != 0)
    throw DimensionError("shapes not broadcastable: " + x.shape.str() + " vs " + pe.shape().str());
  // x * s + pe on an embedding nobody has consumed yet: fold into the gather
  // (one kernel forward, the scale into the scatter backward; same roundings:
  // s * E[id] then + pe, and s * go per position before the scatter sum)
  Node& xn = nodes_[(size_t)x.index];
  if(xn.op == "embed" && x.index == (int)nodes_.size() - 1 && (size_t)x.index >= computed_ &&
     xn.alias < 0 && x.shape.rank() == 3 && pe.shape().rank() == 2 &&
     pe.shape()[0] == x.shape[1] && pe.shape()[1] == x.shape[2]) {
    auto ea = std::static_pointer_cast<EmbedAux>(xn.aux);
    if(ea->scale == 1.f && !ea->pe) {
      ea->scale = s;
      ea->pe = sharedConst(pe);
      ea->t = x.shape[1];
      xn.op = "embedPosenc";
      return x;
    }
  }
  Node n;
  n.op = "posenc";
  n.shape = x.shape;
  n.inputs = {x.index};
  auto c = sharedConst(pe);
  n.aux = c;
  int64_t period = pe.size();
  n.fwd = [c, s, period](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_scale_add_periodic(n.value.dev(), g.valPtr(n.inputs[0]), s, c->devc(),
                                 n.value.size(), period, stream()));
  };
  n.bwd = [s](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    auto d = g.gradDst(n.inputs[0]);
    if(d.accumulate)
      MTKC(mtkc_axpy(d.ptr, go, s, n.shape.size(), stream()));
    else
      MTKC(mtkc_scale_shift(d.ptr, go, s, 0.f, n.shape.size(), stream()));
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::maskBlend(NodeRef a, NodeRef b, const Tensor& m) {
  checkRef(a);
  checkRef(b);
  if(a.shape != b.shape || a.shape.rank() != 2 || m.size() != a.shape[0])
    throw DimensionError("maskBlend shapes: " + a.shape.str() + " " + b.shape.str() + " " +
                         m.shape().str());
  Node n;
  n.op = "maskBlend";
  n.shape = a.shape;
  n.inputs = {a.index, b.index};
  auto dm = sharedConst(m);
  n.aux = dm;
  int64_t rows = a.shape[0], cols = a.shape[1];
  n.fwd = [dm, rows, cols](ExpressionGraph& g, Node& n) {
    MTKC(mtkc_mask_blend(n.value.dev(), g.valPtr(n.inputs[0]), g.valPtr(n.inputs[1]), dm->devc(),
                         rows, cols, stream()));
  };
  n.bwd = [dm, rows, cols](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    auto da = g.gradDst(n.inputs[0]);
    auto db = g.gradDst(n.inputs[1]);
    MTKC(mtkc_mask_blend_backward(da.ptr, db.ptr, go, dm->devc(), rows, cols, da.accumulate,
                                  db.accumulate, stream()));
  };
  return addNode(std::move(n));
}

// ------------------------------------------------------------ attention

namespace {
struct AttAux {
  Tensor probs, mask;
  bool hasMask = false;
};
}  // namespace

NodeRef ExpressionGraph::attention(NodeRef q, NodeRef k, NodeRef v, const Tensor& keyMask,
                                   bool causal, int heads) {
  checkRef(q);
  checkRef(k);
  checkRef(v);
  if(q.shape.rank() != 3 || k.shape.rank() != 3 || v.shape != k.shape)
    throw DimensionError("attention expects q [b,tq,d], k/v [b,tk,d]");
  int64_t b = q.shape[0], tq = q.shape[1], tk = k.shape[1], d = q.shape[2];
  if(k.shape[0] != b || k.shape[2] != d)
    throw DimensionError("attention q/k shapes disagree: " + q.shape.str() + " " + k.shape.str());
  if(d % heads != 0)
    throw DimensionError("model dim " + std::to_string(d) + " not divisible by heads " +
                         std::to_string(heads));
  int64_t dk = d / heads;
  // fully-masked query rows raise like softmaxInto (tensor.cpp:424-425)
  if(!keyMask.empty()) {
    if(keyMask.size() != b * tk)
      throw DimensionError("attention key mask must be [b x tk]");
    const Real* m = keyMask.data();
    for(int64_t bi = 0; bi < b; ++bi) {
      int64_t first = -1;
      for(int64_t j = 0; j < tk && first < 0; ++j)
        if(m[bi * tk + j] != 0)
          first = j;
      if(first < 0 || (causal && first > tk - tq))
        throw NumericError("softmax over a fully-masked row");
    }
  } else if(causal && tk < tq) {
    throw NumericError("softmax over a fully-masked row");
  }
  Node n;
  n.op = "attention";
  n.shape = q.shape;
  n.inputs = {q.index, k.index, v.index};
  auto aux = std::make_shared<AttAux>();
  if(!keyMask.empty()) {
    aux->mask = keyMask;  // shared device copy of the batch mask
    aux->hasMask = true;
  }
  n.aux = aux;
  float scale = (float)(1.0 / std::sqrt((double)dk));  // layers.cpp:106
  const bool tensorCore = Device::get().precision() == Precision::TF32 &&
                          mtkc_attention_tc_supported(tq, tk, dk) &&
                          std::getenv("MTK_ATTN_SIMT") == nullptr;
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    aux->probs = g.allocTensor(Shape({b, (int64_t)heads, tq, tk}));
    // TF32 mode: tensor-core kernels (mma.sync tf32); FP32 mode: the
    // CUDA-core kernels with the reference's summation order
    auto fn = tensorCore ? mtkc_attention_tc : mtkc_attention;
    MTKC(fn(n.value.dev(), d, aux->probs.dev(), g.valPtr(n.inputs[0]), d, g.valPtr(n.inputs[1]),
            g.valPtr(n.inputs[2]), d, aux->hasMask ? aux->mask.devc() : nullptr, b, tq, tk, heads,
            dk, scale, causal ? 1 : 0, Device::get().flags(), stream()));
  };
  n.bwd = [=](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    auto dq = g.gradDst(n.inputs[0]);
    auto dkk = g.gradDst(n.inputs[1]);
    auto dv = g.gradDst(n.inputs[2]);
    if(tensorCore) {
      MTKC(mtkc_attention_tc_backward(go, d, aux->probs.devc(), g.valPtr(n.inputs[0]), d,
                                      g.valPtr(n.inputs[1]), g.valPtr(n.inputs[2]), d, dq.ptr,
                                      dkk.ptr, dv.ptr, b, tq, tk, heads, dk, scale, dq.accumulate,
                                      dkk.accumulate, dv.accumulate, nullptr, stream()));
      return;
    }
    Tensor ds = g.allocTensor(Shape({b, (int64_t)heads, tq, tk}));
    MTKC(mtkc_attention_backward(go, d, aux->probs.devc(), g.valPtr(n.inputs[0]), d,
                                 g.valPtr(n.inputs[1]), g.valPtr(n.inputs[2]), d, dq.ptr, dkk.ptr,
                                 dv.ptr, ds.dev(), b, tq, tk, heads, dk, scale, dq.accumulate,
                                 dkk.accumulate, dv.accumulate, stream()));
  };
  return addNode(std::move(n));
}

std::shared_ptr<RowPacking> RowPacking::fromMask(const Tensor& mask) {
  if(mask.empty() || mask.shape().rank() != 2)
    return nullptr;
  const int64_t b = mask.shape()[0], T = mask.shape()[1];
  const Real* m = mask.data();
  auto p = std::make_shared<RowPacking>();
  p->b = b;
  p->T = T;
  p->off.assign((size_t)b + 1, 0);
  for(int64_t i = 0; i < b; ++i) {
    int64_t len = 0;
    while(len < T && m[i * T + len] != 0)
      ++len;
    for(int64_t t = len; t < T; ++t)
      if(m[i * T + t] != 0)
        return nullptr;  // not a prefix
    if(len == 0)
      return nullptr;
    for(int64_t t = 0; t < len; ++t)
      p->rows.push_back(i * T + t);
    p->off[(size_t)i + 1] = (int32_t)p->rows.size();
    p->maxLen = std::max(p->maxLen, len);
  }
  return p;
}

namespace {
// attentionPacked body: k/v columns [kCol, kCol+d) / [vCol, vCol+d) of rows
// with stride ldk (kvShared: k and v are the same wide node)
NodeRef attentionPackedImpl(ExpressionGraph& g, NodeRef q, NodeRef k, NodeRef v, int64_t kCol,
                            int64_t vCol, int64_t ldk, bool kvShared,
                            const std::shared_ptr<const RowPacking>& qp,
                            const std::shared_ptr<const RowPacking>& kp, bool causal, int heads) {
  using Node = ExpressionGraph::Node;
  const int64_t d = q.shape[1], b = qp->b, tq = qp->maxLen, tk = kp->maxLen;
  if(d % heads != 0)
    throw DimensionError("model dim not divisible by heads");
  const int64_t dk = d / heads;
  if(Device::get().precision() != Precision::TF32 || !mtkc_attention_tc_supported(tq, tk, dk))
    throw ContractError("attentionPacked: needs the TF32 tensor-core attention path");
  for(const RowPacking* rp : {qp.get(), kp.get()})
    if(!rp->dev)
      rp->dev = uploadIntsTo(g, rp->off, &rp->devOff);
  Node n;
  n.op = "attentionPacked";
  n.shape = q.shape;
  n.inputs = kvShared ? std::vector<int>{q.index, k.index} : std::vector<int>{q.index, k.index, v.index};
  auto aux = std::make_shared<AttAux>();
  n.aux = aux;
  const float scale = (float)(1.0 / std::sqrt((double)dk));  // layers.cpp:106
  std::shared_ptr<const RowPacking> QP = qp, KP = kp;
  // sentences bucketed by tile size (16/32/48/64 rows): one launch per
  // non-empty bucket, each with the smallest tile its sentences fit
  struct Bucket {
    int64_t tile, off, n;
  };
  std::vector<Bucket> buckets;
  std::vector<int32_t> ids;
  for(int64_t tile : {16, 32, 48, 64}) {
    const int64_t off = (int64_t)ids.size();
    for(int64_t i = 0; i < b; ++i) {
      const int64_t L = std::max(qp->off[(size_t)i + 1] - qp->off[(size_t)i],
                                 kp->off[(size_t)i + 1] - kp->off[(size_t)i]);
      if(L <= tile && L > tile - 16)
        ids.push_back((int32_t)i);
    }
    if((int64_t)ids.size() > off)
      buckets.push_back(Bucket{tile, off, (int64_t)ids.size() - off});
  }
  int64_t idsOff = 0;
  auto idsBuf = uploadIntsTo(g, ids, &idsOff);
  const int vSlot = kvShared ? 1 : 2;
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    aux->probs = g.allocTensor(Shape({b, (int64_t)heads, tq, tk}));
    for(const Bucket& bk : buckets)
      MTKC(mtkc_attention_tc_varlen_ids(
          n.value.dev(), d, aux->probs.dev(), g.valPtr(n.inputs[0]), d,
          g.valPtr(n.inputs[1]) + kCol, g.valPtr(n.inputs[(size_t)vSlot]) + vCol, ldk,
          (const int32_t*)QP->dev->ptr + QP->devOff, (const int32_t*)KP->dev->ptr + KP->devOff,
          (const int32_t*)idsBuf->ptr + idsOff + bk.off, bk.n, bk.tile, b, tq, tk, heads, dk,
          scale, causal ? 1 : 0, Device::get().flags(), stream()));
  };
  n.bwd = [=](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    auto dq = g.gradDst(n.inputs[0]);
    auto dkk = g.gradDst(n.inputs[1]);
    // shared wide node: this node's k / v columns are written by it alone
    auto dv = kvShared ? dkk : g.gradDst(n.inputs[2]);
    const int accK = kvShared ? 0 : dkk.accumulate, accV = kvShared ? 0 : dv.accumulate;
    for(const Bucket& bk : buckets)  // disjoint rows: every launch keeps the accumulate flags
      MTKC(mtkc_attention_tc_varlen_ids_backward(
          go, d, aux->probs.devc(), g.valPtr(n.inputs[0]), d, g.valPtr(n.inputs[1]) + kCol,
          g.valPtr(n.inputs[(size_t)vSlot]) + vCol, ldk, dq.ptr, dkk.ptr + kCol, dv.ptr + vCol,
          (const int32_t*)QP->dev->ptr + QP->devOff, (const int32_t*)KP->dev->ptr + KP->devOff,
          (const int32_t*)idsBuf->ptr + idsOff + bk.off, bk.n, bk.tile, b, tq, tk, heads, dk,
          scale, dq.accumulate, accK, accV, stream()));
  };
  return g.addNode(std::move(n));
}
}  // namespace

NodeRef ExpressionGraph::attentionPacked(NodeRef q, NodeRef k, NodeRef v,
                                         const std::shared_ptr<const RowPacking>& qp,
                                         const std::shared_ptr<const RowPacking>& kp,
                                         bool causal, int heads) {
  checkRef(q);
  checkRef(k);
  checkRef(v);
  if(!qp || !kp || qp->b != kp->b)
    throw ContractError("attentionPacked: packings of different batches");
  if(q.shape.rank() != 2 || k.shape.rank() != 2 || v.shape != k.shape ||
     q.shape[0] != qp->n() || k.shape[0] != kp->n() || q.shape[1] != k.shape[1])
    throw DimensionError("attentionPacked expects q [nq,d], k/v [nk,d]: " + q.shape.str() +
                         " " + k.shape.str());
  return attentionPackedImpl(*this, q, k, v, 0, 0, q.shape[1], false, qp, kp, causal, heads);
}

NodeRef ExpressionGraph::attentionPacked(NodeRef q, NodeRef kv, int64_t kCol, int64_t vCol,
                                         const std::shared_ptr<const RowPacking>& qp,
                                         const std::shared_ptr<const RowPacking>& kp,
                                         bool causal, int heads) {
  checkRef(q);
  checkRef(kv);
  if(!qp || !kp || qp->b != kp->b)
    throw ContractError("attentionPacked: packings of different batches");
  const int64_t d = q.shape.back();
  if(q.shape.rank() != 2 || kv.shape.rank() != 2 || q.shape[0] != qp->n() ||
     kv.shape[0] != kp->n() || kCol < 0 || vCol < 0 || kCol + d > kv.shape[1] ||
     vCol + d > kv.shape[1])
    throw DimensionError("attentionPacked: q " + q.shape.str() + " kv " + kv.shape.str());
  return attentionPackedImpl(*this, q, kv, kv, kCol, vCol, kv.shape[1], true, qp, kp, causal,
                             heads);
}

NodeRef ExpressionGraph::affineMulti(NodeRef x, const std::vector<NodeRef>& Ws,
                                     const std::vector<NodeRef>& bs) {
  checkRef(x);
  if(Ws.empty() || Ws.size() != bs.size() || Ws.size() > MTKC_COPY_MAX_JOBS / 2)
    throw ContractError("affineMulti: 1..16 weight/bias pairs");
  const int64_t K = x.shape.back(), rows = x.shape.size() / K;
  std::vector<int64_t> cols, offs;
  int64_t N = 0;
  for(size_t i = 0; i < Ws.size(); ++i) {
    checkRef(Ws[i]);
    checkRef(bs[i]);
    if(Ws[i].shape.rank() != 2 || Ws[i].shape[0] != K || bs[i].shape.size() != Ws[i].shape[1])
      throw DimensionError("affineMulti: W " + Ws[i].shape.str() + " b " + bs[i].shape.str());
    offs.push_back(N);
    cols.push_back(Ws[i].shape[1]);
    N += Ws[i].shape[1];
  }
  std::vector<int64_t> dims = x.shape.dims();
  dims.back() = N;
  Node n;
  n.op = "affineMulti";
  n.shape = Shape(dims);
  n.inputs = {x.index};
  for(auto& w : Ws)
    n.inputs.push_back(w.index);
  for(auto& b : bs)
    n.inputs.push_back(b.index);
  struct MultiAux {
    Tensor wcat, bcat;
  };
  auto aux = std::make_shared<MultiAux>();
  n.aux = aux;
  const int64_t P = (int64_t)Ws.size();
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    aux->wcat = g.allocTensor(Shape({K, N}));
    aux->bcat = g.allocTensor(Shape({N}));
    std::vector<mtkc_copy_job> jobs;
    for(int64_t i = 0; i < P; ++i) {  // [W_0|W_1|..] and [b_0|b_1|..]
      jobs.push_back(mtkc_copy_job{g.valPtr(n.inputs[(size_t)(1 + i)]), aux->wcat.dev() + offs[(size_t)i],
                                   K, cols[(size_t)i], cols[(size_t)i], N, 0});
      jobs.push_back(mtkc_copy_job{g.valPtr(n.inputs[(size_t)(1 + P + i)]),
                                   aux->bcat.dev() + offs[(size_t)i], 1, cols[(size_t)i],
                                   cols[(size_t)i], N, 0});
    }
    MTKC(mtkc_copy_many(jobs.data(), (int)jobs.size(), stream()));
    gemm(rows, N, K, g.valPtr(n.inputs[0]), K, false, aux->wcat.devc(), N, false, n.value.dev(),
         N, 0.f, aux->bcat.devc());
  };
  n.bwd = [=](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    if(g.node(g.resolve(n.inputs[0])).needsGrad) {  // dx (+)= dY [W..]^T
      auto dx = g.gradDst(n.inputs[0]);
      gemm(rows, K, N, go, N, false, aux->wcat.devc(), N, true, dx.ptr, K,
           dx.accumulate ? 1.f : 0.f);
    }
    // d[W..] = x^T dY with the bias gradients as its operand sums, then
    // scattered to the parameters
    Tensor dw = g.allocTensor(Shape({K, N}));
    Tensor db = g.allocTensor(Shape({N}));
    gemm(K, N, rows, g.valPtr(n.inputs[0]), K, true, go, N, false, dw.dev(), N, 0.f, nullptr,
         MTKC_EPI_NONE, nullptr, 1, 0, 0, 0, db.dev(), MTKC_COLSUM_B, 0);
    std::vector<mtkc_copy_job> jobs;
    for(int64_t i = 0; i < P; ++i) {
      auto gw = g.gradDst(n.inputs[(size_t)(1 + i)]);
      auto gb = g.gradDst(n.inputs[(size_t)(1 + P + i)]);
      jobs.push_back(mtkc_copy_job{dw.devc() + offs[(size_t)i], gw.ptr, K, cols[(size_t)i], N,
                                   cols[(size_t)i], gw.accumulate});
      jobs.push_back(mtkc_copy_job{db.devc() + offs[(size_t)i], gb.ptr, 1, cols[(size_t)i], N,
                                   cols[(size_t)i], gb.accumulate});
    }
    MTKC(mtkc_copy_many(jobs.data(), (int)jobs.size(), stream()));
  };
  return addNode(std::move(n));
}

// ------------------------------------------------------------- LSTM cell

namespace {
struct LstmAux {
  Tensor pre, cache;
};
}  // namespace

NodeRef ExpressionGraph::lstmCell(NodeRef x, NodeRef h, NodeRef c, NodeRef W, NodeRef U,
                                  NodeRef bias) {
  for(const NodeRef* r : {&x, &h, &c, &W, &U, &bias})
    checkRef(*r);
  const int64_t b = h.shape[0], d = h.shape.back(), in = x.shape.back();
  if(h.shape.rank() != 2 || c.shape != h.shape || x.shape.rank() != 2 || x.shape[0] != b ||
     W.shape != Shape({in, 4 * d}) || U.shape != Shape({d, 4 * d}) || bias.shape.size() != 4 * d)
    throw DimensionError("lstmCell shapes: x " + x.shape.str() + " h " + h.shape.str() + " c " +
                         c.shape.str() + " W " + W.shape.str() + " U " + U.shape.str());
  Node n;
  n.op = "lstmCell";
  n.shape = Shape({b, 2 * d});
  n.inputs = {x.index, h.index, c.index, W.index, U.index, bias.index};
  auto aux = std::make_shared<LstmAux>();
  n.aux = aux;
  n.fwd = [=](ExpressionGraph& g, Node& n) {
    aux->pre = g.allocTensor(Shape({b, 4 * d}));
    aux->cache = g.allocTensor(Shape({b, 5 * d}));
    float* pre = aux->pre.dev();
    // h*U first, then x*W accumulated into the same buffer (gruPre's order)
    gemm(b, 4 * d, d, g.valPtr(n.inputs[1]), d, false, g.valPtr(n.inputs[4]), 4 * d, false, pre,
         4 * d, 0.f);
    gemm(b, 4 * d, in, g.valPtr(n.inputs[0]), in, false, g.valPtr(n.inputs[3]), 4 * d, false, pre,
         4 * d, 1.f);
    MTKC(mtkc_lstm_forward(pre, g.valPtr(n.inputs[5]), g.valPtr(n.inputs[2]), n.value.dev(),
                           aux->cache.dev(), b, d, stream()));
  };
  n.bwd = [=](ExpressionGraph& g, Node& n) {
    const float* go = g.gradSrc(n);
    Tensor dpre = g.allocTensor(Shape({b, 4 * d}));
    const bool needC = g.node(g.resolve(n.inputs[2])).needsGrad;
    ExpressionGraph::GradDst dc{};
    if(needC)
      dc = g.gradDst(n.inputs[2]);
    MTKC(mtkc_lstm_backward(go, aux->cache.devc(), g.valPtr(n.inputs[2]), dpre.dev(),
                            needC ? dc.ptr : nullptr, needC ? dc.accumulate : 0, b, d, stream()));
    const float* dp = dpre.devc();
    auto want = [&](int slot) { return g.node(g.resolve(n.inputs[(size_t)slot])).needsGrad; };
    if(want(0)) {  // dx += dpre W^T
      auto dx = g.gradDst(n.inputs[0]);
      gemm(b, in, 4 * d, dp, 4 * d, false, g.valPtr(n.inputs[3]), 4 * d, true, dx.ptr, in,
           dx.accumulate ? 1.f : 0.f);
    }
    if(want(1)) {  // dh += dpre U^T
      auto dh = g.gradDst(n.inputs[1]);
      gemm(b, d, 4 * d, dp, 4 * d, false, g.valPtr(n.inputs[4]), 4 * d, true, dh.ptr, d,
           dh.accumulate ? 1.f : 0.f);
    }
    if(want(3)) {  // dW += x^T dpre
      auto dW = g.gradDst(n.inputs[3]);
      gemm(in, 4 * d, b, g.valPtr(n.inputs[0]), in, true, dp, 4 * d, false, dW.ptr, 4 * d,
           dW.accumulate ? 1.f : 0.f);
    }
    if(want(4)) {  // dU += h^T dpre
      auto dU = g.gradDst(n.inputs[4]);
      gemm(d, 4 * d, b, g.valPtr(n.inputs[1]), d, true, dp, 4 * d, false, dU.ptr, 4 * d,
           dU.accumulate ? 1.f : 0.f);
    }
    if(want(5)) {  // db += colsum(dpre)
      auto db = g.gradDst(n.inputs[5]);
      Device& dev = Device::get();
      MTKC(mtkc_colsum(db.ptr, dp, b, 4 * d, db.accumulate, dev.scratch(64 << 20),
                       dev.scratchBytes(), stream()));
    }
  };
  return addNode(std::move(n));
}

NodeRef ExpressionGraph::lstmState(NodeRef cell) {
  return slice(cell, 1, 0, cell.shape[1] / 2);
}

NodeRef ExpressionGraph::lstmCellState(NodeRef cell) {
  return slice(cell, 1, cell.shape[1] / 2, cell.shape[1] / 2);
}

// -------------------------------------------------------------- dropout


NodeRef ExpressionGraph::dropoutMask(const Shape& shape, Real p) {
  if(p >= Real(1) || p < Real(0))
    throw ContractError("dropout probability must be in [0, 1)");
  if(!inference_ && p != Real(0) && Device::get().deviceDropout()) {
    // throughput mode: the mask is generated on the device from one draw of
    // the graph RNG (kernels/dropout.cu), nothing is uploaded
    const uint64_t key = rng_();
    Node n;
    n.op = "dropoutMask";
    n.shape = shape;
    n.fwd = [key, p](ExpressionGraph&, Node& n) {
      MTKC(mtkc_dropout_mask(n.value.dev(), n.value.size(), (float)p, key, stream()));
    };
    return addNode(std::move(n));
  }
  Tensor mask(shape);
  if(inference_ || p == Real(0)) {
    mask.fill(1);
  } else {
    std::uniform_real_distribution<double> u(0.0, 1.0);
    Real keepInv = Real(1) / (Real(1) - p);
    Real* m = mask.data();
    for(int64_t i = 0; i < mask.size(); ++i)
      m[i] = u(rng_) >= (double)p ? keepInv : Real(0);
  }
  return constant(mask);
}

NodeRef ExpressionGraph::dropout(NodeRef x, Real p, int variationalAxis) {
  checkRef(x);
  if(p >= Real(1) || p < Real(0))
    throw ContractError("dropout probability must be in [0, 1)");
  if(inference_ || p == Real(0))
    return x;
  std::vector<int64_t> dims = x.shape.dims();
  if(variationalAxis >= 0) {
    if(variationalAxis >= x.shape.rank())
      throw ContractError("variational axis out of range");
    dims[(size_t)variationalAxis] = 1;
  }
  if(Device::get().deviceDropout()) {
    // y = x * m with m recomputed from (key, mask index) forward and backward
    const uint64_t key = rng_();
    const int axis = variationalAxis;
    int64_t inner = 1, axisLen = 1;
    if(axis >= 0) {
      axisLen = x.shape[axis];
      for(int i = axis + 1; i < x.shape.rank(); ++i)
        inner *= x.shape[i];
    }
    Node n;
    n.op = "dropout";
    n.shape = x.shape;
    n.inputs = {x.index};
    n.aux = std::make_shared<DropoutAux>(DropoutAux{key, (float)p, inner, axisLen});
    n.fwd = [](ExpressionGraph& g, Node& n) {
      auto* a = static_cast<DropoutAux*>(n.aux.get());
      MTKC(mtkc_dropout(n.value.dev(), g.valPtr(n.inputs[0]), nullptr, n.value.size(), a->inner,
                        a->axisLen, a->p, a->key, stream()));
    };
    n.bwd = [](ExpressionGraph& g, Node& n) {
      auto* a = static_cast<DropoutAux*>(n.aux.get());
      const float* go = g.gradSrc(n);
      auto d = g.gradDst(n.inputs[0]);
      MTKC(mtkc_dropout_backward(d.ptr, go, n.shape.size(), a->inner, a->axisLen, a->p, a->key,
                                 d.accumulate, stream()));
    };
    return addNode(std::move(n));
  }
  NodeRef mask = dropoutMask(Shape(dims), p);
  return mul(x, mask);
}

// -------------------------------------------------------- cross entropy

namespace {
struct CeAux {
  std::shared_ptr<DeviceBuffer> tg;
  int64_t tgOff = 0;
  Tensor mask, stats, rowLoss;
  bool hasMask = false;
  Real count = 0;
  // fused forward+backward (crossEntropyFused): the gradient replaced the
  // logits in the forward, for this loss seed
  bool fused = false;
  Real scale = 1;
};
}  // namespace

NodeRef ExpressionGraph::crossEntropy(NodeRef logits, const IntMat& targets, const Tensor& mask) {
  return crossEntropy(logits, targets, mask, false);
}

NodeRef ExpressionGraph::crossEntropy(NodeRef logits, const IntMat& targets, const Tensor& mask,
                                      bool fusedBackward) {
  checkRef(logits);
  int64_t vocab = logits.shape.back();
  int64_t positions = logits.shape.size() / vocab;
  if(targets.size() != positions)
    throw DimensionError("cross entropy target count mismatch");
  if(!mask.empty() && mask.size() != positions)
    throw DimensionError("cross entropy mask count mismatch");
  for(int32_t id : targets.data)
    if(id < 0 || id >= vocab)
      throw DataError("target id " + std::to_string(id) + " out of vocabulary of size " +
                      std::to_string(vocab));
  auto aux = std::make_shared<CeAux>();
  aux->tg = uploadIntsTo(*this, targets.data, &aux->tgOff);
  Real count = 0;
  if(mask.empty()) {
    count = (Real)positions;
  } else {
    const Real* m = mask.data();
    for(int64_t r = 0; r < positions; ++r)  // graph.cpp:898-902 (sum of m in row order)
      if(m[r] != Real(0))
        count += m[r];
    aux->mask = mask;  // shared device copy of the batch mask
    aux->hasMask = true;
  }
  aux->count = count;
  Node n;
  n.op = "crossEntropy";
  n.shape = Shape({1});
  n.inputs = {logits.index};
  n.aux = aux;
  // Fused path (TF32 training, the logits' only consumer is this loss and the
  // loss is the backward root): one pass writes the loss AND the gradient
  // over the logits for the graph's current loss seed.
  aux->fused = fusedBackward && Device::get().precision() == Precision::TF32 &&
               mtkc_xent_fused_supported(vocab) && !inference_ &&
               !nodes_[(size_t)resolve(logits.index)].isParam;
  aux->scale = lossScale_;
  n.fwd = [aux, vocab, positions](ExpressionGraph& g, Node& n) {
    if(aux->count == Real(0))
      throw ContractError("cross entropy over a fully-masked batch");
    aux->stats = g.allocTensor(Shape({positions, 2}));
    aux->rowLoss = g.allocTensor(Shape({positions}));
    if(aux->fused) {
      Node& L = g.node(g.resolve(n.inputs[0]));
      MTKC(mtkc_xent_fused(L.value.dev(), (const int32_t*)aux->tg->ptr + aux->tgOff,
                           aux->hasMask ? aux->mask.devc() : nullptr, positions, vocab,
                           (float)aux->scale, aux->rowLoss.dev(), n.value.dev(), aux->count,
                           stream()));
      return;
    }
    // TF32 mode: the one-pass kernels (the FP32 path keeps the reference's order)
    const bool fast = Device::get().precision() == Precision::TF32;
    MTKC((fast ? mtkc_xent_forward_fast : mtkc_xent_forward)(g.valPtr(n.inputs[0]), (const int32_t*)aux->tg->ptr + aux->tgOff,
                           aux->hasMask ? aux->mask.devc() : nullptr, positions, vocab,
                           aux->stats.dev(), aux->rowLoss.dev(), n.value.dev(), aux->count,
                           stream()));
  };
  n.bwd = [aux, vocab, positions](ExpressionGraph& g, Node& n) {
    if(aux->fused) {  // the logits buffer already holds their gradient
      Node& L = g.node(g.resolve(n.inputs[0]));
      if(g.lossScale() != aux->scale || L.gradLive || !L.grad.empty())
        throw ContractError("fused cross entropy: the loss seed changed or the logits have "
                            "other consumers");
      L.grad = L.value;
      L.gradLive = true;
      return;
    }
    const float* go = g.gradSrc(n);
    auto d = g.gradDst(n.inputs[0]);
    const bool fast = Device::get().precision() == Precision::TF32;
    MTKC((fast ? mtkc_xent_backward_fast : mtkc_xent_backward)(d.ptr, g.valPtr(n.inputs[0]), aux->stats.devc(),
                            (const int32_t*)aux->tg->ptr + aux->tgOff,
                            aux->hasMask ? aux->mask.devc() : nullptr, go, positions, vocab,
                            aux->count, d.accumulate, stream()));
  };
  return addNode(std::move(n));
}

// ------------------------------------------------------------ execution

void ExpressionGraph::forward() {
  for(size_t i = computed_; i < nodes_.size(); ++i) {
    Node& n = nodes_[i];
    if(n.alias >= 0) {
      Node& root = nodes_[(size_t)resolve((int)i)];
      n.value = root.value.reshaped(n.shape);
      continue;
    }
    if(n.fwd) {
      if(n.value.empty())
        n.value = allocTensor(n.shape);
      n.fwd(*this, n);
      if(checkFinite_) {
        Device& d = Device::get();
        MTKC(mtkc_check_finite(n.value.devc(), n.value.size(), d.flags(), d.stream()));
        try {
          d.checkFlags("op " + n.op);
        } catch(const NumericError&) {
          throw NumericError("non-finite value produced by op '" + n.op + "' (node " +
                             std::to_string(i) + ")");
        }
      }
    }
  }
  computed_ = nodes_.size();
}

void ExpressionGraph::backward(NodeRef loss) { backward(loss, nullptr); }

void ExpressionGraph::backward(NodeRef loss, const std::function<void(int)>& afterNode) {
  checkRef(loss);
  ++backwardCount_;
  if(inference_)
    throw ContractError("backward() called on an inference-mode graph");
  if(loss.shape.size() != 1)
    throw ContractError("loss must be scalar-shaped, got " + loss.shape.str());
  if(computed_ < nodes_.size())
    forward();
  for(auto& n : nodes_)
    if(!n.isParam) {
      n.gradLive = false;
      n.gradGated = true;
    }
  {
    auto d = gradDst(loss.index);
    MTKC(mtkc_fill(d.ptr, lossScale_, 1, stream()));
  }
  static const bool noDefer = getenv("MTK_LN_NODEFER") != nullptr;
  lnPending_.clear();  // a sweep that threw leaves nothing behind
  lnDefer_ = !afterNode && !noDefer;
  for(int i = loss.index; i >= 0; --i) {
    Node& n = nodes_[(size_t)i];
    if(!(n.alias >= 0 || !n.bwd || !n.gradLive || !n.needsGrad))
      n.bwd(*this, n);
    if(afterNode)
      afterNode(i);
  }
  flushLnParams();
  lnDefer_ = false;
}

void ExpressionGraph::deferLnParams(float* dgain, float* dbias, const float* partials,
                                    int64_t blocks, int64_t d, int accumulate) {
  lnPending_.push_back({dgain, dbias, partials, blocks, d, accumulate});
  if(lnPending_.size() >= 32)
    flushLnParams();
}

void ExpressionGraph::flushLnParams() {
  if(lnPending_.empty())
    return;
  std::vector<mtkc_ln_param_job> jobs;
  jobs.reserve(lnPending_.size());
  for(const auto& p : lnPending_)
    jobs.push_back({p.dgain, p.dbias, p.partials, p.blocks, p.d, p.accumulate});
  lnPending_.clear();
  MTKC(mtkc_layernorm_param_reduce_many(jobs.data(), (int)jobs.size(), stream()));
}

std::vector<ExpressionGraph::GradBucket> ExpressionGraph::gradBuckets(int64_t targetElems) const {
  // lowest consumer index per (alias-resolved) node
  std::vector<int> firstUse(nodes_.size(), INT_MAX);
  for(size_t i = 0; i < nodes_.size(); ++i)
    for(int in : nodes_[i].inputs) {
      int r = resolve(in);
      firstUse[(size_t)r] = std::min(firstUse[(size_t)r], (int)i);
    }
  struct P {
    int64_t off;
    int ready;
  };
  std::vector<P> ps;
  for(auto& [name, p] : params_) {
    auto it = paramNode_.find(name);
    int ready = it == paramNode_.end() ? INT_MAX : firstUse[(size_t)it->second];
    ps.push_back({p.offset, ready});
  }
  std::sort(ps.begin(), ps.end(), [](const P& a, const P& b) { return a.off < b.off; });
  std::vector<GradBucket> out;
  const int64_t used = pool_.used();
  for(size_t k = 0; k < ps.size();) {
    GradBucket b{ps[k].off, 0, INT_MAX};
    size_t j = k;
    for(; j < ps.size(); ++j) {
      int64_t next = j + 1 < ps.size() ? ps[j + 1].off : used;
      b.readyAfter = std::min(b.readyAfter, ps[j].ready);
      b.end = next;
      if(b.end - b.begin >= targetElems) {
        ++j;
        break;
      }
    }
    if(k == 0)
      b.begin = 0;
    out.push_back(b);
    k = j;
  }
  return out;
}

void ExpressionGraph::realizeParamGradsRange(int64_t begin, int64_t end) {
  for(auto& [name, p] : params_)
    if(!p.gradLive && p.offset >= begin && p.offset < end) {
      p.grad.setZero();
      p.gradLive = true;
    }
}

void ExpressionGraph::clear() {
  nodes_.clear();
  paramNode_.clear();
  dotCache_.clear();
  computed_ = 0;
  ++generation_;
  arena_.reset();
}

Tensor& ExpressionGraph::paramValue(const std::string& name) {
  auto it = params_.find(name);
  if(it == params_.end())
    throw ContractError("unknown parameter: " + name);
  return it->second.value;
}

Tensor& ExpressionGraph::paramGrad(const std::string& name) {
  auto it = params_.find(name);
  if(it == params_.end())
    throw ContractError("unknown parameter: " + name);
  Param& p = it->second;
  if(!p.gradLive) {
    p.grad.setZero();
    p.gradLive = true;
  }
  return p.grad;
}

int64_t ExpressionGraph::paramOffset(const std::string& name) const {
  auto it = params_.find(name);
  if(it == params_.end())
    throw ContractError("unknown parameter: " + name);
  return it->second.offset;
}

void ExpressionGraph::zeroGrads() {
  for(auto& [name, p] : params_)
    p.gradLive = false;  // logically zero; the first contributor writes
}

void ExpressionGraph::syncParamViews() {
  // dev() uploads pending host edits and marks the host caches stale, so a
  // later host read sees what device-side updates (Adam, EMA apply) wrote
  for(auto& [name, p] : params_) {
    p.value.dev();
    if(p.gradLive)
      p.grad.dev();
  }
}

void ExpressionGraph::realizeParamGrads() {
  for(auto& [name, p] : params_)
    if(!p.gradLive) {
      p.grad.setZero();
      p.gradLive = true;
    }
}

}  // namespace mtk
