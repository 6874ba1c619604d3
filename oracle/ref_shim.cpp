// TEST INFRASTRUCTURE ONLY -- extern "C" shim over the UNMODIFIED reference
// (mtk, /root/reference/proj) so pytest and bench.py's CPU arm can drive it
// through ctypes.  Every entry point calls the reference's own public API;
// nothing here re-implements reference arithmetic.  Built by oracle/Makefile
// into oracle/_ref/libmtkref.so; the product library never links it.
//
// Entry points and the reference API they exercise:
//   ref_batches_make      -> makeBatches            (src/data.cpp:226-282)
//   ref_model_create      -> buildModel + registerParams (src/models.cpp:663-674, 728-745)
//   ref_loss_grads        -> buildLoss/forward/zeroGrads/backward (models.cpp:649-661,
//                            graph.cpp:928-967) -- one worker of trainSync (train.cpp:226-237)
//   ref_adam_update       -> Adam::update + AveragedParameters::update (train.cpp:49-79)
//   ref_train             -> train() / trainSync     (train.cpp:200-300, 408-420)
//   ref_matmul            -> matmulInto              (tensor.cpp:258-306)
//   ref_op_*              -> single graph ops with a seeded upstream gradient
#include "mtk/search.h"
#include "mtk/serialize.h"
#include "mtk/train.h"

#include <cctype>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

using namespace mtk;

namespace {
thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch(const DimensionError& e) {
    return fail(1, e.what());
  } catch(const NumericError& e) {
    return fail(2, e.what());
  } catch(const ContractError& e) {
    return fail(3, e.what());
  } catch(const DataError& e) {
    return fail(4, e.what());
  } catch(const IoError& e) {
    return fail(5, e.what());
  } catch(const std::exception& e) {
    return fail(6, e.what());
  }
}

struct RefExamples {
  std::vector<Example> ex;
};
struct RefBatches {
  std::vector<Batch> b;
};
struct RefModel {
  ModelConfig cfg;
  Model model;
  std::unique_ptr<ExpressionGraph> g;
  std::unique_ptr<Adam> adam;
  std::unique_ptr<AveragedParameters> avg;
};

Shape shapeOf(int rank, const int64_t* dims) {
  return Shape(std::vector<int64_t>(dims, dims + rank));
}

Tensor tensorOf(int rank, const int64_t* dims, const float* data) {
  Shape s = shapeOf(rank, dims);
  return Tensor(s, std::vector<Real>(data, data + s.size()));
}

// loss = sum(out * G): seeds d(out) = G exactly (graph.cpp:164-169 mul bwd,
// :489-505 sum bwd).
NodeRef seededLoss(ExpressionGraph& g, NodeRef out, const float* G) {
  NodeRef gc = g.constant(Tensor(out.shape, std::vector<Real>(G, G + out.shape.size())));
  NodeRef prod = g.mul(out, gc);
  return g.reduce(ReduceOp::Sum, g.reshape(prod, Shape({1, out.shape.size()})), 1);
}

void copyOut(const Tensor& t, float* dst) {
  if(dst)
    std::memcpy(dst, t.data(), sizeof(float) * (size_t)t.size());
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ------------------------------------------------------------- examples

void* ref_examples_create(int64_t n, const int32_t* srcTok, const int64_t* srcOff,
                          const int32_t* tgtTok, const int64_t* tgtOff) {
  auto* h = new RefExamples;
  h->ex.resize((size_t)n);
  for(int64_t i = 0; i < n; ++i) {
    Example& e = h->ex[(size_t)i];
    e.sources = {std::vector<int32_t>(srcTok + srcOff[i], srcTok + srcOff[i + 1])};
    if(tgtTok) {
      e.target.assign(tgtTok + tgtOff[i], tgtTok + tgtOff[i + 1]);
      e.hasTarget = true;
    }
    e.id = (size_t)i;
  }
  return h;
}

// extra source streams (ape-dual / custom multi-source models): stream s of
// example i is tokens [off[s*(n+1)+i], off[s*(n+1)+i+1]) of tok
void ref_examples_add_stream(void* h, int64_t n, const int32_t* tok, const int64_t* off) {
  auto* e = static_cast<RefExamples*>(h);
  for(int64_t i = 0; i < n; ++i)
    e->ex[(size_t)i].sources.emplace_back(tok + off[i], tok + off[i + 1]);
}

void ref_examples_free(void* h) { delete static_cast<RefExamples*>(h); }

// -------------------------------------------------------------- batches

void* ref_batches_make(void* ex, int64_t budget, uint64_t seed, int shuffle) {
  auto* h = new RefBatches;
  int rc = guard([&] {
    BatchOptions bo;
    bo.tokenBudget = budget;
    bo.seed = seed;
    bo.shuffle = shuffle != 0;
    h->b = makeBatches(static_cast<RefExamples*>(ex)->ex, bo);
  });
  if(rc) {
    delete h;
    return nullptr;
  }
  return h;
}

int64_t ref_batches_count(void* h) { return (int64_t)static_cast<RefBatches*>(h)->b.size(); }

// dims = {rows, srcCols, tgtCols}
void ref_batch_shape(void* h, int64_t i, int64_t* dims) {
  const Batch& b = static_cast<RefBatches*>(h)->b[(size_t)i];
  dims[0] = b.rows();
  dims[1] = b.sourceIds.empty() ? 0 : b.sourceIds[0].cols;
  dims[2] = b.hasTarget ? b.targetIds.cols : 0;
}

void ref_batch_get(void* h, int64_t i, int32_t* srcIds, float* srcMask, int32_t* tgtIds,
                   float* tgtMask, int64_t* sentIds) {
  const Batch& b = static_cast<RefBatches*>(h)->b[(size_t)i];
  if(!b.sourceIds.empty()) {
    std::memcpy(srcIds, b.sourceIds[0].data.data(), 4 * (size_t)b.sourceIds[0].size());
    copyOut(b.sourceMasks[0], srcMask);
  }
  if(b.hasTarget) {
    std::memcpy(tgtIds, b.targetIds.data.data(), 4 * (size_t)b.targetIds.size());
    copyOut(b.targetMask, tgtMask);
  }
  for(size_t r = 0; r < b.sentenceIds.size(); ++r)
    sentIds[r] = (int64_t)b.sentenceIds[r];
}

void ref_batches_free(void* h) { delete static_cast<RefBatches*>(h); }

// ---------------------------------------------------------------- model

void* ref_model_create(const char* cfgText, uint64_t seed) {
  auto* h = new RefModel;
  int rc = guard([&] {
    h->cfg = ModelConfig::parse(cfgText);
    h->model = buildModel(h->cfg);
    h->g = std::make_unique<ExpressionGraph>(seed);
    h->model.registerParams(*h->g);
    h->g->clear();
    h->adam = std::make_unique<Adam>(adamDefaultsFor(h->cfg));
    h->avg = std::make_unique<AveragedParameters>();
  });
  if(rc) {
    delete h;
    return nullptr;
  }
  return h;
}

void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

int64_t ref_param_count(void* h) {
  return (int64_t)static_cast<RefModel*>(h)->g->paramNames().size();
}

const char* ref_param_name(void* h, int64_t i) {
  return static_cast<RefModel*>(h)->g->paramNames()[(size_t)i].c_str();
}

int ref_param_shape(void* h, const char* name, int64_t* dims) {
  const Shape& s = static_cast<RefModel*>(h)->g->paramValue(name).shape();
  for(int i = 0; i < s.rank(); ++i)
    dims[i] = s[i];
  return s.rank();
}

int ref_param_get(void* h, const char* name, float* out) {
  return guard([&] { copyOut(static_cast<RefModel*>(h)->g->paramValue(name), out); });
}

int ref_param_set(void* h, const char* name, const float* in) {
  return guard([&] {
    Tensor& t = static_cast<RefModel*>(h)->g->paramValue(name);
    std::memcpy(t.data(), in, sizeof(float) * (size_t)t.size());
  });
}

int ref_grad_get(void* h, const char* name, float* out) {
  return guard([&] { copyOut(static_cast<RefModel*>(h)->g->paramGrad(name), out); });
}

int ref_grad_set(void* h, const char* name, const float* in) {
  return guard([&] {
    Tensor& t = static_cast<RefModel*>(h)->g->paramGrad(name);
    std::memcpy(t.data(), in, sizeof(float) * (size_t)t.size());
  });
}

// which: 0 = Adam m, 1 = Adam v, 2 = EMA average
int ref_state_get(void* h, int which, const char* name, float* out) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    auto& store = which == 0 ? m->adam->firstMoments()
                  : which == 1 ? m->adam->secondMoments()
                               : m->avg->values();
    copyOut(store.at(name), out);
  });
}

int64_t ref_adam_step(void* h) { return static_cast<RefModel*>(h)->adam->step(); }

// One worker's share of a trainSync update (train.cpp:226-237): clear, seed,
// buildLoss, forward, zeroGrads, backward.  Gradients stay in the graph.
int ref_loss_grads(void* h, void* bs, int64_t i, uint64_t graphSeed, double* loss,
                   float* tokens) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    ExpressionGraph& g = *m->g;
    g.clear();
    g.setSeed(graphSeed);
    Real tc = 0;
    NodeRef l = m->model.buildLoss(g, static_cast<RefBatches*>(bs)->b[(size_t)i], &tc);
    g.forward();
    g.zeroGrads();
    g.backward(l);
    *loss = (double)l.val().at(0);
    if(tokens)
      *tokens = (float)tc;
  });
}

// Forward-only logits of the teacher-forced decoder (for one-shot checks).
int ref_forward_loss(void* h, void* bs, int64_t i, uint64_t graphSeed, double* loss) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    ExpressionGraph& g = *m->g;
    g.clear();
    g.setSeed(graphSeed);
    NodeRef l = m->model.buildLoss(g, static_cast<RefBatches*>(bs)->b[(size_t)i]);
    g.forward();
    *loss = (double)l.val().at(0);
  });
}

int ref_adam_update(void* h, float lr) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    m->adam->update(*m->g, lr);
    m->avg->update(*m->g);
  });
}

int ref_train(void* h, void* ex, int workers, int64_t budget, uint64_t seed, int64_t epochs,
              int64_t maxUpdates, float lrBase, int64_t warmup, double* finalLoss,
              int64_t* updates) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    TrainOptions o;
    o.workers = workers;
    o.tokenBudget = budget;
    o.seed = seed;
    o.epochs = epochs;
    o.maxUpdates = maxUpdates;
    o.lr.base = lrBase;
    o.lr.warmup = warmup;
    TrainResult r = train(m->model, static_cast<RefExamples*>(ex)->ex, *m->g, *m->adam,
                          *m->avg, o);
    *finalLoss = r.finalLoss;
    *updates = r.updates;
  });
}

// train() with async = true: trainAsync (train.cpp:302-404)
int ref_train_async(void* h, void* ex, int workers, int64_t budget, uint64_t seed,
                    int64_t epochs, int64_t maxUpdates, float lrBase, int64_t warmup,
                    double* finalLoss, int64_t* updates) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    TrainOptions o;
    o.workers = workers;
    o.async = true;
    o.tokenBudget = budget;
    o.seed = seed;
    o.epochs = epochs;
    o.maxUpdates = maxUpdates;
    o.lr.base = lrBase;
    o.lr.warmup = warmup;
    TrainResult r = train(m->model, static_cast<RefExamples*>(ex)->ex, *m->g, *m->adam,
                          *m->avg, o);
    *finalLoss = r.finalLoss;
    *updates = r.updates;
  });
}

// train() with checkpointing / resume (train.cpp:284-287, 407-418)
int ref_train_ckpt(void* h, void* ex, int workers, int64_t budget, uint64_t seed, int64_t epochs,
                   int64_t maxUpdates, float lrBase, int64_t warmup, const char* ckptPath,
                   int64_t ckptEvery, const char* resumeFrom, double* finalLoss,
                   int64_t* updates) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    TrainOptions o;
    o.workers = workers;
    o.tokenBudget = budget;
    o.seed = seed;
    o.epochs = epochs;
    o.maxUpdates = maxUpdates;
    o.lr.base = lrBase;
    o.lr.warmup = warmup;
    o.checkpointPath = ckptPath ? ckptPath : "";
    o.checkpointEvery = ckptEvery;
    o.resumeFrom = resumeFrom ? resumeFrom : "";
    TrainResult r = train(m->model, static_cast<RefExamples*>(ex)->ex, *m->g, *m->adam,
                          *m->avg, o);
    *finalLoss = r.finalLoss;
    *updates = r.updates;
  });
}

int ref_save_model(void* h, const char* path) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    saveModel(path, m->cfg, *m->g);
  });
}

int ref_load_params(void* h, const char* path) {
  return guard([&] { loadParams(readModelFile(path), *static_cast<RefModel*>(h)->g); });
}

int ref_save_checkpoint(void* h, const char* path, int64_t update, int64_t epoch,
                        int64_t batch) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    saveCheckpoint(path, m->cfg, *m->g, *m->adam, *m->avg, update, epoch, batch);
  });
}

int ref_load_checkpoint(void* h, const char* path, int64_t* counters) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    loadCheckpoint(path, *m->g, *m->adam, *m->avg, counters[0], counters[1], counters[2]);
  });
}

// search.cpp:66-187 beamSearch on batch i with this model (one scorer).
// Output per sentence, hypotheses in rank order: out_counts[sentence] =
// number of hypotheses; hypothesis h: out_lens[h] tokens appended to
// out_tokens, out_scores[h] = score.  Capacities: max_hyps, max_tokens.
int ref_beam_search(void* h, void* bs, int64_t i, int beam, double alpha, int64_t lenFactor,
                    int64_t* out_counts, int64_t* out_lens, double* out_scores,
                    int32_t* out_tokens, int64_t max_hyps, int64_t max_tokens) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    const Batch& b = static_cast<RefBatches*>(bs)->b[(size_t)i];
    Scorer sc{"m0", &m->model, m->g.get(), 1.0};
    SearchOptions o;
    o.beamSize = beam;
    o.alpha = alpha;
    o.maxLengthFactor = lenFactor;
    auto res = beamSearch({sc}, b, o);
    int64_t nh = 0, nt = 0;
    for(size_t s = 0; s < res.size(); ++s) {
      out_counts[s] = (int64_t)res[s].size();
      for(auto& hyp : res[s]) {
        if(nh >= max_hyps || nt + (int64_t)hyp.tokens.size() > max_tokens)
          throw ContractError("ref_beam_search: output capacity");
        out_lens[nh] = (int64_t)hyp.tokens.size();
        out_scores[nh] = hyp.score;
        for(auto t : hyp.tokens)
          out_tokens[nt++] = t;
        ++nh;
      }
    }
  });
}

// search.cpp:189-215 scoreBatch: per row the total log-probability
int ref_score_batch(void* h, void* bs, int64_t i, double* out_scores) {
  return guard([&] {
    auto* m = static_cast<RefModel*>(h);
    const Batch& b = static_cast<RefBatches*>(bs)->b[(size_t)i];
    Scorer sc{"m0", &m->model, m->g.get(), 1.0};
    auto res = scoreBatch(sc, b);
    for(size_t r = 0; r < res.size(); ++r)
      out_scores[r] = res[r].score;
  });
}

int64_t ref_parameter_total(const char* cfgText) {
  int64_t n = -1;
  guard([&] { n = parameterTotal(ModelConfig::parse(cfgText)); });
  return n;
}

// ------------------------------------------------------------ op level

int ref_matmul(int ra, const int64_t* da, const float* a, int rb, const int64_t* db,
               const float* b, int rc, const int64_t* dc, float* c, int transA, int transB,
               float alpha, float beta) {
  return guard([&] {
    Tensor ta = tensorOf(ra, da, a), tb = tensorOf(rb, db, b);
    Tensor tc = tensorOf(rc, dc, c);
    matmulInto(tc, ta, tb, transA != 0, transB != 0, alpha, beta);
    copyOut(tc, c);
  });
}

// dot node fwd + bwd (graph.cpp:293-332), d(out) = G
int ref_op_dot(int ra, const int64_t* da, const float* a, int rb, const int64_t* db,
               const float* b, int transA, int transB, const float* G, float* out, float* ga,
               float* gb) {
  return guard([&] {
    ExpressionGraph g(1);
    NodeRef na = g.param("a", shapeOf(ra, da),
                         inits::fromVector(std::vector<Real>(a, a + shapeOf(ra, da).size())));
    NodeRef nb = g.param("b", shapeOf(rb, db),
                         inits::fromVector(std::vector<Real>(b, b + shapeOf(rb, db).size())));
    NodeRef o = g.dot(na, nb, transA != 0, transB != 0);
    NodeRef loss = seededLoss(g, o, G);
    g.forward();
    g.zeroGrads();
    g.backward(loss);
    copyOut(o.val(), out);
    copyOut(g.paramGrad("a"), ga);
    copyOut(g.paramGrad("b"), gb);
  });
}

int ref_op_layernorm(int64_t rows, int64_t d, const float* x, const float* gain,
                     const float* bias, const float* G, float* out, float* gx, float* gg,
                     float* gbias) {
  return guard([&] {
    ExpressionGraph g(1);
    NodeRef nx = g.param("x", Shape({rows, d}),
                         inits::fromVector(std::vector<Real>(x, x + rows * d)));
    NodeRef ng = g.param("g", Shape({d}), inits::fromVector(std::vector<Real>(gain, gain + d)));
    NodeRef nb = g.param("b", Shape({d}), inits::fromVector(std::vector<Real>(bias, bias + d)));
    NodeRef o = g.layerNorm(nx, ng, nb);
    NodeRef loss = seededLoss(g, o, G);
    g.forward();
    g.zeroGrads();
    g.backward(loss);
    copyOut(o.val(), out);
    copyOut(g.paramGrad("x"), gx);
    copyOut(g.paramGrad("g"), gg);
    copyOut(g.paramGrad("b"), gbias);
  });
}

// softmax over the last axis of x [rank dims], optional broadcastable mask
int ref_op_softmax(int rx, const int64_t* dx, const float* x, int rm, const int64_t* dm,
                   const float* mask, const float* G, float* out, float* gx) {
  return guard([&] {
    ExpressionGraph g(1);
    Shape sx = shapeOf(rx, dx);
    NodeRef nx = g.param("x", sx, inits::fromVector(std::vector<Real>(x, x + sx.size())));
    Tensor m = mask ? tensorOf(rm, dm, mask) : Tensor();
    NodeRef o = g.softmax(nx, m);
    NodeRef loss = seededLoss(g, o, G);
    g.forward();
    g.zeroGrads();
    g.backward(loss);
    copyOut(o.val(), out);
    copyOut(g.paramGrad("x"), gx);
  });
}

// masked mean cross-entropy (graph.cpp:859-924); logits [b x t x V]
int ref_op_xent(int64_t b, int64_t t, int64_t V, const float* logits, const int32_t* targets,
                const float* mask, double* loss, float* glogits) {
  return guard([&] {
    ExpressionGraph g(1);
    NodeRef nl = g.param("l", Shape({b, t, V}),
                         inits::fromVector(std::vector<Real>(logits, logits + b * t * V)));
    IntMat tg(b, t);
    std::memcpy(tg.data.data(), targets, 4 * (size_t)(b * t));
    Tensor m = mask ? Tensor(Shape({b, t}), std::vector<Real>(mask, mask + b * t)) : Tensor();
    NodeRef l = g.crossEntropy(nl, tg, m);
    g.forward();
    g.zeroGrads();
    g.backward(l);
    *loss = (double)l.val().at(0);
    copyOut(g.paramGrad("l"), glogits);
  });
}

// embedding gather + scatter-add (graph.cpp:595-622)
int ref_op_embed(int64_t V, int64_t e, const float* table, int64_t rows, int64_t cols,
                 const int32_t* ids, const float* G, float* out, float* gtable) {
  return guard([&] {
    ExpressionGraph g(1);
    NodeRef nt = g.param("E", Shape({V, e}),
                         inits::fromVector(std::vector<Real>(table, table + V * e)));
    IntMat im(rows, cols);
    std::memcpy(im.data.data(), ids, 4 * (size_t)(rows * cols));
    NodeRef o = g.embed(nt, im);
    NodeRef loss = seededLoss(g, o, G);
    g.forward();
    g.zeroGrads();
    g.backward(loss);
    copyOut(o.val(), out);
    copyOut(g.paramGrad("E"), gtable);
  });
}

// MultiHeadAttention::apply (layers.cpp:89-126) with identity q/k/v/o
// projections and zero biases, so out == the attention core; returns the
// gradients of the q/k/v inputs for d(out) = G.
int ref_op_mha(int64_t b, int64_t tq, int64_t tk, int64_t d, int heads, const float* q,
               const float* k, const float* v, const float* keyMask, int causal,
               const float* G, float* out, float* gq, float* gk, float* gv) {
  return guard([&] {
    ExpressionGraph g(1);
    std::vector<Real> eye((size_t)(d * d), Real(0));
    for(int64_t i = 0; i < d; ++i)
      eye[(size_t)(i * d + i)] = 1;
    for(const char* n : {"q", "k", "v", "o"}) {
      g.param(std::string("mha.") + n + "W", Shape({d, d}), inits::fromVector(eye));
      g.param(std::string("mha.") + n + "B", Shape({d}), inits::zeros());
    }
    NodeRef nq = g.param("xq", Shape({b, tq, d}), inits::fromVector(std::vector<Real>(q, q + b * tq * d)));
    NodeRef nk = g.param("xk", Shape({b, tk, d}), inits::fromVector(std::vector<Real>(k, k + b * tk * d)));
    NodeRef nv = g.param("xv", Shape({b, tk, d}), inits::fromVector(std::vector<Real>(v, v + b * tk * d)));
    MultiHeadAttention mha{"mha", d, heads};
    Tensor km = keyMask ? Tensor(Shape({b, tk}), std::vector<Real>(keyMask, keyMask + b * tk)) : Tensor();
    NodeRef o = mha.apply(g, nq, nk, nv, km, causal != 0);
    NodeRef loss = seededLoss(g, o, G);
    g.forward();
    g.zeroGrads();
    g.backward(loss);
    copyOut(o.val(), out);
    copyOut(g.paramGrad("xq"), gq);
    copyOut(g.paramGrad("xk"), gk);
    copyOut(g.paramGrad("xv"), gv);
  });
}

// fused GRU block (graph.cpp:648-813). Param order in `w` (each row-major):
// Uz Ur Uh [d x d], bz br bh [d], then (if e > 0) Wz Wr Wx [e x d], then (if
// ln) lnGz lnBz lnGr lnBr (+ lnGx lnBx if e > 0) [d]. Gradients come back in
// the same packed order in `gw`.
int ref_op_gru(int64_t b, int64_t e, int64_t d, int ln, const float* h, const float* x,
               const float* w, const float* G, float* out, float* gh, float* gx, float* gw) {
  return guard([&] {
    ExpressionGraph g(1);
    const float* p = w;
    std::vector<std::string> order;
    auto mk = [&](const std::string& name, Shape s) {
      NodeRef r = g.param(name, s, inits::fromVector(std::vector<Real>(p, p + s.size())));
      p += s.size();
      order.push_back(name);
      return r;
    };
    GruParams gp;
    gp.Uz = mk("Uz", Shape({d, d}));
    gp.Ur = mk("Ur", Shape({d, d}));
    gp.Uh = mk("Uh", Shape({d, d}));
    gp.bz = mk("bz", Shape({d}));
    gp.br = mk("br", Shape({d}));
    gp.bh = mk("bh", Shape({d}));
    if(e > 0) {
      gp.Wz = mk("Wz", Shape({e, d}));
      gp.Wr = mk("Wr", Shape({e, d}));
      gp.Wx = mk("Wx", Shape({e, d}));
    }
    if(ln) {
      gp.lnGz = mk("lnGz", Shape({d}));
      gp.lnBz = mk("lnBz", Shape({d}));
      gp.lnGr = mk("lnGr", Shape({d}));
      gp.lnBr = mk("lnBr", Shape({d}));
      if(e > 0) {
        gp.lnGx = mk("lnGx", Shape({d}));
        gp.lnBx = mk("lnBx", Shape({d}));
      }
    }
    NodeRef nh = g.param("h", Shape({b, d}), inits::fromVector(std::vector<Real>(h, h + b * d)));
    NodeRef nx;
    if(e > 0)
      nx = g.param("x", Shape({b, e}), inits::fromVector(std::vector<Real>(x, x + b * e)));
    NodeRef o = g.gruCell(nh, nx, gp, ln != 0);
    NodeRef loss = seededLoss(g, o, G);
    g.forward();
    g.zeroGrads();
    g.backward(loss);
    copyOut(o.val(), out);
    copyOut(g.paramGrad("h"), gh);
    if(e > 0)
      copyOut(g.paramGrad("x"), gx);
    float* q = gw;
    for(auto& name : order) {
      const Tensor& t = g.paramGrad(name);
      std::memcpy(q, t.data(), sizeof(float) * (size_t)t.size());
      q += t.size();
    }
  });
}

}  // extern "C"

// ---------------------------------------------------------------- op programs
// A tiny stack program over the reference's ExpressionGraph op constructors
// (graph.h:72-110), for op-level parity of the elementwise / broadcast /
// reduce / layout rows (graph.cpp:139-524).  Tokens (whitespace separated):
//   pK                  push parameter K (inputs[K], named "pK")
//   dup                 push the top node again (self-operand cases)
//   add sub mul div     binary, trailing-dim broadcast (graph.cpp:139-237)
//   tanh sigmoid relu exp log neg        unary (graph.cpp:239-268)
//   scale:S adds:S      scale / addScalar
//   reshape:d0,d1,...   transpose:p0,p1,...
//   concat:N:AXIS       slice:AXIS:START:LEN      gather:r0,r1,...
//   reduce:OP:AXIS:KEEP (OP = sum|max|mean|argmax)   softmax
// The top of the stack is the output; loss = sum(out * G).
extern "C" int ref_op_program(const char* prog, int nin, const int* ranks, const int64_t* dims,
                              const float* const* data, const float* G, float* out,
                              int64_t out_cap, int64_t* out_dims, int* out_rank,
                              float* const* grads) {
  return guard([&] {
    ExpressionGraph g(1);
    std::vector<NodeRef> stack, params;
    std::vector<std::string> names;
    const int64_t* d = dims;
    for(int i = 0; i < nin; ++i) {
      Shape s = shapeOf(ranks[i], d);
      d += ranks[i];
      names.push_back("p" + std::to_string(i));
      params.push_back(g.param(names.back(), s,
                               inits::fromVector(std::vector<Real>(data[i], data[i] + s.size()))));
    }
    auto pop = [&] {
      if(stack.empty())
        throw ContractError("op program: stack underflow");
      NodeRef r = stack.back();
      stack.pop_back();
      return r;
    };
    auto split = [](const std::string& s, char c) {
      std::vector<std::string> out;
      std::stringstream ss(s);
      std::string tok;
      while(std::getline(ss, tok, c))
        out.push_back(tok);
      return out;
    };
    std::stringstream ps(prog);
    std::string tok;
    while(ps >> tok) {
      auto f = split(tok, ':');
      const std::string& op = f[0];
      if(op[0] == 'p' && op.size() > 1 && std::isdigit((unsigned char)op[1])) {
        stack.push_back(params[(size_t)std::stoi(op.substr(1))]);
      } else if(op == "dup") {
        NodeRef t = pop();
        stack.push_back(t);
        stack.push_back(t);
      } else if(op == "add" || op == "sub" || op == "mul" || op == "div") {
        NodeRef b = pop(), a = pop();
        stack.push_back(op == "add" ? g.add(a, b)
                        : op == "sub" ? g.sub(a, b)
                        : op == "mul" ? g.mul(a, b)
                                      : g.div(a, b));
      } else if(op == "tanh") {
        stack.push_back(g.tanh(pop()));
      } else if(op == "sigmoid") {
        stack.push_back(g.sigmoid(pop()));
      } else if(op == "relu") {
        stack.push_back(g.relu(pop()));
      } else if(op == "exp") {
        stack.push_back(g.exp(pop()));
      } else if(op == "log") {
        stack.push_back(g.log(pop()));
      } else if(op == "neg") {
        stack.push_back(g.neg(pop()));
      } else if(op == "scale") {
        stack.push_back(g.scale(pop(), (Real)std::stod(f.at(1))));
      } else if(op == "adds") {
        stack.push_back(g.addScalar(pop(), (Real)std::stod(f.at(1))));
      } else if(op == "reshape") {
        std::vector<int64_t> s;
        for(auto& x : split(f.at(1), ','))
          s.push_back(std::stoll(x));
        stack.push_back(g.reshape(pop(), Shape(s)));
      } else if(op == "transpose") {
        std::vector<int> p;
        for(auto& x : split(f.at(1), ','))
          p.push_back(std::stoi(x));
        stack.push_back(g.transpose(pop(), p));
      } else if(op == "concat") {
        int n = std::stoi(f.at(1)), axis = std::stoi(f.at(2));
        std::vector<NodeRef> parts((size_t)n);
        for(int i = n - 1; i >= 0; --i)
          parts[(size_t)i] = pop();
        stack.push_back(g.concat(parts, axis));
      } else if(op == "slice") {
        stack.push_back(g.slice(pop(), std::stoi(f.at(1)), std::stoll(f.at(2)), std::stoll(f.at(3))));
      } else if(op == "gather") {
        std::vector<int64_t> rows;
        for(auto& x : split(f.at(1), ','))
          rows.push_back(std::stoll(x));
        stack.push_back(g.gatherRows(pop(), rows));
      } else if(op == "reduce") {
        const std::string& r = f.at(1);
        ReduceOp ro = r == "sum" ? ReduceOp::Sum
                      : r == "max" ? ReduceOp::Max
                      : r == "mean" ? ReduceOp::Mean
                                    : ReduceOp::Argmax;
        stack.push_back(g.reduce(ro, pop(), std::stoi(f.at(2)), std::stoi(f.at(3)) != 0));
      } else if(op == "softmax") {
        stack.push_back(g.softmax(pop()));
      } else if(op == "dot") {  // dot[:transA:transB] (graph.cpp:293-332)
        NodeRef b = pop(), a = pop();
        const bool ta = f.size() > 1 && f[1] == "1", tb = f.size() > 2 && f[2] == "1";
        stack.push_back(g.dot(a, b, ta, tb));
      } else {
        throw ContractError("op program: unknown token " + tok);
      }
    }
    NodeRef o = pop();
    if(o.shape.size() > out_cap)
      throw ContractError("op program: output buffer too small");
    *out_rank = (int)o.shape.rank();
    for(int i = 0; i < o.shape.rank(); ++i)
      out_dims[i] = o.shape[i];
    NodeRef loss = seededLoss(g, o, G);
    g.forward();
    g.zeroGrads();
    g.backward(loss);
    copyOut(o.val(), out);
    for(int i = 0; i < nin; ++i)
      copyOut(g.paramGrad(names[(size_t)i]), grads[i]);
  });
}
