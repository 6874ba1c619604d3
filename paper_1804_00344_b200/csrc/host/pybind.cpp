// Python binding of the C++ host framework (module `_mtk`).  Mirrors the
// reference's public C++ API names so the parity tests read like the
// reference's own suites; tensors cross as numpy arrays (host copies).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <sstream>

#include "mtk/device.h"
#include "mtk/search.h"
#include "mtk/train.h"

namespace py = pybind11;
using namespace mtk;

namespace {

using FArr = py::array_t<float, py::array::c_style | py::array::forcecast>;
using IArr = py::array_t<int32_t, py::array::c_style | py::array::forcecast>;

Shape shapeOf(const py::sequence& s) {
  std::vector<int64_t> d;
  for(auto v : s)
    d.push_back(v.cast<int64_t>());
  return Shape(d);
}

py::tuple tupleOf(const Shape& s) {
  py::tuple t(s.rank());
  for(int i = 0; i < s.rank(); ++i)
    t[i] = s[i];
  return t;
}

FArr toNumpy(const Tensor& t) {
  FArr out(t.shape().dims());
  const Real* p = t.data();
  std::memcpy(out.mutable_data(), p, sizeof(float) * (size_t)t.size());
  return out;
}

Tensor fromNumpy(FArr a) {
  std::vector<int64_t> dims(a.shape(), a.shape() + a.ndim());
  if(dims.empty())
    dims.push_back(1);
  std::vector<Real> v(a.data(), a.data() + a.size());
  return Tensor(Shape(dims), std::move(v));
}

IntMat intMatOf(IArr a) {
  if(a.ndim() != 2)
    throw DimensionError("id matrix must be 2-d");
  IntMat m(a.shape(0), a.shape(1));
  std::memcpy(m.data.data(), a.data(), sizeof(int32_t) * (size_t)m.size());
  return m;
}

ParamInit initOf(py::object init) {
  if(py::isinstance<py::str>(init)) {
    std::string s = init.cast<std::string>();
    if(s == "zeros")
      return inits::zeros();
    if(s == "ones")
      return inits::ones();
    if(s == "glorot")
      return inits::glorotUniform();
    throw ContractError("unknown init " + s);
  }
  if(py::isinstance<py::float_>(init) || py::isinstance<py::int_>(init))
    return inits::constant(init.cast<float>());
  FArr a = init.cast<FArr>();
  return inits::fromVector(std::vector<Real>(a.data(), a.data() + a.size()));
}

struct Examples {
  std::vector<Example> ex;
};

}  // namespace

PYBIND11_MODULE(_mtk, m) {
  m.doc() = "B200-native mtk training step (C++ host over sm_100a kernels)";

  static py::exception<Error> exError(m, "Error", PyExc_RuntimeError);
  static py::exception<DimensionError> exDim(m, "DimensionError", exError.ptr());
  static py::exception<NumericError> exNum(m, "NumericError", exError.ptr());
  static py::exception<ContractError> exCon(m, "ContractError", exError.ptr());
  static py::exception<DataError> exData(m, "DataError", exError.ptr());
  static py::exception<IoError> exIo(m, "IoError", exError.ptr());
  py::register_exception_translator([](std::exception_ptr p) {
    try {
      if(p)
        std::rethrow_exception(p);
    } catch(const DimensionError& e) {
      py::set_error(exDim, e.what());
    } catch(const NumericError& e) {
      py::set_error(exNum, e.what());
    } catch(const ContractError& e) {
      py::set_error(exCon, e.what());
    } catch(const DataError& e) {
      py::set_error(exData, e.what());
    } catch(const IoError& e) {
      py::set_error(exIo, e.what());
    } catch(const Error& e) {
      py::set_error(exError, e.what());
    }
  });

  // ---------------------------------------------------------- device
  m.def("select_device", &Device::selectDevice);
  m.def("set_precision", [](const std::string& p) {
    Device::get().setPrecision(p == "fp32" ? Precision::FP32 : Precision::TF32);
  });
  m.def("precision", [] { return Device::get().precision() == Precision::FP32 ? "fp32" : "tf32"; });
  m.def("set_dropout_rng", [](const std::string& r) {
    if(r != "auto" && r != "host" && r != "device")
      throw ContractError("dropout rng must be auto, host or device");
    Device::get().setDropoutRng(r == "host" ? DropoutRng::Host
                                : r == "device" ? DropoutRng::Device : DropoutRng::Auto);
  });
  m.def("dropout_rng", [] { return Device::get().deviceDropout() ? "device" : "host"; });
  m.def("sync", [] { Device::get().sync(); });
  m.def("check_flags", [] { Device::get().checkFlags("explicit check"); });
  m.def("launch_count", [] { return (uint64_t)mtkc_launch_count(); });
  m.def("h2d_bytes", [] { return (uint64_t)mtkc_h2d_bytes(); });
  m.def("d2h_bytes", [] { return (uint64_t)mtkc_d2h_bytes(); });
  m.def("prof_enable", [](int on) { MTKC(mtkc_prof_enable(on)); });
  m.def("gpu_sleep", [](int64_t us) { MTKC(mtkc_gpu_sleep(us, Device::get().stream())); });
  // CUDA events on the compute stream (the stream every kernel runs on)
  m.def("event_record", [] {
    void* e = nullptr;
    MTKC(mtkc_event_create(&e));
    MTKC(mtkc_event_record(e, Device::get().stream()));
    return (uintptr_t)e;
  });
  m.def("event_elapsed_ms_keep", [](uintptr_t a, uintptr_t b) {  // events stay alive
    Device::get().sync();
    float ms = 0;
    MTKC(mtkc_event_elapsed_ms((void*)a, (void*)b, &ms));
    return ms;
  });
  m.def("event_destroy", [](uintptr_t a) { mtkc_event_destroy((void*)a); });
  m.def("event_elapsed_ms", [](uintptr_t a, uintptr_t b) {
    Device::get().sync();
    float ms = 0;
    MTKC(mtkc_event_elapsed_ms((void*)a, (void*)b, &ms));
    mtkc_event_destroy((void*)a);
    mtkc_event_destroy((void*)b);
    return ms;
  });
  m.def("prof_report", [] {
    std::vector<char> buf(1 << 16);
    MTKC(mtkc_prof_report(buf.data(), buf.size()));
    return std::string(buf.data());
  });
  m.def("sm_count", [] { return Device::get().sms(); });
  m.def("stream_handle", [] { return (uintptr_t)Device::get().stream(); });
  m.def("nccl_unique_id", [] {
    char id[128];
    MTKC(mtkc_nccl_unique_id(id));
    return py::bytes(id, 128);
  });
  m.def("comm_ranks", [] { return commRanks(); });
  m.def(
      "rank_share",
      [](const std::vector<double>& tokens, int workers, int world, int rank) {
        std::vector<std::pair<int, float>> out;
        for(auto& s : rankShare(tokens, workers, world, rank))
          out.emplace_back(s.worker, s.weight);
        return out;
      },
      py::arg("tokens"), py::arg("workers"), py::arg("world"), py::arg("rank"));
  m.def(
      "set_distributed",
      [](int rank, int world, py::bytes id, bool forceComm) {
        std::string s = id;
        setDistributed(rank, world, s.data(), forceComm);
      },
      py::arg("rank"), py::arg("world"), py::arg("id"), py::arg("force_comm") = false);

  // ---------------------------------------------------------- tensors
  py::class_<Tensor>(m, "Tensor")
      .def(py::init([](FArr a) { return fromNumpy(a); }))
      .def_property_readonly("shape", [](const Tensor& t) { return tupleOf(t.shape()); })
      .def("numpy", [](const Tensor& t) { return toNumpy(t); })
      .def("dev_ptr", [](const Tensor& t) { return (uintptr_t)t.devc(); });

  py::class_<NodeRef>(m, "NodeRef")
      .def(py::init<>())
      .def_property_readonly("shape", [](const NodeRef& r) { return tupleOf(r.shape); })
      .def_readonly("index", &NodeRef::index)
      .def("valid", &NodeRef::valid)
      .def("val", [](const NodeRef& r) { return toNumpy(r.val()); })
      .def("grad", [](const NodeRef& r) { return toNumpy(r.grad()); });

  py::class_<GruParams>(m, "GruParams")
      .def(py::init<>())
      .def_readwrite("Wz", &GruParams::Wz)
      .def_readwrite("Uz", &GruParams::Uz)
      .def_readwrite("bz", &GruParams::bz)
      .def_readwrite("Wr", &GruParams::Wr)
      .def_readwrite("Ur", &GruParams::Ur)
      .def_readwrite("br", &GruParams::br)
      .def_readwrite("Wx", &GruParams::Wx)
      .def_readwrite("Uh", &GruParams::Uh)
      .def_readwrite("bh", &GruParams::bh)
      .def_readwrite("lnGz", &GruParams::lnGz)
      .def_readwrite("lnBz", &GruParams::lnBz)
      .def_readwrite("lnGr", &GruParams::lnGr)
      .def_readwrite("lnBr", &GruParams::lnBr)
      .def_readwrite("lnGx", &GruParams::lnGx)
      .def_readwrite("lnBx", &GruParams::lnBx);

  py::enum_<ReduceOp>(m, "ReduceOp")
      .value("Sum", ReduceOp::Sum)
      .value("Max", ReduceOp::Max)
      .value("Mean", ReduceOp::Mean)
      .value("Argmax", ReduceOp::Argmax);

  using G = ExpressionGraph;
  py::class_<G>(m, "ExpressionGraph")
      .def(py::init<uint64_t, bool>(), py::arg("seed") = 0, py::arg("inference") = false)
      .def("param",
           [](G& g, const std::string& name, py::sequence shape, py::object init) {
             return g.param(name, shapeOf(shape), initOf(init));
           },
           py::arg("name"), py::arg("shape"), py::arg("init") = "glorot")
      .def("constant", [](G& g, FArr a) { return g.constant(fromNumpy(a)); })
      .def("add", &G::add)
      .def("sub", &G::sub)
      .def("mul", &G::mul)
      .def("div", &G::div)
      .def("tanh", &G::tanh)
      .def("sigmoid", &G::sigmoid)
      .def("relu", &G::relu)
      .def("exp", &G::exp)
      .def("log", &G::log)
      .def("neg", &G::neg)
      .def("scale", &G::scale)
      .def("add_scalar", &G::addScalar)
      .def("dot", &G::dot, py::arg("a"), py::arg("b"), py::arg("trans_a") = false,
           py::arg("trans_b") = false)
      .def("affine", &G::affine, py::arg("x"), py::arg("w"), py::arg("b"),
           py::arg("trans_w") = false)
      .def("affine_relu", &G::affineRelu)
      .def("reshape", [](G& g, NodeRef a, py::sequence s) { return g.reshape(a, shapeOf(s)); })
      .def("transpose", &G::transpose)
      .def("concat", &G::concat)
      .def("slice", &G::slice)
      .def("gather_rows", &G::gatherRows)
      .def("reduce", &G::reduce, py::arg("op"), py::arg("a"), py::arg("axis"),
           py::arg("keep_axis") = false)
      .def("softmax",
           [](G& g, NodeRef a, py::object mask) {
             return g.softmax(a, mask.is_none() ? Tensor() : fromNumpy(mask.cast<FArr>()));
           },
           py::arg("a"), py::arg("mask") = py::none())
      .def("layer_norm", &G::layerNorm, py::arg("x"), py::arg("gain"), py::arg("bias"),
           py::arg("eps") = 1e-9f)
      .def("embed", [](G& g, NodeRef t, IArr ids) { return g.embed(t, intMatOf(ids)); })
      .def("gru_cell", &G::gruCell)
      .def("dropout", &G::dropout, py::arg("x"), py::arg("p"), py::arg("variational_axis") = -1)
      .def("dropout_mask",
           [](G& g, py::sequence shape, float p) { return g.dropoutMask(shapeOf(shape), p); })
      .def("residual_add", &G::residualAdd, py::arg("r"), py::arg("z"))
      .def("lstm_cell", &G::lstmCell)
      .def("lstm_state", &G::lstmState)
      .def("lstm_cell_state", &G::lstmCellState)
      .def("cross_entropy",
           [](G& g, NodeRef l, IArr targets, py::object mask) {
             return g.crossEntropy(l, intMatOf(targets),
                                   mask.is_none() ? Tensor() : fromNumpy(mask.cast<FArr>()));
           },
           py::arg("logits"), py::arg("targets"), py::arg("mask") = py::none())
      .def("attention",
           [](G& g, NodeRef q, NodeRef k, NodeRef v, py::object mask, bool causal, int heads) {
             return g.attention(q, k, v,
                                mask.is_none() ? Tensor() : fromNumpy(mask.cast<FArr>()), causal,
                                heads);
           })
      .def("scale_add_const",
           [](G& g, NodeRef x, float s, FArr pe) { return g.scaleAddConst(x, s, fromNumpy(pe)); })
      .def("mask_blend",
           [](G& g, NodeRef a, NodeRef b, FArr m) { return g.maskBlend(a, b, fromNumpy(m)); })
      .def("forward", &G::forward)
      .def("backward", [](G& g, NodeRef loss) { g.backward(loss); })
      .def("clear", &G::clear)
      .def("set_seed", &G::setSeed)
      .def("set_loss_scale", &G::setLossScale)
      .def("node_count", &G::nodeCount)
      .def("param_names", &G::paramNames)
      .def("has_param", &G::hasParam)
      .def("param_value", [](G& g, const std::string& n) { return toNumpy(g.paramValue(n)); })
      .def("param_grad", [](G& g, const std::string& n) { return toNumpy(g.paramGrad(n)); })
      .def("set_param",
           [](G& g, const std::string& n, FArr a) {
             Tensor& t = g.paramValue(n);
             if((int64_t)a.size() != t.size())
               throw DimensionError("set_param size mismatch for " + n);
             MTKC(mtkc_memcpy_h2d(t.dev(), a.data(), sizeof(float) * (size_t)a.size(),
                                  Device::get().stream()));
             Device::get().sync();
           })
      .def("zero_grads", &G::zeroGrads)
      .def("arena_high_water", [](G& g) { return g.arena().highWaterBytes(); })
      .def("param_pool_size", [](G& g) { return g.pool().used(); });

  // ---------------------------------------------------------- arena (tensor.h:43-61)
  py::class_<Arena>(m, "Arena")
      .def(py::init<size_t>(), py::arg("capacity_bytes"))
      .def("alloc", [](Arena& a, int64_t elems) { a.alloc(elems); })
      .def("reset", &Arena::reset)
      .def("capacity", &Arena::capacity)
      .def("outstanding_bytes", &Arena::outstandingBytes)
      .def("high_water_bytes", &Arena::highWaterBytes);

  // ---------------------------------------------------------- data
  py::class_<Examples>(m, "Examples")
      .def(py::init([](py::list sources, py::list targets, py::list extra) {
             Examples e;
             size_t n = py::len(sources);
             e.ex.resize(n);
             for(size_t i = 0; i < n; ++i) {
               auto s = sources[i].cast<std::vector<int32_t>>();
               e.ex[i].sources = {s};
               for(auto stream : extra)  // further source streams (multi-source models)
                 e.ex[i].sources.push_back(
                     stream.cast<py::list>()[i].cast<std::vector<int32_t>>());
               if(py::len(targets)) {
                 e.ex[i].target = targets[i].cast<std::vector<int32_t>>();
                 e.ex[i].hasTarget = true;
               }
               e.ex[i].id = i;
             }
             return e;
           }),
           py::arg("sources"), py::arg("targets"), py::arg("extra_streams") = py::list())
      .def("__len__", [](const Examples& e) { return e.ex.size(); });

  // SURVEY.md 8(d) synthetic generator (same formula as synth.py)
  m.def("synth_examples", [](int64_t n, int64_t vocab, int64_t start) {
    auto sm = [](uint64_t x) {
      uint64_t z = x + 0x9e3779b97f4a7c15ull;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      return z ^ (z >> 31);
    };
    Examples e;
    e.ex.resize((size_t)n);
    for(int64_t k = 0; k < n; ++k) {
      uint64_t i = (uint64_t)(start + k);
      int64_t ls = 16 + (int64_t)(sm(1234ull * 1000003ull + i) % 17);
      int64_t lt = 16 + (int64_t)(sm(5678ull * 1000003ull + i) % 17);
      std::vector<int32_t> s((size_t)ls), t((size_t)lt);
      for(int64_t j = 0; j < ls; ++j)
        s[(size_t)j] = (int32_t)(2 + sm((i << 20) ^ (uint64_t)j ^ 0xabcull) % (uint64_t)(vocab - 2));
      for(int64_t j = 0; j < lt; ++j)
        t[(size_t)j] = (int32_t)(2 + sm((i << 20) ^ (uint64_t)j ^ 0xdefull) % (uint64_t)(vocab - 2));
      e.ex[(size_t)k].sources = {s};
      e.ex[(size_t)k].target = t;
      e.ex[(size_t)k].hasTarget = true;
      e.ex[(size_t)k].id = (size_t)k;
    }
    return e;
  }, py::arg("n"), py::arg("vocab"), py::arg("start") = 0);

  py::class_<Batch>(m, "Batch")
      .def(py::init([](IArr srcIds, FArr srcMask, IArr tgtIds, FArr tgtMask) {
        Batch b;
        b.sourceIds = {intMatOf(srcIds)};
        b.sourceMasks = {fromNumpy(srcMask)};
        b.targetIds = intMatOf(tgtIds);
        b.targetMask = fromNumpy(tgtMask);
        b.hasTarget = true;
        for(int64_t r = 0; r < b.rows(); ++r)
          b.sentenceIds.push_back((size_t)r);
        return b;
      }))
      .def("rows", &Batch::rows)
      .def("target_tokens", &Batch::targetTokenCount)
      .def("padded_slots",  // rows x (padded source + padded target length)
           [](const Batch& b) {
             int64_t n = 0;
             for(auto& s : b.sourceIds)
               n += s.size();
             return n + b.targetIds.size();
           })
      .def("source_tokens", &Batch::sourceTokenCount)
      .def("src_ids",
           [](const Batch& b) {
             const IntMat& im = b.sourceIds[0];
             IArr a({im.rows, im.cols});
             std::memcpy(a.mutable_data(), im.data.data(), 4 * (size_t)im.size());
             return a;
           })
      .def("tgt_ids",
           [](const Batch& b) {
             IArr a({b.targetIds.rows, b.targetIds.cols});
             std::memcpy(a.mutable_data(), b.targetIds.data.data(), 4 * (size_t)b.targetIds.size());
             return a;
           })
      .def("src_mask", [](const Batch& b) { return toNumpy(b.sourceMasks[0]); })
      .def("tgt_mask", [](const Batch& b) { return toNumpy(b.targetMask); })
      .def("sentence_ids", [](const Batch& b) { return b.sentenceIds; });

  m.def("make_batches",
        [](const Examples& e, int64_t budget, uint64_t seed, bool shuffle) {
          BatchOptions o;
          o.tokenBudget = budget;
          o.seed = seed;
          o.shuffle = shuffle;
          return makeBatches(e.ex, o);
        },
        py::arg("examples"), py::arg("budget"), py::arg("seed") = 1, py::arg("shuffle") = true);

  // ---------------------------------------------------------- models
  py::class_<ModelConfig>(m, "ModelConfig")
      .def_static("parse", &ModelConfig::parse)
      .def("serialize", &ModelConfig::serialize)
      .def_readwrite("architecture", &ModelConfig::architecture)
      .def_readwrite("emb_dim", &ModelConfig::embDim)
      .def_readwrite("state_dim", &ModelConfig::stateDim)
      .def_readwrite("source_vocab", &ModelConfig::sourceVocab)
      .def_readwrite("target_vocab", &ModelConfig::targetVocab)
      .def_readwrite("heads", &ModelConfig::heads)
      .def_readwrite("layers", &ModelConfig::layers)
      .def_readwrite("dropout", &ModelConfig::dropout)
      .def_readwrite("tying", &ModelConfig::tying)
      .def_readwrite("layer_norm", &ModelConfig::layerNorm);

  py::class_<Model, std::shared_ptr<Model>>(m, "Model")
      .def(py::init([](const std::string& cfg) {
        return std::make_shared<Model>(buildModel(ModelConfig::parse(cfg)));
      }))
      .def_property_readonly("config", [](const Model& mo) { return mo.config; })
      .def("register_params", &Model::registerParams)
      .def("build_loss", [](const Model& mo, G& g, const Batch& b) { return mo.buildLoss(g, b); });

  // decoding (search.cpp): per sentence [(tokens, score, token_scores), ...]
  m.def(
      "beam_search",
      [](const Model& mo, G& g, const Batch& b, int beam, double alpha, int64_t lenFactor) {
        SearchOptions o;
        o.beamSize = beam;
        o.alpha = alpha;
        o.maxLengthFactor = lenFactor;
        auto res = beamSearch({Scorer{"m0", &mo, &g, 1.0}}, b, o);
        py::list out;
        for(auto& list : res) {
          py::list hyps;
          for(auto& h : list)
            hyps.append(py::make_tuple(h.tokens, h.score, h.tokenScores));
          out.append(hyps);
        }
        return out;
      },
      py::arg("model"), py::arg("graph"), py::arg("batch"), py::arg("beam") = 5,
      py::arg("alpha") = 0.6, py::arg("max_length_factor") = 3);
  m.def("score_batch", [](const Model& mo, G& g, const Batch& b) {
    auto res = scoreBatch(Scorer{"m0", &mo, &g, 1.0}, b);
    py::list out;
    for(auto& h : res)
      out.append(py::make_tuple(h.tokens, h.score, h.tokenScores));
    return out;
  });

  m.def("parameter_total", [](const std::string& cfg) {
    return parameterTotal(ModelConfig::parse(cfg));
  });

  // ---------------------------------------------------------- training
  py::class_<AdamConfig>(m, "AdamConfig")
      .def(py::init<>())
      .def_readwrite("beta1", &AdamConfig::beta1)
      .def_readwrite("beta2", &AdamConfig::beta2)
      .def_readwrite("eps", &AdamConfig::eps);
  m.def("adam_defaults_for",
        [](const std::string& cfg) { return adamDefaultsFor(ModelConfig::parse(cfg)); });

  py::class_<AveragedParameters, std::shared_ptr<AveragedParameters>>(m, "AveragedParameters")
      .def(py::init<float>(), py::arg("beta") = 0.9999f)
      .def("update", &AveragedParameters::update)
      .def("apply_to", &AveragedParameters::applyTo)
      .def("value", [](AveragedParameters& a, G& g, const std::string& n) {
        return toNumpy(a.value(g, n));
      });

  py::class_<Adam, std::shared_ptr<Adam>>(m, "Adam")
      .def(py::init<AdamConfig>(), py::arg("config") = AdamConfig())
      .def("update",
           [](Adam& a, G& g, float lr, AveragedParameters* avg) { a.update(g, lr, avg); },
           py::arg("g"), py::arg("lr"), py::arg("avg") = nullptr)
      .def("step", &Adam::step)
      .def("set_step", &Adam::setStep)
      .def("first_moment",
           [](Adam& a, G& g, const std::string& n) { return toNumpy(a.firstMoment(g, n)); })
      .def("second_moment",
           [](Adam& a, G& g, const std::string& n) { return toNumpy(a.secondMoment(g, n)); })
      .def("update_tensor", [](Adam& a, const std::string& name, FArr value, FArr grad, float lr,
                               int64_t step) {
        Tensor v = fromNumpy(value), gr = fromNumpy(grad);
        a.updateTensor(name, v, gr, lr, step);
        return toNumpy(v);
      });

  py::class_<LrSchedule>(m, "LrSchedule")
      .def(py::init<>())
      .def_readwrite("base", &LrSchedule::base)
      .def_readwrite("warmup", &LrSchedule::warmup)
      .def("__call__", &LrSchedule::operator());

  py::class_<TrainOptions>(m, "TrainOptions")
      .def(py::init<>())
      .def_readwrite("workers", &TrainOptions::workers)
      .def_readwrite("async_", &TrainOptions::async)
      .def_readwrite("token_budget", &TrainOptions::tokenBudget)
      .def_readwrite("seed", &TrainOptions::seed)
      .def_readwrite("epochs", &TrainOptions::epochs)
      .def_readwrite("max_updates", &TrainOptions::maxUpdates)
      .def_readwrite("lr", &TrainOptions::lr)
      .def_readwrite("average_beta", &TrainOptions::averageBeta)
      .def_readwrite("log_every", &TrainOptions::logEvery)
      .def_readwrite("checkpoint_path", &TrainOptions::checkpointPath)
      .def_readwrite("checkpoint_every", &TrainOptions::checkpointEvery)
      .def_readwrite("resume_from", &TrainOptions::resumeFrom)
      .def_readwrite("overlap_allreduce", &TrainOptions::overlapAllreduce)
      .def_readwrite("bucket_elems", &TrainOptions::bucketElems);
  m.def("save_model", [](const std::string& path, const std::string& cfg, G& g) {
    saveModel(path, ModelConfig::parse(cfg), g);
  });
  m.def("load_params", [](const std::string& path, G& g) { loadParams(readModelFile(path), g); });
  m.def("read_model_config", [](const std::string& path) {
    return readModelFile(path).config.serialize();
  });
  m.def("save_checkpoint", [](const std::string& path, const std::string& cfg, G& g, Adam& adam,
                              AveragedParameters& avg, int64_t update, int64_t epoch,
                              int64_t batch) {
    saveCheckpoint(path, ModelConfig::parse(cfg), g, adam, avg, update, epoch, batch);
  });
  m.def("load_checkpoint", [](const std::string& path, G& g, Adam& adam, AveragedParameters& avg) {
    int64_t u = 0, e = 0, b = 0;
    loadCheckpoint(path, g, adam, avg, u, e, b);
    return py::make_tuple(u, e, b);
  });

  py::class_<TrainResult>(m, "TrainResult")
      .def_readonly("updates", &TrainResult::updates)
      .def_readonly("epochs", &TrainResult::epochs)
      .def_readonly("final_loss", &TrainResult::finalLoss);

  m.def("train",
        [](Model& model, const Examples& data, G& master, Adam& adam, AveragedParameters& avg,
           TrainOptions opts) {
          std::ostringstream log;
          opts.log = &log;
          TrainResult r = train(model, data.ex, master, adam, avg, opts);
          return py::make_tuple(r, log.str());
        });

  py::class_<UpdateResult>(m, "UpdateResult")
      .def_readonly("loss", &UpdateResult::loss)
      .def_readonly("tokens", &UpdateResult::tokens);

  py::class_<SyncStepper>(m, "SyncStepper")
      .def(py::init<const Model&, G&, Adam&, AveragedParameters&, const TrainOptions&>(),
           py::keep_alive<1, 2>(), py::keep_alive<1, 3>(), py::keep_alive<1, 4>(),
           py::keep_alive<1, 5>())
      .def("update",
           [](SyncStepper& s, const std::vector<const Batch*>& batches, int64_t u, bool read) {
             return s.update(batches, u, read);
           },
           py::arg("batches"), py::arg("update_index"), py::arg("read_loss") = true)
      .def("update_pipelined",
           [](SyncStepper& s, const std::vector<const Batch*>& batches, int64_t u) {
             return s.updatePipelined(batches, u);
           },
           py::arg("batches"), py::arg("update_index"))
      .def("flush_pipelined", &SyncStepper::flushPipelined)
      .def("host_times", &SyncStepper::hostTimes)
      .def("buckets_issued", &SyncStepper::bucketsIssued);

  m.def("mix_seed", &mixSeed);
}
