// Adam + EMA, learning-rate schedule and synchronous data-parallel training
// (reference: src/train.cpp).
#include "mtk/train.h"

#include <algorithm>
#include <chrono>
#include <memory>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <ostream>

#include "mtk/device.h"

namespace mtk {

AdamConfig adamDefaultsFor(const ModelConfig& config) {  // train.cpp:11-20
  bool transformer = config.architecture == "transformer" || config.decoderKind == "transformer";
  AdamConfig c;
  if(transformer) {
    c.beta2 = Real(0.98);
    c.eps = Real(1e-9);
  }
  return c;
}

namespace {
int* adamFlag() { return Device::get().flags() + 1; }

std::shared_ptr<DeviceBuffer> zeroBuffer(int64_t n) {
  auto b = std::make_shared<DeviceBuffer>((size_t)n);
  MTKC(mtkc_memset(b->ptr, 0, (size_t)n * sizeof(float), Device::get().stream()));
  return b;
}

// grow a pool-layout buffer to n elements, keeping its prefix
void growTo(std::shared_ptr<DeviceBuffer>& b, int64_t& have, int64_t n) {
  if(b && have >= n)
    return;
  auto nb = zeroBuffer(n);
  if(b && have > 0)
    MTKC(mtkc_memcpy_d2d(nb->ptr, b->ptr, (size_t)have * sizeof(float), Device::get().stream()));
  b = nb;
  have = n;
}
}  // namespace

// ------------------------------------------------------------------ Adam

void Adam::ensure(ExpressionGraph& g) {
  int64_t n = g.pool().used();
  int64_t have = n_;
  growTo(m_, have, n);
  have = n_;
  growTo(v_, have, n);
  n_ = std::max(n_, n);
}

void Adam::resetMoments(ExpressionGraph& g, bool present) {
  ensure(g);
  haveMoments_ = present;
  Device& d = Device::get();
  MTKC(mtkc_memset(m_->ptr, 0, (size_t)n_ * sizeof(float), d.stream()));
  MTKC(mtkc_memset(v_->ptr, 0, (size_t)n_ * sizeof(float), d.stream()));
}

void Adam::launch(ExpressionGraph& g, Real lr, AveragedParameters* avg) {
  ensure(g);
  haveMoments_ = true;
  g.syncParamViews();  // host edits uploaded, host caches invalidated
  g.realizeParamGrads();
  Device& d = Device::get();
  int64_t n = g.pool().used();
  // While earlier updates are unchecked the flag stays sticky: once a
  // non-finite gradient is seen every later update is skipped on the device.
  if(!pending_)
    MTKC(mtkc_memset(adamFlag(), 0, sizeof(int), d.stream()));
  float* grads = g.pool().grads()->ptr;
  // a step whose forward/backward raised a device error (bad token id,
  // fully-masked softmax row, division by zero) must not train the model:
  // the reference throws before any update (graph.cpp:602-606)
  MTKC(mtkc_flag_or(adamFlag(), d.flags(), d.stream()));
  MTKC(mtkc_check_finite(grads, n, adamFlag(), d.stream()));
  int64_t step = step_ + 1;
  Real corr1 = Real(1) - (Real)std::pow((double)cfg_.beta1, (double)step);  // train.cpp:37-38
  Real corr2 = Real(1) - (Real)std::pow((double)cfg_.beta2, (double)step);
  float* avgPtr = avg ? avg->ensure(g) : nullptr;
  MTKC(mtkc_adam_ema(g.pool().values()->ptr, grads, m_->ptr, v_->ptr, avgPtr, n, lr, cfg_.beta1,
                     cfg_.beta2, cfg_.eps, corr1, corr2, avg ? avg->beta() : 0.f, avg ? 1 : 0,
                     /*zero_grad=*/0, adamFlag(), d.stream()));
  if(!pending_)
    verifiedStep_ = step_;
  step_ = step;
  pending_ = true;
  lastGraph_ = &g;
  g.zeroGrads();  // consumed by the update (train.cpp:57); lazily zero, memory kept
}

void Adam::checkDeferred() {
  if(!pending_)
    return;
  pending_ = false;
  Device& d = Device::get();
  int flag = 0;
  MTKC(mtkc_memcpy_d2h(&flag, adamFlag(), sizeof(int), d.stream()));
  d.sync();
  if(!flag) {
    verifiedStep_ = step_;
    return;
  }
  // the flag is sticky while updates are unchecked: every update after the
  // last verified one was skipped on the device (parameters unchanged)
  step_ = verifiedStep_;
  d.checkFlags("training step");  // device errors of the step: their own exception types
  if(!(flag & MTKC_FLAG_NONFINITE))
    throw NumericError("training step rejected by a device error; update aborted");
  ExpressionGraph& g = *lastGraph_;
  std::vector<float> host((size_t)g.pool().used());
  MTKC(mtkc_memcpy_d2h(host.data(), g.pool().grads()->ptr, host.size() * sizeof(float),
                       d.stream()));
  d.sync();
  std::string bad = "?";
  for(auto& name : g.paramNames()) {
    int64_t off = g.paramOffset(name), sz = g.paramValue(name).size();
    bool finite = true;
    for(int64_t i = 0; i < sz && finite; ++i)
      finite = std::isfinite(host[(size_t)(off + i)]);
    if(!finite) {
      bad = name;
      break;
    }
  }
  throw NumericError("non-finite gradient for parameter " + bad + "; update aborted");
}

void Adam::updateAsync(ExpressionGraph& g, Real lr, AveragedParameters* avg) {
  launch(g, lr, avg);
}

void Adam::update(ExpressionGraph& g, Real lr, AveragedParameters* avg) {
  launch(g, lr, avg);
  checkDeferred();
}

void Adam::updateTensor(const std::string& name, Tensor& value, const Tensor& grad, Real lr,
                        int64_t step) {
  if(!grad.allFinite())
    throw NumericError("non-finite gradient for parameter " + name + "; update aborted");
  auto it = single_.find(name);
  if(it == single_.end()) {
    Tensor m(value.shape()), v(value.shape());
    it = single_.emplace(name, std::make_pair(m, v)).first;
  }
  Tensor& m = it->second.first;
  Tensor& v = it->second.second;
  Real corr1 = Real(1) - (Real)std::pow((double)cfg_.beta1, (double)step);
  Real corr2 = Real(1) - (Real)std::pow((double)cfg_.beta2, (double)step);
  // a private copy of the gradient keeps the caller's tensor untouched
  Tensor gcopy = grad.copy();
  MTKC(mtkc_adam_ema(value.dev(), gcopy.dev(), m.dev(), v.dev(), nullptr, value.size(), lr,
                     cfg_.beta1, cfg_.beta2, cfg_.eps, corr1, corr2, 0.f, 0, 0, nullptr,
                     Device::get().stream()));
}

static Tensor poolView(ExpressionGraph& g, const std::shared_ptr<DeviceBuffer>& buf,
                       const std::string& name) {
  return Tensor(g.paramValue(name).shape(), buf, g.paramOffset(name));
}

Tensor Adam::firstMoment(ExpressionGraph& g, const std::string& name) {
  ensure(g);
  return poolView(g, m_, name);
}

Tensor Adam::secondMoment(ExpressionGraph& g, const std::string& name) {
  ensure(g);
  return poolView(g, v_, name);
}

Real LrSchedule::operator()(int64_t step) const {  // train.cpp:61-67
  if(step < 0)
    throw ContractError("negative lr step");
  if(step <= warmup)
    return base * (Real)step / (Real)warmup;
  return base * (Real)std::sqrt((double)warmup / (double)step);
}

// ---------------------------------------------------- AveragedParameters

float* AveragedParameters::ensure(ExpressionGraph& g) {
  growTo(buf_, n_, g.pool().used());
  return buf_->ptr;
}

void AveragedParameters::reset() {
  buf_.reset();
  n_ = 0;
}

void AveragedParameters::update(ExpressionGraph& g) {  // train.cpp:69-79
  g.syncParamViews();
  float* a = ensure(g);
  MTKC(mtkc_ema(a, g.pool().values()->ptr, g.pool().used(), beta_, Device::get().stream()));
}

void AveragedParameters::applyTo(ExpressionGraph& g) const {
  if(!buf_)
    return;
  g.syncParamViews();
  MTKC(mtkc_memcpy_d2d(g.pool().values()->ptr, buf_->ptr,
                       (size_t)std::min<int64_t>(n_, g.pool().used()) * sizeof(float),
                       Device::get().stream()));
}

Tensor AveragedParameters::value(ExpressionGraph& g, const std::string& name) {
  ensure(g);
  return poolView(g, buf_, name);
}

// ---------------------------------------------------------- distributed

namespace {
DistContext g_dist;
}

DistContext& distContext() { return g_dist; }

void setDistributed(int rank, int world, const void* ncclId128, bool forceComm) {
  Device::get();
  if(g_dist.comm) {  // re-initialisation (tests): drop the old communicator
    mtkc_nccl_comm_destroy(g_dist.comm);
    g_dist.comm = nullptr;
  }
  g_dist.rank = rank;
  g_dist.world = world;
  if(world > 1) {
    // SMs left to NCCL while buckets overlap the backward: NCCL's channels
    // are capped to match (defaults only; the user's NCCL_* settings win)
    const char* e = std::getenv("MTK_NCCL_SMS");
    g_dist.ncclSms = e ? std::max(0, std::atoi(e)) : 8;
    if(g_dist.ncclSms > 0) {
      std::string n = std::to_string(g_dist.ncclSms);
      setenv("NCCL_MAX_NCHANNELS", n.c_str(), 0);
      setenv("NCCL_MAX_CTAS", n.c_str(), 0);
    }
  }
  if(world > 1 || forceComm)
    MTKC(mtkc_nccl_comm_init(&g_dist.comm, world, rank, ncclId128));
}

int commRanks() {
  if(!g_dist.comm)
    return 1;
  int n = 0;
  MTKC(mtkc_nccl_comm_count(g_dist.comm, &n));
  return n;
}

// ---------------------------------------------------------- checkpoints

void saveCheckpoint(const std::string& path, const ModelConfig& config, ExpressionGraph& g,
                    Adam& adam, AveragedParameters& average, int64_t update, int64_t epoch,
                    int64_t batchIndex) {  // train.cpp:123-139
  adam.checkDeferred();
  std::vector<std::pair<std::string, Tensor>> tensors;
  for(auto& name : g.paramNames())
    tensors.emplace_back(name, g.paramValue(name));
  // the reference keeps moments / averages in std::maps: name order
  std::vector<std::string> sorted = g.paramNames();
  std::sort(sorted.begin(), sorted.end());
  if(adam.hasMoments()) {
    for(auto& name : sorted)
      tensors.emplace_back("adam.m." + name, adam.firstMoment(g, name));
    for(auto& name : sorted)
      tensors.emplace_back("adam.v." + name, adam.secondMoment(g, name));
  }
  if(!average.empty())
    for(auto& name : sorted)
      tensors.emplace_back("avg." + name, average.value(g, name));
  Tensor counters(Shape({4}), {(Real)update, (Real)epoch, (Real)batchIndex,
                               (Real)adam.step()});
  tensors.emplace_back("trainer.counters", counters);
  writeModelFile(path, config, tensors);
}

void loadCheckpoint(const std::string& path, ExpressionGraph& g, Adam& adam,
                    AveragedParameters& average, int64_t& update, int64_t& epoch,
                    int64_t& batchIndex) {  // train.cpp:141-164
  ModelFile file = readModelFile(path);
  loadParams(file, g);
  adam.checkDeferred();
  bool haveM = false, haveAvg = false;
  for(auto& [name, t] : file.tensors) {
    haveM = haveM || name.rfind("adam.m.", 0) == 0 || name.rfind("adam.v.", 0) == 0;
    haveAvg = haveAvg || name.rfind("avg.", 0) == 0;
  }
  // moments / averages absent from the file start from zero, as the
  // reference's cleared maps do at the next update
  adam.resetMoments(g, haveM);
  average.reset();
  if(haveAvg)
    average.ensure(g);
  for(auto& [name, t] : file.tensors) {
    auto fill = [&](Tensor dst, const char* what) {
      if(dst.shape() != t.shape())
        throw DataError(std::string(what) + " " + name + " shape mismatch in " + path);
      dst.copyFrom(t);
    };
    if(name.rfind("adam.m.", 0) == 0 && g.hasParam(name.substr(7)))
      fill(adam.firstMoment(g, name.substr(7)), "moment");
    else if(name.rfind("adam.v.", 0) == 0 && g.hasParam(name.substr(7)))
      fill(adam.secondMoment(g, name.substr(7)), "moment");
    else if(name.rfind("avg.", 0) == 0 && g.hasParam(name.substr(4)))
      fill(average.value(g, name.substr(4)), "average");
  }
  const Tensor* counters = file.find("trainer.counters");
  if(!counters || counters->size() != 4)
    throw DataError("checkpoint lacks trainer counters: " + path);
  update = (int64_t)counters->at(0);
  epoch = (int64_t)counters->at(1);
  batchIndex = (int64_t)counters->at(2);
  adam.setStep((int64_t)counters->at(3));
}

// ----------------------------------------------------------- training

uint64_t mixSeed(uint64_t seed, int64_t update, int worker) {  // train.cpp:170-176
  uint64_t h = hash64("update");
  h ^= seed + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h ^= (uint64_t)update * 0xbf58476d1ce4e5b9ull;
  h ^= (uint64_t)(worker + 1) * 0x94d049bb133111ebull;
  return h;
}

SyncStepper::SyncStepper(const Model& model, ExpressionGraph& g, Adam& adam,
                         AveragedParameters& avg, const TrainOptions& opts)
    : model_(model), g_(g), adam_(adam), avg_(avg), opts_(opts) {
  if(opts.workers < 1)
    throw ContractError("training needs at least one worker");
  lossAcc_ = std::make_shared<DeviceBuffer>(64);
  // pinned loss slots and their events for updatePipelined: allocated here,
  // not on the first pipelined call (a pinned allocation costs milliseconds)
  void* p = nullptr;
  MTKC(mtkc_host_alloc_pinned(&p, 4 * sizeof(float)));
  pinned_ = (float*)p;
  MTKC(mtkc_event_create(&slotEvent_[0]));
  MTKC(mtkc_event_create(&slotEvent_[1]));
}

const int* Adam::flagWord() { return adamFlag(); }

SyncStepper::~SyncStepper() {
  for(void* e : slotEvent_)
    if(e)
      mtkc_event_destroy(e);
  if(pinned_)
    mtkc_host_free_pinned(pinned_);
  for(void* e : events_)
    mtkc_event_destroy(e);
  if(commDone_)
    mtkc_event_destroy(commDone_);
  if(commStream_)
    mtkc_stream_destroy(commStream_);
}

std::vector<WorkerShare> rankShare(const std::vector<double>& tokens, int workers, int world,
                                   int rank) {
  if(world < 1 || rank < 0 || rank >= world)
    throw ContractError("rank outside the communicator");
  if(workers % world != 0)
    throw ContractError("workers must be a multiple of the number of ranks");
  const int take = (int)tokens.size();
  if(take < 1 || take > workers)
    throw ContractError("an update takes between 1 and `workers` batches");
  double total = 0;
  for(double t : tokens)
    total += t;
  const int L = workers / world;
  std::vector<WorkerShare> out;
  for(int j = 0; j < L; ++j) {
    int i = rank * L + j;
    if(i >= take)
      break;
    out.push_back({i, (Real)tokens[(size_t)i] / (Real)total});  // train.cpp:262-266
  }
  return out;
}

UpdateResult SyncStepper::update(const std::vector<const Batch*>& batches, int64_t updateIndex,
                                 bool readLoss) {
  DistContext& dc = distContext();
  int W = opts_.workers;
  int take = (int)batches.size();
  std::vector<double> tokens((size_t)take);
  double total = 0;
  for(int i = 0; i < take; ++i) {
    tokens[(size_t)i] = (double)batches[(size_t)i]->targetTokenCount();
    total += tokens[(size_t)i];
  }
  const std::vector<WorkerShare> share = rankShare(tokens, W, dc.world, dc.rank);
  Device& d = Device::get();
  MTKC(mtkc_memset(lossAcc_->ptr, 0, sizeof(float), d.stream()));
  g_.zeroGrads();
  const bool exchange = dc.comm != nullptr;
  const bool overlap = exchange && opts_.overlapAllreduce;
  if(overlap && !commStream_) {
    MTKC(mtkc_stream_create(&commStream_));
    MTKC(mtkc_event_create(&commDone_));
  }
  // the rank's last local worker (its backward finalises the gradients)
  const int lastLocal = (int)share.size() - 1;
  bool issuedAll = false;
  for(int j = 0; j < (int)share.size(); ++j) {
    const int i = share[(size_t)j].worker;
    g_.clear();
    g_.setSeed(mixSeed(opts_.seed, updateIndex, i));
    const Real w = share[(size_t)j].weight;
    g_.setLossScale(w);
    auto t0 = std::chrono::steady_clock::now();
    NodeRef loss = model_.buildLoss(g_, *batches[(size_t)i]);
    auto t1 = std::chrono::steady_clock::now();
    g_.forward();
    auto t2 = std::chrono::steady_clock::now();
    if(overlap && j == lastLocal) {
      // Bucketed all-reduce overlapped with the backward sweep: a bucket is
      // a contiguous range of the flat gradient pool; once the sweep has
      // passed the lowest-index consumer of every parameter in it, the
      // compute stream records an event and the comm stream all-reduces
      // the range while the backward continues.
      // Every rank issues the buckets in the same graph-independent order
      // (descending pool offset: parameters created last, whose gradients
      // the sweep finalises first, go first), each once it and all buckets
      // before it are final -- NCCL needs identical collective sequences
      // on all ranks, whatever each rank's batch shape.
      auto buckets = g_.gradBuckets(opts_.bucketElems);
      std::stable_sort(buckets.begin(), buckets.end(),
                       [](const ExpressionGraph::GradBucket& a,
                          const ExpressionGraph::GradBucket& b) { return a.begin > b.begin; });
      while(events_.size() < buckets.size()) {
        void* e = nullptr;
        MTKC(mtkc_event_create(&e));
        events_.push_back(e);
      }
      size_t next = 0;
      float* grads = g_.pool().grads()->ptr;
      auto issue = [&](size_t k) {
        const auto& b = buckets[k];
        g_.realizeParamGradsRange(b.begin, b.end);
        MTKC(mtkc_event_record(events_[k], d.stream()));
        MTKC(mtkc_stream_wait_event(commStream_, events_[k]));
        MTKC(mtkc_allreduce_sum(dc.comm, grads + b.begin, b.end - b.begin, commStream_));
        ++bucketsIssued_;
      };
      // from the first bucket on, the persistent GEMMs leave SMs to NCCL
      const bool capSms = dc.world > 1 && dc.ncclSms > 0;
      bool capped = false;
      auto issueCapped = [&](size_t k) {
        if(capSms && !capped) {
          int sms = 0;
          MTKC(mtkc_sm_count(&sms));
          MTKC(mtkc_gemm_set_sm_limit(std::max(1, sms - dc.ncclSms)));
          capped = true;
        }
        issue(k);
      };
      g_.backward(loss, [&](int node) {
        while(next < buckets.size() && buckets[next].readyAfter >= node)
          issueCapped(next++);
      });
      while(next < buckets.size())
        issueCapped(next++);
      if(capped)
        MTKC(mtkc_gemm_set_sm_limit(0));
      issuedAll = true;
    } else {
      g_.backward(loss);
    }
    auto t3 = std::chrono::steady_clock::now();
    hostTimes_[0] += std::chrono::duration<double, std::milli>(t1 - t0).count();
    hostTimes_[1] += std::chrono::duration<double, std::milli>(t2 - t1).count();
    hostTimes_[2] += std::chrono::duration<double, std::milli>(t3 - t2).count();
    MTKC(mtkc_axpy(lossAcc_->ptr, loss.val().devc(), w, 1, d.stream()));
  }
  g_.setLossScale(1);
  if(exchange) {
    if(issuedAll) {
      // compute stream waits for the last bucket before Adam reads the pool
      MTKC(mtkc_event_record(commDone_, commStream_));
      MTKC(mtkc_stream_wait_event(d.stream(), commDone_));
    } else if(overlap) {
      // rank without a batch at the epoch tail: zero gradients, the same
      // bucket sequence as the working ranks (identical collective order)
      g_.realizeParamGrads();
      auto buckets = g_.gradBuckets(opts_.bucketElems);
      std::stable_sort(buckets.begin(), buckets.end(),
                       [](const ExpressionGraph::GradBucket& a,
                          const ExpressionGraph::GradBucket& b) { return a.begin > b.begin; });
      float* grads = g_.pool().grads()->ptr;
      for(auto& b : buckets)
        MTKC(mtkc_allreduce_sum(dc.comm, grads + b.begin, b.end - b.begin, d.stream()));
    } else {
      // overlap disabled: the whole pool in one all-reduce
      g_.realizeParamGrads();
      MTKC(mtkc_allreduce_sum(dc.comm, g_.pool().grads()->ptr, g_.pool().used(), d.stream()));
    }
    MTKC(mtkc_allreduce_sum(dc.comm, lossAcc_->ptr, 1, d.stream()));
  }
  Real lr = opts_.lr(adam_.step() + 1);
  adam_.updateAsync(g_, lr, &avg_);
  UpdateResult r;
  r.tokens = total;
  if(readLoss) {
    float l = 0;
    MTKC(mtkc_memcpy_d2h(&l, lossAcc_->ptr, sizeof(float), d.stream()));
    adam_.checkDeferred();  // synchronises
    d.checkFlags("training step");
    r.loss = l;
  }
  return r;
}

UpdateResult SyncStepper::collect(int slot) {
  UpdateResult r;
  r.tokens = slotTokens_[slot];
  MTKC(mtkc_event_sync(slotEvent_[slot]));
  const int flag = reinterpret_cast<const int*>(pinned_)[2 * slot + 1];
  if(flag) {
    pipeCount_ = 0;  // the pipeline restarts after the error
    adam_.checkDeferred();  // synchronises, rolls back the skipped updates, throws
  }
  adam_.markVerified(slotStep_[slot]);
  r.loss = pinned_[2 * slot];
  return r;
}

UpdateResult SyncStepper::updatePipelined(const std::vector<const Batch*>& batches,
                                          int64_t updateIndex) {
  Device& d = Device::get();
  UpdateResult launched = update(batches, updateIndex, false);
  const int slot = (int)(pipeCount_ & 1);
  MTKC(mtkc_memcpy_d2h(pinned_ + 2 * slot, lossAcc_->ptr, sizeof(float), d.stream()));
  MTKC(mtkc_memcpy_d2h(pinned_ + 2 * slot + 1, Adam::flagWord(), sizeof(int), d.stream()));
  MTKC(mtkc_event_record(slotEvent_[slot], d.stream()));
  slotTokens_[slot] = launched.tokens;
  slotStep_[slot] = adam_.step();
  ++pipeCount_;
  if(pipeCount_ == 1) {
    UpdateResult r;
    r.loss = std::nan("");
    return r;
  }
  return collect(1 - slot);  // the previous update
}

UpdateResult SyncStepper::flushPipelined() {
  if(pipeCount_ == 0)
    return UpdateResult{};
  UpdateResult r = collect((int)((pipeCount_ - 1) & 1));
  pipeCount_ = 0;
  Device::get().checkFlags("training step");
  return r;
}

namespace {
void logLine(const TrainOptions& opts, int64_t update, int64_t epoch, double loss, Real lr,
             double wps) {
  if(!opts.log || opts.logEvery <= 0 || update % opts.logEvery != 0)
    return;
  (*opts.log) << "update=" << update << " epoch=" << epoch << " loss=" << loss
              << " lr=" << (double)lr << " wps=" << wps << "\n";
}

// trainAsync (train.cpp:302-404) on one GPU.  The reference's hogwild
// workers are threads that read a shared parameter store, compute one
// batch's gradients and update the store per tensor under a lock, in
// whatever order they finish.  Here W worker graphs run in rounds: every
// worker of a round reads the shared (master) parameters, computes its
// batch (flat epoch-major batch list, seed mixSeed(seed, batch + update, 0)
// as train.cpp:343), then the updates are applied to the master in worker
// order -- one admissible interleaving of the reference's threads, each
// update computed on parameters at most W-1 updates old.  W = 1 is
// deterministic and equals the reference's single-worker run.
TrainResult trainAsyncB200(Model& model, const std::vector<Example>& data,
                           ExpressionGraph& master, Adam& adam, AveragedParameters& average,
                           const TrainOptions& opts, int64_t update, int64_t startEpoch,
                           int64_t startBatch) {
  std::vector<Batch> batches;
  std::vector<int64_t> epochOf;
  for(int64_t epoch = startEpoch; epoch < opts.epochs; ++epoch) {
    BatchOptions bo;
    bo.tokenBudget = opts.tokenBudget;
    bo.seed = opts.seed + (uint64_t)epoch;
    bo.shuffle = true;
    auto eb = makeBatches(data, bo);  // epochBatches, train.cpp:183-190
    for(size_t i = epoch == startEpoch ? (size_t)startBatch : 0; i < eb.size(); ++i) {
      batches.push_back(std::move(eb[i]));
      epochOf.push_back(epoch);
    }
  }
  const int W = opts.workers;
  std::vector<std::unique_ptr<ExpressionGraph>> workers;
  for(int w = 0; w < W; ++w) {
    workers.push_back(std::make_unique<ExpressionGraph>(opts.seed));
    model.registerParams(*workers.back());
  }
  Device& dev = Device::get();
  const size_t bytes = (size_t)master.pool().used() * sizeof(float);
  TrainResult res;
  double lastLoss = 0;
  int64_t tokensSeen = 0;
  auto t0 = std::chrono::steady_clock::now();
  for(size_t i = 0; i < batches.size();) {
    int64_t take = std::min<int64_t>(W, (int64_t)(batches.size() - i));
    if(opts.maxUpdates >= 0)
      take = std::min<int64_t>(take, opts.maxUpdates - ((int64_t)i + update));
    if(take <= 0)
      break;
    master.syncParamViews();
    std::vector<NodeRef> losses((size_t)take);
    std::vector<Real> tokens((size_t)take, 0);
    for(int64_t k = 0; k < take; ++k) {  // read the store, compute the batch
      ExpressionGraph& g = *workers[(size_t)k];
      g.syncParamViews();
      MTKC(mtkc_memcpy_d2d(g.pool().values()->ptr, master.pool().values()->ptr, bytes,
                           dev.stream()));
      g.clear();
      g.setSeed(mixSeed(opts.seed, (int64_t)i + k + update, 0));
      losses[(size_t)k] = model.buildLoss(g, batches[i + (size_t)k], &tokens[(size_t)k]);
      g.forward();
      g.zeroGrads();
      g.backward(losses[(size_t)k]);
      g.realizeParamGrads();
    }
    for(int64_t k = 0; k < take; ++k) {  // apply the updates in worker order
      ExpressionGraph& g = *workers[(size_t)k];
      master.realizeParamGrads();
      MTKC(mtkc_memcpy_d2d(master.pool().grads()->ptr, g.pool().grads()->ptr, bytes,
                           dev.stream()));
      const int64_t step = adam.step() + 1;
      const Real lr = opts.lr(step);
      adam.update(master, lr, &average);
      lastLoss = (double)losses[(size_t)k].val().at(0);
      tokensSeen += (int64_t)tokens[(size_t)k];
      double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      logLine(opts, step, epochOf[i + (size_t)k], lastLoss, lr,
              secs > 0 ? (double)tokensSeen / secs : 0);
    }
    i += (size_t)take;
  }
  res.updates = adam.step();
  res.epochs = opts.epochs;
  res.finalLoss = lastLoss;
  if(!opts.checkpointPath.empty())
    saveCheckpoint(opts.checkpointPath, model.config, master, adam, average, res.updates,
                   opts.epochs, 0);
  return res;
}
}  // namespace

TrainResult train(Model& model, const std::vector<Example>& data, ExpressionGraph& master,
                  Adam& adam, AveragedParameters& average, const TrainOptions& opts) {
  // train.cpp:407-418 + trainSync :200-300
  if(opts.workers < 1)
    throw ContractError("training needs at least one worker");
  model.registerParams(master);
  master.clear();
  int64_t update = 0, startEpoch = 0, startBatch = 0;
  if(!opts.resumeFrom.empty())
    loadCheckpoint(opts.resumeFrom, master, adam, average, update, startEpoch, startBatch);
  if(opts.async) {
    if(distContext().world > 1)
      throw ContractError("asynchronous training runs on one process (world size 1)");
    return trainAsyncB200(model, data, master, adam, average, opts, update, startEpoch,
                          startBatch);
  }
  SyncStepper stepper(model, master, adam, average, opts);
  TrainResult res;
  auto t0 = std::chrono::steady_clock::now();
  int64_t tokensSeen = 0;
  for(int64_t epoch = startEpoch; epoch < opts.epochs; ++epoch) {
    BatchOptions bo;
    bo.tokenBudget = opts.tokenBudget;
    bo.seed = opts.seed + (uint64_t)epoch;
    bo.shuffle = true;
    auto batches = makeBatches(data, bo);  // epochBatches, train.cpp:183-190
    double epochLoss = 0;
    int64_t epochUpdates = 0;
    for(size_t idx = (epoch == startEpoch ? (size_t)startBatch : 0); idx < batches.size();) {
      int take = (int)std::min<size_t>((size_t)opts.workers, batches.size() - idx);
      std::vector<const Batch*> ptrs;
      for(int i = 0; i < take; ++i)
        ptrs.push_back(&batches[idx + (size_t)i]);
      Real lr = opts.lr(adam.step() + 1);
      UpdateResult r = stepper.update(ptrs, update);
      ++update;
      idx += (size_t)take;
      epochLoss += r.loss;
      ++epochUpdates;
      tokensSeen += (int64_t)r.tokens;
      double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      logLine(opts, update, epoch, r.loss, lr, secs > 0 ? (double)tokensSeen / secs : 0);
      if(!opts.checkpointPath.empty() && opts.checkpointEvery > 0 &&
         update % opts.checkpointEvery == 0 && distContext().rank == 0)
        saveCheckpoint(opts.checkpointPath, model.config, master, adam, average, update, epoch,
                       (int64_t)idx);
      if(opts.maxUpdates >= 0 && update >= opts.maxUpdates) {
        res.updates = update;
        res.epochs = epoch + 1;
        res.finalLoss = epochUpdates ? epochLoss / (double)epochUpdates : 0;
        return res;
      }
    }
    res.finalLoss = epochUpdates ? epochLoss / (double)epochUpdates : res.finalLoss;
    res.epochs = epoch + 1;
  }
  res.updates = update;
  return res;
}

}  // namespace mtk
