// Optimiser, schedule, parameter averaging and synchronous data-parallel
// training (reference: include/mtk/train.h, src/train.cpp).
//
// B200 design: every parameter, gradient, Adam moment and EMA shadow is one
// flat device buffer in the graph's parameter-pool layout, so the update is
// one fused kernel (Adam + EMA, 36 B/param) and the data-parallel exchange
// is one NCCL all-reduce over the flat gradient buffer.  Worker gradients
// are pre-weighted by tokens_i/total through the backward seed, which makes
// the all-reduce sum equal the reference's worker-ordered weighted combine
// (train.cpp:254-269).
#pragma once

#include <iosfwd>
#include <algorithm>
#include <map>

#include "mtk/serialize.h"

namespace mtk {

struct AdamConfig {
  Real beta1 = Real(0.9);
  Real beta2 = Real(0.999);
  Real eps = Real(1e-8);
};

AdamConfig adamDefaultsFor(const ModelConfig& config);

class AveragedParameters;

class Adam {
public:
  explicit Adam(AdamConfig config = AdamConfig()) : cfg_(config) {}

  // One update from the accumulated gradients, then zero them
  // (train.cpp:49-59).  Throws NumericError and leaves every parameter
  // untouched if any gradient is non-finite.  When `avg` is given the EMA
  // update is fused into the same pass.
  void update(ExpressionGraph& g, Real lr, AveragedParameters* avg = nullptr);
  // Same, but the non-finite check is deferred to checkDeferred() (no host
  // synchronisation inside the step).
  void updateAsync(ExpressionGraph& g, Real lr, AveragedParameters* avg = nullptr);
  void checkDeferred();
  // every update up to and including optimizer step `step` was verified
  // error-free on the device (pipelined loss read): none of them counts
  // toward a rollback any more
  void markVerified(int64_t step) { verifiedStep_ = std::max(verifiedStep_, step); }
  // device word of the pending updates: MTKC_FLAG_NONFINITE for a non-finite
  // gradient, plus the device error bits of the step (bad ids, fully-masked
  // rows, division by zero) -- any bit makes the update a no-op
  static const int* flagWord();
  // Single-tensor variant (train.cpp:30-47) with its own moments per name.
  void updateTensor(const std::string& name, Tensor& value, const Tensor& grad, Real lr,
                    int64_t step);

  int64_t step() const { return step_; }
  const AdamConfig& config() const { return cfg_; }
  void setStep(int64_t s) { step_ = verifiedStep_ = s; }
  // moment views for checkpointing (names in graph order)
  Tensor firstMoment(ExpressionGraph& g, const std::string& name);
  Tensor secondMoment(ExpressionGraph& g, const std::string& name);
  // moments exist once an update ran or a checkpoint supplied them
  bool hasMoments() const { return haveMoments_; }
  void resetMoments(ExpressionGraph& g, bool present);  // zero m, v (checkpoint load)

private:
  void ensure(ExpressionGraph& g);
  void launch(ExpressionGraph& g, Real lr, AveragedParameters* avg);
  AdamConfig cfg_;
  int64_t step_ = 0;
  std::shared_ptr<DeviceBuffer> m_, v_;
  int64_t n_ = 0;
  bool haveMoments_ = false;
  bool pending_ = false;
  int64_t verifiedStep_ = 0;  // last optimizer step known to have been applied
  ExpressionGraph* lastGraph_ = nullptr;
  std::map<std::string, std::pair<Tensor, Tensor>> single_;  // updateTensor moments
};

struct LrSchedule {
  Real base = Real(0.0003);
  int64_t warmup = 16000;
  Real operator()(int64_t step) const;
};

class AveragedParameters {
public:
  explicit AveragedParameters(Real beta = Real(0.9999)) : beta_(beta) {}
  void update(ExpressionGraph& g);  // avg <- beta*avg + (1-beta)*params
  void applyTo(ExpressionGraph& g) const;
  bool empty() const { return !buf_; }
  Real beta() const { return beta_; }
  Tensor value(ExpressionGraph& g, const std::string& name);
  float* ensure(ExpressionGraph& g);  // flat shadow in pool layout (zero-initialised)
  void reset();                       // drop the shadow (next update starts from zero)

private:
  Real beta_;
  std::shared_ptr<DeviceBuffer> buf_;
  int64_t n_ = 0;
};

// Data-parallel context: one process per GPU; `workers` in TrainOptions is
// the total worker count across ranks (the reference's threads).
struct DistContext {
  int rank = 0;
  int world = 1;
  void* comm = nullptr;  // ncclComm_t
  int ncclSms = 0;       // SMs the GEMMs leave to NCCL while buckets overlap the backward
};
// world == 1 with forceComm creates a one-rank NCCL communicator, so the
// exchange path (buckets, streams, events) runs on a single GPU too.
void setDistributed(int rank, int world, const void* ncclId128, bool forceComm = false);
DistContext& distContext();
// ranks in the NCCL communicator (1 without one)
int commRanks();

struct TrainOptions {
  int workers = 1;
  bool async = false;
  int64_t tokenBudget = 256;
  uint64_t seed = 1;
  int64_t epochs = 1;
  int64_t maxUpdates = -1;
  LrSchedule lr;
  Real averageBeta = Real(0.9999);
  std::string checkpointPath;
  int64_t checkpointEvery = 0;
  std::string resumeFrom;
  int64_t logEvery = 0;
  std::ostream* log = nullptr;
  // data-parallel gradient exchange: bucketed NCCL all-reduces issued on a
  // communication stream during the backward sweep (each bucket as soon as
  // its gradients are final), or one all-reduce after the backward
  bool overlapAllreduce = true;
  int64_t bucketElems = (int64_t)8 << 20;  // 32 MiB of fp32 gradients
};

struct TrainResult {
  int64_t updates = 0;
  int64_t epochs = 0;
  double finalLoss = 0;
};

// One synchronous update: this rank's share of `batches` (worker i =
// rank*L + j handles batches[i]), weighted gradients, NCCL all-reduce,
// fused Adam + EMA.  Stateless apart from the objects passed in.
struct UpdateResult {
  double loss = 0;   // token-weighted mean loss over all workers
  double tokens = 0;  // total target tokens of the update
};
class SyncStepper {
public:
  SyncStepper(const Model& model, ExpressionGraph& g, Adam& adam, AveragedParameters& avg,
              const TrainOptions& opts);
  // launches the update; the returned loss is read from the device
  // (one synchronisation) unless `readLoss` is false.
  UpdateResult update(const std::vector<const Batch*>& batches, int64_t updateIndex,
                      bool readLoss = true);
  // Pipelined variant for training loops: launches update `updateIndex`,
  // queues an asynchronous copy of its loss (and of the non-finite flag) to
  // pinned host memory, then waits only for the PREVIOUS update's copy and
  // returns that update's result (loss NaN on the first call).  The host
  // stays one update ahead of the device; errors surface one update late.
  UpdateResult updatePipelined(const std::vector<const Batch*>& batches, int64_t updateIndex);
  // result of the last pipelined update (waits for it)
  UpdateResult flushPipelined();
  // accumulated host milliseconds in graph build / forward / backward
  std::vector<double> hostTimes() const { return {hostTimes_[0], hostTimes_[1], hostTimes_[2]}; }

private:
  double hostTimes_[3] = {0, 0, 0};
  const Model& model_;
  ExpressionGraph& g_;
  Adam& adam_;
  AveragedParameters& avg_;
  TrainOptions opts_;
  std::shared_ptr<DeviceBuffer> lossAcc_;
  void* commStream_ = nullptr;       // NCCL stream (bucketed all-reduce)
  std::vector<void*> events_;        // compute -> comm "bucket ready" events
  void* commDone_ = nullptr;         // comm -> compute "exchange finished"
  int64_t bucketsIssued_ = 0;        // telemetry (tests)
  // pipelined loss read: two pinned slots {loss, flag} and their events
  float* pinned_ = nullptr;
  void* slotEvent_[2] = {nullptr, nullptr};
  double slotTokens_[2] = {0, 0};
  int64_t slotStep_[2] = {0, 0};     // optimizer step each slot's update launched
  int64_t pipeCount_ = 0;
  UpdateResult collect(int slot);

public:
  int64_t bucketsIssued() const { return bucketsIssued_; }
  ~SyncStepper();
};

uint64_t mixSeed(uint64_t seed, int64_t update, int worker);

// The workers one rank runs in a synchronous update (train.cpp:221-269):
// worker i handles batches[i]; with L = workers / world, rank r runs workers
// r*L .. r*L+L-1 that have a batch (ranks past the epoch tail run none and
// contribute zero gradients), each weighted tokens_i / total -- the weights
// of all ranks sum to 1, so the NCCL sum of the pre-scaled gradients is the
// reference's combine.  Pure host logic: identical on every rank.
struct WorkerShare {
  int worker;
  Real weight;
};
std::vector<WorkerShare> rankShare(const std::vector<double>& tokens, int workers, int world,
                                   int rank);

// Checkpoints (train.cpp:121-164): parameters, then "adam.m.<name>",
// "adam.v.<name>" and "avg.<name>" in name order once they exist, then
// "trainer.counters" = {update, epoch, batchIndex, adam step} -- the
// reference's MTK1 layout, so checkpoints move between the two builds.
void saveCheckpoint(const std::string& path, const ModelConfig& config, ExpressionGraph& g,
                    Adam& adam, AveragedParameters& average, int64_t update, int64_t epoch,
                    int64_t batchIndex);
void loadCheckpoint(const std::string& path, ExpressionGraph& g, Adam& adam,
                    AveragedParameters& average, int64_t& update, int64_t& epoch,
                    int64_t& batchIndex);

TrainResult train(Model& model, const std::vector<Example>& data, ExpressionGraph& master,
                  Adam& adam, AveragedParameters& average, const TrainOptions& opts);

}  // namespace mtk
