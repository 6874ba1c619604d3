// Token-budget batching, bit-exact with the reference (src/data.cpp:149-282).
#include "mtk/data.h"

#include <algorithm>

namespace mtk {

int64_t Batch::sourceTokenCount() const {
  if(sourceMasks.empty())
    return 0;
  int64_t n = 0;
  for(Real v : sourceMasks[0].toVector())
    n += v != 0;
  return n;
}

int64_t Batch::targetTokenCount() const {
  if(!hasTarget)
    return 0;
  int64_t n = 0;
  for(Real v : targetMask.toVector())
    n += v != 0;
  return n;
}

namespace {

// Pad one stream: every row gets its tokens then one </s>; extent is the
// longest (len + 1), at least 1 (data.cpp:149-166).
void padStream(const std::vector<const std::vector<int32_t>*>& seqs, IntMat& ids, Tensor& mask) {
  int64_t b = (int64_t)seqs.size();
  int64_t width = 1;
  for(auto* s : seqs)
    width = std::max<int64_t>(width, (int64_t)s->size() + 1);
  ids = IntMat(b, width);
  std::vector<Real> m((size_t)(b * width), Real(0));
  for(int64_t r = 0; r < b; ++r) {
    const auto& s = *seqs[(size_t)r];
    std::copy(s.begin(), s.end(), ids.data.begin() + r * width);
    ids.at(r, (int64_t)s.size()) = Vocabulary::kEos;
    std::fill(m.begin() + r * width, m.begin() + r * width + (int64_t)s.size() + 1, Real(1));
  }
  mask = Tensor(Shape({b, width}), std::move(m));
}

int64_t streamLen(const Example& ex, size_t stream, bool target) {
  return (int64_t)(target ? ex.target.size() : ex.sources[stream].size()) + 1;
}

// Padded slot count of a group with per-stream running maxima
// (paddedCost, data.cpp:193-215).
struct GroupCost {
  std::vector<int64_t> srcMax;
  int64_t tgtMax = 1;
  int64_t rows = 0;
  bool hasTarget = false;

  explicit GroupCost(const Example& first)
      : srcMax(first.sources.size(), 1), hasTarget(first.hasTarget) {}
  int64_t costWith(const Example* ex) const {
    int64_t b = rows + (ex ? 1 : 0);
    int64_t total = 0;
    for(size_t s = 0; s < srcMax.size(); ++s)
      total += b * std::max(srcMax[s], ex ? streamLen(*ex, s, false) : 1);
    if(hasTarget)
      total += b * std::max(tgtMax, ex ? streamLen(*ex, 0, true) : 1);
    return total;
  }
  void add(const Example& ex) {
    for(size_t s = 0; s < srcMax.size(); ++s)
      srcMax[s] = std::max(srcMax[s], streamLen(ex, s, false));
    if(hasTarget)
      tgtMax = std::max(tgtMax, streamLen(ex, 0, true));
    ++rows;
  }
};

int64_t exampleLength(const Example& ex) {  // data.cpp:217-224
  int64_t n = 0;
  for(auto& s : ex.sources)
    n += (int64_t)s.size() + 1;
  if(ex.hasTarget)
    n += (int64_t)ex.target.size() + 1;
  return n;
}

}  // namespace

Batch padBatch(const std::vector<const Example*>& group) {
  if(group.empty())
    throw ContractError("cannot pad an empty batch");
  size_t arity = group[0]->sources.size();
  Batch batch;
  batch.sourceIds.resize(arity);
  batch.sourceMasks.resize(arity);
  std::vector<const std::vector<int32_t>*> seqs(group.size());
  for(size_t s = 0; s < arity; ++s) {
    for(size_t i = 0; i < group.size(); ++i)
      seqs[i] = &group[i]->sources[s];
    padStream(seqs, batch.sourceIds[s], batch.sourceMasks[s]);
  }
  batch.hasTarget = group[0]->hasTarget;
  if(batch.hasTarget) {
    for(size_t i = 0; i < group.size(); ++i)
      seqs[i] = &group[i]->target;
    padStream(seqs, batch.targetIds, batch.targetMask);
  }
  for(auto* ex : group)
    batch.sentenceIds.push_back(ex->id);
  return batch;
}

std::vector<Batch> makeBatches(const std::vector<Example>& examples, const BatchOptions& opts,
                               size_t* skippedCount) {
  size_t skipped = 0;
  std::vector<const Example*> order;
  order.reserve(examples.size());
  for(auto& ex : examples) {
    GroupCost lone(ex);
    if(lone.costWith(&ex) > opts.tokenBudget) {
      ++skipped;
      continue;
    }
    order.push_back(&ex);
  }
  if(opts.shuffle) {
    Rng rng(opts.seed);
    std::shuffle(order.begin(), order.end(), rng);
  }
  size_t window = opts.sortWindow;
  if(window == 0) {
    int64_t avgLen = 1;
    if(!order.empty()) {
      int64_t total = 0;
      for(auto* ex : order)
        total += exampleLength(*ex);
      avgLen = std::max<int64_t>(1, total / (int64_t)order.size());
    }
    window = (size_t)std::max<int64_t>(1, 100 * opts.tokenBudget / avgLen);
  }
  std::vector<Batch> batches;
  std::vector<const Example*> win, group;
  for(size_t start = 0; start < order.size(); start += window) {
    size_t end = std::min(order.size(), start + window);
    win.assign(order.begin() + (long)start, order.begin() + (long)end);
    std::stable_sort(win.begin(), win.end(), [](const Example* a, const Example* b) {
      return exampleLength(*a) < exampleLength(*b);
    });
    group.clear();
    std::unique_ptr<GroupCost> cost;
    for(auto* ex : win) {
      if(!group.empty() && cost->costWith(ex) > opts.tokenBudget) {
        batches.push_back(padBatch(group));
        group.clear();
      }
      if(group.empty())
        cost = std::make_unique<GroupCost>(*ex);
      group.push_back(ex);
      cost->add(*ex);
    }
    if(!group.empty())
      batches.push_back(padBatch(group));
  }
  if(opts.shuffle) {
    Rng rng(opts.seed ^ 0x9e3779b97f4a7c15ull);
    std::shuffle(batches.begin(), batches.end(), rng);
  }
  if(skippedCount)
    *skippedCount = skipped;
  return batches;
}

}  // namespace mtk
