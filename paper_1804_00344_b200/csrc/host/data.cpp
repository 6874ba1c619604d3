// Token-budget batching, bit-exact with the reference (src/data.cpp:149-282).
#include "mtk/data.h"

#include <algorithm>
#include <fstream>
#include <sstream>

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

// ----------------------------------------------------------- Vocabulary
// (reference data.cpp:13-122; same reserved ids, ordering and errors)

Vocabulary::Vocabulary() {
  add("</s>");
  add("<unk>");
}

void Vocabulary::add(const std::string& token) {
  if(tok2id_.count(token))
    throw DataError("duplicate token in vocabulary: " + token);
  tok2id_[token] = (int32_t)id2tok_.size();
  id2tok_.push_back(token);
}

namespace {
std::vector<std::string> splitTokens(const std::string& line) {
  std::vector<std::string> out;
  std::istringstream is(line);
  std::string tok;
  while(is >> tok)
    out.push_back(tok);
  return out;
}
}  // namespace

Vocabulary Vocabulary::build(const std::vector<std::string>& corpusPaths, size_t maxSize) {
  std::unordered_map<std::string, int64_t> freq;
  bool any = false;
  for(auto& path : corpusPaths)
    for(auto& line : readLines(path))
      for(auto& tok : splitTokens(line)) {
        ++freq[tok];
        any = true;
      }
  if(!any)
    throw DataError("cannot build a vocabulary from an empty corpus");
  std::vector<std::pair<std::string, int64_t>> sorted(freq.begin(), freq.end());
  std::sort(sorted.begin(), sorted.end(), [](const auto& a, const auto& b) {
    if(a.second != b.second)
      return a.second > b.second;  // descending frequency
    return a.first < b.first;      // ties lexicographic
  });
  Vocabulary v;
  for(auto& [tok, n] : sorted) {
    if((size_t)v.size() >= maxSize)
      break;
    if(tok == "</s>" || tok == "<unk>")
      throw DataError("reserved token redefined in corpus: " + tok);
    v.add(tok);
  }
  return v;
}

Vocabulary Vocabulary::load(const std::string& path) {
  std::ifstream in(path);
  if(!in)
    throw IoError("cannot open vocabulary file: " + path);
  Vocabulary v;
  v.id2tok_.clear();
  v.tok2id_.clear();
  std::string line;
  while(std::getline(in, line)) {
    if(!line.empty() && line.back() == '\r')
      line.pop_back();
    v.add(line);
  }
  if(v.size() < 2 || v.id2tok_[0] != "</s>" || v.id2tok_[1] != "<unk>")
    throw DataError("vocabulary file must start with </s> and <unk>: " + path);
  return v;
}

void Vocabulary::save(const std::string& path) const {
  std::ofstream out(path);
  if(!out)
    throw IoError("cannot write vocabulary file: " + path);
  for(auto& tok : id2tok_)
    out << tok << "\n";
}

int32_t Vocabulary::id(const std::string& token) const {
  auto it = tok2id_.find(token);
  return it == tok2id_.end() ? kUnk : it->second;
}

const std::string& Vocabulary::token(int32_t id) const {
  if(id < 0 || id >= size())
    throw DataError("token id out of range: " + std::to_string(id));
  return id2tok_[(size_t)id];
}

std::vector<int32_t> Vocabulary::encode(const std::string& line) const {
  std::vector<int32_t> out;
  for(auto& tok : splitTokens(line))
    out.push_back(id(tok));
  return out;
}

std::string Vocabulary::decode(const std::vector<int32_t>& ids) const {
  std::string out;
  for(size_t i = 0; i < ids.size(); ++i) {
    if(ids[i] == kEos)
      break;
    if(!out.empty())
      out += ' ';
    out += token(ids[i]);
  }
  return out;
}

// ------------------------------------------------------------- corpus IO

std::vector<std::string> readLines(const std::string& path) {
  std::ifstream in(path);
  if(!in)
    throw IoError("cannot open file: " + path);
  std::vector<std::string> lines;
  std::string line;
  while(std::getline(in, line)) {
    if(!line.empty() && line.back() == '\r')
      line.pop_back();
    lines.push_back(line);
  }
  return lines;
}

std::vector<Example> readParallelCorpus(const std::vector<std::string>& sourcePaths,
                                        const std::string& targetPath,
                                        const std::vector<const Vocabulary*>& sourceVocabs,
                                        const Vocabulary* targetVocab) {
  std::vector<std::vector<std::string>> sourceLines;
  for(auto& p : sourcePaths)
    sourceLines.push_back(readLines(p));
  std::vector<std::string> targetLines;
  if(!targetPath.empty())
    targetLines = readLines(targetPath);
  size_t n = sourceLines.empty() ? targetLines.size() : sourceLines[0].size();
  for(auto& s : sourceLines)
    if(s.size() != n)
      throw DataError("corpus streams are not sentence-aligned");
  if(!targetPath.empty() && targetLines.size() != n)
    throw DataError("target corpus not aligned with source corpus");
  std::vector<Example> out;
  for(size_t i = 0; i < n; ++i) {
    Example ex;
    ex.id = i;
    for(size_t s = 0; s < sourceLines.size(); ++s)
      ex.sources.push_back(sourceVocabs[s]->encode(sourceLines[s][i]));
    if(!targetPath.empty()) {
      ex.target = targetVocab->encode(targetLines[i]);
      ex.hasTarget = true;
    }
    out.push_back(std::move(ex));
  }
  return out;
}

std::vector<int32_t> invertR2l(std::vector<int32_t> tokens) {
  std::reverse(tokens.begin(), tokens.end());
  return tokens;
}

}  // namespace mtk
