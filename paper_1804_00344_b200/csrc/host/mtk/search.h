// Decoding on the training kernels (reference include/mtk/search.h, §8(f)3):
// lockstep batched beam search over an ensemble and forced-decoding scores.
// The decoder steps run on the device (Decoder::step one token at a time,
// DecoderState::select to reorder hypotheses); the per-step log-softmax and
// candidate selection follow the reference's host arithmetic (double
// precision, same tie rules), so n-best lists match it.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "mtk/models.h"

namespace mtk {

struct Scorer {
  std::string name;
  const Model* model = nullptr;
  ExpressionGraph* graph = nullptr;
  double weight = 1.0;
};

struct Hypothesis {
  std::vector<int32_t> tokens;  // no start symbol; trailing </s> when emitted
  double score = 0;             // ensemble-mean log-probability
  std::vector<double> tokenScores;
  std::vector<std::pair<std::string, double>> components;  // per-scorer totals
};

struct SearchOptions {
  int beamSize = 5;
  double alpha = 0.6;           // rank by score / length^alpha
  int nBest = 1;
  int64_t maxLengthFactor = 3;  // times the source length
  int64_t maxLengthBase = 50;   // cap for models without a source
};

std::vector<std::vector<Hypothesis>> beamSearch(const std::vector<Scorer>& scorers,
                                                const Batch& batch, const SearchOptions& opts);
std::vector<Hypothesis> scoreBatch(const Scorer& scorer, const Batch& batch);

struct TranslateOptions : SearchOptions {
  int64_t tokenBudget = 512;
};

struct TranslateOutput {
  std::vector<std::string> best;               // one line per input, input order
  std::vector<std::string> nbestLines;         // "id ||| text ||| F0=.. ||| score"
  std::vector<std::vector<Hypothesis>> nbest;  // per input, ranked
  double wordsPerSecond = 0;
};

// A corpus: length-sorted batches, beam search, original order restored,
// right-to-left output re-inverted (reference search.cpp:285-349).
TranslateOutput translateLines(const std::vector<Scorer>& scorers, const Vocabulary& targetVocab,
                               const std::vector<std::vector<std::string>>& sourceStreams,
                               const std::vector<Vocabulary>& sourceVocabs,
                               const TranslateOptions& opts);
std::string formatNBestLine(size_t id, const std::string& text, const Hypothesis& h);

double lengthNormalizedScore(const Hypothesis& h, double alpha);
void rankHypotheses(std::vector<Hypothesis>& hyps, double alpha);

}  // namespace mtk
