// mtk-b200: the reference's `mtk` command line (tools/mtk.cpp) for the
// training path, on the B200 backend.
//
// Subcommands: vocab, train, translate, score; same option names,
// defaults, `--config` option files (key: value per line, command line wins,
// tools/mtk.cpp:429-456) and exit codes: 0 success, 1 usage error, 2 data/io
// error, 3 numeric error (tools/mtk.cpp:546-594).  CLI11 (absent from the
// reference tree) is replaced by a small option table.  rescore / bleu are
// not provided.
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iomanip>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "mtk/data.h"
#include "mtk/models.h"
#include "mtk/search.h"
#include "mtk/serialize.h"
#include "mtk/train.h"

using namespace mtk;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --------------------------------------------------------- option table

struct Opt {
  enum Kind { Str, StrList, Int, Num, Flag } kind;
  void* dst;
  bool required = false;
  std::string help;
  bool given = false;
};

struct Command {
  std::string name, help;
  std::map<std::string, Opt> opts;  // key without "--"
  void add(const std::string& key, Opt::Kind k, void* dst, const std::string& help,
           bool required = false) {
    opts[key] = Opt{k, dst, required, help};
  }
  void usage(std::ostream& os) const {
    os << "usage: mtk-b200 " << name << " [options]   (" << help << ")\n";
    for(auto& [k, o] : opts)
      os << "  --" << k << (o.kind == Opt::Flag ? "" : " <value>") << (o.required ? " (required)" : "")
         << "  " << o.help << "\n";
  }
};

int64_t toInt(const std::string& v, const std::string& key) {
  try {
    size_t used = 0;
    int64_t x = std::stoll(v, &used);
    if(used != v.size())
      throw std::invalid_argument(v);
    return x;
  } catch(const std::exception&) {
    throw UsageError("option --" + key + " expects an integer, got '" + v + "'");
  }
}

double toNum(const std::string& v, const std::string& key) {
  try {
    size_t used = 0;
    double x = std::stod(v, &used);
    if(used != v.size())
      throw std::invalid_argument(v);
    return x;
  } catch(const std::exception&) {
    throw UsageError("option --" + key + " expects a number, got '" + v + "'");
  }
}

bool parseFlagValue(const std::string& v, const std::string& key) {  // config.cpp parseFlag
  if(v == "true" || v == "1")
    return true;
  if(v == "false" || v == "0")
    return false;
  throw DataError("option '" + key + "' expects true/false, got '" + v + "'");
}

std::string strip(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r");
  if(a == std::string::npos)
    return "";
  size_t b = s.find_last_not_of(" \t\r");
  return s.substr(a, b - a + 1);
}

// "key: value" per line, '#' comments (config.cpp:20-47)
std::map<std::string, std::string> readConfigFile(const std::string& path) {
  std::ifstream in(path);
  if(!in)
    throw IoError("cannot open config file: " + path);
  std::map<std::string, std::string> out;
  std::string line;
  size_t lineNo = 0;
  while(std::getline(in, line)) {
    ++lineNo;
    size_t hash = line.find('#');
    if(hash != std::string::npos)
      line = line.substr(0, hash);
    line = strip(line);
    if(line.empty())
      continue;
    size_t colon = line.find(':');
    if(colon == std::string::npos)
      throw DataError("malformed config line " + std::to_string(lineNo) + " in " + path + ": " +
                      line);
    std::string key = strip(line.substr(0, colon)), value = strip(line.substr(colon + 1));
    if(key.empty())
      throw DataError("empty key on config line " + std::to_string(lineNo) + " in " + path);
    if(out.count(key))
      throw DataError("duplicate config key '" + key + "' in " + path);
    out[key] = value;
  }
  return out;
}

std::vector<std::string> splitWs(const std::string& s) {
  std::istringstream in(s);
  std::vector<std::string> out;
  std::string tok;
  while(in >> tok)
    out.push_back(tok);
  return out;
}

void assign(Opt& o, const std::string& key, const std::vector<std::string>& vals) {
  switch(o.kind) {
    case Opt::Flag:
      *(bool*)o.dst = true;
      break;
    case Opt::Str:
      if(vals.size() != 1)
        throw UsageError("option --" + key + " expects one value");
      *(std::string*)o.dst = vals[0];
      break;
    case Opt::StrList:
      if(vals.empty())
        throw UsageError("option --" + key + " expects at least one value");
      *(std::vector<std::string>*)o.dst = vals;
      break;
    case Opt::Int:
      if(vals.size() != 1)
        throw UsageError("option --" + key + " expects one value");
      *(int64_t*)o.dst = toInt(vals[0], key);
      break;
    case Opt::Num:
      if(vals.size() != 1)
        throw UsageError("option --" + key + " expects one value");
      *(double*)o.dst = toNum(vals[0], key);
      break;
  }
  o.given = true;
}

// command line first (it wins), then --config values for options not given
void parse(Command& cmd, const std::vector<std::string>& args) {
  std::string configPath;
  for(size_t i = 0; i < args.size();) {
    const std::string& a = args[i];
    if(a == "--help" || a == "-h") {
      cmd.usage(std::cout);
      std::exit(0);
    }
    if(a.rfind("--", 0) != 0)
      throw UsageError("unexpected argument '" + a + "'");
    std::string key = a.substr(2);
    std::vector<std::string> vals;
    size_t j = i + 1;
    while(j < args.size() && args[j].rfind("--", 0) != 0)
      vals.push_back(args[j++]);
    if(key == "config") {
      if(vals.size() != 1)
        throw UsageError("--config expects one file");
      configPath = vals[0];
    } else {
      auto it = cmd.opts.find(key);
      if(it == cmd.opts.end())
        throw UsageError("unknown option --" + key);
      if(it->second.kind == Opt::Flag && !vals.empty())
        throw UsageError("flag --" + key + " takes no value");
      assign(it->second, key, vals);
    }
    i = j;
  }
  if(!configPath.empty()) {
    for(auto& [key, value] : readConfigFile(configPath)) {
      auto it = cmd.opts.find(key);
      if(it == cmd.opts.end() || key == "config")
        throw DataError("unknown option '" + key + "' in config file " + configPath);
      if(it->second.given)
        continue;
      if(it->second.kind == Opt::Flag) {
        if(parseFlagValue(value, key))
          assign(it->second, key, {});
      } else {
        assign(it->second, key, splitWs(value));
      }
    }
  }
  for(auto& [k, o] : cmd.opts)
    if(o.required && !o.given)
      throw UsageError("missing required option --" + k);
}

uint64_t defaultSeed() {  // tools/mtk.cpp:22-31
  const char* s = std::getenv("MTK_SEED");
  if(!s)
    return 1;
  try {
    return (uint64_t)std::stoull(s);
  } catch(const std::exception&) {
    throw DataError(std::string("MTK_SEED is not an integer: ") + s);
  }
}

// ------------------------------------------------------------ subcommands

struct VocabArgs {
  std::vector<std::string> corpora;
  std::string output;
  int64_t maxSize = 32000;
};

struct TrainArgs {  // tools/mtk.cpp:50-75 (same defaults)
  std::string modelPath;
  std::vector<std::string> trainSets;  // sources..., target
  std::vector<std::string> vocabs;
  std::string arch = "s2s-shallow";
  std::string customEncoders, customDecoder;
  int64_t embDim = 64, stateDim = 128;
  int64_t heads = 4, layers = 2;
  double dropout = 0.1;
  std::string tying = "none";
  bool layerNorm = false, rightLeft = false, postNorm = false;
  int64_t epochs = 1, maxUpdates = -1;
  int64_t miniBatchTokens = 256;
  int64_t workers = 1;
  bool async = false;
  double lrBase = 0.0003;
  int64_t warmup = 16000;
  double averageBeta = 0.9999;
  int64_t saveEvery = 0;
  std::string resume;
  int64_t logEvery = 100;
  bool quiet = false;
  int64_t seed = -1;
};

int runVocab(const VocabArgs& a) {  // tools/mtk.cpp:159-164
  Vocabulary v = Vocabulary::build(a.corpora, (size_t)a.maxSize);
  v.save(a.output);
  std::cerr << "built vocabulary of " << v.size() << " tokens\n";
  return 0;
}

int runTrain(const TrainArgs& a) {  // tools/mtk.cpp:166-241
  if(a.trainSets.size() < 2)
    throw DataError("--train-sets needs at least one source file and one target file");
  if(a.vocabs.size() != a.trainSets.size())
    throw DataError("--vocabs must list one vocabulary per training file");
  size_t streams = a.trainSets.size() - 1;
  std::vector<Vocabulary> vocabs;
  for(auto& p : a.vocabs)
    vocabs.push_back(Vocabulary::load(p));
  std::vector<const Vocabulary*> srcV;
  std::vector<std::string> srcPaths;
  for(size_t i = 0; i < streams; ++i) {
    srcV.push_back(&vocabs[i]);
    srcPaths.push_back(a.trainSets[i]);
    if(vocabs[i].size() != vocabs[0].size())
      throw DataError("all source vocabularies must have the same size");
  }
  auto data = readParallelCorpus(srcPaths, a.trainSets.back(), srcV, &vocabs.back());
  if(a.rightLeft)
    for(auto& ex : data)
      ex.target = invertR2l(ex.target);

  ModelConfig cfg;
  cfg.architecture = a.arch;
  cfg.encoderKind = a.customEncoders;
  cfg.decoderKind = a.customDecoder;
  cfg.sourceVocab = vocabs[0].size();
  cfg.targetVocab = vocabs.back().size();
  cfg.embDim = a.embDim;
  cfg.stateDim = a.stateDim;
  cfg.heads = (int)a.heads;
  cfg.layers = (int)a.layers;
  cfg.dropout = (Real)a.dropout;
  cfg.tying = a.tying;
  cfg.layerNorm = a.layerNorm;
  cfg.rightLeft = a.rightLeft;
  cfg.postNorm = a.postNorm;
  cfg.sourceArity = (int)streams;

  uint64_t seed = a.seed >= 0 ? (uint64_t)a.seed : defaultSeed();
  Model model = buildModel(cfg);
  ExpressionGraph master(seed);
  Adam adam(adamDefaultsFor(cfg));
  AveragedParameters average((Real)a.averageBeta);

  TrainOptions opts;
  opts.workers = (int)a.workers;
  opts.async = a.async;
  opts.tokenBudget = a.miniBatchTokens;
  opts.seed = seed;
  opts.epochs = a.epochs;
  opts.maxUpdates = a.maxUpdates;
  opts.lr.base = (Real)a.lrBase;
  opts.lr.warmup = a.warmup;
  opts.averageBeta = (Real)a.averageBeta;
  opts.checkpointPath = a.saveEvery > 0 ? a.modelPath + ".ckpt" : "";
  opts.checkpointEvery = a.saveEvery;
  opts.resumeFrom = a.resume;
  opts.logEvery = a.quiet ? 0 : a.logEvery;
  opts.log = a.quiet ? nullptr : &std::cerr;

  TrainResult res = train(model, data, master, adam, average, opts);
  saveModel(a.modelPath, cfg, master);
  if(!average.empty()) {
    ExpressionGraph avgGraph(seed);
    model.registerParams(avgGraph);
    for(auto& name : master.paramNames())
      avgGraph.paramValue(name).copyFrom(master.paramValue(name));
    average.applyTo(avgGraph);
    saveModel(a.modelPath + ".avg", cfg, avgGraph);
  }
  if(!a.quiet)
    std::cerr << "finished: updates=" << res.updates << " epochs=" << res.epochs
              << " loss=" << res.finalLoss << "\n";
  return 0;
}

struct TranslateArgs {  // tools/mtk.cpp:77-88
  std::vector<std::string> models, vocabs, inputs;
  std::string output = "-";
  std::string nBestFile;
  int64_t beamSize = 5;
  double alpha = 0.6;
  int64_t nBest = 1;
  int64_t miniBatchTokens = 512;
  int64_t maxLengthFactor = 3;
};

struct ScoreArgs {  // tools/mtk.cpp:90-96
  std::string model;
  std::vector<std::string> vocabs, inputs;
  std::string output = "-";
  int64_t miniBatchTokens = 512;
};

struct Loaded {
  std::unique_ptr<ExpressionGraph> graph;
  Model model;
};

Loaded loadOne(const std::string& path) {  // tools/mtk.cpp:130-135
  Loaded lm;
  lm.graph = std::make_unique<ExpressionGraph>(1, /*inference=*/true);
  lm.model = loadModel(path, *lm.graph);
  return lm;
}

std::ostream& openOutput(const std::string& path, std::ofstream& file) {
  if(path == "-")
    return std::cout;
  file.open(path);
  if(!file)
    throw IoError("cannot write output file: " + path);
  return file;
}

int runTranslate(const TranslateArgs& a) {  // tools/mtk.cpp:243-292
  std::vector<Loaded> loaded;
  for(auto& p : a.models)
    loaded.push_back(loadOne(p));
  const ModelConfig& c0 = loaded[0].model.config;
  for(auto& lm : loaded) {
    if(lm.model.config.targetVocab != c0.targetVocab)
      throw DataError("ensemble members disagree on the target vocabulary size");
    if(lm.model.config.rightLeft != c0.rightLeft)
      throw DataError("cannot ensemble left-to-right and right-to-left models");
    if(lm.model.config.sourceArity != c0.sourceArity)
      throw DataError("ensemble members disagree on the number of source streams");
  }
  if((int64_t)a.inputs.size() != (int64_t)c0.sourceArity)
    throw DataError("expected " + std::to_string(c0.sourceArity) + " input file(s)");
  if(a.vocabs.size() != a.inputs.size() + 1)
    throw DataError("--vocabs must list the source vocabularies plus the target vocabulary");
  std::vector<Vocabulary> vocabs;
  for(auto& p : a.vocabs)
    vocabs.push_back(Vocabulary::load(p));
  std::vector<Scorer> scorers;
  for(size_t i = 0; i < loaded.size(); ++i)
    scorers.push_back({"F" + std::to_string(i), &loaded[i].model, loaded[i].graph.get(), 1.0});
  std::vector<std::vector<std::string>> streams;
  for(auto& p : a.inputs)
    streams.push_back(readLines(p));
  std::vector<Vocabulary> srcVocabs(vocabs.begin(), vocabs.end() - 1);
  TranslateOptions opts;
  opts.beamSize = (int)a.beamSize;
  opts.alpha = a.alpha;
  opts.nBest = (int)a.nBest;
  opts.maxLengthFactor = a.maxLengthFactor;
  opts.tokenBudget = a.miniBatchTokens;
  TranslateOutput result = translateLines(scorers, vocabs.back(), streams, srcVocabs, opts);
  std::ofstream file;
  std::ostream& out = openOutput(a.output, file);
  for(auto& line : result.best)
    out << line << "\n";
  if(!a.nBestFile.empty()) {
    std::ofstream nb(a.nBestFile);
    if(!nb)
      throw IoError("cannot write n-best file: " + a.nBestFile);
    for(auto& line : result.nbestLines)
      nb << line << "\n";
  }
  std::cerr << "translated " << result.best.size() << " sentences, " << std::fixed
            << std::setprecision(1) << result.wordsPerSecond << " words/s\n";
  return 0;
}

int runScore(const ScoreArgs& a) {  // tools/mtk.cpp:294-340
  Loaded lm = loadOne(a.model);
  const ModelConfig& cfg = lm.model.config;
  if((int64_t)a.inputs.size() != (int64_t)cfg.sourceArity + 1)
    throw DataError("expected " + std::to_string(cfg.sourceArity) +
                    " source file(s) plus one target file");
  if(a.vocabs.size() != a.inputs.size())
    throw DataError("--vocabs must list one vocabulary per input file");
  std::vector<Vocabulary> vocabs;
  for(auto& p : a.vocabs)
    vocabs.push_back(Vocabulary::load(p));
  std::vector<const Vocabulary*> srcV;
  std::vector<std::string> srcPaths;
  for(size_t i = 0; i + 1 < a.inputs.size(); ++i) {
    srcV.push_back(&vocabs[i]);
    srcPaths.push_back(a.inputs[i]);
  }
  auto data = readParallelCorpus(srcPaths, a.inputs.back(), srcV, &vocabs.back());
  if(cfg.rightLeft)
    for(auto& ex : data)
      ex.target = invertR2l(ex.target);
  std::vector<Hypothesis> results(data.size());
  BatchOptions bo;
  bo.tokenBudget = a.miniBatchTokens;
  bo.shuffle = false;
  Scorer scorer{"F0", &lm.model, lm.graph.get(), 1.0};
  for(auto& batch : makeBatches(data, bo)) {
    auto scored = scoreBatch(scorer, batch);
    for(size_t r = 0; r < scored.size(); ++r)
      results[batch.sentenceIds[r]] = std::move(scored[r]);
  }
  std::ofstream file;
  std::ostream& out = openOutput(a.output, file);
  out << std::fixed << std::setprecision(6);
  for(size_t i = 0; i < results.size(); ++i) {
    out << i << ' ' << results[i].score;
    for(double sc : results[i].tokenScores)
      out << ' ' << sc;
    out << "\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  VocabArgs va;
  Command vocab{"vocab", "build a vocabulary from corpora", {}};
  vocab.add("corpus", Opt::StrList, &va.corpora, "input text files", true);
  vocab.add("output", Opt::Str, &va.output, "vocabulary file to write", true);
  vocab.add("max-size", Opt::Int, &va.maxSize, "maximum vocabulary size");

  TrainArgs ta;
  Command train{"train", "train a model", {}};
  train.add("model", Opt::Str, &ta.modelPath, "model file to write", true);
  train.add("train-sets", Opt::StrList, &ta.trainSets, "source file(s) then target file", true);
  train.add("vocabs", Opt::StrList, &ta.vocabs, "vocabulary per training file", true);
  train.add("arch", Opt::Str, &ta.arch,
            "s2s-shallow | s2s-deep | transformer | lm | ape-dual | hard-att | custom");
  train.add("custom-encoders", Opt::Str, &ta.customEncoders, "encoder kinds for --arch custom");
  train.add("custom-decoder", Opt::Str, &ta.customDecoder, "decoder kind for --arch custom");
  train.add("emb-dim", Opt::Int, &ta.embDim, "embedding dimension");
  train.add("state-dim", Opt::Int, &ta.stateDim, "recurrent state dimension");
  train.add("heads", Opt::Int, &ta.heads, "attention heads");
  train.add("layers", Opt::Int, &ta.layers, "transformer depth");
  train.add("dropout", Opt::Num, &ta.dropout, "dropout probability");
  train.add("tying", Opt::Str, &ta.tying, "none | source-target | all");
  train.add("layer-norm", Opt::Flag, &ta.layerNorm, "layer normalization");
  train.add("right-left", Opt::Flag, &ta.rightLeft, "train on inverted target sentences");
  train.add("post-norm", Opt::Flag, &ta.postNorm, "post-norm transformer blocks");
  train.add("epochs", Opt::Int, &ta.epochs, "training epochs");
  train.add("max-updates", Opt::Int, &ta.maxUpdates, "stop after this many updates");
  train.add("mini-batch-tokens", Opt::Int, &ta.miniBatchTokens, "token budget per batch");
  train.add("workers", Opt::Int, &ta.workers, "data-parallel workers");
  train.add("async", Opt::Flag, &ta.async, "asynchronous updates instead of synchronous");
  train.add("lr", Opt::Num, &ta.lrBase, "base learning rate");
  train.add("warmup", Opt::Int, &ta.warmup, "learning-rate warmup steps");
  train.add("average-beta", Opt::Num, &ta.averageBeta, "parameter averaging decay");
  train.add("save-every", Opt::Int, &ta.saveEvery, "checkpoint every N updates");
  train.add("resume", Opt::Str, &ta.resume, "checkpoint to resume from");
  train.add("log-every", Opt::Int, &ta.logEvery, "log every N updates");
  train.add("quiet", Opt::Flag, &ta.quiet, "suppress progress output");
  train.add("seed", Opt::Int, &ta.seed, "random seed (default: MTK_SEED or 1)");

  TranslateArgs xa;
  Command translate{"translate", "translate text", {}};
  translate.add("models", Opt::StrList, &xa.models, "model file(s); several = ensemble", true);
  translate.add("vocabs", Opt::StrList, &xa.vocabs, "source vocab(s) then target vocab", true);
  translate.add("input", Opt::StrList, &xa.inputs, "input file per source stream", true);
  translate.add("output", Opt::Str, &xa.output, "output file ('-' = stdout)");
  translate.add("n-best-file", Opt::Str, &xa.nBestFile, "write the n-best list here");
  translate.add("beam-size", Opt::Int, &xa.beamSize, "beam size");
  translate.add("alpha", Opt::Num, &xa.alpha, "length normalization exponent");
  translate.add("n-best", Opt::Int, &xa.nBest, "hypotheses per sentence in the n-best list");
  translate.add("mini-batch-tokens", Opt::Int, &xa.miniBatchTokens, "token budget per batch");
  translate.add("max-length-factor", Opt::Int, &xa.maxLengthFactor,
                "maximum output length as a multiple of the source length");

  ScoreArgs sa;
  Command score{"score", "force-decode and print log-probabilities", {}};
  score.add("model", Opt::Str, &sa.model, "model file", true);
  score.add("vocabs", Opt::StrList, &sa.vocabs, "vocabulary per input file", true);
  score.add("input", Opt::StrList, &sa.inputs, "source file(s) then target file", true);
  score.add("output", Opt::Str, &sa.output, "output file ('-' = stdout)");
  score.add("mini-batch-tokens", Opt::Int, &sa.miniBatchTokens, "token budget per batch");

  std::vector<std::string> args(argv + 1, argv + argc);
  Command* cmd = nullptr;
  try {
    if(args.empty() || args[0] == "--help" || args[0] == "-h") {
      std::cerr << "usage: mtk-b200 {vocab|train|translate|score} [options]; --help per "
                   "subcommand\n";
      return args.empty() ? 1 : 0;
    }
    if(args[0] == "vocab")
      cmd = &vocab;
    else if(args[0] == "train")
      cmd = &train;
    else if(args[0] == "translate")
      cmd = &translate;
    else if(args[0] == "score")
      cmd = &score;
    else
      throw UsageError("unknown subcommand '" + args[0] + "' (vocab, train, translate, score)");
    parse(*cmd, std::vector<std::string>(args.begin() + 1, args.end()));
  } catch(const UsageError& e) {
    std::cerr << e.what() << "\n";
    return 1;
  } catch(const DataError& e) {
    std::cerr << "data error: " << e.what() << "\n";
    return 2;
  } catch(const IoError& e) {
    std::cerr << "io error: " << e.what() << "\n";
    return 2;
  }
  try {
    if(cmd == &vocab)
      return runVocab(va);
    if(cmd == &train)
      return runTrain(ta);
    if(cmd == &translate)
      return runTranslate(xa);
    return runScore(sa);
  } catch(const DataError& e) {
    std::cerr << "data error: " << e.what() << "\n";
    return 2;
  } catch(const IoError& e) {
    std::cerr << "io error: " << e.what() << "\n";
    return 2;
  } catch(const NumericError& e) {
    std::cerr << "numeric error: " << e.what() << "\n";
    return 3;
  } catch(const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
