// mtk-b200: the reference's `mtk` command line (tools/mtk.cpp) for the
// training path, on the B200 backend.
//
// Subcommands: vocab, train (the §8(f) training driver); same option names,
// defaults, `--config` option files (key: value per line, command line wins,
// tools/mtk.cpp:429-456) and exit codes: 0 success, 1 usage error, 2 data/io
// error, 3 numeric error (tools/mtk.cpp:546-594).  CLI11 (absent from the
// reference tree) is replaced by a small option table.  Decoding subcommands
// (translate, score, rescore, bleu) are outside the training path.
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "mtk/data.h"
#include "mtk/models.h"
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

  std::vector<std::string> args(argv + 1, argv + argc);
  Command* cmd = nullptr;
  try {
    if(args.empty() || args[0] == "--help" || args[0] == "-h") {
      std::cerr << "usage: mtk-b200 {vocab|train} [options]; --help per subcommand\n";
      return args.empty() ? 1 : 0;
    }
    if(args[0] == "vocab")
      cmd = &vocab;
    else if(args[0] == "train")
      cmd = &train;
    else
      throw UsageError("unknown subcommand '" + args[0] + "' (vocab, train)");
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
    return cmd == &vocab ? runVocab(va) : runTrain(ta);
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
