// Drop-in check: the reference's UNMODIFIED model code (src/models.cpp,
// src/layers.cpp, src/encdec.cpp, compiled from /root/reference by
// tests/dropin/Makefile against this build's headers csrc/host/mtk/*.h) runs
// one training step on the B200 backend (libmtkhost.so / libmtkcuda.so):
// buildModel -> registerParams -> buildLoss -> forward -> backward
// (reference call sites: train.cpp:232-235, models.cpp:629-674).
//
// Test infrastructure (tests/test_dropin_gpu.py compares the output with the
// reference oracle); not part of the product.
//
// usage: dropin_step <config-file> <sentences> <token-budget> <graph-seed> <out-file>
// out-file: f64 loss, i64 target tokens, i64 #params, then per parameter
//           i64 name length, name bytes, i64 element count, f32 gradient.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>

#include "mtk/data.h"
#include "mtk/device.h"
#include "mtk/graph.h"
#include "mtk/models.h"

using namespace mtk;

static uint64_t splitmix(uint64_t x) {
  uint64_t z = x + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  if(argc != 6) {
    std::fprintf(stderr, "usage: %s config sentences budget seed out\n", argv[0]);
    return 2;
  }
  std::ifstream cf(argv[1]);
  std::stringstream ss;
  ss << cf.rdbuf();
  ModelConfig cfg = ModelConfig::parse(ss.str());
  const int64_t n = std::atoll(argv[2]);
  const int64_t budget = std::atoll(argv[3]);
  const uint64_t seed = std::strtoull(argv[4], nullptr, 0);
  // SURVEY.md 8(d) synthetic corpus (same formula as paper_1804_00344_b200/synth.py)
  std::vector<Example> ex((size_t)n);
  const uint64_t V = (uint64_t)cfg.sourceVocab;
  for(int64_t k = 0; k < n; ++k) {
    const uint64_t i = (uint64_t)k;
    const int64_t ls = 16 + (int64_t)(splitmix(1234ull * 1000003ull + i) % 17);
    const int64_t lt = 16 + (int64_t)(splitmix(5678ull * 1000003ull + i) % 17);
    std::vector<int32_t> s((size_t)ls), t((size_t)lt);
    for(int64_t j = 0; j < ls; ++j)
      s[(size_t)j] = (int32_t)(2 + splitmix((i << 20) ^ (uint64_t)j ^ 0xabcull) % (V - 2));
    for(int64_t j = 0; j < lt; ++j)
      t[(size_t)j] = (int32_t)(2 + splitmix((i << 20) ^ (uint64_t)j ^ 0xdefull) % (V - 2));
    ex[(size_t)k].sources = {s};
    ex[(size_t)k].target = t;
    ex[(size_t)k].hasTarget = true;
    ex[(size_t)k].id = (size_t)k;
  }
  BatchOptions bo;
  bo.tokenBudget = budget;
  bo.seed = 1;
  std::vector<Batch> batches = makeBatches(ex, bo);
  if(batches.size() != 1) {
    std::fprintf(stderr, "expected one batch, got %zu\n", batches.size());
    return 3;
  }
  Model model = buildModel(cfg);
  ExpressionGraph g(1);
  model.registerParams(g);
  g.clear();
  g.setSeed(seed);
  Real tokens = 0;
  NodeRef loss = model.buildLoss(g, batches[0], &tokens);
  g.forward();
  g.zeroGrads();
  g.backward(loss);
  const double lv = (double)loss.val().toVector()[0];
  std::ofstream out(argv[5], std::ios::binary);
  const int64_t tok = batches[0].targetTokenCount();
  const auto names = g.paramNames();
  const int64_t np = (int64_t)names.size();
  out.write((const char*)&lv, 8);
  out.write((const char*)&tok, 8);
  out.write((const char*)&np, 8);
  for(const auto& name : names) {
    const int64_t len = (int64_t)name.size();
    out.write((const char*)&len, 8);
    out.write(name.data(), len);
    std::vector<Real> gr = g.paramGrad(name).toVector();
    const int64_t cnt = (int64_t)gr.size();
    out.write((const char*)&cnt, 8);
    out.write((const char*)gr.data(), cnt * (int64_t)sizeof(Real));
  }
  std::printf("dropin loss %.9g tokens %lld params %lld launches %llu\n", lv, (long long)tok,
              (long long)np, (unsigned long long)mtkc_launch_count());
  return 0;
}
