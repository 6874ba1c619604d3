// MTK1 model / checkpoint container (reference: include/mtk/serialize.h,
// src/serialize.cpp).  The on-disk layout is the reference's, byte for byte:
//   "MTK1", u32 version 1, u64-length-prefixed config text, then entries of
//   [u32 name length, name, u32 rank, u64 dims..., little-endian f32 data]
//   terminated by a zero name length.
// Files written by the reference load here unchanged and vice versa.
//
// B200 note: tensors in a ModelFile are host-staged (the file is a host
// object); saveModel / saveCheckpoint read the flat device parameter pool
// (and the flat Adam / EMA buffers) with one device-to-host copy each and
// slice it per parameter, loadParams uploads one flat pool image.
#pragma once

#include "mtk/models.h"

namespace mtk {

struct ModelFile {
  ModelConfig config;
  std::vector<std::pair<std::string, Tensor>> tensors;  // in file order

  const Tensor* find(const std::string& name) const;
};

void writeModelFile(const std::string& path, const ModelConfig& config,
                    const std::vector<std::pair<std::string, Tensor>>& tensors);
ModelFile readModelFile(const std::string& path);

// every graph parameter under its own name, in creation order
void saveModel(const std::string& path, const ModelConfig& config, ExpressionGraph& g);
// fills an existing graph's parameters (names and shapes must match exactly;
// dotted names without a matching parameter -- optimizer state -- are skipped)
void loadParams(const ModelFile& file, ExpressionGraph& g);
Model loadModel(const std::string& path, ExpressionGraph& g);

}  // namespace mtk
