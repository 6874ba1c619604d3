// Fused GRU block (gruCell, reference graph.cpp:648-813).
#include "mtk/device.h"
#include "mtk/graph.h"

namespace mtk {

NodeRef ExpressionGraph::gruCell(NodeRef state, NodeRef input, const GruParams& p,
                                 bool layerNorm) {
  (void)state;
  (void)input;
  (void)p;
  (void)layerNorm;
  throw ContractError("gruCell: not built yet");
}

}  // namespace mtk
