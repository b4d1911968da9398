// rst/cc_forest.hpp -- connectivity phase (reference: include/rst/cc_forest.hpp:14-42).
#pragma once

#include <vector>

#include "rst/graph.hpp"
#include "rst/step_engine.hpp"

namespace rst {

enum class HookMode { kMin, kMax };

struct SpanningForest {
  std::vector<Vertex> labels;      // converged representative per vertex
  std::vector<EdgeId> tree_edges;  // ascending edge ids
};

// Exact synchronous min/max-alternating hooking on the GPU; labels and
// tree edges are bit-identical to the reference.
SpanningForest cc_spanning_forest(const Graph& g, StepEngine& engine);

}  // namespace rst
