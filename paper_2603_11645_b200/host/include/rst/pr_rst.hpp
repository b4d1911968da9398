// rst/pr_rst.hpp -- path-reversal RST (reference: include/rst/pr_rst.hpp:94-95).
#pragma once

#include "rst/graph.hpp"
#include "rst/rooted_forest.hpp"
#include "rst/step_engine.hpp"

namespace rst {

RootedForest pr_rst(const Graph& g, Vertex root, StepEngine& engine, std::int64_t jump_batch = 5);

}  // namespace rst
