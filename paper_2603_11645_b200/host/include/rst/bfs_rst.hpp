// rst/bfs_rst.hpp -- BFS baseline (reference: include/rst/bfs_rst.hpp:23).
#pragma once

#include "rst/graph.hpp"
#include "rst/rooted_forest.hpp"
#include "rst/step_engine.hpp"

namespace rst {

// Direction-optimising BFS; parent = smallest-id neighbour one level up,
// other components rooted at their smallest vertex (roots in that order).
RootedForest bfs_rst(const Graph& g, Vertex root, StepEngine& engine);

}  // namespace rst
