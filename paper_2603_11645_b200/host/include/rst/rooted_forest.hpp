// rst/rooted_forest.hpp -- the output type (reference:
// include/rst/rooted_forest.hpp:14-36).
#pragma once

#include <iosfwd>
#include <utility>
#include <vector>

#include "rst/types.hpp"

namespace rst {

struct RootedForest {
  std::vector<Vertex> parent;        // parent[r] == r exactly for roots
  std::vector<Vertex> roots;
  std::vector<std::int64_t> levels;  // BFS only
};

struct DepthStats {
  std::vector<std::pair<Vertex, std::int64_t>> per_root;
  std::int64_t max_depth = 0;
};

DepthStats forest_depth(const RootedForest& f);
void write_parent_array(std::ostream& out, const std::vector<Vertex>& parent);
std::vector<Vertex> read_parent_array(std::istream& in);
RootedForest forest_from_parent(std::vector<Vertex> parent);

}  // namespace rst
