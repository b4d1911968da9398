// rst/validate.hpp -- verification (reference: include/rst/validate.hpp:16-47).
#pragma once

#include <string>
#include <vector>

#include "rst/graph.hpp"
#include "rst/rooted_forest.hpp"

namespace rst {

// Sequential host helpers kept for callers of the reference API.
std::vector<Vertex> oracle_components(const Graph& g);
std::vector<Vertex> oracle_root_tree(std::int64_t n, const std::vector<Edge>& tree_edges, Vertex root);
std::vector<std::int64_t> oracle_bfs_levels(const Graph& g, Vertex root);

struct ValidationReport {
  bool valid = true;
  std::vector<std::string> errors;
  void fail(std::string msg) {
    valid = false;
    if (errors.size() < 32) errors.push_back(std::move(msg));
  }
};

// Rooted-spanning-forest check, run on the GPU (rstg_validate) plus the
// declared-roots consistency check on the host.
ValidationReport validate_rooted_forest(const Graph& g, const RootedForest& f,
                                        Vertex required_root = kNone);

}  // namespace rst
