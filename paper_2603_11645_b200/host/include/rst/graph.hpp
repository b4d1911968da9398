// rst/graph.hpp -- graph data model and ingestion of the drop-in API
// (reference: include/rst/graph.hpp:17-94). Host-side plumbing; the device
// copy lives in the C-ABI handle (include/rstg.h).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "rst/types.hpp"

namespace rst {

struct EdgeList {
  Vertex num_vertices = 0;
  std::vector<Edge> edges;
  std::vector<std::int64_t> original_ids;  // sparse external ids, empty = identity
};

// CSR + normalized edge list; edge id = index into `edges`.
struct Graph {
  Vertex n = 0;
  std::int64_t m = 0;
  std::vector<std::int64_t> offsets;
  std::vector<Vertex> neighbors;
  std::vector<EdgeId> edge_origin;
  std::vector<Edge> edges;

  std::span<const Vertex> neighbors_of(Vertex u) const {
    return {neighbors.data() + offsets[static_cast<std::size_t>(u)],
            neighbors.data() + offsets[static_cast<std::size_t>(u) + 1]};
  }
  std::int64_t degree(Vertex u) const {
    return offsets[static_cast<std::size_t>(u) + 1] - offsets[static_cast<std::size_t>(u)];
  }
  bool has_edge(Vertex u, Vertex v) const;
};

class ParseError : public std::runtime_error {
 public:
  ParseError(std::int64_t line, const std::string& what);
  std::int64_t line() const { return line_; }

 private:
  std::int64_t line_;
};

void normalize(EdgeList& el);
EdgeList load_edge_list(std::istream& in);
void write_edge_list(std::ostream& out, const EdgeList& el);
Graph build_csr(const EdgeList& el);
EdgeList to_edge_list(const Graph& g);

EdgeList gen_path(Vertex n);
EdgeList gen_star(Vertex n);
EdgeList gen_grid(Vertex rows, Vertex cols);
EdgeList gen_random(Vertex n, double p, std::uint64_t seed);
EdgeList gen_complete(Vertex n);
// Benchmark shapes of SURVEY.md Appendix B (extensions): road_usa-shaped
// mesh R x R, Graph500 Kronecker scale/edge factor.
EdgeList gen_road(Vertex R, double p = 0.2026);
EdgeList gen_kron(int scale, int edge_factor = 16);

struct GenSpec {
  enum class Kind { path, star, grid, random, complete, road, kron };
  Kind kind = Kind::path;
  Vertex n = 0;
  Vertex rows = 0, cols = 0;
  double p = 0.0;
};

GenSpec parse_gen_spec(const std::string& spec);
EdgeList generate(const GenSpec& spec, std::uint64_t seed = 0);

}  // namespace rst
