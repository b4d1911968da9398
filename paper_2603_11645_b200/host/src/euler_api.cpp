// euler_api.cpp -- the reference's arc-level Euler-tour API
// (euler_rooting.hpp:18-59) over the device kernels of csrc/euler_api.cu and
// rstg_k_list_rank. Same layout, values and errors as the reference; the
// engine is charged the steps the reference's step-synchronous version
// charges (one per parallel_for_step, a sort as ceil(log2 E) steps, one per
// Wyllie round), so step-counting callers read the same numbers.
#include <algorithm>
#include <bit>
#include <stdexcept>
#include <vector>

#include "rst/device.hpp"
#include "rst/euler_rooting.hpp"

namespace rst {

EulerStructure build_euler(std::int64_t n, const std::vector<Edge>& tree_edges,
                           StepEngine& engine) {
  static_assert(sizeof(Edge) == 2 * sizeof(std::int64_t), "Edge must be two int64");
  const std::int64_t T = static_cast<std::int64_t>(tree_edges.size());
  const std::int64_t E = 2 * T;
  EulerStructure es;
  es.num_vertices = n;
  es.num_arcs = E;
  es.from.resize(static_cast<std::size_t>(E));
  es.to.resize(static_cast<std::size_t>(E));
  es.first.resize(static_cast<std::size_t>(n));
  es.last.resize(static_cast<std::size_t>(n));
  es.next.resize(static_cast<std::size_t>(E));
  rstg_check(rstg_k_build_euler(n, reinterpret_cast<const int64_t*>(tree_edges.data()), T,
                                es.from.data(), es.to.data(), es.first.data(), es.last.data(),
                                es.next.data()));
  const std::int64_t sort_steps = ceil_log2(std::max<std::int64_t>(E, 2));
  engine.charge(1, std::max(n, E));
  engine.charge(sort_steps, E * sort_steps);
  engine.charge(1, E);
  return es;
}

void compute_successor(EulerStructure& es, StepEngine& engine) {
  const std::int64_t E = es.num_arcs;
  es.succ.resize(static_cast<std::size_t>(E));
  rstg_check(rstg_k_compute_successor(es.num_vertices, E, es.from.data(), es.first.data(),
                                      es.next.data(), es.succ.data()));
  engine.charge(1, E);
}

void break_cycles(EulerStructure& es, const std::vector<Vertex>& roots, StepEngine& engine) {
  if (es.succ.empty() && es.num_arcs > 0)
    throw std::runtime_error("break_cycles called before compute_successor");
  rstg_check(rstg_k_break_cycles(es.num_vertices, es.num_arcs, es.last.data(), roots.data(),
                                 static_cast<std::int64_t>(roots.size()), es.succ.data()));
  engine.charge(1, static_cast<std::int64_t>(roots.size()));
}

std::vector<std::int64_t> list_rank(const EulerStructure& es, StepEngine& engine) {
  const std::int64_t E = es.num_arcs;
  std::vector<std::int64_t> rank(static_cast<std::size_t>(E));
  if (E > 0) rstg_check(rstg_k_list_rank(E, es.succ.data(), rank.data()));
  // pred clear + pred link + init, then one step per doubling round: the
  // reference stops after the first round in which no jump reaches a
  // second ancestor, i.e. bit_width(longest rank) rounds (at least one)
  engine.charge(3, 3 * E);
  if (E > 0) {
    const auto top = static_cast<std::uint64_t>(*std::max_element(rank.begin(), rank.end()));
    const std::int64_t rounds = std::max<std::int64_t>(1, std::bit_width(top));
    engine.charge(rounds, rounds * E);
  }
  return rank;
}

RootedForest derive_parents(const EulerStructure& es, const std::vector<std::int64_t>& rank,
                            const std::vector<Vertex>& roots, StepEngine& engine) {
  const std::int64_t n = es.num_vertices;
  RootedForest f;
  f.parent.resize(static_cast<std::size_t>(n));
  f.roots = roots;
  std::sort(f.roots.begin(), f.roots.end());
  rstg_check(rstg_k_derive_parents(n, es.num_arcs, es.from.data(), es.to.data(), rank.data(),
                                   f.parent.data()));
  engine.charge(1, n);
  engine.charge(1, es.num_arcs / 2);
  return f;
}

}  // namespace rst
