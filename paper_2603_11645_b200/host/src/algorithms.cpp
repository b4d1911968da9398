// algorithms.cpp -- the reference's C++ entry points, each one call into
// the CUDA pipeline behind the C ABI (include/rstg.h):
//   bfs_rst            bfs_rst.hpp:23         -> rstg_run(RSTG_BFS)
//   cc_spanning_forest cc_forest.hpp:42       -> rstg_cc_spanning_forest
//   euler_root_forest  euler_rooting.hpp:63   -> rstg_euler_root_forest
//   cc_euler_rst       euler_rooting.hpp:69   -> rstg_run(RSTG_CC_EULER)
//   pr_rst             pr_rst.hpp:94          -> rstg_run(RSTG_PR_RST)
// Nothing is computed on the host: without a GPU these throw.
#include <string>
#include <vector>

#include "rst/bfs_rst.hpp"
#include "rst/cc_forest.hpp"
#include "rst/device.hpp"
#include "rst/euler_rooting.hpp"
#include "rst/pr_rst.hpp"

namespace rst {

namespace {

void check_root(const Graph& g, Vertex root) {
  if (root < 0 || root >= g.n)
    throw std::runtime_error("root " + std::to_string(root) + " out of range");
}

RootedForest run(const Graph& g, int algo, Vertex root, std::int64_t jump_batch,
                 StepEngine& engine) {
  check_root(g, root);
  rstg_graph* h = device_graph(g, engine.device());
  RootedForest f;
  f.parent.resize(static_cast<std::size_t>(g.n));
  f.roots.resize(static_cast<std::size_t>(g.n));
  if (algo == RSTG_BFS) f.levels.resize(static_cast<std::size_t>(g.n));
  int64_t nroots = 0;
  rstg_stats st{};
  rstg_check(rstg_run(h, algo, root, jump_batch, f.parent.data(),
                      algo == RSTG_BFS ? f.levels.data() : nullptr, f.roots.data(), &nroots,
                      &st));
  f.roots.resize(static_cast<std::size_t>(nroots));
  engine.record_device(st.steps, st.work, st.launches, st.device_ms);
  return f;
}

}  // namespace

RootedForest bfs_rst(const Graph& g, Vertex root, StepEngine& engine) {
  return run(g, RSTG_BFS, root, 5, engine);
}

RootedForest cc_euler_rst(const Graph& g, Vertex root, StepEngine& engine) {
  return run(g, RSTG_CC_EULER, root, 5, engine);
}

RootedForest pr_rst(const Graph& g, Vertex root, StepEngine& engine, std::int64_t jump_batch) {
  return run(g, RSTG_PR_RST, root, jump_batch, engine);
}

SpanningForest cc_spanning_forest(const Graph& g, StepEngine& engine) {
  rstg_graph* h = device_graph(g, engine.device());
  SpanningForest sf;
  sf.labels.resize(static_cast<std::size_t>(g.n));
  sf.tree_edges.resize(static_cast<std::size_t>(std::max<std::int64_t>(g.n, 1)));
  int64_t T = 0;
  rstg_stats st{};
  rstg_check(rstg_cc_spanning_forest(h, sf.labels.data(), sf.tree_edges.data(), &T, &st));
  sf.tree_edges.resize(static_cast<std::size_t>(T));
  engine.record_device(st.steps, st.work, st.launches, st.device_ms);
  return sf;
}

RootedForest euler_root_forest(std::int64_t n, const std::vector<Edge>& tree_edges,
                               const std::vector<Vertex>& labels, Vertex designated_root,
                               StepEngine& engine) {
  static_assert(sizeof(Edge) == 2 * sizeof(std::int64_t), "Edge must be two int64");
  RootedForest f;
  f.parent.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  f.roots.resize(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
  int64_t nroots = 0;
  rstg_check(rstg_euler_root_forest(
      n, reinterpret_cast<const int64_t*>(tree_edges.data()),
      static_cast<int64_t>(tree_edges.size()), labels.data(),
      static_cast<int64_t>(labels.size()), designated_root, engine.device(), f.parent.data(),
      f.roots.data(), &nroots));
  f.parent.resize(static_cast<std::size_t>(n));
  f.roots.resize(static_cast<std::size_t>(nroots));
  return f;
}

}  // namespace rst
