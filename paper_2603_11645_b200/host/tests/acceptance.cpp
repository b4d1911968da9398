// rst_acceptance -- the acceptance contract of the reference
// (proj/tests/acceptance.cpp, 9 criteria) evaluated against the B200
// engine through its drop-in C++ API. One PASS/FAIL line per criterion;
// the exit code is the number of failures. Step counts are the engine's
// device barriers (deterministic per input), so the step-scaling criteria
// test the same asymptotics: BFS one barrier per level, cc-euler and
// pr-rst logarithmic.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <numeric>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "rst/bench.hpp"
#include "rst/bfs_rst.hpp"
#include "rst/cc_forest.hpp"
#include "rst/euler_rooting.hpp"
#include "rst/graph.hpp"
#include "rst/pr_rst.hpp"
#include "rst/rooted_forest.hpp"
#include "rst/validate.hpp"
#include "rstg.h"

using namespace rst;

namespace {

int failures = 0;

void verdict(int id, bool ok, const std::string& what) {
  std::printf("%s  criterion %d: %s\n", ok ? "PASS" : "FAIL", id, what.c_str());
  if (!ok) ++failures;
}

Graph from_edges(Vertex n, std::vector<Edge> e) {
  EdgeList el;
  el.num_vertices = n;
  el.edges = std::move(e);
  normalize(el);
  return build_csr(el);
}

Graph gen(const std::string& spec, std::uint64_t seed = 0) {
  return build_csr(generate(parse_gen_spec(spec), seed));
}

std::vector<Edge> random_tree(Vertex n, std::mt19937_64& rng) {
  std::vector<Edge> t;
  for (Vertex v = 1; v < n; ++v) t.push_back({static_cast<Vertex>(rng() % static_cast<std::uint64_t>(v)), v});
  return t;
}

std::vector<Vertex> canon(const std::vector<Vertex>& lab) {
  std::vector<Vertex> first(lab.size(), kNone), out(lab.size());
  for (std::size_t v = 0; v < lab.size(); ++v) {
    auto& f = first[static_cast<std::size_t>(lab[v])];
    if (f == kNone) f = static_cast<Vertex>(v);
    out[v] = f;
  }
  return out;
}

std::vector<Vertex> forest_labels(const std::vector<Vertex>& parent) {
  std::vector<Vertex> lab(parent.size());
  for (std::size_t v = 0; v < parent.size(); ++v) {
    Vertex x = static_cast<Vertex>(v);
    while (parent[static_cast<std::size_t>(x)] != x) x = parent[static_cast<std::size_t>(x)];
    lab[v] = x;
  }
  return canon(lab);
}

}  // namespace

int main() {
  std::setvbuf(stdout, nullptr, _IOLBF, 0);
  std::printf("rooted spanning tree acceptance suite (B200 engine)\n");
  struct DS {
    std::string name;
    Graph g;
  };
  std::vector<DS> suite;
  suite.push_back({"path:10000", gen("path:10000")});
  suite.push_back({"star:10000", gen("star:10000")});
  suite.push_back({"grid:100:100", gen("grid:100:100")});
  for (std::uint64_t s = 1; s <= 5; ++s)
    suite.push_back({"random:2000:0.005 seed=" + std::to_string(s), gen("random:2000:0.005", s)});
  suite.push_back({"two-triangles", from_edges(6, {{0, 1}, {1, 2}, {0, 2}, {3, 4}, {4, 5}, {3, 5}})});
  suite.push_back({"single-vertex", gen("path:1")});

  // 1: valid forests with n - c tree edges, within the budget
  std::vector<std::vector<RunResult>> runs(suite.size());
  const auto t0 = std::chrono::steady_clock::now();
  for (std::size_t d = 0; d < suite.size(); ++d)
    for (AlgoKind a : kAllAlgos) runs[d].push_back(run_algorithm(suite[d].g, a, RunOptions{}));
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  {
    int ok = 0, total = 0;
    std::string bad;
    for (std::size_t d = 0; d < suite.size(); ++d) {
      const Graph& g = suite[d].g;
      const std::vector<Vertex> labels = oracle_components(g);
      const std::set<Vertex> comps(labels.begin(), labels.end());
      for (std::size_t a = 0; a < 3; ++a) {
        ++total;
        const RootedForest& f = runs[d][a].forest;
        std::int64_t te = 0;
        for (Vertex v = 0; v < g.n; ++v) te += f.parent[static_cast<std::size_t>(v)] != v;
        if (validate_rooted_forest(g, f, 0).valid && te == g.n - static_cast<std::int64_t>(comps.size()))
          ++ok;
        else if (bad.empty())
          bad = suite[d].name + "/" + algo_name(kAllAlgos[a]);
      }
    }
    verdict(1, ok == total && secs < 10.0,
            std::to_string(ok) + "/" + std::to_string(total) + " forests valid in " +
                std::to_string(secs) + "s" + (bad.empty() ? "" : ", first failure " + bad));
  }

  // 2: partitions vs union-find; Euler rooting exact on random trees
  {
    bool parts = true;
    for (std::size_t d = 0; d < suite.size(); ++d) {
      StepEngine e;
      const auto want = oracle_components(suite[d].g);
      parts = parts && canon(cc_spanning_forest(suite[d].g, e).labels) == want &&
              forest_labels(runs[d][2].forest.parent) == want;
    }
    std::mt19937_64 rng(20260815);
    int exact = 0;
    for (int t = 0; t < 100; ++t) {
      const Vertex n = 1 + static_cast<Vertex>(rng() % 256);
      const auto te = random_tree(n, rng);
      const Vertex root = static_cast<Vertex>(rng() % static_cast<std::uint64_t>(n));
      StepEngine e;
      const auto f = euler_root_forest(n, te, std::vector<Vertex>(static_cast<std::size_t>(n), 0), root, e);
      exact += f.parent == oracle_root_tree(n, te, root);
    }
    verdict(2, parts && exact == 100,
            std::string("partitions ") + (parts ? "match" : "differ") + "; euler rooting exact on " +
                std::to_string(exact) + "/100 random trees");
  }

  // 3 + 4: step scaling on path(2^k)
  std::vector<std::int64_t> sb, sc, sp;
  for (int k = 10; k <= 14; ++k) {
    const Graph g = gen("path:" + std::to_string(1 << k));
    StepEngine eb, ec, ep;
    bfs_rst(g, 0, eb);
    cc_euler_rst(g, 0, ec);
    pr_rst(g, 0, ep);
    sb.push_back(eb.steps());
    sc.push_back(ec.steps());
    sp.push_back(ep.steps());
  }
  {
    bool bfs_ok = true, cc_ok = true;
    for (int i = 0; i < 5; ++i) {
      const std::int64_t lo = (std::int64_t{1} << (10 + i)) - 1;
      bfs_ok = bfs_ok && sb[i] >= lo && sb[i] <= lo + 3;
      cc_ok = cc_ok && double(sc[i]) / (10 + i) <= double(sc[0]) / 10.0 * 1.2;
    }
    const double pr_growth = double(sp[4]) / double(sp[0]);
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "bfs steps %lld..%lld (%s), cc-euler steps %lld..%lld (%s), pr-rst growth %.2f (%s)",
                  (long long)sb[0], (long long)sb[4], bfs_ok ? "ok" : "violated", (long long)sc[0],
                  (long long)sc[4], cc_ok ? "ok" : "violated", pr_growth,
                  pr_growth <= 2.1 ? "ok" : "violated");
    verdict(3, bfs_ok && cc_ok && pr_growth <= 2.1, buf);
    const double gb = double(sb[4]) / sb[0], gc = double(sc[4]) / sc[0];
    std::snprintf(buf, sizeof buf, "bfs grows %.2fx (floor 15x), cc-euler grows %.2fx (cap 1.5x)", gb, gc);
    verdict(4, gb >= 15.0 && gc <= 1.5, buf);
  }

  // 5: BFS depth equals the root's eccentricity
  {
    bool ok = true;
    for (std::size_t d = 0; d < suite.size(); ++d) {
      std::int64_t ecc = 0;
      for (auto l : oracle_bfs_levels(suite[d].g, 0)) ecc = std::max(ecc, l);
      std::int64_t dep = 0;
      for (const auto& [r, dd] : forest_depth(runs[d][0].forest).per_root)
        if (r == 0) dep = dd;
      ok = ok && dep == ecc;
    }
    verdict(5, ok, ok ? "bfs depth equals the root's eccentricity on every graph"
                      : "bfs depth deviates from the eccentricity");
  }

  // 6: device list ranking is a bijection onto positions; Euler rooting of
  //    random trees (seed 424242) exact
  {
    std::mt19937_64 rng(424242);
    int bij = 0, rooted = 0;
    for (int t = 0; t < 100; ++t) {
      const std::int64_t E = 2 + static_cast<std::int64_t>(rng() % 509);
      std::vector<std::int64_t> perm(static_cast<std::size_t>(E));
      std::iota(perm.begin(), perm.end(), 0);
      std::shuffle(perm.begin(), perm.end(), rng);
      std::vector<std::int64_t> succ(static_cast<std::size_t>(E), -1), rank(static_cast<std::size_t>(E));
      for (std::int64_t i = 0; i + 1 < E; ++i) succ[static_cast<std::size_t>(perm[static_cast<std::size_t>(i)])] = perm[static_cast<std::size_t>(i + 1)];
      if (rstg_k_list_rank(E, succ.data(), rank.data()) == RSTG_OK) {
        bool good = true;
        for (std::int64_t i = 0; i < E; ++i) good = good && rank[static_cast<std::size_t>(perm[static_cast<std::size_t>(i)])] == i;
        bij += good;
      }
      const Vertex n = 2 + static_cast<Vertex>(rng() % 255);
      const auto te = random_tree(n, rng);
      StepEngine e;
      rooted += euler_root_forest(n, te, std::vector<Vertex>(static_cast<std::size_t>(n), 0), 0, e).parent ==
                oracle_root_tree(n, te, 0);
    }
    verdict(6, bij == 100 && rooted == 100,
            "list ranking exact on " + std::to_string(bij) + "/100 lists, euler rooting exact on " +
                std::to_string(rooted) + "/100 trees");
  }

  // 7: reruns are bit-identical (parents, steps, work)
  {
    bool ok = true;
    std::vector<DS> dets;
    dets.push_back({"path:4096", gen("path:4096")});
    dets.push_back({"grid:50:50", gen("grid:50:50")});
    dets.push_back({"random:1000:0.01", gen("random:1000:0.01", 3)});
    dets.push_back({"two-triangles", from_edges(6, {{0, 1}, {1, 2}, {0, 2}, {3, 4}, {4, 5}, {3, 5}})});
    for (auto& d : dets)
      for (AlgoKind a : kAllAlgos) {
        RunOptions one, many;
        many.workers = 8;
        const auto r1 = run_algorithm(d.g, a, one), r2 = run_algorithm(d.g, a, one),
                   r8 = run_algorithm(d.g, a, many);
        ok = ok && r1.forest.parent == r2.forest.parent && r1.forest.parent == r8.forest.parent &&
             r1.report.steps == r2.report.steps && r1.report.steps == r8.report.steps &&
             r1.report.work == r8.report.work;
      }
    verdict(7, ok, ok ? "12 graph/algorithm pairs bit-identical across reruns" : "nondeterminism");
  }

  // 8: bench protocol
  {
    BenchProbe probe;
    const auto rec = bench_row(gen("path:2048"), "gen:path:2048", AlgoKind::kBfs, RunOptions{}, &probe);
    auto s = probe.timed_ms;
    std::sort(s.begin(), s.end());
    const bool ok = probe.executions == 6 && s.size() == 5 && rec.median_ms == s[2];
    verdict(8, ok, std::to_string(probe.executions) + " executions, median of 5 timed");
  }

  // 9: jump-batch invariance
  {
    const Graph g = gen("path:4096");
    StepEngine e1, e5;
    const auto f1 = pr_rst(g, 0, e1, 1), f5 = pr_rst(g, 0, e5, 5);
    verdict(9, f1.parent == f5.parent && e5.steps() <= e1.steps(),
            "parents identical across batch 1 and 5, steps " + std::to_string(e5.steps()) +
                " <= " + std::to_string(e1.steps()));
  }

  if (failures == 0)
    std::printf("all 9 criteria passed\n");
  else
    std::printf("%d criteria FAILED\n", failures);
  return failures;
}
