// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, which
// oracle/Makefile compiles from the sources under /root/reference/proj/core
// (with -Drst=rst_ref so its symbols cannot collide with anything else) into
// oracle/_ref/librst_ref.so. Nothing here re-implements an algorithm: every
// entry point builds the reference's own Graph and calls the reference's own
// public functions (bench.hpp:36 run_algorithm, cc_forest.hpp:42,
// euler_rooting.hpp:63-69, validate.hpp:46-47, graph.hpp:71-94).
// Used by tests/ (golden fixtures, oracle pinning) and by bench.py's
// cpu_baseline / --impl reference legs.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
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

namespace {
thread_local std::string g_err;

rst::Graph make_graph(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev) {
  rst::EdgeList el;
  el.num_vertices = n;
  el.edges.resize(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) el.edges[static_cast<size_t>(i)] = {eu[i], ev[i]};
  return rst::build_csr(el);
}

void copy_forest(const rst::RootedForest& f, int64_t* parent, int64_t* levels,
                 int64_t* roots, int64_t* num_roots) {
  if (parent) std::memcpy(parent, f.parent.data(), f.parent.size() * sizeof(int64_t));
  if (levels && !f.levels.empty())
    std::memcpy(levels, f.levels.data(), f.levels.size() * sizeof(int64_t));
  if (roots) std::memcpy(roots, f.roots.data(), f.roots.size() * sizeof(int64_t));
  if (num_roots) *num_roots = static_cast<int64_t>(f.roots.size());
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// One-shot: build the Graph, run the strategy through run_algorithm.
int ref_run(int algo, int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
            int64_t root, int workers, int64_t jump_batch, int64_t* parent,
            int64_t* levels, int64_t* roots, int64_t* num_roots, int64_t* steps,
            int64_t* work) {
  try {
    rst::Graph g = make_graph(n, m, eu, ev);
    rst::RunOptions opt;
    opt.root = root;
    opt.workers = workers;
    opt.jump_batch = jump_batch;
    rst::RunResult r = rst::run_algorithm(g, static_cast<rst::AlgoKind>(algo), opt);
    copy_forest(r.forest, parent, levels, roots, num_roots);
    if (steps) *steps = r.report.steps;
    if (work) *work = r.report.work;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Prebuilt graph handle so a timing loop measures run_algorithm only.
void* ref_graph_create(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev) {
  try {
    return new rst::Graph(make_graph(n, m, eu, ev));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_graph_destroy(void* h) { delete static_cast<rst::Graph*>(h); }

// Times exactly what bench_row times (bench.cpp:73-76): run_algorithm,
// including its StepEngine construction. Returns wall ms, <0 on error.
double ref_graph_run(void* h, int algo, int64_t root, int workers, int64_t jump_batch,
                     int64_t* parent) {
  try {
    const rst::Graph& g = *static_cast<rst::Graph*>(h);
    rst::RunOptions opt;
    opt.root = root;
    opt.workers = workers;
    opt.jump_batch = jump_batch;
    auto t0 = std::chrono::steady_clock::now();
    rst::RunResult r = rst::run_algorithm(g, static_cast<rst::AlgoKind>(algo), opt);
    auto t1 = std::chrono::steady_clock::now();
    if (parent) std::memcpy(parent, r.forest.parent.data(), r.forest.parent.size() * 8);
    return std::chrono::duration<double, std::milli>(t1 - t0).count();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

int ref_cc_spanning_forest(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                           int workers, int64_t* labels, int64_t* tree_edges,
                           int64_t* num_tree_edges, int64_t* steps) {
  try {
    rst::Graph g = make_graph(n, m, eu, ev);
    rst::StepEngine e(workers);
    rst::SpanningForest sf = rst::cc_spanning_forest(g, e);
    std::memcpy(labels, sf.labels.data(), sf.labels.size() * sizeof(int64_t));
    std::memcpy(tree_edges, sf.tree_edges.data(), sf.tree_edges.size() * sizeof(int64_t));
    *num_tree_edges = static_cast<int64_t>(sf.tree_edges.size());
    if (steps) *steps = e.steps();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_euler_root_forest(int64_t n, int64_t T, const int64_t* tu, const int64_t* tv,
                          const int64_t* labels, int64_t nlabels, int64_t designated_root,
                          int64_t* parent, int64_t* roots, int64_t* num_roots) {
  try {
    std::vector<rst::Edge> te(static_cast<size_t>(T));
    for (int64_t i = 0; i < T; ++i) te[static_cast<size_t>(i)] = {tu[i], tv[i]};
    std::vector<rst::Vertex> lab(labels, labels + nlabels);
    rst::StepEngine e;
    rst::RootedForest f = rst::euler_root_forest(n, te, lab, designated_root, e);
    copy_forest(f, parent, nullptr, roots, num_roots);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Reference Euler internals on a forest, for rank golden vectors.
int ref_euler_ranks(int64_t n, int64_t T, const int64_t* tu, const int64_t* tv,
                    const int64_t* roots, int64_t nroots, int64_t* succ, int64_t* rank) {
  try {
    std::vector<rst::Edge> te(static_cast<size_t>(T));
    for (int64_t i = 0; i < T; ++i) te[static_cast<size_t>(i)] = {tu[i], tv[i]};
    rst::StepEngine e;
    rst::EulerStructure es = rst::build_euler(n, te, e);
    rst::compute_successor(es, e);
    std::vector<rst::Vertex> rv(roots, roots + nroots);
    rst::break_cycles(es, rv, e);
    std::memcpy(succ, es.succ.data(), es.succ.size() * sizeof(int64_t));
    std::vector<int64_t> rk = rst::list_rank(es, e);
    std::memcpy(rank, rk.data(), rk.size() * sizeof(int64_t));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_validate(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                 const int64_t* parent, const int64_t* roots, int64_t nroots,
                 int64_t required_root) {
  try {
    rst::Graph g = make_graph(n, m, eu, ev);
    rst::RootedForest f;
    f.parent.assign(parent, parent + n);
    f.roots.assign(roots, roots + nroots);
    rst::ValidationReport r = rst::validate_rooted_forest(g, f, required_root);
    g_err = r.errors.empty() ? "" : r.errors.front();
    return r.valid ? 1 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Reference generators ("path:10", "grid:5:7", "random:500:0.004", ...).
// Two calls: first with eu == nullptr returns m and n; then fills.
int64_t ref_generate(const char* spec, uint64_t seed, int64_t* n_out, int64_t* eu,
                     int64_t* ev) {
  try {
    rst::EdgeList el = rst::generate(rst::parse_gen_spec(spec), seed);
    *n_out = el.num_vertices;
    if (eu) {
      for (size_t i = 0; i < el.edges.size(); ++i) {
        eu[i] = el.edges[i].u;
        ev[i] = el.edges[i].v;
      }
    }
    return static_cast<int64_t>(el.edges.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// load_edge_list (graph.cpp:48-127) over an in-memory text. Returns m
// (normalized), fills n, the edges (when eu != nullptr) and original_ids
// (when ids != nullptr; *nids = their count); -1 on any exception, with
// *err_line = the ParseError line (or -1 for other errors).
int64_t ref_load_edge_list(const char* text, int64_t len, int64_t* n_out, int64_t* eu,
                           int64_t* ev, int64_t* ids, int64_t* nids, int64_t* err_line) {
  *err_line = -1;
  try {
    std::istringstream in(std::string(text, static_cast<size_t>(len)));
    rst::EdgeList el = rst::load_edge_list(in);
    *n_out = el.num_vertices;
    *nids = static_cast<int64_t>(el.original_ids.size());
    if (eu) {
      for (size_t i = 0; i < el.edges.size(); ++i) {
        eu[i] = el.edges[i].u;
        ev[i] = el.edges[i].v;
      }
    }
    if (ids) std::memcpy(ids, el.original_ids.data(), el.original_ids.size() * sizeof(int64_t));
    return static_cast<int64_t>(el.edges.size());
  } catch (const rst::ParseError& e) {
    g_err = e.what();
    *err_line = e.line();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int64_t ref_forest_depth(int64_t n, const int64_t* parent) {
  try {
    rst::RootedForest f = rst::forest_from_parent(std::vector<int64_t>(parent, parent + n));
    return rst::forest_depth(f).max_depth;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
