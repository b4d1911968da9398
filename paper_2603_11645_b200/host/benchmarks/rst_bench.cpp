// rst_bench -- microbenchmark driver, the drop-in for the reference's
// proj/benchmarks/algo_bench.cpp (google-benchmark is not available here).
// Same case families (path 2^10/2^12/2^14, grid 32x32 and 100x100,
// random(n, 0.005)) x the three strategies; reports wall ms per
// run_algorithm call (host graph in, host parents out), device ms, and the
// steps / n counters. `--shapes` adds the BASELINE.json shapes (grid 1024^2,
// road-like 24M mesh, path 16M) with the same protocol.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

#include "rst/bench.hpp"
#include "rst/graph.hpp"

namespace {

struct Case {
  std::string name;
  std::string spec;
};

void run_case(const Case& c, int reps) {
  const rst::Graph g = rst::build_csr(rst::generate(rst::parse_gen_spec(c.spec), 1));
  for (rst::AlgoKind algo : rst::kAllAlgos) {
    if (algo == rst::AlgoKind::kBfs && g.n > (1 << 22) && c.spec.rfind("path", 0) == 0) continue;
    rst::RunOptions opt;
    rst::run_algorithm(g, algo, opt);  // warm-up + upload
    std::vector<double> wall;
    rst::RunResult last;
    for (int i = 0; i < reps; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      last = rst::run_algorithm(g, algo, opt);
      wall.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                         .count());
    }
    std::sort(wall.begin(), wall.end());
    std::printf("%-22s %-9s n=%-10lld m=%-10lld wall_ms=%9.3f steps=%lld\n", c.name.c_str(),
                rst::algo_name(algo), static_cast<long long>(g.n), static_cast<long long>(g.m),
                wall[wall.size() / 2], static_cast<long long>(last.report.steps));
  }
}

}  // namespace

int main(int argc, char** argv) {
  bool shapes = false;
  int reps = 5;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--shapes") shapes = true;
    if (a == "--reps" && i + 1 < argc) reps = std::max(1, std::atoi(argv[++i]));
  }
  std::vector<Case> cases;
  for (int k : {10, 12, 14}) cases.push_back({"BM_Path/" + std::to_string(1 << k), "path:" + std::to_string(1 << k)});
  for (int s : {32, 100}) cases.push_back({"BM_Grid/" + std::to_string(s), "grid:" + std::to_string(s) + ":" + std::to_string(s)});
  for (int k : {10, 12, 14})
    cases.push_back({"BM_Random/" + std::to_string(1 << k), "random:" + std::to_string(1 << k) + ":0.005"});
  if (shapes) {
    cases.push_back({"grid-1024^2", "grid:1024:1024"});
    cases.push_back({"road-24M", "road:4899"});
    cases.push_back({"path-16M", "path:16777216"});
  }
  try {
    for (const Case& c : cases) run_case(c, reps);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
