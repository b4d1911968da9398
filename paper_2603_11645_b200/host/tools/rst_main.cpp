// rst -- command-line driver of the B200 engine, the drop-in for the
// reference's proj/tools/rst_main.cpp: same subcommands (run, bench, stats,
// gen, validate), flags, output formats and exit codes (0 ok, 1 invalid
// result / error, 2 usage). CLI11 and nlohmann/json are not available, so
// the argument parser and the JSON writer are hand-rolled.
#include <charconv>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "rst/bench.hpp"
#include "rst/bfs_rst.hpp"
#include "rst/graph.hpp"
#include "rst/rooted_forest.hpp"
#include "rst/validate.hpp"

namespace {

struct Args {
  std::vector<std::string> positional;
  std::map<std::string, std::vector<std::string>> opts;
  std::map<std::string, bool> flags;
};

const char* kUsage =
    "usage: rst <run|bench|stats|gen|validate> ...\n"
    "  rst run <source> [bfs|cc-euler|pr-rst] [--algo A] [--dump-parents F] [--json]\n"
    "  rst bench <sources...> [--algo A]... [--out F]\n"
    "  rst stats <source>\n"
    "  rst gen <path|star|grid|random|complete|road|kron> <params...> [--out F]\n"
    "  rst validate <source> <parents>\n"
    "common: --root R --seed S --workers W (1..256) --jump-batch J (1..20) --device D\n"
    "sources: a file path or gen:<spec>\n";

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

Args parse_args(int argc, char** argv, int from) {
  static const char* value_opts[] = {"--root", "--seed",   "--workers", "--jump-batch",
                                     "--algo", "--out",    "--dump-parents", "--device"};
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string s = argv[i];
    if (s == "--json") {
      a.flags["--json"] = true;
      continue;
    }
    if (s.rfind("--", 0) == 0) {
      std::string key = s, val;
      const auto eq = s.find('=');
      if (eq != std::string::npos) {
        key = s.substr(0, eq);
        val = s.substr(eq + 1);
      } else {
        bool known = false;
        for (const char* o : value_opts) known = known || key == o;
        if (!known) throw UsageError("unknown option " + key);
        if (i + 1 >= argc) throw UsageError(key + " needs a value");
        val = argv[++i];
      }
      a.opts[key].push_back(val);
      continue;
    }
    a.positional.push_back(s);
  }
  return a;
}

template <class T>
T num(const std::string& s, const char* what) {
  T v{};
  auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc{} || r.ptr != s.data() + s.size())
    throw UsageError(std::string(what) + ": not a number: " + s);
  return v;
}

struct Common {
  std::int64_t root = 0;
  std::uint64_t seed = 0;
  int workers = 1;
  std::int64_t jump_batch = 5;
  int device = 0;
  bool root_given = false;
};

Common common(const Args& a) {
  Common c;
  auto last = [&](const char* k) -> const std::string* {
    auto it = a.opts.find(k);
    return it == a.opts.end() ? nullptr : &it->second.back();
  };
  if (auto v = last("--root")) {
    c.root = num<std::int64_t>(*v, "--root");
    c.root_given = true;
  }
  if (auto v = last("--seed")) c.seed = num<std::uint64_t>(*v, "--seed");
  if (auto v = last("--workers")) {
    c.workers = num<int>(*v, "--workers");
    if (c.workers < 1 || c.workers > 256) throw UsageError("--workers: value not in range 1 to 256");
  }
  if (auto v = last("--jump-batch")) {
    c.jump_batch = num<std::int64_t>(*v, "--jump-batch");
    if (c.jump_batch < 1 || c.jump_batch > 20)
      throw UsageError("--jump-batch: value not in range 1 to 20");
  }
  if (auto v = last("--device")) c.device = num<int>(*v, "--device");
  return c;
}

rst::RunOptions run_options(const Common& c) {
  rst::RunOptions o;
  o.root = c.root;
  o.workers = c.workers;
  o.jump_batch = c.jump_batch;
  o.device = c.device;
  return o;
}

rst::Graph load_graph(const std::string& src, std::uint64_t seed) {
  return rst::build_csr(rst::load_source(src, seed));
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

std::string json_num(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, r.ptr);
}

int cmd_run(const Args& a) {
  if (a.positional.empty()) throw UsageError("run: source is required");
  const Common c = common(a);
  std::string algo_s = a.positional.size() > 1 ? a.positional[1] : "bfs";
  if (auto it = a.opts.find("--algo"); it != a.opts.end()) algo_s = it->second.back();
  const auto algo = rst::parse_algo(algo_s);
  if (!algo) {
    std::cerr << "unknown algorithm: " << algo_s << "\n";
    return 2;
  }
  const std::string& source = a.positional[0];
  const rst::Graph g = load_graph(source, c.seed);
  const rst::RunResult res = rst::run_algorithm(g, *algo, run_options(c));
  const rst::ValidationReport rep = rst::validate_rooted_forest(g, res.forest, c.root);
  const rst::DepthStats depth = rst::forest_depth(res.forest);
  if (auto it = a.opts.find("--dump-parents"); it != a.opts.end()) {
    std::ofstream out(it->second.back());
    if (!out) {
      std::cerr << "cannot write " << it->second.back() << "\n";
      return 1;
    }
    rst::write_parent_array(out, res.forest.parent);
  }
  if (a.flags.count("--json")) {
    // keys in sorted order, two-space indent (the reference's json dump)
    std::map<std::string, std::string> j;
    j["source"] = json_str(source);
    j["algorithm"] = json_str(algo_s);
    j["n"] = std::to_string(g.n);
    j["m"] = std::to_string(g.m);
    j["root"] = std::to_string(c.root);
    j["steps"] = std::to_string(res.report.steps);
    j["work"] = std::to_string(res.report.work);
    j["wall_ms"] = json_num(res.report.wall_ms);
    j["tree_depth"] = std::to_string(depth.max_depth);
    j["components"] = std::to_string(res.forest.roots.size());
    j["valid"] = rep.valid ? "true" : "false";
    std::cout << "{\n";
    std::size_t i = 0;
    for (const auto& [k, v] : j) std::cout << "  \"" << k << "\": " << v << (++i < j.size() ? ",\n" : "\n");
    std::cout << "}\n";
  } else {
    std::cout << "source      " << source << "\n"
              << "algorithm   " << algo_s << "\n"
              << "n           " << g.n << "\n"
              << "m           " << g.m << "\n"
              << "root        " << c.root << "\n"
              << "steps       " << res.report.steps << "\n"
              << "work        " << res.report.work << "\n"
              << "wall_ms     " << res.report.wall_ms << "\n"
              << "tree_depth  " << depth.max_depth << "\n"
              << "components  " << res.forest.roots.size() << "\n"
              << "valid       " << (rep.valid ? "true" : "false") << "\n";
  }
  if (!rep.valid) {
    for (const auto& e : rep.errors) std::cerr << "validation: " << e << "\n";
    return 1;
  }
  return 0;
}

int cmd_bench(const Args& a) {
  if (a.positional.empty()) throw UsageError("bench: at least one source is required");
  const Common c = common(a);
  std::vector<std::string> names = {"bfs", "cc-euler", "pr-rst"};
  if (auto it = a.opts.find("--algo"); it != a.opts.end()) names = it->second;
  std::vector<rst::AlgoKind> algos;
  for (const auto& nm : names) {
    const auto k = rst::parse_algo(nm);
    if (!k) {
      std::cerr << "unknown algorithm: " << nm << "\n";
      return 2;
    }
    algos.push_back(*k);
  }
  std::ofstream file;
  if (auto it = a.opts.find("--out"); it != a.opts.end()) {
    file.open(it->second.back());
    if (!file) {
      std::cerr << "cannot write " << it->second.back() << "\n";
      return 1;
    }
  }
  std::ostream& out = file.is_open() ? file : std::cout;
  rst::write_csv_header(out);
  bool ok = true;
  for (const auto& src : a.positional) {
    const rst::Graph g = load_graph(src, c.seed);
    for (rst::AlgoKind k : algos) {
      const rst::BenchRecord r = rst::bench_row(g, src, k, run_options(c));
      rst::write_csv_row(out, r);
      ok = ok && r.valid;
    }
  }
  return ok ? 0 : 1;
}

int cmd_stats(const Args& a) {
  if (a.positional.empty()) throw UsageError("stats: source is required");
  const Common c = common(a);
  const rst::Graph g = load_graph(a.positional[0], c.seed);
  rst::StepEngine engine(c.workers, c.device);
  const rst::RootedForest f = rst::bfs_rst(g, c.root, engine);
  std::int64_t depth = 0;
  for (const auto& [r, d] : rst::forest_depth(f).per_root)
    if (r == c.root) depth = d;
  std::cout << "n           " << g.n << "\n"
            << "m           " << g.m << "\n"
            << "components  " << f.roots.size() << "\n"
            << "depth       " << depth << "\n";
  return 0;
}

int cmd_gen(const Args& a) {
  if (a.positional.empty()) throw UsageError("gen: kind is required");
  const Common c = common(a);
  std::string spec = a.positional[0];
  for (std::size_t i = 1; i < a.positional.size(); ++i) spec += ":" + a.positional[i];
  const rst::EdgeList el = rst::generate(rst::parse_gen_spec(spec), c.seed);
  std::ofstream file;
  if (auto it = a.opts.find("--out"); it != a.opts.end()) {
    file.open(it->second.back());
    if (!file) {
      std::cerr << "cannot write " << it->second.back() << "\n";
      return 1;
    }
  }
  rst::write_edge_list(file.is_open() ? static_cast<std::ostream&>(file) : std::cout, el);
  return 0;
}

int cmd_validate(const Args& a) {
  if (a.positional.size() < 2) throw UsageError("validate: source and parents are required");
  const Common c = common(a);
  const rst::Graph g = load_graph(a.positional[0], c.seed);
  std::ifstream in(a.positional[1]);
  if (!in) {
    std::cerr << "file not found: " << a.positional[1] << "\n";
    return 1;
  }
  const rst::RootedForest f = rst::forest_from_parent(rst::read_parent_array(in));
  const rst::ValidationReport rep =
      rst::validate_rooted_forest(g, f, c.root_given ? c.root : rst::kNone);
  if (rep.valid) {
    std::cout << "valid rooted spanning forest (" << f.roots.size() << " components)\n";
    return 0;
  }
  for (const auto& e : rep.errors) std::cerr << "violation: " << e << "\n";
  return 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage;
    return 2;
  }
  const std::string sub = argv[1];
  try {
    const Args a = parse_args(argc, argv, 2);
    if (sub == "run") return cmd_run(a);
    if (sub == "bench") return cmd_bench(a);
    if (sub == "stats") return cmd_stats(a);
    if (sub == "gen") return cmd_gen(a);
    if (sub == "validate") return cmd_validate(a);
    std::cerr << kUsage;
    return 2;
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\n" << kUsage;
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
