// device.cpp -- per-thread cache of device graph handles for host Graphs,
// and the mapping of C-ABI status codes to the reference's exception types.
#include "rst/device.hpp"

#include <stdexcept>
#include <vector>

namespace rst {

namespace {

struct Entry {
  const Graph* g = nullptr;
  const void* offsets = nullptr;
  const void* neighbors = nullptr;
  const void* edges = nullptr;
  std::int64_t n = -1, m = -1;
  int device = -1;
  rstg_graph* handle = nullptr;
};

struct Cache {
  std::vector<Entry> entries;
  ~Cache() {
    for (auto& e : entries)
      if (e.handle) rstg_graph_destroy(e.handle);
  }
};

thread_local Cache t_cache;
constexpr std::size_t kMaxEntries = 4;

}  // namespace

void rstg_check(int rc) {
  if (rc == RSTG_OK) return;
  const std::string msg = rstg_last_error();
  if (rc == RSTG_ERR_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

rstg_graph* device_graph(const Graph& g, int device) {
  for (auto& e : t_cache.entries) {
    if (e.g == &g && e.n == g.n && e.m == g.m && e.device == device &&
        e.offsets == g.offsets.data() && e.neighbors == g.neighbors.data() &&
        e.edges == static_cast<const void*>(g.edges.data()))
      return e.handle;
  }
  if (t_cache.entries.size() >= kMaxEntries) {
    rstg_graph_destroy(t_cache.entries.front().handle);
    t_cache.entries.erase(t_cache.entries.begin());
  }
  static_assert(sizeof(Edge) == 2 * sizeof(std::int64_t), "Edge must be two int64");
  rstg_graph* h = nullptr;
  const bool csr = static_cast<std::int64_t>(g.offsets.size()) == g.n + 1 &&
                   static_cast<std::int64_t>(g.neighbors.size()) == 2 * g.m &&
                   static_cast<std::int64_t>(g.edge_origin.size()) == 2 * g.m;
  rstg_check(rstg_graph_create(csr ? g.offsets.data() : nullptr,
                               csr ? g.neighbors.data() : nullptr,
                               csr ? g.edge_origin.data() : nullptr,
                               reinterpret_cast<const int64_t*>(g.edges.data()), g.n, g.m, device,
                               &h));
  Entry e;
  e.g = &g;
  e.offsets = g.offsets.data();
  e.neighbors = g.neighbors.data();
  e.edges = g.edges.data();
  e.n = g.n;
  e.m = g.m;
  e.device = device;
  e.handle = h;
  t_cache.entries.push_back(e);
  return h;
}

void drop_device_graphs() {
  for (auto& e : t_cache.entries)
    if (e.handle) rstg_graph_destroy(e.handle);
  t_cache.entries.clear();
}

}  // namespace rst
