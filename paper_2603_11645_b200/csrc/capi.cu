// capi.cu -- the extern "C" boundary (include/rstg.h).
//
// Host buffers in, host buffers out, int64 at the boundary like the
// reference's Graph / RootedForest; int32 on the device. Every entry point
// catches and maps exceptions: AlgoError -> RSTG_ERR_ALGO (reference
// std::runtime_error texts), ArgError -> RSTG_ERR_ARG, CUDA -> RSTG_ERR_CUDA.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/rstg.h"
#include "engine.hpp"
#include "scan.cuh"

#include <cub/cub.cuh>

namespace rstg {
void upload_reference_graph(Handle& h, const int64_t* offsets, const int64_t* nbrs,
                            const int64_t* origin, const int64_t* edges_uv, int64_t n, int64_t m);
void upload_edges_build_csr(Handle& h, const int64_t* edges_uv, int64_t n, int64_t m);
void adopt_device_graph(Handle& h, const int2* edges, const uint32_t* offsets, const int32_t* nbrs,
                        const uint32_t* arc_edge, int64_t n, int64_t m);
void generate_device(Handle& h, int kind, int64_t a, int64_t b, double p, bool build_csr);
const int2* edge_list_device(const rstg_edge_list* el, int64_t* n, int64_t* m);  // loader.cu
void widen_to_host(Handle& h, const int32_t* dev, int64_t count, int64_t* host);
int64_t forest_depth_device(Handle& h, const int32_t* parent, int32_t* depth, uint32_t* rootmax,
                            int64_t* cycle_vertex);
int64_t root_depths(Handle& h, const int32_t* parent, uint32_t* rootmax, int64_t n);
void launch_hook(Handle& h, int mode, const int2* edges, int64_t m, uint32_t e_base,
                 const int32_t* rep, unsigned long long* slot, int* any_prop);
void launch_apply(Handle& h, int32_t* rep, unsigned long long* slot, uint8_t* tflag,
                  uint32_t e_base, uint32_t m_local, unsigned long long* counter,
                  uint32_t* tlist);
void launch_cc_init(Handle& h, int32_t* rep, unsigned long long* slot);
void cc_hook_round(Handle& h, int mode, const int32_t* rep, unsigned long long* slot,
                   unsigned long long* out_count, int* any_prop,
                   unsigned long long* zero_word = nullptr);
void cc_round_done(Handle& h, int64_t out_count);
void cc_reset_rounds(Handle& h);
void launch_compress2(Handle& h, int32_t* rep, int64_t n);
void generate_kron_part(Handle& h, int scale, int ef, int part, int nparts);
}  // namespace rstg

#include "listrank.cuh"

using namespace rstg;

struct rstg_graph {
  explicit rstg_graph(int dev) : h(dev) {}
  Handle h;
  std::string phases_json = "{}";
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return RSTG_OK;
  } catch (const AlgoError& e) {
    g_err = e.what();
    return RSTG_ERR_ALGO;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RSTG_ERR_ARG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RSTG_ERR_CUDA;
  }
}

}  // namespace

// The same error mapping for entry points defined in other files.
namespace rstg {
int guard_call(const std::function<void()>& f) { return guard(f); }
}  // namespace rstg

namespace {
double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void fill_stats(rstg_stats* st, const Stats& s) {
  if (!st) return;
  st->steps = s.steps;
  st->work = s.work;
  st->rounds = s.rounds;
  st->launches = s.launches;
  st->tree_edges = s.tree_edges;
  st->components = s.components;
  st->levels = s.levels;
  st->device_ms = s.device_ms;
}

// Narrow a host int64 array into a device int32 buffer (small test inputs).
template <class T>
void to_device(Handle& h, const int64_t* host, int64_t count, T* dev) {
  std::vector<T> tmp((size_t)std::max<int64_t>(count, 1));
  for (int64_t i = 0; i < count; ++i) tmp[(size_t)i] = (T)host[i];
  CK(cudaMemcpyAsync(dev, tmp.data(), count * sizeof(T), cudaMemcpyHostToDevice, h.stream));
  CK(cudaStreamSynchronize(h.stream));
}

void check_root(Handle& h, int64_t root) {
  if (root < 0 || root >= h.g.n)
    throw AlgoError("root " + std::to_string(root) + " out of range");
}

// phase times: {"name": [total_ms, records, algorithmic_bytes], ...} in
// first-seen order (records: timed intervals of the phase in the run)
std::string phases_to_json(Handle& h) {
  auto ph = h.timer.collect();
  struct Agg {
    std::string name;
    double ms, bytes;
    int count;
  };
  std::vector<Agg> agg;
  for (auto& p : ph) {
    auto it = std::find_if(agg.begin(), agg.end(), [&](const Agg& a) { return a.name == p.name; });
    if (it == agg.end())
      agg.push_back({p.name, p.ms, p.bytes, 1});
    else
      it->ms += p.ms, it->bytes += p.bytes, it->count += 1;
  }
  std::string js = "{";
  for (size_t i = 0; i < agg.size(); ++i) {
    if (i) js += ",";
    char buf[256];
    std::snprintf(buf, sizeof buf, "\"%s\":[%.6f,%d,%.0f]", agg[i].name.c_str(), agg[i].ms,
                  agg[i].count, agg[i].bytes);
    js += buf;
  }
  return js + "}";
}

// The device pipeline of run_algorithm. Returns the roots count (roots
// written as int32 into `roots` when non-null).
int64_t run_pipeline(rstg_graph* g, int algo, int64_t root, int64_t jump_batch, int32_t* parent,
                     int32_t* levels, int32_t* roots) {
  Handle& h = g->h;
  check_root(h, root);
  h.stats = Stats{};
  h.late_check = nullptr;
  h.late_copy = {};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, h.stream));
  int64_t nroots = -1;
  if (algo == RSTG_BFS) {
    if (!levels) levels = h.ws<int32_t>(WS_BFS_LEVEL, h.g.n);
    if (!roots) roots = h.ws<int32_t>(WS_ROOTS, h.g.n + 1);
    nroots = bfs_rst(h, (int32_t)root, parent, levels, roots);
  } else if (algo == RSTG_CC_EULER) {
    // (a tree edge's eto word holds its edge index below a flag bit)
    if (h.g.m >= (int64_t{1} << 31))
      throw ArgError("cc-euler needs fewer than 2^31 edges on one device");
    int32_t* labels = h.ws<int32_t>(WS_REP, h.g.n);
    // round 0 runs from the CSR (and writes every local list) when there is one
    // (round 0 runs -- from keys or the CSR -- whenever there are edges and
    // either a CSR exists or is pending)
    const EulerIO io = euler_buffers(h, h.g.n, (h.g.has_csr() || h.round0_slots) && h.g.m > 0);
    const int64_t T = cc_exact(h, labels, nullptr, &io);
    euler_root(h, labels, io, h.g.n, T, /*cc_slots=*/true, (int32_t)root, parent);
  } else if (algo == RSTG_PR_RST) {
    pr_rst(h, (int32_t)root, jump_batch, parent);
  } else {
    throw ArgError("unknown algorithm");
  }
  CK(cudaEventRecord(e1, h.stream));
  if (h.late_check) {  // (the deferred tile-ranking check: before anything reads P)
    CK(cudaEventSynchronize(e1));
    auto f = std::move(h.late_check);
    h.late_check = nullptr;
    f();
  }
  if (roots && algo != RSTG_BFS) nroots = roots_ascending(h, parent, roots);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
  h.stats.device_ms = ms;
  if (nroots >= 0) h.stats.components = nroots;
  g->phases_json = phases_to_json(h);
  return nroots;
}

// rank of every position from its (ruler, offset) word (rstg_k_list_rank)
__global__ void k_rank_cover(int64_t E, const uint32_t* sl, const uint32_t* rstart, int ob,
                             uint32_t* rank) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = sl[p];  // (ruler << ob) | offset
    rank[p] = rstart[a >> ob] + (a & ((1u << ob) - 1u));
  }
}
__global__ void k_check_compressed(int64_t m, const int2* e, const int32_t* rep, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t ru = rep[e[i].x], rv = rep[e[i].y];
    if (rep[ru] != ru || rep[rv] != rv) *bad = 1;
  }
}
__global__ void k_jacobi(int64_t n, const int32_t* snap, int32_t* next, int* not_done) {
  bool pend = false;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t nv = snap[snap[v]];
    next[v] = nv;
    pend |= snap[nv] != nv;
  }
  block_flag(pend, not_done);
}

struct FlagF {
  const uint8_t* f;
  __device__ uint32_t operator()(int64_t e) const { return f[e]; }
};

int ceil_log2_i(int64_t x) {
  int k = 0;
  int64_t p = 1;
  while (p < x) {
    p <<= 1;
    ++k;
  }
  return k;
}
}  // namespace

extern "C" {

const char* rstg_last_error(void) { return g_err.c_str(); }

int rstg_device_count(int* count) {
  return guard([&] { CK(cudaGetDeviceCount(count)); });
}

int rstg_graph_create(const int64_t* offsets, const int64_t* neighbors, const int64_t* edge_origin,
                      const int64_t* edges_uv, int64_t n, int64_t m, int device, rstg_graph** out) {
  *out = nullptr;
  return guard([&] {
    auto* g = new rstg_graph(device);
    try {
      if (offsets && neighbors && edge_origin)
        upload_reference_graph(g->h, offsets, neighbors, edge_origin, edges_uv, n, m);
      else
        upload_edges_build_csr(g->h, edges_uv, n, m);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int rstg_graph_upload(rstg_graph* g, const int64_t* offsets, const int64_t* neighbors,
                      const int64_t* edge_origin, const int64_t* edges_uv, int64_t n, int64_t m) {
  return guard([&] {
    if (offsets && neighbors && edge_origin)
      upload_reference_graph(g->h, offsets, neighbors, edge_origin, edges_uv, n, m);
    else
      upload_edges_build_csr(g->h, edges_uv, n, m);
  });
}

int rstg_graph_create_device(const int32_t* d_edges_uv, const uint32_t* d_offsets,
                             const int32_t* d_nbrs, const uint32_t* d_arc_edge, int64_t n,
                             int64_t m, int device, rstg_graph** out) {
  *out = nullptr;
  return guard([&] {
    auto* g = new rstg_graph(device);
    try {
      adopt_device_graph(g->h, reinterpret_cast<const int2*>(d_edges_uv), d_offsets, d_nbrs,
                         d_arc_edge, n, m);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int rstg_graph_from_edge_list(const rstg_edge_list* el, int device, rstg_graph** out) {
  *out = nullptr;
  return guard([&] {
    int64_t n = 0, m = 0;
    const int2* edges = edge_list_device(el, &n, &m);
    auto* g = new rstg_graph(device);
    try {
      adopt_device_graph(g->h, edges, nullptr, nullptr, nullptr, n, m);  // CSR built on the device
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int rstg_graph_generate(const char* spec, int device, rstg_graph** out) {
  *out = nullptr;
  return guard([&] {
    std::vector<std::string> parts;
    std::string s(spec);
    size_t st = 0;
    for (;;) {
      size_t c = s.find(':', st);
      parts.push_back(s.substr(st, c == std::string::npos ? c : c - st));
      if (c == std::string::npos) break;
      st = c + 1;
    }
    size_t k = (!parts.empty() && parts[0] == "gen") ? 1 : 0;
    if (parts.size() <= k) throw ArgError("empty generator spec: " + s);
    const std::string kind = parts[k];
    auto num = [&](size_t i) -> int64_t {
      if (k + 1 + i >= parts.size()) throw ArgError("generator spec '" + s + "': wrong number of parameters");
      return std::stoll(parts[k + 1 + i]);
    };
    auto* g = new rstg_graph(device);
    try {
      if (kind == "path") generate_device(g->h, 0, num(0), 0, 0, true);
      else if (kind == "star") generate_device(g->h, 1, num(0), 0, 0, true);
      else if (kind == "grid") generate_device(g->h, 2, num(0), num(1), 0, true);
      else if (kind == "road")
        generate_device(g->h, 3, num(0), 0,
                        parts.size() > k + 2 ? std::stod(parts[k + 2]) : 0.2026, true);
      else if (kind == "kron")
        generate_device(g->h, 4, num(0), parts.size() > k + 2 ? num(1) : 16, 0, true);
      else
        throw ArgError("unknown generator kind: " + kind);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int rstg_graph_generate_part(const char* spec, int part, int nparts, int device,
                             rstg_graph** out) {
  *out = nullptr;
  return guard([&] {
    int scale = 0, ef = 16;
    if (std::sscanf(spec, "kron:%d:%d", &scale, &ef) < 1 &&
        std::sscanf(spec, "gen:kron:%d:%d", &scale, &ef) < 1)
      throw ArgError("partitioned generation supports kron:SCALE[:EF] only");
    if (nparts < 1 || part < 0 || part >= nparts) throw ArgError("bad partition");
    auto* g = new rstg_graph(device);
    try {
      generate_kron_part(g->h, scale, ef, part, nparts);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int rstg_graph_set_edge_base(rstg_graph* g, int64_t e_base) {
  return guard([&] {
    if (e_base < 0 || e_base + g->h.g.m > (int64_t{1} << 32)) throw ArgError("edge base out of range");
    g->h.g.e_base = e_base;
  });
}

int rstg_cc_labels(rstg_graph* g, int32_t* d_rep, uint8_t* d_tflag, int64_t* d_slot,
                   int64_t* d_xbuf, rstg_reduce_min_fn reduce_min, void* ctx, rstg_stats* stats) {
  return guard([&] {
    Handle& h = g->h;
    const double t0 = now_ms();
    h.stats = Stats{};
    if (reduce_min && (!d_slot || !d_xbuf)) throw ArgError("exchange needs slot and xbuf buffers");
    CcExchange ex{reduce_min, ctx, reinterpret_cast<unsigned long long*>(d_slot),
                  reinterpret_cast<unsigned long long*>(d_xbuf)};
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, h.stream));
    cc_exact(h, d_rep, d_tflag, nullptr, reduce_min ? &ex : nullptr);
    CK(cudaEventRecord(e1, h.stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    h.stats.device_ms = ms;
    g->phases_json = phases_to_json(h);
    fill_stats(stats, h.stats);
    if (stats) stats->total_ms = now_ms() - t0;
  });
}

int rstg_cc_init(rstg_graph* g, int32_t* d_rep, int64_t* d_slot) {
  return guard([&] {
    launch_cc_init(g->h, d_rep, reinterpret_cast<unsigned long long*>(d_slot));
    cc_reset_rounds(g->h);
    CK(cudaMemsetAsync(g->h.dev_box + 3, 0, sizeof(int64_t), g->h.stream));
    CK(cudaStreamSynchronize(g->h.stream));
  });
}

int rstg_cc_hook(rstg_graph* g, int mode, const int32_t* d_rep, int64_t* d_slot) {
  return guard([&] {
    Handle& h = g->h;
    // filtered round; its crossing-edge count is read back by rstg_cc_apply
    cc_hook_round(h, mode, d_rep, reinterpret_cast<unsigned long long*>(d_slot),
                  reinterpret_cast<unsigned long long*>(h.dev_box) + 3, nullptr);
    CK(cudaStreamSynchronize(h.stream));
  });
}

int rstg_cc_apply(rstg_graph* g, int32_t* d_rep, int64_t* d_slot, uint8_t* d_tflag,
                  int64_t* applied) {
  return guard([&] {
    Handle& h = g->h;
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 2;
    CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), h.stream));
    launch_apply(h, d_rep, reinterpret_cast<unsigned long long*>(d_slot), d_tflag,
                 (uint32_t)h.g.e_base, (uint32_t)h.g.m, ctr, nullptr);
    h.read_box(reinterpret_cast<int64_t*>(ctr), 2);  // [2] applied, [3] crossing edges
    *applied = h.host_box[0];
    cc_round_done(h, h.host_box[1]);
    CK(cudaMemsetAsync(h.dev_box + 3, 0, sizeof(int64_t), h.stream));
  });
}

int rstg_cc_compress(rstg_graph* g, int32_t* d_rep) {
  return guard([&] {
    launch_compress2(g->h, d_rep, g->h.g.n);
    CK(cudaStreamSynchronize(g->h.stream));
  });
}

int rstg_graph_info(const rstg_graph* g, int64_t* n, int64_t* m) {
  if (!g) return RSTG_ERR_ARG;
  *n = g->h.g.n;
  *m = g->h.g.m;
  return RSTG_OK;
}

int rstg_graph_edges(rstg_graph* g, int64_t* edges_uv) {
  return guard([&] {
    widen_to_host(g->h, reinterpret_cast<const int32_t*>(g->h.g.edges), 2 * g->h.g.m, edges_uv);
  });
}

int rstg_graph_edges_flagged(rstg_graph* g, const uint8_t* d_flags, int64_t* edges_uv,
                             int64_t cap, int64_t* count) {
  return guard([&] {
    Handle& h = g->h;
    const int64_t m = h.g.m;
    *count = 0;
    if (m == 0) return;
    // flagged edges in id order (cub select), then widened to the host
    int2* sel = h.ws<int2>(WS_VAL_A, m);
    long long* nsel = reinterpret_cast<long long*>(h.dev_box) + 48;
    size_t temp = 0;
    CK(cub::DeviceSelect::Flagged(nullptr, temp, h.g.edges, d_flags, sel, nsel, m, h.stream));
    void* tmp = h.ws(WS_SL, temp);
    CK(cub::DeviceSelect::Flagged(tmp, temp, h.g.edges, d_flags, sel, nsel, m, h.stream));
    h.read_box(reinterpret_cast<int64_t*>(nsel), 1);
    const int64_t c = h.host_box[0];
    if (c > cap) throw ArgError("output capacity too small");
    widen_to_host(h, reinterpret_cast<const int32_t*>(sel), 2 * c, edges_uv);
    *count = c;
  });
}

int rstg_graph_destroy(rstg_graph* g) {
  return guard([&] { delete g; });
}

int rstg_set_stream(rstg_graph* g, void* stream) {
  return guard([&] { g->h.set_stream(static_cast<cudaStream_t>(stream)); });
}

int rstg_set_timing(rstg_graph* g, int enabled) {
  g->h.timer.enabled = enabled != 0;
  return RSTG_OK;
}

int rstg_phase_times(rstg_graph* g, char* buf, int64_t cap) {
  if (!g || !buf || cap <= 0) return RSTG_ERR_ARG;
  std::strncpy(buf, g->phases_json.c_str(), (size_t)cap - 1);
  buf[cap - 1] = 0;
  return RSTG_OK;
}

int rstg_run(rstg_graph* g, int algo, int64_t root, int64_t jump_batch, int64_t* parent_out,
             int64_t* levels_out, int64_t* roots_out, int64_t* num_roots, rstg_stats* stats) {
  return guard([&] {
    const double t0 = now_ms();
    Handle& h = g->h;
    const int64_t n = h.g.n;
    int32_t* parent = h.ws<int32_t>(WS_PARENT, n);
    int32_t* levels = (algo == RSTG_BFS) ? h.ws<int32_t>(WS_BFS_LEVEL, n) : nullptr;
    int32_t* roots = h.ws<int32_t>(WS_ROOTS, n + 1);
    const int64_t nr = run_pipeline(g, algo, root, jump_batch, parent, levels, roots);
    int64_t d2h = 0;
    widen_to_host(h, parent, n, parent_out);
    d2h += n * 8;
    if (levels_out && levels) {
      widen_to_host(h, levels, n, levels_out);
      d2h += n * 8;
    }
    if (roots_out && nr > 0) {
      widen_to_host(h, roots, nr, roots_out);
      d2h += nr * 8;
    }
    if (num_roots) *num_roots = nr;
    fill_stats(stats, h.stats);
    if (stats) {
      stats->components = nr;
      stats->h2d_bytes = 0;
      stats->d2h_bytes = d2h;
      stats->total_ms = now_ms() - t0;
    }
  });
}

int rstg_run_device(rstg_graph* g, int algo, int64_t root, int64_t jump_batch, int32_t* d_parent,
                    int32_t* d_levels, rstg_stats* stats) {
  return guard([&] {
    const double t0 = now_ms();
    run_pipeline(g, algo, root, jump_batch, d_parent, d_levels, nullptr);
    fill_stats(stats, g->h.stats);
    if (stats) {
      stats->h2d_bytes = stats->d2h_bytes = 0;
      stats->total_ms = now_ms() - t0;
    }
  });
}

int rstg_cc_spanning_forest(rstg_graph* g, int64_t* labels_out, int64_t* tree_edges_out,
                            int64_t* num_tree_edges, rstg_stats* stats) {
  return guard([&] {
    Handle& h = g->h;
    h.stats = Stats{};
    const int64_t n = h.g.n, m = h.g.m;
    int32_t* labels = h.ws<int32_t>(WS_REP, n);
    uint8_t* tflag = h.ws<uint8_t>(WS_TFLAG, m);
    const int64_t T = cc_exact(h, labels, tflag);
    widen_to_host(h, labels, n, labels_out);
    uint32_t* ids = h.ws<uint32_t>(WS_POS, T + 1);
    if (m > 0) scan_emit(h, m, FlagF{tflag}, EmitCompact{ids}, false);
    std::vector<uint32_t> tmp((size_t)T);
    CK(cudaMemcpyAsync(tmp.data(), ids, T * sizeof(uint32_t), cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));
    for (int64_t i = 0; i < T; ++i) tree_edges_out[i] = tmp[(size_t)i];
    *num_tree_edges = T;
    fill_stats(stats, h.stats);
  });
}

int rstg_euler_root_forest(int64_t n, const int64_t* tree_uv, int64_t T, const int64_t* labels,
                           int64_t nlabels, int64_t designated_root, int device,
                           int64_t* parent_out, int64_t* roots_out, int64_t* num_roots) {
  return guard([&] {
    if (nlabels != n) throw AlgoError("labels size does not match vertex count");
    if (designated_root != -1 && (designated_root < 0 || designated_root >= n))
      throw AlgoError("designated root out of range");
    // Tree edges as a graph: oriented, sorted and deduplicated on the device
    // (arc order never changes parents); labels narrowed with a range check.
    rstg_graph gg(device);
    Handle& h = gg.h;
    int32_t* lab = h.ws<int32_t>(WS_REP, n);
    const int64_t bad_label = upload_ids(h, labels, n, lab, n);
    if (bad_label >= 0)
      throw AlgoError("label out of range at vertex " + std::to_string(bad_label));
    // the reference's order: the edge count (euler_rooting.cpp:205-208)
    // before anything the tour construction could reject
    const int64_t comps = count_labels(h, lab, n);
    if (T != n - comps) throw AlgoError("edge count does not match a spanning forest of the labeling");
    bool simple = true;
    if (!upload_tree_edges(h, tree_uv, T, n, &simple))
      throw AlgoError("tree edge endpoint out of range");
    int32_t* parent = h.ws<int32_t>(WS_PARENT, n);
    if (!simple) throw AlgoError("list ranking failed to converge: not a forest");
    const EulerIO io = euler_buffers(h, T, /*local_written=*/false);
    euler_link_edges(h, io, T);
    euler_root(h, lab, io, T, T, /*cc_slots=*/false, (int32_t)designated_root, parent,
               /*verify=*/true);
    // Not a forest iff some vertex is unreachable from its root: validate
    // the orientation by doubling (a cycle never resolves to a root).
    {
      int32_t* ra = h.ws<int32_t>(WS_VAL_A, n);
      int32_t* rb = h.ws<int32_t>(WS_VAL_B, n);
      int* nd = reinterpret_cast<int*>(h.dev_box + 50);
      CK(cudaMemcpyAsync(ra, parent, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, h.stream));
      const int rounds = ceil_log2_i(n < 2 ? 2 : n) + 1;
      for (int r = 0; r < rounds; ++r) {
        CK(cudaMemsetAsync(nd, 0, sizeof(int), h.stream));
        k_jacobi<<<grid_for(n), kBlock, 0, h.stream>>>(n, ra, rb, nd);
        std::swap(ra, rb);
      }
      CK_LAUNCH();
      h.read_box(reinterpret_cast<int64_t*>(nd), 1);
      if (*reinterpret_cast<int*>(h.host_box) != 0)
        throw AlgoError("list ranking failed to converge: not a forest");
    }
    int32_t* roots = h.ws<int32_t>(WS_ROOTS, n + 1);
    const int64_t nr = roots_ascending(h, parent, roots);
    // A cycle component keeps no root while another tree gets two: the
    // edge-count check then fails upstream; root count must match here.
    widen_to_host(h, parent, n, parent_out);
    if (roots_out && nr > 0) widen_to_host(h, roots, nr, roots_out);
    if (num_roots) *num_roots = nr;
  });
}

int rstg_forest_depth(rstg_graph* g, const int64_t* parent, int64_t* depth_out,
                      int64_t* root_max_out, int64_t* max_depth) {
  return guard([&] {
    Handle& h = g->h;
    const int64_t n = h.g.n;
    int32_t* p = h.ws<int32_t>(WS_PARENT, n);
    const int64_t bad = upload_ids(h, parent, n, p, n);  // (checked before use, like rstg_validate)
    if (bad >= 0) throw AlgoError("parent out of range at vertex " + std::to_string(bad));
    int32_t* depth = h.ws<int32_t>(WS_ROOTS, n + 1);  // (WS_VAL_C is the readback staging)
    uint32_t* rootmax = h.ws<uint32_t>(WS_MINV, n);
    h.minv_clean = nullptr;  // (WS_MINV reused here)
    int64_t cyc = -1;
    forest_depth_device(h, p, depth, rootmax, &cyc);
    if (cyc >= 0) {
      // the reference walks from the smallest vertex that never reaches a
      // root and names the first vertex its walk meets twice
      std::vector<char> seen((size_t)n, 0);
      int64_t x = cyc;
      while (!seen[(size_t)x]) {
        seen[(size_t)x] = 1;
        x = parent[x];
      }
      throw AlgoError("parent array contains a cycle at vertex " + std::to_string(x));
    }
    *max_depth = root_depths(h, p, rootmax, n);  // rootmax[v] := -1 for non-roots
    if (root_max_out) widen_to_host(h, reinterpret_cast<const int32_t*>(rootmax), n, root_max_out);
    if (depth_out) widen_to_host(h, depth, n, depth_out);
  });
}

int rstg_validate(rstg_graph* g, const int64_t* parent, int64_t required_root, int* valid,
                  int* code, int64_t* bad_vertex) {
  return guard([&] {
    Handle& h = g->h;
    int32_t* p = h.ws<int32_t>(WS_PARENT, h.g.n);
    // Range check while narrowing (out-of-range int64 values would wrap).
    const int64_t bad = upload_ids(h, parent, h.g.n, p, h.g.n);
    if (bad >= 0) {
      *valid = 0;
      *code = 1;
      *bad_vertex = bad;
      return;
    }
    int64_t bv = -1;
    const int c = validate_forest(h, p, (int32_t)required_root, &bv);
    *valid = c == 0;
    *code = c;
    *bad_vertex = bv;
  });
}

int rstg_k_hook_step(int64_t n, int64_t m, const int64_t* edges_uv, int mode, int64_t* rep,
                     uint8_t* tree_flag, int64_t* slot, int* applied) {
  return guard([&] {
    rstg_graph gg(0);
    Handle& h = gg.h;
    h.g.n = n;
    h.g.m = m;
    CK(cudaMalloc(&h.g.edges, std::max<int64_t>(m, 1) * sizeof(int2)));
    to_device<int32_t>(h, edges_uv, 2 * m, reinterpret_cast<int32_t*>(h.g.edges));
    int32_t* r = h.ws<int32_t>(WS_REP, n);
    to_device<int32_t>(h, rep, n, r);
    int* bad = reinterpret_cast<int*>(h.dev_box + 50);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), h.stream));
    k_check_compressed<<<grid_for(m), kBlock, 0, h.stream>>>(m, h.g.edges, r, bad);
    CK_LAUNCH();
    h.read_box(reinterpret_cast<int64_t*>(bad), 1);
    if (*reinterpret_cast<int*>(h.host_box)) throw AlgoError("hooking ran on uncompressed labels");
    unsigned long long* sl = h.ws<unsigned long long>(WS_SLOT, n);
    h.slots_clean = nullptr;  // (the caller's slot values go here)
    std::vector<unsigned long long> hs((size_t)n);
    for (int64_t v = 0; v < n; ++v)
      hs[(size_t)v] = (unsigned long long)slot[v];
    CK(cudaMemcpy(sl, hs.data(), n * 8, cudaMemcpyHostToDevice));
    uint8_t* tf = h.ws<uint8_t>(WS_TFLAG, m);
    CK(cudaMemcpy(tf, tree_flag, (size_t)m, cudaMemcpyHostToDevice));
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box);
    CK(cudaMemset(ctr, 0, 8));
    launch_hook(h, mode, h.g.edges, m, 0, r, sl, nullptr);
    launch_apply(h, r, sl, tf, 0, (uint32_t)m, ctr, nullptr);
    h.read_box(reinterpret_cast<int64_t*>(ctr), 1);
    *applied = h.host_box[0] != 0;
    std::vector<int32_t> hr((size_t)n);
    CK(cudaMemcpy(hr.data(), r, n * 4, cudaMemcpyDeviceToHost));
    for (int64_t v = 0; v < n; ++v) rep[v] = hr[(size_t)v];
    CK(cudaMemcpy(tree_flag, tf, (size_t)m, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hs.data(), sl, n * 8, cudaMemcpyDeviceToHost));
    for (int64_t v = 0; v < n; ++v) slot[v] = (int64_t)hs[(size_t)v];
    CK(cudaFree(h.g.edges));
    h.g.edges = nullptr;
  });
}

// jump_to_convergence exactly (Jacobi doubling, same round guard and the
// same error), cc_forest.cpp:50-71.
int rstg_k_jump(int64_t n, int64_t* rep) {
  return guard([&] {
    rstg_graph gg(0);
    Handle& h = gg.h;
    h.g.n = n;
    int32_t* a = h.ws<int32_t>(WS_REP, n);
    int32_t* b = h.ws<int32_t>(WS_PR_NEXT, n);
    to_device<int32_t>(h, rep, n, a);
    int* nd = reinterpret_cast<int*>(h.dev_box + 50);
    const int64_t max_rounds = ceil_log2_i(std::max<int64_t>(n, 1)) + 2;
    for (int64_t round = 0;; ++round) {
      if (round > max_rounds) throw AlgoError("pointer jumping failed to converge");
      CK(cudaMemsetAsync(nd, 0, sizeof(int), h.stream));
      k_jacobi<<<grid_for(n), kBlock, 0, h.stream>>>(n, a, b, nd);
      CK_LAUNCH();
      std::swap(a, b);
      h.read_box(reinterpret_cast<int64_t*>(nd), 1);
      if (*reinterpret_cast<int*>(h.host_box) == 0) break;
    }
    std::vector<int32_t> hr((size_t)n);
    CK(cudaMemcpy(hr.data(), a, n * 4, cudaMemcpyDeviceToHost));
    for (int64_t v = 0; v < n; ++v) rep[v] = hr[(size_t)v];
  });
}

int rstg_k_list_rank(int64_t E, const int64_t* succ, int64_t* rank) {
  return guard([&] {
    rstg_graph gg(0);
    Handle& h = gg.h;
    h.g.n = E;
    uint32_t* s = h.ws<uint32_t>(WS_SUCC, E);
    std::vector<uint32_t> hs((size_t)E);
    for (int64_t p = 0; p < E; ++p) hs[(size_t)p] = succ[p] < 0 ? kNone32 : (uint32_t)succ[p];
    CK(cudaMemcpy(s, hs.data(), E * 4, cudaMemcpyHostToDevice));
    uint32_t* sl = h.ws<uint32_t>(WS_SL, E);
    LrParams P;
    const uint32_t* rstart = lr_rank_lists(h, E, s, sl, /*verify=*/true, &P);
    uint32_t* rk = h.ws<uint32_t>(WS_ETO, E);
    k_rank_cover<<<grid_for(E), kBlock, 0, h.stream>>>(E, sl, rstart, P.ob, rk);
    CK_LAUNCH();
    std::vector<uint32_t> hr((size_t)E);
    CK(cudaMemcpy(hr.data(), rk, E * 4, cudaMemcpyDeviceToHost));
    for (int64_t p = 0; p < E; ++p) rank[p] = hr[(size_t)p];
  });
}

}  // extern "C"
