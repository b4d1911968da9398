// loader.cu -- the edge-list / MatrixMarket loader (load_edge_list,
// graph.cpp:48-127) for large real inputs (road_usa, europe_osm:
// PAPER.md:175-179), B200-first:
//
//   parse      the text buffer is cut at line boundaries into one chunk per
//              host thread; each thread tokenizes its lines (std::from_chars,
//              the reference's rules: '\n' lines, a trailing '\r' dropped,
//              blanks and tabs separate tokens, '#'/'%' comment lines, an
//              optional MatrixMarket size line after a "%%" banner) into
//              int64 pairs. Errors carry the 1-based line number of the
//              FIRST offending line in file order, whatever the chunking.
//   ids        on the device: all 2m endpoints radix-sorted and
//              deduplicated; dense when count == max + 1 (edges kept as
//              read), else every endpoint is remapped to its rank by binary
//              search over the sorted ids (original_ids keeps the table).
//   normalize  on the device (graph.cpp:39-46): self-loops dropped, (u, v)
//              oriented u < v, radix-sorted, deduplicated -- the input of
//              build_csr, and of rstg_graph_from_edge_list without a host
//              round trip.
#include <cub/cub.cuh>

#include <algorithm>
#include <charconv>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rstg.h"
#include "engine.hpp"

namespace rstg {

int guard_call(const std::function<void()>& f);  // capi.cu
void adopt_device_graph(Handle& h, const int2* edges, const uint32_t* offsets, const int32_t* nbrs,
                        const uint32_t* arc_edge, int64_t n, int64_t m);
void widen_to_host(Handle& h, const int32_t* dev, int64_t count, int64_t* host);

namespace {

struct ParseFail {
  int64_t line = -1;  // 1-based; -1: none
  std::string what;
};

bool is_blank(char c) { return c == ' ' || c == '\t'; }

// One line of the reference's loop body (graph.cpp:60-92) minus the
// header bookkeeping: 0 = blank/comment, 1 = pair (vals), 2 = error.
// ntok_out = token count (for the MatrixMarket size-line test).
int parse_line(const char* b, const char* e, int64_t vals[3], int* ntok_out, std::string* err) {
  if (e > b && e[-1] == '\r') --e;
  const char* p = b;
  while (p < e && is_blank(*p)) ++p;
  if (p == e) return 0;
  if (*p == '#' || *p == '%') return 0;
  int ntok = 0;
  while (p < e) {
    while (p < e && is_blank(*p)) ++p;
    if (p == e) break;
    const char* q = p;
    while (q < e && !is_blank(*q)) ++q;
    if (ntok < 3) {
      auto r = std::from_chars(p, q, vals[ntok]);
      if (r.ec != std::errc{} || r.ptr != q) {
        *err = "expected integer, got '" + std::string(p, q) + "'";
        return 2;
      }
    }
    ++ntok;
    p = q;
  }
  *ntok_out = ntok;
  return 1;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0;  // '\n'-terminated lines (+1 for an unterminated tail)
  std::vector<long long> uv;
  int64_t err_local = -1;  // 0-based line within the chunk
  std::string err;
};

void parse_chunk(Chunk& c) {
  const char* p = c.b;
  int64_t ln = 0;
  while (p < c.e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(c.e - p)));
    const char* le = nl ? nl : c.e;
    int64_t vals[3];
    int ntok = 0;
    std::string err;
    const int k = parse_line(p, le, vals, &ntok, &err);
    if (k == 2 || (k == 1 && ntok != 2) || (k == 1 && (vals[0] < 0 || vals[1] < 0))) {
      if (k == 1)
        err = ntok != 2 ? "expected 2 integer tokens, got " + std::to_string(ntok)
                        : std::string("negative vertex id");
      c.err_local = ln;
      c.err = err;
      return;
    }
    if (k == 1) {
      c.uv.push_back(vals[0]);
      c.uv.push_back(vals[1]);
    }
    ++ln;
    p = nl ? nl + 1 : c.e;
  }
  c.lines = ln;
}

// The whole text: pairs in file order, or the first error.
std::vector<long long> parse_text(const char* text, int64_t len, int threads, ParseFail* fail) {
  std::vector<long long> out;
  const char* end = text + len;
  // Sequential prefix up to the first data line: the MatrixMarket banner
  // ("%%...") must precede it for a 3-token first data line to be the size
  // line that is skipped (graph.cpp:86-90).
  const char* p = text;
  int64_t line = 0;
  bool saw_mm = false;
  while (p < end) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
    const char* le = nl ? nl : end;
    ++line;
    const char* s = p;
    const char* se = (le > p && le[-1] == '\r') ? le - 1 : le;
    while (s < se && is_blank(*s)) ++s;
    if (s == se || *s == '#' || *s == '%') {
      if (s + 1 < se && s[0] == '%' && s[1] == '%') saw_mm = true;
      p = nl ? nl + 1 : end;
      continue;
    }
    // the first data line
    int64_t vals[3];
    int ntok = 0;
    std::string err;
    const int k = parse_line(p, le, vals, &ntok, &err);
    if (k == 2) {
      fail->line = line;
      fail->what = err;
      return out;
    }
    if (!(saw_mm && ntok == 3)) {
      if (ntok != 2) {
        fail->line = line;
        fail->what = "expected 2 integer tokens, got " + std::to_string(ntok);
        return out;
      }
      if (vals[0] < 0 || vals[1] < 0) {
        fail->line = line;
        fail->what = "negative vertex id";
        return out;
      }
      out.push_back(vals[0]);
      out.push_back(vals[1]);
    }
    p = nl ? nl + 1 : end;
    break;
  }
  // The rest in parallel, chunks cut after a '\n'.
  const int64_t rest = end - p;
  int T = std::max(1, threads);
  if (rest < (int64_t{1} << 20)) T = 1;
  std::vector<Chunk> chunks(T);
  const char* cb = p;
  for (int t = 0; t < T; ++t) {
    const char* ce = (t == T - 1) ? end : p + rest * (t + 1) / T;
    if (ce < cb) ce = cb;
    if (t < T - 1 && ce < end) {
      const char* nl = static_cast<const char*>(memchr(ce, '\n', (size_t)(end - ce)));
      ce = nl ? nl + 1 : end;
    }
    chunks[t].b = cb;
    chunks[t].e = ce;
    cb = ce;
  }
  if (T == 1) {
    parse_chunk(chunks[0]);
  } else {
    std::vector<std::thread> th;
    th.reserve(T);
    for (int t = 0; t < T; ++t) th.emplace_back(parse_chunk, std::ref(chunks[t]));
    for (auto& x : th) x.join();
  }
  int64_t base = line;
  size_t total = out.size();
  for (auto& c : chunks) {
    if (c.err_local >= 0) {
      fail->line = base + c.err_local + 1;
      fail->what = c.err;
      return out;
    }
    base += c.lines;
    total += c.uv.size();
  }
  out.reserve(total);
  for (auto& c : chunks) {
    out.insert(out.end(), c.uv.begin(), c.uv.end());
    std::vector<long long>().swap(c.uv);
  }
  return out;
}

// ---- device side ----------------------------------------------------------
__global__ void k_ids(int64_t count, const long long* __restrict__ uv, unsigned long long* ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    ids[i] = (unsigned long long)uv[i];
}
// endpoint -> rank in the sorted distinct ids (the reference's remap)
__global__ void k_remap(int64_t count, const long long* __restrict__ uv,
                        const unsigned long long* __restrict__ ids, int64_t nid, bool dense,
                        int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = (unsigned long long)uv[i];
    if (dense) {
      out[i] = (int32_t)x;
      continue;
    }
    int64_t lo = 0, hi = nid;  // lower_bound
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ids[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    out[i] = (int32_t)lo;
  }
}
__global__ void k_keys(int64_t m, const int2* __restrict__ e, unsigned long long* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 x = e[i];
    const uint32_t a = (uint32_t)min(x.x, x.y), b = (uint32_t)max(x.x, x.y);
    keys[i] = (x.x == x.y) ? ~0ull : (((unsigned long long)a << 32) | b);
  }
}
__global__ void k_unkey(int64_t m, const unsigned long long* __restrict__ keys, int2* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    out[i] = make_int2((int)(k >> 32), (int)(uint32_t)k);
  }
}

// Scoped device buffer.
template <class T>
struct Dev {
  T* p = nullptr;
  explicit Dev(int64_t count) { CK(cudaMalloc(&p, std::max<int64_t>(count, 1) * sizeof(T))); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

// sorted distinct values of keys[0, count) into out (count returned)
int64_t sort_unique(Handle& h, unsigned long long* keys, unsigned long long* out, int64_t count,
                    int end_bit) {
  Dev<unsigned long long> sorted(count);
  size_t t1 = 0, t2 = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, keys, sorted.p, count, 0, end_bit, h.stream));
  long long* nsel = reinterpret_cast<long long*>(h.dev_box) + 48;
  CK(cub::DeviceSelect::Unique(nullptr, t2, sorted.p, out, nsel, count, h.stream));
  Dev<char> tmp((int64_t)std::max(t1, t2));
  CK(cub::DeviceRadixSort::SortKeys(tmp.p, t1, keys, sorted.p, count, 0, end_bit, h.stream));
  CK(cub::DeviceSelect::Unique(tmp.p, t2, sorted.p, out, nsel, count, h.stream));
  h.read_box(reinterpret_cast<int64_t*>(nsel), 1);
  return h.host_box[0];
}

}  // namespace
}  // namespace rstg

using namespace rstg;

// A normalized edge list on the device (EdgeList, graph.hpp:17-23).
struct rstg_edge_list {
  explicit rstg_edge_list(int dev) : h(dev) {}
  ~rstg_edge_list() { cudaFree(edges); }
  Handle h;
  int2* edges = nullptr;
  int64_t n = 0, m = 0;
  std::vector<int64_t> original_ids;  // sparse external ids (empty: identity)
};

namespace {
thread_local int64_t t_err_line = -1;
}

extern "C" {

int rstg_parse_edge_text(const char* text, int64_t len, int threads, int64_t* uv_out, int64_t cap,
                         int64_t* count, int64_t* err_line) {
  *err_line = -1;
  *count = 0;
  ParseFail f;
  int rc = guard_call([&] {
    std::vector<long long> uv = parse_text(text, len, threads, &f);
    if (f.line >= 0) throw ArgError("line " + std::to_string(f.line) + ": " + f.what);
    const int64_t c = (int64_t)uv.size() / 2;
    *count = c;
    if (uv_out && c <= cap) std::memcpy(uv_out, uv.data(), uv.size() * sizeof(long long));
  });
  if (rc == RSTG_ERR_ARG && f.line >= 0) {
    *err_line = f.line;
    return RSTG_ERR_PARSE;
  }
  return rc;
}

int rstg_edge_list_load(const char* text, int64_t len, int threads, int device,
                        rstg_edge_list** out, int64_t* err_line) {
  *out = nullptr;
  t_err_line = -1;
  if (err_line) *err_line = -1;
  ParseFail f;
  int rc = guard_call([&] {
    std::vector<long long> uv = parse_text(text, len, threads, &f);
    if (f.line >= 0) throw ArgError("line " + std::to_string(f.line) + ": " + f.what);
    if (uv.empty()) throw AlgoError("empty edge-list input: no data lines");
    auto* el = new rstg_edge_list(device);
    try {
      Handle& h = el->h;
      const int64_t two_m = (int64_t)uv.size(), m = two_m / 2;
      Dev<long long> duv(two_m);
      CK(cudaMemcpyAsync(duv.p, uv.data(), two_m * sizeof(long long), cudaMemcpyHostToDevice,
                         h.stream));
      std::vector<long long>().swap(uv);  // (the copy above is synchronous for pageable memory)
      // distinct ids: dense (count == max + 1) or remapped to their ranks
      Dev<unsigned long long> ids(two_m), uniq(two_m);
      k_ids<<<grid_for(two_m), kBlock, 0, h.stream>>>(two_m, duv.p, ids.p);
      CK_LAUNCH();
      const int64_t nid = sort_unique(h, ids.p, uniq.p, two_m, 64);
      unsigned long long maxid = 0;
      CK(cudaMemcpy(&maxid, uniq.p + nid - 1, sizeof(maxid), cudaMemcpyDeviceToHost));
      const bool dense = (unsigned long long)nid == maxid + 1;
      const int64_t n = dense ? (int64_t)maxid + 1 : nid;
      if (n > (int64_t{1} << 31)) throw AlgoError("graph too large: vertex ids exceed 2^31");
      Dev<int32_t> r(two_m);
      k_remap<<<grid_for(two_m), kBlock, 0, h.stream>>>(two_m, duv.p, uniq.p, nid, dense, r.p);
      CK_LAUNCH();
      if (!dense) {
        el->original_ids.resize((size_t)nid);
        CK(cudaMemcpy(el->original_ids.data(), uniq.p, nid * sizeof(int64_t),
                      cudaMemcpyDeviceToHost));
      }
      // normalize (graph.cpp:39-46): the self-loop sentinel sorts last
      Dev<unsigned long long> keys(m), ukeys(m);
      k_keys<<<grid_for(m), kBlock, 0, h.stream>>>(m, reinterpret_cast<const int2*>(r.p), keys.p);
      CK_LAUNCH();
      int64_t mm = sort_unique(h, keys.p, ukeys.p, m, 64);
      if (mm > 0) {
        unsigned long long last = 0;
        CK(cudaMemcpy(&last, ukeys.p + mm - 1, sizeof(last), cudaMemcpyDeviceToHost));
        if (last == ~0ull) --mm;
      }
      if (mm > (int64_t{1} << 32)) throw AlgoError("too many edges");
      CK(cudaMalloc(&el->edges, std::max<int64_t>(mm, 1) * sizeof(int2)));
      if (mm > 0) k_unkey<<<grid_for(mm), kBlock, 0, h.stream>>>(mm, ukeys.p, el->edges);
      CK_LAUNCH();
      CK(cudaStreamSynchronize(h.stream));
      el->n = n;
      el->m = mm;
    } catch (...) {
      delete el;
      throw;
    }
    *out = el;
  });
  if (rc == RSTG_ERR_ARG && f.line >= 0) {
    t_err_line = f.line;
    if (err_line) *err_line = f.line;
    return RSTG_ERR_PARSE;
  }
  return rc;
}

int rstg_edge_list_info(const rstg_edge_list* el, int64_t* n, int64_t* m, int64_t* n_original_ids) {
  *n = el->n;
  *m = el->m;
  if (n_original_ids) *n_original_ids = (int64_t)el->original_ids.size();
  return RSTG_OK;
}

int rstg_edge_list_copy(rstg_edge_list* el, int64_t* edges_uv, int64_t* original_ids) {
  return guard_call([&] {
    if (edges_uv && el->m > 0)
      widen_to_host(el->h, reinterpret_cast<const int32_t*>(el->edges), 2 * el->m, edges_uv);
    if (original_ids && !el->original_ids.empty())
      std::memcpy(original_ids, el->original_ids.data(), el->original_ids.size() * sizeof(int64_t));
  });
}

int rstg_edge_list_destroy(rstg_edge_list* el) {
  delete el;
  return RSTG_OK;
}

}  // extern "C"

// rstg_graph_from_edge_list lives in capi.cu (it owns rstg_graph).
namespace rstg {
const int2* edge_list_device(const rstg_edge_list* el, int64_t* n, int64_t* m) {
  *n = el->n;
  *m = el->m;
  return el->edges;
}
}  // namespace rstg
