// graph.cu -- device graph ingestion.
//
//   * upload of the reference's host Graph (graph.hpp:29-43: int64 CSR +
//     edge list) narrowed to int32/uint32 on the device;
//   * CSR construction on the device from a normalized edge list with the
//     exact layout of build_csr (graph.cpp:133-172): per vertex the
//     back-arcs to smaller neighbours (ascending) then the forward arcs
//     (ascending); edge_origin = edge id;
//   * normalize (graph.cpp:39-46) on the device: drop self-loops, orient
//     u < v, sort, dedup;
//   * device generators for the benchmark shapes (path, star, grid, the
//     road mesh and Graph500 Kronecker of SURVEY.md Appendix B), producing
//     exactly the host generators' edge lists.
// Sorting here (normalize, back-arc grouping) uses CUB's radix sort: graph
// ingestion is outside the RST hot path.
#include <algorithm>
#include <cub/cub.cuh>

#include "engine.hpp"
#include "graphgen.hpp"
#include "scan.cuh"

namespace rstg {

// ------------------------------------------------------------ narrowing
template <class T>
__global__ void k_narrow(int64_t count, const long long* __restrict__ in, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)in[i];
}
__global__ void k_widen(int64_t count, const int32_t* __restrict__ in, long long* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Device int32 -> host int64. Pinned destinations are written directly by
// the widening kernel over the host link (no staging round trip).
void widen_to_host(Handle& h, const int32_t* dev, int64_t count, int64_t* host) {
  if (count <= 0) return;
  if (is_pinned(host)) {
    k_widen<<<grid_for(count), kBlock, 0, h.stream>>>(count, dev, reinterpret_cast<long long*>(host));
    CK_LAUNCH();
    CK(cudaStreamSynchronize(h.stream));
    return;
  }
  const int64_t chunk = int64_t{1} << 24;
  long long* stage = h.ws<long long>(WS_VAL_C, std::min(count, chunk));
  for (int64_t off = 0; off < count; off += chunk) {
    const int64_t c = std::min(chunk, count - off);
    k_widen<<<grid_for(c), kBlock, 0, h.stream>>>(c, dev + off, stage);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(host + off, stage, c * sizeof(int64_t), cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));  // stage reused by the next chunk
  }
}

// int64 host array -> device int32/uint32. Pinned sources are read directly
// by the narrowing kernel (zero-copy over the host link); pageable ones go
// through a staging buffer.
// Checked variant (caller id arrays): every value must lie in [0, hi); the
// index of the first one that does not is returned (-1: all in range).
__global__ void k_narrow_checked(int64_t count, const long long* __restrict__ in, int32_t* out,
                                 int64_t base, long long hi, long long* first_bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = in[i];
    if (v < 0 || v >= hi) atomicMin(first_bad, (long long)(base + i));
    out[i] = (int32_t)v;
  }
}
int64_t upload_ids(Handle& h, const int64_t* host, int64_t count, int32_t* dev, int64_t hi) {
  if (count <= 0) return -1;
  long long* bad = reinterpret_cast<long long*>(h.dev_box + 57);
  const long long inf = INT64_MAX;
  CK(cudaMemcpyAsync(bad, &inf, sizeof(inf), cudaMemcpyHostToDevice, h.stream));
  if (is_pinned(host)) {
    k_narrow_checked<<<grid_for(count), kBlock, 0, h.stream>>>(
        count, reinterpret_cast<const long long*>(host), dev, 0, hi, bad);
    CK_LAUNCH();
  } else {
    const int64_t chunk = int64_t{1} << 24;
    long long* stage = h.ws<long long>(WS_VAL_C, std::min(count, chunk));
    for (int64_t off = 0; off < count; off += chunk) {
      const int64_t c = std::min(chunk, count - off);
      CK(cudaMemcpyAsync(stage, host + off, c * sizeof(int64_t), cudaMemcpyHostToDevice, h.stream));
      k_narrow_checked<<<grid_for(c), kBlock, 0, h.stream>>>(c, stage, dev + off, off, hi, bad);
      CK_LAUNCH();
      if (off + c < count) CK(cudaStreamSynchronize(h.stream));  // stage reused
    }
  }
  h.read_box(reinterpret_cast<int64_t*>(bad), 1);
  return h.host_box[0] == INT64_MAX ? -1 : h.host_box[0];
}

template <class T>
static void upload_narrow(Handle& h, const int64_t* host, int64_t count, T* dev) {
  if (count <= 0) return;
  if (is_pinned(host)) {
    k_narrow<T><<<grid_for(count), kBlock, 0, h.stream>>>(
        count, reinterpret_cast<const long long*>(host), dev);
    CK_LAUNCH();
    return;
  }
  const int64_t chunk = int64_t{1} << 24;  // 16M elements = 128 MB staging
  long long* stage = h.ws<long long>(WS_VAL_C, std::min(count, chunk));
  for (int64_t off = 0; off < count; off += chunk) {
    const int64_t c = std::min(chunk, count - off);
    CK(cudaMemcpyAsync(stage, host + off, c * sizeof(int64_t), cudaMemcpyHostToDevice, h.stream));
    k_narrow<T><<<grid_for(c), kBlock, 0, h.stream>>>(c, stage, dev + off);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(h.stream));  // stage reused by the next chunk
  }
}

static void alloc_graph(Handle& h, int64_t n, int64_t m, bool csr) {
  h.round0_slots = nullptr;  // (new edges: any upload keys are stale)
  h.edge_locality = -1;
  h.tile_segments = -1;
  if (n < 0) throw ArgError("negative vertex count");
  if (n >= (int64_t{1} << 31)) throw ArgError("graph too large: vertex ids exceed 2^31");
  if (m > (int64_t{1} << 32)) throw ArgError("too many edges");
  if (h.g.edges && h.g.n == n && h.g.m == m && (h.g.offsets != nullptr) == csr) return;  // reuse
  h.free_graph();
  h.g.n = n;
  h.g.m = m;
  CK(cudaMalloc(&h.g.edges, std::max<int64_t>(m, 1) * sizeof(int2)));
  if (csr) {
    if (2 * m >= (int64_t{1} << 32)) throw ArgError("CSR needs 2m < 2^32 arcs");
    CK(cudaMalloc(&h.g.offsets, (n + 1) * sizeof(uint32_t)));
    CK(cudaMalloc(&h.g.nbrs, std::max<int64_t>(2 * m, 1) * sizeof(int32_t)));
    CK(cudaMalloc(&h.g.arc_edge, std::max<int64_t>(2 * m, 1) * sizeof(uint32_t)));
  }
}

// Host Graph of the reference (graph.hpp:29-43) -> device.
void upload_reference_graph(Handle& h, const int64_t* offsets, const int64_t* nbrs,
                            const int64_t* origin, const int64_t* edges_uv, int64_t n, int64_t m) {
  const bool csr = offsets != nullptr && 2 * m < (int64_t{1} << 32);
  alloc_graph(h, n, m, csr);
  h.g.csr_pending = false;
  h.round0_slots = nullptr;
  h.edge_locality = -1;
  h.tile_segments = -1;
  if (csr) {
    upload_narrow<uint32_t>(h, offsets, n + 1, h.g.offsets);
    upload_narrow<int32_t>(h, nbrs, 2 * m, h.g.nbrs);
    upload_narrow<uint32_t>(h, origin, 2 * m, h.g.arc_edge);
  }
  upload_narrow<int32_t>(h, edges_uv, 2 * m, reinterpret_cast<int32_t*>(h.g.edges));
  CK(cudaStreamSynchronize(h.stream));
}

// ------------------------------------------------------ CSR on device
__global__ void k_degrees(int64_t m, const int2* __restrict__ e, uint32_t* fdeg, uint32_t* bdeg) {
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < m;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool ok = i < m;
    const int2 uv = ok ? e[i] : make_int2(-1, -1);
    // warp-aggregate equal endpoints (runs of equal u are contiguous)
    const unsigned fu = __match_any_sync(0xffffffffu, uv.x);
    const unsigned fv = __match_any_sync(0xffffffffu, uv.y);
    const int lane = threadIdx.x & 31;
    if (ok && (__ffs(fu) - 1) == lane) atomicAdd(&fdeg[uv.x], (uint32_t)__popc(fu));
    if (ok && (__ffs(fv) - 1) == lane) atomicAdd(&bdeg[uv.y], (uint32_t)__popc(fv));
  }
}
__global__ void k_keys_v(int64_t m, const int2* __restrict__ e, uint32_t* keys, uint32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (uint32_t)e[i].y;
    vals[i] = (uint32_t)i;
  }
}
__global__ void k_place_forward(int64_t m, const int2* __restrict__ e, const uint32_t* __restrict__ off,
                                const uint32_t* __restrict__ bdeg, const uint32_t* __restrict__ fs,
                                int32_t* nbrs, uint32_t* arc_edge) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 uv = e[i];
    const uint32_t pos = off[uv.x] + bdeg[uv.x] + ((uint32_t)i - fs[uv.x]);
    nbrs[pos] = uv.y;
    arc_edge[pos] = (uint32_t)i;
  }
}
__global__ void k_place_back(int64_t m, const int2* __restrict__ e, const uint32_t* __restrict__ skey,
                             const uint32_t* __restrict__ sval, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ bs, int32_t* nbrs, uint32_t* arc_edge) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = skey[k], i = sval[k];
    const uint32_t pos = off[v] + ((uint32_t)k - bs[v]);
    nbrs[pos] = e[i].x;
    arc_edge[pos] = i;
  }
}

namespace {
struct ArrF {
  const uint32_t* a;
  __device__ uint32_t operator()(int64_t i) const { return a[i]; }
};
struct SumF {
  const uint32_t* a;
  const uint32_t* b;
  __device__ uint32_t operator()(int64_t i) const { return a[i] + b[i]; }
};
}  // namespace

// build_csr (graph.cpp:133-172) on the device for h.g.edges (normalized).
void build_csr_device(Handle& h) {
  const int64_t n = h.g.n, m = h.g.m;
  const cudaStream_t s = h.stream;
  uint32_t* fdeg = h.ws<uint32_t>(WS_TF, n + 1);
  uint32_t* bdeg = h.ws<uint32_t>(WS_MINV, n + 1);
  h.minv_clean = nullptr;  // (WS_MINV reused here)
  uint32_t* fs = h.ws<uint32_t>(WS_HEADS, n + 1);
  uint32_t* bs = h.ws<uint32_t>(WS_RPOS, n + 1);
  CK(cudaMemsetAsync(fdeg, 0, (n + 1) * sizeof(uint32_t), s));
  CK(cudaMemsetAsync(bdeg, 0, (n + 1) * sizeof(uint32_t), s));
  if (m > 0) {
    k_degrees<<<grid_for(m), kBlock, 0, s>>>(m, h.g.edges, fdeg, bdeg);
    CK_LAUNCH();
  }
  scan_emit(h, n, SumF{fdeg, bdeg}, EmitExcl{h.g.offsets, n}, false);
  scan_emit(h, n, ArrF{fdeg}, EmitExcl{fs, n}, false);
  scan_emit(h, n, ArrF{bdeg}, EmitExcl{bs, n}, false);
  if (n == 0) CK(cudaMemsetAsync(h.g.offsets, 0, sizeof(uint32_t), s));
  if (m == 0) {
    CK(cudaStreamSynchronize(s));
    h.g.csr_pending = false;
    return;
  }
  k_place_forward<<<grid_for(m), kBlock, 0, s>>>(m, h.g.edges, h.g.offsets, bdeg, fs, h.g.nbrs,
                                                h.g.arc_edge);
  CK_LAUNCH();
  // back arcs: stable sort of edge ids by v
  uint32_t* kin = h.ws<uint32_t>(WS_ATO, m);
  uint32_t* vin = h.ws<uint32_t>(WS_AFROM, m);
  uint32_t* kout = h.ws<uint32_t>(WS_SUCC, m);
  uint32_t* vout = h.ws<uint32_t>(WS_REV, m);
  k_keys_v<<<grid_for(m), kBlock, 0, s>>>(m, h.g.edges, kin, vin);
  CK_LAUNCH();
  int end_bit = 1;
  while (end_bit < 32 && ((int64_t)1 << end_bit) < n) ++end_bit;
  size_t temp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, kin, kout, vin, vout, (int64_t)m, 0, end_bit, s));
  void* tmp = h.ws(WS_SL, temp);
  CK(cub::DeviceRadixSort::SortPairs(tmp, temp, kin, kout, vin, vout, (int64_t)m, 0, end_bit, s));
  k_place_back<<<grid_for(m), kBlock, 0, s>>>(m, h.g.edges, kout, vout, h.g.offsets, bs, h.g.nbrs,
                                             h.g.arc_edge);
  CK_LAUNCH();
  CK(cudaStreamSynchronize(s));
  h.g.csr_pending = false;
}

// ------------------------------------------------------ normalize on device
__global__ void k_pack_keys(int64_t m, const int2* __restrict__ raw, unsigned long long* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 e = raw[i];
    const uint32_t a = (uint32_t)min(e.x, e.y), b = (uint32_t)max(e.x, e.y);
    keys[i] = (e.x == e.y) ? ~0ull : (((unsigned long long)a << 32) | b);
  }
}
__global__ void k_unpack_keys(int64_t m, const unsigned long long* __restrict__ keys, int2* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    out[i] = make_int2((int)(k >> 32), (int)(uint32_t)k);
  }
}

// normalize (graph.cpp:39-46): keys -> sorted unique edges; returns m.
int64_t normalize_keys_device(Handle& h, unsigned long long* keys, int64_t count, int64_t n,
                              int2* out) {
  const cudaStream_t s = h.stream;
  unsigned long long* sorted = h.ws<unsigned long long>(WS_VAL_B, count);
  int end_bit = 1;
  while (end_bit < 64 && ((uint64_t)1 << end_bit) <= ((uint64_t)n << 32)) ++end_bit;
  end_bit = 64;  // self-loop sentinel is all ones
  size_t temp = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, temp, keys, sorted, count, 0, end_bit, s));
  void* tmp = h.ws(WS_SL, temp);
  CK(cub::DeviceRadixSort::SortKeys(tmp, temp, keys, sorted, count, 0, end_bit, s));
  long long* nsel = reinterpret_cast<long long*>(h.dev_box) + 48;
  size_t temp2 = 0;
  CK(cub::DeviceSelect::Unique(nullptr, temp2, sorted, keys, nsel, count, s));
  void* tmp2 = h.ws(WS_SL, temp2);
  CK(cub::DeviceSelect::Unique(tmp2, temp2, sorted, keys, nsel, count, s));
  h.read_box(reinterpret_cast<int64_t*>(nsel), 1);
  int64_t m = h.host_box[0];
  // drop the self-loop sentinel (sorted last)
  if (m > 0) {
    unsigned long long last = 0;
    CK(cudaMemcpy(&last, keys + m - 1, sizeof(last), cudaMemcpyDeviceToHost));
    if (last == ~0ull) --m;
  }
  if (m > 0) {
    k_unpack_keys<<<grid_for(m), kBlock, 0, s>>>(m, keys, out);
    CK_LAUNCH();
  }
  CK(cudaStreamSynchronize(s));
  return m;
}

bool upload_tree_edges(Handle& h, const int64_t* tree_uv, int64_t T, int64_t n, bool* simple) {
  alloc_graph(h, n, T, 2 * T < (int64_t{1} << 32));
  h.g.csr_pending = h.g.offsets != nullptr;
  *simple = true;
  if (T == 0) return true;
  unsigned long long* keys = h.ws<unsigned long long>(WS_VAL_A, T);
  int2* raw = reinterpret_cast<int2*>(keys);  // (packed in place below)
  if (upload_ids(h, tree_uv, 2 * T, reinterpret_cast<int32_t*>(raw), n) >= 0) return false;
  k_pack_keys<<<grid_for(T), kBlock, 0, h.stream>>>(T, raw, keys);
  CK_LAUNCH();
  *simple = normalize_keys_device(h, keys, T, n, h.g.edges) == T;
  return true;
}

// ------------------------------------------------------ device generators
namespace {
struct GridCount {  // grid (graph.cpp:198-210) and road mesh
  int64_t rows, cols;
  uint64_t thr;
  bool road;
  __device__ uint32_t operator()(int64_t id) const {
    const int64_t r = id / cols, c = id % cols;
    uint32_t k = (c + 1 < cols) ? 1u : 0u;
    if (r + 1 < rows && (!road || road_vertical((uint64_t)id, thr))) ++k;
    return k;
  }
};
struct GridEmit {
  GridCount gc;
  int2* out;
  __device__ void operator()(int64_t id, uint32_t p, uint32_t k) const {
    if (!k) return;
    const int64_t r = id / gc.cols, c = id % gc.cols;
    if (c + 1 < gc.cols) out[p++] = make_int2((int)id, (int)(id + 1));
    if (r + 1 < gc.rows && (!gc.road || road_vertical((uint64_t)id, gc.thr)))
      out[p] = make_int2((int)id, (int)(id + gc.cols));
  }
};
}  // namespace

__global__ void k_gen_path(int64_t n, int2* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_int2((int)i, (int)(i + 1));
}
__global__ void k_gen_star(int64_t n, int2* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_int2(0, (int)(i + 1));
}
__global__ void k_gen_kron(int64_t tuples, int scale, unsigned long long* keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tuples;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u, v;
    kron_tuple((uint64_t)e, scale, &u, &v);
    u = kron_perm(u, scale);
    v = kron_perm(v, scale);
    const uint64_t a = u < v ? u : v, b = u < v ? v : u;
    keys[e] = (u == v) ? ~0ull : ((a << 32) | b);
  }
}

// kind: 0 path(n) 1 star(n) 2 grid(rows, cols) 3 road(R, p) 4 kron(scale, ef)
void generate_device(Handle& h, int kind, int64_t a, int64_t b, double p, bool build_csr) {
  const cudaStream_t s = h.stream;
  if (kind == 0 || kind == 1) {
    if (a < 1) throw ArgError(kind == 0 ? "path: n must be >= 1" : "star: n must be >= 1");
    alloc_graph(h, a, a - 1, build_csr);
    if (a > 1) {
      if (kind == 0)
        k_gen_path<<<grid_for(a), kBlock, 0, s>>>(a, h.g.edges);
      else
        k_gen_star<<<grid_for(a), kBlock, 0, s>>>(a, h.g.edges);
      CK_LAUNCH();
    }
  } else if (kind == 2 || kind == 3) {
    const int64_t rows = a, cols = (kind == 2) ? b : a;
    if (rows < 1 || cols < 1) throw ArgError("grid: dimensions must be >= 1");
    GridCount gc{rows, cols, road_threshold(p), kind == 3};
    const int64_t n = rows * cols;
    int2* tmp = reinterpret_cast<int2*>(h.ws<unsigned long long>(WS_VAL_B, 2 * n + 1));
    const uint32_t m = scan_emit(h, n, gc, GridEmit{gc, tmp}, true);
    alloc_graph(h, n, m, build_csr);
    CK(cudaMemcpyAsync(h.g.edges, tmp, (size_t)m * sizeof(int2), cudaMemcpyDeviceToDevice, s));
  } else if (kind == 4) {
    const int scale = (int)a;
    const int64_t tuples = b << scale;
    if (scale < 1 || scale > 30) throw ArgError("kron: scale must be in [1, 30]");
    unsigned long long* keys = h.ws<unsigned long long>(WS_VAL_A, tuples);
    k_gen_kron<<<grid_for(tuples), kBlock, 0, s>>>(tuples, scale, keys);
    CK_LAUNCH();
    int2* tmp = reinterpret_cast<int2*>(h.ws<unsigned long long>(WS_VAL_C, tuples));
    const int64_t m = normalize_keys_device(h, keys, tuples, int64_t{1} << scale, tmp);
    alloc_graph(h, int64_t{1} << scale, m, build_csr && 2 * m < (int64_t{1} << 32));
    CK(cudaMemcpyAsync(h.g.edges, tmp, (size_t)m * sizeof(int2), cudaMemcpyDeviceToDevice, s));
  } else {
    throw ArgError("unknown generator kind");
  }
  CK(cudaStreamSynchronize(s));
  if (h.g.offsets) build_csr_device(h);
}

// ---- Kronecker partition by smaller endpoint (multi-GPU CC) -------------
// Edges of the globally normalized list are sorted by u = min endpoint, so
// the edges with u in [lo, hi) form one contiguous range of the global
// list. A part is generated in sub-ranges (each sort <= 2^29 keys) and
// appended in order.
__global__ void k_kron_count(int64_t tuples, int scale, uint32_t lo, uint32_t hi, int nsub,
                             unsigned long long* counts) {
  __shared__ unsigned long long sc[64];
  for (int i = threadIdx.x; i < nsub; i += blockDim.x) sc[i] = 0;
  __syncthreads();
  const uint64_t span = hi - lo;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tuples;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u, v;
    kron_tuple((uint64_t)e, scale, &u, &v);
    u = kron_perm(u, scale);
    v = kron_perm(v, scale);
    const uint64_t a = u < v ? u : v;
    if (u == v || a < lo || a >= hi) continue;
    const int sub = (int)(((a - lo) * (uint64_t)nsub) / span);
    atomicAdd(&sc[sub], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nsub; i += blockDim.x)
    if (sc[i]) atomicAdd(&counts[i], sc[i]);
}
__global__ void k_kron_emit(int64_t tuples, int scale, uint32_t lo, uint32_t hi, int nsub, int sub,
                            unsigned long long* keys, unsigned long long* ctr) {
  const uint64_t span = hi - lo;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tuples;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u, v;
    kron_tuple((uint64_t)e, scale, &u, &v);
    u = kron_perm(u, scale);
    v = kron_perm(v, scale);
    const uint64_t a = u < v ? u : v, b = u < v ? v : u;
    if (u == v || a < lo || a >= hi) continue;
    if ((int)(((a - lo) * (uint64_t)nsub) / span) != sub) continue;
    keys[atomicAdd(ctr, 1ull)] = (a << 32) | b;
  }
}

void generate_kron_part(Handle& h, int scale, int ef, int part, int nparts) {
  if (scale < 1 || scale > 30) throw ArgError("kron: scale must be in [1, 30]");
  const cudaStream_t s = h.stream;
  const int64_t n = int64_t{1} << scale, tuples = (int64_t)ef << scale;
  const uint32_t lo = (uint32_t)(n * part / nparts), hi = (uint32_t)(n * (part + 1) / nparts);
  const int64_t sub_target = int64_t{1} << 29;
  // expected tuples in the part ~ tuples / nparts (skewed ids are permuted)
  int nsub = (int)std::min<int64_t>(64, std::max<int64_t>(1, (tuples / nparts) / sub_target + 1));
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(h.dev_box) + 160;  // [160,224)
  CK(cudaMemsetAsync(counts, 0, 64 * sizeof(unsigned long long), s));
  k_kron_count<<<grid_for(tuples), kBlock, 0, s>>>(tuples, scale, lo, hi, nsub, counts);
  CK_LAUNCH();
  h.read_box(reinterpret_cast<int64_t*>(counts), nsub);
  std::vector<int64_t> cnt(h.host_box, h.host_box + nsub);
  int64_t total = 0, maxc = 1;
  for (int64_t c : cnt) {
    total += c;
    maxc = std::max(maxc, c);
  }
  h.free_graph();
  int2* edges = nullptr;
  CK(cudaMalloc(&edges, std::max<int64_t>(total, 1) * sizeof(int2)));
  unsigned long long* keys = h.ws<unsigned long long>(WS_VAL_A, maxc);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 224;
  int64_t m = 0;
  for (int sub = 0; sub < nsub; ++sub) {
    if (cnt[sub] == 0) continue;
    CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
    k_kron_emit<<<grid_for(tuples), kBlock, 0, s>>>(tuples, scale, lo, hi, nsub, sub, keys, ctr);
    CK_LAUNCH();
    m += normalize_keys_device(h, keys, cnt[sub], n, edges + m);
  }
  h.release(WS_VAL_A);
  h.release(WS_VAL_B);
  h.release(WS_SL);
  h.g.n = n;
  h.g.m = m;
  h.g.edges = edges;
  h.g.e_base = 0;
}

// Narrows a chunk of int64 (u, v) pairs into the device edge list and
// records round 0's hook proposal of each edge on the way: with every rep a
// singleton, min-mode hooking offers slot[v] the key (u << 32 | e) (u < v
// in a normalized list), the smallest of which is v's first neighbour --
// exactly what the CSR-direct round 0 reads (cc.cu).
//
// It also checks the input the way build_csr does (graph.cpp:145-156): the
// first edge (in list order) with an endpoint out of [0, n) or a self-loop
// is recorded in err[0] / err[1] (atomicMin of its index) and gets no key;
// err[2] is raised when an edge is not strictly above its predecessor
// (unsorted or duplicate: "EdgeList not normalized").
__global__ void k_narrow_edges(int64_t count, const long long* __restrict__ in, int2* out,
                               uint32_t e_first, int64_t n, unsigned long long* slot,
                               long long* err, int2 prev_last) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const long long u = in[2 * i], v = in[2 * i + 1];
    const int64_t id = (int64_t)e_first + i;
    if (u < 0 || u >= n || v < 0 || v >= n) {
      atomicMin(&err[0], (long long)id);
      out[i] = make_int2(0, 0);
      continue;
    }
    if (u == v) atomicMin(&err[1], (long long)id);
    const int2 e = make_int2((int)u, (int)v);
    out[i] = e;
    long long pu, pv;
    if (i > 0) {
      pu = in[2 * i - 2];
      pv = in[2 * i - 1];
    } else {
      pu = prev_last.x;
      pv = prev_last.y;
    }
    if ((i > 0 || e_first > 0) && !(pu < u || (pu == u && pv < v))) err[2] = 1;
    if (e.x != e.y) {  // (build_csr admits u > v: the loser is max(u, v) either way)
      const int lo = min(e.x, e.y), hi = max(e.x, e.y);
      const unsigned long long key = pack_key((uint32_t)lo, (uint32_t)id);
      if (key < slot[hi]) atomicMin(&slot[hi], key);
    }
  }
}
__global__ void k_fill_u64(int64_t count, unsigned long long* p, unsigned long long v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

void ensure_csr(Handle& h) {
  if (!h.g.csr_pending) return;
  const Stats keep = h.stats;  // ingestion, not the algorithm: reruns count alike
  build_csr_device(h);
  h.stats = keep;
  h.g.csr_pending = false;
}

// Round 0's hook keys from the device edge list (a graph uploaded for an
// earlier build whose keys were consumed, no CSR built, or one rank's
// partition). The smaller endpoint of every edge gets the sentinel
// kKeyEdge (above every real key, below empty): after round 0 a slot still
// empty marks an isolated vertex, which then never enters the roots list
// (the CSR path knows degrees; this path learns them here, and across ranks
// the MIN exchange carries the sentinel like any key).
__global__ void k_round0_keys(int64_t m, const int2* __restrict__ edges, uint32_t e_base,
                              unsigned long long* slot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 e = edges[i];
    if (e.x != e.y) {
      const int lo = min(e.x, e.y), hi = max(e.x, e.y);
      const unsigned long long key = pack_key((uint32_t)lo, e_base + (uint32_t)i);
      if (key < slot[hi]) atomicMin(&slot[hi], key);
      if (slot[lo] == kKeyInf) atomicMin(&slot[lo], kKeyEdge);
    }
  }
}
void launch_round0_keys(Handle& h, unsigned long long* slot) {
  k_round0_keys<<<grid_for(h.g.m), kBlock, 0, h.stream>>>(h.g.m, h.g.edges, (uint32_t)h.g.e_base,
                                                          slot);
  CK_LAUNCH();
}
bool round0_keys_from_edges(Handle& h, unsigned long long* slot) {
  // (a built CSR serves round 0 directly; without one -- pending, or a
  // graph too large for 32-bit arc offsets -- the keys come from the edges)
  if ((h.g.has_csr() && !h.g.csr_pending) || h.g.m == 0) return false;
  if (h.slots_clean != slot || h.g.n > h.slots_clean_n) {
    k_fill_u64<<<grid_for(h.g.n), kBlock, 0, h.stream>>>(h.g.n, slot, kKeyInf);
    CK_LAUNCH();
  }
  launch_round0_keys(h, slot);
  return true;
}

// Normalized int64 edge list (the reference EdgeList) -> device graph.
// The edges stream in through two staging buffers (DMA of chunk k + 1
// overlaps the narrowing of chunk k), round 0's hook keys are computed on
// the way, and the CSR is left pending: cc-euler never needs it.
void upload_edges_build_csr(Handle& h, const int64_t* edges_uv, int64_t n, int64_t m) {
  alloc_graph(h, n, m, 2 * m < (int64_t{1} << 32));
  h.g.csr_pending = h.g.offsets != nullptr;
  unsigned long long* slot = h.ws<unsigned long long>(WS_SLOT, n);
  const cudaStream_t s = h.stream;
  if ((h.slots_clean != slot || n > h.slots_clean_n) && n > 0) {
    k_fill_u64<<<grid_for(n), kBlock, 0, s>>>(n, slot, kKeyInf);
    CK_LAUNCH();
  }
  h.slots_clean = nullptr;
  h.round0_slots = nullptr;
  h.edge_locality = -1;
  h.tile_segments = -1;
  if (m > 0) {
    if (!h.copy_stream) CK(cudaStreamCreateWithFlags(&h.copy_stream, cudaStreamNonBlocking));
    const int64_t chunk = int64_t{1} << 22;  // edges per staging buffer (32 MB of int64 pairs)
    long long* stage = h.ws<long long>(WS_VAL_C, 2 * 2 * chunk);
    long long* err = reinterpret_cast<long long*>(h.dev_box + 54);  // [54,57): input checks
    const long long err_init[3] = {INT64_MAX, INT64_MAX, 0};
    CK(cudaMemcpyAsync(err, err_init, sizeof(err_init), cudaMemcpyHostToDevice, s));
    int2 last = make_int2(0, 0);
    cudaEvent_t copied[2], consumed[2];
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&consumed[b], cudaEventDisableTiming));
      CK(cudaEventRecord(consumed[b], s));
    }
    for (int64_t off = 0, k = 0; off < m; off += chunk, ++k) {
      const int b = (int)(k & 1);
      const int64_t c = std::min(chunk, m - off);
      long long* buf = stage + b * 2 * chunk;
      CK(cudaStreamWaitEvent(h.copy_stream, consumed[b], 0));
      CK(cudaMemcpyAsync(buf, edges_uv + 2 * off, c * 2 * sizeof(int64_t), cudaMemcpyHostToDevice,
                         h.copy_stream));
      CK(cudaEventRecord(copied[b], h.copy_stream));
      CK(cudaStreamWaitEvent(s, copied[b], 0));
      k_narrow_edges<<<grid_for(c), kBlock, 0, s>>>(c, buf, h.g.edges + off, (uint32_t)off, n,
                                                     slot, err, last);
      CK_LAUNCH();
      CK(cudaEventRecord(consumed[b], s));
      // the chunk's last edge, for the next chunk's order check (host copy:
      // the source array is the caller's)
      last = make_int2((int)std::clamp<int64_t>(edges_uv[2 * (off + c) - 2], -1, n),
                       (int)std::clamp<int64_t>(edges_uv[2 * (off + c) - 1], -1, n));
    }
    CK(cudaStreamSynchronize(s));
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(copied[b]);
      cudaEventDestroy(consumed[b]);
    }
    h.read_box(reinterpret_cast<int64_t*>(err), 3);
    const int64_t bad_range = h.host_box[0], bad_loop = h.host_box[1], unsorted = h.host_box[2];
    if (bad_range != INT64_MAX || bad_loop != INT64_MAX || unsorted) {
      // the reference's build_csr order: per edge range then self-loop, then the sort check
      const char* what = bad_range < bad_loop ? "edge endpoint out of range"
                         : bad_loop != INT64_MAX ? "self-loop in normalized EdgeList"
                                                 : "EdgeList not normalized";
      h.free_graph();
      h.slots_clean = nullptr;
      throw ArgError(what);
    }
    h.round0_slots = slot;
  } else if (h.g.offsets) {
    build_csr_device(h);
    h.g.csr_pending = false;
  }
  CK(cudaStreamSynchronize(s));
}

// Device int32 arrays -> handle-owned copies.
void adopt_device_graph(Handle& h, const int2* edges, const uint32_t* offsets, const int32_t* nbrs,
                        const uint32_t* arc_edge, int64_t n, int64_t m) {
  const bool csr = offsets != nullptr;
  alloc_graph(h, n, m, csr || 2 * m < (int64_t{1} << 32));
  const cudaStream_t s = h.stream;
  CK(cudaMemcpyAsync(h.g.edges, edges, m * sizeof(int2), cudaMemcpyDeviceToDevice, s));
  if (csr) {
    CK(cudaMemcpyAsync(h.g.offsets, offsets, (n + 1) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h.g.nbrs, nbrs, 2 * m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h.g.arc_edge, arc_edge, 2 * m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
  } else if (h.g.offsets) {
    build_csr_device(h);
  }
}

}  // namespace rstg
