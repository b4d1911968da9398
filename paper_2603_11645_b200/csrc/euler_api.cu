// euler_api.cu -- the reference's arc-level Euler-tour API on the device
// (euler_rooting.hpp:18-59): build_euler, compute_successor, break_cycles,
// derive_parents. list_rank is rstg_k_list_rank (capi.cu).
//
// These are the fine-grained entry points the reference's unit and
// acceptance tests call (acceptance.cpp:295-315, test_euler.cpp). The
// production cc-euler pipeline never materialises this structure: it links
// rotation lists while hooking (euler.cu). Here the arrays are the
// reference's own layout -- int64, arc i = tree edge i forward, arc i + T
// backward, rev(e) = (e + E/2) mod E -- so a caller holding an
// EulerStructure gets the same values the reference computes:
//   * build_euler: arcs ordered by (from, to) with one device radix sort
//     (the reference's std::sort, charged as a parallel sort), then each
//     sorted position links to the next arc of the same tail;
//   * compute_successor: succ[e] = next[rev e], else first[from[rev e]];
//   * break_cycles: succ[rev(last[r])] = NONE per root with arcs;
//   * derive_parents: the higher-ranked arc of each pair returns from the
//     child.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <functional>
#include <string>

#include "../../include/rstg.h"
#include "engine.hpp"

namespace rstg {
namespace {

// int64 scratch on the device for the duration of one call.
struct DevI64 {
  long long* p = nullptr;
  explicit DevI64(int64_t count) {
    CK(cudaMalloc(&p, std::max<int64_t>(count, 1) * sizeof(long long)));
  }
  ~DevI64() { cudaFree(p); }
  DevI64(const DevI64&) = delete;
  DevI64& operator=(const DevI64&) = delete;
};

void up(Handle& h, long long* dev, const int64_t* host, int64_t count) {
  if (count > 0)
    CK(cudaMemcpyAsync(dev, host, count * sizeof(long long), cudaMemcpyHostToDevice, h.stream));
}
void down(Handle& h, int64_t* host, const long long* dev, int64_t count) {
  if (count > 0)
    CK(cudaMemcpyAsync(host, dev, count * sizeof(long long), cudaMemcpyDeviceToHost, h.stream));
  CK(cudaStreamSynchronize(h.stream));
}

__global__ void k_arcs(int64_t T, int64_t n, const long long* __restrict__ uv, long long* from,
                       long long* to, unsigned long long* keys, long long* ids, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i < T ? i : i - T;
    const long long u = uv[2 * e], v = uv[2 * e + 1];
    if (u < 0 || u >= n || v < 0 || v >= n) {
      *bad = 1;
      keys[i] = ~0ull;
      ids[i] = i;
      continue;
    }
    const long long f = i < T ? u : v, t = i < T ? v : u;
    from[i] = f;
    to[i] = t;
    keys[i] = ((unsigned long long)f << 32) | (unsigned long long)(uint32_t)t;
    ids[i] = i;
  }
}

__global__ void k_chains(int64_t E, const unsigned long long* __restrict__ skeys,
                         const long long* __restrict__ perm, long long* first, long long* last,
                         long long* next) {
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < E;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const long long e = perm[pos];
    const unsigned long long v = skeys[pos] >> 32;
    if (pos == 0 || (skeys[pos - 1] >> 32) != v) first[v] = e;
    if (pos == E - 1 || (skeys[pos + 1] >> 32) != v) {
      last[v] = e;
      next[e] = -1;
    } else {
      next[e] = perm[pos + 1];
    }
  }
}

__global__ void k_successor(int64_t E, const long long* __restrict__ from,
                            const long long* __restrict__ first, const long long* __restrict__ next,
                            long long* succ) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (e + E / 2) % E;
    const long long nx = next[r];
    succ[e] = nx != -1 ? nx : first[from[r]];
  }
}

__global__ void k_cut(int64_t nroots, int64_t E, const long long* __restrict__ roots,
                      const long long* __restrict__ last, long long* succ) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nroots;
       i += (int64_t)gridDim.x * blockDim.x) {
    const long long l = last[roots[i]];
    if (l != -1) succ[(l + E / 2) % E] = -1;
  }
}

__global__ void k_derive(int64_t n, int64_t T, const long long* __restrict__ from,
                         const long long* __restrict__ to, const long long* __restrict__ rank,
                         long long* parent) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ret = rank[i] > rank[i + T] ? i : i + T;
    parent[from[ret]] = to[ret];
  }
}
__global__ void k_iota(int64_t n, long long* a) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    a[v] = v;
}

}  // namespace
}  // namespace rstg

namespace rstg {
int guard_call(const std::function<void()>& f);  // capi.cu
}
using namespace rstg;

extern "C" {

int rstg_k_build_euler(int64_t n, const int64_t* tree_uv, int64_t T, int64_t* from, int64_t* to,
                       int64_t* first, int64_t* last, int64_t* next) {
  return guard_call([&] {
    if (n < 0 || T < 0) throw ArgError("negative size");
    Handle h(0);
    const int64_t E = 2 * T;
    DevI64 uv(2 * T), f(E), t(E), ids(E), sids(E), fi(n), la(n), nx(E);
    DevI64 keys(E), skeys(E);  // (u64 keys in int64 storage)
    CK(cudaMemsetAsync(fi.p, 0xFF, std::max<int64_t>(n, 1) * 8, h.stream));  // kNone
    CK(cudaMemsetAsync(la.p, 0xFF, std::max<int64_t>(n, 1) * 8, h.stream));
    if (E > 0) {
      up(h, uv.p, tree_uv, 2 * T);
      int* bad = reinterpret_cast<int*>(h.dev_box + 50);
      CK(cudaMemsetAsync(bad, 0, sizeof(int), h.stream));
      auto* k = reinterpret_cast<unsigned long long*>(keys.p);
      auto* sk = reinterpret_cast<unsigned long long*>(skeys.p);
      k_arcs<<<grid_for(E), kBlock, 0, h.stream>>>(T, n, uv.p, f.p, t.p, k, ids.p, bad);
      CK_LAUNCH();
      h.read_box(reinterpret_cast<int64_t*>(bad), 1);
      if (*reinterpret_cast<int*>(h.host_box)) throw AlgoError("tree edge endpoint out of range");
      size_t temp = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, k, sk, ids.p, sids.p, E, 0, 64, h.stream));
      void* tmp = h.ws(WS_SL, temp);
      CK(cub::DeviceRadixSort::SortPairs(tmp, temp, k, sk, ids.p, sids.p, E, 0, 64, h.stream));
      k_chains<<<grid_for(E), kBlock, 0, h.stream>>>(E, sk, sids.p, fi.p, la.p, nx.p);
      CK_LAUNCH();
    }
    down(h, from, f.p, E);
    down(h, to, t.p, E);
    down(h, first, fi.p, n);
    down(h, last, la.p, n);
    down(h, next, nx.p, E);
  });
}

int rstg_k_compute_successor(int64_t n, int64_t E, const int64_t* from, const int64_t* first,
                             const int64_t* next, int64_t* succ) {
  return guard_call([&] {
    if (E <= 0) return;
    Handle h(0);
    DevI64 f(E), fi(n), nx(E), s(E);
    up(h, f.p, from, E);
    up(h, fi.p, first, n);
    up(h, nx.p, next, E);
    k_successor<<<grid_for(E), kBlock, 0, h.stream>>>(E, f.p, fi.p, nx.p, s.p);
    CK_LAUNCH();
    down(h, succ, s.p, E);
  });
}

int rstg_k_break_cycles(int64_t n, int64_t E, const int64_t* last, const int64_t* roots,
                        int64_t nroots, int64_t* succ) {
  return guard_call([&] {
    if (E <= 0 || nroots <= 0) return;
    Handle h(0);
    DevI64 la(n), r(nroots), s(E);
    up(h, la.p, last, n);
    up(h, r.p, roots, nroots);
    up(h, s.p, succ, E);
    k_cut<<<grid_for(nroots), kBlock, 0, h.stream>>>(nroots, E, r.p, la.p, s.p);
    CK_LAUNCH();
    down(h, succ, s.p, E);
  });
}

int rstg_k_derive_parents(int64_t n, int64_t E, const int64_t* from, const int64_t* to,
                          const int64_t* rank, int64_t* parent) {
  return guard_call([&] {
    if (n <= 0) return;
    Handle h(0);
    const int64_t T = E / 2;
    DevI64 f(E), t(E), rk(E), p(n);
    up(h, f.p, from, E);
    up(h, t.p, to, E);
    up(h, rk.p, rank, E);
    k_iota<<<grid_for(n), kBlock, 0, h.stream>>>(n, p.p);
    if (T > 0) k_derive<<<grid_for(T), kBlock, 0, h.stream>>>(n, T, f.p, t.p, rk.p, p.p);
    CK_LAUNCH();
    down(h, parent, p.p, n);
  });
}

}  // extern "C"
