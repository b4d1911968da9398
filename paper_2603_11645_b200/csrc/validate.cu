// validate.cu -- device validity check of a rooted spanning forest, the
// semantics of validate_rooted_forest (validate.cpp:108-211) without the
// host-side O(n+m) oracle:
//   1 parent out of range            (validate.cpp:122-126)
//   2 parent edge not a graph edge   (:137-145; binary search, graph.cpp:29-33)
//   3 parent chain cycle             (:148-172; doubling with a round cap)
//   4 a component with != 1 root     (:174-191)
//   5 chain reaches another component(:192-199)
//   6 required root is not a root    (:201-209)
// Component labels come from the device CC. Used for configurations whose
// host oracle does not fit (Kron-28) and as the GPU-side "valid" column.
#include "engine.hpp"

namespace rstg {

enum : int { V_RANGE = 1, V_EDGE, V_CYCLE, V_ROOTS, V_COMP, V_REQUIRED };

__global__ void k_val_edges(int64_t n, const int32_t* __restrict__ parent,
                            const uint32_t* __restrict__ off, const int32_t* __restrict__ nbrs,
                            int32_t* root0, unsigned long long* bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = parent[v];
    root0[v] = p;
    if (p < 0 || p >= n) {
      atomicMin(bad, ((unsigned long long)V_RANGE << 40) | (unsigned long long)v);
      root0[v] = (int32_t)v;
      continue;
    }
    if (p == (int32_t)v) continue;
    uint32_t lo = off[v], hi = off[v + 1];
    const uint32_t end = hi;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (nbrs[mid] < p)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo >= end || nbrs[lo] != p)
      atomicMin(bad, ((unsigned long long)V_EDGE << 40) | (unsigned long long)v);
  }
}

// One doubling round: b[v] = a[a[v]].
__global__ void k_val_double(int64_t n, const int32_t* __restrict__ a, int32_t* __restrict__ b) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    b[v] = a[a[v]];
}
// After enough doubling every acyclic chain ends on a true root; a vertex
// whose resolved ancestor is not self-parented sits on (or above) a cycle.
// (Fixed points of the doubled map alone are not enough: an even cycle
// collapses into them, cf. cc_forest.hpp:33-39.)
__global__ void k_val_cycle(int64_t n, const int32_t* __restrict__ root,
                            const int32_t* __restrict__ parent, unsigned long long* bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = root[v];
    if (parent[x] != x) atomicMin(bad, ((unsigned long long)V_CYCLE << 40) | (unsigned long long)v);
  }
}

__global__ void k_val_count_roots(int64_t n, const int32_t* parent, const int32_t* lab,
                                  uint32_t* cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    if (parent[v] == (int32_t)v) atomicAdd(&cnt[lab[v]], 1u);
}

__global__ void k_val_comp(int64_t n, const int32_t* root, const int32_t* lab,
                           const uint32_t* cnt, unsigned long long* bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (cnt[lab[v]] != 1u)
      atomicMin(bad, ((unsigned long long)V_ROOTS << 40) | (unsigned long long)v);
    if (lab[root[v]] != lab[v])
      atomicMin(bad, ((unsigned long long)V_COMP << 40) | (unsigned long long)v);
  }
}

static int ceil_log2_i(int64_t x) {
  int k = 0;
  int64_t p = 1;
  while (p < x) {
    p <<= 1;
    ++k;
  }
  return k;
}

int validate_forest(Handle& h, const int32_t* parent, int32_t required_root,
                    int64_t* bad_vertex) {
  const int64_t n = h.g.n;
  ensure_csr(h);
  if (!h.g.has_csr()) throw ArgError("validation needs the graph's CSR");
  const cudaStream_t s = h.stream;
  int32_t* ra = h.ws<int32_t>(WS_VAL_B, n);
  int32_t* rb = h.ws<int32_t>(WS_VAL_C, n);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(h.dev_box) + 40;
  CK(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s));
  const unsigned g = grid_for(n);
  k_val_edges<<<g, kBlock, 0, s>>>(n, parent, h.g.offsets, h.g.nbrs, ra, bad);
  CK_LAUNCH();
  // Doubling: after ceil(log2 n)+1 rounds every acyclic chain is resolved.
  const int rounds = ceil_log2_i(n < 2 ? 2 : n) + 1;
  for (int r = 0; r < rounds; ++r) {
    k_val_double<<<g, kBlock, 0, s>>>(n, ra, rb);
    CK_LAUNCH();
    std::swap(ra, rb);
  }
  k_val_cycle<<<g, kBlock, 0, s>>>(n, ra, parent, bad);
  CK_LAUNCH();
  h.read_box(reinterpret_cast<int64_t*>(bad), 1);
  unsigned long long b = (unsigned long long)h.host_box[0];
  if (b != kAllOnes) {
    *bad_vertex = (int64_t)(b & 0xffffffffffull);
    return (int)(b >> 40);
  }
  // Components: labels from the device CC, one root per label.
  int32_t* lab = h.ws<int32_t>(WS_VAL_A, n);
  cc_labels_fast(h, lab);
  uint32_t* cnt = h.ws<uint32_t>(WS_MINV, n);
  h.minv_clean = nullptr;  // (WS_MINV reused here)
  CK(cudaMemsetAsync(cnt, 0, n * sizeof(uint32_t), s));
  k_val_count_roots<<<g, kBlock, 0, s>>>(n, parent, lab, cnt);
  k_val_comp<<<g, kBlock, 0, s>>>(n, ra, lab, cnt, bad);
  CK_LAUNCH();
  h.read_box(reinterpret_cast<int64_t*>(bad), 1);
  b = (unsigned long long)h.host_box[0];
  if (b != kAllOnes) {
    *bad_vertex = (int64_t)(b & 0xffffffffffull);
    return (int)(b >> 40);
  }
  if (required_root >= 0) {
    int32_t pr = 0;
    CK(cudaMemcpyAsync(h.host_box, parent + required_root, sizeof(int32_t),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    pr = *reinterpret_cast<int32_t*>(h.host_box);
    if (pr != required_root) {
      *bad_vertex = required_root;
      return V_REQUIRED;
    }
  }
  *bad_vertex = -1;
  return 0;
}

}  // namespace rstg

namespace rstg {

// ---- forest_depth (rooted_forest.cpp:12-95) on the device ----------------
// Distance to the root by Jacobi doubling over (jump, distance) pairs: a
// round doubles every jump, so ceil(log2 depth) + 1 rounds settle all; a
// pointer still short of a root after ceil(log2 n) + 2 rounds is on a
// cycle. Per-root maxima by atomicMax on the root's slot.
__global__ void k_depth_init(int64_t n, const int32_t* __restrict__ parent, int2* jd) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = parent[v];
    jd[v] = make_int2(p, p == (int32_t)v ? 0 : 1);
  }
}
__global__ void k_depth_round(int64_t n, const int2* __restrict__ a, int2* __restrict__ b,
                              int* flags, int round) {
  if (round > 0 && flags[round - 1] == 0) return;
  bool changed = false;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int2 x = a[v];
    const int2 y = a[x.x];
    b[v] = make_int2(y.x, x.y + y.y);
    changed |= y.x != x.x;
  }
  block_flag(changed, &flags[round]);
}
__global__ void k_depth_finish(int64_t n, const int2* __restrict__ jd, const int32_t* __restrict__ parent,
                               int32_t* depth, unsigned int* rootmax, int* cycle_at) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int2 x = jd[v];
    if (parent[x.x] != x.x) {  // never reached a root: a cycle
      atomicMin(cycle_at, (int)v);
      continue;
    }
    depth[v] = x.y;
    atomicMax(&rootmax[x.x], (unsigned int)x.y);
  }
}

// Per-root maxima in the reference's layout (rooted_forest.cpp: -1 for a
// non-root) and the deepest tree's depth.
__global__ void k_root_depths(int64_t n, const int32_t* __restrict__ parent, uint32_t* rootmax,
                              unsigned int* best) {
  unsigned int b = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (parent[v] == (int32_t)v)
      b = max(b, rootmax[v]);
    else
      rootmax[v] = 0xFFFFFFFFu;  // (int32 -1 when widened)
  }
  b = __reduce_max_sync(0xffffffffu, b);
  if ((threadIdx.x & 31) == 0 && b) atomicMax(best, b);
}
int64_t root_depths(Handle& h, const int32_t* parent, uint32_t* rootmax, int64_t n) {
  unsigned int* best = reinterpret_cast<unsigned int*>(h.dev_box + 42);
  CK(cudaMemsetAsync(h.dev_box + 42, 0, sizeof(int64_t), h.stream));
  if (n > 0) k_root_depths<<<grid_for(n), kBlock, 0, h.stream>>>(n, parent, rootmax, best);
  CK_LAUNCH();
  h.read_box(h.dev_box + 42, 1);
  return (int64_t)*reinterpret_cast<unsigned int*>(h.host_box);
}

int64_t forest_depth_device(Handle& h, const int32_t* parent, int32_t* depth, uint32_t* rootmax,
                            int64_t* cycle_vertex) {
  const int64_t n = h.g.n;
  const cudaStream_t s = h.stream;
  int2* a = h.ws<int2>(WS_VAL_A, n);
  int2* b = h.ws<int2>(WS_VAL_B, n);
  int* flags = reinterpret_cast<int*>(h.dev_box + 128);  // 64 ints
  int* cyc = reinterpret_cast<int*>(h.dev_box + 41);
  CK(cudaMemsetAsync(flags, 0, 64 * sizeof(int), s));
  CK(cudaMemsetAsync(rootmax, 0, n * sizeof(uint32_t), s));
  CK(cudaMemsetAsync(cyc, 0x7F, sizeof(int), s));
  const unsigned g = grid_for(n);
  k_depth_init<<<g, kBlock, 0, s>>>(n, parent, a);
  int rounds = 2;
  while ((int64_t{1} << (rounds - 2)) < n) ++rounds;
  for (int r = 0; r < rounds && r < 64; ++r) {
    k_depth_round<<<g, kBlock, 0, s>>>(n, a, b, flags, r);
    std::swap(a, b);  // (a round that changed nothing leaves b unwritten: both equal)
  }
  k_depth_finish<<<g, kBlock, 0, s>>>(n, a, parent, depth, rootmax, cyc);
  CK_LAUNCH();
  h.read_box(reinterpret_cast<int64_t*>(cyc), 1);
  const int c = *reinterpret_cast<int*>(h.host_box);
  *cycle_vertex = c == 0x7F7F7F7F ? -1 : c;
  return rounds;
}

}  // namespace rstg
