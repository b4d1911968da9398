// euler.cu -- Euler-tour rooting of the CC spanning forest
// (euler_root_forest, euler_rooting.cpp:180-215), sort-free and CSR-free.
//
// The reference lays out arcs i=(u->v), i+T=(v->u), host-std::sorts them by
// (from, to) to chain each vertex's arcs (euler_rooting.cpp:49-72), and
// derives succ(e) = next(rev e) else first(from(rev e)) (:76-87). Any
// rotation system (any circular order of each vertex's arcs) yields an
// Euler tour of the same tree, and a tree with a fixed root has exactly one
// parent array, so the order is free. Here:
//   * the apply step of the CC appends tree-edge ids to a list (no scan of
//     the m edges or the 2m CSR arcs);
//   * each tree edge claims a slot in both endpoints' arc segments with a
//     warp-aggregated atomicAdd (segment offsets = scan of tree degrees);
//     the thread that placed both arcs writes to/rev/succ for both, so
//     compute_successor and break_cycles (:89-102: the wrap into a root's
//     first arc is cut) cost no search;
//   * ranks come from sparse ruling-set list ranking (listrank.cu);
//   * derive_parents (:155-178): in each arc pair the higher-ranked arc is
//     the return arc, parent[from] = to.
// Roots: the designated root for its label, the smallest vertex of every
// other label (:190-203).
#include "engine.hpp"
#include "scan.cuh"

namespace rstg {

const uint32_t* list_rank_rulers(Handle& h, int64_t E, const uint32_t* succ, int stride,
                                 const uint32_t* heads, int64_t H, uint32_t* sl,
                                 int64_t* R_out, bool verify);

// min_vertex per label (euler_rooting.cpp:190-195); labels are vertex ids.
__global__ void k_min_vertex(int64_t n, const int32_t* __restrict__ lab, uint32_t* minv) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = lab[v];
    if ((uint32_t)v < minv[l]) atomicMin(&minv[l], (uint32_t)v);
  }
}
void launch_min_vertex(Handle& h, const int32_t* lab, uint32_t* minv) {
  k_min_vertex<<<grid_for(h.g.n), kBlock, 0, h.stream>>>(h.g.n, lab, minv);
  CK_LAUNCH();
  h.stats.step(h.g.n);
}
__global__ void k_override_root(const int32_t* lab, uint32_t* minv, int32_t root) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && root >= 0) minv[lab[root]] = (uint32_t)root;
}
__global__ void k_mark_roots(int64_t n, const int32_t* __restrict__ lab,
                             const uint32_t* __restrict__ minv, uint8_t* isroot,
                             int32_t* parent, uint32_t* tdeg, unsigned long long* count) {
  uint32_t c = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool r = minv[lab[v]] == (uint32_t)v;
    isroot[v] = r;
    parent[v] = (int32_t)v;  // derive_parents :167
    tdeg[v] = 0;
    c += r;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

// Tree degrees + each arc's slot inside its tail's segment. Tree edge i is
// tsrc[i] (kNone32 = no edge), or graph edge i when tsrc is null.
__global__ void __launch_bounds__(kBlock)
    k_tree_slots(int64_t N, const uint32_t* __restrict__ tsrc, const int2* __restrict__ edges,
                 uint32_t e_base, uint32_t* tdeg, uint2* __restrict__ lpos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = tsrc ? tsrc[i] : (uint32_t)i;
    if (e == kNone32) continue;
    const int2 uv = edges[e - e_base];
    const uint32_t pu = atomicAdd(&tdeg[uv.x], 1u);
    const uint32_t pv = atomicAdd(&tdeg[uv.y], 1u);
    lpos[i] = make_uint2(pu, pv);
  }
}

// Both arcs of tree edge i: {to, rev} records plus the separate succ array
// the list-ranking walk chases (4-byte entries keep 8 successors per
// sector). compute_successor :83-86 and the break_cycles cut :96-101.
__global__ void __launch_bounds__(kBlock)
    k_tree_arcs(int64_t N, const uint32_t* __restrict__ tsrc, const int2* __restrict__ edges,
                uint32_t e_base, const uint2* __restrict__ lpos, const uint32_t* __restrict__ tf,
                const uint8_t* __restrict__ isroot, uint2* __restrict__ arc,
                uint32_t* __restrict__ succ) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = tsrc ? tsrc[i] : (uint32_t)i;
    if (e == kNone32) continue;
    const int2 uv = edges[e - e_base];
    const uint2 lp = lpos[i];
    const uint32_t u = (uint32_t)uv.x, v = (uint32_t)uv.y;
    const uint32_t fu = tf[u], eu = tf[u + 1], fv = tf[v], ev = tf[v + 1];
    const uint32_t p1 = fu + lp.x;  // u -> v
    const uint32_t p2 = fv + lp.y;  // v -> u
    arc[p1] = make_uint2(v, p2);
    succ[p1] = (p2 + 1 < ev) ? p2 + 1 : (isroot[v] ? kNone32 : fv);
    arc[p2] = make_uint2(u, p1);
    succ[p2] = (p1 + 1 < eu) ? p1 + 1 : (isroot[u] ? kNone32 : fu);
  }
}

namespace {
struct ArrF {
  const uint32_t* a;
  __device__ uint32_t operator()(int64_t i) const { return a[i]; }
};
struct HeadFlag {  // roots with at least one tree arc: their first arc heads a list
  const uint8_t* isroot;
  const uint32_t* tf;
  __device__ uint32_t operator()(int64_t x) const {
    return (isroot[x] && tf[x] < tf[x + 1]) ? 1u : 0u;
  }
};
struct EmitHeadArc {
  const uint32_t* tf;
  uint32_t* heads;
  __device__ void operator()(int64_t x, uint32_t p, uint32_t v) const {
    if (v) heads[p] = tf[x];
  }
};
}  // namespace

// derive_parents (:172-176) on (ruler, offset) ranks; from(p) = to(rev p).
__global__ void __launch_bounds__(kBlock)
    k_orient(int64_t E, const uint2* __restrict__ arc, const uint32_t* __restrict__ sl,
             const uint32_t* __restrict__ rstart, int32_t* __restrict__ parent) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint2 ap = arc[p];
    const uint32_t q = ap.y;
    if ((uint32_t)p > q) continue;
    const uint32_t to_q = arc[q].x;  // = from(p)
    const uint32_t a = sl[p], b = sl[q];  // (ruler << 7) | offset
    const uint32_t rp = rstart[a >> 7] + (a & 127u);
    const uint32_t rq = rstart[b >> 7] + (b & 127u);
    // the higher-ranked arc returns from the child: parent[from] = to
    if (rp > rq)
      parent[to_q] = (int32_t)ap.x;
    else
      parent[ap.x] = (int32_t)to_q;
  }
}

void euler_root(Handle& h, const int32_t* labels, const uint32_t* tsrc, int64_t N, int64_t T,
                int32_t designated_root, int32_t* parent, bool verify) {
  const int64_t n = h.g.n;
  uint32_t* minv = h.ws<uint32_t>(WS_MINV, n);
  uint8_t* isroot = h.ws<uint8_t>(WS_ISROOT, n);
  uint32_t* tdeg = h.ws<uint32_t>(WS_POS, n + 1);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 4;

  h.timer.begin(h.stream, "euler.roots");
  CK(cudaMemsetAsync(minv, 0xFF, n * sizeof(uint32_t), h.stream));
  CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), h.stream));
  k_min_vertex<<<grid_for(n), kBlock, 0, h.stream>>>(n, labels, minv);
  k_override_root<<<1, 32, 0, h.stream>>>(labels, minv, designated_root);
  k_mark_roots<<<grid_for(n), kBlock, 0, h.stream>>>(n, labels, minv, isroot, parent, tdeg, ctr);
  CK_LAUNCH();
  h.stats.step(n, 3);
  h.read_box(reinterpret_cast<int64_t*>(ctr), 1);
  const int64_t comps = h.host_box[0];
  h.stats.components = comps;
  h.timer.end(h.stream);
  if (T != n - comps)  // euler_rooting.cpp:205-208
    throw AlgoError("edge count does not match a spanning forest of the labeling");
  const int64_t E = 2 * T;
  if (E == 0) return;

  h.timer.begin(h.stream, "euler.arcs");
  if (!tsrc) N = T;
  uint2* lpos = h.ws<uint2>(WS_VAL_B, N);
  k_tree_slots<<<grid_for(N), kBlock, 0, h.stream>>>(N, tsrc, h.g.edges, (uint32_t)h.g.e_base,
                                                    tdeg, lpos);
  CK_LAUNCH();
  h.stats.step(N);
  uint32_t* tf = h.ws<uint32_t>(WS_TF, n + 1);
  scan_emit(h, n, ArrF{tdeg}, EmitExcl{tf, n}, false);
  uint2* arc = h.ws<uint2>(WS_ATO, E);
  uint32_t* succ = h.ws<uint32_t>(WS_SUCC, E);
  k_tree_arcs<<<grid_for(N), kBlock, 0, h.stream>>>(N, tsrc, h.g.edges, (uint32_t)h.g.e_base,
                                                   lpos, tf, isroot, arc, succ);
  CK_LAUNCH();
  h.stats.step(N);
  uint32_t* heads = h.ws<uint32_t>(WS_HEADS, n + 1);
  const int64_t H = scan_emit(h, n, HeadFlag{isroot, tf}, EmitHeadArc{tf, heads}, true);
  h.timer.end(h.stream);

  uint32_t* sl = h.ws<uint32_t>(WS_SL, E);
  int64_t R = 0;
  const uint32_t* rstart = list_rank_rulers(h, E, succ, 1, heads, H, sl, &R, verify);
  h.timer.begin(h.stream, "euler.orient");
  k_orient<<<grid_for(E), kBlock, 0, h.stream>>>(E, arc, sl, rstart, parent);
  CK_LAUNCH();
  h.stats.step(E);
  h.timer.end(h.stream);
}

}  // namespace rstg
