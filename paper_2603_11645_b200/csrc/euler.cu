// euler.cu -- Euler-tour rooting of the CC spanning forest
// (euler_root_forest, euler_rooting.cpp:180-215), sort-free.
//
// The reference builds arcs i=(u->v), i+T=(v->u) per tree edge and host
// std::sorts them by (from, to) (euler_rooting.cpp:49-56). Here the CSR is
// already (from, to)-sorted (build_csr keeps neighbour lists ascending,
// graph.cpp:159-171), so the tree adjacency is a stream compaction of the
// CSR arcs whose edge is flagged: position = exclusive scan of the flags.
//   succ(x->y) = next arc after (y->x) in y's list, wrapping to y's first
//                (compute_successor :76-87); the wrap is cut when y is a root
//                (break_cycles :89-102: succ[rev(last[r])] = none).
//   rev(x->y)  = binary search of x in y's sorted tree list.
//   ranks      = sparse ruling-set list ranking (listrank.cu).
//   parent     = for each arc pair the higher-ranked arc is the return arc
//                (derive_parents :155-178).
// Roots are the designated root for its label and the smallest vertex of
// every other label (:190-203). The result is unique given the tree-edge
// set and the root set, so it equals the reference bit-for-bit.
#include "engine.hpp"
#include "scan.cuh"

namespace rstg {

const uint32_t* list_rank_rulers(Handle& h, int64_t E, const uint32_t* succ,
                                 const uint32_t* heads, int64_t H, unsigned long long* sl,
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
                             int32_t* parent, unsigned long long* count) {
  uint32_t c = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool r = minv[lab[v]] == (uint32_t)v;
    isroot[v] = r;
    parent[v] = (int32_t)v;  // derive_parents :167
    c += r;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

namespace {
struct TreeArcFlag {
  const uint32_t* arc_edge;
  const uint8_t* tflag;
  __device__ uint32_t operator()(int64_t j) const { return tflag[arc_edge[j]]; }
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

__global__ void k_tree_offsets(int64_t n, const uint32_t* __restrict__ offsets,
                               const uint32_t* __restrict__ pos, uint32_t* tf) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n;
       x += (int64_t)gridDim.x * blockDim.x)
    tf[x] = pos[offsets[x]];
}

__global__ void __launch_bounds__(kBlock)
    k_fill_arcs(int64_t A, const uint32_t* __restrict__ arc_edge, const int32_t* __restrict__ nbrs,
                const int2* __restrict__ edges, const uint8_t* __restrict__ tflag,
                const uint32_t* __restrict__ pos, uint32_t* __restrict__ ato,
                uint32_t* __restrict__ afrom) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < A;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = arc_edge[j];
    if (!tflag[e]) continue;
    const uint32_t p = pos[j];
    const int32_t y = nbrs[j];
    const int2 uv = edges[e];
    ato[p] = (uint32_t)y;
    afrom[p] = (uint32_t)(uv.x ^ uv.y ^ y);  // the other endpoint
  }
}

// succ + rev + cut (compute_successor :83-86, break_cycles :96-101).
__global__ void __launch_bounds__(kBlock)
    k_successor(int64_t E, const uint32_t* __restrict__ ato, const uint32_t* __restrict__ afrom,
                const uint32_t* __restrict__ tf, const uint8_t* __restrict__ isroot,
                uint32_t* __restrict__ succ, uint32_t* __restrict__ rev) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = afrom[p], y = ato[p];
    uint32_t lo = tf[y], hi = tf[y + 1];
    const uint32_t end = hi;
    while (lo < hi) {  // lower_bound of x in y's ascending tree list
      uint32_t mid = (lo + hi) >> 1;
      if (ato[mid] < x)
        lo = mid + 1;
      else
        hi = mid;
    }
    rev[p] = lo;
    succ[p] = (lo + 1 < end) ? lo + 1 : (isroot[y] ? kNone32 : tf[y]);
  }
}

// derive_parents (:172-176) on (ruler, offset) ranks.
__global__ void __launch_bounds__(kBlock)
    k_orient(int64_t E, const uint32_t* __restrict__ rev, const unsigned long long* __restrict__ sl,
             const uint32_t* __restrict__ rstart, const uint32_t* __restrict__ ato,
             const uint32_t* __restrict__ afrom, int32_t* __restrict__ parent) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t q = rev[p];
    if ((uint32_t)p > q) continue;
    const unsigned long long a = sl[p], b = sl[q];
    const uint32_t rp = rstart[a >> 32] + (uint32_t)a;
    const uint32_t rq = rstart[b >> 32] + (uint32_t)b;
    const uint32_t ret = rp > rq ? (uint32_t)p : q;
    parent[afrom[ret]] = (int32_t)ato[ret];
  }
}

// Full ranks per arc (for the rank-level parity tests only).
__global__ void k_ranks(int64_t E, const unsigned long long* sl, const uint32_t* rstart,
                        uint32_t* rank) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E;
       p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long a = sl[p];
    rank[p] = rstart[a >> 32] + (uint32_t)a;
  }
}

// Shared tail once succ is known: rank lists from `heads`, orient.
static void rank_and_orient(Handle& h, int64_t E, const uint32_t* succ, const uint32_t* rev,
                            const uint32_t* ato, const uint32_t* afrom, const uint32_t* heads,
                            int64_t H, int32_t* parent, uint32_t* ranks_out, bool verify) {
  unsigned long long* sl = h.ws<unsigned long long>(WS_SL, E);
  int64_t R = 0;
  const uint32_t* rstart = list_rank_rulers(h, E, succ, heads, H, sl, &R, verify);
  h.timer.begin(h.stream, "euler.orient");
  k_orient<<<grid_for(E), kBlock, 0, h.stream>>>(E, rev, sl, rstart, ato, afrom, parent);
  CK_LAUNCH();
  h.stats.step(E);
  if (ranks_out) {
    k_ranks<<<grid_for(E), kBlock, 0, h.stream>>>(E, sl, rstart, ranks_out);
    CK_LAUNCH();
  }
  h.timer.end(h.stream);
}

void euler_root(Handle& h, const int32_t* labels, const uint8_t* tflag, int64_t T,
                int32_t designated_root, int32_t* parent, bool verify) {
  const int64_t n = h.g.n, m = h.g.m, A = 2 * m;
  if (!h.g.has_csr()) throw ArgError("euler rooting needs the graph's CSR");
  uint32_t* minv = h.ws<uint32_t>(WS_MINV, n);
  uint8_t* isroot = h.ws<uint8_t>(WS_ISROOT, n);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 4;

  h.timer.begin(h.stream, "euler.roots");
  CK(cudaMemsetAsync(minv, 0xFF, n * sizeof(uint32_t), h.stream));
  CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), h.stream));
  k_min_vertex<<<grid_for(n), kBlock, 0, h.stream>>>(n, labels, minv);
  k_override_root<<<1, 32, 0, h.stream>>>(labels, minv, designated_root);
  k_mark_roots<<<grid_for(n), kBlock, 0, h.stream>>>(n, labels, minv, isroot, parent, ctr);
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
  uint32_t* pos = h.ws<uint32_t>(WS_POS, A + 1);
  const uint32_t got = scan_emit(h, A, TreeArcFlag{h.g.arc_edge, tflag}, EmitExcl{pos, A}, true);
  if ((int64_t)got != E) throw AlgoError("tree flags inconsistent with tree edge count");
  uint32_t* tf = h.ws<uint32_t>(WS_TF, n + 1);
  uint32_t* ato = h.ws<uint32_t>(WS_ATO, E);
  uint32_t* afrom = h.ws<uint32_t>(WS_AFROM, E);
  k_tree_offsets<<<grid_for(n + 1), kBlock, 0, h.stream>>>(n, h.g.offsets, pos, tf);
  k_fill_arcs<<<grid_for(A), kBlock, 0, h.stream>>>(A, h.g.arc_edge, h.g.nbrs, h.g.edges, tflag,
                                                    pos, ato, afrom);
  CK_LAUNCH();
  h.stats.step(n, 1);
  h.stats.step(A, 1);
  h.timer.end(h.stream);

  h.timer.begin(h.stream, "euler.succ");
  uint32_t* succ = h.ws<uint32_t>(WS_SUCC, E);
  uint32_t* rev = h.ws<uint32_t>(WS_REV, E);
  k_successor<<<grid_for(E), kBlock, 0, h.stream>>>(E, ato, afrom, tf, isroot, succ, rev);
  CK_LAUNCH();
  h.stats.step(E);
  uint32_t* heads = h.ws<uint32_t>(WS_HEADS, n + 1);
  const int64_t H = scan_emit(h, n, HeadFlag{isroot, tf}, EmitHeadArc{tf, heads}, true);
  h.timer.end(h.stream);

  rank_and_orient(h, E, succ, rev, ato, afrom, heads, H, parent, nullptr, verify);
}

}  // namespace rstg
