// euler.cu -- Euler-tour rooting of a spanning forest (euler_root_forest,
// euler_rooting.cpp:180-215), sort-free, scan-free and CSR-free.
//
// The reference lays out arcs i=(u->v), i+T=(v->u), host-std::sorts them by
// (from, to) to chain each vertex's arcs (euler_rooting.cpp:49-72), and
// derives succ(e) = next(rev e) else first(from(rev e)) (:76-87). Any
// rotation system (any circular order of each vertex's arcs) yields an
// Euler tour of the same tree, and a tree with a fixed root has exactly one
// parent array, so the order is free. Here:
//   * the CC apply step links every new tree edge into the rotation lists
//     of its endpoints (link_tree_edge, engine.hpp): arcs i and N + i per
//     slot, so rev(p) = p +- N and successors are written at link time;
//   * one vertex pass (k_euler_fix) picks the roots -- the designated root
//     for its label, the smallest vertex of every other label (:190-203) --,
//     closes each non-root list into a cycle (the wrap of compute_successor)
//     and leaves the roots' lists open (break_cycles, :96-101), and
//     registers the list-ranking rulers (hash-selected arcs, the tours'
//     first arcs) with warp-aggregated id claims;
//   * ranks come from sparse ruling-set list ranking (listrank.cu);
//   * derive_parents (:155-178): in each arc pair the higher-ranked arc is
//     the return arc, parent[from] = to.
#include <algorithm>
#include <cstdlib>

#include "engine.hpp"
#include "listrank.cuh"

namespace rstg {

// min_vertex per label (euler_rooting.cpp:190-195) on its own (the BFS
// seeds use it); labels are vertex ids, lanes sharing one issue one atomic.
__global__ void __launch_bounds__(kBlock)
    k_min_vertex(int64_t n, const int32_t* __restrict__ lab, uint32_t* minv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < n; b += stride) {
    const int64_t v = b + threadIdx.x;
    const int32_t l = v < n ? lab[v] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    if (v < n && (threadIdx.x & 31) == __ffs(peers) - 1 && (uint32_t)v < minv[l])
      atomicMin(&minv[l], (uint32_t)v);
  }
}
void launch_min_vertex(Handle& h, const int32_t* lab, uint32_t* minv) {
  k_min_vertex<<<grid_for(h.g.n), kBlock, 0, h.stream>>>(h.g.n, lab, minv);
  CK_LAUNCH();
  h.stats.step(h.g.n);
}

__global__ void k_override_root(const int32_t* lab, uint32_t* minv, int32_t root, bool cc_slots) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && root >= 0)
    minv[cc_slots ? find_root_ro(lab, root) : lab[root]] = (uint32_t)root;  // (lazy CC labels)
}

// Labels present (explicit forests: caller labels need not be rep roots).
__global__ void k_mark_labels(int64_t n, const int32_t* __restrict__ lab, uint8_t* present) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    present[lab[v]] = 1;
}

__global__ void k_count_present(int64_t n, const uint8_t* __restrict__ present,
                                unsigned long long* count) {
  unsigned c = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    c += present[v];
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}
int64_t count_labels(Handle& h, const int32_t* labels, int64_t n) {
  if (n == 0) return 0;
  uint8_t* present = h.ws<uint8_t>(WS_ISROOT, n);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(h.dev_box) + 4;
  CK(cudaMemsetAsync(present, 0, (size_t)n, h.stream));
  CK(cudaMemsetAsync(cnt, 0, sizeof(*cnt), h.stream));
  k_mark_labels<<<grid_for(n), kBlock, 0, h.stream>>>(n, labels, present);
  k_count_present<<<grid_for(n), kBlock, 0, h.stream>>>(n, present, cnt);
  CK_LAUNCH();
  h.read_box(reinterpret_cast<int64_t*>(cnt), 1);
  return h.host_box[0];
}

// Vertex pass, in tiles of kFixItems x kBlock vertices claimed in order:
//   * min_vertex per label (euler_rooting.cpp:190-195): lanes sharing a
//     label (one giant component: all of them) issue one atomicMin;
//   * the label list (one entry per component) for the root pass;
//   * rotation cycles: round 0 closed every local list already; a vertex
//     with a remote list gets local + remote spliced into one cycle;
//   * the list-ranking rulers among its slot's arcs (cc_slots: slot v holds
//     a tree edge iff lab[v] != v), one id claim per tile, so ruler ids
//     follow positions.
// Most vertices touch two coalesced words here (label, remote head).
constexpr int kFixItems = 8;
__global__ void __launch_bounds__(kBlock)
    k_euler_fix(int64_t n, const int32_t* lab, const uint8_t* __restrict__ present,
                uint32_t* minv, EulerIO io, bool cc_slots, uint32_t* labels_out,
                unsigned long long* nlabels, uint32_t* rpos, uint32_t* sl, unsigned long long* ctr,
                unsigned long long* tiles, int logk, int ob, uint32_t cap, bool rulers,
                bool mark_empty) {
  constexpr int64_t kTile = (int64_t)kFixItems * kBlock;
  __shared__ unsigned long long s_tile;
  __shared__ uint32_t s_nl;
  __shared__ unsigned long long s_lb;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_tile = atomicAdd(tiles, 1ull);
      s_nl = 0;
    }
    __syncthreads();
    const int64_t base = (int64_t)s_tile * kTile;
    if (base >= n) break;
    uint32_t flags = 0;  // 2 bits per item: arc v, arc N + v; bit 16+k: label
    uint32_t h2[kFixItems];
    // CC labels may be lazy (cc_exact with Euler): resolved here without a
    // compression write-back (every later pass only tests lab[v] == v).
    // The loads of all items go out together, level by level -- labels,
    // their labels, then the rare deeper walks -- as do the remote heads:
    // one item's chain at a time left this pass latency-bound.
    int32_t lb[kFixItems];
#pragma unroll
    for (int k = 0; k < kFixItems; ++k) {
      const int64_t v = base + k * kBlock + threadIdx.x;
      lb[k] = v < n ? __ldcs(&lab[v]) : -1;
      h2[k] = v < n ? __ldcs(&io.rhead[v]) : kNone32;
    }
    if (cc_slots) {
      int32_t l2[kFixItems];
#pragma unroll
      for (int k = 0; k < kFixItems; ++k) l2[k] = lb[k] >= 0 ? lab[lb[k]] : -1;
#pragma unroll
      for (int k = 0; k < kFixItems; ++k)
        if (l2[k] != lb[k]) lb[k] = find_root_ro(lab, l2[k]);
    }
#pragma unroll
    for (int k = 0; k < kFixItems; ++k) {
      const int64_t v = base + k * kBlock + threadIdx.x;
      const int32_t l = lb[k];
      const unsigned peers = __match_any_sync(0xffffffffu, l);
      if (v >= n) continue;
      if ((threadIdx.x & 31) == __ffs(peers) - 1 && (uint32_t)v < minv[l])
        atomicMin(&minv[l], (uint32_t)v);  // the group's lowest lane has its smallest vertex
      if (present ? present[v] != 0 : l == (int32_t)v) flags |= 1u << (16 + k);
      if (mark_empty && l == (int32_t)v) {  // (cc slots: a root's slot holds no tree edge)
        io.S[v] = kEmptySlot;
        io.S[io.nslots + v] = kEmptySlot;
      }
      if (rulers && cc_slots && l != (int32_t)v) {
        if (lr_hash_ruler((uint32_t)v, logk)) flags |= 1u << (2 * k);
        if (lr_hash_ruler(io.nslots + (uint32_t)v, logk)) flags |= 2u << (2 * k);
      }
    }
    // Splices, their loads batched across the items (independent lists):
    // local tail -> remote head and remote tail -> local head, or the remote
    // list closed into a cycle of its own when there is no local list.
    // (the splice loads of all items first: lists of distinct vertices)
    uint32_t h1[kFixItems], t1[kFixItems], t2[kFixItems];
#pragma unroll
    for (int k = 0; k < kFixItems; ++k) {
      const int64_t v = base + k * kBlock + threadIdx.x;
      const bool sp = h2[k] != kNone32;
      h1[k] = sp ? io.vhead[v] : kNone32;
      t1[k] = sp ? io.vtail[v] : kNone32;
      t2[k] = sp ? io.rtail[v] : kNone32;
    }
#pragma unroll
    for (int k = 0; k < kFixItems; ++k) {
      if (h2[k] == kNone32) continue;
      const int64_t v = base + k * kBlock + threadIdx.x;
      if (h1[k] != kNone32) {  // local tail -> remote head, remote tail -> local head
        io.S[arc_rev(t1[k], io.nslots)] = h2[k];
        io.S[arc_rev(t2[k], io.nslots)] = h1[k];
      } else {
        io.S[arc_rev(t2[k], io.nslots)] = h2[k];
        io.vhead[v] = h2[k];
      }
      // the spliced cycle is (vhead .. t2): the root pass reads only
      // vhead/vtail, and the remote list is left empty for the next build
      io.vtail[v] = t2[k];
      io.rhead[v] = kNone32;
    }
    uint32_t id = rulers ? lr_block_claim(__popc(flags & 0xFFFFu), ctr) : 0u;
    const uint32_t nl = __popc(flags >> 16);
    uint32_t li = nl ? atomicAdd(&s_nl, nl) : 0u;
    __syncthreads();
    if (threadIdx.x == 0 && s_nl) s_lb = atomicAdd(nlabels, (unsigned long long)s_nl);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kFixItems; ++k) {
      const uint32_t v = (uint32_t)(base + k * kBlock + threadIdx.x);
      if (flags & (1u << (2 * k))) lr_put(id++, v, rpos, sl, ob, cap);
      if (flags & (2u << (2 * k))) lr_put(id++, io.nslots + v, rpos, sl, ob, cap);
      if (flags & (1u << (16 + k))) labels_out[s_lb + li++] = v;
    }
  }
}

constexpr int64_t kResetMax = 1 << 16;

// The min table between builds: all-ones, or flagged dirty by the root pass
// (many components: it skipped the reset) and filled here.
__global__ void k_fill_if_dirty(uint32_t* __restrict__ minv, int64_t n, const int* dirty,
                                unsigned long long* box) {
  // (and the pass's counters: dev_box [4] labels, [8] ruler ids, [13] tiles)
  if (blockIdx.x == 0 && threadIdx.x < 3) box[threadIdx.x == 0 ? 4 : threadIdx.x == 1 ? 8 : 13] = 0;
  if (!*dirty) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    minv[i] = kNone32;
}

// Root pass over the labels: the root of label x is minv[x] (the designated
// root already stored for its label): parent[r] = r (derive_parents :167),
// its rotation cycle opened just before its first arc (break_cycles
// :96-101) and that first arc registered as the head ruler of its tour.
__global__ void __launch_bounds__(kBlock)
    k_euler_roots(uint32_t* __restrict__ labels, const unsigned long long* nlabels,
                  uint32_t* __restrict__ minv, EulerIO io, int32_t* parent, uint32_t* rpos,
                  uint32_t* sl, unsigned long long* ctr, int logk, int ob, uint32_t cap,
                  bool rulers, int* minv_dirty, bool keep_roots) {
  const int64_t L = (int64_t)*nlabels;
  // few labels: reset their min entries here; many: leave them, flagged
  // for the fill before the next build (cheaper than a scattered reset)
  const bool reset = L <= kResetMax;
  if (blockIdx.x == 0 && threadIdx.x == 0) *minv_dirty = reset ? 0 : 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < L; b += stride) {
    const int64_t i = b + threadIdx.x;
    uint32_t hd = kNone32;
    if (i < L) {
      const uint32_t r = minv[labels[i]];
      if (reset) minv[labels[i]] = kNone32;
      parent[r] = (int32_t)r;
      if (keep_roots) labels[i] = r;  // (the roots, for a deferred re-orientation)
      hd = io.vhead[r];  // the combined cycle (k_euler_fix spliced the remote list)
      if (hd != kNone32)
        io.S[arc_rev(io.vtail[r], io.nslots)] = kNone32;  // the tour ends back at the root
    }
    if (!rulers) continue;  // (block-uniform)
    const bool head = hd != kNone32 && !lr_hash_ruler(hd, logk);
    const uint32_t id = lr_block_claim(head ? 1u : 0u, ctr);
    if (head) lr_put(id, hd, rpos, sl, ob, cap);
  }
}

// parent[r] = r again for the roots k_euler_roots kept in the label list.
__global__ void k_reset_roots(const uint32_t* __restrict__ roots, const unsigned long long* count,
                              int32_t* parent) {
  const int64_t L = (int64_t)*count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L;
       i += (int64_t)gridDim.x * blockDim.x)
    parent[roots[i]] = (int32_t)roots[i];
}

// Hash-selected rulers of explicit slots [0, T) (all occupied).
__global__ void __launch_bounds__(kBlock)
    k_register_slots(int64_t T, uint32_t nslots, uint32_t* rpos, uint32_t* sl,
                     unsigned long long* ctr, int logk, int ob, uint32_t cap) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < T; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b + threadIdx.x;
    const bool a0 = i < T && lr_hash_ruler((uint32_t)i, logk);
    const bool a1 = i < T && lr_hash_ruler(nslots + (uint32_t)i, logk);
    uint32_t id = lr_block_claim((uint32_t)a0 + (uint32_t)a1, ctr);
    if (a0) lr_put(id++, (uint32_t)i, rpos, sl, ob, cap);
    if (a1) lr_put(id++, nslots + (uint32_t)i, rpos, sl, ob, cap);
  }
}

__global__ void k_link_edges(int64_t T, const int2* __restrict__ edges, EulerIO io) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 e = edges[i];
    link_tree_edge(io, (uint32_t)i, (uint32_t)e.x, (uint32_t)e.y, (uint32_t)i);
  }
}

// derive_parents (:172-176) on (ruler, offset) ranks, one thread per slot.
__global__ void __launch_bounds__(kBlock)
    k_orient(int64_t N, const int32_t* __restrict__ lab, bool cc_slots,
             const uint32_t* __restrict__ eto, const int2* __restrict__ edges,
             const uint32_t* __restrict__ sl,  // the rank words
             const uint32_t* __restrict__ rstart, int ob, int32_t* __restrict__ parent) {
  const uint32_t mask = (1u << ob) - 1u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (cc_slots && lab[i] == (int32_t)i) continue;  // no tree edge in this slot
    const uint2 t = eto_ends(eto[i], (uint32_t)i, edges);  // (b, a): arc i = a -> b, N + i = b -> a
    const uint32_t wp = sl[i], wq = sl[N + i];
    const uint32_t rp = rstart[wp >> ob] + (wp & mask);
    const uint32_t rq = rstart[wq >> ob] + (wq & mask);
    // the higher-ranked arc returns from the child: parent[from] = to
    if (rp > rq)
      parent[t.y] = (int32_t)t.x;  // a -> b returns: parent[a] = b
    else
      parent[t.x] = (int32_t)t.y;  // b -> a returns: parent[b] = a
  }
}

// derive_parents on tile ranks (tilerank.cu): rank = segstart[seg] + off.
__global__ void __launch_bounds__(kBlock)
    k_orient_tiles(int64_t N, const uint32_t* __restrict__ eto, const int2* __restrict__ edges,
                   const uint32_t* __restrict__ seg,
                   const uint16_t* __restrict__ off, const uint32_t* __restrict__ segstart,
                   int32_t* __restrict__ parent) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t sp = seg[i];
    if (sp == kNone32) continue;  // no tree edge in this slot (the tile pass marked it)
    const uint2 t = eto_ends(eto[i], (uint32_t)i, edges);  // (b, a): arc i = a -> b, N + i = b -> a
    const uint32_t rp = segstart[sp] + off[i];
    const uint32_t rq = segstart[seg[N + i]] + off[N + i];
    if (rp > rq)
      parent[t.y] = (int32_t)t.x;  // a -> b returns: parent[a] = b
    else
      parent[t.x] = (int32_t)t.y;  // b -> a returns: parent[b] = a
  }
}

EulerIO euler_buffers(Handle& h, int64_t N, bool local_written) {
  EulerIO io;
  io.nslots = (uint32_t)N;
  io.eto = h.ws<uint32_t>(WS_ETO, N);
  io.S = h.ws<uint32_t>(WS_SUCC, 2 * N);
  io.vhead = h.ws<uint32_t>(WS_VHEAD, h.g.n);
  io.vtail = h.ws<uint32_t>(WS_VTAIL, h.g.n);
  io.rhead = h.ws<uint32_t>(WS_RHEAD, h.g.n);
  io.rtail = h.ws<uint32_t>(WS_RTAIL, h.g.n);
  if (!local_written) CK(cudaMemsetAsync(io.vhead, 0xFF, (size_t)h.g.n * sizeof(uint32_t), h.stream));
  // the remote heads are all-NONE between builds (k_euler_fix resets what it
  // splices); a fresh buffer, or one a failed build left dirty, is filled
  if (h.rhead_clean != io.rhead || h.g.n > h.rhead_clean_n)
    CK(cudaMemsetAsync(io.rhead, 0xFF, (size_t)h.g.n * sizeof(uint32_t), h.stream));
  h.rhead_clean = nullptr;  // (until the vertex pass has consumed the lists)
  return io;
}

void euler_link_edges(Handle& h, const EulerIO& io, int64_t T) {
  if (T <= 0) return;
  k_link_edges<<<grid_for(T), kBlock, 0, h.stream>>>(T, h.g.edges, io);
  CK_LAUNCH();
  h.stats.step(T);
}

// Edge locality sample: how many of `samples` evenly spaced edges join
// vertex ids less than kLocalSpan apart.
constexpr int kLocalSpan = 4096;
constexpr int kLocalitySamples = 1 << 16;
__global__ void k_edge_locality(const int2* __restrict__ edges, int64_t m, int samples,
                                unsigned long long* cnt) {
  uint32_t c = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < samples; i += gridDim.x * blockDim.x) {
    const int2 e = edges[(int64_t)i * m / samples];
    c += abs(e.y - e.x) < kLocalSpan;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

static int edge_locality(Handle& h) {
  if (h.edge_locality < 0) {
    const int64_t m = h.g.m;
    if (m == 0 || h.g.edges == nullptr) {
      h.edge_locality = 0;
    } else {
      const int samples = (int)std::min<int64_t>(m, kLocalitySamples);
      unsigned long long* cnt = reinterpret_cast<unsigned long long*>(h.dev_box) + 17;
      CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t), h.stream));
      k_edge_locality<<<64, kBlock, 0, h.stream>>>(h.g.edges, m, samples, cnt);
      CK_LAUNCH();
      h.read_box(h.dev_box + 17, 1);
      h.edge_locality = (int)(100 * h.host_box[0] / samples);
    }
  }
  return h.edge_locality;
}

void euler_root(Handle& h, const int32_t* labels, const EulerIO& io, int64_t N, int64_t T,
                bool cc_slots, int32_t designated_root, int32_t* parent, bool verify) {
  const int64_t n = h.g.n;
  const int64_t E = 2 * N;  // arc position space (holes where a slot is empty)
  // lists = tours of components with an edge: at most min(T, n - T) heads
  // (the explicit, unverified input may have more: bound by n there)
  const LrParams P = lr_params(E, verify ? n : std::min<int64_t>(T, n - T) + 1, 2 * T);
  uint32_t* minv = h.ws<uint32_t>(WS_MINV, n);
  uint32_t* rpos = h.ws<uint32_t>(WS_RPOS, P.cap);
  uint32_t* sl = h.ws<uint32_t>(WS_SL, E);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 8;
  unsigned long long* comps = reinterpret_cast<unsigned long long*>(h.dev_box) + 4;
  unsigned long long* tiles = reinterpret_cast<unsigned long long*>(h.dev_box) + 13;
  const cudaStream_t s = h.stream;

  uint32_t* lablist = h.ws<uint32_t>(WS_LABELS, n + 1);
  // labels + remote heads read, min table written, one label entry per component
  h.timer.begin(s, "euler.roots", 4.0 * n + 4.0 * n + 4.0 * n);
  // The min table is all-ones between builds: the root pass resets every
  // entry it consumes, so only a fresh (or foreign-used) buffer is filled.
  int* minv_dirty = reinterpret_cast<int*>(h.dev_box + 19);
  // (entries past the last build's n may hold an older, larger build's values)
  if (h.minv_clean != minv || n > h.minv_clean_n) {
    CK(cudaMemsetAsync(minv, 0xFF, n * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(minv_dirty, 0, sizeof(int), s));
    CK(cudaMemsetAsync(h.dev_box + 4, 0, sizeof(int64_t), s));
    CK(cudaMemsetAsync(h.dev_box + 8, 0, sizeof(int64_t), s));
    CK(cudaMemsetAsync(h.dev_box + 13, 0, sizeof(int64_t), s));
  } else {  // (the counters are zeroed by the same launch)
    k_fill_if_dirty<<<grid_for(n), kBlock, 0, s>>>(minv, n, minv_dirty,
                                                   reinterpret_cast<unsigned long long*>(h.dev_box));
  }
  h.minv_clean = nullptr;  // (until the root pass below has run)
  uint8_t* present = nullptr;
  if (!cc_slots) {
    present = h.ws<uint8_t>(WS_ISROOT, n);
    CK(cudaMemsetAsync(present, 0, (size_t)n, s));
    k_mark_labels<<<grid_for(n), kBlock, 0, s>>>(n, labels, present);
  }
  // tile-contracted ranking (tilerank.cu) or the ruling-set walk
  // (a vertex-slot tour moves between nearby slots exactly when tree edges
  // join nearby ids; RSTG_LR_TILES=0/1 forces the choice)
  const char* tiles_env = getenv("RSTG_LR_TILES");
  const bool use_tiles =
      !verify && (tiles_env ? atoi(tiles_env) != 0 : cc_slots && edge_locality(h) >= 50);
  k_euler_fix<<<grid_for((n + kFixItems - 1) / kFixItems), kBlock, 0, s>>>(
      n, labels, present, minv, io, cc_slots, lablist, comps, rpos, sl, ctr, tiles, P.logk0, P.ob,
      (uint32_t)P.cap, !use_tiles, use_tiles && cc_slots);
  h.rhead_clean = io.rhead;
  h.rhead_clean_n = n;
  k_override_root<<<1, 32, 0, s>>>(labels, minv, designated_root, cc_slots);
  k_euler_roots<<<grid_for(n), kBlock, 0, s>>>(lablist, comps, minv, io, parent, rpos, sl, ctr,
                                               P.logk0, P.ob, (uint32_t)P.cap, !use_tiles,
                                               minv_dirty, use_tiles);
  h.minv_clean = minv;
  h.minv_clean_n = n;
  if (!use_tiles && !cc_slots && T > 0)
    k_register_slots<<<grid_for(T), kBlock, 0, s>>>(T, io.nslots, rpos, sl, ctr, P.logk0, P.ob,
                                                    (uint32_t)P.cap);
  CK_LAUNCH();
  h.stats.step(n, cc_slots ? 3 : 5);
  h.timer.end(s);
  if (verify) {
    h.read_box(reinterpret_cast<int64_t*>(comps), 1);
    const int64_t nc = h.host_box[0];
    h.stats.components = nc;
    if (T != n - nc)  // euler_rooting.cpp:205-208
      throw AlgoError("edge count does not match a spanning forest of the labeling");
  }
  if (T == 0) return;

  if (use_tiles) {
    // (cc slots: the vertex pass marked the empty slots in S, no labels needed)
    const TileRank tr = lr_rank_tiles(h, P, N, io.S, cc_slots ? nullptr : labels, cc_slots, T,
                                      verify);
    // seg of every slot; per tree edge eto, the other seg, two offsets, two starts, parent
    // compulsory: per slot its arc's segment word 4 B + offset 2 B; per tree
    // edge its eto word 4 B, the other arc's word 4 B + offset 2 B, the
    // parent 4 B (segment starts: one small L2-resident table)
    h.timer.begin(s, "euler.orient", 6.0 * N + 14.0 * T);
    const uint32_t* eto = io.eto;
    const int2* edges = h.g.edges;
    k_orient_tiles<<<grid_for(N), kBlock, 0, s>>>(N, eto, edges, tr.seg, tr.off, tr.segstart,
                                                  parent);
    CK_LAUNCH();
    h.stats.step(N);
    h.timer.end(s);
    if (h.late_copy.src) {
      CK(cudaMemcpyAsync(h.host_box + 32, h.late_copy.src, h.late_copy.words * sizeof(int64_t),
                         cudaMemcpyDeviceToHost, s));
      h.late_copy = {};
    }
    if (tr.deferred)
      h.late_check = [&h, P, N, tr, eto, edges, parent, lablist, comps] {
        if (tile_rank_settle(h, P, N, tr)) {
          // re-derive from the recomputed ranks: the roots first (the first
          // orientation, on wrong ranks, may have given a root a parent)
          k_reset_roots<<<grid_for(N), kBlock, 0, h.stream>>>(lablist, comps, parent);
          k_orient_tiles<<<grid_for(N), kBlock, 0, h.stream>>>(N, eto, edges, tr.seg, tr.off,
                                                               tr.segstart, parent);
          CK_LAUNCH();
          CK(cudaStreamSynchronize(h.stream));
        }
      };
    return;
  }
  const uint32_t* rstart = lr_rank(h, P, E, io.S, sl, rpos, ctr, verify, 2 * T, nullptr);

  h.timer.begin(s, "euler.orient", 8.0 * N + 12.0 * T + 4.0 * T);
  k_orient<<<grid_for(N), kBlock, 0, s>>>(N, labels, cc_slots, io.eto, h.g.edges,
                                          sl, rstart, P.ob, parent);
  CK_LAUNCH();
  h.stats.step(N);
  h.timer.end(s);
}

}  // namespace rstg
