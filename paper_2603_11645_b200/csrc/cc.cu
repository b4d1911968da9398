#include <cstdio>
#include <cstdlib>
// cc.cu -- exact GConn-style connectivity: edge-parallel hooking with
// spanning-edge capture + pointer-jumping shortcutting.
//
// Restates cc_spanning_forest (cc_forest.cpp:73-102) bit-exactly:
//   * hook (cc_forest.cpp:18-35): per edge e=(u,v) with ru != rv the loser
//     root's slot takes min(pack(winner, e)); min mode loser = max(ru,rv),
//     max mode loser = min(ru,rv); the smallest (winner, e) wins in both.
//     One 64-bit atomicMin per proposal, skipped when a plain load already
//     shows a smaller-or-equal key (slots only decrease inside the kernel).
//   * apply (cc_forest.cpp:39-46): rep[v] = winner, tree_flag[e] = 1.
//   * jump_to_convergence (cc_forest.cpp:50-71): the Jacobi fixed point is
//     "every vertex points at the root of its rep tree", which does not
//     depend on the evaluation order, so two-level shortcutting (shared-
//     memory tiles, then the exit set in one cooperative launch) replaces
//     the ceil(log2 L) doubling barriers over all n.
//   * the apply step (and the CSR-direct round 0) also links every new
//     tree edge into the Euler rotation lists (link_tree_edge), so the
//     Euler construction needs no pass of its own.
// Hook rounds stay synchronous: proposals read
// reps frozen by the previous kernel boundary.
#include <cooperative_groups.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "engine.hpp"
#include "scan.cuh"

namespace cg = cooperative_groups;

namespace rstg {

__global__ void k_cc_init(int64_t n, int32_t* rep, unsigned long long* slot) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (rep) rep[v] = (int32_t)v;
    if (slot) slot[v] = kKeyInf;
  }
}

// hook_step edge pass (cc_forest.cpp:18-35) / graft proposals (pr_rst.cpp:82-99).
// Active-edge filtering: an edge whose endpoints share a rep stays internal
// forever (components only merge), so a round may append the edges it
// still saw crossing to out_list and the next round visits only those
// (in_list). Proposals -- and therefore the result -- are unchanged.
// Tiles of kHookItems x kBlock edges: all loads of a tile are issued before
// the dependent rep gathers (kHookItems independent chains per thread), and the
// crossing edges of a tile are compacted with one block scan and a single
// atomicAdd on the output cursor.
// Items per thread and resident CTAs: 4 edges per thread at full occupancy
// (32 registers, 8 x 256 threads per SM) beat 8 at half occupancy (64
// registers): RMAT-24 hooks 3.66 -> 3.43 ms, road 0.14 -> 0.12 ms
#ifndef RSTG_HOOK_ITEMS
#define RSTG_HOOK_ITEMS 4
#endif
#ifndef RSTG_HOOK_MINB
#define RSTG_HOOK_MINB 8
#endif
constexpr int kHookItems = RSTG_HOOK_ITEMS;
constexpr int kHookTile = kHookItems * kBlock;

// Hook rounds after round 0 skip the full compression pass (lazy mode): a
// vertex's rep may then point at an old root that has since hooked, so the
// root is found by walking up (find_root, engine.hpp). Roots are frozen for
// the whole hook kernel (apply runs later), so the root found equals the
// fully compressed label -- the proposals are exactly those of hook_step on
// compressed labels.
template <int MODE, bool WRITE>
__global__ void __launch_bounds__(kBlock, RSTG_HOOK_MINB)
    k_hook(const int2* __restrict__ edges, int64_t count, uint32_t e_base,
           const uint32_t* __restrict__ in_list, int32_t* rep,
           unsigned long long* __restrict__ slot, int* any_proposal, uint32_t* __restrict__ out_list,
           unsigned long long* out_count, bool lazy, unsigned long long* zero_word) {
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_total;
  bool proposed = false;
  // a counter the next kernel on the stream accumulates into (the round's
  // apply), cleared here instead of by a memset launch
  if (zero_word && blockIdx.x == 0 && threadIdx.x == 0) *zero_word = 0;
  for (int64_t tile = blockIdx.x; tile * kHookTile < count; tile += gridDim.x) {
    const int64_t base = tile * kHookTile;
    uint32_t idx[kHookItems];
    int2 e[kHookItems];
#pragma unroll
    for (int k = 0; k < kHookItems; ++k) {
      const int64_t i = base + k * kBlock + threadIdx.x;
      idx[k] = (i < count) ? (in_list ? __ldcs(&in_list[i]) : (uint32_t)i) : kNone32;
    }
    // the edge stream is read once: evict-first loads keep the L2 for the
    // rep gathers and slot atomics
#pragma unroll
    for (int k = 0; k < kHookItems; ++k)
      e[k] = (idx[k] != kNone32) ? __ldcs(&edges[idx[k]]) : make_int2(0, 0);
    // reps of both endpoints of all items first (independent loads), then
    // in lazy mode their reps (independent again), then the rare deeper walks
    int32_t ru[kHookItems], rv[kHookItems];
#pragma unroll
    for (int k = 0; k < kHookItems; ++k) {
      ru[k] = rep[e[k].x];
      rv[k] = rep[e[k].y];
    }
    if (lazy) {
      int32_t gu[kHookItems], gv[kHookItems];
#pragma unroll
      for (int k = 0; k < kHookItems; ++k) {
        gu[k] = rep[ru[k]];
        gv[k] = rep[rv[k]];
      }
#pragma unroll
      for (int k = 0; k < kHookItems; ++k) {
        if (gu[k] != ru[k]) ru[k] = find_root(rep, e[k].x);
        if (gv[k] != rv[k]) rv[k] = find_root(rep, e[k].y);
      }
    }
    uint32_t ncross = 0;
#pragma unroll
    for (int k = 0; k < kHookItems; ++k) {
      const int32_t lo = min(ru[k], rv[k]), hi = max(ru[k], rv[k]);
      if (idx[k] == kNone32 || lo == hi) {
        idx[k] = kNone32;
        continue;
      }
      ++ncross;
      const int32_t winner = MODE == 0 ? lo : hi;
      const int32_t loser = MODE == 0 ? hi : lo;
      const unsigned long long key = pack_key((uint32_t)winner, e_base + idx[k]);
      if (key < slot[loser]) atomicMin(&slot[loser], key);
    }
    proposed |= ncross > 0;
    if (WRITE) {
      uint32_t off = block_excl_scan(ncross, &s_total);
      if (threadIdx.x == 0) s_base = s_total ? atomicAdd(out_count, (unsigned long long)s_total) : 0;
      __syncthreads();
      const unsigned long long ob = s_base + off;
#pragma unroll
      for (int k = 0, j = 0; k < kHookItems; ++k)
        if (idx[k] != kNone32) out_list[ob + j++] = idx[k];
      __syncthreads();
    }
  }
  if (any_proposal) block_flag(proposed, any_proposal);
}

// Apply step (cc_forest.cpp:39-46); counts applied hooks (= new tree
// edges). A root hooks at most once over the whole run (it is never a root
// again), so tedge[v] = the edge that hooked v is a collision-free record
// of the tree-edge set, indexed by vertex, for the Euler construction.
__global__ void __launch_bounds__(kBlock)
    k_apply(int64_t n, int32_t* __restrict__ rep, unsigned long long* __restrict__ slot,
            uint8_t* __restrict__ tflag, uint32_t e_base, uint32_t m_local,
            unsigned long long* counter, uint32_t* __restrict__ tedge) {
  uint32_t cnt = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = slot[v];
    if (key == kKeyInf) continue;
    rep[v] = (int32_t)(key >> 32);
    const uint32_t eg = (uint32_t)key;
    const uint32_t e = eg - e_base;
    if (tflag && e < m_local) tflag[e] = 1;
    if (tedge) tedge[v] = eg;
    slot[v] = kKeyInf;
    ++cnt;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ uint32_t ws[kBlock / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kBlock / 32; ++w) t += ws[w];
    if (t) atomicAdd(counter, (unsigned long long)t);
  }
}

// ---- two-level shortcutting ---------------------------------------------
#ifndef RSTG_JUMP_BATCH
#define RSTG_JUMP_BATCH 4
#endif
constexpr int kJumpBatch = RSTG_JUMP_BATCH;  // entries in flight per thread in k_jump_x
#ifndef RSTG_JUMP_HOPS
#define RSTG_JUMP_HOPS 4  // pointer hops per entry per round of k_jump_x
#endif

// Level 1 (k_tile_resolve): each CTA owns a tile of kTileV consecutive
// vertices held in shared memory and follows every pointer while it stays
// inside the tile (in-smem doubling), so rep[v] becomes either a root or the
// first ancestor outside v's tile. Those out-of-tile targets X are appended
// (deduplicated by a bitmap, warp-aggregated) to a list as they are found.
// Level 2: one cooperative kernel pointer-jumps X in place (its pointers
// stay inside X or hit roots), a grid barrier per doubling round, stopping
// on the device once a round changes nothing; a last gather
// rep[v] = rep[rep[v]] finishes. Passes over all n: 2 (tile, final gather)
// instead of ~log2(depth), no host round trip.
// 8K vertices per tile (32 KB of shared memory, two 1024-thread CTAs per
// SM). Measured on the road mesh: 32K-vertex tiles (one CTA per SM) keep
// more pointers inside the tile but lose more to the lower occupancy.
#ifndef RSTG_CC_TILEV
#define RSTG_CC_TILEV 8192
#endif
constexpr int kTileV = RSTG_CC_TILEV;
constexpr int kTileThreads = 1024;
constexpr size_t kTileSmem = kTileV * sizeof(int32_t);

// Sources of the tile's pointers (fused with the level-1 resolve so the new
// reps never round-trip through HBM before shortcutting):
//   kSrcRep    rep as is
//   kSrcApply  apply step first: hooked roots take their slot's winner
//              (cc_forest.cpp:39-46), the slot is reset, the edge recorded
//   kSrcRound0 the first hook round computed directly from the CSR: with
//              every rep a singleton, min-mode hooking gives v the key
//              min over neighbours u < v of (u, e), i.e. v's first CSR
//              neighbour (lists ascending) with its unique edge id
//   kSrcRound0Slot  the same round 0 with the hook keys already in the
//              slots (the edge upload computed them as the edges streamed
//              in, graph.cu): no CSR needed
enum { kSrcRep = 0, kSrcApply = 1, kSrcRound0 = 2, kSrcRound0Slot = 3 };

struct RoundIO {
  unsigned long long* slot;
  uint8_t* tflag;               // tree-edge flags by local edge id (nullable)
  uint32_t e_base, m_local;
  unsigned long long* counter;  // += hooks applied
  const uint32_t* offsets;
  const int32_t* nbrs;
  const uint32_t* arc_edge;
  const int2* edges;
  bool link;                    // link new tree edges into the Euler rotation lists
  EulerIO eu;
  uint32_t* roots;              // round 0: vertices left as roots (nullable)
  unsigned long long* nroots;
  bool edge_sentinel;           // round-0 slots carry kKeyEdge (empty = isolated)
  // PR-RST's first graft round (identity forest): a hooked v gets parent u
  // and the skip structure's level 0 its entry (pr.cu)
  int32_t* pr_parent;
  const uint32_t* pr_pos;
  uint32_t* pr_q0;
};

// Run shortcut before the in-tile doubling: a vertex whose pointer is its
// left neighbour (p = v - 1, inside the tile) continues that neighbour's
// run. One block-wide max-scan over the tile (blocked layout: a thread owns
// kTileV / kTileThreads consecutive vertices) gives every vertex the first
// vertex h of its run, and s[v] = s[h] jumps the whole run at once (h keeps
// its pointer, so no entry is read while it is written). Locally numbered
// graphs chain along runs (a mesh row, a path): the doubling then only has
// the runs' heads left -- two or three rounds instead of ~log2(row). A tile
// with few such pointers (power-law graphs) skips it after one barrier.
__device__ __forceinline__ void run_shortcut(int32_t* s, int64_t base, int cnt) {
  constexpr int kB = kTileV / kTileThreads;
  static_assert(kB % 4 == 0 && kB <= 32, "blocked layout: a multiple of 4 vertices per thread");
  __shared__ int s_wmax[kTileThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int i0 = t * kB;
  int32_t pv[kB];
#pragma unroll
  for (int q = 0; q < kB / 4; ++q) {
    const int4 a = reinterpret_cast<const int4*>(s)[kB / 4 * t + q];
    pv[4 * q] = a.x;
    pv[4 * q + 1] = a.y;
    pv[4 * q + 2] = a.z;
    pv[4 * q + 3] = a.w;
  }
  uint32_t left = 0;
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    const int i = i0 + j;
    if (i > 0 && i < cnt && (int64_t)pv[j] == base + i - 1) left |= 1u << j;
  }
  if (__syncthreads_count(__popc(left)) < kTileV / 8) return;  // (block-uniform)
  // inclusive max-scan of "run start" indices: a non-left vertex starts a run
  int key[kB];
  int m = -1;
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    if (!(left >> j & 1)) m = i0 + j;
    key[j] = m;
  }
  int incl = m;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = max(incl, y);
  }
  int excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = -1;
  if (lane == 31) s_wmax[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = s_wmax[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = max(w, y);
    }
    const int we = __shfl_up_sync(0xffffffffu, w, 1);
    s_wmax[lane] = lane == 0 ? -1 : we;  // (exclusive over the warps)
  }
  __syncthreads();
  const int prefix = max(excl, s_wmax[warp]);
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    if (!(left >> j & 1)) continue;
    const int h = key[j] >= 0 ? key[j] : prefix;  // (a left vertex always has a start before it)
    pv[j] = s[h];                                  // the run start's own pointer
  }
  __syncthreads();  // (every read of a run start done before the writes)
#pragma unroll
  for (int j = 0; j < kB; ++j)
    if (left >> j & 1) s[i0 + j] = pv[j];
  __syncthreads();
}

template <int SRC>
__global__ void __launch_bounds__(kTileThreads, kTileV > 8192 ? 1 : 2)
    k_tile_resolve(int64_t n, int32_t* rep, uint32_t* xbits, uint32_t* xlist,
                   unsigned long long* xcount, RoundIO io) {
  extern __shared__ int32_t s[];  // kTileV reps (+ 2 x kTileV list words when linking round 0)
  __shared__ uint32_t s_cnt;
  const int64_t base = (int64_t)blockIdx.x * kTileV;
  const int cnt = (int)min((int64_t)kTileV, n - base);
  // Round 0 links its tree edges (u, v), u = v's first neighbour, into
  // shared-memory rotation lists whenever u lies in the tile (nearly
  // always: u is an adjacent id on meshes), then splices each tile list
  // into the global one with a single atomic (see the flush below).
  constexpr bool kLocal = SRC == kSrcRound0 || SRC == kSrcRound0Slot;
  uint32_t* s_head = reinterpret_cast<uint32_t*>(s + kTileV);
  uint32_t* s_tail = s_head + kTileV;
  if (threadIdx.x == 0) s_cnt = 0;
  if (kLocal && io.link) {
    for (int i = threadIdx.x; i < kTileV; i += kTileThreads) s_head[i] = kNone32;
    __syncthreads();
  }
  uint32_t hooked = 0;
  uint32_t rootmask = 0;  // round 0: items of this thread that stay roots
  // Round 0: the tile's first neighbours are fetched in two batched passes
  // -- all offsets into shared memory, then all neighbour reads into
  // registers -- so a thread keeps its 8 items' loads in flight together
  // instead of paying two dependent latencies per item in turn.
  constexpr int kItems = kTileV / kTileThreads;
  int32_t fnb[kItems];
  if (SRC == kSrcRound0) {
    uint32_t* s_o = reinterpret_cast<uint32_t*>(s);  // (reps go here later)
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int i = threadIdx.x + k * kTileThreads;
      if (i < cnt) s_o[i] = io.offsets[base + i];
    }
    __syncthreads();
    const uint32_t o_end = io.offsets[base + cnt];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int i = threadIdx.x + k * kTileThreads;
      fnb[k] = INT32_MAX;
      if (i < cnt) {
        const uint32_t o = s_o[i], o1 = i + 1 < cnt ? s_o[i + 1] : o_end;
        if (o < o1) fnb[k] = io.nbrs[o];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k) {  // (unrolled: fnb stays in registers)
    const int i = threadIdx.x + k * kTileThreads;
    if (i >= cnt) break;
    const int64_t v = base + i;
    int32_t r;
    if (SRC == kSrcRep) {
      r = rep[v];
    } else if (SRC == kSrcApply) {
      const unsigned long long key = io.slot[v];
      r = rep[v];
      if (key != kKeyInf) {
        r = (int32_t)(key >> 32);
        io.slot[v] = kKeyInf;
        ++hooked;
        const uint32_t e = (uint32_t)key - io.e_base;
        if (io.tflag && e < io.m_local) io.tflag[e] = 1;
        if (io.link) {
          const int2 ab = io.edges[e];
          link_tree_edge(io.eu, (uint32_t)v, (uint32_t)ab.x, (uint32_t)ab.y, e);
        }
      }
    } else {
      r = (int32_t)v;
      // cleared below if v hooks; an isolated vertex (no neighbour: the CSR
      // path knows, and so do slots keyed with the kKeyEdge sentinel) can
      // never hook, so it stays off the roots list that every later apply
      // and roots jump walks (RMAT-24: 7.9M of 16.8M)
      if (SRC == kSrcRound0 && fnb[k] != INT32_MAX) rootmask |= 1u << k;
      {
        int32_t u = INT32_MAX;
        uint32_t ekey = kNone32;  // (kSrcRound0Slot: the edge id from the key)
        if (SRC == kSrcRound0) {
          u = fnb[k];
        } else {
          const unsigned long long key = io.slot[v];
          if (!io.edge_sentinel || key != kKeyInf) rootmask |= 1u << k;
          if (key < kKeyEdge) {
            u = (int32_t)(key >> 32);
            ekey = (uint32_t)key;
          }
          if (key != kKeyInf) io.slot[v] = kKeyInf;  // (keeps the slots clean for the next rounds)
        }
        if (u < r) {  // hooked onto its smallest neighbour by edge (u, v)
          rootmask &= ~(1u << k);
          r = u;
          ++hooked;
          if (io.tflag) {
            const uint32_t e = SRC == kSrcRound0 ? io.arc_edge[io.offsets[v]] : ekey - io.e_base;
            if (e < io.m_local) io.tflag[e] = 1;
          }
          if (SRC == kSrcRound0 && io.pr_parent) {
            io.pr_parent[v] = u;
            io.pr_q0[io.pr_pos[v]] = io.pr_pos[u];
          }
          if (io.link) {
            const uint32_t pa = (uint32_t)v, qa = io.eu.nslots + (uint32_t)v;  // pa: u -> v, qa: v -> u
            io.eu.eto[v] = (uint32_t)u;  // (b = v, the slot: one word per tree edge)
            const int64_t lu = (int64_t)u - base;
            uint32_t nu;
            if (lu >= 0) {  // u < v, so lu < cnt
              nu = atomicExch(&s_head[lu], pa);
              if (nu == kNone32) s_tail[lu] = pa;
            } else {
              nu = atomicExch(&io.eu.rhead[u], pa);
              if (nu == kNone32) io.eu.rtail[u] = pa;
            }
            const uint32_t nv = atomicExch(&s_head[i], qa);
            if (nv == kNone32) s_tail[i] = qa;
            io.eu.S[pa] = nv;  // S[pa] = next(qa), S[qa] = next(pa)
            io.eu.S[qa] = nu;
          }
        } else if (SRC == kSrcRound0 && io.pr_parent) {  // (a root: PR-RST's identity entries)
          io.pr_parent[v] = (int32_t)v;
          const uint32_t pv = io.pr_pos[v];
          io.pr_q0[pv] = pv;
        }
      }
    }
    s[i] = r;
  }
  if (kLocal && io.roots) {  // the round-0 roots, appended with one atomic per tile
    __shared__ uint32_t s_rc;
    __shared__ unsigned long long s_rb;
    if (threadIdx.x == 0) s_rc = 0;
    __syncthreads();
    uint32_t pos = rootmask ? atomicAdd(&s_rc, (uint32_t)__popc(rootmask)) : 0u;
    __syncthreads();
    if (threadIdx.x == 0) s_rb = s_rc ? atomicAdd(io.nroots, (unsigned long long)s_rc) : 0ull;
    __syncthreads();
    for (uint32_t mk = rootmask; mk; mk &= mk - 1)
      io.roots[s_rb + pos++] = (uint32_t)(base + threadIdx.x + (__ffs(mk) - 1) * kTileThreads);
  }
  if (kLocal && io.link) {
    // the tile's lists become the vertices' local lists (plain stores;
    // links from other tiles went to the remote lists), each closed into
    // its rotation cycle right away: next(tail) = head (the Euler pass
    // re-splices the few vertices that also have a remote list, and opens
    // the roots' cycles)
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += kTileThreads) {
      const uint32_t hd = s_head[i];
      io.eu.vhead[base + i] = hd;
      if (hd != kNone32) {
        // the tail is kept so a later splice needs no load of S: loading S
        // right after other warps stored into the same sectors costs 3.4x
        // in k_euler_fix (163 -> 553 us on road)
        const uint32_t tl = s_tail[i];
        io.eu.vtail[base + i] = tl;
        io.eu.S[arc_rev(tl, io.eu.nslots)] = hd;
      }
    }
  }
  if (SRC != kSrcRep) {
    for (int o = 16; o > 0; o >>= 1) hooked += __shfl_xor_sync(0xffffffffu, hooked, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && hooked) atomicAdd(&s_cnt, hooked);
  }
  __syncthreads();
  if (SRC != kSrcRep && threadIdx.x == 0 && s_cnt) atomicAdd(io.counter, (unsigned long long)s_cnt);
  run_shortcut(s, base, cnt);
  for (;;) {
    bool changed = false;
    for (int i = threadIdx.x; i < cnt; i += kTileThreads) {
      const int32_t p = s[i];
      const int64_t lp = (int64_t)p - base;
      if (lp >= 0 && lp < cnt) {
        const int32_t q = s[lp];
        if (q != p) {
          s[i] = q;
          changed = true;
        }
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
  // Exit targets: written back with the reps, deduplicated (warp match,
  // then a bitmap), collected in shared memory (s[] is free once the reps
  // are out) and appended with ONE global atomic per tile -- a per-warp
  // atomic on the shared counter serialises on a single address.
  // The bitmap round trips run after the candidates are compacted: one
  // candidate per thread per pass, so a tile waits about one L2 latency
  // for them, not one per item of the busiest thread (and without the
  // registers that batching across a thread's items would need).
  constexpr int kPer = kTileV / kTileThreads;
  __shared__ uint32_t s_xn, s_new, s_wr;
  __shared__ unsigned long long s_xb;
  uint32_t pk[kPer];
  uint32_t cand = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int i = threadIdx.x + k * kTileThreads;
    const int32_t p = i < cnt ? s[i] : -1;
    pk[k] = (uint32_t)p;
    const unsigned same = __match_any_sync(0xffffffffu, p);
    if (i < cnt) {
      rep[base + i] = p;
      const int64_t lp = (int64_t)p - base;
      if ((lp < 0 || lp >= cnt) && (threadIdx.x & 31) == __ffs(same) - 1) cand |= 1u << k;
    }
  }
  if (threadIdx.x == 0) s_xn = s_new = s_wr = 0;
  __syncthreads();  // s[] reads done
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    if (cand & (1u << k)) s[atomicAdd(&s_xn, 1u)] = (int32_t)pk[k];
  __syncthreads();
  const uint32_t nc = s_xn;
  for (uint32_t j = threadIdx.x; j < nc; j += kTileThreads) {
    // many vertices share one exit target (a big component's root): a
    // plain L2 read skips the atomic once the bit is set
    const uint32_t p = (uint32_t)s[j];
    const uint32_t bit = 1u << (p & 31);
    if (!(ld_cg(&xbits[p >> 5]) & bit) && !(atomicOr(&xbits[p >> 5], bit) & bit)) {
      s[j] = (int32_t)(p | 0x80000000u);  // (ids < 2^31: the top bit marks a new target)
      atomicAdd(&s_new, 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) s_xb = s_new ? atomicAdd(xcount, (unsigned long long)s_new) : 0ull;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < nc; j += kTileThreads) {
    const uint32_t p = (uint32_t)s[j];
    if (p & 0x80000000u) xlist[s_xb + atomicAdd(&s_wr, 1u)] = p & 0x7FFFFFFFu;
  }
}

// In-place doubling over the exit set, all rounds in one cooperative
// launch. flags: 3 rotating "changed" words (zeroed before the launch).
__global__ void __launch_bounds__(kBlock)
    k_jump_x(const uint32_t* __restrict__ list, const unsigned long long* xcount, int32_t* rep,
             int* flags, int max_rounds, uint32_t* xbits) {
  cg::grid_group grid = cg::this_grid();
  const int64_t X = (int64_t)*xcount;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < max_rounds; ++r) {
    if (gtid == 0) flags[(r + 1) % 3] = 0;  // read by everyone two barriers ago
    bool changed = false;
    // kJumpBatch entries per thread at a time: their loads of one hop level
    // are issued together (independent chains), not one chain after another
    for (int64_t i0 = gtid; i0 < X; i0 += kJumpBatch * gsize) {
      uint32_t v[kJumpBatch];
      int32_t p[kJumpBatch], x[kJumpBatch];
      bool live[kJumpBatch];
#pragma unroll
      for (int k = 0; k < kJumpBatch; ++k) {
        const int64_t i = i0 + k * gsize;
        live[k] = i < X;
        v[k] = live[k] ? list[i] : 0u;
        // the exit-set bitmap holds exactly the listed entries' bits: the
        // first round clears them, so it is all-zero for the next pass
        if (xbits && r == 0 && live[k]) xbits[v[k] >> 5] = 0u;
      }
#pragma unroll
      for (int k = 0; k < kJumpBatch; ++k) p[k] = live[k] ? ld_cg(&rep[v[k]]) : 0;
#pragma unroll
      for (int k = 0; k < kJumpBatch; ++k) {
        x[k] = live[k] ? ld_cg(&rep[p[k]]) : 0;
        live[k] = live[k] && x[k] != p[k];  // p a root: nothing to do
      }
      bool walk[kJumpBatch];
#pragma unroll
      for (int k = 0; k < kJumpBatch; ++k) walk[k] = live[k];
#pragma unroll
      for (int hop = 1; hop < RSTG_JUMP_HOPS; ++hop) {
#pragma unroll
        for (int k = 0; k < kJumpBatch; ++k) {
          if (!walk[k]) continue;
          const int32_t y = ld_cg(&rep[x[k]]);
          if (y == x[k]) walk[k] = false;
          else x[k] = y;
        }
      }
#pragma unroll
      for (int k = 0; k < kJumpBatch; ++k) {
        if (!live[k]) continue;
        rep[v[k]] = x[k];
        changed = true;
      }
    }
    if (__syncthreads_or(changed) && threadIdx.x == 0) flags[r % 3] = 1;
    grid.sync();
    if (*((volatile int*)&flags[r % 3]) == 0) break;
  }
}

__global__ void __launch_bounds__(kBlock) k_final_gather(int64_t n, int32_t* rep) {
  // kJumpBatch vertices per thread at a time: all their loads before any
  // store (a store to rep would otherwise order the next vertex's loads)
  const int64_t g = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < n; v0 += kJumpBatch * g) {
    int32_t p[kJumpBatch], q[kJumpBatch];
#pragma unroll
    for (int k = 0; k < kJumpBatch; ++k) p[k] = v0 + k * g < n ? rep[v0 + k * g] : 0;
#pragma unroll
    for (int k = 0; k < kJumpBatch; ++k) q[k] = v0 + k * g < n ? rep[p[k]] : 0;
#pragma unroll
    for (int k = 0; k < kJumpBatch; ++k)
      if (v0 + k * g < n && q[k] != p[k]) rep[v0 + k * g] = q[k];
  }
}

// One shortcutting pass (optionally fused with the round's apply step or
// the CSR first round): tile resolve, then the exit set, then the gather.
// Zeroes up to kZeroRanges word ranges in one launch (the counters and
// bitmaps a phase accumulates into), instead of one memset launch each.
constexpr int kZeroRanges = 6;
struct ZeroRanges {
  uint32_t* p[kZeroRanges];
  uint32_t words[kZeroRanges];
  int k;
  void add(void* ptr, size_t bytes) {
    p[k] = static_cast<uint32_t*>(ptr);
    words[k++] = (uint32_t)(bytes / 4);
  }
};
__global__ void k_zero_ranges(ZeroRanges z) {
  for (int r = 0; r < z.k; ++r)
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < z.words[r];
         i += gridDim.x * blockDim.x)
      z.p[r][i] = 0;
}

void resolve_round(Handle& h, int32_t* rep, int64_t n, int src, const RoundIO& io,
                   const ZeroRanges* extra = nullptr) {
  if (n <= 0) return;
  const int64_t words = (n + 31) / 32;
  uint32_t* xbits = h.ws<uint32_t>(WS_XBITS, words);
  uint32_t* xlist = h.ws<uint32_t>(WS_HEADS, n + 1);
  unsigned long long* xcount = reinterpret_cast<unsigned long long*>(h.dev_box) + 5;
  int* flags = reinterpret_cast<int*>(h.dev_box + 6);  // 3 ints in dev_box[6..7]
  // (host-side setup first, so that the zeroing and the tile pass launch
  // back to back: the GPU otherwise idles between them)
  const unsigned tiles = (unsigned)((n + kTileV - 1) / kTileV);
  static int coop_blocks = 0;
  ensure_dyn_smem((const void*)k_tile_resolve<kSrcApply>, kTileSmem);
  ensure_dyn_smem((const void*)k_tile_resolve<kSrcRound0>, 3 * kTileSmem);
  ensure_dyn_smem((const void*)k_tile_resolve<kSrcRound0Slot>, 3 * kTileSmem);
  ensure_dyn_smem((const void*)k_tile_resolve<kSrcRep>, kTileSmem);
  if (!coop_blocks) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jump_x, kBlock, 0));
    coop_blocks = std::max(1, per_sm) * num_sms();
  }
  {
    ZeroRanges z = extra ? *extra : ZeroRanges{};
    if (!extra) z.k = 0;
    // (the bitmap is all-zero after a completed pass: its exit-set jump
    // clears the bits it set)
    if (h.xbits_clean != xbits || words > h.xbits_clean_words)
      z.add(xbits, (size_t)words * sizeof(uint32_t));
    h.xbits_clean = nullptr;
    z.add(h.dev_box + 5, 3 * sizeof(int64_t));
    uint32_t most = 0;  // (the grid covers the largest range actually zeroed)
    for (int r = 0; r < z.k; ++r) most = std::max(most, z.words[r]);
    k_zero_ranges<<<(unsigned)std::min<int64_t>(1184, ((int64_t)most + 1023) / 1024), 1024, 0,
                    h.stream>>>(z);
    CK_LAUNCH();
  }
  if (src == kSrcApply)
    k_tile_resolve<kSrcApply><<<tiles, kTileThreads, kTileSmem, h.stream>>>(n, rep, xbits, xlist,
                                                                            xcount, io);
  else if (src == kSrcRound0Slot)
    k_tile_resolve<kSrcRound0Slot><<<tiles, kTileThreads, io.link ? 3 * kTileSmem : kTileSmem,
                                     h.stream>>>(n, rep, xbits, xlist, xcount, io);
  else if (src == kSrcRound0)
    k_tile_resolve<kSrcRound0><<<tiles, kTileThreads, io.link ? 3 * kTileSmem : kTileSmem,
                                 h.stream>>>(n, rep, xbits, xlist, xcount, io);
  else
    k_tile_resolve<kSrcRep><<<tiles, kTileThreads, kTileSmem, h.stream>>>(n, rep, xbits, xlist,
                                                                          xcount, io);
  CK_LAUNCH();
  h.stats.step(n);
  int rounds = 2;
  while ((int64_t{1} << (rounds - 2)) < n) ++rounds;  // X-forest depth <= |X| <= n
  const unsigned long long* xc = xcount;
  void* args[] = {(void*)&xlist, (void*)&xc, (void*)&rep, (void*)&flags, (void*)&rounds,
                  (void*)&xbits};
  CK(cudaLaunchCooperativeKernel((void*)k_jump_x, dim3(coop_blocks), dim3(kBlock), args, 0,
                                 h.stream));
  h.xbits_clean = xbits;
  h.xbits_clean_words = words;
  h.stats.step(n);
  k_final_gather<<<grid_for(n), kBlock, 0, h.stream>>>(n, rep);
  CK_LAUNCH();
  h.stats.step(n);
  static const bool dbg = getenv("RSTG_CC_DEBUG") != nullptr;
  if (dbg) {
    h.read_box(h.dev_box + 5, 1);
    fprintf(stderr, "resolve_round src %d: n %lld, exit set %lld\n", src, (long long)n,
            (long long)h.host_box[0]);
  }
}

// The same jumping for a short list (<= kJumpSmallMax entries: meshes have a
// few thousand round-0 roots), on chip: one CTA hashes the list's vertices
// into shared memory, maps each entry's pointer to a list index (one global
// load per entry), jumps the indices in shared memory and writes the roots
// back. A pointer that leaves the list (not expected: hooks join roots)
// stays as it is -- labels stay valid ancestors either way.
constexpr int kJumpSmallMax = 8192;
constexpr int kJumpHash = 2 * kJumpSmallMax;
constexpr size_t kJumpSmallSmem = kJumpHash * (sizeof(uint32_t) + sizeof(uint16_t)) +
                                  kJumpSmallMax * (sizeof(uint16_t) + sizeof(uint32_t));
constexpr int kJumpPer = kJumpSmallMax / 1024;
// (one block of 1024 threads; smem: kJumpSmallSmem bytes)
__device__ __forceinline__ void jump_small_block(const uint32_t* __restrict__ list,
                                                 const unsigned long long* count, int32_t* rep,
                                                 uint32_t* hkey) {
  uint32_t* lst = hkey + kJumpHash;   // the list
  uint16_t* hval = reinterpret_cast<uint16_t*>(lst + kJumpSmallMax);  // list index
  uint16_t* par = hval + kJumpHash;  // index of the entry's pointer target
  const unsigned long long cnt = *count;
  const int X = cnt < (unsigned long long)kJumpSmallMax ? (int)cnt : kJumpSmallMax;
  const int tid = threadIdx.x;
  // every global load of a thread in flight at once: its entries, then
  // their pointers
  uint32_t v[kJumpPer], p[kJumpPer];
#pragma unroll
  for (int k = 0; k < kJumpPer; ++k) v[k] = tid + k * 1024 < X ? list[tid + k * 1024] : 0u;
#pragma unroll
  for (int k = 0; k < kJumpPer; ++k) p[k] = tid + k * 1024 < X ? (uint32_t)ld_cg(&rep[v[k]]) : 0u;
  for (int h = tid; h < kJumpHash; h += 1024) hkey[h] = 0;
  __syncthreads();
  auto slot_of = [](uint32_t x) { return (x * 0x9E3779B1u) >> (32 - 14); };  // 14 bits
#pragma unroll
  for (int k = 0; k < kJumpPer; ++k) {
    const int i = tid + k * 1024;
    if (i >= X) continue;
    lst[i] = v[k];
    for (uint32_t h = slot_of(v[k]);; h = (h + 1) & (kJumpHash - 1)) {
      const uint32_t key = atomicCAS(&hkey[h], 0u, v[k] + 1);
      if (key == 0 || key == v[k] + 1) {
        hval[h] = (uint16_t)i;
        break;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kJumpPer; ++k) {
    const int i = tid + k * 1024;
    if (i >= X) continue;
    uint16_t j = (uint16_t)i;  // not in the list: leave the entry alone
    for (uint32_t h = slot_of(p[k]);; h = (h + 1) & (kJumpHash - 1)) {
      const uint32_t key = hkey[h];
      if (key == p[k] + 1) {
        j = hval[h];
        break;
      }
      if (key == 0) break;
    }
    par[i] = j;
  }
  __syncthreads();
  for (int r = 0; r < 32; ++r) {  // in place: an entry always holds an ancestor
    int changed = 0;
    for (int i = tid; i < X; i += 1024) {
      const uint16_t a = par[i], b = par[a];
      if (a != b) {
        par[i] = b;
        changed = 1;
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
#pragma unroll
  for (int k = 0; k < kJumpPer; ++k) {
    const int i = tid + k * 1024;
    if (i >= X) continue;
    const uint32_t t = lst[par[i]];
    if (t != v[k] && t != p[k]) rep[v[k]] = (int32_t)t;
  }
}
__global__ void __launch_bounds__(1024)
    k_jump_small(const uint32_t* __restrict__ list, const unsigned long long* count, int32_t* rep) {
  extern __shared__ uint32_t hkey[];  // vertex + 1, 0 = empty
  jump_small_block(list, count, rep, hkey);
}

// Pointer-jumps the entries of a vertex list in place (one cooperative
// launch, device-side stop): the chains among round-0 roots after a lazy round.
void jump_list(Handle& h, int32_t* rep, int64_t n, const uint32_t* list,
               const unsigned long long* count) {
  int* flags = reinterpret_cast<int*>(h.dev_box + 6);  // 3 ints in dev_box[6..7]
  CK(cudaMemsetAsync(h.dev_box + 6, 0, 2 * sizeof(int64_t), h.stream));
  static int coop_blocks = 0;
  if (!coop_blocks) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jump_x, kBlock, 0));
    coop_blocks = std::max(1, per_sm) * num_sms();
  }
  int rounds = 2;
  while ((int64_t{1} << (rounds - 2)) < n) ++rounds;
  uint32_t* no_bits = nullptr;
  void* args[] = {(void*)&list, (void*)&count, (void*)&rep, (void*)&flags, (void*)&rounds,
                  (void*)&no_bits};
  CK(cudaLaunchCooperativeKernel((void*)k_jump_x, dim3(coop_blocks), dim3(kBlock), args, 0,
                                 h.stream));
  h.stats.step(n);
}

// Compression after lazy rounds: every pointer chain runs through former
// roots only (a vertex's first hop lands on a root of some earlier round),
// so pointer-jumping the round-0 roots list in place (one cooperative
// launch) and one gather rep[v] = rep[rep[v]] compress the whole forest.
void compress_via_roots(Handle& h, int32_t* rep, int64_t n, const uint32_t* roots,
                        const unsigned long long* nroots) {
  int* flags = reinterpret_cast<int*>(h.dev_box + 6);  // 3 ints in dev_box[6..7]
  CK(cudaMemsetAsync(h.dev_box + 6, 0, 2 * sizeof(int64_t), h.stream));
  static int coop_blocks = 0;
  if (!coop_blocks) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jump_x, kBlock, 0));
    coop_blocks = std::max(1, per_sm) * num_sms();
  }
  int rounds = 2;
  while ((int64_t{1} << (rounds - 2)) < n) ++rounds;
  uint32_t* no_bits = nullptr;
  void* args[] = {(void*)&roots, (void*)&nroots, (void*)&rep, (void*)&flags, (void*)&rounds,
                  (void*)&no_bits};
  CK(cudaLaunchCooperativeKernel((void*)k_jump_x, dim3(coop_blocks), dim3(kBlock), args, 0,
                                 h.stream));
  h.stats.step(n);
  k_final_gather<<<grid_for(n), kBlock, 0, h.stream>>>(n, rep);
  CK_LAUNCH();
  h.stats.step(n);
}

void launch_compress2(Handle& h, int32_t* rep, int64_t n) {
  resolve_round(h, rep, n, kSrcRep, RoundIO{});
}

static void launch_hook_k(Handle& h, int mode, const int2* edges, int64_t count, uint32_t e_base,
                          const uint32_t* in_list, const int32_t* rep_c, unsigned long long* slot,
                          int* any_prop, uint32_t* out_list, unsigned long long* out_count,
                          unsigned long long* zero_word = nullptr) {
  const unsigned grid = grid_for((count + kHookItems - 1) / kHookItems);
  int32_t* rep = const_cast<int32_t*>(rep_c);  // lazy mode path-compresses
  const bool lazy = h.cc_lazy;
  if (mode == 0 && out_list)
    k_hook<0, true><<<grid, kBlock, 0, h.stream>>>(edges, count, e_base, in_list, rep, slot,
                                                   any_prop, out_list, out_count, lazy, zero_word);
  else if (mode == 0)
    k_hook<0, false><<<grid, kBlock, 0, h.stream>>>(edges, count, e_base, in_list, rep, slot,
                                                    any_prop, out_list, out_count, lazy, zero_word);
  else if (out_list)
    k_hook<1, true><<<grid, kBlock, 0, h.stream>>>(edges, count, e_base, in_list, rep, slot,
                                                   any_prop, out_list, out_count, lazy, zero_word);
  else
    k_hook<1, false><<<grid, kBlock, 0, h.stream>>>(edges, count, e_base, in_list, rep, slot,
                                                    any_prop, out_list, out_count, lazy, zero_word);
  CK_LAUNCH();
  h.stats.step(count);
}

void launch_hook(Handle& h, int mode, const int2* edges, int64_t m, uint32_t e_base,
                 const int32_t* rep, unsigned long long* slot, int* any_prop) {
  launch_hook_k(h, mode, edges, m, e_base, nullptr, rep, slot, any_prop, nullptr, nullptr);
}

// Filtered hook round on the handle's edges. Round 0 sees every edge cross
// (all reps distinct), so filtering starts by recording round 1's crossing
// edges; later rounds visit only the previous round's list.
// *out_count (device) must be zero; pass its host value to cc_round_done.
void cc_hook_round(Handle& h, int mode, const int32_t* rep, unsigned long long* slot,
                   unsigned long long* out_count, int* any_prop, unsigned long long* zero_word) {
  const int64_t m = h.g.m;
  const uint32_t eb = (uint32_t)h.g.e_base;
  bool launched = false;
  if (h.cc_round == 0 || m == 0 || h.cc_round < h.cc_filter_from) {
    if (m > 0) {
      launch_hook_k(h, mode, h.g.edges, m, eb, nullptr, rep, slot, any_prop, nullptr, nullptr,
                    zero_word);
      launched = true;
    }
  } else if (h.cc_active < 0) {
    uint32_t* out = h.ws<uint32_t>(WS_ELIST0, m);
    launch_hook_k(h, mode, h.g.edges, m, eb, nullptr, rep, slot, any_prop, out, out_count,
                  zero_word);
    launched = true;
  } else {
    const uint32_t* in = h.ws<uint32_t>(h.cc_list ? WS_ELIST1 : WS_ELIST0, m);
    uint32_t* out = h.ws<uint32_t>(h.cc_list ? WS_ELIST0 : WS_ELIST1, m);
    if (h.cc_active > 0) {
      launch_hook_k(h, mode, h.g.edges, h.cc_active, eb, in, rep, slot, any_prop, out, out_count,
                    zero_word);
      launched = true;
    }
  }
  if (zero_word && !launched) CK(cudaMemsetAsync(zero_word, 0, sizeof(*zero_word), h.stream));
}
void cc_round_done(Handle& h, int64_t out_count) {
  if (h.cc_round >= 1 && h.cc_round >= h.cc_filter_from && h.g.m > 0) {
    if (h.cc_active >= 0) h.cc_list ^= 1;
    h.cc_active = out_count;
  }
  ++h.cc_round;
}
bool round0_keys_from_edges(Handle& h, unsigned long long* slot);
void launch_round0_keys(Handle& h, unsigned long long* slot);

void cc_reset_rounds(Handle& h) {
  h.cc_lazy = false;
  h.cc_round = 0;
  h.cc_active = -1;
  h.cc_list = 0;
  // Active-edge filtering records the edges a round still saw crossing; on
  // a dense graph the first hook round sees most edges cross the round-0
  // trees (RMAT-24: 219M of 260M), so its list costs more to write and to
  // gather from than a second full pass over the edge stream: start the
  // lists one round later there (RSTG_CC_FILTER_FROM overrides: 1 or 2).
  static const int forced = [] {
    const char* e = getenv("RSTG_CC_FILTER_FROM");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  h.cc_filter_from = forced ? forced : (h.g.m > 4 * h.g.n ? 2 : 1);
}

void launch_apply(Handle& h, int32_t* rep, unsigned long long* slot, uint8_t* tflag,
                  uint32_t e_base, uint32_t m_local, unsigned long long* counter,
                  uint32_t* tlist) {
  k_apply<<<grid_for(h.g.n), kBlock, 0, h.stream>>>(h.g.n, rep, slot, tflag, e_base, m_local,
                                                     counter, tlist);
  CK_LAUNCH();
  h.stats.step(h.g.n);
}

// Lazy-mode apply (cc_forest.cpp:39-46) over the current roots only: a
// root with a proposal takes its winner (rep[r] = winner, slot reset, tree
// edge recorded / linked); the others stay roots for the next round.
// list == nullptr: the roots are all vertices [0, n).
__global__ void __launch_bounds__(kBlock)
    k_apply_roots(const uint32_t* __restrict__ list, const unsigned long long* count, int64_t n,
                  int32_t* rep, RoundIO io, uint32_t* out_list, unsigned long long* out_count,
                  unsigned long long* zero2) {
  const int64_t R = list ? (int64_t)*count : n;
  // the next hook round's counters (crossing count, any-proposal flag): the
  // host has read them already
  if (zero2 && blockIdx.x == 0 && threadIdx.x < 2) zero2[threadIdx.x] = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  __shared__ uint32_t s_n, s_h;
  __shared__ unsigned long long s_b;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < R; b += stride) {
    if (threadIdx.x == 0) s_n = s_h = 0;
    __syncthreads();
    const int64_t i = b + threadIdx.x;
    bool keep = false;
    uint32_t r = 0;
    if (i < R) {
      r = list ? list[i] : (uint32_t)i;
      const unsigned long long key = io.slot[r];
      if (key == kKeyInf) {
        keep = true;
      } else {
        rep[r] = (int32_t)(key >> 32);
        io.slot[r] = kKeyInf;
        const uint32_t e = (uint32_t)key - io.e_base;
        if (io.tflag && e < io.m_local) io.tflag[e] = 1;
        if (io.link) {
          const int2 ab = io.edges[e];
          link_tree_edge(io.eu, r, (uint32_t)ab.x, (uint32_t)ab.y, e);
        }
        atomicAdd(&s_h, 1u);
      }
    }
    const uint32_t pos = keep ? atomicAdd(&s_n, 1u) : 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
      s_b = s_n ? atomicAdd(out_count, (unsigned long long)s_n) : 0ull;
      if (s_h) atomicAdd(io.counter, (unsigned long long)s_h);
    }
    __syncthreads();
    if (keep) out_list[s_b + pos] = r;
    __syncthreads();
  }
}

void launch_cc_init(Handle& h, int32_t* rep, unsigned long long* slot) {
  k_cc_init<<<grid_for(h.g.n), kBlock, 0, h.stream>>>(h.g.n, rep, slot);
  CK_LAUNCH();
  h.stats.step(h.g.n);
}

// ---- the tail rounds, on the device ---------------------------------------
// Once few edges still cross (meshes: a few thousand after the first hook
// round) and the round-0 roots list is short, a round's kernels take a few
// microseconds and its host round trip (the counter read, then the next
// launches) takes longer than they do. The tail runs all remaining rounds
// in ONE cooperative launch with the same steps as the host loop -- apply
// over the current roots, the round-0 roots jump (block 0, in shared
// memory), the next filtered lazy hook -- a grid barrier between steps and
// the stop decision (no proposal) on the device. Proposals, hooks and
// labels are those of the host loop: only the order of list entries
// differs, which no result depends on.
constexpr int kTailThreads = 1024;
constexpr int64_t kTailMaxEdges = int64_t{1} << 20;
struct TailArgs {
  RoundIO io;                   // apply: slot, tflag, edges, link, eu; io.counter = hooks total
  int32_t* rep;
  uint32_t* elist[2];           // crossing-edge lists (ping-pong); round r's in elist[cur]
  unsigned long long* lcount;   // their lengths (2 words): lcount[cur] = first_count
  int64_t first_count;
  int cur;
  uint32_t* rl[3];              // roots lists: [0] the round-0 roots, [1], [2] current
  unsigned long long* rcount;   // their lengths (dev_box[20..22])
  int in;                       // the list round r's apply reads (0, 1 or 2)
  int mode;                     // round r + 1's hook mode
  int* any;                     // proposal flag (dev_box[2])
  unsigned long long* out;      // [0] hook rounds run, [1] hooks of the last productive
                                // round, [2] rounds exhausted flag
  int64_t rounds_left;          // (cc_forest.cpp:88: the round cap)
  unsigned long long hooks_before;  // hooks applied before round r's apply
  // speculative launch (right after round r's hook, before the host reads
  // its counters): the counts come from the device and the tail runs only
  // if round r proposed, the round-0 roots list is short and few edges
  // cross (out[3] = 1 when it ran)
  bool speculative;
  const unsigned long long* cross_dev;  // round r's crossing count (dev_box[1])
  int64_t max_cross;
};

// appends v to list/count with one atomic per warp
__device__ __forceinline__ void warp_append(bool keep, uint32_t v, uint32_t* list,
                                            unsigned long long* count) {
  const unsigned ball = __ballot_sync(0xffffffffu, keep);
  if (!ball) return;
  const int lane = threadIdx.x & 31, leader = __ffs(ball) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(ball));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (keep) list[base + __popc(ball & ((1u << lane) - 1u))] = v;
}

__global__ void __launch_bounds__(kTailThreads, 1) k_cc_tail(TailArgs a) {
  extern __shared__ uint32_t jump_smem[];  // block 0's roots jump
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  int in = a.in, cur = a.cur, mode = a.mode;
  unsigned long long rounds = 0, last_hooks = 0, hooks_before = a.hooks_before;
  unsigned long long first = (unsigned long long)a.first_count;
  if (a.speculative) {
    const bool go = *(volatile int*)a.any != 0 &&
                    *(volatile unsigned long long*)&a.rcount[0] <= (unsigned long long)kJumpSmallMax &&
                    *(volatile const unsigned long long*)a.cross_dev <= (unsigned long long)a.max_cross;
    if (gtid == 0) a.out[3] = go ? 1 : 0;
    if (!go) return;  // (uniform: every thread read the same words)
    first = *(volatile const unsigned long long*)a.cross_dev;
    hooks_before = *(volatile unsigned long long*)a.io.counter;
    grid.sync();  // (every thread has read the counters before any apply adds)
  }
  if (gtid == 0) {
    a.lcount[cur] = first;  // (read two barriers later)
    a.out[2] = 0;
  }
  for (;;) {
    // ---- apply (cc_forest.cpp:39-46) over the current roots
    const int out = in == 1 ? 2 : 1;
    {
      const int64_t R = (int64_t)*(volatile unsigned long long*)&a.rcount[in];
      const uint32_t* list = a.rl[in];
      uint32_t hooked = 0;
      for (int64_t b = gtid - (threadIdx.x & 31); b < R; b += gsize) {  // (warp-uniform trips)
        const int64_t i = b + (threadIdx.x & 31);
        bool keep = false;
        uint32_t r = 0;
        if (i < R) {
          r = list[i];
          const unsigned long long key = a.io.slot[r];
          if (key == kKeyInf) {
            keep = true;
          } else {
            a.rep[r] = (int32_t)(key >> 32);
            a.io.slot[r] = kKeyInf;
            const uint32_t e = (uint32_t)key - a.io.e_base;
            if (a.io.tflag && e < a.io.m_local) a.io.tflag[e] = 1;
            if (a.io.link) {
              const int2 ab = a.io.edges[e];
              link_tree_edge(a.io.eu, r, (uint32_t)ab.x, (uint32_t)ab.y, e);
            }
            ++hooked;
          }
        }
        warp_append(keep, r, a.rl[out], &a.rcount[out]);
      }
      for (int o = 16; o > 0; o >>= 1) hooked += __shfl_xor_sync(0xffffffffu, hooked, o);
      if ((threadIdx.x & 31) == 0 && hooked) atomicAdd(a.io.counter, (unsigned long long)hooked);
    }
    grid.sync();
    // ---- the round-0 roots jump (block 0); the next round's counters zeroed
    if (blockIdx.x == 0) {
      jump_small_block(a.rl[0], &a.rcount[0], a.rep, jump_smem);
    } else if (blockIdx.x == 1 && threadIdx.x == 0) {
      a.lcount[cur ^ 1] = 0;
      *a.any = 0;
      if (in != 0) a.rcount[in] = 0;  // (the list just consumed is the next output)
    }
    {
      const unsigned long long t = *(volatile unsigned long long*)a.io.counter;  // (after the barrier)
      last_hooks = t - hooks_before;
      hooks_before = t;
    }
    grid.sync();
    // ---- the next hook round (lazy: roots found by walking up), over the
    // edges the previous round saw crossing
    {
      const int64_t M = (int64_t)*(volatile unsigned long long*)&a.lcount[cur];
      const uint32_t* el = a.elist[cur];
      bool proposed = false;
      for (int64_t b = gtid - (threadIdx.x & 31); b < M; b += gsize) {
        const int64_t i = b + (threadIdx.x & 31);
        bool cross = false;
        uint32_t idx = 0;
        if (i < M) {
          idx = el[i];
          const int2 e = a.io.edges[idx];
          const int32_t ru = find_root(a.rep, e.x), rv = find_root(a.rep, e.y);
          if (ru != rv) {
            cross = true;
            const int32_t lo = min(ru, rv), hi = max(ru, rv);
            const int32_t winner = mode == 0 ? lo : hi, loser = mode == 0 ? hi : lo;
            const unsigned long long key = pack_key((uint32_t)winner, a.io.e_base + idx);
            if (key < a.io.slot[loser]) atomicMin(&a.io.slot[loser], key);
          }
        }
        proposed |= cross;
        warp_append(cross, idx, a.elist[cur ^ 1], &a.lcount[cur ^ 1]);
      }
      if (__any_sync(0xffffffffu, proposed) && (threadIdx.x & 31) == 0) *a.any = 1;
    }
    grid.sync();
    ++rounds;
    if (*(volatile int*)a.any == 0) break;  // a round without proposals (cc_forest.cpp:91)
    if ((int64_t)rounds >= a.rounds_left) {
      if (gtid == 0) a.out[2] = 1;
      break;
    }
    cur ^= 1;
    in = out;
    mode ^= 1;
  }
  if (gtid == 0) {
    a.out[0] = rounds;
    a.out[1] = last_hooks;
  }
}

// Edge-partitioned rounds (multi-GPU): the proposals of
// every rank's local edges are MIN-combined before each apply --
// combine_min (cc_forest.cpp:34) across ranks. Round 0 exchanges the dense
// slot array (every vertex may get a key); later rounds only the slots of
// the current roots, gathered in roots-list order (the list is replicated:
// identical on every rank), so the exchange shrinks with the roots.
__global__ void k_gather_slots(const uint32_t* __restrict__ list, int64_t count,
                               const unsigned long long* __restrict__ slot,
                               unsigned long long* buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = slot[list[i]];
}
__global__ void k_scatter_slots(const uint32_t* __restrict__ list, int64_t count,
                                const unsigned long long* __restrict__ buf,
                                unsigned long long* slot, int* any) {
  bool a = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = buf[i];
    slot[list[i]] = k;
    a |= k != kKeyInf;
  }
  if (__any_sync(0xffffffffu, a) && (threadIdx.x & 31) == 0) *any = 1;
}
__global__ void k_any_slot(int64_t n, const unsigned long long* __restrict__ slot, int* any) {
  bool a = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a |= slot[i] != kKeyInf;
  if (__any_sync(0xffffffffu, a) && (threadIdx.x & 31) == 0) *any = 1;
}
static void exchange(Handle& h, const CcExchange& ex, int which, int64_t count) {
  if (count <= 0) return;
  // the caller's collective is enqueued on the handle's stream (the
  // caller sets it: rstg_set_stream) after the proposals
  if (ex.reduce_min(ex.ctx, which, count) != 0) throw AlgoError("slot exchange failed");
}

// PR-RST's first graft round from the CSR (pr.cu): the same round 0 as the
// CC's (min-mode proposals over singleton reps = each vertex's first
// neighbour), fused with its apply and shortcutting, with the graft's
// reversal (singleton paths: parent[v] = u) done on the way. Returns the
// grafts; the vertices left as roots go to `roots` (count in *nroots).
int64_t pr_round0(Handle& h, int32_t* rep, int32_t* parent, const uint32_t* pos, uint32_t* q0,
                  uint32_t* roots, unsigned long long* nroots) {
  const int64_t n = h.g.n;
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(h.dev_box);
  RoundIO io{};
  io.e_base = (uint32_t)h.g.e_base;
  io.m_local = (uint32_t)h.g.m;
  io.counter = counter;
  io.offsets = h.g.offsets;
  io.nbrs = h.g.nbrs;
  io.arc_edge = h.g.arc_edge;
  io.edges = h.g.edges;
  io.roots = roots;
  io.nroots = nroots;
  io.pr_parent = parent;
  io.pr_pos = pos;
  io.pr_q0 = q0;
  ZeroRanges z{};
  z.add(counter, sizeof(unsigned long long));
  z.add(nroots, sizeof(unsigned long long));
  resolve_round(h, rep, n, kSrcRound0, io, &z);
  h.read_box(h.dev_box, 1);
  return h.host_box[0];
}

int64_t cc_exact(Handle& h, int32_t* rep, uint8_t* tflag, const EulerIO* euler,
                 const CcExchange* ex) {
  const int64_t n = h.g.n, m = h.g.m;
  unsigned long long* slot = ex ? ex->slot : h.ws<unsigned long long>(WS_SLOT, n);
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(h.dev_box);
  bool keyed, keys_from_edges = false;
  if (ex) {
    keys_from_edges = true;
    // every rank's round-0 keys (local edges, global ids), MIN-combined
    k_cc_init<<<grid_for(n), kBlock, 0, h.stream>>>(n, nullptr, slot);
    CK_LAUNCH();
    if (m > 0) launch_round0_keys(h, slot);
    exchange(h, *ex, 0, n);
    keyed = n > 0;
  } else {
    // round 0 from the keys the edge upload left in the slots, else (no
    // CSR built) from keys recomputed over the edge list, else the CSR
    const bool upload_keys = h.round0_slots == slot && m > 0;
    keys_from_edges = !upload_keys && round0_keys_from_edges(h, slot);
    keyed = upload_keys || keys_from_edges;
  }
  h.round0_slots = nullptr;
  const bool round0 = keyed || (h.g.has_csr() && m > 0);  // writes every rep itself
  const bool slots_ok = keyed || (h.slots_clean == slot && n <= h.slots_clean_n);
  if (!ex) h.slots_clean = nullptr;  // until this build completes
  h.timer.begin(h.stream, "cc.init", (round0 ? 0.0 : 4.0 * n) + (slots_ok ? 0.0 : 8.0 * n));
  if (!round0 || !slots_ok) {
    k_cc_init<<<grid_for(n), kBlock, 0, h.stream>>>(n, round0 ? nullptr : rep,
                                                     slots_ok ? nullptr : slot);
    CK_LAUNCH();
  }
  // the init step (cc_forest.cpp:82) counts whether or not it had work left
  h.stats.step(n, (!round0 || !slots_ok) ? 1 : 0);
  if (tflag && m > 0) CK(cudaMemsetAsync(tflag, 0, (size_t)m, h.stream));
  // the counters of the build: [0] hooks, [1] crossing, [2] any proposal,
  // [20..22] roots counts -- zeroed in one launch (with round 0's exit-set
  // state when round 0 runs)
  ZeroRanges zc{};
  zc.add(counter, 3 * sizeof(unsigned long long));
  zc.add(counter + 20, 3 * sizeof(unsigned long long));
  h.timer.end(h.stream);
  int mode = 0;  // HookMode::kMin first (cc_forest.cpp:87)
  int* any = reinterpret_cast<int*>(h.dev_box + 2);
  // roots lists: [0] the round-0 roots (kept: every former root), [1] and
  // [2] the current roots, ping-pong
  uint32_t* rlist = h.ws<uint32_t>(WS_CCROOTS, 3 * n + 3);
  uint32_t* rl[3] = {rlist, rlist + n + 1, rlist + 2 * n + 2};
  // dev_box [20] round-0 roots, [21] current roots in, [22] out
  unsigned long long* rcount = reinterpret_cast<unsigned long long*>(h.dev_box) + 20;
  RoundIO io{slot, tflag, (uint32_t)h.g.e_base, (uint32_t)m, counter, h.g.offsets, h.g.nbrs,
             h.g.arc_edge, h.g.edges, euler != nullptr, euler ? *euler : EulerIO{}, rl[0], rcount,
             keys_from_edges};
  cc_reset_rounds(h);
  int64_t round = 0;
  if (round0) {
    // round 0 (min mode over singleton reps) straight from the CSR (or the
    // upload's keys), fused with its apply and shortcutting
    // offsets, first neighbour, rep; a tree edge (arc head 4 B + successors 8 B) per vertex
    h.timer.begin(h.stream, "cc.round0", 4.0 * (n + 1) + 8.0 * n + (euler ? 12.0 * n : 0.0));
    resolve_round(h, rep, n, keyed ? kSrcRound0Slot : kSrcRound0, io, &zc);
    zc.k = 0;
    h.timer.end(h.stream);
    cc_round_done(h, 0);
    round = 1;
    mode = 1;
  }
  // Rounds >= 1 run lazy: no compression pass per round (hooks find roots,
  // apply touches the current roots only), one find pass at the end.
  const bool have_r0 = round == 1;  // round 0 collected the roots
  if (zc.k) {  // (no round 0: the counters still need their zeros)
    k_zero_ranges<<<1, 32, 0, h.stream>>>(zc);
    CK_LAUNCH();
  }
  // roots list rl[i] has its count in rcount[i]; apply reads list `in`
  // and writes list `out` (1 and 2 alternate after the round-0 list)
  const uint32_t* in_list = have_r0 ? rl[0] : nullptr;  // nullptr: all vertices
  int in = 0, out = 1;
  auto compress = [&]() {
    if (have_r0)
      compress_via_roots(h, rep, n, rl[0], rcount);
    else
      resolve_round(h, rep, n, kSrcRep, RoundIO{});
  };
  h.cc_lazy = false;  // the first hook sees compressed reps (round 0 compressed, or singletons)
  static const bool jump_roots = [] {
    const char* e = getenv("RSTG_CC_JUMP_ROOTS");
    return e ? atoi(e) != 0 : true;
  }();
  int64_t total = 0, last_hooks = 0, prev_total = 0, tail_last_hooks = -1;
  // the device-side tail rounds (k_cc_tail)
  static const bool tail_on = [] {
    const char* e = getenv("RSTG_CC_TAIL");
    return e ? atoi(e) != 0 : true;
  }();
  auto tail_args = [&](int64_t first_count, int cur, int in_idx, int next_mode,
                       int64_t hooks_before, int64_t at_round, bool speculative) {
    unsigned long long* box = reinterpret_cast<unsigned long long*>(h.dev_box);
    TailArgs ta{};
    ta.io = io;
    ta.rep = rep;
    ta.elist[0] = h.ws<uint32_t>(WS_ELIST0, m);
    ta.elist[1] = h.ws<uint32_t>(WS_ELIST1, m);
    ta.lcount = box + 24;
    ta.first_count = first_count;
    ta.cur = cur;
    ta.rl[0] = rl[0];
    ta.rl[1] = rl[1];
    ta.rl[2] = rl[2];
    ta.rcount = rcount;
    ta.in = in_idx;
    ta.mode = next_mode;
    ta.any = any;
    ta.out = box + 26;
    ta.rounds_left = std::max<int64_t>(n + 1 - at_round, 1);
    ta.hooks_before = (unsigned long long)hooks_before;
    ta.speculative = speculative;
    ta.cross_dev = box + 1;
    ta.max_cross = std::min<int64_t>(kTailMaxEdges, n / 4);
    return ta;
  };
  auto launch_tail = [&](TailArgs& ta) {
    ensure_dyn_smem((const void*)k_cc_tail, kJumpSmallSmem);
    void* args[] = {(void*)&ta};
    // (one block per SM: measured on road, 8 or 32 blocks cost more than
    // the cheaper barriers save -- the lazy finds need the parallelism)
    static const int tail_blocks_env = [] {
      const char* e = getenv("RSTG_CC_TAIL_BLOCKS");
      return e ? atoi(e) : 0;
    }();
    const int blocks = tail_blocks_env > 0 ? std::min(tail_blocks_env, num_sms()) : num_sms();
    CK(cudaLaunchCooperativeKernel((void*)k_cc_tail, dim3(blocks), dim3(kTailThreads), args,
                                   kJumpSmallSmem, h.stream));
  };
  for (;; ++round) {
    if (round > n + 1) {
      h.cc_lazy = false;
      throw AlgoError("hooking failed to converge");
    }
    // (counter[1], counter[2] are zero here: the build's zeroing, then each apply)
    // compulsory: each visited edge 8 B (+ 4 B list entry when filtered),
    // the rep array once (4 B per vertex, at most two gathers per edge),
    // 4 B per crossing edge appended (added once the count is read)
    const bool filtered = h.cc_round >= 2 && h.cc_active >= 0;
    const double visited = filtered ? (double)h.cc_active : (double)m;
    const char* hook_phase = mode == 0 ? "cc.hook_min" : "cc.hook_max";
    h.timer.begin(h.stream, hook_phase,
                  visited * (filtered ? 12.0 : 8.0) + std::min(4.0 * n, 8.0 * visited));
    // (the hook clears the count this round's apply appends to)
    cc_hook_round(h, mode, rep, slot, counter + 1, any, rcount + out);
    h.timer.end(h.stream);
    // The first listed round on a sparse graph: launch the device-side tail
    // right away; it checks its own conditions on the device and returns at
    // once when they fail, so the host reads this round's counters once.
    const bool spec_tail = tail_on && !ex && have_r0 && jump_roots && h.cc_round == 1 &&
                           h.cc_filter_from == 1 && m > 0;
    TailArgs ta{};
    if (spec_tail) {
      h.timer.begin(h.stream, "cc.tail", 0.0);
      ta = tail_args(-1, /*cur=*/0, in, mode ^ 1, total, round, true);
      launch_tail(ta);
      h.timer.end(h.stream);
    }
    // hooks so far, crossing, any; [20] the round-0 roots count, [20 + in]
    // the current roots count (same read)
    h.read_box(reinterpret_cast<int64_t*>(counter), spec_tail ? 30 : 23);
    if (spec_tail && h.host_box[29]) {  // the tail ran every remaining round
      if (h.host_box[28]) {
        h.cc_lazy = false;
        throw AlgoError("hooking failed to converge");
      }
      total = h.host_box[0];
      tail_last_hooks = h.host_box[27];
      h.stats.rounds = round + 1 + h.host_box[26];
      h.stats.step(n, 1);
      for (int64_t t = 0; t < h.host_box[26]; ++t) h.stats.step(n, 0);
      h.cc_lazy = true;
      break;
    }
    if (h.cc_round >= 1 && m > 0) h.timer.add_bytes(hook_phase, 4.0 * h.host_box[1]);
    const int64_t r0_count = have_r0 ? h.host_box[20] : 0;
    const int64_t cur_roots = have_r0 ? h.host_box[20 + in] : n;
    prev_total = total;
    total = h.host_box[0];
    bool proposed = h.host_box[2] != 0;
    if (ex) {
      // proposals of all ranks (they target current roots only), then the
      // global "any proposal" decides the stop on every rank alike
      h.timer.begin(h.stream, "cc.exchange", 16.0 * cur_roots);
      CK(cudaMemsetAsync(any, 0, sizeof(int), h.stream));
      if (have_r0) {
        const int64_t R = h.host_box[20 + in];
        if (R > 0) {
          // the roots list is filled by atomics (tile / block order varies
          // from rank to rank): sort it by id so position i names the same
          // root on every rank
          uint32_t* list = const_cast<uint32_t*>(in_list);
          uint32_t* sorted = h.ws<uint32_t>(WS_XSORT, R);
          int bits = 1;
          while (bits < 32 && (int64_t{1} << bits) < n) ++bits;
          size_t temp = 0;
          CK(cub::DeviceRadixSort::SortKeys(nullptr, temp, list, sorted, (int)R, 0, bits, h.stream));
          void* tmp = h.ws(WS_XTMP, temp);
          CK(cub::DeviceRadixSort::SortKeys(tmp, temp, list, sorted, (int)R, 0, bits, h.stream));
          CK(cudaMemcpyAsync(list, sorted, R * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h.stream));
          k_gather_slots<<<grid_for(R), kBlock, 0, h.stream>>>(in_list, R, slot, ex->xbuf);
          CK_LAUNCH();
          exchange(h, *ex, 1, R);
          k_scatter_slots<<<grid_for(R), kBlock, 0, h.stream>>>(in_list, R, ex->xbuf, slot, any);
          CK_LAUNCH();
        }
      } else {
        exchange(h, *ex, 0, n);
        k_any_slot<<<grid_for(n), kBlock, 0, h.stream>>>(n, slot, any);
        CK_LAUNCH();
      }
      h.timer.end(h.stream);
      h.read_box(reinterpret_cast<int64_t*>(counter) + 2, 1);
      proposed = *reinterpret_cast<int*>(h.host_box) != 0;
    }
    if (getenv("RSTG_CC_DEBUG"))
      fprintf(stderr, "cc round %lld mode %d: visited %.0f, hooks so far %lld, crossing %lld, lazy %d, r0 %lld\n",
              (long long)round, mode, visited, (long long)total, (long long)h.host_box[1], (int)h.cc_lazy,
              (long long)r0_count);
    cc_round_done(h, h.host_box[1]);
    h.stats.rounds = round + 1;
    // a round without proposals applies nothing (cc_forest.cpp:91)
    if (!proposed) break;
    // the remaining rounds on the device (see k_cc_tail) once they are small
    if (tail_on && !ex && have_r0 && jump_roots && r0_count <= kJumpSmallMax && h.cc_active >= 0 &&
        h.cc_active <= kTailMaxEdges && h.cc_active <= n / 4) {
      // per round: the crossing list read and rewritten (4 + 4 B), each edge
      // 8 B and its two roots (~4 B each), the current roots' slots (16 B)
      h.timer.begin(h.stream, "cc.tail", 24.0 * (double)h.cc_active + 16.0 * (double)cur_roots);
      TailArgs tb = tail_args(h.cc_active, h.cc_list, in, mode ^ 1, total, round, false);
      launch_tail(tb);
      h.timer.end(h.stream);
      h.read_box(h.dev_box, 29);
      const int64_t tail_rounds = h.host_box[26];
      if (h.host_box[28]) {
        h.cc_lazy = false;
        throw AlgoError("hooking failed to converge");
      }
      total = h.host_box[0];
      tail_last_hooks = h.host_box[27];
      h.stats.rounds = round + 1 + tail_rounds;
      h.stats.step(n, 1);
      for (int64_t t = 0; t < tail_rounds; ++t) h.stats.step(n, 0);
      h.cc_lazy = true;
      break;
    }
    // per current root: list entry 4 B, slot 8 B, rep or next-list entry 4 B
    h.timer.begin(h.stream, "cc.apply", 16.0 * cur_roots);
    k_apply_roots<<<grid_for(n), kBlock, 0, h.stream>>>(in_list, rcount + in, n, rep, io, rl[out],
                                                        rcount + out, counter + 1);
    CK_LAUNCH();
    h.stats.step(n);
    in_list = rl[out];
    in = out;
    out = out == 1 ? 2 : 1;
    h.timer.end(h.stream);
    mode ^= 1;
    // Lazy finds cost extra gathers per active edge endpoint; while many
    // edges are still active one compression pass over n is cheaper (the
    // two-level resolve: hook chains of one round may be long).
    if (h.cc_active < 0 || h.cc_active > n / 4) {  // (-1: no list yet, every edge active)
      h.timer.begin(h.stream, "cc.compress", 8.0 * n);
      compress();
      h.timer.end(h.stream);
      h.cc_lazy = false;
    } else {
      h.cc_lazy = true;
      // Hooks of one round chain roots to roots (a winner may itself have
      // been hooked), so lazy finds would walk those chains from every
      // active edge. Every chain runs through round-0 roots only: jumping
      // that list (one cooperative launch, no pass over n) leaves every
      // vertex at most two hops from its root.
      // A short list (meshes: a few thousand local minima) is jumped by one
      // CTA, with block barriers instead of grid barriers.
      if (have_r0 && jump_roots && total > prev_total) {
        h.timer.begin(h.stream, "cc.jump_roots", 8.0 * r0_count);
        if (r0_count <= kJumpSmallMax) {
          ensure_dyn_smem((const void*)k_jump_small, kJumpSmallSmem);
          k_jump_small<<<1, 1024, kJumpSmallSmem, h.stream>>>(rl[0], rcount, rep);
          CK_LAUNCH();
          h.stats.step(n);
        } else {
          jump_list(h, rep, n, rl[0], rcount);
        }
        h.timer.end(h.stream);
      }
    }
    last_hooks = -total;  // completed when the next round reads the hook total
  }
  last_hooks = tail_last_hooks >= 0 ? tail_last_hooks : last_hooks + total;
  // Labels left lazy by the last productive round: the Euler vertex pass
  // resolves them itself with find_root when that round hooked few roots
  // (short chains); otherwise, and for every other caller, compress here.
  if (h.cc_lazy && (!euler || last_hooks > n / 64)) {
    h.timer.begin(h.stream, "cc.final", 8.0 * n);
    compress();
    h.timer.end(h.stream);
  }
  h.cc_lazy = false;
  h.stats.tree_edges = total;
  if (!ex) {
    h.slots_clean = slot;
    h.slots_clean_n = n;
  }
  return total;
}

void cc_labels_fast(Handle& h, int32_t* labels) { cc_exact(h, labels, nullptr, nullptr); }

}  // namespace rstg
