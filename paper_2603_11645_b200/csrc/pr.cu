// pr.cu -- PR-RST path-reversal rooted spanning tree (pr_rst.cpp:267-314).
//
// Rounds of {graft, mark, check, reverse, jump} exactly as the reference
// (graft_round :72-133, mark_paths :135-164, the check :281-288,
// reverse_paths :178-204, batched_jump :216-252), each on the B200 as a
// sweep over the set it concerns rather than over all n vertices:
//
//   graft     proposals: k_hook (shared with the CC, active-edge filtered);
//             resolve + update over the CURRENT ROOTS list only (a graft
//             proposal targets a root), which is compacted as it goes.
//   mark      the reference marks the path from each graft endpoint u to
//             its tree root by doubling over an n x L "special ancestor"
//             table rebuilt every round (:254-265) -- L full sweeps to
//             rebuild, L more to mark. Here the ancestor structure is a
//             randomised skip list over the parent forest: vertex v has
//             level lvl(v) = trailing ones of a hash of v (P[lvl >= k] =
//             2^-k), and ptr_k[v], for lvl(v) >= k, is v's nearest proper
//             ancestor of level >= k (or its tree root). Rebuilding level k
//             walks ptr_{k-1} from the n/2^k vertices of level >= k,
//             expected 2 hops each: O(n) work per round instead of O(n L).
//             The structure lives in POSITION space: vertices sorted by
//             descending level (ids ascending within a level), so level >= k
//             is the prefix [0, C_k) and ptr_k is a dense array of C_k
//             positions (level 0: the parent forest, n entries); a root
//             points at itself. All levels take ~2n words (192 MB on road,
//             not n x L = 2.4 GB), every level is written coalesced, and a
//             walk at level k >= 3 stays inside an L2-resident array.
//             Marking then touches only path vertices: an ascent from each
//             endpoint climbs the levels (expected O(log n) hops) to the
//             root, and a descent fills, level by level from the top, the
//             gaps between consecutive marked vertices of the level above
//             (expected O(1) hops per walker per level). The marked set is
//             exactly the reference's (all ancestors of each endpoint), kept
//             as per-level frontier queues in HBM.
//   check     over the grafted roots (each marked and still a root).
//   reverse   over the marked queues only.
//   jump      rep stays fully converged between rounds, so after a graft
//             only the grafted roots' pointers chain: they are pointer-
//             jumped as a list (one cooperative launch), then one gather
//             rep[v] = rep[rep[v]] -- the converged reps batched_jump ends
//             with, whatever the batch.
// Tree edges and converged reps equal the CC's (same proposals, same
// rounds); the parents are those of the reference's path reversals.
// The designated root's tree is re-rooted at the end (:298-303).
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include "engine.hpp"

namespace cg = cooperative_groups;

namespace rstg {

void cc_hook_round(Handle& h, int mode, const int32_t* rep, unsigned long long* slot,
                   unsigned long long* out_count, int* any_prop,
                   unsigned long long* zero_word = nullptr);
void cc_round_done(Handle& h, int64_t out_count);
void cc_reset_rounds(Handle& h);
void compress_via_roots(Handle& h, int32_t* rep, int64_t n, const uint32_t* roots,
                        const unsigned long long* nroots);
void launch_compress2(Handle& h, int32_t* rep, int64_t n);
int64_t pr_round0(Handle& h, int32_t* rep, int32_t* parent, const uint32_t* pos, uint32_t* q0,
                  uint32_t* roots, unsigned long long* nroots);

namespace {

constexpr int kMaxLvl = 31;        // levels 0..K, K <= 31 (n < 2^31)

// Device control block (u64 words in WS_BFS_CTRL).
enum PrCtl : int {
  P_NROOTS_IN = 0,  // current roots list length
  P_NROOTS_OUT,     // next roots list length
  P_NGRAFT,         // grafts this round (seeds / grafted roots)
  P_CROSSING,       // crossing edges of the graft proposals
  P_ANY,            // int: any proposal (block_flag)
  P_BAD_REV,        // int: reversal found a marked vertex with no source
  P_MCNT0 = 8,      // P_MCNT0 + b: marked vertices of exact level b
  P_NWORDS = P_MCNT0 + kMaxLvl + 2
};

__device__ __forceinline__ uint32_t vertex_level(uint32_t v, int K) {
  unsigned long long x = (unsigned long long)v + 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  x ^= x >> 31;
  return min((uint32_t)__ffsll((long long)~x) - 1u, (uint32_t)K);  // trailing ones
}
// (the identity forest: parent/rep unless the fused round 0 writes them;
// scratch/mark/slot unless the last build left them clean)
__global__ void k_pr_init(int64_t n, int K, int32_t* parent, int32_t* rep, int32_t* scratch,
                          uint8_t* mark, uint8_t* lv, unsigned long long* slot,
                          unsigned long long* hist) {
  __shared__ unsigned int s_h[kMaxLvl + 1];
  for (int i = threadIdx.x; i <= kMaxLvl; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (parent) parent[v] = rep[v] = (int32_t)v;
    if (scratch) {
      scratch[v] = -1;
      mark[v] = 0;
    }
    if (slot) slot[v] = kKeyInf;
    if (hist) {  // (the level order is being built: levels and their histogram)
      const uint32_t l = vertex_level((uint32_t)v, K);
      lv[v] = (uint8_t)l;
      atomicAdd(&s_h[l], 1u);
    }
  }
  __syncthreads();
  if (hist)
    for (int i = threadIdx.x; i <= K; i += blockDim.x)
      if (s_h[i]) atomicAdd(&hist[i], (unsigned long long)s_h[i]);
}

// Sort keys of the level order: descending level = ascending (K - level);
// a stable radix sort keeps ids ascending within a level, so level >= k is
// the prefix [0, C_k) of the result and its walks sweep ids in order.
__global__ void k_pr_level_keys(int64_t n, int K, const uint8_t* __restrict__ lv, uint32_t* keys,
                                uint32_t* ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    keys[v] = (uint32_t)(K - lv[v]);
    ids[v] = (uint32_t)v;
  }
}

// The level structure in position space (passed by value): C[k] = number
// of positions of level >= k (C[0] = n, C[K + 1] = 0); the level-k array
// (k = 0: parents) starts at off[k] of one buffer Q and covers [0, C[k]).
struct PrLv {
  uint32_t C[kMaxLvl + 2];
  unsigned long long off[kMaxLvl + 2];
  int K;
};
// level of position x (C in shared memory): levels are small (mean 1)
__device__ __forceinline__ int level_of_pos(const uint32_t* sC, int K, uint32_t x) {
  int l = 0;
  while (l < K && x < sC[l + 1]) ++l;
  return l;
}

// Levels k0 .. K of the rebuild in ONE cooperative launch (small levels:
// C_k below ~2^18 positions, L2-resident; a grid barrier between levels).
__global__ void __launch_bounds__(kBlock) k_pr_rebuild_tail(int k0, PrLv L, uint32_t* Q) {
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  for (int k = k0; k <= L.K && L.C[k] > 0; ++k) {
    const uint32_t* __restrict__ in = Q + L.off[k - 1];
    uint32_t* __restrict__ out = Q + L.off[k];
    const uint32_t lo = L.C[k], hi = L.C[k - 1];
    for (int64_t i = gtid; i < (int64_t)lo; i += gsize) {
      uint32_t x = ld_cg(&in[i]);  // (written by the previous level, this launch)
      while (x >= lo && x < hi) {
        const uint32_t y = ld_cg(&in[x]);
        if (y == x) break;
        x = y;
      }
      out[i] = x;
    }
    grid.sync();
  }
}

// pos[byl[i]] = i (once per graph size, with the level order)
__global__ void k_pr_pos(int64_t n, const uint32_t* __restrict__ byl, uint32_t* __restrict__ pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pos[byl[i]] = (uint32_t)i;
}

// Level 0 of the structure: the parent forest in positions (a root points
// at itself), Q0[i] = pos[parent[byl[i]]]. The identity at the start; every
// parent write after that (the first round's direct grafts, each reversal)
// updates its entry, so no rebuild pass over n is needed for it.
__global__ void k_pr_q0_identity(int64_t n, uint32_t* __restrict__ q0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    q0[i] = (uint32_t)i;
}

// Level k >= 1 for the positions [0, C[k]): walk the level-(k-1) pointers
// to the first position of level >= k, or to the tree root (a position at
// or past C[k-1] can only be a root: non-roots reached at level k-1 have
// level >= k-1; a root of level k-1 points at itself).
template <int kB>
__global__ void __launch_bounds__(kBlock)
    k_pr_rebuild(int k, PrLv L, uint32_t* __restrict__ Q) {
  const uint32_t* __restrict__ in = Q + L.off[k - 1];
  uint32_t* __restrict__ out = Q + L.off[k];
  const uint32_t cnt = L.C[k], lo = L.C[k], hi = L.C[k - 1];
  const int64_t g = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < cnt; i0 += kB * g) {
    uint32_t x[kB];
    bool walk[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int64_t i = i0 + j * g;
      x[j] = i < cnt ? in[i] : 0u;
      walk[j] = i < cnt;
    }
    // the walks of kB positions advance together (their loads in flight at once)
    for (;;) {
      bool any = false;
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if (!walk[j]) continue;
        if (x[j] < lo || x[j] >= hi) {
          walk[j] = false;
          continue;
        }
        const uint32_t y = in[x[j]];
        if (y == x[j]) walk[j] = false;
        else x[j] = y;
        any = true;
      }
      if (!any) break;
    }
#pragma unroll
    for (int j = 0; j < kB; ++j)
      if (i0 + j * g < cnt) out[i0 + j * g] = x[j];
  }
}

// Append x to the marked queue of its exact level (bucket b occupies
// [base_b, base_b + capacity_b) of mk: the descending-level layout of byl).
__device__ __forceinline__ void enqueue(uint32_t* mk, const unsigned long long* bbase,
                                        unsigned long long* mcnt, int b, int32_t x) {
  const unsigned long long p = atomicAdd(&mcnt[b], 1ull);
  mk[bbase[b] + p] = (uint32_t)x;
}

// graft_round resolve (pr_rst.cpp:112-122) over the current roots: root v
// with a proposal loses to the key's winner; u = the endpoint in v's tree
// (marked: it starts the path to reverse), w = the other (u's new parent).
// seeds[i] = u and grafted[i] = v share one index.
__global__ void k_pr_resolve(const uint32_t* __restrict__ list, const unsigned long long* cnt,
                             int64_t n, const int2* __restrict__ edges, uint32_t e_base,
                             const int32_t* __restrict__ rep, const unsigned long long* __restrict__ slot,
                             uint8_t* mark, int32_t* scratch, uint32_t* seeds, uint32_t* grafted,
                             unsigned long long* ngraft, int32_t* direct_parent,
                             const uint32_t* __restrict__ pos, uint32_t* __restrict__ q0) {
  const int64_t R = list ? (int64_t)*cnt : n;
  __shared__ uint32_t s_n;
  __shared__ unsigned long long s_b;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < R; b += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int64_t i = b + threadIdx.x;
    bool g = false;
    uint32_t v = 0;
    int32_t u = 0;
    if (i < R) {
      v = list ? list[i] : (uint32_t)i;
      const unsigned long long key = slot[v];
      if (key != kKeyInf) {
        const int2 uv = edges[(uint32_t)key - e_base];
        u = (rep[uv.x] == (int32_t)v) ? uv.x : uv.y;
        const int32_t w = (u == uv.x) ? uv.y : uv.x;
        if (direct_parent) {
          // the identity forest (no reversal yet): u = v is a singleton
          // tree, its path to reverse is u alone -- reverse_paths reduces
          // to parent[u] = w (no marking, no queues, no check needed)
          direct_parent[u] = w;
          q0[pos[u]] = pos[w];
        } else {
          mark[u] = 1;
          scratch[u] = w;
        }
        g = true;
      }
    }
    // one claim per block (round 0 grafts nearly every vertex)
    const uint32_t pos = g ? atomicAdd(&s_n, 1u) : 0u;
    __syncthreads();
    if (threadIdx.x == 0) s_b = s_n ? atomicAdd(ngraft, (unsigned long long)s_n) : 0ull;
    __syncthreads();
    if (g && !direct_parent) {
      seeds[s_b + pos] = (uint32_t)u;
      grafted[s_b + pos] = v;
    }
    __syncthreads();
  }
}

// graft_round update (pr_rst.cpp:123-128): rep = winner; the roots that did
// not graft form the next roots list.
__global__ void __launch_bounds__(kBlock)
    k_pr_update(const uint32_t* __restrict__ list, const unsigned long long* cnt, int64_t n,
                int32_t* rep, unsigned long long* slot, uint32_t* out_list,
                unsigned long long* out_cnt) {
  const int64_t R = list ? (int64_t)*cnt : n;
  __shared__ uint32_t s_n;
  __shared__ unsigned long long s_b;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < R; b += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int64_t i = b + threadIdx.x;
    bool keep = false;
    uint32_t v = 0;
    if (i < R) {
      v = list ? list[i] : (uint32_t)i;
      const unsigned long long key = slot[v];
      if (key == kKeyInf) {
        keep = true;
      } else {
        rep[v] = (int32_t)(key >> 32);
        slot[v] = kKeyInf;
      }
    }
    const uint32_t pos = keep ? atomicAdd(&s_n, 1u) : 0u;
    __syncthreads();
    if (threadIdx.x == 0) s_b = s_n ? atomicAdd(out_cnt, (unsigned long long)s_n) : 0ull;
    __syncthreads();
    if (keep) out_list[s_b + pos] = v;
    __syncthreads();
  }
}

// Marking, ascent: from each seed u climb to its tree root -- at level k
// (starting at lvl(u)) follow ptr_k; a vertex of a higher level lifts the
// climb to that level. Every vertex passed is on the path: marked and
// queued by its exact level. Seeds themselves are queued first, block-
// aggregated (round 0 has ~n/2 seeds, all singleton roots: `identity`,
// the forest before any reversal, needs no climb). Positions throughout;
// the vertex id (byl) is looked up only to mark and queue.
__global__ void __launch_bounds__(kBlock)
    k_pr_ascend(const uint32_t* __restrict__ seeds, const unsigned long long* nseeds,
                const uint32_t* __restrict__ Q, PrLv L, const uint32_t* __restrict__ byl,
                const uint32_t* __restrict__ pos, bool identity, uint8_t* mark, uint32_t* mk,
                const unsigned long long* __restrict__ bbase, unsigned long long* mcnt) {
  __shared__ unsigned int s_c[kMaxLvl + 1];
  __shared__ unsigned long long s_b[kMaxLvl + 1];
  __shared__ uint32_t sC[kMaxLvl + 2];
  for (int i = threadIdx.x; i < kMaxLvl + 2; i += blockDim.x) sC[i] = L.C[i];
  const int K = L.K;
  const int64_t S = (int64_t)*nseeds;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < S; b0 += (int64_t)gridDim.x * blockDim.x) {
    for (int i = threadIdx.x; i <= kMaxLvl; i += blockDim.x) s_c[i] = 0;
    __syncthreads();
    const int64_t i = b0 + threadIdx.x;
    int32_t u = -1;
    uint32_t c = 0;
    int l = 0;
    unsigned slot = 0;
    if (i < S) {
      u = (int32_t)seeds[i];
      c = pos[u];
      l = level_of_pos(sC, K, c);
      slot = atomicAdd(&s_c[l], 1u);
    }
    __syncthreads();
    for (int j = threadIdx.x; j <= kMaxLvl; j += blockDim.x)
      s_b[j] = s_c[j] ? atomicAdd(&mcnt[j], (unsigned long long)s_c[j]) : 0ull;
    __syncthreads();
    if (u >= 0) {
      mk[bbase[l] + s_b[l] + slot] = (uint32_t)u;
      int k = l;
      while (!identity) {
        const uint32_t x = Q[L.off[k] + c];  // ptr_k(c): c has level >= k
        if (x == c) break;                    // c is its tree's root
        const uint32_t vx = byl[x];
        mark[vx] = 1;
        const int lx = level_of_pos(sC, K, x);
        enqueue(mk, bbase, mcnt, lx, (int32_t)vx);
        if (x >= sC[k]) break;  // below level k: only the root is reached that way
        if (lx > k) k = lx;
        c = x;
      }
    }
    __syncthreads();
  }
}

// Marking, descent at level j: every marked vertex a of level > j walks
// ptr_j up to the next vertex of level > j (or the root), marking the
// level-j vertices of that gap (queued into bucket j, not read here).
__global__ void __launch_bounds__(kBlock)
    k_pr_descend(int j, const uint32_t* __restrict__ Q, PrLv L, const uint32_t* __restrict__ byl,
                 const uint32_t* __restrict__ pos, uint8_t* mark, uint32_t* mk,
                 const unsigned long long* __restrict__ bbase, unsigned long long* mcnt) {
  const int b = j + 1 + (int)blockIdx.y;  // this block row's bucket (level b > j)
  if (b > L.K) return;
  const int64_t T = (int64_t)mcnt[b];
  const uint32_t* q = mk + bbase[b];
  const uint32_t* __restrict__ in = Q + L.off[j];
  const uint32_t lo = L.C[j + 1], hi = L.C[j];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t pa = pos[q[i]];
    uint32_t x = in[pa];
    if (x == pa) continue;  // a root
    while (x >= lo && x < hi) {  // level exactly j (past hi: a lower root)
      const uint32_t y = in[x];
      if (y == x) break;  // the root (the ascent marked it)
      const uint32_t vx = byl[x];
      mark[vx] = 1;
      enqueue(mk, bbase, mcnt, j, (int32_t)vx);
      x = y;
    }
  }
}

// The top descent levels (K-1 .. jmin) in ONE block, a block barrier
// between levels: their walkers are few (a path holds ~2^-j of its
// vertices at level >= j), so one launch per level was launch latency.
__global__ void __launch_bounds__(1024)
    k_pr_descend_top(int jmin, const uint32_t* __restrict__ Q, PrLv L,
                     const uint32_t* __restrict__ byl, const uint32_t* __restrict__ pos,
                     uint8_t* mark, uint32_t* mk, const unsigned long long* __restrict__ bbase,
                     unsigned long long* mcnt) {
  __shared__ unsigned long long s_pre[kMaxLvl + 3];
  const int K = L.K;
  for (int j = K - 1; j >= jmin; --j) {
    if (threadIdx.x == 0) {  // walkers: buckets j+1 .. K
      unsigned long long acc = 0;
      for (int b = j + 1; b <= K; ++b) {
        s_pre[b] = acc;
        acc += *(volatile unsigned long long*)&mcnt[b];
      }
      s_pre[K + 1] = acc;
    }
    __syncthreads();
    const unsigned long long total = s_pre[K + 1];
    const uint32_t* __restrict__ in = Q + L.off[j];
    const uint32_t lo = L.C[j + 1], hi = L.C[j];
    for (unsigned long long t = threadIdx.x; t < total; t += blockDim.x) {
      int b = j + 1;
      while (b < K && t >= s_pre[b + 1]) ++b;
      const uint32_t a = mk[bbase[b] + (t - s_pre[b])];
      const uint32_t pa = pos[a];
      uint32_t x = in[pa];
      if (x == pa) continue;  // a root
      while (x >= lo && x < hi) {  // level exactly j
        const uint32_t y = in[x];
        if (y == x) break;
        const uint32_t vx = byl[x];
        mark[vx] = 1;
        enqueue(mk, bbase, mcnt, j, (int32_t)vx);
        x = y;
      }
    }
    __syncthreads();  // (level j's queue complete before level j - 1 reads it)
    __threadfence_block();
  }
}

// mark_path for ONE seed by walking the parents (level 0 of the skip
// structure, kept current by every parent write) -- the re-rooting's path
// when it is short: no rebuild of the stale upper levels for one path.
// Marks and queues exactly what the ascent + descent would (every ancestor
// of u, by exact level); *ok = 0 when the path is longer than `cap`.
__global__ void k_pr_short_path(int32_t u, const uint32_t* __restrict__ q0, PrLv L,
                                const uint32_t* __restrict__ byl, const uint32_t* __restrict__ pos,
                                uint8_t* mark, uint32_t* mk, const unsigned long long* __restrict__ bbase,
                                unsigned long long* mcnt, int cap, int* ok) {
  auto level_of = [&](uint32_t x) {
    int l = 0;
    while (l < L.K && x < L.C[l + 1]) ++l;
    return l;
  };
  uint32_t c = pos[u];
  enqueue(mk, bbase, mcnt, level_of(c), u);  // (the seed, as the ascent queues it)
  for (int hop = 0; hop < cap; ++hop) {
    const uint32_t x = q0[c];
    if (x == c) {  // c is the tree root
      *ok = 1;
      return;
    }
    const uint32_t vx = byl[x];
    mark[vx] = 1;
    enqueue(mk, bbase, mcnt, level_of(x), (int32_t)vx);
    c = x;
  }
  *ok = 0;
}

// mark_paths for every seed of a round by walking the parents (level 0 of
// the skip structure is always current), one thread per seed, when every
// path is short: the seeds' paths lie in different trees (one seed per
// grafted root), so they are disjoint and each vertex is queued once.
// *ok is cleared when some path is longer than `cap` (the caller then
// rebuilds the structure and marks by ascent and descent; the marks set
// here are a subset of those and are set again).
__global__ void k_pr_short_paths(const uint32_t* __restrict__ seeds,
                                 const unsigned long long* nseeds,
                                 const uint32_t* __restrict__ q0, PrLv L,
                                 const uint32_t* __restrict__ byl, const uint32_t* __restrict__ pos,
                                 uint8_t* mark, uint32_t* mk,
                                 const unsigned long long* __restrict__ bbase,
                                 unsigned long long* mcnt, int cap, int* ok) {
  auto level_of = [&](uint32_t x) {
    int l = 0;
    while (l < L.K && x < L.C[l + 1]) ++l;
    return l;
  };
  const int64_t S = (int64_t)*nseeds;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = (int32_t)seeds[i];
    uint32_t c = pos[u];
    enqueue(mk, bbase, mcnt, level_of(c), u);
    int hop = 0;
    for (; hop < cap; ++hop) {
      if (*(volatile int*)ok == 0) return;  // (another path was too long: give up early)
      const uint32_t x = q0[c];
      if (x == c) break;  // c is the tree root
      const uint32_t vx = byl[x];
      mark[vx] = 1;
      enqueue(mk, bbase, mcnt, level_of(x), (int32_t)vx);
      c = x;
    }
    if (hop == cap) *ok = 0;
  }
}

// The check (pr_rst.cpp:281-288): each grafted root is marked and still a
// root; records the smallest offending (r, u).
__global__ void k_pr_check(const uint32_t* __restrict__ grafted, const uint32_t* __restrict__ seeds,
                           const unsigned long long* ngraft, const uint8_t* mark,
                           const int32_t* parent, unsigned long long* bad) {
  const int64_t G = (int64_t)*ngraft;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < G;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = grafted[i];
    if (!mark[r] || parent[r] != (int32_t)r)
      atomicMin(bad, ((unsigned long long)r << 32) | seeds[i]);
  }
}

// reverse_paths (pr_rst.cpp:186-201) over the marked vertices only; block
// row y walks the queue of level y.
__global__ void k_pr_reverse_a(const uint32_t* mk, const unsigned long long* bbase,
                               const unsigned long long* mcnt, const int32_t* __restrict__ parent,
                               int32_t* scratch) {
  const int b = (int)blockIdx.y;
  const int64_t T = (int64_t)mcnt[b];
  const uint32_t* q = mk + bbase[b];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = (int32_t)q[i];
    const int32_t p = parent[v];
    if (p != v) scratch[p] = v;
  }
}
__global__ void k_pr_reverse_b(const uint32_t* mk, const unsigned long long* bbase,
                               const unsigned long long* mcnt, uint8_t* mark, int32_t* parent,
                               int32_t* scratch, int* bad_rev, const uint32_t* __restrict__ pos,
                               uint32_t* __restrict__ q0) {
  const int b = (int)blockIdx.y;
  const int64_t T = (int64_t)mcnt[b];
  const uint32_t* q = mk + bbase[b];
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = (int32_t)q[i];
    const int32_t s = scratch[v];
    if (s < 0) {
      bad = true;
      continue;
    }
    parent[v] = s;
    q0[pos[v]] = pos[s];  // (level 0 of the skip structure follows the parents)
    scratch[v] = -1;
    mark[v] = 0;
  }
  block_flag(bad, bad_rev);
}
__global__ void k_set_i32(int32_t* p, int32_t v) { *p = v; }
__global__ void k_set_u8(uint8_t* p, uint8_t v) { *p = v; }
__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }
__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

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

void pr_rst(Handle& h, int32_t root, int64_t jump_batch, int32_t* parent) {
  const int64_t n = h.g.n;
  const int K = std::min(std::max(ceil_log2_i(std::max<int64_t>(n, 1)), 1), kMaxLvl);
  int32_t* rep = h.ws<int32_t>(WS_REP, n);
  int32_t* scratch = h.ws<int32_t>(WS_PR_SCRATCH, n);
  uint8_t* mark = h.ws<uint8_t>(WS_PR_ONPATH, n);
  uint8_t* lv = h.ws<uint8_t>(WS_PR_FRESH, n);
  uint32_t* seeds = h.ws<uint32_t>(WS_PR_GU, n + 1);
  uint32_t* grafted = h.ws<uint32_t>(WS_PR_NEXT, n + 1);
  uint32_t* byl = h.ws<uint32_t>(WS_PR_BYL, n + 1);
  uint32_t* mk = h.ws<uint32_t>(WS_PR_MK, n + 1);
  uint32_t* pos = h.ws<uint32_t>(WS_PR_POS, n + 1);
  uint32_t* rlist = h.ws<uint32_t>(WS_CCROOTS, 3 * n + 3);
  uint32_t* rl[2] = {rlist, rlist + n + 1};
  unsigned long long* slot = h.ws<unsigned long long>(WS_SLOT, n);
  cc_reset_rounds(h);       // (graft rounds use the CC's active-edge lists)
  h.round0_slots = nullptr;  // (and overwrite an upload's round-0 keys)
  unsigned long long* pc =
      reinterpret_cast<unsigned long long*>(h.ws<unsigned long long>(WS_BFS_CTRL, P_NWORDS + 2 * (kMaxLvl + 2)));
  unsigned long long* bbase = pc + P_NWORDS;           // bucket b base in mk
  unsigned long long* cursor = bbase + (kMaxLvl + 2);  // histogram, then byl cursors
  unsigned long long* mcnt = pc + P_MCNT0;
  int* any = reinterpret_cast<int*>(pc + P_ANY);
  int* bad_rev = reinterpret_cast<int*>(pc + P_BAD_REV);
  unsigned long long* bad_mark = reinterpret_cast<unsigned long long*>(h.dev_box) + 16;
  const unsigned g = grid_for(n);
  const cudaStream_t s = h.stream;

  // ---- init: identity forest (make_pr_state :40-70) and vertex levels.
  // The level order (vertices sorted by descending level, ids ascending
  // within a level, so level-k walks sweep ids in order) and the counts C_k
  // depend on n only: built once per graph size, kept with the handle.
  // What a build leaves behind is the identity's state again for scratch
  // (-1), mark (0) and the slots (INF) -- every entry it sets is reset by the
  // reversal or the update that consumes it -- and the fused round 0 (a
  // built CSR) writes every parent and rep itself: the init writes only what
  // is not known to hold (nothing, on a repeated build of a CSR graph).
  const bool fused0 = h.g.has_csr() && !h.g.csr_pending && h.g.m > 0 && n > 0;
  const bool slots_ok = h.slots_clean == slot && n <= h.slots_clean_n;
  const bool marks_ok = h.pr_clean == scratch && h.pr_clean_mark == mark && n <= h.pr_clean_n;
  h.slots_clean = nullptr;  // graft rounds use the slots (clean again at the end)
  h.pr_clean = nullptr;
  h.timer.begin(s, "pr.init", (fused0 ? 0.0 : 8.0 * n) + (marks_ok ? 0.0 : 5.0 * n) +
                                  (slots_ok ? 0.0 : 8.0 * n));
  CK(cudaMemsetAsync(pc, 0, (P_NWORDS + 2 * (kMaxLvl + 2)) * sizeof(unsigned long long), s));
  const bool cached = h.pr_levels_n == n && h.pr_levels_byl == byl && (int)h.pr_levels_C.size() == K + 2;
  if (!cached || !fused0 || !marks_ok || !slots_ok) {
    k_pr_init<<<g, kBlock, 0, s>>>(n, K, fused0 ? nullptr : parent, rep, marks_ok ? nullptr : scratch,
                                   mark, lv, slots_ok ? nullptr : slot, cached ? nullptr : cursor);
    CK_LAUNCH();
  }
  CK(cudaMemsetAsync(bad_mark, 0xFF, sizeof(unsigned long long), s));
  unsigned long long* cbase = h.ws<unsigned long long>(WS_PR_CBASE, kMaxLvl + 2);
  if (!cached) {
    h.read_box(reinterpret_cast<int64_t*>(cursor), K + 1);
    std::vector<int64_t> C(K + 2, 0);  // C[k] = #level >= k
    for (int k = K; k >= 0; --k) C[k] = C[k + 1] + h.host_box[k];
    // bucket b of the marked queues (and level b of byl) starts at C[b+1]
    std::vector<unsigned long long> hb(kMaxLvl + 2, 0);
    for (int b = 0; b <= K; ++b) hb[b] = (unsigned long long)C[b + 1];
    CK(cudaMemcpy(cbase, hb.data(), hb.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    if (n > 0) {
      // stable radix sort of (K - level) over ids in order
      uint32_t* keys = h.ws<uint32_t>(WS_VAL_A, 2 * n);
      uint32_t* ids = reinterpret_cast<uint32_t*>(h.ws<uint32_t>(WS_VAL_B, 2 * n));
      k_pr_level_keys<<<g, kBlock, 0, s>>>(n, K, lv, keys, ids);
      CK_LAUNCH();
      int bits = 1;
      while ((1 << bits) <= K) ++bits;
      size_t temp = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys, keys + n, ids, byl, (int)n, 0, bits, s));
      void* tmp = h.ws(WS_SL, temp);
      CK(cub::DeviceRadixSort::SortPairs(tmp, temp, keys, keys + n, ids, byl, (int)n, 0, bits, s));
    }
    if (n > 0) {
      k_pr_pos<<<g, kBlock, 0, s>>>(n, byl, pos);
      CK_LAUNCH();
    }
    CK(cudaStreamSynchronize(s));
    h.pr_levels_C = C;
    h.pr_levels_n = n;
    h.pr_levels_byl = byl;
  }
  const std::vector<int64_t>& C = h.pr_levels_C;
  PrLv L{};
  L.K = K;
  {
    unsigned long long o = 0;
    for (int k = 0; k <= K + 1; ++k) {
      L.C[k] = (uint32_t)C[k];
      L.off[k] = o;
      o += (unsigned long long)C[k];
    }
  }
  // the skip structure in position space: level k (k = 0: parents) at
  // off[k], C[k] entries -- sum_k C[k] = n + the sum of the levels, about
  // 2n (sized exactly: the sum is random)
  uint32_t* Q = h.ws<uint32_t>(WS_PR_ANC, (size_t)L.off[K + 1] + 1);
  if (n > 0 && !fused0) {  // (the fused round 0 writes every level-0 entry)
    k_pr_q0_identity<<<g, kBlock, 0, s>>>(n, Q);
    CK_LAUNCH();
  }
  CK(cudaMemcpyAsync(bbase, cbase, (kMaxLvl + 2) * sizeof(unsigned long long),
                     cudaMemcpyDeviceToDevice, s));
  h.stats.step(n, 3);
  h.timer.end(s);

  // the skip structure lags the parent forest after a reversal; before the
  // first one the forest is the identity (every vertex its own root): the
  // first marking needs no structure at all
  bool forest_dirty = false, identity = true;
  auto rebuild = [&]() {
    h.timer.begin(s, "pr.rebuild", 0.0);
    double bytes = 0;  // (level 0 is kept current by the parent writes)
    // big levels one launch each; the small ones (C_k < 2^18) in one
    // cooperative launch (they were bound by launch latency)
    static const int64_t small_level = [] {
      const char* e = getenv("RSTG_PR_SMALL_LEVEL");
      return e ? atoll(e) : (int64_t{1} << 18);
    }();
    static int tail_blocks = 0;
    if (!tail_blocks) {
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pr_rebuild_tail, kBlock, 0));
      tail_blocks = std::max(1, std::min(per_sm, 4)) * num_sms();
    }
    for (int k = 1; k <= K && C[k] > 0; ++k) {
      // per position of level >= k: the level-(k-1) entry in (4 B), ~1 more
      // hop (4 B), the entry out (4 B)
      if (C[k] < small_level) {
        for (int kk = k; kk <= K && C[kk] > 0; ++kk) bytes += (double)C[kk] * 12.0;
        int k0 = k;
        void* args[] = {(void*)&k0, (void*)&L, (void*)&Q};
        CK(cudaLaunchCooperativeKernel((void*)k_pr_rebuild_tail, dim3(tail_blocks), dim3(kBlock),
                                       args, 0, s));
        h.stats.step(C[k]);
        break;
      }
      bytes += (double)C[k] * 12.0;
      (n > (int64_t{1} << 22) ? k_pr_rebuild<4> : k_pr_rebuild<1>)
          <<<grid_for(C[k]), kBlock, 0, s>>>(k, L, Q);
      h.stats.step(C[k]);
    }
    CK_LAUNCH();
    h.timer.add_bytes(bytes);
    h.timer.end(s);
    forest_dirty = false;
  };
  // marked set of one round: all ancestors of every seed (mark_paths :135-164)
  int64_t round_roots = n;  // roots before the current round's grafts (bounds its seeds)
  auto run_marking = [&]() {
    if (forest_dirty) {
      // Few grafts (a round with few roots left): every path walked on the
      // parents while they are all short, instead of rebuilding the stale
      // structure for a few paths. A walk that exceeds the cap stops them
      // all (bounded loss: cap hops) and the structure is rebuilt.
      const char* e = getenv("RSTG_PR_SHORT_PATHS");
      const int cap = e ? atoi(e) : 32;  // (road pr-rst 2.06 -> 1.77 ms; RMAT unchanged)
      const char* e2 = getenv("RSTG_PR_SHORT_PATHS_ROOTS");
      const int64_t max_roots = e2 ? atoll(e2) : 8192;
      if (cap > 0 && round_roots <= max_roots) {
        h.timer.begin(s, "pr.mark", 0.0);
        int* ok = reinterpret_cast<int*>(h.dev_box + 60);
        k_set_i32<<<1, 1, 0, s>>>(ok, 1);
        CK(cudaMemsetAsync(mcnt, 0, (kMaxLvl + 2) * sizeof(unsigned long long), s));
        k_pr_short_paths<<<g, kBlock, 0, s>>>(seeds, pc + P_NGRAFT, Q, L, byl, pos, mark, mk,
                                              bbase, mcnt, cap, ok);
        CK_LAUNCH();
        h.read_box(h.dev_box + 60, 1);
        h.timer.end(s);
        if (*reinterpret_cast<const int*>(h.host_box) != 0) return;  // (the structure stays stale)
      }
      rebuild();
    }
    h.timer.begin(s, "pr.mark", 0.0);
    CK(cudaMemsetAsync(mcnt, 0, (kMaxLvl + 2) * sizeof(unsigned long long), s));
    k_pr_ascend<<<g, kBlock, 0, s>>>(seeds, pc + P_NGRAFT, Q, L, byl, pos, identity, mark, mk,
                                     bbase, mcnt);
    h.stats.step(n);
    // level-j walkers are the queues of levels > j: one block row each,
    // sized by the expected queue (n / 2^(b+1) path vertices at most)
    // (one launch per level: a single cooperative launch with a grid
    // barrier per level measured slower -- the gap walks dominate, not the
    // launches)
    if (!identity) {
      static const int top_from = [] {
        const char* e = getenv("RSTG_PR_TOP_LEVEL");
        return e ? atoi(e) : 6;  // (road pr.mark 0.52 -> 0.43 ms at 6, 0.44 at 10)
      }();
      int j = K - 1;
      if (top_from > 0 && K - 1 >= top_from) {
        k_pr_descend_top<<<1, 1024, 0, s>>>(top_from, Q, L, byl, pos, mark, mk, bbase, mcnt);
        h.stats.step(n);
        j = top_from - 1;
      }
      for (; j >= 0; --j) {
        const int64_t expect = std::max<int64_t>(C[j + 1] - C[j + 2], 1);
        const unsigned gx = std::min<unsigned>(grid_for(expect), 2 * (unsigned)num_sms());
        k_pr_descend<<<dim3(gx, K - j), kBlock, 0, s>>>(j, Q, L, byl, pos, mark, mk, bbase, mcnt);
        h.stats.step(n);
      }
    }
    CK_LAUNCH();
    h.timer.end(s);
  };
  auto run_reverse = [&]() {
    const dim3 dg(2 * num_sms(), K + 1);
    k_pr_reverse_a<<<dg, kBlock, 0, s>>>(mk, bbase, mcnt, parent, scratch);
    k_pr_reverse_b<<<dg, kBlock, 0, s>>>(mk, bbase, mcnt, mark, parent, scratch, bad_rev, pos, Q);
    CK_LAUNCH();
    h.stats.step(n);
    h.stats.step(n);
    forest_dirty = true;
    identity = false;
  };

  // batched_jump's guard (pr_rst.cpp:218-219) fires only once a graft happened.
  const bool batch_ok = jump_batch >= 1 && jump_batch <= 20;
  const int64_t max_barriers =
      batch_ok ? (ceil_log2_i(std::max<int64_t>(n, 1)) + jump_batch - 1) / jump_batch + 2 : 0;
  const uint32_t* in_list = nullptr;  // nullptr: every vertex is a root
  int out = 0;
  int mode = 0;
  int64_t first_round = 0;
  if (fused0) {  // (a built CSR)
    // The first graft round from the CSR, fused with its resolve, update,
    // reversal (singleton paths) and jump: the CC's round-0 tile pass
    // (cc.cu pr_round0). Grafts, parents and converged reps are those of the
    // round-0 loop below; the roots left go to rl[0].
    h.timer.begin(s, "pr.round0", 4.0 * (n + 1) + 8.0 * n + 12.0 * n);
    const int64_t grafts0 = pr_round0(h, rep, parent, pos, Q, rl[0], pc + P_NROOTS_IN);
    h.timer.end(s);
    // batched_jump's guard (pr_rst.cpp:218-219) fires once a graft happened
    if (grafts0 > 0 && !batch_ok) throw AlgoError("jump batch out of range [1, 20]");
    h.stats.step(n, 4);
    cc_round_done(h, 0);  // (the next graft round starts the active-edge lists)
    in_list = rl[0];
    out = 1;
    mode = 1;
    identity = false;
    forest_dirty = true;
    first_round = 1;
  }
  for (int64_t round = first_round;; ++round) {
    if (round > n + 1) throw AlgoError("grafting failed to converge");
    h.timer.begin(s, "pr.graft", 0.0);
    // graft proposals with active-edge filtering (as in the CC: an edge
    // inside one tree stays inside; the proposals are unchanged)
    CK(cudaMemsetAsync(pc + P_CROSSING, 0, 3 * sizeof(unsigned long long), s));
    const double visited = (h.cc_round >= 2 && h.cc_active >= 0) ? (double)h.cc_active : (double)h.g.m;
    h.timer.add_bytes(visited * 16.0);
    cc_hook_round(h, mode, rep, slot, pc + P_CROSSING, any);
    h.read_box(reinterpret_cast<int64_t*>(pc), P_ANY + 1);
    const int64_t crossing = h.host_box[P_CROSSING];
    const bool proposed = static_cast<int>(h.host_box[P_ANY]) != 0;
    const int64_t nroots = in_list ? h.host_box[P_NROOTS_IN] : n;
    round_roots = nroots;
    cc_round_done(h, crossing);
    h.timer.end(s);
    h.stats.rounds = round + 1;
    if (!proposed) break;  // no graft (:279)
    if (!batch_ok) throw AlgoError("jump batch out of range [1, 20]");

    h.timer.begin(s, "pr.resolve", 24.0 * nroots);
    CK(cudaMemsetAsync(pc + P_NROOTS_OUT, 0, 2 * sizeof(unsigned long long), s));  // out, ngraft
    // (the first graft round on the identity forest reverses singleton
    // paths: the resolve sets the parents itself)
    const bool direct = identity;
    k_pr_resolve<<<grid_for(nroots), kBlock, 0, s>>>(in_list, pc + P_NROOTS_IN, n, h.g.edges,
                                                     (uint32_t)h.g.e_base, rep, slot, mark,
                                                     scratch, seeds, grafted, pc + P_NGRAFT,
                                                     direct ? parent : nullptr, pos, Q);
    k_pr_update<<<grid_for(nroots), kBlock, 0, s>>>(in_list, pc + P_NROOTS_IN, n, rep, slot,
                                                    rl[out], pc + P_NROOTS_OUT);
    CK(cudaMemcpyAsync(pc + P_NROOTS_IN, pc + P_NROOTS_OUT, sizeof(unsigned long long),
                       cudaMemcpyDeviceToDevice, s));
    CK_LAUNCH();
    in_list = rl[out];
    out ^= 1;
    h.stats.step(n);
    h.stats.step(n);
    h.timer.end(s);

    if (direct) {
      identity = false;
      forest_dirty = true;
    } else {
      run_marking();
      h.timer.begin(s, "pr.reverse", 0.0);
      k_pr_check<<<grid_for(nroots), kBlock, 0, s>>>(grafted, seeds, pc + P_NGRAFT, mark, parent,
                                                     bad_mark);
      h.stats.step(n);
      run_reverse();
      CK_LAUNCH();
      h.timer.end(s);
    }

    // converged reps again (batched_jump's result, :216-252): the grafted
    // roots' chains are jumped as a list, then one gather over n
    h.timer.begin(s, "pr.jump", 8.0 * n);
    if (nroots > n / 8)
      launch_compress2(h, rep, n);  // many grafts (round 0: long hook chains): tile shortcutting
    else
      compress_via_roots(h, rep, n, grafted, pc + P_NGRAFT);
    h.stats.step(n, std::max<int64_t>(max_barriers / 2, 1) - 1);
    h.timer.end(s);
    // deferred error checks of this round (+ the marked count, for the
    // phases' algorithmic bytes)
    h.read_box(reinterpret_cast<int64_t*>(pc), P_MCNT0 + K + 1);
    const bool badrev = static_cast<int>(h.host_box[P_BAD_REV]) != 0;
    double marked = 0;
    for (int b = 0; b <= K; ++b) marked += (double)h.host_box[P_MCNT0 + b];
    const double grafts = (double)h.host_box[P_NGRAFT];
    // mark: per marked vertex its queue entry 4 B + mark byte, ~2 hops of
    // pointer + level byte; reverse: queue entry, parent, scratch (twice),
    // mark; per graft the check and the root bit; jump: the grafted list
    h.timer.add_bytes("pr.mark", marked * (4.0 + 1.0 + 2.0 * 5.0));
    h.timer.add_bytes("pr.reverse", marked * 21.0 + grafts * 14.0);
    h.timer.add_bytes("pr.jump", grafts * 8.0);
    h.read_box(reinterpret_cast<int64_t*>(bad_mark), 1);
    const unsigned long long bm = (unsigned long long)h.host_box[0];
    if (bm != kAllOnes)
      throw AlgoError("path marking corrupted: " + std::to_string(bm >> 32) +
                      " is not the root above " + std::to_string((uint32_t)bm));
    if (badrev) throw AlgoError("reversal found a marked vertex with no source");
    mode ^= 1;
  }

  // Re-root the designated root's tree (pr_rst.cpp:298-303).
  CK(cudaMemcpyAsync(h.host_box, rep + root, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int32_t emergent = *reinterpret_cast<int32_t*>(h.host_box);
  if (emergent != root) {
    h.timer.begin(s, "pr.reroot", 0.0);
    // mark_path(root, emergent) :166-176: one seed
    k_set_u32<<<1, 1, 0, s>>>(seeds, (uint32_t)root);
    k_set_u32<<<1, 1, 0, s>>>(grafted, (uint32_t)emergent);
    k_set_u64<<<1, 1, 0, s>>>(pc + P_NGRAFT, 1ull);
    k_set_u8<<<1, 1, 0, s>>>(mark + root, 1);
    CK_LAUNCH();
    bool marked = false;
    if (forest_dirty) {
      // one path: walk it on the (current) parents while it is short,
      // instead of rebuilding the whole skip structure for it
      const char* cap_env = getenv("RSTG_PR_SHORT_PATH");  // (per call: the tests force the fallback)
      const int cap = cap_env ? atoi(cap_env) : 512;
      if (cap > 0) {
        int* ok = reinterpret_cast<int*>(h.dev_box + 60);  // (dev_box [60]: the short-path flag)
        CK(cudaMemsetAsync(mcnt, 0, (kMaxLvl + 2) * sizeof(unsigned long long), s));
        k_pr_short_path<<<1, 1, 0, s>>>(root, Q, L, byl, pos, mark, mk, bbase, mcnt, cap, ok);
        CK_LAUNCH();
        h.read_box(h.dev_box + 60, 1);
        marked = *reinterpret_cast<const int*>(h.host_box) != 0;
      }
    }
    h.timer.end(s);
    round_roots = n;  // (its one path was tried above: rebuild if that failed)
    if (!marked) run_marking();
    h.timer.begin(s, "pr.reroot", 0.0);
    k_pr_check<<<1, 32, 0, s>>>(grafted, seeds, pc + P_NGRAFT, mark, parent, bad_mark);
    k_set_i32<<<1, 1, 0, s>>>(scratch + root, root);  // reverse_path :212
    run_reverse();
    CK_LAUNCH();
    h.read_box(reinterpret_cast<int64_t*>(pc), P_BAD_REV + 1);
    const bool badrev = static_cast<int>(h.host_box[P_BAD_REV]) != 0;
    h.read_box(reinterpret_cast<int64_t*>(bad_mark), 1);
    h.timer.end(s);
    const unsigned long long bm = (unsigned long long)h.host_box[0];
    if (bm != kAllOnes)
      throw AlgoError("path marking corrupted: " + std::to_string(bm >> 32) +
                      " is not the root above " + std::to_string((uint32_t)bm));
    if (badrev) throw AlgoError("reversal found a marked vertex with no source");
  }
  // every slot, scratch entry and mark this build set was reset by the step
  // that consumed it: the next build may skip their fills
  h.slots_clean = slot;
  h.slots_clean_n = n;
  h.pr_clean = scratch;
  h.pr_clean_mark = mark;
  h.pr_clean_n = n;
}

}  // namespace rstg
