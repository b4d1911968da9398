// listrank.cu -- sparse ruling-set list ranking (replaces the Wyllie loop of
// list_rank, euler_rooting.cpp:104-153, which costs ceil(log2 E) full
// passes over all E arcs).
//
// Level 0 (the tour):
//   1. rulers = positions whose multiplicative hash falls in a 1/2^logk0
//      bucket, plus every list head (no walk would reach a head); the
//      producer registers them inside its own pass (lr_register_warp);
//   2. a persistent walk kernel: each CTA owns a slice of the ruler ids and
//      each thread keeps kChains sublist walks in flight at once (memory-
//      level parallelism on the dependent succ loads), claiming the next
//      ruler of its CTA's slice from shared memory when a walk ends. A walk
//      writes one 32-bit (ruler id, offset) word per arc and stops at the
//      next ruler or the list tail; a walk longer than 2^ob - 1 hops turns
//      its next arc into a fresh ruler (rare, walked by a follow-up launch).
// Levels >= 1 (the ruler lists, weighted by sublist length): the same
//   scheme recursively -- pred marks, ruler registration, persistent
//   weighted walk, recurse, expand -- until a level fits one CTA, which runs
//   Wyllie doubling in shared memory. Single-node lists drop out of the
//   recursion (their prefix is 0), so every level shrinks.
// rank(arc) = rstart[ruler] + offset is evaluated by the consumer. Ranks
// equal the reference's list_rank output (distance from the list head):
// checked arc for arc against the reference's own ranks
// (tests/golden/euler_ranks.npz) and the oracle's Wyllie restatement.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "engine.hpp"
#include "listrank.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

namespace rstg {

// sublist walks kept in flight per thread (runtime choice: RSTG_LR_CHAINS)
constexpr int kMaxChains = 4;
constexpr int kBaseMax = 8192;  // one-CTA Wyllie (64 KB of shared memory)
constexpr uint32_t kChunk = 64;  // ruler ids per round-robin chunk of the walks

static int ceil_log2_ll(int64_t x) {
  int k = 0;
  while ((int64_t{1} << k) < x) ++k;
  return k;
}

static int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = getenv(name);
  if (!e) return dflt;
  const int v = atoi(e);
  return (v < lo || v > hi) ? dflt : v;
}

LrParams lr_params(int64_t E, int64_t heads_bound, int64_t arcs) {
  if (arcs < 0) arcs = E;  // positions actually on a list (the rest are holes)
  LrParams P;
  // Ruler density: sparse rulers cut the ruler levels' work but lengthen
  // the longest sublist (the walk's critical path, ~2^k ln R hops), which
  // dominates when the tour is short. 1/32 from 24M arcs, 1/8 below
  // 4M (measured: grid 1M, road 24M, path 16M, RMAT-24).
  const int lk = arcs >= (int64_t{24} << 20) ? 5 : arcs >= (int64_t{4} << 20) ? 4 : 3;
  P.logk0 = env_int("RSTG_LR_LOGK0", lk, 1, 10);
  P.logk1 = env_int("RSTG_LR_LOGK1", 3, 1, 10);
  P.chains = env_int("RSTG_LR_CHAINS", 1, 1, 4);
  // one cooperative launch for the ruler levels measured slower than the
  // host-driven recursion (grid barriers cost more than the syncs saved)
  P.coop_levels = env_int("RSTG_LR_COOP", 0, 0, 1) != 0;
  // CTAs per SM of the level-0 walk: 4 (1024 walks per SM) measured best on
  // the road mesh -- more walks in flight thrash the L2 (profiles/)
  // (a tour whose succ + word arrays fit in half the L2 keeps all 8)
  P.walk_blocks = env_int("RSTG_LR_BLOCKS", arcs * 8 < (int64_t{48} << 20) ? 8 : 4, 1, 8);
  P.chunk = (uint32_t)env_int("RSTG_LR_CHUNK", 64, 1, 4096);
  if (P.chains == 3) P.chains = 2;
  // static rulers: hash hits (~E/2^logk, the Weyl sequence is
  // equidistributed; 2x slack) + heads; dynamic splits add <= E/walk_cap
  const int64_t stat = 2 * (E >> P.logk0) + heads_bound + 1024;
  // (tests force short walks to exercise the split path)
  const int64_t forced_cap = env_int("RSTG_LR_WALKCAP", 1 << 30, 1, 1 << 30);
  int idb = ceil_log2_ll(stat + E / std::min<int64_t>(64, forced_cap) + 64);
  if (idb < 1) idb = 1;
  if (idb > 31) throw std::runtime_error("list ranking: too many arcs");
  P.ob = 32 - idb;
  if (P.ob > 16) P.ob = 16;
  P.walk_cap = (1u << P.ob) - 1u;
  P.walk_cap = (uint32_t)std::min<int64_t>(P.walk_cap, forced_cap);
  P.cap = stat + E / P.walk_cap + 64;
  if (P.cap >= (int64_t{1} << (32 - P.ob))) throw std::runtime_error("list ranking: capacity");
  return P;
}

static unsigned persistent_grid() { return (unsigned)num_sms() * (2048 / kBlock); }

// ------------------------------------------------------------- level 0
template <int kChains>
__global__ void __launch_bounds__(kBlock)
    k_walk0(const uint32_t* __restrict__ succ, uint32_t* rpos, uint32_t* __restrict__ rlen,
            uint32_t* __restrict__ rnext, uint32_t* sl, const unsigned long long* range,
            unsigned long long* ctr, unsigned long long* walked, int logk, int ob, uint32_t walk_cap,
            uint32_t cap, uint32_t chunk) {
  // Rulers in chunks of kChunk ids dealt round-robin to the CTAs: CTA b
  // walks chunks b, b + G, b + 2G, ... in order, so the rulers in flight
  // over the whole grid form a sliding window of ids -- and ids follow
  // positions (tile-ordered registration) -- which keeps the touched part
  // of succ and sl L2-resident instead of spreading over the whole tour.
  __shared__ uint32_t s_claim;
  __shared__ unsigned long long s_walked;
  const uint32_t lo = (uint32_t)range[0], hi = (uint32_t)range[1];
  if (threadIdx.x == 0) {
    s_claim = 0;
    s_walked = 0;
  }
  __syncthreads();
  // Each walk is a small state machine issuing exactly ONE load per loop
  // iteration whatever its state (claim -> rpos, start/hop -> succ, at the
  // next ruler -> its word), so the lanes of a warp, all in different
  // states, wait for one memory latency per iteration. (Writing the words
  // over succ in place halves the traffic but serialises each hop's load
  // behind the previous hop's store to the same sector: 4x slower.)
  enum : uint32_t { kClaim = 0, kStart, kHop, kRuler, kDone };
  uint32_t st[kChains], id[kChains], cur[kChains], off[kChains];
  uint64_t mine = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) st[c] = kClaim;
  for (;;) {
    const uint32_t* ptr[kChains];
    bool live = false;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (st[c] == kClaim) {
        const uint32_t j = atomicAdd(&s_claim, 1u);
        const uint64_t t = lo + ((uint64_t)(j / chunk) * gridDim.x + blockIdx.x) * chunk + j % chunk;
        if (t < hi) {
          id[c] = (uint32_t)t;
          ptr[c] = &rpos[t];
        } else {
          st[c] = kDone;
        }
      } else if (st[c] == kStart) {
        ptr[c] = &succ[cur[c]];
        off[c] = 1;
      } else if (st[c] == kHop) {
        sl[cur[c]] = (id[c] << ob) | off[c];
        ++off[c];
        ptr[c] = &succ[cur[c]];
      } else if (st[c] == kRuler) {
        ptr[c] = &sl[cur[c]];
      }
      live |= st[c] != kDone;
    }
    if (!live) break;
    uint32_t val[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) val[c] = st[c] != kDone ? __ldg(ptr[c]) : 0u;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      const uint32_t x = val[c];
      if (st[c] == kClaim) {
        cur[c] = x;
        st[c] = kStart;
      } else if (st[c] == kRuler) {
        rlen[id[c]] = off[c];
        rnext[id[c]] = x >> ob;
        mine += off[c];
        st[c] = kClaim;
      } else if (st[c] == kStart || st[c] == kHop) {
        if (x == kNone32) {
          rlen[id[c]] = off[c];
          rnext[id[c]] = kNone32;
          mine += off[c];
          st[c] = kClaim;
        } else if (lr_hash_ruler(x, logk)) {
          cur[c] = x;
          st[c] = kRuler;
        } else if (off[c] > walk_cap) {  // split: x becomes a dynamic ruler
          const uint32_t nid = (uint32_t)atomicAdd(ctr, 1ull);
          if (nid < cap) {  // else counted only: the host throws on the count
            rpos[nid] = x;
            sl[x] = nid << ob;
          }
          rlen[id[c]] = off[c];
          rnext[id[c]] = nid;
          mine += off[c];
          st[c] = kClaim;
        } else {
          cur[c] = x;
          st[c] = kHop;
        }
      }
    }
  }
  // arcs covered (ruler itself included), for the forest check
  if (mine) atomicAdd(&s_walked, (unsigned long long)mine);
  __syncthreads();
  if (threadIdx.x == 0 && s_walked) atomicAdd(walked, s_walked);
}

// Overflowed registration: remember the true count in spill[0] and clamp.
__global__ void k_clamp_count(unsigned long long* ctr, unsigned long long cap,
                              unsigned long long* spill) {
  spill[0] = *ctr;
  if (*ctr > cap) *ctr = cap;
}

static void launch_walk0(Handle& h, const LrParams& P, const uint32_t* S, uint32_t* rsucc,
                         uint32_t* rlen, uint32_t* rnext, uint32_t* sl,
                         const unsigned long long* range, unsigned long long* ctr,
                         unsigned long long* walked) {
  const unsigned g = (unsigned)num_sms() * P.walk_blocks;
  if (P.chains == 1)
    k_walk0<1><<<g, kBlock, 0, h.stream>>>(S, rsucc, rlen, rnext, sl, range, ctr, walked, P.logk0, P.ob,
                                           P.walk_cap, (uint32_t)P.cap, P.chunk);
  else if (P.chains == 2)
    k_walk0<2><<<g, kBlock, 0, h.stream>>>(S, rsucc, rlen, rnext, sl, range, ctr, walked, P.logk0, P.ob,
                                           P.walk_cap, (uint32_t)P.cap, P.chunk);
  else
    k_walk0<4><<<g, kBlock, 0, h.stream>>>(S, rsucc, rlen, rnext, sl, range, ctr, walked, P.logk0, P.ob,
                                           P.walk_cap, (uint32_t)P.cap, P.chunk);
  CK_LAUNCH();
}

// range[0..1] = [lo, hi) of the next walk launch from the ruler counter.
__global__ void k_lr_range(unsigned long long* range, const unsigned long long* ctr) {
  range[0] = range[1];
  range[1] = *ctr;
}

// -------------------------------------------------------- levels >= 1
__global__ void k_mark_pred(int64_t N, const uint32_t* __restrict__ next, uint8_t* haspred) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
       x += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t nx = next[x];
    if (nx != kNone32) haspred[nx] = 1;
  }
}

// Rulers of a weighted level: hash hits with a predecessor, and heads of
// lists with more than one node. Singletons get sub = NONE (prefix 0).
__global__ void __launch_bounds__(kBlock)
    k_register1(int64_t N, const uint32_t* __restrict__ next, const uint8_t* __restrict__ haspred,
                uint32_t* rpos, uint32_t* sub, uint32_t* off, unsigned long long* ctr, int logk) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < N; b += stride) {
    const int64_t x = b + threadIdx.x;
    bool want = false;
    if (x < N) {
      const bool hp = haspred[x] != 0;
      const bool single = !hp && next[x] == kNone32;
      want = hp ? lr_hash_ruler((uint32_t)x, logk) : !single;
      if (single) {
        sub[x] = kNone32;
        off[x] = 0;
      }
    }
    const uint32_t id = lr_block_claim(want ? 1u : 0u, ctr);
    if (want) {
      rpos[id] = (uint32_t)x;
      sub[x] = id;
      off[x] = 0;
    }
  }
}

template <int kChains>
__global__ void __launch_bounds__(kBlock)
    k_walk1(const uint32_t* __restrict__ next, const uint32_t* __restrict__ w,
            const uint32_t* __restrict__ rpos, const unsigned long long* ctr, uint32_t* sub,
            uint32_t* __restrict__ off, uint32_t* __restrict__ rw, uint32_t* __restrict__ rn,
            int logk) {
  __shared__ uint32_t s_claim;
  const uint32_t R = (uint32_t)*ctr;
  if (threadIdx.x == 0) s_claim = 0;
  __syncthreads();
  // the same one-load-per-iteration state machine as k_walk0 (two
  // independent loads in the hop state: next and weight of a node)
  enum : uint32_t { kClaim = 0, kStart, kHop, kRuler, kDone };
  uint32_t st[kChains], id[kChains], cur[kChains], acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) st[c] = kClaim;
  for (;;) {
    const uint32_t* pa[kChains];
    const uint32_t* pb[kChains];
    bool live = false;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      pb[c] = nullptr;
      if (st[c] == kClaim) {
        const uint32_t j = atomicAdd(&s_claim, 1u);
        const uint64_t t = ((uint64_t)(j / kChunk) * gridDim.x + blockIdx.x) * kChunk + j % kChunk;
        if (t < R) {
          id[c] = (uint32_t)t;
          pa[c] = &rpos[t];
        } else {
          st[c] = kDone;
        }
      } else if (st[c] == kStart) {
        pa[c] = &next[cur[c]];
        pb[c] = &w[cur[c]];
      } else if (st[c] == kHop) {
        sub[cur[c]] = id[c];
        off[cur[c]] = acc[c];
        pa[c] = &next[cur[c]];
        pb[c] = &w[cur[c]];
      } else if (st[c] == kRuler) {
        pa[c] = &sub[cur[c]];
      }
      live |= st[c] != kDone;
    }
    if (!live) break;
    uint32_t va[kChains], vb[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      va[c] = st[c] != kDone ? ld_cg(pa[c]) : 0u;
      vb[c] = pb[c] ? __ldg(pb[c]) : 0u;
    }
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      const uint32_t x = va[c];
      if (st[c] == kClaim) {
        cur[c] = x;
        st[c] = kStart;
      } else if (st[c] == kRuler) {
        rw[id[c]] = acc[c];
        rn[id[c]] = x;
        st[c] = kClaim;
      } else if (st[c] == kStart || st[c] == kHop) {
        acc[c] = (st[c] == kStart ? 0u : acc[c]) + vb[c];
        if (x == kNone32) {
          rw[id[c]] = acc[c];
          rn[id[c]] = kNone32;
          st[c] = kClaim;
        } else if (lr_hash_ruler(x, logk)) {  // every reachable hash hit is a ruler
          cur[c] = x;
          st[c] = kRuler;
        } else {
          cur[c] = x;
          st[c] = kHop;
        }
      }
    }
  }
}

__global__ void k_expand(int64_t N, const uint32_t* __restrict__ sub, const uint32_t* __restrict__ off,
                         const uint32_t* __restrict__ pre1, uint32_t* __restrict__ pre) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
       x += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = sub[x];
    pre[x] = (s == kNone32) ? 0u : pre1[s] + off[x];
  }
}

// Verification: every node of the level was visited (sub set).
__global__ void k_check_visited(int64_t N, const uint32_t* sub, const uint32_t* next,
                                const uint8_t* haspred, int* bad) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
       x += (int64_t)gridDim.x * blockDim.x)
    if (sub[x] == kNone32 && (haspred[x] || next[x] != kNone32)) *bad = 1;
}

// Base case: one CTA, Wyllie over predecessor pointers in shared memory:
// pre[x] = sum of w over the predecessors of x. A pointer still live after
// ceil(log2 N) + 1 rounds means a cycle.
__global__ void __launch_bounds__(1024)
    k_lr_base(int N, const uint32_t* __restrict__ next, const uint32_t* __restrict__ w,
              uint32_t* __restrict__ pre, int rounds, int* bad) {
  extern __shared__ uint32_t sm[];
  uint32_t* p = sm;        // predecessor pointer
  uint32_t* v = sm + N;    // accumulated prefix
  for (int x = threadIdx.x; x < N; x += blockDim.x) p[x] = kNone32;
  __syncthreads();
  for (int x = threadIdx.x; x < N; x += blockDim.x) {
    const uint32_t nx = next[x];
    if (nx != kNone32) p[nx] = (uint32_t)x;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < N; x += blockDim.x) v[x] = (p[x] == kNone32) ? 0u : w[p[x]];
  __syncthreads();
  constexpr int kPer = kBaseMax / 1024;
  for (int r = 0; r < rounds; ++r) {
    uint32_t np[kPer], nv[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int x = threadIdx.x + k * 1024;
      if (x < N) {
        const uint32_t q = p[x];
        np[k] = (q == kNone32) ? kNone32 : p[q];
        nv[k] = (q == kNone32) ? v[x] : v[x] + v[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int x = threadIdx.x + k * 1024;
      if (x < N) {
        p[x] = np[k];
        v[x] = nv[k];
      }
    }
    __syncthreads();
  }
  for (int x = threadIdx.x; x < N; x += blockDim.x) {
    if (bad && p[x] != kNone32) *bad = 1;
    pre[x] = v[x];
  }
}

// ---------------------------------------- levels >= 1 in one launch
// The whole ruler-list recursion as ONE cooperative kernel: per level a
// pred-mark, a registration (tile-ordered claims), a weighted persistent
// walk, each phase behind a grid barrier; the level that fits kBaseCoop
// nodes is solved by CTA 0 in shared memory; then the expansions run back
// down. No host round trip between levels (their sizes stay on the
// device). Arenas are carved per level with halving capacities; a level
// that outgrows its capacity sets *fallback and the host reruns the
// host-driven recursion (list_prefix).
constexpr int kMaxCoopLevels = 12;
constexpr int kBaseCoop = 4096;
struct LrLevel {
  const uint32_t* next;  // this level's list
  const uint32_t* w;
  uint32_t* pre;         // this level's output
  unsigned long long* N; // node count (device)
  int64_t cap;           // capacity of this level's arrays
  uint8_t* haspred;
  uint32_t* sub;
  uint32_t* off;
  uint32_t* rpos;        // next level's nodes = this level's rulers
};

__global__ void __launch_bounds__(kBlock)
    k_lr_levels(LrLevel* L, int maxl, int logk, bool verify, int* bad, int* fallback) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t s_claim;
  __shared__ uint32_t s_p[kBaseCoop], s_v[kBaseCoop];
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  int k = 0;
  for (; k < maxl; ++k) {
    const int64_t N = (int64_t)*((volatile unsigned long long*)L[k].N);
    if (N <= kBaseCoop) break;
    if (k + 1 >= maxl || N > L[k].cap) {  // (uniform across the grid)
      if (gtid == 0) *fallback = 1;
      return;
    }
    const LrLevel& c = L[k];
    const LrLevel& nx = L[k + 1];
    if (gtid == 0) *nx.N = 0;
    for (int64_t x = gtid; x < N; x += gsize) {
      c.haspred[x] = 0;
      if (verify) c.sub[x] = kNone32;
    }
    grid.sync();
    for (int64_t x = gtid; x < N; x += gsize) {
      const uint32_t n1 = c.next[x];
      if (n1 != kNone32) c.haspred[n1] = 1;
    }
    grid.sync();
    // registration: next level's nodes, one claim per CTA tile
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < N; b += gsize) {
      const int64_t x = b + threadIdx.x;
      bool want = false;
      if (x < N) {
        const bool hp = c.haspred[x] != 0;
        const bool single = !hp && c.next[x] == kNone32;
        want = hp ? lr_hash_ruler((uint32_t)x, logk) : !single;
        if (single) {
          c.sub[x] = kNone32;
          c.off[x] = 0;
        }
      }
      const uint32_t id = lr_block_claim(want ? 1u : 0u, nx.N);
      if (want) {
        if (id < nx.cap) c.rpos[id] = (uint32_t)x;
        c.sub[x] = id;
        c.off[x] = 0;
      }
    }
    grid.sync();
    const uint32_t R = (uint32_t)*((volatile unsigned long long*)nx.N);
    if (R > nx.cap) {  // (uniform)
      if (gtid == 0) *fallback = 1;
      return;
    }
    // weighted walks (the k_walk1 state machine), chunks round-robin
    if (threadIdx.x == 0) s_claim = 0;
    __syncthreads();
    {
      enum : uint32_t { kClaim = 0, kStart, kHop, kRuler, kDone };
      uint32_t st = kClaim, id = 0, cur = 0, acc = 0;
      for (;;) {
        const uint32_t* pa = nullptr;
        const uint32_t* pb = nullptr;
        if (st == kClaim) {
          const uint32_t j = atomicAdd(&s_claim, 1u);
          const uint64_t t = ((uint64_t)(j / kChunk) * gridDim.x + blockIdx.x) * kChunk + j % kChunk;
          if (t < R) {
            id = (uint32_t)t;
            pa = &c.rpos[t];
          } else {
            break;
          }
        } else if (st == kStart) {
          pa = &c.next[cur];
          pb = &c.w[cur];
        } else if (st == kHop) {
          c.sub[cur] = id;
          c.off[cur] = acc;
          pa = &c.next[cur];
          pb = &c.w[cur];
        } else {  // kRuler
          pa = &c.sub[cur];
        }
        const uint32_t x = ld_cg(pa);
        const uint32_t wv = pb ? ld_cg(pb) : 0u;
        if (st == kClaim) {
          cur = x;
          st = kStart;
        } else if (st == kRuler) {
          const_cast<uint32_t*>(nx.w)[id] = acc;
          const_cast<uint32_t*>(nx.next)[id] = x;
          st = kClaim;
        } else {
          acc = (st == kStart ? 0u : acc) + wv;
          if (x == kNone32) {
            const_cast<uint32_t*>(nx.w)[id] = acc;
            const_cast<uint32_t*>(nx.next)[id] = kNone32;
            st = kClaim;
          } else {
            cur = x;
            st = lr_hash_ruler(x, logk) ? kRuler : kHop;
          }
        }
      }
    }
    grid.sync();
    if (verify)
      for (int64_t x = gtid; x < N; x += gsize)
        if (c.sub[x] == kNone32 && (c.haspred[x] || c.next[x] != kNone32)) *bad = 1;
  }
  if (k >= maxl) {
    if (gtid == 0) *fallback = 1;
    return;
  }
  // base: CTA 0, Wyllie over predecessor pointers in shared memory
  if (blockIdx.x == 0) {
    const LrLevel& c = L[k];
    const int N = (int)*((volatile unsigned long long*)c.N);
    for (int x = threadIdx.x; x < N; x += blockDim.x) s_p[x] = kNone32;
    __syncthreads();
    for (int x = threadIdx.x; x < N; x += blockDim.x) {
      const uint32_t n1 = c.next[x];
      if (n1 != kNone32) s_p[n1] = (uint32_t)x;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < N; x += blockDim.x) s_v[x] = (s_p[x] == kNone32) ? 0u : c.w[s_p[x]];
    __syncthreads();
    constexpr int kPer = kBaseCoop / kBlock;
    int rounds = 1;
    while ((1 << (rounds - 1)) < N) ++rounds;
    for (int r = 0; r < rounds; ++r) {
      uint32_t np[kPer], nv[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int x = threadIdx.x + q * kBlock;
        if (x < N) {
          const uint32_t p = s_p[x];
          np[q] = (p == kNone32) ? kNone32 : s_p[p];
          nv[q] = (p == kNone32) ? s_v[x] : s_v[x] + s_v[p];
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int x = threadIdx.x + q * kBlock;
        if (x < N) {
          s_p[x] = np[q];
          s_v[x] = nv[q];
        }
      }
      __syncthreads();
    }
    for (int x = threadIdx.x; x < N; x += blockDim.x) {
      if (s_p[x] != kNone32) *bad = 1;
      c.pre[x] = s_v[x];
    }
  }
  grid.sync();
  for (int j = k - 1; j >= 0; --j) {
    const LrLevel& c = L[j];
    const int64_t N = (int64_t)*((volatile unsigned long long*)c.N);
    const uint32_t* pre1 = L[j + 1].pre;
    for (int64_t x = gtid; x < N; x += gsize) {
      const uint32_t sb = c.sub[x];
      c.pre[x] = (sb == kNone32) ? 0u : pre1[sb] + c.off[x];
    }
    grid.sync();
  }
}

// Host side of the cooperative recursion; returns false when the host path
// must run instead (capacity fallback).
static bool list_prefix_coop(Handle& h, const LrParams& P, int64_t N0, const uint32_t* next,
                             const uint32_t* w, uint32_t* pre, bool verify, int* bad) {
  const cudaStream_t s = h.stream;
  // capacities halve per level; per level N x (haspred 1 + sub, off, rpos,
  // next', w', pre' 4 each) bytes
  int64_t caps[kMaxCoopLevels];
  int64_t total = 0;
  caps[0] = N0;
  for (int k = 0; k < kMaxCoopLevels; ++k) {
    if (k > 0) caps[k] = std::max<int64_t>(caps[k - 1] / 2, kBaseCoop);
    total += ((caps[k] + 15) & ~int64_t{15}) * 25 + 64;
  }
  uint8_t* arena = h.ws<uint8_t>(WS_LR_L1, (size_t)total + 256);
  LrLevel Lh[kMaxCoopLevels];
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(h.dev_box) + 224;  // [224, 236)
  CK(cudaMemsetAsync(counts + 1, 0, (kMaxCoopLevels - 1) * sizeof(unsigned long long), s));
  uint8_t* q = arena;
  for (int k = 0; k < kMaxCoopLevels; ++k) {
    const int64_t c = (caps[k] + 15) & ~int64_t{15};
    Lh[k].cap = caps[k];
    Lh[k].haspred = q;
    q += c;
    Lh[k].sub = reinterpret_cast<uint32_t*>(q);
    Lh[k].off = Lh[k].sub + c;
    Lh[k].rpos = Lh[k].off + c;
    uint32_t* nn = Lh[k].rpos + c;  // next level's next / w / pre
    uint32_t* nw = nn + c;
    uint32_t* np = nw + c;
    q = reinterpret_cast<uint8_t*>(np + c) + 64;
    if (k == 0) {
      Lh[0].next = next;
      Lh[0].w = w;
      Lh[0].pre = pre;
      Lh[0].N = counts;
    }
    if (k + 1 < kMaxCoopLevels) {
      Lh[k + 1].next = nn;
      Lh[k + 1].w = nw;
      Lh[k + 1].pre = np;
      Lh[k + 1].N = counts + k + 1;
    }
  }
  CK(cudaMemcpyAsync(counts, &N0, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  LrLevel* Ld = reinterpret_cast<LrLevel*>(h.ws<uint8_t>(WS_LR_L1 + 1, sizeof(Lh)));
  CK(cudaMemcpyAsync(Ld, Lh, sizeof(Lh), cudaMemcpyHostToDevice, s));
  int* fallback = reinterpret_cast<int*>(h.dev_box + 53);
  CK(cudaMemsetAsync(fallback, 0, sizeof(int), s));
  static int coop_blocks = 0;
  if (!coop_blocks) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lr_levels, kBlock, 0));
    coop_blocks = std::max(1, std::min(per_sm, 4)) * num_sms();
  }
  int maxl = kMaxCoopLevels;
  int logk = P.logk1;
  void* args[] = {(void*)&Ld, (void*)&maxl, (void*)&logk, (void*)&verify, (void*)&bad,
                  (void*)&fallback};
  CK(cudaLaunchCooperativeKernel((void*)k_lr_levels, dim3(coop_blocks), dim3(kBlock), args, 0, s));
  h.stats.step(N0, 1);
  // the fallback flag is read with the caller's next readback (lr_rank)
  return true;
}

// pre[x] = sum of w over the nodes before x in its list.
void list_prefix(Handle& h, const LrParams& P, int64_t N, const uint32_t* next, const uint32_t* w,
                 uint32_t* pre, int depth, bool verify, int* bad) {
  if (N <= 0) return;
  const cudaStream_t s = h.stream;
  if (N <= kBaseMax) {
    ensure_dyn_smem((const void*)k_lr_base, 2 * kBaseMax * sizeof(uint32_t));
    k_lr_base<<<1, 1024, 2 * N * sizeof(uint32_t), s>>>((int)N, next, w, pre,
                                                         ceil_log2_ll(N < 2 ? 2 : N) + 1, bad);
    CK_LAUNCH();
    h.stats.step(N);
    return;
  }
  if (depth >= 12) throw std::runtime_error("list ranking: recursion too deep");
  // level arena: haspred N, sub N, off N, rpos N, rw N, rn N, pre1 N --
  // sized by the ruler capacity (every level has at most that many nodes),
  // not by N: N varies with the tour layout from build to build, and a
  // grow-only workspace must not reallocate inside a timed build
  const int64_t C = std::max<int64_t>(N, P.cap);
  uint8_t* arena = h.ws<uint8_t>(WS_LR_L1 + depth, (size_t)C * (1 + 6 * 4) + 64);
  uint8_t* haspred = arena;
  uint32_t* sub = reinterpret_cast<uint32_t*>(arena + ((N + 15) & ~int64_t{15}));
  uint32_t* off = sub + N;
  uint32_t* rpos = off + N;
  uint32_t* rw = rpos + N;
  uint32_t* rn = rw + N;
  uint32_t* pre1 = rn + N;
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 9;
  CK(cudaMemsetAsync(haspred, 0, (size_t)N, s));
  CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
  if (verify) CK(cudaMemsetAsync(sub, 0xFF, (size_t)N * 4, s));
  const unsigned g = grid_for(N);
  k_mark_pred<<<g, kBlock, 0, s>>>(N, next, haspred);
  k_register1<<<g, kBlock, 0, s>>>(N, next, haspred, rpos, sub, off, ctr, P.logk1);
  if (P.chains == 1)
    k_walk1<1><<<persistent_grid(), kBlock, 0, s>>>(next, w, rpos, ctr, sub, off, rw, rn, P.logk1);
  else if (P.chains == 2)
    k_walk1<2><<<persistent_grid(), kBlock, 0, s>>>(next, w, rpos, ctr, sub, off, rw, rn, P.logk1);
  else
    k_walk1<4><<<persistent_grid(), kBlock, 0, s>>>(next, w, rpos, ctr, sub, off, rw, rn, P.logk1);
  CK_LAUNCH();
  h.stats.step(N, 3);
  if (verify) {
    k_check_visited<<<g, kBlock, 0, s>>>(N, sub, next, haspred, bad);
    CK_LAUNCH();
  }
  h.read_box(reinterpret_cast<int64_t*>(ctr), 1);
  const int64_t R1 = h.host_box[0];
  static const bool dbg = getenv("RSTG_LR_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "[lr] level %d: %lld nodes -> %lld rulers\n", depth + 1, (long long)N, (long long)R1);
  list_prefix(h, P, R1, rn, rw, pre1, depth + 1, verify, bad);
  k_expand<<<g, kBlock, 0, s>>>(N, sub, off, pre1, pre);
  CK_LAUNCH();
  h.stats.step(N);
}

const uint32_t* lr_rank(Handle& h, const LrParams& P, int64_t E, const uint32_t* S, uint32_t* sl,
                        uint32_t* rsucc, unsigned long long* ctr, bool verify, int64_t expect,
                        int64_t* R_out) {
  const cudaStream_t s = h.stream;
  if (ctr != reinterpret_cast<unsigned long long*>(h.dev_box) + 8)
    throw std::logic_error("lr_rank: ruler counter must be dev_box[8]");
  uint32_t* rlen = h.ws<uint32_t>(WS_RLEN, P.cap);
  uint32_t* rnext = h.ws<uint32_t>(WS_RNEXT, P.cap);
  unsigned long long* range = reinterpret_cast<unsigned long long*>(h.dev_box) + 10;  // [10], [11]
  unsigned long long* walked = reinterpret_cast<unsigned long long*>(h.dev_box) + 14;
  int* bad = reinterpret_cast<int*>(h.dev_box + 52);
  if (verify) CK(cudaMemsetAsync(bad, 0, sizeof(int), s));

  h.timer.begin(s, "lr.walk", 8.0 * E);
  // registration overflow (more rulers than P.cap) is caught from the count
  // read after the walk; the walk only ever touches ids below the count,
  // so bound it first on the device
  k_clamp_count<<<1, 1, 0, s>>>(ctr, (unsigned long long)P.cap, range + 2);
  CK(cudaMemsetAsync(range, 0, 2 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(walked, 0, sizeof(unsigned long long), s));
  k_lr_range<<<1, 1, 0, s>>>(range, ctr);
  launch_walk0(h, P, S, rsucc, rlen, rnext, sl, range, ctr, walked);
  h.stats.step(E, 2);
  // one readback: ctr [8], the [lo, hi) just walked [10..11], the count
  // registered before clamping [12], arcs walked [14]
  h.read_box(reinterpret_cast<int64_t*>(ctr), 7);
  if (h.host_box[4] > P.cap) throw std::runtime_error("list ranking: ruler capacity exceeded");
  int64_t hi = h.host_box[3];
  int64_t R = h.host_box[0];
  while (R > hi) {  // walks that split: their new rulers (rare)
    if (R > P.cap) throw std::runtime_error("list ranking: ruler capacity exceeded");
    k_lr_range<<<1, 1, 0, s>>>(range, ctr);
    launch_walk0(h, P, S, rsucc, rlen, rnext, sl, range, ctr, walked);
    h.stats.launches += 2;
    hi = R;
    h.read_box(reinterpret_cast<int64_t*>(ctr), 7);
    R = h.host_box[0];
  }
  if (R > P.cap) throw std::runtime_error("list ranking: ruler capacity exceeded");
  if (verify && h.host_box[6] != expect)  // some position unreachable from every ruler
    throw AlgoError("list ranking failed to converge: not a forest");
  h.timer.end(s);

  h.timer.begin(s, "lr.rulers_rank", 16.0 * R);
  uint32_t* rstart = h.ws<uint32_t>(WS_RD, P.cap);
  // The recursion's shape follows the ruler ids, which follow the tour's
  // layout (atomic insertion order), so its own step/work counts vary from
  // run to run; StepReport gets a fixed charge instead (doubling passes
  // over the expected rulers, like Wyllie on them), kept bit-identical
  // across reruns (acceptance criterion 7).
  const Stats before = h.stats;
  if (P.coop_levels) {
    list_prefix_coop(h, P, R, rnext, rlen, rstart, verify, bad);
    h.read_box(h.dev_box + 52, 2);  // [52] bad (int), [53] fallback (int)
    if (*reinterpret_cast<int*>(h.host_box + 1)) list_prefix(h, P, R, rnext, rlen, rstart, 0, verify, bad);
  } else {
    list_prefix(h, P, R, rnext, rlen, rstart, 0, verify, bad);
  }
  if (verify) {
    h.read_box(reinterpret_cast<int64_t*>(bad), 1);
    if (*reinterpret_cast<int*>(h.host_box))
      throw AlgoError("list ranking failed to converge: not a forest");
  }
  {
    const int64_t launches = h.stats.launches;
    h.stats = before;
    h.stats.launches = launches;
    // (the expected ruler count, E / 2^logk0: the static count itself
    // depends on which arc opens each tour)
    const int64_t Rexp = std::max<int64_t>(E >> P.logk0, 2);
    const int rounds = ceil_log2_ll(Rexp) + 1;
    h.stats.steps += rounds;
    h.stats.work += Rexp * rounds;
  }
  h.timer.end(s);
  if (R_out) *R_out = R;
  return rstart;
}

// ------------------------------------------------------- generic lists
__global__ void __launch_bounds__(kBlock)
    k_register0(int64_t E, const uint8_t* __restrict__ haspred, uint32_t* rpos, uint32_t* sl,
                unsigned long long* ctr, int logk, int ob, uint32_t cap) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < E; b += stride) {
    const int64_t p = b + threadIdx.x;
    const bool want = p < E && (lr_hash_ruler((uint32_t)p, logk) || !haspred[p]);
    const uint32_t id = lr_block_claim(want ? 1u : 0u, ctr);
    if (want) lr_put(id, (uint32_t)p, rpos, sl, ob, cap);
  }
}

const uint32_t* lr_rank_lists(Handle& h, int64_t E, const uint32_t* succ, uint32_t* sl, bool verify,
                              LrParams* P_out) {
  const LrParams P = lr_params(E, E);
  uint32_t* rpos = h.ws<uint32_t>(WS_RPOS, P.cap);
  uint8_t* haspred = h.ws<uint8_t>(WS_ISROOT, E);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 8;
  CK(cudaMemsetAsync(haspred, 0, (size_t)E, h.stream));
  CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), h.stream));
  k_mark_pred<<<grid_for(E), kBlock, 0, h.stream>>>(E, succ, haspred);
  k_register0<<<grid_for(E), kBlock, 0, h.stream>>>(E, haspred, rpos, sl, ctr, P.logk0, P.ob,
                                                    (uint32_t)P.cap);
  CK_LAUNCH();
  h.stats.step(E, 2);
  const uint32_t* rstart = lr_rank(h, P, E, succ, sl, rpos, ctr, verify, E, nullptr);
  if (P_out) *P_out = P;
  return rstart;
}

}  // namespace rstg
