// tilerank.cu -- Euler-tour ranking by tile contraction.
//
// The tour of a locally numbered tree (meshes, paths, grids: a tree edge
// joins nearby vertex ids, and tree edge slots are vertex ids) mostly
// steps between nearby slots. A CTA takes a tile of kSlots consecutive
// slots -- its arcs i and N + i -- and ranks them on chip:
//   1. the successor of every arc of the tile is read once (all loads of
//      a thread in flight together) and kept in shared memory as a local
//      index when it stays in the tile; a segment is a maximal run of
//      tour successors inside the tile, its head the arc without an
//      in-tile predecessor;
//   2. rulers = the heads plus one arc in 16 by index (one per thread);
//      every ruler walks to the next ruler in shared memory, writing each
//      arc it passes (ruler << 16 | offset) and the reached ruler's
//      (predecessor ruler << 16 | distance) -- O(arcs) work, ~16 hops a walk;
//   3. pointer jumping over the rulers alone (a few hundred per tile)
//      gives every ruler its head and offset; the tile publishes its head
//      count as soon as it is known and takes its first segment id by
//      decoupled look-back, so segment ids follow the tile order; every
//      arc writes (segment, offset), every segment its length and exit
//      (the arc after its last one).
// The segments form lists again -- one per tour, shorter by the
// contraction factor, and local again because their ids are in tile order
// -- so the same contraction is applied to them, weighted by segment
// length (k_tile_rank_w), level after level until one tile holds a whole
// list; the prefixes are then expanded back down. No host round trip
// between levels: counts stay on the device, grids are sized by a bound,
// and a level that overflows its bound makes the caller fall back to
// list_prefix (recursive ruling sets, listrank.cu).
// A tour that jumps between tiles (random vertex ids) gains little: the
// caller (euler.cu) then keeps the ruling-set walk, chosen per graph from
// an edge-locality sample.
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "engine.hpp"
#include "listrank.cuh"

namespace rstg {

constexpr int kTileRankThreads = 1024;

// nx[] packs a 15-bit local index with a ruler flag. Level kernels (<= 16K
// nodes) mark "successor leaves the tile / list end" with kTileExit; the
// level-1 kernel (up to 32K arcs: every 15-bit value is an arc) marks it by
// pointing the arc at itself, and uses kTileExit only as the index mask.
constexpr uint16_t kTileExit = 0x7FFF;
constexpr uint16_t kTileRuler = 0x8000;  // flag on nx[li]: li is a ruler

// Tile-ordered numbering, single pass (decoupled look-back): tile ids are
// taken in launch order from state[0], each tile publishes its count and
// then its inclusive prefix in state[1 + tile] (flag in the top two bits,
// value below, one 64-bit word: no separate fence for the payload). A tile
// only waits on tiles that took their ids earlier, so it cannot deadlock.
// Segment ids in tile order keep the segment list local: the next level
// contracts it by tiles again.
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = kLbAgg - 1;
__device__ __forceinline__ uint32_t tile_take(unsigned long long* state) {
  return (uint32_t)atomicAdd(state, 1ull);
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// Publishes the tile's count as soon as it is known (before the walks), so
// that by the time the tile needs its prefix the tiles before it have
// mostly published theirs.
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void tile_publish(unsigned long long* state, uint32_t tile,
                                             uint32_t count) {
  // (a store, not an atomic: the flag and value are one word, and nothing
  // waits on a returned value)
  st_relaxed_gpu(&state[1 + tile], (tile == 0 ? kLbInc : kLbAgg) | count);
}
// The look-back by one whole warp (all 32 lanes call it): each step reads
// 32 predecessors' words at once and stops at the nearest inclusive prefix
// -- one L2 round trip per 32 tiles instead of one per tile (a thread
// walking back alone left the rest of its CTA waiting at the barrier).
__device__ __forceinline__ uint32_t tile_prefix_warp(unsigned long long* state, uint32_t tile,
                                                     uint32_t count) {
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long* st = state + 1;
  unsigned long long excl = 0;
  for (int64_t base = (int64_t)tile - 1; base >= 0; base -= 32) {
    const int64_t p = base - (int64_t)lane;
    unsigned long long v;
    unsigned inc;
    for (;;) {
      v = p >= 0 ? ld_relaxed_gpu(&st[p]) : kLbInc;  // (before tile 0: an inclusive 0)
      inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
      const unsigned lim = inc ? (2u << (__ffs(inc) - 1)) - 1u : 0xffffffffu;  // lanes that count
      if (!(__ballot_sync(0xffffffffu, (v >> 62) == 0) & lim)) break;  // all of them published
    }
    const unsigned first = inc ? (unsigned)__ffs(inc) - 1u : 31u;
    unsigned long long add = lane <= first ? (v & kLbVal) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
    excl += add;
    if (inc) break;
  }
  if (lane == 0) st_relaxed_gpu(&st[tile], kLbInc | (excl + count));
  return (uint32_t)excl;
}

template <int kSlots>
constexpr size_t tile_rank_smem() {
  return 2 * kSlots * (sizeof(uint32_t) + sizeof(uint16_t) + sizeof(uint8_t));
}

// CTAs per SM: shared memory (228 KB per SM, 1 KB reserved per CTA) or threads
template <int kSlots, int kThreads>
constexpr int tile_rank_blocks() {
  constexpr int by_smem = 233472 / (int)(tile_rank_smem<kSlots>() + 1024);
  constexpr int by_threads = 2048 / kThreads;
  return by_smem < by_threads ? by_smem : by_threads;
}

// Local arc index: slot j of the tile -> arc j (t0 + j) and kSlots + j
// (N + t0 + j). All index math is 32-bit: arcs are u32 (2N < 2^32).
template <int kSlots, int kThreads, int kStride>
__global__ void __launch_bounds__(kThreads, tile_rank_blocks<kSlots, kThreads>())
    k_tile_rank(uint32_t N, const uint32_t* __restrict__ S, const int32_t* __restrict__ lab,
                bool cc_slots, uint32_t T, uint32_t* __restrict__ seg, uint16_t* __restrict__ off,
                uint32_t* __restrict__ seg_len, uint32_t* __restrict__ seg_exit,
                unsigned long long* nseg, unsigned long long* state,
                unsigned long long* walked) {
  static_assert(2 * kSlots <= kTileExit + 1, "local arc index must fit 15 bits");
  constexpr int kArcs = 2 * kSlots;
  constexpr int kPer = kSlots / kThreads;  // slots per thread
  constexpr int kOwn = 2 * kPer;           // arcs per thread
  static_assert(kOwn <= 32, "own-arc masks are 32 bits");
  extern __shared__ uint32_t word[];  // arc: ruler << 16 | offset; ruler: pred ruler << 16 | dist
  // local successor | ruler flag; an arc whose successor leaves the tile
  // (or ends the tour) points at itself
  uint16_t* nx = reinterpret_cast<uint16_t*>(word + kArcs);
  uint16_t* hid = nx;  // (after the walks) head -> local segment number
  // has an in-tile predecessor: plain byte stores (racing stores all write
  // 1), not bitmap atomics -- a path's warp would hit one word 32 times
  uint8_t* haspred = reinterpret_cast<uint8_t*>(nx + kArcs);
  __shared__ uint32_t s_nh, s_walk, s_tile, s_base;
  __shared__ int s_rounds;
  if (threadIdx.x == 0) s_tile = tile_take(state);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t t0 = tile * (uint32_t)kSlots;
  const uint32_t cnt = min((uint32_t)kSlots, N - t0);  // slots in this tile
  const uint32_t tid = threadIdx.x;
  // own arc q: slot j = tid + (q >> 1) * kThreads, local j + (q & 1) * kSlots
  auto local_of = [&](int q) -> uint32_t { return tid + (q >> 1) * kThreads + (q & 1) * kSlots; };
  auto global_of = [&](int q) -> uint32_t {
    return t0 + tid + (q >> 1) * kThreads + ((q & 1) ? N : 0u);
  };
  if (tid == 0) s_nh = s_walk = 0;
  for (int w = tid; w < kArcs / 16; w += kThreads) reinterpret_cast<uint4*>(haspred)[w] = uint4{0, 0, 0, 0};
  // 1. loads: validity of each own slot, then the successors of its arcs
  //    (staged in word[], free until the walks)
  uint32_t vmask = 0;  // own arcs that exist
  const uint32_t last = N - 1;  // loads are unconditional (clamped): all in flight at once
  // (cc_slots with lab == nullptr: the Euler vertex pass marked every empty
  // slot's successor words kEmptySlot, so validity comes with the S loads
  // below and the labels are not read at all)
  if (cc_slots && lab) {
    int32_t lv[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) lv[k] = __ldcs(&lab[min(t0 + tid + k * kThreads, last)]);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint32_t j = tid + k * kThreads;
      vmask |= (j < cnt && lv[k] != (int32_t)(t0 + j)) ? 3u << (2 * k) : 0u;
    }
  } else if (!cc_slots) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint32_t j = tid + k * kThreads;
      vmask |= (j < cnt && t0 + j < T) ? 3u << (2 * k) : 0u;
    }
  }
  const bool marked = cc_slots && !lab;
  constexpr int kBatch = kOwn < 16 ? kOwn : 16;
#pragma unroll
  for (int q0 = 0; q0 < kOwn; q0 += kBatch) {
    uint32_t y[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const uint32_t j = min(t0 + tid + ((q0 + q) >> 1) * kThreads, last);
      // (default caching, not evict-first: each segment tail re-reads its
      // successor at the end of the tile, from L2)
      y[q] = __ldg(&S[((q0 + q) & 1) ? N + j : j]);
    }
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      word[local_of(q0 + q)] = y[q];
      if (marked && !((q0 + q) & 1) && tid + ((q0 + q) >> 1) * kThreads < cnt &&
          y[q] != kEmptySlot)
        vmask |= 3u << (q0 + q);  // (both arcs of the slot)
    }
  }
  __syncthreads();  // haspred zeroed
  uint32_t tmask = 0;  // own arcs whose successor leaves the tile (segment tails)
#pragma unroll
  for (int q = 0; q < kOwn; ++q) {
    if (!(vmask >> q & 1)) continue;
    const uint32_t li = local_of(q);
    const uint32_t v = word[li];
    uint32_t ls = li;
    if (v - t0 < cnt) ls = v - t0;                              // forward arc in the tile
    else if (v - N - t0 < cnt && v >= N) ls = v - N - t0 + kSlots;  // reverse arc in the tile
    if (v == kNone32) ls = li;
    if (ls != li) haspred[ls] = 1;
    else tmask |= 1u << q;
    nx[li] = (uint16_t)ls;
  }
  __syncthreads();
  // 2. rulers: heads, and own arc q == tid % kOwn (one arc in kOwn by index)
  uint32_t hmask = 0, rmask = 0;
#pragma unroll
  for (int q = 0; q < kOwn; ++q) {
    const uint32_t li = local_of(q);
    const bool head = (vmask >> q & 1) && !haspred[li];
    const bool ruler = head || ((vmask >> q & 1) && q % kStride == (int)(tid % kStride));
    hmask |= head ? 1u << q : 0u;
    rmask |= ruler ? 1u << q : 0u;
    if (ruler) nx[li] |= kTileRuler;
    if (head) word[li] = li << 16;
  }
  const uint32_t hbase = hmask ? atomicAdd(&s_nh, (uint32_t)__popc(hmask)) : 0u;
  __syncthreads();
  if (tid == 0) tile_publish(state, tile, s_nh);
  for (uint32_t m = rmask; m; m &= m - 1) {
    const uint32_t r = local_of(__ffs(m) - 1);
    uint32_t cur = nx[r] & kTileExit, o = 1;
    if (cur == r) continue;  // its successor leaves the tile
    for (;;) {
      const uint32_t v = nx[cur];
      word[cur] = r << 16 | o;
      const uint32_t nxt = v & kTileExit;
      if ((v & kTileRuler) || nxt == cur) break;
      cur = nxt;
      ++o;
    }
  }
  __syncthreads();
  // 3. pointer jumping over the rulers that are not heads
  int r = 0;
  for (; r < 16; ++r) {
    int changed = 0;
    for (uint32_t m = rmask & ~hmask; m; m &= m - 1) {
      const uint32_t li = local_of(__ffs(m) - 1);
      const uint32_t v = word[li];
      const uint32_t p = v >> 16;
      const uint32_t w = word[p];
      if ((w >> 16) == p) continue;  // p is a head: done
      word[li] = (w & 0xFFFF0000u) | ((v + w) & 0xFFFFu);
      changed = 1;
    }
    if (!__syncthreads_or(changed)) break;
  }
  if (walked && tid == 0) s_rounds = r;
  {
    uint32_t k = hbase;
    for (uint32_t m = hmask; m; m &= m - 1) hid[local_of(__ffs(m) - 1)] = (uint16_t)k++;
  }
  __syncthreads();
  if (tid < 32) {
    const uint32_t b = tile_prefix_warp(state, tile, s_nh);
    if (tid == 0) {
      s_base = b;
      if (tile == gridDim.x - 1) *nseg = b + s_nh;
    }
  }
  __syncthreads();
  const uint32_t sbase = s_base;
#pragma unroll
  for (int q = 0; q < kOwn; ++q) {
    if (!(vmask >> q & 1)) {  // no arc: marked for the orient pass
      if (tid + (q >> 1) * kThreads < cnt) __stcs(&seg[global_of(q)], kNone32);
      continue;
    }
    uint32_t w = word[local_of(q)], o = 0;
    if (!(rmask >> q & 1)) {  // (ruler, offset) -> the ruler's (head, offset)
      o = w & 0xFFFFu;
      w = word[w >> 16];
    }
    o += w & 0xFFFFu;
    const uint32_t sid = sbase + hid[w >> 16];
    const uint32_t x = global_of(q);
    __stcs(&seg[x], sid);
    __stcs(&off[x], (uint16_t)o);
    if (tmask >> q & 1) {
      seg_len[sid] = o + 1;
      seg_exit[sid] = __ldg(&S[x]);  // the next segment's head (or NONE; L2: staged above)
    }
  }
  if (walked) {
    atomicAdd(&s_walk, (uint32_t)__popc(vmask));
    __syncthreads();
    if (tid == 0) {
      atomicAdd(walked, (unsigned long long)s_walk);
      atomicMax(reinterpret_cast<unsigned long long*>(walked) + 1, (unsigned long long)s_rounds);
    }
  }
}

// Level >= 2: the same contraction on a weighted list -- node i of
// [0, n), successor next[i] (NONE at the end), weight w[i] (its segment
// length below). A tile is kNodes consecutive node ids (tile-ordered ids
// from the level below make these neighbours on the tour). Each node gets
// its next-level segment and its weighted offset in it (the sum of the
// weights before it); each segment its weight and last node.
template <int kNodes>
constexpr size_t tile_rank_w_smem() {
  return kNodes * (sizeof(unsigned long long) + sizeof(uint16_t) + sizeof(uint8_t));
}

template <int kNodes, int kThreads, int kStride>
__global__ void __launch_bounds__(kThreads, kNodes > 8192 ? 1 : 2048 / kThreads)
    k_tile_rank_w(const unsigned long long* n_dev, const uint32_t* __restrict__ exit_in,
                  const uint32_t* __restrict__ seg_in, const uint32_t* __restrict__ w,
                  uint32_t* __restrict__ seg,
                  uint32_t* __restrict__ off, uint32_t* __restrict__ seg_len,
                  uint32_t* __restrict__ seg_exit, unsigned long long* nseg,
                  unsigned long long* state, int* overflow) {
  static_assert(kNodes <= kTileExit, "local node index must fit 15 bits");
  constexpr int kPer = kNodes / kThreads;
  static_assert(kPer <= 32, "own-node masks are 32 bits");
  // node: ruler << 32 | weighted offset; ruler: pred ruler << 32 | distance;
  // before the walks: the node's own weight
  extern __shared__ unsigned long long wd[];
  uint16_t* nx = reinterpret_cast<uint16_t*>(wd + kNodes);  // local successor | ruler flag
  uint16_t* hid = nx;
  uint8_t* haspred = reinterpret_cast<uint8_t*>(nx + kNodes);
  __shared__ uint32_t s_nh, s_tile, s_base;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    s_tile = tile_take(state);
    s_nh = 0;
  }
  for (int k = tid; k < kNodes / 16; k += kThreads)
    reinterpret_cast<uint4*>(haspred)[k] = uint4{0, 0, 0, 0};
  __syncthreads();
  // node count from the level below (on the device: no host round trip);
  // the grid is sized by a bound, tiles past the count leave at once
  const uint32_t n = (uint32_t)*n_dev;
  const uint32_t ntiles = (n + kNodes - 1) / kNodes;
  if (blockIdx.x == 0 && ntiles > gridDim.x && tid == 0) *overflow = 1;
  const uint32_t tile = s_tile;
  if (tile >= ntiles) return;
  const uint32_t t0 = tile * (uint32_t)kNodes;
  const uint32_t cnt = min((uint32_t)kNodes, n - t0);
  const uint32_t last = n - 1;
  // successor of node i (a segment of the level below): the segment
  // headed by the element after its last one, next = seg_in[exit_in[i]]
  // (computed here, not by a separate pass)
  uint32_t y[kPer], wt[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t i = min(t0 + tid + k * kThreads, last);
    y[k] = __ldcs(&exit_in[i]);
    wt[k] = __ldcs(&w[i]);
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) y[k] = y[k] == kNone32 ? kNone32 : seg_in[y[k]];
  uint32_t vmask = 0, tmask = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t j = tid + k * kThreads;
    if (j >= cnt) continue;
    vmask |= 1u << k;
    const uint32_t ls = (y[k] != kNone32 && y[k] - t0 < cnt) ? y[k] - t0 : kTileExit;
    if (ls != kTileExit) haspred[ls] = 1;
    else tmask |= 1u << k;
    nx[j] = (uint16_t)ls;
    wd[j] = wt[k];
  }
  __syncthreads();
  uint32_t hmask = 0, rmask = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t j = tid + k * kThreads;
    const bool head = (vmask >> k & 1) && !haspred[j];
    const bool ruler = head || ((vmask >> k & 1) && k % kStride == (int)(tid % kStride));
    hmask |= head ? 1u << k : 0u;
    rmask |= ruler ? 1u << k : 0u;
    if (ruler) nx[j] |= kTileRuler;
  }
  const uint32_t hbase = hmask ? atomicAdd(&s_nh, (uint32_t)__popc(hmask)) : 0u;
  __syncthreads();
  if (tid == 0) tile_publish(state, tile, s_nh);
  // heads: (self, 0); a head is never reached by a walk, and every ruler's
  // own weight is in a register
  for (uint32_t m = hmask; m; m &= m - 1) {
    const uint32_t j = tid + (__ffs(m) - 1) * kThreads;
    wd[j] = (unsigned long long)j << 32;
  }
  for (uint32_t m = rmask; m; m &= m - 1) {
    const int k = __ffs(m) - 1;
    const uint32_t r = tid + k * kThreads;
    uint32_t cur = nx[r] & kTileExit;
    unsigned long long acc = wt[k];
    while (cur != kTileExit) {
      const uint32_t v = nx[cur];
      if (v & kTileRuler) {
        wd[cur] = (unsigned long long)r << 32 | acc;
        break;
      }
      const uint32_t wc = (uint32_t)wd[cur];  // its weight (one walk visits a node)
      wd[cur] = (unsigned long long)r << 32 | acc;
      acc += wc;
      cur = v & kTileExit;
    }
  }
  __syncthreads();
  for (int r = 0; r < 16; ++r) {
    int changed = 0;
    for (uint32_t m = rmask & ~hmask; m; m &= m - 1) {
      const uint32_t j = tid + (__ffs(m) - 1) * kThreads;
      const unsigned long long v = wd[j];
      const uint32_t p = (uint32_t)(v >> 32);
      const unsigned long long u = wd[p];
      if ((uint32_t)(u >> 32) == p) continue;
      wd[j] = (u & 0xFFFFFFFF00000000ull) | (uint32_t)(v + u);
      changed = 1;
    }
    if (!__syncthreads_or(changed)) break;
  }
  {
    uint32_t c = hbase;
    for (uint32_t m = hmask; m; m &= m - 1) hid[tid + (__ffs(m) - 1) * kThreads] = (uint16_t)c++;
  }
  __syncthreads();
  if (tid < 32) {
    const uint32_t b = tile_prefix_warp(state, tile, s_nh);
    if (tid == 0) {
      s_base = b;
      if (tile == ntiles - 1) *nseg = b + s_nh;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (!(vmask >> k & 1)) continue;
    const uint32_t j = tid + k * kThreads;
    unsigned long long v = wd[j];
    uint32_t o = 0;
    if (!(rmask >> k & 1)) {
      o = (uint32_t)v;
      v = wd[v >> 32];
    }
    o += (uint32_t)v;
    const uint32_t sid = s_base + hid[v >> 32];
    __stcs(&seg[t0 + j], sid);
    __stcs(&off[t0 + j], o);
    if (tmask >> k & 1) {
      seg_len[sid] = o + wt[k];
      seg_exit[sid] = y[k];  // this level's node after the segment (or NONE)
    }
  }
}

// next segment of each segment: the one its exit arc heads
__global__ void k_seg_link(const unsigned long long* nseg, const uint32_t* __restrict__ seg_exit,
                           const uint32_t* __restrict__ seg, uint32_t* __restrict__ seg_next) {
  const int64_t R = (int64_t)*nseg;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t ex = seg_exit[i];
    seg_next[i] = ex == kNone32 ? kNone32 : seg[ex];
  }
}

// pre[i] = pre_up[seg[i]] + off[i] over the n_dev nodes of a level
// (nothing when a level overflowed: counts may then exceed the arenas,
// which are sized by the bounds; the caller falls back)
__global__ void k_tile_expand(const unsigned long long* n_dev, const uint32_t* __restrict__ seg,
                              const uint32_t* __restrict__ off, const uint32_t* __restrict__ pre_up,
                              uint32_t* __restrict__ pre, const int* overflow) {
  if (*overflow) return;
  const int64_t n = (int64_t)*n_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pre[i] = pre_up[seg[i]] + off[i];
}

namespace {
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
template <class K>
void set_smem(K kern, size_t smem) {
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
}
constexpr int kLevelNodes = 8192;
constexpr int kBigLevelNodes = 16384;
constexpr int kLevelThreads = 1024;
}  // namespace

// Weighted prefix of a tile-ordered list (levels >= 2 of the contraction):
// pre[i] = sum of len over the nodes before i on its list. Each level
// contracts by tiles; the top (<= one tile) is ranked by the same kernel as
// a single tile, whose segments are then whole lists. No host round trip:
// node counts stay on the device and each grid is sized for contraction of
// at least 3x per level (3.6-4x is typical on locally numbered tours); a level that needs more tiles, or a
// top with more than one tile, raises `overflow` and the caller falls back
// to list_prefix. Returns false on overflow. deferred: R is only a bound
// (the previous build's count plus a margin); nothing is read back here --
// the counts and the overflow flag go to host_box[32..49) asynchronously
// and the caller settles them after its final sync (tile_rank_settle).
static bool tile_prefix_levels(Handle& h, int64_t R, const uint32_t* S, const uint32_t* seg1,
                               const uint32_t* exit1, const uint32_t* len1, uint32_t* pre1,
                               bool dbg, bool deferred) {
  const cudaStream_t s = h.stream;
  constexpr int kMaxLevels = WS_TL_LAST - WS_TL2;
  // level l: its nodes are the segments of level l - 1 (level 0: of the
  // arcs); node i's successor is seg_in[exit[i]], exit[i] the element of
  // level l - 1 after its last one
  struct Level {
    const uint32_t* exit;
    const uint32_t* seg_in;
    const uint32_t* len;
    uint32_t* pre;
    uint32_t* seg;  // up-mapping of this level's nodes
    uint32_t* off;
    int64_t bound;  // node-count bound (grid sizing)
    int tile;       // nodes per tile: 16K (one CTA per SM, twice the
                    // contraction of 8K at two CTAs per SM; see big_tiles)
  } L[kMaxLevels + 2];
  L[0] = Level{exit1, seg1, len1, pre1, nullptr, nullptr, R, 0};
  const int contract = std::max(2, env_int("RSTG_LR_TILECONTRACT", 3));
  // 16K-node tiles at every level (2; 1: only once one wave of them covers
  // a level, 0: never): they contract 7-12x where 8K tiles contract ~4x, so
  // one level fewer; measured on road, rulers_rank 0.293 -> 0.283 ms
  static const int big_tiles = env_int("RSTG_LR_BIGTILES", 2);
  const int64_t big_max = big_tiles == 2 ? INT64_MAX
                          : big_tiles ? (int64_t)num_sms() * kBigLevelNodes : 0;
  int top = 0;
  for (;;) {
    const int64_t b = L[top].bound;
    L[top].tile = b <= big_max ? kBigLevelNodes : kLevelNodes;
    size_t cap = kLevelNodes;
    while ((int64_t)cap < b) cap <<= 1;  // stable across builds
    uint32_t* a = h.ws<uint32_t>(WS_TL2 + top, 5 * cap);
    L[top].seg = a;
    L[top].off = a + cap;
    if (b <= L[top].tile) break;
    if (top == kMaxLevels - 1) return false;
    // the next level's nodes: at most a third of these (bound; 3.6-4x is
    // typical), else overflow (RSTG_LR_TILECONTRACT overrides the factor:
    // the tests force the fallback with a large one)
    // (16K tiles contract 7-12x on road: bounded by 5x there)
    const int c = L[top].tile == kBigLevelNodes ? std::max(contract, 5) : contract;
    L[top + 1] = Level{a + 2 * cap, L[top].seg, a + 3 * cap, a + 4 * cap, nullptr, nullptr,
                       std::max<int64_t>((b + c - 1) / c, 1), 0};
    ++top;
  }
  // one control block, zeroed by one memset: node counts [0, 16) (count 0 =
  // the segment count the level-1 kernel left in dev_box[8], copied), the
  // overflow flag [16], then each level's tile counter + look-back states
  size_t words = 32;
  for (int l = 0; l <= top; ++l)
    words += (l == top ? 1 : (L[l].bound + L[l].tile - 1) / L[l].tile) + 1;
  unsigned long long* blk = h.ws<unsigned long long>(WS_TL_LAST, words);
  unsigned long long* cnt = blk;
  int* overflow = reinterpret_cast<int*>(blk + 16);
  CK(cudaMemsetAsync(blk, 0, words * sizeof(unsigned long long), s));
  CK(cudaMemcpyAsync(cnt, h.dev_box + 8, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
  static const int wstride = env_int("RSTG_LR_WSTRIDE", 4);
  constexpr size_t smem = tile_rank_w_smem<kLevelNodes>();
  constexpr size_t smem_big = tile_rank_w_smem<kBigLevelNodes>();
  auto kern = wstride >= 8   ? k_tile_rank_w<kLevelNodes, kLevelThreads, 8>
              : wstride >= 4 ? k_tile_rank_w<kLevelNodes, kLevelThreads, 4>
                             : k_tile_rank_w<kLevelNodes, kLevelThreads, 2>;
  auto kern_big = wstride >= 8   ? k_tile_rank_w<kBigLevelNodes, kLevelThreads, 16>
                  : wstride >= 4 ? k_tile_rank_w<kBigLevelNodes, kLevelThreads, 8>
                                 : k_tile_rank_w<kBigLevelNodes, kLevelThreads, 4>;
  set_smem(kern, smem);
  set_smem(kern_big, smem_big);
  unsigned long long* state = blk + 32;
  for (int l = 0; l <= top; ++l) {
    const bool is_top = l == top;
    const bool big = L[l].tile == kBigLevelNodes;
    const unsigned tiles = is_top ? 1u : (unsigned)((L[l].bound + L[l].tile - 1) / L[l].tile);
    // the top is one tile: its segments are whole lists and its offsets
    // the prefixes; its segment outputs go to scratch
    uint32_t* scratch = h.ws<uint32_t>(WS_RA, 4 * (size_t)kBigLevelNodes);
    const int kScr = kBigLevelNodes;
    (big ? kern_big : kern)<<<tiles, kLevelThreads, big ? smem_big : smem, s>>>(
        cnt + l, L[l].exit, L[l].seg_in, L[l].len, is_top ? scratch : L[l].seg,
        is_top ? L[l].pre : L[l].off,
        is_top ? scratch + kScr : const_cast<uint32_t*>(L[l + 1].len),
        is_top ? scratch + 2 * kScr : const_cast<uint32_t*>(L[l + 1].exit), cnt + l + 1,
        state, overflow);
    CK_LAUNCH();
    state += tiles + 1;
  }
  for (int l = top - 1; l >= 0; --l) {
    k_tile_expand<<<grid_for(L[l].bound), kBlock, 0, s>>>(cnt + l, L[l].seg, L[l].off,
                                                          L[l + 1].pre, L[l].pre, overflow);
    CK_LAUNCH();
  }
  if (deferred) {
    h.late_copy = {blk, 17};  // (enqueued by the caller after the orientation)
    return true;
  }
  h.read_box(reinterpret_cast<int64_t*>(blk), 17);  // counts, overflow
  if (dbg) {
    for (int l = 0; l <= top; ++l)
      fprintf(stderr, "lr.tiles level %d: %lld nodes\n", l + 2, (long long)h.host_box[l]);
  }
  return *reinterpret_cast<int*>(&h.host_box[16]) == 0;
}

// The segments' ranks by the generic list ranking (levels that stall).
static void tile_fallback(Handle& h, const LrParams& Q, int64_t R, const uint32_t* seg,
                          const uint32_t* seg_exit, const uint32_t* seg_len, uint32_t* seg_next,
                          uint32_t* segstart, const unsigned long long* nseg) {
  k_seg_link<<<grid_for(R), kBlock, 0, h.stream>>>(nseg, seg_exit, seg, seg_next);
  CK_LAUNCH();
  list_prefix(h, Q, R, seg_next, seg_len, segstart, 0, false, nullptr);
}

TileRank lr_rank_tiles(Handle& h, const LrParams& P, int64_t N, const uint32_t* S,
                       const int32_t* lab, bool cc_slots, int64_t T, bool verify) {
  const cudaStream_t s = h.stream;
  const int64_t E = 2 * N;
  uint32_t* seg = h.ws<uint32_t>(WS_SL, E);
  uint16_t* off = h.ws<uint16_t>(WS_TOFF, E);
  // segments <= arcs: sized by E (a fixed bound: no reallocation per build)
  uint32_t* seg_len = h.ws<uint32_t>(WS_RLEN, E + 1);
  uint32_t* seg_exit = h.ws<uint32_t>(WS_RNEXT, E + 1);
  uint32_t* seg_next = h.ws<uint32_t>(WS_RPOS, E + 1);
  uint32_t* segstart = h.ws<uint32_t>(WS_RD, E + 1);
  unsigned long long* nseg = reinterpret_cast<unsigned long long*>(h.dev_box) + 8;
  unsigned long long* walked = reinterpret_cast<unsigned long long*>(h.dev_box) + 14;
  static const int slots_env = env_int("RSTG_LR_TILESLOTS", 8192);
  static const bool dbg = getenv("RSTG_LR_DEBUG") != nullptr;
  const int slots = slots_env <= 2048 ? 2048 : slots_env <= 4096 ? 4096 : slots_env <= 8192 ? 8192 : 16384;
  const unsigned tiles = (unsigned)((N + slots - 1) / slots);
  unsigned long long* state = h.ws<unsigned long long>(WS_TSTATE, (size_t)tiles + 1);
  h.timer.begin(s, "lr.tiles", 12.0 * E);  // succ read + segment id + offset per arc
  CK(cudaMemsetAsync(state, 0, ((size_t)tiles + 1) * sizeof(unsigned long long), s));
  if (verify || dbg) CK(cudaMemsetAsync(h.dev_box + 14, 0, 2 * sizeof(int64_t), s));
  auto launch = [&](auto kern, int threads, size_t smem) {
    set_smem(kern, smem);
    kern<<<tiles, threads, smem, s>>>((uint32_t)N, S, lab, cc_slots, (uint32_t)T, seg, off,
                                      seg_len, seg_exit, nseg, state,
                                      verify || dbg ? walked : nullptr);
  };
  static const int stride1 = env_int("RSTG_LR_STRIDE", 16);
  if (slots == 16384)
    launch(k_tile_rank<16384, 1024, 32>, 1024, tile_rank_smem<16384>());
  else if (slots == 2048)
    launch(k_tile_rank<2048, 256, 16>, 256, tile_rank_smem<2048>());
  else if (slots == 4096)
    launch(k_tile_rank<4096, 512, 16>, 512, tile_rank_smem<4096>());
  else if (stride1 <= 4)
    launch(k_tile_rank<8192, 1024, 4>, 1024, tile_rank_smem<8192>());
  else if (stride1 <= 8)
    launch(k_tile_rank<8192, 1024, 8>, 1024, tile_rank_smem<8192>());
  else
    launch(k_tile_rank<8192, 1024, 16>, 1024, tile_rank_smem<8192>());
  CK_LAUNCH();
  h.stats.step(E, 2);
  // The segment count sizes the level grids. A repeated build of the same
  // graph takes it from the previous build (plus a margin: the count
  // depends only on the tree and, by one segment, on the root) instead of
  // a host round trip here; the levels raise their overflow flag if the
  // bound was short, and the settle step after the build re-ranks then.
  const bool deferred = !verify && !dbg && h.tile_segments >= 0;
  int64_t R;
  if (deferred) {
    R = std::min<int64_t>(E, h.tile_segments + h.tile_segments / 8 + 8192);
    const int forced = env_int("RSTG_LR_SEGBOUND", 0);  // (tests: a short bound)
    if (forced > 0) R = forced;
  } else {
    h.read_box(h.dev_box + 8, 8);  // [8] segments, [14] arcs walked, [15] jump rounds
    R = h.host_box[0];
    h.tile_segments = R;
    if (dbg)
      fprintf(stderr, "lr.tiles: %lld arcs -> %lld segments (%.1fx), %lld jump rounds\n",
              (long long)(2 * T), (long long)R, R ? 2.0 * T / R : 0.0, (long long)h.host_box[7]);
    if (verify && h.host_box[6] != 2 * T)  // a cycle inside a tile has no head
      throw AlgoError("list ranking failed to converge: not a forest");
  }
  h.timer.end(s);

  h.timer.begin(s, "lr.rulers_rank", 16.0 * R);
  // fixed StepReport charge (the segment count follows the tour layout)
  const Stats before = h.stats;
  LrParams Q = P;
  Q.cap = std::max<int64_t>(P.cap, E + 1);  // (level arenas sized by the fixed bound)
  const int levels_env = env_int("RSTG_LR_TILELEVELS", 1);  // (0: segments by list_prefix)
  bool late = false;
  if (levels_env && R * 4 <= E) {
    if (tile_prefix_levels(h, R, S, seg, seg_exit, seg_len, segstart, dbg, deferred))
      late = deferred;
    else
      tile_fallback(h, Q, R, seg, seg_exit, seg_len, seg_next, segstart, nseg);
  } else {
    if (deferred) {  // (the exact count is needed here)
      h.read_box(h.dev_box + 8, 1);
      R = h.host_box[0];
      h.tile_segments = R;
    }
    tile_fallback(h, Q, R, seg, seg_exit, seg_len, seg_next, segstart, nseg);
  }
  const int64_t launches = h.stats.launches;
  h.stats = before;
  h.stats.launches = launches;
  const int64_t Rexp = std::max<int64_t>(E >> P.logk0, 2);
  int rounds = 1;
  while ((int64_t{1} << (rounds - 1)) < Rexp) ++rounds;
  h.stats.steps += rounds;
  h.stats.work += Rexp * rounds;
  h.timer.end(s);
  return TileRank{seg, off, segstart, late};
}

bool tile_rank_settle(Handle& h, const LrParams& P, int64_t N, const TileRank& tr) {
  if (!tr.deferred) return false;
  const int64_t R = h.host_box[32];  // level-1 segment count (copied with the flag)
  const bool overflow = *reinterpret_cast<const int*>(&h.host_box[32 + 16]) != 0;
  h.tile_segments = R;
  if (!overflow) return false;
  const int64_t E = 2 * N;
  LrParams Q = P;
  Q.cap = std::max<int64_t>(P.cap, E + 1);
  tile_fallback(h, Q, R, tr.seg, h.ws<uint32_t>(WS_RNEXT, E + 1), h.ws<uint32_t>(WS_RLEN, E + 1),
                h.ws<uint32_t>(WS_RPOS, E + 1), const_cast<uint32_t*>(tr.segstart),
                reinterpret_cast<unsigned long long*>(h.dev_box) + 8);
  return true;
}

}  // namespace rstg
