// listrank.cuh -- sparse ruling-set list ranking: device helpers shared by
// the producers of the lists (euler.cu registers rulers inside its own
// passes) and the ranking driver (listrank.cu).
//
// Level 0 (the Euler tour, E arcs, succ[] NONE-terminated): a position p is
// a ruler when hash(p) falls in a 1/2^logk bucket, or when it heads a list.
// Its word is sl[p] = (ruler id << ob) | offset, offset = hops from the
// ruler (the ruler itself has offset 0); rank(p) = rstart[id] + offset.
#pragma once

#include "common.cuh"
#include "scan.cuh"

namespace rstg {

struct LrParams {
  int logk0 = 5;      // level-0 ruler density 1/2^logk0
  int logk1 = 3;      // ruler density of the ruler-list levels
  int chains = 1;     // walks in flight per thread (more thrash the L2)
  bool coop_levels = false;  // ruler-list levels in one cooperative launch
  int walk_blocks = 4;  // CTAs per SM of the level-0 walk
  uint32_t chunk = 64;  // ruler ids per round-robin chunk
  int ob = 10;        // offset bits of the level-0 word
  uint32_t walk_cap;  // longest walk before a split, (1 << ob) - 1
  int64_t cap;        // ruler-id capacity
};

#ifdef __CUDACC__
__device__ __forceinline__ bool lr_hash_ruler(uint32_t p, int logk) {
  return ((p * 0x9E3779B1u) >> (32 - logk)) == 0u;
}

// Registers position p as a ruler for every lane with want set. All 32
// lanes of the warp must call it together (warp-aggregated id claim).
// Ids at or beyond cap are counted but not stored (the caller checks the
// count against cap and throws).
__device__ __forceinline__ void lr_register_warp(bool want, uint32_t p, uint32_t* rpos, uint32_t* sl,
                                                 unsigned long long* ctr, int ob, uint32_t cap) {
  const unsigned mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(mask) - 1) base = (uint32_t)atomicAdd(ctr, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
  if (want) {
    const uint32_t id = base + __popc(mask & ((1u << lane) - 1u));
    if (id < cap) {
      rpos[id] = p;
      sl[p] = id << ob;
    }
  }
}

// Tile-ordered id claim: CTA-wide exclusive scan of per-thread counts and
// one global atomic per CTA tile, so the ids of a tile's rulers are one
// contiguous range (the persistent walk hands a CTA a contiguous id range:
// its chains then start in one region of the tour and share cache lines)
// and the counter sees one atomic per tile, not per warp. Every thread of
// the CTA must call it; returns the thread's first id.
__device__ __forceinline__ uint32_t lr_block_claim(uint32_t c, unsigned long long* ctr) {
  __shared__ uint32_t s_total;
  __shared__ uint32_t s_base;
  const uint32_t off = block_excl_scan(c, &s_total);
  if (threadIdx.x == 0) s_base = s_total ? (uint32_t)atomicAdd(ctr, (unsigned long long)s_total) : 0u;
  __syncthreads();
  const uint32_t b = s_base + off;
  __syncthreads();
  return b;
}
// Registers position p as ruler `id`: rpos[id] = p, sl[p] = id << ob.
__device__ __forceinline__ void lr_put(uint32_t id, uint32_t p, uint32_t* rpos, uint32_t* sl, int ob,
                                       uint32_t cap) {
  if (id < cap) {
    rpos[id] = p;
    sl[p] = id << ob;
  }
}
#endif

class Handle;
// E positions (holes included), at most heads_bound lists, `arcs` positions
// actually on the lists (-1: all E).
LrParams lr_params(int64_t E, int64_t heads_bound, int64_t arcs = -1);

// Walks every registered ruler (ids [0, *ctr) on the device, positions in
// rpos) over succ and fills sl, for every position a walk reached, with
// its word (ruler id << ob) | offset; then ranks the ruler lists. Returns
// rstart (device, by ruler id): rank(p) = rstart[sl[p] >> ob] + (sl[p] & mask).
// When verify, the walks must cover exactly `expect` positions (else a
// cycle without a ruler exists) and the ruler lists must be acyclic, or
// the reference's "list ranking failed to converge: not a forest" is thrown.
const uint32_t* lr_rank(Handle& h, const LrParams& P, int64_t E, const uint32_t* succ, uint32_t* sl,
                        uint32_t* rpos, unsigned long long* ctr, bool verify, int64_t expect,
                        int64_t* R_out);

// pre[x] = sum of w over the nodes before x in its list (recursive ruling
// sets; level arenas sized by max(N, P.cap)).
void list_prefix(Handle& h, const LrParams& P, int64_t N, const uint32_t* next, const uint32_t* w,
                 uint32_t* pre, int depth, bool verify, int* bad);

// Tile-contracted ranking of the Euler tour (tilerank.cu): each CTA ranks
// the arcs of a tile of consecutive slots on chip (maximal runs of tour
// successors inside the tile = segments, numbered in tile order), then the
// segment list is contracted by tiles again, level after level (list_prefix
// when that stalls). rank(x) = segstart[seg[x]] + off[x].
struct TileRank {
  const uint32_t* seg;       // 2N segment id per arc
  const uint16_t* off;       // 2N offset within the segment
  const uint32_t* segstart;  // rank of each segment's first arc
  // The upper levels ran on a grid sized from the previous build's segment
  // count: their overflow flag and the real count are copied to
  // host_box[32..49) asynchronously; tile_rank_settle() checks them after
  // the build's final sync (and re-ranks the segments when they overflowed).
  bool deferred = false;
};
TileRank lr_rank_tiles(Handle& h, const LrParams& P, int64_t N, const uint32_t* S,
                       const int32_t* lab, bool cc_slots, int64_t T, bool verify);
// After the stream has synced: true when the deferred levels overflowed and
// segstart has been recomputed on the stream (the caller re-derives the
// parents); records the segment count for the next build either way.
bool tile_rank_settle(Handle& h, const LrParams& P, int64_t N, const TileRank& tr);

// Generic entry (rstg_k_list_rank, explicit lists): registers hash rulers
// and every list head (positions without a predecessor), then lr_rank.
const uint32_t* lr_rank_lists(Handle& h, int64_t E, const uint32_t* succ, uint32_t* sl, bool verify,
                              LrParams* P_out);

}  // namespace rstg
