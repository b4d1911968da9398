// scan.cuh -- tiled exclusive scan / stream compaction over a functor.
//
// Three passes (tile counts -> scan of tile counts -> tile rescan + emit).
// The input is a device functor f(i) -> uint32 (typically a flag computed
// on the fly from graph arrays), so no n-sized input array is needed; the
// emit functor consumes (i, exclusive prefix, value) in coalesced order.
// Memory: one uint32 per 4096-element tile.
#pragma once

#include "common.cuh"
#include "engine.hpp"

namespace rstg {

constexpr int kScanItems = 16;
constexpr int kScanTile = kBlock * kScanItems;  // 4096
#define RSTG_PAD(i) ((i) + ((i) >> 5))

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

// Exclusive block scan of one value per thread; returns prefix, *total set.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[kBlock / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = warp_incl_scan(v);
  if (lane == 31) warp_sums[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = (lane < kBlock / 32) ? warp_sums[lane] : 0;
    uint32_t si = warp_incl_scan(s);
    if (lane < kBlock / 32) warp_sums[lane] = si - s;
    if (lane == kBlock / 32 - 1) *total = si;
  }
  __syncthreads();
  uint32_t r = warp_sums[wid] + inc - v;
  __syncthreads();
  return r;
}

template <class F>
__global__ void __launch_bounds__(kBlock) k_scan_tile_count(F f, int64_t n, uint32_t* partial) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t sum = 0;
#pragma unroll 4
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k * kBlock + threadIdx.x;
    if (i < n) sum += f(i);
  }
  __shared__ uint32_t tot;
  block_excl_scan(sum, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// In-place exclusive scan of `count` partials by one CTA; partial[count] = total.
__global__ void k_scan_partials(uint32_t* partial, int64_t count);

template <class F, class Emit>
__global__ void __launch_bounds__(kBlock)
    k_scan_tile_emit(F f, int64_t n, const uint32_t* partial, Emit emit) {
  __shared__ uint32_t vals[RSTG_PAD(kScanTile)];
  __shared__ uint32_t pref[RSTG_PAD(kScanTile)];
  __shared__ uint32_t tot;
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
#pragma unroll 4
  for (int k = 0; k < kScanItems; ++k) {
    int li = k * kBlock + threadIdx.x;
    int64_t i = base + li;
    vals[RSTG_PAD(li)] = (i < n) ? f(i) : 0u;
  }
  __syncthreads();
  uint32_t local[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int li = threadIdx.x * kScanItems + k;
    local[k] = s;
    s += vals[RSTG_PAD(li)];
  }
  uint32_t tp = block_excl_scan(s, &tot) + partial[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int li = threadIdx.x * kScanItems + k;
    pref[RSTG_PAD(li)] = tp + local[k];
  }
  __syncthreads();
#pragma unroll 4
  for (int k = 0; k < kScanItems; ++k) {
    int li = k * kBlock + threadIdx.x;
    int64_t i = base + li;
    if (i < n) emit(i, pref[RSTG_PAD(li)], vals[RSTG_PAD(li)]);
  }
}

// Runs the scan; returns the total (one host sync) when want_total.
template <class F, class Emit>
uint32_t scan_emit(Handle& h, int64_t n, F f, Emit emit, bool want_total, int slot = WS_SCAN) {
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  uint32_t* partial = h.ws<uint32_t>(slot, tiles + 1);
  if (tiles > 0) {
    k_scan_tile_count<<<(unsigned)tiles, kBlock, 0, h.stream>>>(f, n, partial);
    CK_LAUNCH();
  }
  k_scan_partials<<<1, 1024, 0, h.stream>>>(partial, tiles);
  CK_LAUNCH();
  if (tiles > 0) {
    k_scan_tile_emit<<<(unsigned)tiles, kBlock, 0, h.stream>>>(f, n, partial, emit);
    CK_LAUNCH();
  }
  h.stats.step(n, 3);
  if (!want_total) return 0;
  CK(cudaMemcpyAsync(h.host_box, partial + tiles, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                     h.stream));
  CK(cudaStreamSynchronize(h.stream));
  return *reinterpret_cast<uint32_t*>(h.host_box);
}

// out[i] = exclusive prefix for i in [0,n), out[n] = total.
struct EmitExcl {
  uint32_t* out;
  int64_t n;
  __device__ void operator()(int64_t i, uint32_t p, uint32_t v) const {
    out[i] = p;
    if (i == n - 1) out[n] = p + v;
  }
};
// Stream compaction: out[p] = i for flagged i (ascending order kept).
struct EmitCompact {
  uint32_t* out;
  __device__ void operator()(int64_t i, uint32_t p, uint32_t v) const {
    if (v) out[p] = (uint32_t)i;
  }
};

}  // namespace rstg
