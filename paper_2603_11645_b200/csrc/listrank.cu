// listrank.cu -- sparse ruling-set list ranking (replaces the Wyllie loop of
// list_rank, euler_rooting.cpp:104-153, which costs ceil(log2 E) full
// passes over all E arcs).
//
//   1. rulers = every arc whose multiplicative hash falls in a 1/K bucket
//      (found by one index-only pass, ids handed out by warp-aggregated
//      atomics), plus every list head (heads have no predecessor, so no
//      walk would ever reach them);
//   2. one thread per ruler walks its sublist (succ chain) until the next
//      ruler or the list tail, writing a 32-bit (ruler id, offset) word per
//      arc; a walk longer than kWalkCap turns the next arc into a fresh
//      ruler and stops, so a launch is bounded by kWalkCap dependent loads
//      and the geometric tail is handled by a few short follow-up launches;
//   3. the ruler list (about E/K nodes) is prefix-summed by Jacobi pointer
//      jumping on packed (prefix, jump) words;
//   4. rank(arc) = rstart[ruler] + offset, evaluated by the consumer.
// Ranks equal the reference's list_rank output (distance from the head):
// checked arc for arc against the reference's own ranks
// (tests/golden/euler_ranks.npz) and the oracle's Wyllie restatement.
#include "engine.hpp"
#include "scan.cuh"

namespace rstg {

constexpr int kLogK = 5;  // ruler density 1/32
constexpr uint32_t kWalkCap = 64;
constexpr int kOffBits = 7;  // sl word = (ruler id << 7) | offset, offset <= kWalkCap
constexpr uint32_t kOffMask = (1u << kOffBits) - 1u;
constexpr uint32_t kMaxRulers = (1u << (32 - kOffBits)) - 2u;  // all-ones = unvisited
static_assert(kWalkCap <= kOffMask, "offset field too narrow");

__device__ __forceinline__ bool is_hash_ruler(uint32_t p) {
  return ((p * 0x9E3779B1u) >> (32 - kLogK)) == 0u;
}

// Hash rulers: an index-only pass; each 4096-position tile counts its
// rulers with a block scan and claims its id range with one atomicAdd.
// sl[ruler] = (id, 0).
constexpr int kRulerItems = 16;
__global__ void __launch_bounds__(kBlock)
    k_find_rulers(int64_t E, uint32_t* __restrict__ rpos, uint32_t* __restrict__ sl,
                  unsigned long long* counter) {
  __shared__ uint32_t s_total;
  __shared__ unsigned long long s_base;
  const int64_t tile_len = (int64_t)kBlock * kRulerItems;
  for (int64_t tile = blockIdx.x; tile * tile_len < E; tile += gridDim.x) {
    const int64_t p0 = tile * tile_len + (int64_t)threadIdx.x * kRulerItems;
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < kRulerItems; ++k) {
      const int64_t p = p0 + k;
      mine |= (p < E && is_hash_ruler((uint32_t)p)) ? (1u << k) : 0u;
    }
    const uint32_t off = block_excl_scan(__popc(mine), &s_total);
    if (threadIdx.x == 0) s_base = s_total ? atomicAdd(counter, (unsigned long long)s_total) : 0;
    __syncthreads();
    uint32_t id = (uint32_t)s_base + off;
    while (mine) {
      const int k = __ffs(mine) - 1;
      mine &= mine - 1;
      rpos[id] = (uint32_t)(p0 + k);
      sl[p0 + k] = id << kOffBits;
      ++id;
    }
    __syncthreads();
  }
}

__global__ void k_append_heads(const uint32_t* heads, int64_t H, uint32_t* rpos, uint32_t* sl,
                               unsigned long long* counter) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < H;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t hd = heads[i];
    if (is_hash_ruler(hd)) continue;
    const uint32_t id = (uint32_t)atomicAdd(counter, 1ull);
    rpos[id] = hd;
    sl[hd] = id << kOffBits;
  }
}

// One thread per ruler in [lo, hi). Dynamic rulers are appended at
// *rcount (device counter) and walked by the next launch.
__global__ void __launch_bounds__(kBlock)
    k_walk(const uint32_t* __restrict__ succ, int stride, uint32_t* rpos, uint32_t* __restrict__ rlen,
           uint32_t* __restrict__ rnext, uint32_t* sl, uint32_t lo, uint32_t hi,
           unsigned long long* rcount) {
  const int64_t t = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= hi) return;
  const uint32_t i = (uint32_t)t;
  const uint32_t tag = i << kOffBits;
  uint32_t cur = succ[(size_t)rpos[i] * stride];
  uint32_t off = 1;
  uint32_t nxt = kNone32;
  for (;;) {
    if (cur == kNone32) break;
    if (is_hash_ruler(cur)) {
      nxt = ld_cg(&sl[cur]) >> kOffBits;
      break;
    }
    if (off > kWalkCap) {  // split: cur becomes a new ruler
      const uint32_t nid = (uint32_t)atomicAdd(rcount, 1ull);
      rpos[nid] = cur;
      sl[cur] = nid << kOffBits;
      nxt = nid;
      break;
    }
    sl[cur] = tag | off;
    ++off;
    cur = succ[(size_t)cur * stride];
  }
  rlen[i] = off;
  rnext[i] = nxt;
}

// pred over the ruler list, packed Wyllie word (prefix << 32 | jump).
__global__ void k_ruler_pred(int64_t R, const uint32_t* rnext, uint32_t* pred) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t nx = rnext[i];
    if (nx != kNone32) pred[nx] = (uint32_t)i;
  }
}
__global__ void k_ruler_wyllie_init(int64_t R, const uint32_t* pred, const uint32_t* rlen,
                                    unsigned long long* w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = pred[i];
    w[i] = (p == kNone32) ? (unsigned long long)kNone32 : (((unsigned long long)rlen[p] << 32) | p);
  }
}
__global__ void k_ruler_wyllie(int64_t R, const unsigned long long* __restrict__ w,
                               unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = w[i];
    const uint32_t j = (uint32_t)x;
    if (j == kNone32) {
      out[i] = x;
      continue;
    }
    const unsigned long long y = w[j];
    out[i] = (((x >> 32) + (y >> 32)) << 32) | (y & 0xffffffffull);
  }
}
// Verification (only for caller-supplied structures that may not be
// forests): every ruler chain must have ended and every arc been visited.
__global__ void k_lr_verify(int64_t R, const unsigned long long* w, int64_t E, const uint32_t* sl,
                            int* bad) {
  const int64_t total = R > E ? R : E;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < R && (uint32_t)w[i] != kNone32) *bad = 1;
    if (i < E && sl[i] == kNone32) *bad = 1;
  }
}
__global__ void k_ruler_extract(int64_t R, const unsigned long long* w, uint32_t* rstart) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x)
    rstart[i] = (uint32_t)(w[i] >> 32);
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

// Returns rstart (device, R entries); sl filled for every arc:
// rank(p) = rstart[sl[p] >> 7] + (sl[p] & 127).
const uint32_t* list_rank_rulers(Handle& h, int64_t E, const uint32_t* succ, int stride,
                                 const uint32_t* heads, int64_t H, uint32_t* sl, int64_t* R_out,
                                 bool verify) {
  const int64_t cap = E / (1 << kLogK) * 2 + H + E / kWalkCap + 64;
  uint32_t* rpos = h.ws<uint32_t>(WS_RPOS, cap);
  uint32_t* rlen = h.ws<uint32_t>(WS_RLEN, cap);
  uint32_t* rnext = h.ws<uint32_t>(WS_RNEXT, cap);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 8;

  h.timer.begin(h.stream, "lr.rulers");
  if (verify) CK(cudaMemsetAsync(sl, 0xFF, E * sizeof(uint32_t), h.stream));
  CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), h.stream));
  k_find_rulers<<<grid_for(E), kBlock, 0, h.stream>>>(E, rpos, sl, ctr);
  if (H > 0) k_append_heads<<<grid_for(H), kBlock, 0, h.stream>>>(heads, H, rpos, sl, ctr);
  CK_LAUNCH();
  h.stats.step(E, H > 0 ? 2 : 1);
  h.read_box(reinterpret_cast<int64_t*>(ctr), 1);
  uint32_t R = (uint32_t)h.host_box[0];
  if ((int64_t)R > cap) throw std::runtime_error("ruler capacity exceeded");
  h.timer.end(h.stream);

  // Walks; dynamic rulers are counted from R upwards.
  h.timer.begin(h.stream, "lr.walk");
  uint32_t lo = 0, hi = R;
  while (lo < hi) {
    if ((int64_t)hi + (int64_t)(hi - lo) > std::min<int64_t>(cap, kMaxRulers))
      throw std::runtime_error("list ranking: ruler capacity exceeded");
    const unsigned grid = (unsigned)((hi - lo + kBlock - 1) / kBlock);
    k_walk<<<grid, kBlock, 0, h.stream>>>(succ, stride, rpos, rlen, rnext, sl, lo, hi, ctr);
    CK_LAUNCH();
    h.stats.launches++;
    h.read_box(reinterpret_cast<int64_t*>(ctr), 1);
    lo = hi;
    hi = (uint32_t)h.host_box[0];
  }
  // Counters stay deterministic although the number of follow-up walks
  // (dynamic rulers) depends on the tour layout: one logical barrier, E arcs.
  h.stats.steps++;
  h.stats.work += E;
  const int64_t R_static = R;
  R = hi;
  h.timer.end(h.stream);

  // Prefix over the ruler lists.
  h.timer.begin(h.stream, "lr.rulers_rank");
  // sized by the deterministic capacity, not R (R varies with the tour
  // layout; a grow-only buffer must not reallocate inside the timed loop)
  uint32_t* pred = h.ws<uint32_t>(WS_RA, cap);
  unsigned long long* wa = h.ws<unsigned long long>(WS_RB, cap);
  unsigned long long* wb = h.ws<unsigned long long>(WS_RC, cap);
  uint32_t* rstart = h.ws<uint32_t>(WS_RD, cap);
  CK(cudaMemsetAsync(pred, 0xFF, R * sizeof(uint32_t), h.stream));
  const unsigned g = grid_for(R);
  k_ruler_pred<<<g, kBlock, 0, h.stream>>>(R, rnext, pred);
  k_ruler_wyllie_init<<<g, kBlock, 0, h.stream>>>(R, pred, rlen, wa);
  CK_LAUNCH();
  h.stats.step(R_static, 2);
  // round count from the deterministic capacity (>= ceil(log2 R) + 1)
  const int rounds = ceil_log2_i(cap < 2 ? 2 : cap) + 1;
  for (int r = 0; r < rounds; ++r) {
    k_ruler_wyllie<<<g, kBlock, 0, h.stream>>>(R, wa, wb);
    CK_LAUNCH();
    h.stats.step(R_static);
    std::swap(wa, wb);
  }
  k_ruler_extract<<<g, kBlock, 0, h.stream>>>(R, wa, rstart);
  CK_LAUNCH();
  h.stats.step(R_static);
  if (verify) {
    int* bad = reinterpret_cast<int*>(h.dev_box + 52);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), h.stream));
    k_lr_verify<<<grid_for(std::max<int64_t>(R, E)), kBlock, 0, h.stream>>>(R, wa, E, sl, bad);
    CK_LAUNCH();
    h.read_box(reinterpret_cast<int64_t*>(bad), 1);
    if (*reinterpret_cast<int*>(h.host_box))
      throw AlgoError("list ranking failed to converge: not a forest");
  }
  h.timer.end(h.stream);
  if (R_out) *R_out = R;
  return rstart;
}

}  // namespace rstg
