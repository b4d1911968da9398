// listrank.cu -- sparse ruling-set list ranking (replaces the Wyllie loop of
// list_rank, euler_rooting.cpp:104-153, which costs ceil(log2 E) full
// passes over all E arcs).
//
//   1. rulers = every arc whose multiplicative hash falls in a 1/K bucket,
//      plus every list head (heads have no predecessor, so no walk would
//      ever reach them);
//   2. one thread per ruler walks its sublist (succ chain) until the next
//      ruler or the list tail, writing (ruler id, offset) per arc; a walk
//      longer than kWalkCap spawns a fresh ruler and stops, so one launch
//      is bounded by kWalkCap dependent loads and the geometric tail is
//      handled by a few short follow-up launches;
//   3. the ruler list (about E/K nodes) is prefix-summed by Jacobi pointer
//      jumping on packed (prefix, jump) words;
//   4. rank(arc) = rstart[ruler] + offset, evaluated by the consumer.
// Ranks equal the reference's list_rank output (distance from the head);
// the property is checked arc-for-arc in tests/test_gpu_parity.py.
#include "engine.hpp"
#include "scan.cuh"

namespace rstg {

constexpr int kLogK = 5;  // ruler density 1/32
constexpr uint32_t kWalkCap = 128;

__device__ __forceinline__ bool is_hash_ruler(uint32_t p) {
  return ((p * 0x9E3779B1u) >> (32 - kLogK)) == 0u;
}

namespace {
struct HashRulerFlag {
  __device__ uint32_t operator()(int64_t p) const { return is_hash_ruler((uint32_t)p) ? 1u : 0u; }
};
}  // namespace

__global__ void k_append_heads(const uint32_t* heads, int64_t H, uint32_t* rpos, uint32_t R0,
                               unsigned long long* counter) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < H;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t hd = heads[i];
    if (is_hash_ruler(hd)) continue;
    uint32_t k = (uint32_t)atomicAdd(counter, 1ull);
    rpos[R0 + k] = hd;
  }
}

__global__ void k_init_rulers(const uint32_t* rpos, int64_t R, unsigned long long* sl) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x)
    sl[rpos[i]] = (unsigned long long)i << 32;
}

// Walk sublists of rulers [lo, hi). Dynamic rulers are appended at
// *rcount (device counter) and walked by the next launch.
__global__ void __launch_bounds__(kBlock)
    k_walk(const uint32_t* __restrict__ succ, int stride, uint32_t* rpos, uint32_t* __restrict__ rlen,
           uint32_t* __restrict__ rnext, unsigned long long* sl, uint32_t lo, uint32_t hi,
           unsigned long long* rcount) {
  for (int64_t t = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < hi;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)t;
    const unsigned long long tag = (unsigned long long)i << 32;
    uint32_t cur = succ[(size_t)rpos[i] * stride];
    uint32_t off = 1;
    uint32_t nxt = kNone32;
    for (;;) {
      if (cur == kNone32) break;
      if (is_hash_ruler(cur)) {
        nxt = (uint32_t)(ld_cg(&sl[cur]) >> 32);
        break;
      }
      if (off > kWalkCap) {  // split: cur becomes a new ruler
        uint32_t nid = (uint32_t)atomicAdd(rcount, 1ull);
        rpos[nid] = cur;
        sl[cur] = (unsigned long long)nid << 32;
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
}

// pred over the ruler list, packed Wyllie word (prefix << 32 | jump).
__global__ void k_ruler_pred(int64_t R, const uint32_t* rnext, uint32_t* pred) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t nx = rnext[i];
    if (nx != kNone32) pred[nx] = (uint32_t)i;
  }
}
__global__ void k_ruler_wyllie_init(int64_t R, const uint32_t* pred, const uint32_t* rlen,
                                    unsigned long long* w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t p = pred[i];
    w[i] = (p == kNone32) ? (unsigned long long)kNone32
                          : (((unsigned long long)rlen[p] << 32) | p);
  }
}
__global__ void k_ruler_wyllie(int64_t R, const unsigned long long* __restrict__ w,
                               unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long x = w[i];
    uint32_t j = (uint32_t)x;
    if (j == kNone32) {
      out[i] = x;
      continue;
    }
    unsigned long long y = w[j];
    out[i] = (((x >> 32) + (y >> 32)) << 32) | (y & 0xffffffffull);
  }
}
// Verification (only for caller-supplied structures that may not be
// forests): every ruler chain must have ended and every arc been visited.
__global__ void k_lr_verify(int64_t R, const unsigned long long* w, int64_t E,
                            const unsigned long long* sl, int* bad) {
  const int64_t total = R > E ? R : E;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < R && (uint32_t)w[i] != kNone32) *bad = 1;
    if (i < E && sl[i] == ~0ull) *bad = 1;
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

// Returns rstart (device, R entries); sl filled for every arc.
const uint32_t* list_rank_rulers(Handle& h, int64_t E, const uint32_t* succ, int stride,
                                 const uint32_t* heads, int64_t H, unsigned long long* sl,
                                 int64_t* R_out, bool verify) {
  const int64_t cap = E / (1 << kLogK) * 2 + H + E / kWalkCap + 64;
  uint32_t* rpos = h.ws<uint32_t>(WS_RPOS, cap);
  uint32_t* rlen = h.ws<uint32_t>(WS_RLEN, cap);
  uint32_t* rnext = h.ws<uint32_t>(WS_RNEXT, cap);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(h.dev_box) + 8;

  h.timer.begin(h.stream, "lr.rulers");
  if (verify) CK(cudaMemsetAsync(sl, 0xFF, E * sizeof(unsigned long long), h.stream));
  const uint32_t R0 = scan_emit(h, E, HashRulerFlag{}, EmitCompact{rpos}, true);
  if ((int64_t)R0 + H > cap) throw std::runtime_error("ruler capacity exceeded");
  CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), h.stream));
  if (H > 0) {
    k_append_heads<<<grid_for(H), kBlock, 0, h.stream>>>(heads, H, rpos, R0, ctr);
    CK_LAUNCH();
    h.stats.step(H);
  }
  h.read_box(reinterpret_cast<int64_t*>(ctr), 1);
  uint32_t R = R0 + (uint32_t)h.host_box[0];
  k_init_rulers<<<grid_for(R), kBlock, 0, h.stream>>>(rpos, R, sl);
  CK_LAUNCH();
  h.stats.step(R);
  h.timer.end(h.stream);

  // Walks; dynamic rulers are counted from R upwards.
  h.timer.begin(h.stream, "lr.walk");
  h.host_box[0] = R;
  CK(cudaMemcpyAsync(ctr, h.host_box, sizeof(unsigned long long), cudaMemcpyHostToDevice,
                     h.stream));
  uint32_t lo = 0, hi = R;
  while (lo < hi) {
    if ((int64_t)hi + (int64_t)(hi - lo) > cap) throw std::runtime_error("walk capacity");
    k_walk<<<grid_for(hi - lo), kBlock, 0, h.stream>>>(succ, stride, rpos, rlen, rnext, sl, lo, hi,
                                                        ctr);
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
