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
//     depend on the evaluation order, so one asynchronous path-halving
//     kernel replaces the ceil(log2 L) doubling barriers.
// Hook rounds stay synchronous: proposals read
// reps frozen by the previous kernel boundary.
#include "engine.hpp"
#include "scan.cuh"

namespace rstg {

__global__ void k_cc_init(int64_t n, int32_t* rep, unsigned long long* slot) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    rep[v] = (int32_t)v;
    slot[v] = kKeyInf;
  }
}

// hook_step edge pass (cc_forest.cpp:18-35) / graft proposals (pr_rst.cpp:82-99).
template <int MODE>
__global__ void __launch_bounds__(kBlock)
    k_hook(const int2* __restrict__ edges, int64_t m, uint32_t e_base,
           const int32_t* __restrict__ rep, unsigned long long* __restrict__ slot,
           int* any_proposal) {
  bool proposed = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 e = edges[i];
    const int32_t ru = rep[e.x], rv = rep[e.y];
    if (ru == rv) continue;
    const int32_t lo = min(ru, rv), hi = max(ru, rv);
    const int32_t winner = MODE == 0 ? lo : hi;
    const int32_t loser = MODE == 0 ? hi : lo;
    const unsigned long long key = pack_key((uint32_t)winner, e_base + (uint32_t)i);
    proposed = true;
    if (key < slot[loser]) atomicMin(&slot[loser], key);
  }
  if (any_proposal) block_flag(proposed, any_proposal);
}

// Apply step (cc_forest.cpp:39-46); counts applied hooks = new tree edges.
__global__ void __launch_bounds__(kBlock)
    k_apply(int64_t n, int32_t* __restrict__ rep, unsigned long long* __restrict__ slot,
            uint8_t* __restrict__ tflag, uint32_t e_base, uint32_t m_local,
            unsigned long long* counter) {
  uint32_t cnt = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = slot[v];
    if (key == kKeyInf) continue;
    rep[v] = (int32_t)(key >> 32);
    const uint32_t e = (uint32_t)key - e_base;
    if (tflag && e < m_local) tflag[e] = 1;
    slot[v] = kKeyInf;
    ++cnt;
  }
  // block reduce
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

// Asynchronous pointer jumping to the fixed point of
// jump_to_convergence: every rep[v] ends at the root of v's rep tree.
// Each step reads an ancestor; any value ever stored in rep[x] is a proper
// ancestor of x (roots never change), so the walk strictly ascends and the
// path-halving stores only shorten other threads' walks.
__global__ void __launch_bounds__(kBlock) k_compress(int64_t n, int32_t* rep) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t p = rep[v];
    if (p == (int32_t)v) continue;
    int32_t gp = ld_cg(&rep[p]);
    if (gp == p) continue;
    do {
      rep[v] = gp;
      p = gp;
      gp = ld_cg(&rep[p]);
    } while (gp != p);
  }
}

// One in-place doubling round rep[v] = rep[rep[v]] (the Jacobi step of
// jump_to_convergence, evaluated in place: a fresher read only jumps
// further). A round that changes nothing proves every rep[v] is a root
// (roots are the only fixed points of a forest), so later rounds exit on
// the device without a host round trip.
template <int HOPS>
__global__ void __launch_bounds__(kBlock) k_jump_round(int64_t n, int32_t* rep, int* flags,
                                                       int round) {
  if (round > 0 && flags[round - 1] == 0) return;
  bool changed = false;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = rep[v];
    int32_t x = rep[p];
    if (x == p) continue;
#pragma unroll
    for (int hop = 1; hop < HOPS; ++hop) {
      const int32_t y = rep[x];
      if (y == x) break;
      x = y;
    }
    rep[v] = x;
    changed = true;
  }
  block_flag(changed, &flags[round]);
}

static int jump_hops() {
  static int hops = 0;
  if (hops == 0) {
    const char* e = getenv("RSTG_JUMP_HOPS");
    hops = e ? atoi(e) : 1;
    if (hops != 1 && hops != 2 && hops != 4 && hops != 8) hops = 1;
  }
  return hops;
}

void launch_jump_rounds(Handle& h, int32_t* rep, int64_t n) {
  int rounds = 2;
  while ((int64_t{1} << (rounds - 2)) < n) ++rounds;  // ceil(log2 n) + 2
  int* flags = reinterpret_cast<int*>(h.dev_box + 128);  // 64 ints (dev_box[128..159])
  CK(cudaMemsetAsync(flags, 0, 64 * sizeof(int), h.stream));
  const unsigned g = grid_for(n);
  const int hops = jump_hops();
  for (int r = 0; r < rounds && r < 64; ++r) {
    if (hops == 1) k_jump_round<1><<<g, kBlock, 0, h.stream>>>(n, rep, flags, r);
    else if (hops == 2) k_jump_round<2><<<g, kBlock, 0, h.stream>>>(n, rep, flags, r);
    else if (hops == 4) k_jump_round<4><<<g, kBlock, 0, h.stream>>>(n, rep, flags, r);
    else k_jump_round<8><<<g, kBlock, 0, h.stream>>>(n, rep, flags, r);
    h.stats.step(n);
  }
  CK_LAUNCH();
}

// ---- two-level shortcutting ---------------------------------------------
// Level 1 (k_tile_resolve): each CTA owns a tile of kTileV consecutive
// vertices held in shared memory and follows every pointer while it stays
// inside the tile (in-smem doubling), so rep[v] becomes either a root or the
// first ancestor outside v's tile. Those out-of-tile targets X are flagged.
// Level 2: X is compacted and pointer-jumped on its own (its pointers stay
// inside X or hit roots); a last gather rep[v] = rep[rep[v]] finishes.
// Passes over all n: 3 (tile, compaction, final) instead of ~log2(depth);
// the jumping runs on |X|, which is tiny for chains (path: one per tile).
constexpr int kTileV = 8192;
constexpr int kTileThreads = 1024;

__global__ void __launch_bounds__(kTileThreads)
    k_tile_resolve(int64_t n, int32_t* rep, uint8_t* isx) {
  __shared__ int32_t s[kTileV];
  const int64_t base = (int64_t)blockIdx.x * kTileV;
  const int cnt = (int)min((int64_t)kTileV, n - base);
  for (int i = threadIdx.x; i < cnt; i += kTileThreads) s[i] = rep[base + i];
  __syncthreads();
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
  for (int i = threadIdx.x; i < cnt; i += kTileThreads) {
    const int32_t p = s[i];
    rep[base + i] = p;
    const int64_t lp = (int64_t)p - base;
    if (lp < 0 || lp >= cnt) isx[p] = 1;
  }
}

__global__ void __launch_bounds__(kBlock)
    k_jump_list(int64_t count, const uint32_t* __restrict__ list, int32_t* rep, int* flags,
                int round) {
  if (round > 0 && flags[round - 1] == 0) return;
  bool changed = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = list[i];
    const int32_t p = rep[v];
    int32_t x = rep[p];
    if (x == p) continue;
#pragma unroll
    for (int hop = 1; hop < 4; ++hop) {
      const int32_t y = rep[x];
      if (y == x) break;
      x = y;
    }
    rep[v] = x;
    changed = true;
  }
  block_flag(changed, &flags[round]);
}

__global__ void __launch_bounds__(kBlock) k_final_gather(int64_t n, int32_t* rep) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = rep[v];
    const int32_t q = rep[p];
    if (q != p) rep[v] = q;
  }
}

namespace {
struct ByteFlag {
  const uint8_t* f;
  __device__ uint32_t operator()(int64_t i) const { return f[i]; }
};
}  // namespace

void launch_compress2(Handle& h, int32_t* rep, int64_t n) {
  if (n <= 0) return;
  uint8_t* isx = h.ws<uint8_t>(WS_ISROOT, n);
  uint32_t* list = h.ws<uint32_t>(WS_HEADS, n + 1);
  CK(cudaMemsetAsync(isx, 0, (size_t)n, h.stream));
  const unsigned tiles = (unsigned)((n + kTileV - 1) / kTileV);
  k_tile_resolve<<<tiles, kTileThreads, 0, h.stream>>>(n, rep, isx);
  CK_LAUNCH();
  h.stats.step(n);
  const int64_t X = scan_emit(h, n, ByteFlag{isx}, EmitCompact{list}, true);
  if (X > 0) {
    int rounds = 2;
    while ((int64_t{1} << (rounds - 2)) < X + 1) ++rounds;  // X-forest depth <= |X|
    int* flags = reinterpret_cast<int*>(h.dev_box + 128);
    CK(cudaMemsetAsync(flags, 0, 64 * sizeof(int), h.stream));
    const unsigned g = grid_for(X);
    for (int r = 0; r < rounds && r < 64; ++r) {
      k_jump_list<<<g, kBlock, 0, h.stream>>>(X, list, rep, flags, r);
      h.stats.step(X);
    }
    CK_LAUNCH();
  }
  k_final_gather<<<grid_for(n), kBlock, 0, h.stream>>>(n, rep);
  CK_LAUNCH();
  h.stats.step(n);
}

void launch_hook(Handle& h, int mode, const int2* edges, int64_t m, uint32_t e_base,
                 const int32_t* rep, unsigned long long* slot, int* any_prop) {
  const unsigned grid = grid_for(m);
  if (mode == 0)
    k_hook<0><<<grid, kBlock, 0, h.stream>>>(edges, m, e_base, rep, slot, any_prop);
  else
    k_hook<1><<<grid, kBlock, 0, h.stream>>>(edges, m, e_base, rep, slot, any_prop);
  CK_LAUNCH();
  h.stats.step(m);
}

void launch_apply(Handle& h, int32_t* rep, unsigned long long* slot, uint8_t* tflag,
                  uint32_t e_base, uint32_t m_local, unsigned long long* counter) {
  k_apply<<<grid_for(h.g.n), kBlock, 0, h.stream>>>(h.g.n, rep, slot, tflag, e_base, m_local,
                                                     counter);
  CK_LAUNCH();
  h.stats.step(h.g.n);
}

void launch_compress(Handle& h, int32_t* rep, int64_t n) {
  k_compress<<<grid_for(n), kBlock, 0, h.stream>>>(n, rep);
  CK_LAUNCH();
  h.stats.step(n);
}

void launch_cc_init(Handle& h, int32_t* rep, unsigned long long* slot) {
  k_cc_init<<<grid_for(h.g.n), kBlock, 0, h.stream>>>(h.g.n, rep, slot);
  CK_LAUNCH();
  h.stats.step(h.g.n);
}

int64_t cc_exact(Handle& h, int32_t* rep, uint8_t* tflag) {
  const int64_t n = h.g.n, m = h.g.m;
  unsigned long long* slot = h.ws<unsigned long long>(WS_SLOT, n);
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(h.dev_box);
  h.timer.begin(h.stream, "cc.init");
  launch_cc_init(h, rep, slot);
  if (tflag && m > 0) CK(cudaMemsetAsync(tflag, 0, (size_t)m, h.stream));
  CK(cudaMemsetAsync(counter, 0, 2 * sizeof(unsigned long long), h.stream));
  h.timer.end(h.stream);
  int mode = 0;  // HookMode::kMin first (cc_forest.cpp:87)
  uint64_t prev = 0;
  for (int64_t round = 0;; ++round) {
    if (round > n + 1) throw AlgoError("hooking failed to converge");
    h.timer.begin(h.stream, mode == 0 ? "cc.hook_min" : "cc.hook_max");
    launch_hook(h, mode, h.g.edges, m, (uint32_t)h.g.e_base, rep, slot, nullptr);
    h.timer.end(h.stream);
    h.timer.begin(h.stream, "cc.apply");
    launch_apply(h, rep, slot, tflag, (uint32_t)h.g.e_base, (uint32_t)m, counter);
    h.timer.end(h.stream);
    h.read_box(reinterpret_cast<int64_t*>(counter), 1);
    const uint64_t total = (uint64_t)h.host_box[0];
    h.stats.rounds = round + 1;
    if (total == prev) break;  // no hook applied this round (cc_forest.cpp:91)
    prev = total;
    h.timer.begin(h.stream, "cc.compress");
    launch_compress2(h, rep, n);
    h.timer.end(h.stream);
    mode ^= 1;
  }
  h.stats.tree_edges = (int64_t)prev;
  return (int64_t)prev;
}

void cc_labels_fast(Handle& h, int32_t* labels) { cc_exact(h, labels, nullptr); }

}  // namespace rstg
