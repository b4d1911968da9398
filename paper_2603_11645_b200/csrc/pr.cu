// pr.cu -- PR-RST path-reversal rooted spanning tree (pr_rst.cpp:267-314).
//
// Round = {graft, mark, check, reverse, batched jump, rebuild ancestors}
// exactly as the reference, each step a coalesced vertex/edge sweep:
//   graft proposals   k_hook (shared with CC; pr_rst.cpp:82-99)
//   resolve + update  k_graft_resolve / k_graft_update (:112-128)
//   mark_paths        one launch per doubling level k; marks carry the level
//                     they were set in, so "marked before level k" replaces
//                     the reference's cur/fresh double buffer and one kernel
//                     per level suffices (:135-164). A level that adds
//                     nothing stops the remaining launches on the device;
//                     later levels could not add anything either (the marked
//                     set is a contiguous 2^(k+1)-prefix of each chain).
//   reverse_paths     two sweeps (:178-204)
//   batched_jump      Jacobi snapshot hops, 2^batch per barrier (:216-252);
//                     converged barriers exit on the device
//   rebuild ancestors level-major table anc[k*n + v] (:254-265); a level
//                     equal to its predecessor stops the rebuild (all higher
//                     levels are then identical) and mark reads are clamped.
// The only host synchronisation is one flag read per round.
#include "engine.hpp"

namespace rstg {

void launch_hook(Handle& h, int mode, const int2* edges, int64_t m, uint32_t e_base,
                 const int32_t* rep, unsigned long long* slot, int* any_prop);
void cc_hook_round(Handle& h, int mode, const int32_t* rep, unsigned long long* slot,
                   unsigned long long* out_count, int* any_prop);
void cc_round_done(Handle& h, int64_t out_count);
void cc_reset_rounds(Handle& h);

// Device control block layout (int32 words in the WS_BFS_CTRL workspace).
enum PrCtl : int {
  C_ANY = 0,      // any graft proposal this round
  C_BAD_REV,      // reversal found a marked vertex with no source
  C_JUMP_DONE,    // batched jump converged
  C_JUMP_FINAL,   // index (0/1) of the buffer holding the jumped reps
  C_LMAX,         // valid ancestor levels
  C_MARK_STOP,    // marking stopped (a level added nothing)
  C_GREW0,        // C_GREW0 + k: level k added a mark
  C_CHANGED0 = C_GREW0 + 40,  // C_CHANGED0 + k: anc level k differs from k-1
  C_NWORDS = C_CHANGED0 + 40
};

__global__ void k_pr_init(int64_t n, int32_t* parent, int32_t* rep, int32_t* scratch,
                          uint8_t* mark, uint8_t* groot, unsigned long long* slot) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    parent[v] = rep[v] = (int32_t)v;
    scratch[v] = -1;
    mark[v] = 0;
    groot[v] = 0;
    slot[v] = kKeyInf;
  }
}

// make_pr_state's anc[v][k] = v (pr_rst.cpp:60-68): every level of the
// identity table equals level 0, so only level 0 is written and the valid
// level count starts at 1 (reads of higher levels clamp to it).
__global__ void k_anc_identity(int64_t n, int32_t* anc) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    anc[v] = (int32_t)v;
}

// resolve winners against the frozen rep (pr_rst.cpp:112-122)
__global__ void k_graft_resolve(int64_t n, const int2* __restrict__ edges, uint32_t e_base,
                                const int32_t* __restrict__ rep,
                                const unsigned long long* __restrict__ slot,
                                uint8_t* __restrict__ mark, int32_t* __restrict__ scratch,
                                uint8_t* __restrict__ groot, int32_t* __restrict__ gu) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = slot[v];
    if (key == kKeyInf) continue;
    const int2 uv = edges[(uint32_t)key - e_base];
    const int32_t u = (rep[uv.x] == (int32_t)v) ? uv.x : uv.y;
    const int32_t w = (u == uv.x) ? uv.y : uv.x;
    mark[u] = 1;  // seeds carry level tag 1
    scratch[u] = w;
    groot[v] = 1;
    gu[v] = u;
  }
}

// rep update (pr_rst.cpp:123-128)
__global__ void k_graft_update(int64_t n, int32_t* rep, unsigned long long* slot) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = slot[v];
    if (key == kKeyInf) continue;
    rep[v] = (int32_t)(key >> 32);
    slot[v] = kKeyInf;
  }
}

// One mark_paths level k (pr_rst.cpp:146-153). Marked-before-level-k means
// tag in [1, k+1]; new marks get tag k+2.
__global__ void __launch_bounds__(kBlock)
    k_mark_level(int64_t n, int k, const int32_t* __restrict__ anc, uint8_t* mark, int* ctl) {
  if (k > 0 && (ctl[C_MARK_STOP] || !ctl[C_GREW0 + k - 1])) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl[C_MARK_STOP] = 1;
    return;
  }
  const int kk = min(k, ctl[C_LMAX] - 1);
  const int32_t* lvl = anc + (int64_t)kk * n;
  bool grew = false;
  // four marks per load (almost all are 0: one 32-bit test skips them); the
  // mark buffer is padded past n
  const int64_t words = (n + 3) / 4;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t4 = reinterpret_cast<const volatile uint32_t*>(mark)[w];
    if (t4 == 0) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t t = (t4 >> (8 * b)) & 0xFFu;
      const int64_t v = 4 * w + b;
      if (t == 0 || t > (uint32_t)(k + 1) || v >= n) continue;
      const int32_t a = lvl[v];
      if (mark[a] == 0) {
        mark[a] = (uint8_t)(k + 2);
        grew = true;
      }
    }
  }
  block_flag(grew, &ctl[C_GREW0 + k]);
}

// The graft check (pr_rst.cpp:281-288): every grafted root r is marked and
// still a root. Records the smallest offending (r, u).
__global__ void k_graft_check(int64_t n, const uint8_t* groot, const uint8_t* mark,
                              const int32_t* parent, const int32_t* gu,
                              unsigned long long* bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (!groot[v]) continue;
    if (!mark[v] || parent[v] != (int32_t)v)
      atomicMin(bad, ((unsigned long long)v << 32) | (uint32_t)gu[v]);
  }
}
__global__ void k_check_one(int32_t r, int32_t u, const uint8_t* mark, const int32_t* parent,
                            unsigned long long* bad) {
  if (!mark[r] || parent[r] != r) atomicMin(bad, ((unsigned long long)r << 32) | (uint32_t)u);
}
__global__ void k_clear_groot(int64_t n, uint8_t* groot) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    groot[v] = 0;
}

// reverse_paths (pr_rst.cpp:186-190, 191-201)
__global__ void k_reverse_a(int64_t n, const uint8_t* __restrict__ mark,
                            const int32_t* __restrict__ parent, int32_t* scratch) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (!mark[v]) continue;
    const int32_t p = parent[v];
    if (p != (int32_t)v) scratch[p] = (int32_t)v;
  }
}
__global__ void k_reverse_b(int64_t n, uint8_t* mark, int32_t* parent, int32_t* scratch,
                            int* ctl) {
  bool bad = false;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (!mark[v]) continue;
    const int32_t s = scratch[v];
    if (s < 0) {
      bad = true;
      continue;
    }
    parent[v] = s;
    scratch[v] = -1;
    mark[v] = 0;
  }
  block_flag(bad, &ctl[C_BAD_REV]);
}

// One batched_jump barrier (pr_rst.cpp:235-244). Buffers alternate; a
// converged state makes later barriers no-ops.
template <int kB>
__global__ void __launch_bounds__(kBlock)
    k_jump_barrier(int64_t n, int64_t hops, int barrier, int32_t* buf0, int32_t* buf1,
                   int* ctl, int* not_done) {
  if (ctl[C_JUMP_DONE]) return;
  const int32_t* __restrict__ snap = (barrier & 1) ? buf1 : buf0;
  int32_t* __restrict__ next = (barrier & 1) ? buf0 : buf1;
  // kB vertices' chains walked together: each hop's loads issued at once
  bool pending = false;
  const int64_t g = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < n; v0 += kB * g) {
    int32_t x[kB];
    bool walk[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      walk[j] = v0 + j * g < n;
      x[j] = walk[j] ? snap[v0 + j * g] : 0;
    }
    for (int64_t t = 1; t < hops; ++t) {
      bool any = false;
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if (!walk[j]) continue;
        const int32_t nx = snap[x[j]];
        if (nx == x[j]) walk[j] = false;
        else x[j] = nx;
        any |= walk[j];
      }
      if (!any) break;
    }
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      if (v0 + j * g >= n) continue;
      next[v0 + j * g] = x[j];
      if (snap[x[j]] != x[j]) pending = true;
    }
  }
  block_flag(pending, not_done);
}
// Closes barrier `barrier`: converged -> record which buffer holds reps.
__global__ void k_jump_close(int barrier, int* ctl, int* not_done) {
  if (ctl[C_JUMP_DONE]) return;
  if (*not_done == 0) {
    ctl[C_JUMP_DONE] = 1;
    ctl[C_JUMP_FINAL] = (barrier & 1) ? 0 : 1;
  }
  *not_done = 0;
}
__global__ void k_jump_copyback(int64_t n, int32_t* rep, const int32_t* other, const int* ctl) {
  if (ctl[C_JUMP_FINAL] == 0) return;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    rep[v] = other[v];
}

// rebuild_special_ancestors level k >= 1 (pr_rst.cpp:260-264).
template <int kB>
__global__ void __launch_bounds__(kBlock) k_anc_level(int64_t n, int k, int32_t* anc, int* ctl) {
  if (k >= 2 && !ctl[C_CHANGED0 + k - 1]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMin(&ctl[C_LMAX], k);
    return;
  }
  // (distinct levels of one buffer: restrict-qualified so the stores do not
  // order the next vertices' loads; kB vertices' gathers in flight -- 4 on
  // graphs larger than L2, where each gather waits on DRAM)
  const int32_t* __restrict__ prev = anc + (int64_t)(k - 1) * n;
  int32_t* __restrict__ cur = anc + (int64_t)k * n;
  bool changed = false;
  const int64_t g = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < n; v0 += kB * g) {
    int32_t a[kB], b[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) a[j] = v0 + j * g < n ? __ldcs(&prev[v0 + j * g]) : 0;
#pragma unroll
    for (int j = 0; j < kB; ++j) b[j] = v0 + j * g < n ? prev[a[j]] : 0;
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      if (v0 + j * g >= n) continue;
      cur[v0 + j * g] = b[j];
      changed |= (b[j] != a[j]);
    }
  }
  block_flag(changed, &ctl[C_CHANGED0 + k]);
}

__global__ void k_set_i32(int32_t* p, int32_t v) { *p = v; }
__global__ void k_set_u8(uint8_t* p, uint8_t v) { *p = v; }

static int ceil_log2_i(int64_t x) {
  int k = 0;
  int64_t p = 1;
  while (p < x) {
    p <<= 1;
    ++k;
  }
  return k;
}

void pr_rst(Handle& h, int32_t root, int64_t jump_batch, int32_t* parent) {
  // batched gathers pay once a level of the ancestor table (4n bytes) no
  // longer sits in L2
  const bool big = h.g.n > (int64_t{1} << 22);
  const int64_t n = h.g.n, m = h.g.m;
  const int L = std::max(ceil_log2_i(std::max<int64_t>(n, 1)), 1);
  int32_t* rep = h.ws<int32_t>(WS_REP, n);
  int32_t* scratch = h.ws<int32_t>(WS_PR_SCRATCH, n);
  uint8_t* mark = h.ws<uint8_t>(WS_PR_ONPATH, n);
  uint8_t* groot = h.ws<uint8_t>(WS_PR_GROOT, n);
  int32_t* gu = h.ws<int32_t>(WS_PR_GU, n);
  int32_t* nextbuf = h.ws<int32_t>(WS_PR_NEXT, n);
  int32_t* anc = h.ws<int32_t>(WS_PR_ANC, (size_t)n * L);
  unsigned long long* slot = h.ws<unsigned long long>(WS_SLOT, n);
  h.slots_clean = nullptr;  // graft rounds leave slots of their own
  cc_reset_rounds(h);       // (graft rounds use the CC's active-edge lists)
  unsigned long long* crossing = reinterpret_cast<unsigned long long*>(h.dev_box) + 18;
  h.round0_slots = nullptr;  // (and overwrite an upload's round-0 keys)
  int* ctl = reinterpret_cast<int*>(h.ws<int>(WS_BFS_CTRL, C_NWORDS + 8));
  unsigned long long* bad_mark = reinterpret_cast<unsigned long long*>(h.dev_box) + 16;
  int* not_done = ctl + C_NWORDS;
  const unsigned g = grid_for(n);
  const cudaStream_t s = h.stream;

  h.timer.begin(s, "pr.init");
  k_pr_init<<<g, kBlock, 0, s>>>(n, parent, rep, scratch, mark, groot, slot);
  k_anc_identity<<<g, kBlock, 0, s>>>(n, anc);  // make_pr_state :60-68
  CK_LAUNCH();
  CK(cudaMemsetAsync(bad_mark, 0xFF, sizeof(unsigned long long), s));
  h.stats.step(n, 2);
  h.timer.end(s);

  auto run_marking = [&]() {
    CK(cudaMemsetAsync(ctl + C_MARK_STOP, 0, (1 + 40) * sizeof(int), s));
    for (int k = 0; k < L; ++k) {
      k_mark_level<<<g, kBlock, 0, s>>>(n, k, anc, mark, ctl);
      h.stats.step(n);
    }
    CK_LAUNCH();
  };
  auto run_reverse = [&]() {
    k_reverse_a<<<g, kBlock, 0, s>>>(n, mark, parent, scratch);
    k_reverse_b<<<g, kBlock, 0, s>>>(n, mark, parent, scratch, ctl);
    CK_LAUNCH();
    h.stats.step(n);
    h.stats.step(n);
  };
  // ctl[C_LMAX] = 1 initially (identity table: level 0 stands for all).
  {
    int init[C_NWORDS + 8] = {0};
    init[C_LMAX] = 1;
    CK(cudaMemcpyAsync(ctl, init, sizeof(init), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }

  // batched_jump's guard (pr_rst.cpp:218-219) fires only once a graft
  // happened; hops / barrier cap are derived after that check.
  const bool batch_ok = jump_batch >= 1 && jump_batch <= 20;
  const int64_t hops = batch_ok ? (int64_t{1} << jump_batch) : 1;
  const int64_t max_barriers =
      batch_ok ? (ceil_log2_i(std::max<int64_t>(n, 1)) + jump_batch - 1) / jump_batch + 2 : 0;
  int mode = 0;
  for (int64_t round = 0;; ++round) {
    if (round > n + 1) throw AlgoError("grafting failed to converge");
    h.timer.begin(s, "pr.graft");
    // graft proposals with active-edge filtering (as in the CC: an edge
    // inside one tree stays inside; the proposals are unchanged)
    CK(cudaMemsetAsync(ctl + C_ANY, 0, sizeof(int), s));
    CK(cudaMemsetAsync(crossing, 0, sizeof(unsigned long long), s));
    cc_hook_round(h, mode, rep, slot, crossing, ctl + C_ANY);
    CK(cudaMemcpyAsync(h.host_box, ctl, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h.host_box + 1, crossing, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cc_round_done(h, h.host_box[1]);
    h.timer.end(s);
    h.stats.rounds = round + 1;
    if (reinterpret_cast<int*>(h.host_box)[C_ANY] == 0) break;  // no graft (:279)
    if (!batch_ok) throw AlgoError("jump batch out of range [1, 20]");
    h.timer.begin(s, "pr.resolve");
    k_graft_resolve<<<g, kBlock, 0, s>>>(n, h.g.edges, (uint32_t)h.g.e_base, rep, slot, mark,
                                         scratch, groot, gu);
    k_graft_update<<<g, kBlock, 0, s>>>(n, rep, slot);
    CK_LAUNCH();
    h.stats.step(n);
    h.stats.step(n);
    h.timer.end(s);
    h.timer.begin(s, "pr.mark");
    run_marking();
    k_graft_check<<<g, kBlock, 0, s>>>(n, groot, mark, parent, gu, bad_mark);
    k_clear_groot<<<g, kBlock, 0, s>>>(n, groot);
    CK_LAUNCH();
    h.stats.step(n);
    h.timer.end(s);
    h.timer.begin(s, "pr.reverse");
    run_reverse();
    h.timer.end(s);
    h.timer.begin(s, "pr.jump");
    CK(cudaMemsetAsync(ctl + C_JUMP_DONE, 0, 2 * sizeof(int), s));
    CK(cudaMemsetAsync(not_done, 0, sizeof(int), s));
    for (int64_t b = 0; b <= max_barriers; ++b) {
      (big ? k_jump_barrier<4> : k_jump_barrier<1>)<<<g, kBlock, 0, s>>>(n, hops, (int)b, rep,
                                                                        nextbuf, ctl, not_done);
      k_jump_close<<<1, 1, 0, s>>>((int)b, ctl, not_done);
      h.stats.step(n);
    }
    k_jump_copyback<<<g, kBlock, 0, s>>>(n, rep, nextbuf, ctl);
    CK_LAUNCH();
    h.timer.end(s);
    h.timer.begin(s, "pr.anc");
    CK(cudaMemcpyAsync(anc, parent, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(ctl + C_CHANGED0, 0, 40 * sizeof(int), s));
    k_set_i32<<<1, 1, 0, s>>>(ctl + C_LMAX, L);
    for (int k = 1; k < L; ++k) {
      (big ? k_anc_level<4> : k_anc_level<1>)<<<g, kBlock, 0, s>>>(n, k, anc, ctl);
      h.stats.step(n);
    }
    CK_LAUNCH();
    h.timer.end(s);
    // Deferred error checks for this round.
    CK(cudaMemcpyAsync(h.host_box, ctl, C_GREW0 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h.host_box + 8, bad_mark, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int* hc = reinterpret_cast<int*>(h.host_box);
    const unsigned long long bm = (unsigned long long)h.host_box[8];
    if (bm != kAllOnes)
      throw AlgoError("path marking corrupted: " + std::to_string(bm >> 32) +
                      " is not the root above " + std::to_string((uint32_t)bm));
    if (hc[C_BAD_REV]) throw AlgoError("reversal found a marked vertex with no source");
    if (!hc[C_JUMP_DONE]) throw AlgoError("pointer jumping detected a representative cycle");
    mode ^= 1;
  }

  // Re-root the designated root's tree (pr_rst.cpp:298-303).
  CK(cudaMemcpyAsync(h.host_box, rep + root, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int32_t emergent = *reinterpret_cast<int32_t*>(h.host_box);
  if (emergent != root) {
    h.timer.begin(s, "pr.reroot");
    k_set_u8<<<1, 1, 0, s>>>(mark + root, 1);  // mark_path :170
    run_marking();
    k_check_one<<<1, 1, 0, s>>>(emergent, root, mark, parent, bad_mark);  // :172-175
    k_set_i32<<<1, 1, 0, s>>>(scratch + root, root);  // reverse_path :212
    run_reverse();
    CK_LAUNCH();
    CK(cudaMemcpyAsync(h.host_box, ctl, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h.host_box + 8, bad_mark, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    h.timer.end(s);
    const unsigned long long bm = (unsigned long long)h.host_box[8];
    if (bm != kAllOnes)
      throw AlgoError("path marking corrupted: " + std::to_string(bm >> 32) +
                      " is not the root above " + std::to_string((uint32_t)bm));
    if (reinterpret_cast<int*>(h.host_box)[C_BAD_REV])
      throw AlgoError("reversal found a marked vertex with no source");
  }
}

}  // namespace rstg
