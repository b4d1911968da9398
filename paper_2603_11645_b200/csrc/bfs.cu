// bfs.cu -- direction-optimising BFS baseline (bfs_rst, bfs_rst.cpp:10-77).
//
// Exact semantics of the reference's pull BFS:
//   * parent[v] = the smallest-id neighbour one level up (bfs_rst.cpp:49-55,
//     tests/test_bfs.cpp:55-62): top-down levels take atomicMin over every
//     frontier neighbour; bottom-up levels scan the ascending neighbour
//     list and stop at the first frontier hit.
//   * other components are seeded at their smallest vertex, ascending
//     (:58-73). Components are disjoint, so seeding them all at once in one
//     multi-source BFS gives the same levels and parents; their smallest
//     vertices come from the CC labels (only needed when the root's BFS did
//     not reach every vertex).
// One persistent cooperative kernel runs all levels with one grid barrier
// per level (a high-diameter road mesh has ~13K levels; a host round trip
// per level would dominate). Frontier queues live in HBM; the top-down
// expansion maps a frontier vertex to a thread, a warp or the whole grid by
// degree (thread/warp/grid gathering), and Beamer's heuristic switches to
// bottom-up sweeps when the frontier's edges outweigh the unexplored edges.
#include <cooperative_groups.h>

#include "engine.hpp"
#include "scan.cuh"

namespace cg = cooperative_groups;

namespace rstg {

struct BfsCtl {
  int qn[3];                 // light frontier sizes, rotating by level % 3
  int hn[3];                 // heavy frontier sizes (degree >= kHeavyDeg)
  unsigned long long mf[3];  // frontier out-degree sums (Beamer's m_f)
  int levels;                // deepest level reached
  int _pad[3];
  unsigned long long reached;   // vertices taken off a frontier (all levels)
  unsigned long long scanned;   // their out-degree sum: arcs read top-down
  int d;                        // next level to expand (kernels hand over here)
  int done;                     // frontier empty: traversal complete
  unsigned long long vis0;      // Beamer's explored-edge count at the hand-over
};

// Small-frontier mode. A high-diameter graph (road: 13,219 levels, ~1,800
// frontier vertices on average) spends its BFS in grid barriers: a
// cooperative grid of ~1,200 CTAs pays several microseconds per barrier for
// a level whose work is one dependent chain per frontier vertex. While the
// frontier is small, the levels run instead in ONE thread-block cluster
// (kSmallCtas CTAs x 1024 threads, one frontier vertex per thread) whose
// hardware cluster barrier ends each level; the full cooperative grid takes
// over when the frontier grows (hysteresis: small -> big above kSmallExit,
// big -> small below kSmallEnter). The host relaunches only at hand-overs.
constexpr int kSmallThreads = 1024;
constexpr int kSmallExit = 32768;
constexpr int kSmallEnter = 8192;

constexpr int kWarpDeg = 32;
constexpr uint32_t kHeavyDeg = 4096;

struct BfsQueues {
  int32_t* q[2];   // light frontier, by level parity
  int32_t* hq[2];  // heavy frontier, by level parity
};

// Appends v (discovered at level d) to the next frontier; warp-aggregated.
__device__ __forceinline__ void enqueue(int32_t v, uint32_t deg, int32_t* qx, int* qnx,
                                        int32_t* hqx, int* hnx, unsigned long long* mfx) {
  if (deg >= kHeavyDeg) {
    qx = hqx;
    qnx = hnx;
  }
  cg::coalesced_group g = cg::coalesced_threads();
  // Lanes may target two different queues; split by queue.
  const bool heavy = deg >= kHeavyDeg;
  const unsigned hm = g.ballot(heavy);
  const unsigned rank_mask = heavy ? hm : ~hm;
  const int my_rank = __popc(rank_mask & ((1u << g.thread_rank()) - 1u));
  const int cnt = __popc(rank_mask & ((g.size() == 32) ? 0xffffffffu : ((1u << g.size()) - 1u)));
  const int leader = __ffs(rank_mask) - 1;
  int base = 0;
  if ((int)g.thread_rank() == leader) base = atomicAdd(qnx, cnt);
  base = g.shfl(base, leader);
  qx[base + my_rank] = v;
  unsigned long long s = deg;
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long t = g.shfl_down(s, o);
    if ((int)g.thread_rank() + o < (int)g.size()) s += t;
  }
  if (g.thread_rank() == 0) atomicAdd(mfx, s);
}

struct LevelIO {
  int32_t* qx;
  int* qnx;
  int32_t* hqx;
  int* hnx;
  unsigned long long* mfx;
};

// Top-down edge u -> v at level d: smallest frontier neighbour wins.
__device__ __forceinline__ void td_visit(int32_t u, int32_t v, int d, int32_t* level,
                                         int32_t* parent, const uint32_t* offsets,
                                         const LevelIO& io) {
  const int lv = ld_cg(&level[v]);
  if (lv != -1 && lv != d) return;
  if (u < ld_cg(&parent[v])) atomicMin(&parent[v], u);
  if (lv == -1 && atomicCAS(&level[v], -1, d) == -1)
    enqueue(v, offsets[v + 1] - offsets[v], io.qx, io.qnx, io.hqx, io.hnx, io.mfx);
}

__global__ void __launch_bounds__(kBlock)
    k_bfs(int64_t n, int64_t two_m, const uint32_t* __restrict__ offsets,
          const int32_t* __restrict__ nbrs, int32_t* level, int32_t* parent, BfsQueues qs,
          BfsCtl* ctl, int max_levels, int small_enter, unsigned long long small_mf) {
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = gtid >> 5, nwarps = gsize >> 5;
  bool bottom_up = false;
  const int d_start = *((volatile int*)&ctl->d);
  unsigned long long visited_edges = *((volatile unsigned long long*)&ctl->vis0);
  for (int d = d_start; d < d_start + max_levels; ++d) {
    const int ci = d % 3, ni = (d + 1) % 3, zi = (d + 2) % 3;
    const int qn = *((volatile int*)&ctl->qn[ci]);
    const int hn = *((volatile int*)&ctl->hn[ci]);
    const unsigned long long mf = *((volatile unsigned long long*)&ctl->mf[ci]);
    if (qn + hn == 0 || (!bottom_up && qn + hn < small_enter && mf <= small_mf)) {
      // every thread saw the same counters: a uniform exit
      if (gtid == 0) {
        ctl->d = d;
        ctl->done = qn + hn == 0;
        ctl->vis0 = visited_edges;
      }
      return;
    }
    visited_edges += mf;
    if (gtid == 0) {
      ctl->reached += (unsigned long long)(qn + hn);
      ctl->scanned += mf;
      ctl->levels = d - 1;
      ctl->qn[zi] = 0;
      ctl->hn[zi] = 0;
      ctl->mf[zi] = 0;
    }
    // Beamer's direction heuristic (alpha = 14, beta = 24).
    const unsigned long long mu = (unsigned long long)two_m - min(visited_edges, (unsigned long long)two_m);
    const int64_t nf = (int64_t)qn + hn;
    if (!bottom_up && mf * 14ull > mu && nf * 64 > n) bottom_up = true;
    else if (bottom_up && nf * 24 < n) bottom_up = false;
    const int32_t* qc = qs.q[d & 1];
    const int32_t* hqc = qs.hq[d & 1];
    const LevelIO io{qs.q[(d + 1) & 1], &ctl->qn[ni], qs.hq[(d + 1) & 1], &ctl->hn[ni],
                     &ctl->mf[ni]};
    if (!bottom_up) {
      for (int64_t base = warp_id * 32; base < qn; base += nwarps * 32) {
        const int64_t i = base + lane;
        int32_t u = -1;
        uint32_t b = 0, e = 0;
        if (i < qn) {
          u = qc[i];
          b = offsets[u];
          e = offsets[u + 1];
        }
        const uint32_t deg = e - b;
        unsigned wmask = __ballot_sync(0xffffffffu, u >= 0 && deg >= (uint32_t)kWarpDeg);
        while (wmask) {  // warp gathering
          const int src = __ffs(wmask) - 1;
          wmask &= wmask - 1;
          const int32_t wu = __shfl_sync(0xffffffffu, u, src);
          const uint32_t wb = __shfl_sync(0xffffffffu, b, src);
          const uint32_t we = __shfl_sync(0xffffffffu, e, src);
          for (uint32_t j = wb + lane; j < we; j += 32) td_visit(wu, nbrs[j], d, level, parent, offsets, io);
        }
        if (u >= 0 && deg < (uint32_t)kWarpDeg)  // thread gathering
          for (uint32_t j = b; j < e; ++j) td_visit(u, nbrs[j], d, level, parent, offsets, io);
      }
      for (int h = 0; h < hn; ++h) {  // grid gathering for heavy vertices
        const int32_t u = hqc[h];
        const uint32_t b = offsets[u], e = offsets[u + 1];
        for (int64_t j = b + gtid; j < e; j += gsize) td_visit(u, nbrs[j], d, level, parent, offsets, io);
      }
    } else {
      // bottom-up: the first frontier hit in ascending neighbour order
      for (int64_t v = gtid; v < n; v += gsize) {
        if (level[v] != -1) continue;
        const uint32_t b = offsets[v], e = offsets[v + 1];
        for (uint32_t j = b; j < e; ++j) {
          const int32_t u = nbrs[j];
          if (ld_cg(&level[u]) == d - 1) {
            parent[v] = u;
            level[v] = d;
            enqueue((int32_t)v, e - b, io.qx, io.qnx, io.hqx, io.hnx, io.mfx);
            break;
          }
        }
      }
    }
    grid.sync();
  }
  if (gtid == 0) {  // (level cap reached: hand back as is)
    ctl->d = d_start + max_levels;
    ctl->vis0 = visited_edges;
  }
}

// The small-frontier levels: one cluster, top-down only (a small frontier
// never favours bottom-up), one hardware cluster barrier per level. The
// frontier lives in SHARED memory: every CTA keeps the vertices its own
// threads discovered (cur/next queues of kSmallCap entries) with its
// count and degree sum, so a level's critical path holds only the graph
// reads and the level/parent atomics in HBM -- the queue reads, counters
// and appends stay on chip. The totals (termination, hand-over) are read
// across the cluster through distributed shared memory. A CTA's next queue
// can hold at most its current degree sum, so a level whose per-CTA degree
// sum exceeds kSmallCap is handed back to the cooperative grid first.
constexpr int kSmallCap = 16384;
struct SmallQ {
  uint32_t q[2][kSmallCap];
  unsigned int qn[2];
  unsigned int dsum[2];  // degree sum, each degree clamped to kSmallCap + 1 (bounded, exact test)
};

__device__ __forceinline__ void small_enqueue(SmallQ& sq, int nx, int32_t v, uint32_t deg) {
  const unsigned pos = atomicAdd(&sq.qn[nx], 1u);
  sq.q[nx][pos] = (uint32_t)v;
  atomicAdd(&sq.dsum[nx], min(deg, (uint32_t)kSmallCap + 1u));
}
__device__ __forceinline__ void small_visit(int32_t u, int32_t v, int d, int32_t* level,
                                            int32_t* parent, const uint32_t* offsets, SmallQ& sq,
                                            int nx) {
  const int lv = ld_cg(&level[v]);
  if (lv != -1 && lv != d) return;
  if (u < ld_cg(&parent[v])) atomicMin(&parent[v], u);
  if (lv == -1 && atomicCAS(&level[v], -1, d) == -1)
    small_enqueue(sq, nx, v, offsets[v + 1] - offsets[v]);
}

__global__ void __launch_bounds__(kSmallThreads, 1)
    k_bfs_small(const uint32_t* __restrict__ offsets, const int32_t* __restrict__ nbrs,
                int32_t* level, int32_t* parent, BfsQueues qs, BfsCtl* ctl) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  SmallQ& sq = *reinterpret_cast<SmallQ*>(s_raw);
  __shared__ unsigned long long s_tot, s_dtot, s_dmax;
  __shared__ unsigned int s_pre[33];  // frontier prefix over the cluster's queues
  __shared__ const SmallQ* s_rq[32];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank(), C = cl.num_blocks();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int d = ld_cg(&ctl->d);
  int cur = d & 1;
  // entry: the global frontier of level d, dealt round-robin to the CTAs
  {
    const int ci = d % 3;
    const int qn = ld_cg(&ctl->qn[ci]), hn = ld_cg(&ctl->hn[ci]);
    if (threadIdx.x == 0) {
      sq.qn[cur] = 0;
      sq.dsum[cur] = 0;
    }
    __syncthreads();
    for (int i = rank + C * threadIdx.x; i < qn + hn; i += C * blockDim.x) {
      const int32_t v = i < qn ? ld_cg(&qs.q[d & 1][i]) : ld_cg(&qs.hq[d & 1][i - qn]);
      small_enqueue(sq, cur, v, offsets[v + 1] - offsets[v]);
    }
  }
  unsigned long long vis = __ldcg(&ctl->vis0), reached = 0, scanned = 0;
  cl.sync();
  for (;; ++d, cur ^= 1) {
    const int nx = cur ^ 1;
    // frontier totals, the per-queue prefix and the largest per-CTA degree
    // sum, over the cluster (distributed shared memory)
    if (warp == 0) {
      unsigned t = 0, ds = 0;
      if (lane < (int)C) {
        const SmallQ* r = cl.map_shared_rank(&sq, lane);
        s_rq[lane] = r;
        t = r->qn[cur];
        ds = r->dsum[cur];
      }
      unsigned incl = t;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      s_pre[lane + 1] = incl;
      if (lane == 0) s_pre[0] = 0;
      unsigned long long dsum = ds, dm = ds;
      for (int o = 16; o > 0; o >>= 1) {
        dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        dm = max(dm, __shfl_xor_sync(0xffffffffu, dm, o));
      }
      if (lane == 31) s_tot = incl;
      if (lane == 0) {
        s_dtot = dsum;
        s_dmax = dm;
      }
    }
    __syncthreads();
    const unsigned long long total = s_tot, dtot = s_dtot;
    if (total == 0 || s_dmax > (unsigned long long)kSmallCap) break;
    reached += total;
    scanned += dtot;
    vis += dtot;
    if (threadIdx.x == 0) {
      sq.qn[nx] = 0;
      sq.dsum[nx] = 0;
    }
    __syncthreads();
    // the cluster's frontier, dealt evenly over all its threads (entries
    // read from the owning CTA's shared memory); discoveries stay local
    const unsigned tot = (unsigned)total;
    const unsigned ct = rank * blockDim.x + threadIdx.x, cs = C * blockDim.x;
    for (unsigned base = ct - lane; base < tot; base += cs) {
      const unsigned i = base + lane;
      int32_t u = -1;
      uint32_t b = 0, e = 0;
      if (i < tot) {
        int r = 0;
        while (s_pre[r + 1] <= i) ++r;
        u = (int32_t)s_rq[r]->q[cur][i - s_pre[r]];
        b = offsets[u];
        e = offsets[u + 1];
      }
      const uint32_t deg = e - b;
      unsigned wmask = __ballot_sync(0xffffffffu, u >= 0 && deg >= (uint32_t)kWarpDeg);
      while (wmask) {  // warp gathering
        const int src = __ffs(wmask) - 1;
        wmask &= wmask - 1;
        const int32_t wu = __shfl_sync(0xffffffffu, u, src);
        const uint32_t wb = __shfl_sync(0xffffffffu, b, src);
        const uint32_t we = __shfl_sync(0xffffffffu, e, src);
        for (uint32_t j = wb + lane; j < we; j += 32)
          small_visit(wu, nbrs[j], d, level, parent, offsets, sq, nx);
      }
      if (u >= 0 && deg < (uint32_t)kWarpDeg)  // thread gathering
        for (uint32_t j = b; j < e; ++j) small_visit(u, nbrs[j], d, level, parent, offsets, sq, nx);
    }
    cl.sync();
  }
  // every CTA leaves the loop at the same level (the totals are the
  // cluster's), but a CTA may still be reading the others' counters through
  // distributed shared memory: none exits before all have read
  cl.sync();
  // hand-over at level d (not expanded): done, or the frontier back to the
  // global queues for the cooperative grid
  const int ci = d % 3, ni = (d + 1) % 3;
  if (rank == 0 && threadIdx.x == 0) {
    ctl->d = d;
    ctl->done = s_tot == 0;
    ctl->vis0 = vis;
    ctl->reached += reached;
    ctl->scanned += scanned;
    ctl->levels = d - 1;
    ctl->qn[ci] = ctl->hn[ci] = 0;
    ctl->mf[ci] = 0;
    ctl->qn[ni] = ctl->hn[ni] = 0;
    ctl->mf[ni] = 0;
  }
  if (s_tot == 0) return;
  cl.sync();  // (counters zeroed before the appends)
  const unsigned qn = sq.qn[cur];
  for (unsigned i = threadIdx.x; i < qn; i += blockDim.x) {
    const int32_t v = (int32_t)sq.q[cur][i];
    const uint32_t deg = offsets[v + 1] - offsets[v];
    if (deg >= kHeavyDeg) {
      qs.hq[d & 1][atomicAdd(&ctl->hn[ci], 1)] = v;
    } else {
      qs.q[d & 1][atomicAdd(&ctl->qn[ci], 1)] = v;
    }
  }
  unsigned long long dsum = 0;
  for (unsigned i = threadIdx.x; i < qn; i += blockDim.x) {
    const int32_t v = (int32_t)sq.q[cur][i];
    dsum += offsets[v + 1] - offsets[v];
  }
  for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
  if (lane == 0 && dsum) atomicAdd(&ctl->mf[ci], dsum);
}

__global__ void k_bfs_init(int64_t n, int32_t* level, int32_t* parent) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    level[v] = -1;
    parent[v] = 0x7fffffff;
  }
}
__global__ void k_bfs_seed_one(int32_t r, int32_t* level, int32_t* parent, BfsQueues qs,
                               const uint32_t* offsets, BfsCtl* ctl) {
  // level 1 reads ctl index 1 and the odd-parity queues
  const uint32_t deg = offsets[r + 1] - offsets[r];
  level[r] = 0;
  parent[r] = r;
  if (deg >= kHeavyDeg) {
    qs.hq[1][0] = r;
    ctl->hn[1] = 1;
  } else {
    qs.q[1][0] = r;
    ctl->qn[1] = 1;
  }
  ctl->mf[1] = deg;
  ctl->d = 1;
}

namespace {
// Unvisited vertices that are the smallest of their CC label.
struct SeedFlag {
  const int32_t* level;
  const uint32_t* minv;
  const int32_t* lab;
  __device__ uint32_t operator()(int64_t v) const {
    return (level[v] == -1 && minv[lab[v]] == (uint32_t)v) ? 1u : 0u;
  }
};
struct EmitSeed {
  int32_t* roots;  // roots[1 + p]
  int32_t* q;
  int32_t* level;
  int32_t* parent;
  __device__ void operator()(int64_t v, uint32_t p, uint32_t f) const {
    if (!f) return;
    roots[1 + p] = (int32_t)v;
    q[p] = (int32_t)v;
    level[v] = 0;
    parent[v] = (int32_t)v;
  }
};
}  // namespace

void launch_min_vertex(Handle& h, const int32_t* lab, uint32_t* minv);

__global__ void k_seed_ctl(BfsCtl* ctl, unsigned long long edges) {
  ctl->mf[1] = edges;
  ctl->d = 1;
}

__global__ void k_sum_seed_degrees(const int32_t* q, int count, const uint32_t* offsets,
                                   unsigned long long* out) {
  unsigned long long s = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
    s += offsets[q[i] + 1] - offsets[q[i]];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

namespace {
struct Unvisited {
  const int32_t* level;
  __device__ uint32_t operator()(int64_t v) const { return level[v] == -1 ? 1u : 0u; }
};
struct Nop {
  __device__ void operator()(int64_t, uint32_t, uint32_t) const {}
};
}  // namespace

// Cluster size of the small-frontier kernel: 16 CTAs (non-portable) where
// the device schedules it, else 8; 0 = small mode unavailable / disabled
// (RSTG_BFS_SMALL=0).
static int small_cluster_ctas(Handle& h) {
  static int cached = -1;
  if (cached >= 0) return cached;
  cached = 0;
  const char* env = getenv("RSTG_BFS_SMALL");
  if (env && atoi(env) == 0) return cached;
  CK(cudaFuncSetAttribute((const void*)k_bfs_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute((const void*)k_bfs_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sizeof(SmallQ)));
  for (int c : {16, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.dynamicSmemBytes = sizeof(SmallQ);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)k_bfs_small, &cfg) == cudaSuccess &&
        nclusters > 0) {
      cached = c;
      break;
    }
    cudaGetLastError();
  }
  (void)h;
  return cached;
}

// All levels from ctl->d on: the small-frontier cluster kernel while the
// frontier stays small, the cooperative grid while it is large; each kernel
// returns at a hand-over (ctl->d, ctl->done), read back here.
static void run_levels(Handle& h, int32_t* level, int32_t* parent, BfsQueues qs, BfsCtl* ctl,
                       int64_t frontier) {
  static int max_blocks = 0;
  if (max_blocks == 0) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs, kBlock, 0));
    max_blocks = per_sm * num_sms();
  }
  const int cl = small_cluster_ctas(h);
  int64_t n = h.g.n, two_m = 2 * h.g.m;
  const uint32_t* offsets = h.g.offsets;
  const int32_t* nbrs = h.g.nbrs;
  int max_levels = (int)std::min<int64_t>(n + 2, 0x7ffffff0);
  int small_enter = cl ? kSmallEnter : 0;
  // (a frontier whose degree sum could overflow a CTA's shared queue stays
  // on the grid: dealt round-robin, each CTA gets about 1/cl of it)
  unsigned long long small_mf = (unsigned long long)cl * kSmallCap / 4;
  bool small_stalled = false;  // the small kernel handed back without a level
  int d_now = 1;               // (the callers start every traversal at level 1)
  for (;;) {
    const int d_before = d_now;
    const bool small = cl && frontier <= kSmallExit && !small_stalled;
    if (small) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cl);
      cfg.blockDim = dim3(kSmallThreads);
      cfg.dynamicSmemBytes = sizeof(SmallQ);
      cfg.stream = h.stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k_bfs_small, offsets, nbrs, level, parent, qs, ctl));
    } else {
      void* args[] = {&n, &two_m, (void*)&offsets, (void*)&nbrs, &level, &parent, &qs, &ctl,
                      &max_levels, &small_enter, &small_mf};
      CK(cudaLaunchCooperativeKernel((void*)k_bfs, dim3(max_blocks), dim3(kBlock), args, 0,
                                     h.stream));
    }
    h.stats.launches += 1;
    CK(cudaMemcpyAsync(h.host_box, ctl, sizeof(BfsCtl), cudaMemcpyDeviceToHost, h.stream));
    CK(cudaStreamSynchronize(h.stream));
    const BfsCtl* hc = reinterpret_cast<const BfsCtl*>(h.host_box);
    if (hc->done) return;
    small_stalled = small && hc->d == d_before;
    d_now = hc->d;
    frontier = (int64_t)hc->qn[hc->d % 3] + hc->hn[hc->d % 3];
  }
}

int64_t bfs_rst(Handle& h, int32_t root, int32_t* parent, int32_t* level, int32_t* roots) {
  const int64_t n = h.g.n;
  ensure_csr(h);
  if (!h.g.has_csr()) throw ArgError("bfs needs the graph's CSR");
  BfsQueues qs;
  qs.q[0] = h.ws<int32_t>(WS_BFS_Q0, n + 1);
  qs.q[1] = h.ws<int32_t>(WS_BFS_Q1, n + 1);
  int32_t* hq = h.ws<int32_t>(WS_BFS_BITS, 2 * (n + 1));
  qs.hq[0] = hq;
  qs.hq[1] = hq + (n + 1);
  BfsCtl* ctl = reinterpret_cast<BfsCtl*>(h.ws<char>(WS_BFS_CTRL, sizeof(BfsCtl) + 64));
  const cudaStream_t s = h.stream;

  h.timer.begin(s, "bfs.init", 8.0 * n);
  CK(cudaMemsetAsync(ctl, 0, sizeof(BfsCtl), s));
  k_bfs_init<<<grid_for(n), kBlock, 0, s>>>(n, level, parent);
  k_bfs_seed_one<<<1, 1, 0, s>>>(root, level, parent, qs, h.g.offsets, ctl);
  CK_LAUNCH();
  h.stats.step(n);
  h.timer.end(s);

  // compulsory per reached vertex: offsets 8 B, its level and parent 8 B;
  // per arc of a reached vertex 4 B (the neighbour id) -- counted on the
  // device as the frontiers go (ctl->reached, ctl->scanned)
  h.timer.begin(s, "bfs.levels", 0.0);
  run_levels(h, level, parent, qs, ctl, 1);
  h.timer.end(s);
  const BfsCtl* hc = reinterpret_cast<const BfsCtl*>(h.host_box);
  const int levels_root = hc->levels;
  h.timer.add_bytes("bfs.levels", 16.0 * (double)hc->reached + 4.0 * (double)hc->scanned);
  h.stats.levels = levels_root;
  // one barrier per level plus the final empty level (with the init step:
  // depth + 2 for a connected graph, bfs_rst.hpp:19)
  h.stats.steps += levels_root + 1;

  // Anything unreached? Seed every other component at its smallest vertex.
  const uint32_t unvisited = scan_emit(h, n, Unvisited{level}, Nop{}, true);
  h.stats.steps -= 1;  // the restart scan belongs to the final level (bfs_rst.cpp:58)
  *reinterpret_cast<int32_t*>(h.host_box) = root;
  CK(cudaMemcpyAsync(roots, h.host_box, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (unvisited == 0) {
    CK(cudaStreamSynchronize(s));
    return 1;
  }
  h.timer.begin(s, "bfs.seed_components");
  int32_t* lab = h.ws<int32_t>(WS_VAL_A, n);
  cc_labels_fast(h, lab);
  uint32_t* minv = h.ws<uint32_t>(WS_MINV, n);
  h.minv_clean = nullptr;  // (WS_MINV reused here)
  CK(cudaMemsetAsync(minv, 0xFF, n * sizeof(uint32_t), s));
  launch_min_vertex(h, lab, minv);
  // The second phase starts again at level 1 (ctl index 1, odd queues).
  // Seeds all enter the light queue; heavy seeds are then expanded by warp
  // gathering, which is correct, just slower.
  CK(cudaMemsetAsync(ctl, 0, sizeof(BfsCtl), s));
  const uint32_t seeds =
      scan_emit(h, n, SeedFlag{level, minv, lab}, EmitSeed{roots, qs.q[1], level, parent}, true);
  unsigned long long* degsum = reinterpret_cast<unsigned long long*>(h.dev_box) + 30;
  CK(cudaMemsetAsync(degsum, 0, sizeof(unsigned long long), s));
  k_sum_seed_degrees<<<grid_for(seeds), kBlock, 0, s>>>(qs.q[1], (int)seeds, h.g.offsets, degsum);
  CK_LAUNCH();
  h.read_box(reinterpret_cast<int64_t*>(degsum), 1);
  k_seed_ctl<<<1, 1, 0, s>>>(ctl, (unsigned long long)h.host_box[0]);
  *reinterpret_cast<int*>(h.host_box) = (int)seeds;
  CK(cudaMemcpyAsync(&ctl->qn[1], h.host_box, sizeof(int), cudaMemcpyHostToDevice, s));
  CK_LAUNCH();
  h.timer.end(s);
  h.timer.begin(s, "bfs.levels2", 0.0);
  run_levels(h, level, parent, qs, ctl, seeds);
  h.timer.end(s);
  const int lv2 = hc->levels;
  h.timer.add_bytes("bfs.levels2", 16.0 * (double)hc->reached + 4.0 * (double)hc->scanned);
  h.stats.levels = std::max<int64_t>(levels_root, lv2);
  h.stats.steps += lv2 + 2;
  return 1 + (int64_t)seeds;
}

}  // namespace rstg
