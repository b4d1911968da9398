// engine.hpp -- device graph handle, workspace and phase timing.
//
// One Handle per (graph, device, stream). It owns the device copy of the
// graph and a grow-only workspace so repeated builds on the same graph do
// no cudaMalloc inside the timed region. Calls on one handle are
// serialized on its stream (SURVEY.md §8b "Threading").
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "common.cuh"

namespace rstg {

// Counters mirroring StepReport (step_engine.hpp:21-25): `steps` counts
// device-wide barriers (kernel boundaries / grid syncs of the device
// pipeline), `work` counts element updates, plus device-side figures.
struct Stats {
  int64_t steps = 0;
  int64_t work = 0;
  int64_t rounds = 0;    // hook / graft rounds incl. the final empty one
  int64_t launches = 0;  // kernels launched by the library
  int64_t tree_edges = 0;
  int64_t components = 0;
  int64_t levels = 0;    // BFS levels (max over components) / PR mark levels
  double device_ms = 0;  // event-timed device pipeline (when timing on)
  void step(int64_t domain, int64_t launches_ = 1) {
    ++steps;
    work += domain;
    launches += launches_;
  }
};

// Named phase timer on the handle's stream (CUDA events; no host sync
// until collect()).
// Each phase carries its algorithmic bytes (every element the
// phase must touch, once), so the bench's roofline needs no model of its own.
struct PhaseRec {
  std::string name;
  double ms;
  double bytes;
};
class PhaseTimer {
 public:
  void begin(cudaStream_t s, const char* name, double bytes = 0);
  void end(cudaStream_t s);
  // Adds algorithmic bytes to the open phase (known only once it runs).
  void add_bytes(double b) {
    if (enabled && !open_.empty()) recs_[open_.back()].bytes += b;
  }
  // ... or to the latest closed phase of that name (bytes counted on the
  // device, read back after the phase)
  void add_bytes(const char* name, double b) {
    if (!enabled) return;
    for (auto it = recs_.rbegin(); it != recs_.rend(); ++it)
      if (it->name == name) {
        it->bytes += b;
        return;
      }
  }
  // Synchronizes and returns the phases in order; clears.
  std::vector<PhaseRec> collect();
  bool enabled = false;

 private:
  struct Rec {
    std::string name;
    double bytes;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs_;
  std::vector<size_t> open_;  // indices of open phases (phases nest)
  std::vector<cudaEvent_t> pool_;
  size_t used_ = 0;
  cudaEvent_t get();
};

struct DeviceGraph {
  int64_t n = 0, m = 0;
  int64_t e_base = 0;           // global id of edges[0] (edge-partitioned ranks)
  int2* edges = nullptr;        // m normalized (u<v) edges, id = e_base + index
  uint32_t* offsets = nullptr;  // n+1 CSR offsets (nullptr if no CSR)
  int32_t* nbrs = nullptr;      // 2m neighbours, ascending per vertex
  uint32_t* arc_edge = nullptr; // 2m edge_origin
  bool csr_pending = false;     // CSR buffers allocated, built on first use (ensure_csr)
  bool has_csr() const { return offsets != nullptr; }
};

class Handle {
 public:
  explicit Handle(int device);
  void release(int slot);
  ~Handle();
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;

  int device = 0;
  // connectivity round state (active-edge filtering, cc.cu)
  int cc_round = 0;
  int64_t cc_active = -1;  // edges in the current active list, -1 = all
  int cc_list = 0;
  int cc_filter_from = 1;  // first hook round that records its crossing edges
  bool cc_lazy = false;    // hook rounds find roots (no per-round compression)
  // WS_SLOT holds all-empty keys from a completed cc_exact (apply resets
  // every slot it consumes), so the next build skips re-initialising it;
  // any other user of the slot buffer clears this.
  const void* slots_clean = nullptr;
  int64_t slots_clean_n = 0;  // ... for its first slots_clean_n entries (beyond: unknown)
  // Set by the edge upload: WS_SLOT already holds round 0's hook keys
  // (computed while the edges streamed in), consumed by cc_exact.
  const void* round0_slots = nullptr;
  // Percent of sampled edges joining vertex ids less than a rank tile
  // apart (-1: not measured for this graph). Decides the Euler-tour
  // ranking: tile contraction for locally numbered graphs, else ruling sets.
  int edge_locality = -1;
  // Segment count of the last tile-contraction ranking of this graph (-1:
  // none yet): later builds size the level grids from it (with a margin;
  // a larger count raises the device overflow flag) instead of reading the
  // count back mid-build. Reset with edge_locality when the graph changes.
  int64_t tile_segments = -1;
  // Work a build left to check after its final stream sync (the tile
  // ranking's overflow flag, copied asynchronously into host_box[32..]):
  // run by run_late_checks() before anything reads the outputs.
  std::function<void()> late_check;
  // the device words the late check reads (copied to host_box[32..]
  // asynchronously once the last kernel that does not depend on them is
  // enqueued, so the copy does not delay it)
  struct {
    const void* src = nullptr;
    int words = 0;
  } late_copy;
  // WS_MINV holds all-ones left by the Euler root pass (its other users --
  // BFS, validation, degree counts -- clear this when they take the buffer).
  const void* minv_clean = nullptr;
  int64_t minv_clean_n = 0;  // ... for its first minv_clean_n entries
  // WS_RHEAD holds all-NONE left by the Euler vertex pass (it resets every
  // remote list it splices), so a build needs no 4n-byte fill
  const void* rhead_clean = nullptr;
  int64_t rhead_clean_n = 0;
  // WS_XBITS (the exit-set bitmap of the two-level shortcutting) is all-zero
  // after a completed pass: the exit-set jump clears what the tiles set
  const void* xbits_clean = nullptr;
  int64_t xbits_clean_words = 0;
  // PR-RST's scratch (-1) and mark (0) arrays as a completed build leaves
  // them, for their first pr_clean_n entries
  const void* pr_clean = nullptr;
  const void* pr_clean_mark = nullptr;
  int64_t pr_clean_n = 0;
  // PR-RST skip levels (pr.cu): vertex order by level and the counts C_k
  // of vertices of level >= k, valid for graphs of pr_levels_n vertices
  int64_t pr_levels_n = -1;
  const void* pr_levels_byl = nullptr;
  std::vector<int64_t> pr_levels_C;
  cudaStream_t copy_stream = nullptr;  // H2D staging of uploads (lazily created)
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  DeviceGraph g;
  Stats stats;
  PhaseTimer timer;

  // Grow-only named device buffers (slot ids from WsSlot).
  void* ws(int slot, size_t bytes);
  template <class T>
  T* ws(int slot, size_t count) {
    return static_cast<T*>(ws(slot, count * sizeof(T) + 16));
  }
  // Small pinned host mailbox for flag/count readbacks.
  int64_t* host_box = nullptr;
  // Device counters block (256 x int64) zeroed per use by the caller; fixed
  // regions: [0,3] cc, [4] euler roots, [5,7] cc exit set, [8,15] lr / tile ranking,
  // [16] pr bad mark, [17] edge-locality count, [18] pr crossing, [19] euler min-table
  // dirty flag (persists across builds), [20,22] cc roots, [24,29) cc tail rounds, [30] bfs, [40] validate,
  // [48] normalize, [50,53) capi/lr verify, [54,57) edge-upload input checks, [57] upload_ids, [60] pr short path, [128,160) jump-round flags.
  int64_t* dev_box = nullptr;

  // Copies `count` int64 device values into host_box and syncs the stream.
  void read_box(const int64_t* dptr, int count);
  void set_stream(cudaStream_t s);
  void free_graph();

 private:
  std::vector<std::pair<void*, size_t>> bufs_;
};

// Workspace slots. Distinct algorithms may alias slots when they never run
// concurrently on one handle.
enum WsSlot : int {
  WS_REP = 0,     // int32 n       CC reps / labels
  WS_SLOT,        // u64 n         hook / graft slots
  WS_TFLAG,       // u8 m          tree-edge flags
  WS_PARENT,      // int32 n       output parent
  WS_MINV,        // u32 n         min vertex per label
  WS_ISROOT,      // u8 n
  WS_POS,         // u32 2m+1      arc scan
  WS_TF,          // u32 n+1       tree CSR offsets
  WS_ATO,         // u32 E
  WS_AFROM,       // u32 E
  WS_SUCC,        // u32 E
  WS_REV,         // u32 E
  WS_SL,          // u64 E         (ruler id, local offset) per arc
  WS_RPOS,        // u32 R         ruler arc positions
  WS_RLEN,        // u32 R
  WS_RNEXT,       // u32 R
  WS_RA,          // u32/u64 R     Wyllie buffers
  WS_RB,
  WS_RC,
  WS_RD,
  WS_HEADS,       // u32 n
  WS_SCAN,        // u32 scan partials
  WS_SCAN2,
  WS_ROOTS,       // int32 n       roots list
  WS_ELIST0,      // u32 m         active (still crossing) edges, ping
  WS_ELIST1,      // u32 m         pong
  // PR-RST
  WS_PR_SCRATCH,  // int32 n
  WS_PR_ONPATH,   // u8 n
  WS_PR_FRESH,    // u8 n          skip level per vertex (built with the level order)
  WS_PR_GROOT,    // u8 n
  WS_PR_GU,       // u32 n         graft endpoints (marking seeds) of a round
  WS_PR_ANC,      // u32 ~2n       skip structure in position space (level k: C_k entries)
  WS_PR_POS,      // u32 n         position of each vertex in the level order
  WS_PR_NEXT,     // u32 n         grafted roots of a round
  WS_PR_BYL,      // u32 n         vertices by descending skip level
  WS_PR_MK,       // u32 n         marked vertices, one queue per exact level
  WS_PR_CBASE,    // u64 32        queue bases C_{b+1} (kept with pr_levels_n)
  // BFS
  WS_BFS_LEVEL,   // int32 n
  WS_BFS_Q0,      // int32 n
  WS_BFS_Q1,      // int32 n
  WS_BFS_BITS,    // u32 n/32
  WS_BFS_CTRL,    // int64 control block
  // validation
  WS_VAL_A,
  WS_VAL_B,
  WS_VAL_C,
  // Euler tour (euler.cu): rotation lists
  WS_VHEAD,       // u32 n         first arc of each vertex's local rotation list
  WS_VTAIL,       // u32 n         its last arc
  WS_RHEAD,       // u32 n         remote list (atomic prepends): first arc
  WS_RTAIL,       // u32 n         its last arc (the first one inserted)
  WS_ETO,         // u32 2N        arc heads, pairs (2i: a->b, 2i+1: b->a)
  WS_XBITS,       // u32 n/32      exit-set membership bitmap (cc.cu)
  WS_LABELS,      // u32 n         one label per component (euler.cu)
  WS_TOFF,        // u16 2N        offset of each arc in its tile segment (tilerank.cu)
  WS_CCROOTS,     // u32 3(n+1)    round-0 roots + current CC roots, ping-pong (cc.cu)
  WS_TSTATE,      // u64 tiles+1   tile counter + look-back states (tilerank.cu)
  WS_XSORT,       // u32 n         edge-partitioned CC: roots list sorted by id (cc.cu)
  WS_XTMP,        // bytes         its sort's temporary storage
  // tile-contraction levels >= 2 (tilerank.cu), one arena per level
  WS_TL2,
  WS_TL_LAST = WS_TL2 + 8,
  // list-ranking levels >= 1 (listrank.cu), one arena per level
  WS_LR_L1,
  WS_LR_LAST = WS_LR_L1 + 12,
  WS_COUNT
};

// ---- Euler tour as rotation lists (euler.cu) ----------------------------
// Tree edge slot i (of N) with endpoints (a, b), a < b, owns arcs i = (a -> b)
// and N + i = (b -> a): rev(p) = p +- N. The two directions live in
// separate halves so that a tour running along a chain of consecutive slots
// reads 8 successors per 32-byte sector, not 4. Each vertex keeps a singly linked
// list of the arcs leaving it (any rotation order gives the same parent
// array), built by atomicExch prepends the moment a
// tree edge is created (the CC apply step). succ(p) = next(rev p), the arc
// after rev(p) in the list of the vertex p enters (euler_rooting.cpp:83-86);
// it is stored directly: S[rev p] = next(p). The wrap from a list's last
// arc to its first is filled in after the CC, and left open (NONE) for a
// root, which is exactly break_cycles (euler_rooting.cpp:96-101).
//
// Two lists per vertex, concatenated by the vertex pass after the CC: the
// "local" one written by round 0's shared-memory tiles with plain stores
// (vhead/vtail, every vertex covered, so no initialisation; closed into its
// cycle at once), and the "remote" one that every other link prepends to with
// atomicExch (rhead/rtail, NONE-initialised).
struct EulerIO {
  uint32_t nslots;  // N
  uint32_t* eto;    // N words: the tree edge of slot i, arcs i = a -> b, N + i = b -> a:
                    //   a, when b = i (round 0: the vertex that hooked is b), or
                    //   kEtoEdge | e (e = the edge's index in the graph's edge list)
  uint32_t* S;      // 2N  successors
  uint32_t* vhead;  // n   local cycle: its first arc (NONE: no local list)
  uint32_t* vtail;  // n   local cycle: its last arc (S[rev(vtail)] = vhead)
  uint32_t* rhead;  // n   remote list: first arc (NONE-initialised)
  uint32_t* rtail;  // n   remote list: last arc (the first inserted)
};

#ifdef __CUDACC__
// Root of x in a rep forest whose roots are frozen, path-compressing x
// (every value a racing compression stores is a valid ancestor).
__device__ __forceinline__ int32_t find_root(int32_t* rep, int32_t x) {
  const int32_t p = rep[x];
  if (p == x) return x;
  int32_t r = rep[p];
  if (r == p) return p;
  for (;;) {
    const int32_t q = rep[r];
    if (q == r) break;
    r = q;
  }
  rep[x] = r;
  return r;
}

// The same walk without the write-back, for readers that only need the
// root (the Euler vertex pass: later passes test lab[v] == v only).
__device__ __forceinline__ int32_t find_root_ro(const int32_t* rep, int32_t x) {
  int32_t r = rep[x];
  if (r == x) return x;
  for (;;) {
    const int32_t q = rep[r];
    if (q == r) return r;
    r = q;
  }
}

constexpr uint32_t kEtoEdge = 0x80000000u;  // eto word: an edge index, not an endpoint
// The endpoints (b, a) of slot i's tree edge (arc i = a -> b) from its eto word.
__device__ __forceinline__ uint2 eto_ends(uint32_t w, uint32_t i, const int2* __restrict__ edges) {
  if (!(w & kEtoEdge)) return make_uint2(i, w);
  const int2 e = edges[w & ~kEtoEdge];
  return make_uint2((uint32_t)e.y, (uint32_t)e.x);
}
// a tree edge (a, b) = edges[e] on slot `slot` (e < 2^31: checked by the callers' graphs)
__device__ __forceinline__ void link_tree_edge(const EulerIO& io, uint32_t slot, uint32_t a,
                                               uint32_t b, uint32_t e) {
  const uint32_t p = slot, q = io.nslots + slot;  // p: a -> b, q: b -> a
  io.eto[slot] = kEtoEdge | e;
  const uint32_t na = atomicExch(&io.rhead[a], p);  // next(p) = na
  const uint32_t nb = atomicExch(&io.rhead[b], q);  // next(q) = nb
  io.S[p] = nb;  // S[p] = next(rev p) = next(q)
  io.S[q] = na;
  if (na == kNone32) io.rtail[a] = p;
  if (nb == kNone32) io.rtail[b] = q;
}
__device__ __forceinline__ uint32_t arc_rev(uint32_t p, uint32_t nslots) {
  return p < nslots ? p + nslots : p - nslots;
}
#endif

// Caller int64 ids -> device int32, range-checked on the device against
// [0, hi): returns the index of the first out-of-range value, -1 if none.
int64_t upload_ids(Handle& h, const int64_t* host, int64_t count, int32_t* dev, int64_t hi);
// Host int64 (u, v) pairs of an explicit forest -> h.g.edges, oriented,
// sorted and deduplicated on the device (the graph's CSR is left pending).
// Returns false on an endpoint outside [0, n); *simple is false when a
// self-loop or duplicate edge was dropped.
bool upload_tree_edges(Handle& h, const int64_t* tree_uv, int64_t T, int64_t n, bool* simple);
// Builds a pending CSR (uploads defer it: cc-euler never needs it).
void ensure_csr(Handle& h);

// ---- algorithms (device-resident in/out; int32 ids) ----
// cc_spanning_forest (cc_forest.cpp:73-102), exact: labels = converged reps,
// tflag[e] = 1 for tree edges. Returns the number of tree edges.
// tlist (nullable, n entries): tlist[v] = global id of the tree edge that
// hooked root v, or kNone32 (every tree edge appears exactly once).
// euler (nullable): every tree edge is linked into the rotation lists as it
// is created, slot = the vertex it hooked (EulerIO; N = n slots); the labels
// are then left lazy (reps pointing at ancestors), euler_root resolves them.
// ex (nullable): edge-partitioned mode (multi-GPU): the handle holds one
// rank's contiguous edge range (global ids from g.e_base), the slots are
// the caller's, and reduce_min MIN-combines them across the ranks before
// every apply (which 0: slot[0, count) dense; 1: xbuf[0, count), the
// current roots' slots in roots-list order). Labels and tree-edge totals
// are then identical on every rank and equal to the 1-GPU result.
struct CcExchange {
  int (*reduce_min)(void* ctx, int which, int64_t count);
  void* ctx;
  unsigned long long* slot;  // n entries
  unsigned long long* xbuf;  // n entries
};
int64_t cc_exact(Handle& h, int32_t* labels, uint8_t* tflag, const EulerIO* euler = nullptr,
                 const CcExchange* ex = nullptr);
// cc labels only, validity-level (any correct partition; used by BFS
// seeding and the validator). Returns the number of hook rounds.
void cc_labels_fast(Handle& h, int32_t* labels);
// euler_root_forest (euler_rooting.cpp:180-215) on rotation lists already
// linked (EulerIO over N slots): roots, successor wrap, ruler registration,
// list ranking, orientation; parent[n] out (int32 device).
//   cc_slots: slot v holds the edge that hooked v (valid iff labels[v] != v,
//             N = n); otherwise slots [0, T) are all valid.
//   verify:   also prove the structure is a forest (edge count, every arc
//             reached, ruler lists acyclic), else the reference's errors.
void euler_root(Handle& h, const int32_t* labels, const EulerIO& io, int64_t N, int64_t T,
                bool cc_slots, int32_t designated_root, int32_t* parent, bool verify = false);
// Number of distinct labels among labels[0, n) (each in [0, n)).
int64_t count_labels(Handle& h, const int32_t* labels, int64_t n);
// EulerIO buffers of the handle for N slots; the remote lists reset to
// NONE, the local ones too unless round 0 will write them (local_written).
EulerIO euler_buffers(Handle& h, int64_t N, bool local_written);
// Links graph edges [0, T) as tree edges (explicit forests).
void euler_link_edges(Handle& h, const EulerIO& io, int64_t T);
// pr_rst (pr_rst.cpp:267-314)
void pr_rst(Handle& h, int32_t root, int64_t jump_batch, int32_t* parent);
// bfs_rst (bfs_rst.cpp:10-77): parent, levels; roots in discovery order
// written to roots (int32), returns count.
int64_t bfs_rst(Handle& h, int32_t root, int32_t* parent, int32_t* levels, int32_t* roots);
// Roots of a parent array in ascending order; returns count.
int64_t roots_ascending(Handle& h, const int32_t* parent, int32_t* roots);
// Device validity check (validate.cpp:108-211 semantics). Returns 0 when
// valid, else an error code; *bad_vertex receives the first offender.
int validate_forest(Handle& h, const int32_t* parent, int32_t required_root,
                    int64_t* bad_vertex);

}  // namespace rstg
