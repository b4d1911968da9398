/*
 * rstg.h -- C ABI of the B200-native rooted-spanning-tree engine.
 *
 * The drop-in boundary for the three RST strategies of arXiv 2603.11645.
 * Plain pointers and sizes only; every entry point returns RSTG_OK (0) or
 * an error code, with the message in rstg_last_error() (thread-local).
 * Error messages reproduce the reference's exception texts where its tests
 * pin them (SURVEY.md §8b "Error conventions").
 *
 * Reference interfaces replaced (paths under /root/reference/proj/core):
 *   rstg_graph_create*    Graph / build_csr          include/rst/graph.hpp:29-43,71
 *   rstg_edge_list_*      load_edge_list / EdgeList  include/rst/graph.hpp:17-23,60-64
 *   rstg_run              run_algorithm              include/rst/bench.hpp:36
 *                         (bfs_rst bfs_rst.hpp:23, cc_euler_rst
 *                          euler_rooting.hpp:69, pr_rst pr_rst.hpp:94-95)
 *   rstg_cc_spanning_forest  cc_spanning_forest     include/rst/cc_forest.hpp:42
 *   rstg_euler_root_forest   euler_root_forest      include/rst/euler_rooting.hpp:63-66
 *   rstg_validate         validate_rooted_forest     include/rst/validate.hpp:46-47
 *   rstg_forest_depth     forest_depth               include/rst/rooted_forest.hpp:29
 *   rstg_k_*              hook_step / jump_to_convergence / build_euler /
 *                         compute_successor / break_cycles / list_rank /
 *                         derive_parents (cc_forest.hpp:29-40,
 *                         euler_rooting.hpp:18-59): fine-grained entry
 *                         points of the reference's unit/acceptance tests.
 */
#ifndef RSTG_H
#define RSTG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSTG_OK 0
#define RSTG_ERR_ARG 1   /* invalid argument (reference: std::invalid_argument) */
#define RSTG_ERR_ALGO 2  /* algorithm failure (reference: std::runtime_error)   */
#define RSTG_ERR_CUDA 3  /* CUDA runtime error / no device                      */
#define RSTG_ERR_PARSE 4 /* malformed edge-list text (reference: rst::ParseError) */

/* AlgoKind order of bench.hpp:16 */
#define RSTG_BFS 0
#define RSTG_CC_EULER 1
#define RSTG_PR_RST 2

typedef struct rstg_graph rstg_graph;
typedef struct rstg_edge_list rstg_edge_list;

/* Mirrors StepReport (step_engine.hpp:21-25) plus device-side figures. */
typedef struct {
  int64_t steps;      /* device-wide barriers of the pipeline            */
  int64_t work;       /* element updates                                 */
  int64_t rounds;     /* hook / graft rounds (incl. the final empty one) */
  int64_t launches;   /* kernels launched                                */
  int64_t tree_edges; /* spanning-forest edges                           */
  int64_t components; /* roots                                           */
  int64_t levels;     /* BFS levels                                      */
  double device_ms;   /* CUDA-event time of the device pipeline          */
  double total_ms;    /* wall time of the call incl. host<->device copies */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
} rstg_stats;

const char* rstg_last_error(void);
int rstg_device_count(int* count);

/* Graph from the reference's host arrays (int64): offsets[n+1],
 * neighbors[2m], edge_origin[2m], edges_uv[2m] (u,v interleaved, normalized:
 * u < v, lexicographically sorted, unique). CSR arrays may be NULL: the CSR
 * is then built on the device from edges_uv, and edges_uv is checked on the
 * device like build_csr (graph.cpp:145-156): RSTG_ERR_ARG with "edge
 * endpoint out of range", "self-loop in normalized EdgeList" or "EdgeList
 * not normalized". */
int rstg_graph_create(const int64_t* offsets, const int64_t* neighbors,
                      const int64_t* edge_origin, const int64_t* edges_uv, int64_t n,
                      int64_t m, int device, rstg_graph** out);
/* Re-upload a graph of the same kind into an existing handle (reuses its
 * device buffers and workspace when n and m are unchanged). edges_uv streams
 * through two device staging buffers (cudaMemcpyAsync of chunk k+1 overlaps
 * the narrowing of chunk k); pinned CSR arrays are read directly by the
 * narrowing kernel, pageable ones are staged. */
int rstg_graph_upload(rstg_graph* g, const int64_t* offsets, const int64_t* neighbors,
                      const int64_t* edge_origin, const int64_t* edges_uv, int64_t n, int64_t m);
/* Graph from device-resident int32 arrays (copied into the handle).
 * d_offsets/d_nbrs/d_arc_edge may be NULL (CSR built on the device). */
int rstg_graph_create_device(const int32_t* d_edges_uv, const uint32_t* d_offsets,
                             const int32_t* d_nbrs, const uint32_t* d_arc_edge, int64_t n,
                             int64_t m, int device, rstg_graph** out);
/* load_edge_list (graph.hpp:60-64, graph.cpp:48-127) over an in-memory
 * text (edge list or MatrixMarket): parsed by `threads` host threads,
 * then ids densified/remapped and the list normalized on `device`.
 * Errors: RSTG_ERR_PARSE "line N: <what>" with *err_line = N (the
 * reference's ParseError texts); RSTG_ERR_ALGO "empty edge-list input: no
 * data lines" / "graph too large: vertex ids exceed 2^31". */
int rstg_edge_list_load(const char* text, int64_t len, int threads, int device,
                        rstg_edge_list** out, int64_t* err_line);
/* n (num_vertices), m (normalized edges), original-id count (0 = identity ids). */
int rstg_edge_list_info(const rstg_edge_list* el, int64_t* n, int64_t* m, int64_t* n_original_ids);
/* edges_uv[2m] (u < v, sorted) and original_ids[n_original_ids]; either nullable. */
int rstg_edge_list_copy(rstg_edge_list* el, int64_t* edges_uv, int64_t* original_ids);
int rstg_edge_list_destroy(rstg_edge_list* el);
/* Device graph straight from a loaded list (no host round trip; CSR on device). */
int rstg_graph_from_edge_list(const rstg_edge_list* el, int device, rstg_graph** out);
/* The parse stage alone (host threads only, no device): raw pairs in file
 * order into uv_out (when *count <= cap), or RSTG_ERR_PARSE + *err_line. */
int rstg_parse_edge_text(const char* text, int64_t len, int threads, int64_t* uv_out, int64_t cap,
                         int64_t* count, int64_t* err_line);

/* Device generator: "path:N", "star:N", "grid:R:C", "road:R[:p]",
 * "kron:SCALE[:EF]" (SURVEY.md Appendix B shapes; identical edge lists to
 * the host generators). */
int rstg_graph_generate(const char* spec, int device, rstg_graph** out);
int rstg_graph_info(const rstg_graph* g, int64_t* n, int64_t* m);
/* Copies the device edge list out as int64 pairs (2m). */
int rstg_graph_edges(rstg_graph* g, int64_t* edges_uv);
/* The edges whose device flag (uint8 per edge of the handle, e.g. the tree
 * flags of rstg_cc_labels) is set, in id order, as int64 (u, v) pairs;
 * *count = how many (at most cap). SpanningForest::tree_edges as endpoints. */
int rstg_graph_edges_flagged(rstg_graph* g, const uint8_t* d_flags, int64_t* edges_uv,
                             int64_t cap, int64_t* count);
int rstg_graph_destroy(rstg_graph* g);
/* Launch on a caller stream (cudaStream_t) instead of the handle's own. */
int rstg_set_stream(rstg_graph* g, void* cuda_stream);
/* Per-phase CUDA-event timing (read with rstg_phase_times). */
int rstg_set_timing(rstg_graph* g, int enabled);
/* JSON object of the last run, one entry per phase:
 * {"phase": [ms, records, algorithmic_bytes], ...}; records = timed
 * intervals of the phase in the run (a phase may span several launches). */
int rstg_phase_times(rstg_graph* g, char* buf, int64_t cap);

/* run_algorithm (bench.cpp:38-54): parent_out[n] (P[r] = r); levels_out[n]
 * for BFS (nullable); roots_out (capacity n, nullable) in the reference's
 * order: BFS discovery order, cc-euler / pr-rst ascending. */
int rstg_run(rstg_graph* g, int algo, int64_t root, int64_t jump_batch, int64_t* parent_out,
             int64_t* levels_out, int64_t* roots_out, int64_t* num_roots, rstg_stats* stats);
/* Device-resident variant: int32 parent (and levels, nullable) on device. */
int rstg_run_device(rstg_graph* g, int algo, int64_t root, int64_t jump_batch,
                    int32_t* d_parent, int32_t* d_levels, rstg_stats* stats);

/* cc_spanning_forest: labels[n] = converged reps, tree_edges ascending ids. */
int rstg_cc_spanning_forest(rstg_graph* g, int64_t* labels_out, int64_t* tree_edges_out,
                            int64_t* num_tree_edges, rstg_stats* stats);

/* euler_root_forest(n, tree_edges, labels, designated_root) on `device`.
 * tree_uv: T edges as (u,v) pairs; designated_root -1 = none. Checks in the
 * reference's order: label count, designated root, (labels in [0, n)),
 * "edge count does not match a spanning forest of the labeling", then
 * "list ranking failed to converge: not a forest". */
int rstg_euler_root_forest(int64_t n, const int64_t* tree_uv, int64_t T, const int64_t* labels,
                           int64_t nlabels, int64_t designated_root, int device,
                           int64_t* parent_out, int64_t* roots_out, int64_t* num_roots);

/* validate_rooted_forest on the device. *valid = 1/0; *code = 0 or
 * 1 range, 2 non-edge, 3 cycle, 4 roots per component, 5 cross-component,
 * 6 required root; *bad_vertex = first offender. */
int rstg_validate(rstg_graph* g, const int64_t* parent, int64_t required_root, int* valid,
                  int* code, int64_t* bad_vertex);

/* forest_depth (rooted_forest.hpp:29, rooted_forest.cpp:12-95) on the
 * device: depth_out[n] hops to the root (nullable), root_max_out[n] the
 * deepest chain under each root, -1 for non-roots (nullable), *max_depth
 * the overall maximum. Errors: "parent out of range at vertex v",
 * "parent array contains a cycle at vertex v" (the smallest such v). */
int rstg_forest_depth(rstg_graph* g, const int64_t* parent, int64_t* depth_out,
                      int64_t* root_max_out, int64_t* max_depth);

/* ---- edge-partitioned connectivity (multi-GPU) ----
 * Rank r's handle holds a contiguous range of the GLOBAL normalized edge
 * list: global edge id = e_base + local index (hook keys use global ids,
 * so k-rank results equal the 1-rank result bit for bit). rep (int32 n) and
 * slot (int64 n, empty = INT64_MAX) are caller-owned device buffers
 * replicated on every rank; between rstg_cc_hook and rstg_cc_apply the
 * caller MIN-all-reduces slot over the ranks (ncclMin on ncclInt64) --
 * exactly combine_min of hook_step (cc_forest.cpp:34). */
/* Kronecker partition on the device: edges whose smaller endpoint lies in
 * [part*n/nparts, (part+1)*n/nparts), normalized (a contiguous range of the
 * global sorted list). No CSR. */
int rstg_graph_generate_part(const char* spec, int part, int nparts, int device,
                             rstg_graph** out);
int rstg_graph_set_edge_base(rstg_graph* g, int64_t e_base);
/* MIN-combine of hook slots across ranks, called by rstg_cc_labels before
 * every apply: which 0 = d_slot[0, count) (round 0, dense), which 1 =
 * d_xbuf[0, count) (the current roots' slots in roots-list order, the list
 * being identical on every rank). The callee enqueues its collective on the
 * handle's stream (rstg_set_stream) and returns 0, or non-zero on failure. */
typedef int (*rstg_reduce_min_fn)(void* ctx, int which, int64_t count);
/* cc_spanning_forest's labels (cc_forest.cpp:73-102) through the optimised
 * single-GPU round structure (round 0 from hook keys, lazy rounds, roots-
 * list apply). d_rep: int32 n labels out (converged reps); d_tflag (nullable):
 * uint8 flags of the handle's edges that became tree edges. reduce_min NULL:
 * one GPU (d_slot/d_xbuf may be NULL). Otherwise edge-partitioned: the handle
 * holds this rank's edge range (rstg_graph_set_edge_base), d_slot/d_xbuf
 * are caller int64[n] device buffers, and every rank ends with the same
 * labels -- bit-identical to the 1-GPU labels. stats->tree_edges = the
 * global tree-edge count, stats->rounds the hook rounds. */
int rstg_cc_labels(rstg_graph* g, int32_t* d_rep, uint8_t* d_tflag, int64_t* d_slot,
                   int64_t* d_xbuf, rstg_reduce_min_fn reduce_min, void* ctx, rstg_stats* stats);
int rstg_cc_init(rstg_graph* g, int32_t* d_rep, int64_t* d_slot);
int rstg_cc_hook(rstg_graph* g, int mode, const int32_t* d_rep, int64_t* d_slot);
/* applies every non-empty slot (rep[v] = winner, slot reset); local tree
 * flags (nullable, m_local bytes); *applied = hooks applied (all ranks). */
int rstg_cc_apply(rstg_graph* g, int32_t* d_rep, int64_t* d_slot, uint8_t* d_tflag,
                  int64_t* applied);
int rstg_cc_compress(rstg_graph* g, int32_t* d_rep);

/* ---- kernel-level entry points (device kernels, host buffers) ---- */
/* hook_step (cc_forest.cpp:8-48): slot[n] uses INT64_MAX as empty.
 * *applied = 1 if any hook was applied. */
int rstg_k_hook_step(int64_t n, int64_t m, const int64_t* edges_uv, int mode, int64_t* rep,
                     uint8_t* tree_flag, int64_t* slot, int* applied);
/* jump_to_convergence fixed point (cc_forest.cpp:50-71). */
int rstg_k_jump(int64_t n, int64_t* rep);
/* list ranking of NONE(-1)-terminated lists (euler_rooting.cpp:104-153):
 * rank = distance from the list head. */
int rstg_k_list_rank(int64_t E, const int64_t* succ, int64_t* rank);
/* The reference's arc-level Euler API (euler_rooting.hpp:18-59), int64 in
 * its own layout: arc i = tree edge i (u -> v), arc i + T its reverse.
 *   build_euler        euler_rooting.hpp:33-34: from/to/next[2T], first/last[n]
 *   compute_successor  euler_rooting.hpp:38:    succ[E]
 *   break_cycles       euler_rooting.hpp:43-44: succ[rev(last[r])] = -1
 *   derive_parents     euler_rooting.hpp:53-56: parent[n] (roots are the
 *                      caller's, sorted by the C++ mirror) */
int rstg_k_build_euler(int64_t n, const int64_t* tree_uv, int64_t T, int64_t* from, int64_t* to,
                       int64_t* first, int64_t* last, int64_t* next);
int rstg_k_compute_successor(int64_t n, int64_t E, const int64_t* from, const int64_t* first,
                             const int64_t* next, int64_t* succ);
int rstg_k_break_cycles(int64_t n, int64_t E, const int64_t* last, const int64_t* roots,
                        int64_t nroots, int64_t* succ);
int rstg_k_derive_parents(int64_t n, int64_t E, const int64_t* from, const int64_t* to,
                          const int64_t* rank, int64_t* parent);

#ifdef __cplusplus
}
#endif
#endif /* RSTG_H */
