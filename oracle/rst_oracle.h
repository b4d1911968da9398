/*
 * rst_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, sequential restatement of the reference RST algorithms
 * (/root/reference/proj/core). It is the CHECKER for the CUDA product path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product (paper_2603_11645_b200/)
 * never links or calls anything in oracle/.
 *
 * Parity pinning: every function here is checked (tests/test_oracle_*.py)
 * against (a) the golden vectors of the reference's own doctest suites
 * (proj/tests/test_*.cpp) and (b) outputs of the reference itself, compiled
 * from /root/reference by oracle/Makefile into oracle/_ref/ (fixtures in
 * tests/golden/, generator script tests/golden/make_golden.py).
 *
 * All ids are int64 like the reference (types.hpp:7-8). kNone = -1.
 * Return codes: 0 ok, <0 error; og_last_error() gives the reference's
 * exception message for the error paths the reference tests pin.
 */
#ifndef RST_ORACLE_H
#define RST_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* og_last_error(void);
void og_free(void* p);

/* ---- graph ingestion (graph.cpp) ------------------------------------- */
/* normalize (graph.cpp:39-46): drop self-loops, orient u<v, sort, dedup.
 * In place; returns the new edge count. */
int64_t og_normalize(int64_t m, int64_t* eu, int64_t* ev);
/* build_csr (graph.cpp:133-172). offsets[n+1], nbrs[2m], origin[2m]. */
int og_build_csr(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                 int64_t* offsets, int64_t* nbrs, int64_t* origin);

/* ---- generators (graph.cpp:181-235) + the survey's synthetic shapes ---- */
/* Each returns m and mallocs *eu,*ev (free with og_free). Output is
 * normalized. Negative return = invalid argument. */
int64_t og_gen_path(int64_t n, int64_t** eu, int64_t** ev);
int64_t og_gen_star(int64_t n, int64_t** eu, int64_t** ev);
int64_t og_gen_grid(int64_t rows, int64_t cols, int64_t** eu, int64_t** ev);
int64_t og_gen_random(int64_t n, double p, uint64_t seed, int64_t** eu, int64_t** ev);
int64_t og_gen_complete(int64_t n, int64_t** eu, int64_t** ev);
/* road_usa-shaped mesh: R x R lattice, all
 * horizontal edges, vertical edge kept iff splitmix64(0x5eed^id) < p*2^64. */
int64_t og_gen_road(int64_t R, double p, int64_t** eu, int64_t** ev);
/* Graph500 Kronecker, vertex permutation
 * og_kron_perm(), then normalize. n = 2^scale. */
int64_t og_gen_kron(int scale, int edge_factor, int64_t** eu, int64_t** ev);
uint64_t og_splitmix64(uint64_t x);
uint64_t og_kron_perm(uint64_t x, int scale);

/* ---- hot path restatements ------------------------------------------- */
/* cc_spanning_forest (cc_forest.cpp:73-102). labels[n] = converged rep,
 * tree_flag[m] (uint8). Returns number of tree edges, or <0 on error.
 * *rounds_out (nullable) = number of hook rounds incl. the final empty one. */
int64_t og_cc_spanning_forest(int64_t n, int64_t m, const int64_t* eu,
                              const int64_t* ev, int64_t* labels,
                              uint8_t* tree_flag, int64_t* rounds_out);
/* hook_step (cc_forest.cpp:8-48). mode 0 = kMin, 1 = kMax. slot[n] holds
 * packed keys (kKeyInf = INT64_MAX when empty). Returns 1 if any hook was
 * applied, 0 if none, <0 on "hooking ran on uncompressed labels". */
int og_hook_step(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                 int mode, int64_t* rep, uint8_t* tree_flag, int64_t* slot);
/* jump_to_convergence (cc_forest.cpp:50-71). Returns number of doubling
 * rounds (= steps), <0 on "pointer jumping failed to converge". */
int64_t og_jump_to_convergence(int64_t n, int64_t* rep);

/* euler_root_forest (euler_rooting.cpp:180-215). parent[n] out; roots
 * (capacity n) out sorted ascending, *num_roots. designated_root may be -1.
 * ranks_out (nullable, 2T) receives list_rank's output in the reference's
 * arc numbering (arc i = tree edge i u->v, arc i+T = v->u). */
int og_euler_root_forest(int64_t n, int64_t T, const int64_t* tu,
                         const int64_t* tv, const int64_t* labels,
                         int64_t designated_root, int64_t* parent,
                         int64_t* roots, int64_t* num_roots, int64_t* ranks_out);
/* Euler internals on a forest, for the reference's worked examples
 * (build_euler :13-74, compute_successor :76-87, break_cycles :89-102,
 * list_rank :104-153). All arrays 2T (first/last n). */
int og_build_euler(int64_t n, int64_t T, const int64_t* tu, const int64_t* tv,
                   int64_t* from, int64_t* to, int64_t* first, int64_t* last,
                   int64_t* next);
int og_list_rank(int64_t E, const int64_t* succ, int64_t* rank);
/* cc_euler_rst (euler_rooting.cpp:217-226). */
int og_cc_euler_rst(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                    int64_t root, int64_t* parent, int64_t* roots,
                    int64_t* num_roots);

/* pr_rst (pr_rst.cpp:267-314). roots ascending (the reference's scan). */
int og_pr_rst(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
              int64_t root, int64_t jump_batch, int64_t* parent,
              int64_t* roots, int64_t* num_roots);

/* bfs_rst (bfs_rst.cpp:10-77), literal level-synchronous pull restatement
 * (O(n * levels)); needs the CSR. roots in discovery order. */
int og_bfs_rst(int64_t n, const int64_t* offsets, const int64_t* nbrs,
               int64_t root, int64_t* parent, int64_t* levels,
               int64_t* roots, int64_t* num_roots);
/* O(n+m) restatement with identical output. */
int og_bfs_rst_fast(int64_t n, const int64_t* offsets, const int64_t* nbrs,
                    int64_t root, int64_t* parent, int64_t* levels,
                    int64_t* roots, int64_t* num_roots);

/* ---- verification (validate.cpp) ------------------------------------- */
/* oracle_components (validate.cpp:46-53): union-find, smallest id label. */
void og_components(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                   int64_t* label);
/* validate_rooted_forest (validate.cpp:108-211). roots may be NULL (then
 * the self-parent set is used). required_root -1 = none. Returns 1 valid,
 * 0 invalid (og_last_error() holds the first failure). */
int og_validate(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                const int64_t* offsets, const int64_t* nbrs,
                const int64_t* parent, const int64_t* roots, int64_t num_roots,
                int64_t required_root);
/* forest_depth (rooted_forest.cpp:12-95): max depth; <0 on cycle. */
int64_t og_forest_depth(int64_t n, const int64_t* parent);

#ifdef __cplusplus
}
#endif
#endif
