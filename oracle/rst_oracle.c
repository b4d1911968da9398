/*
 * rst_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Sequential plain-C restatement of the reference algorithms. Each function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core). A "step" of the reference's StepEngine
 * (step_engine.hpp:45-57) becomes one sequential loop here; the reference's
 * determinism contract (step_engine.hpp:27-33) guarantees any sequential
 * order of a step's bodies gives the parallel result, so these loops are
 * exact restatements, not approximations.
 */
#include "rst_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KNONE (-1)
#define KEYINF INT64_MAX /* kKeyInf, step_engine.hpp:143 */

static char g_err[256];
static void set_err(const char* s) {
  strncpy(g_err, s, sizeof g_err - 1);
  g_err[sizeof g_err - 1] = 0;
}
const char* og_last_error(void) { return g_err; }
void og_free(void* p) { free(p); }

/* types.hpp:24-32 */
static int ceil_log2(int64_t x) {
  int k = 0;
  int64_t p = 1;
  while (p < x) {
    p <<= 1;
    ++k;
  }
  return k;
}
static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
/* pack_key, step_engine.hpp:137-141 */
static int64_t pack_key(int64_t value, int64_t id) { return (value << 32) | id; }

/* ======================= graph ingestion ============================== */
typedef struct {
  int64_t u, v;
} edge_t;
static int cmp_edge(const void* a, const void* b) {
  const edge_t* x = (const edge_t*)a;
  const edge_t* y = (const edge_t*)b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return 0;
}

/* graph.cpp:39-46 */
int64_t og_normalize(int64_t m, int64_t* eu, int64_t* ev) {
  edge_t* e = (edge_t*)malloc(sizeof(edge_t) * (size_t)(m > 0 ? m : 1));
  int64_t k = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (eu[i] == ev[i]) continue; /* erase_if self-loop */
    int64_t a = eu[i], b = ev[i];
    if (a > b) {
      int64_t t = a;
      a = b;
      b = t;
    }
    e[k].u = a;
    e[k].v = b;
    ++k;
  }
  qsort(e, (size_t)k, sizeof(edge_t), cmp_edge);
  int64_t w = 0;
  for (int64_t i = 0; i < k; ++i) {
    if (w > 0 && e[w - 1].u == e[i].u && e[w - 1].v == e[i].v) continue;
    e[w++] = e[i];
  }
  for (int64_t i = 0; i < w; ++i) {
    eu[i] = e[i].u;
    ev[i] = e[i].v;
  }
  free(e);
  return w;
}

/* graph.cpp:133-172 */
int og_build_csr(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                 int64_t* offsets, int64_t* nbrs, int64_t* origin) {
  if (n < 0) {
    set_err("negative vertex count");
    return -1;
  }
  if (m > ((int64_t)1 << 32)) {
    set_err("too many edges");
    return -1;
  }
  memset(offsets, 0, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < m; ++i) {
    if (eu[i] < 0 || eu[i] >= n || ev[i] < 0 || ev[i] >= n) {
      set_err("edge endpoint out of range");
      return -1;
    }
    if (eu[i] == ev[i]) {
      set_err("self-loop in normalized EdgeList");
      return -1;
    }
    ++offsets[eu[i] + 1];
    ++offsets[ev[i] + 1];
  }
  for (int64_t v = 0; v < n; ++v) offsets[v + 1] += offsets[v];
  for (int64_t i = 1; i < m; ++i) {
    if (eu[i - 1] > eu[i] || (eu[i - 1] == eu[i] && ev[i - 1] >= ev[i])) {
      set_err("EdgeList not normalized");
      return -1;
    }
  }
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t v = 0; v < n; ++v) cursor[v] = offsets[v];
  for (int64_t i = 0; i < m; ++i) {
    int64_t u = eu[i], v = ev[i];
    nbrs[cursor[u]] = v;
    origin[cursor[u]++] = i;
    nbrs[cursor[v]] = u;
    origin[cursor[v]++] = i;
  }
  free(cursor);
  return 0;
}

/* ============================ generators ============================== */
static int64_t alloc_edges(int64_t cap, int64_t** eu, int64_t** ev) {
  *eu = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  *ev = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  return 0;
}

/* graph.cpp:181-188 */
int64_t og_gen_path(int64_t n, int64_t** eu, int64_t** ev) {
  if (n < 1) {
    set_err("path: n must be >= 1");
    return -1;
  }
  alloc_edges(n - 1, eu, ev);
  for (int64_t i = 0; i + 1 < n; ++i) {
    (*eu)[i] = i;
    (*ev)[i] = i + 1;
  }
  return n - 1;
}

/* graph.cpp:190-196 */
int64_t og_gen_star(int64_t n, int64_t** eu, int64_t** ev) {
  if (n < 1) {
    set_err("star: n must be >= 1");
    return -1;
  }
  alloc_edges(n - 1, eu, ev);
  for (int64_t i = 1; i < n; ++i) {
    (*eu)[i - 1] = 0;
    (*ev)[i - 1] = i;
  }
  return n - 1;
}

/* graph.cpp:198-210 */
int64_t og_gen_grid(int64_t rows, int64_t cols, int64_t** eu, int64_t** ev) {
  if (rows < 1 || cols < 1) {
    set_err("grid: dimensions must be >= 1");
    return -1;
  }
  alloc_edges(2 * rows * cols, eu, ev);
  int64_t k = 0;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      int64_t id = r * cols + c;
      if (c + 1 < cols) {
        (*eu)[k] = id;
        (*ev)[k++] = id + 1;
      }
      if (r + 1 < rows) {
        (*eu)[k] = id;
        (*ev)[k++] = id + cols;
      }
    }
  return og_normalize(k, *eu, *ev);
}

/* std::mt19937_64 (the engine gen_random draws from, graph.cpp:216). */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64_t;
static void mt64_seed(mt64_t* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}
static uint64_t mt64_next(mt64_t* s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t MA = 0xB5026F5AA96619E9ULL;
  if (s->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    }
    for (; i < 311; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    }
    uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* graph.cpp:212-235 (fixed-threshold draw on the raw 64-bit stream) */
int64_t og_gen_random(int64_t n, double p, uint64_t seed, int64_t** eu, int64_t** ev) {
  if (n < 1) {
    set_err("random: n must be >= 1");
    return -1;
  }
  if (p < 0.0 || p > 1.0) {
    set_err("random: p must be in [0,1]");
    return -1;
  }
  mt64_t rng;
  mt64_seed(&rng, seed);
  int always = p >= 1.0;
  uint64_t threshold = 0;
  if (!always && p > 0.0) {
    const long double two64 = 18446744073709551616.0L;
    const long double scaled = (long double)p * two64;
    if (scaled >= two64)
      always = 1;
    else
      threshold = (uint64_t)scaled;
  }
  int64_t cap = 1024, k = 0;
  alloc_edges(cap, eu, ev);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t v = u + 1; v < n; ++v) {
      uint64_t r = mt64_next(&rng);
      if (always || r < threshold) {
        if (k == cap) {
          cap *= 2;
          *eu = (int64_t*)realloc(*eu, sizeof(int64_t) * (size_t)cap);
          *ev = (int64_t*)realloc(*ev, sizeof(int64_t) * (size_t)cap);
        }
        (*eu)[k] = u;
        (*ev)[k++] = v;
      }
    }
  return k;
}

/* graph.cpp:237-244 */
int64_t og_gen_complete(int64_t n, int64_t** eu, int64_t** ev) {
  if (n < 1) {
    set_err("complete: n must be >= 1");
    return -1;
  }
  alloc_edges(n * (n - 1) / 2, eu, ev);
  int64_t k = 0;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t v = u + 1; v < n; ++v) {
      (*eu)[k] = u;
      (*ev)[k++] = v;
    }
  return k;
}

/* SURVEY.md Appendix B splitmix64 */
uint64_t og_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* SURVEY.md §8(d)/Appendix B road mesh. Emission order is already the
 * normalized (lexicographic) order. */
int64_t og_gen_road(int64_t R, double p, int64_t** eu, int64_t** ev) {
  if (R < 1) {
    set_err("road: R must be >= 1");
    return -1;
  }
  const uint64_t thr = (uint64_t)(p * 18446744073709551615.0);
  alloc_edges(2 * R * R, eu, ev);
  int64_t k = 0;
  for (int64_t r = 0; r < R; ++r)
    for (int64_t c = 0; c < R; ++c) {
      int64_t id = r * R + c;
      if (c + 1 < R) {
        (*eu)[k] = id;
        (*ev)[k++] = id + 1;
      }
      if (r + 1 < R && og_splitmix64(0x5eedULL ^ (uint64_t)id) < thr) {
        (*eu)[k] = id;
        (*ev)[k++] = id + R;
      }
    }
  return k;
}

/* Seeded bijection on [0, 2^scale): odd multiplies and xorshifts are each
 * invertible modulo 2^scale. Shared definition with the product generator
 * (documented in DESIGN.md). */
uint64_t og_kron_perm(uint64_t x, int scale) {
  const uint64_t mask = (scale >= 64) ? ~0ULL : ((1ULL << scale) - 1ULL);
  int s1 = (scale + 1) / 2, s2 = scale / 3 + 1;
  if (s1 < 1) s1 = 1;
  x = (x + 0x5eedULL) & mask;
  x = (x * 0x9e3779b97f4a7c15ULL) & mask;
  x ^= x >> s1;
  x = (x * 0xd6e8feb86659fd93ULL) & mask;
  x ^= x >> s2;
  x = (x * 0xbf58476d1ce4e5b9ULL) & mask;
  return x;
}

/* SURVEY.md Appendix B Kronecker (A,B,C)=(0.57,0.19,0.19). */
int64_t og_gen_kron(int scale, int edge_factor, int64_t** eu, int64_t** ev) {
  if (scale < 1 || scale > 30 || edge_factor < 1) {
    set_err("kron: bad parameters");
    return -1;
  }
  int64_t tuples = (int64_t)edge_factor << scale;
  alloc_edges(tuples, eu, ev);
  for (int64_t e = 0; e < tuples; ++e) {
    uint64_t u = 0, v = 0;
    for (int b = 0; b < scale; ++b) {
      double r = (double)(og_splitmix64((uint64_t)e * 64ULL + (uint64_t)b) >> 11) *
                 (1.0 / 9007199254740992.0);
      int q = r < 0.57 ? 0 : r < 0.76 ? 1 : r < 0.95 ? 2 : 3;
      u = (u << 1) | (uint64_t)(q >> 1);
      v = (v << 1) | (uint64_t)(q & 1);
    }
    (*eu)[e] = (int64_t)og_kron_perm(u, scale);
    (*ev)[e] = (int64_t)og_kron_perm(v, scale);
  }
  return og_normalize(tuples, *eu, *ev);
}

/* ======================= cc_forest.cpp ================================ */
/* hook_step, cc_forest.cpp:8-48 */
int og_hook_step(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                 int mode, int64_t* r, uint8_t* tree_flag, int64_t* slot) {
  int uncompressed = 0, any = 0;
  for (int64_t e = 0; e < m; ++e) { /* edge step :18-35 */
    int64_t ru = r[eu[e]], rv = r[ev[e]];
    if (r[ru] != ru || r[rv] != rv) {
      uncompressed = 1;
      continue;
    }
    if (ru == rv) continue;
    int64_t winner, loser;
    if (mode == 0) {
      winner = ru < rv ? ru : rv;
      loser = ru < rv ? rv : ru;
    } else {
      winner = ru < rv ? rv : ru;
      loser = ru < rv ? ru : rv;
    }
    int64_t key = pack_key(winner, e);
    if (key < slot[loser]) slot[loser] = key; /* combine_min */
  }
  if (uncompressed) {
    set_err("hooking ran on uncompressed labels");
    return -1;
  }
  for (int64_t v = 0; v < n; ++v) { /* apply step :39-46 */
    int64_t key = slot[v];
    if (key == KEYINF) continue;
    r[v] = key >> 32;
    tree_flag[key & 0xffffffffLL] = 1;
    slot[v] = KEYINF;
    any = 1;
  }
  return any;
}

/* jump_to_convergence, cc_forest.cpp:50-71 (double-buffered Jacobi). */
int64_t og_jump_to_convergence(int64_t n, int64_t* rep) {
  int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* snap = rep;
  int64_t* next = buf;
  const int64_t max_rounds = ceil_log2(max64(n, 1)) + 2;
  int64_t round;
  for (round = 0;; ++round) {
    if (round > max_rounds) {
      free(buf);
      set_err("pointer jumping failed to converge");
      return -1;
    }
    int done = 1;
    for (int64_t v = 0; v < n; ++v) {
      int64_t nv = snap[snap[v]];
      next[v] = nv;
      if (snap[nv] != nv) done = 0;
    }
    int64_t* t = snap;
    snap = next;
    next = t;
    if (done) break;
  }
  if (snap != rep) memcpy(rep, snap, sizeof(int64_t) * (size_t)n);
  free(buf);
  return round + 1;
}

/* cc_spanning_forest, cc_forest.cpp:73-102 */
int64_t og_cc_spanning_forest(int64_t n, int64_t m, const int64_t* eu,
                              const int64_t* ev, int64_t* labels,
                              uint8_t* tree_flag, int64_t* rounds_out) {
  int64_t* slot = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memset(tree_flag, 0, (size_t)m);
  for (int64_t v = 0; v < n; ++v) {
    labels[v] = v;
    slot[v] = KEYINF;
  }
  int mode = 0;
  int64_t round;
  for (round = 0;; ++round) {
    if (round > n + 1) {
      free(slot);
      set_err("hooking failed to converge");
      return -1;
    }
    int h = og_hook_step(n, m, eu, ev, mode, labels, tree_flag, slot);
    if (h < 0) {
      free(slot);
      return -1;
    }
    if (!h) break;
    if (og_jump_to_convergence(n, labels) < 0) {
      free(slot);
      return -1;
    }
    mode = !mode;
  }
  free(slot);
  if (rounds_out) *rounds_out = round + 1;
  int64_t T = 0;
  for (int64_t e = 0; e < m; ++e) T += tree_flag[e] ? 1 : 0;
  return T;
}

/* ======================= euler_rooting.cpp ============================ */
typedef struct {
  int64_t from, to, id;
} arc_t;
static int cmp_arc(const void* a, const void* b) {
  const arc_t* x = (const arc_t*)a;
  const arc_t* y = (const arc_t*)b;
  if (x->from != y->from) return x->from < y->from ? -1 : 1;
  if (x->to != y->to) return x->to < y->to ? -1 : 1;
  return 0;
}

/* build_euler, euler_rooting.cpp:13-74 */
int og_build_euler(int64_t n, int64_t T, const int64_t* tu, const int64_t* tv,
                   int64_t* from, int64_t* to, int64_t* first, int64_t* last,
                   int64_t* next) {
  const int64_t E = 2 * T;
  for (int64_t i = 0; i < n; ++i) first[i] = last[i] = KNONE;
  for (int64_t i = 0; i < T; ++i) {
    from[i] = tu[i];
    to[i] = tv[i];
    from[i + T] = tv[i];
    to[i + T] = tu[i];
  }
  arc_t* perm = (arc_t*)malloc(sizeof(arc_t) * (size_t)(E > 0 ? E : 1));
  for (int64_t i = 0; i < E; ++i) {
    perm[i].from = from[i];
    perm[i].to = to[i];
    perm[i].id = i;
  }
  qsort(perm, (size_t)E, sizeof(arc_t), cmp_arc); /* :49-54 */
  for (int64_t pos = 0; pos < E; ++pos) {         /* :62-72 */
    int64_t e = perm[pos].id;
    int64_t v = from[e];
    if (pos == 0 || perm[pos - 1].from != v) first[v] = e;
    if (pos == E - 1 || perm[pos + 1].from != v) {
      last[v] = e;
      next[e] = KNONE;
    } else {
      next[e] = perm[pos + 1].id;
    }
  }
  free(perm);
  return 0;
}

/* list_rank, euler_rooting.cpp:104-153 (Wyllie over predecessors). */
int og_list_rank(int64_t E, const int64_t* succ, int64_t* rank) {
  size_t sz = sizeof(int64_t) * (size_t)(E > 0 ? E : 1);
  int64_t* pr = (int64_t*)malloc(sz);
  int64_t *ja = (int64_t*)malloc(sz), *jb = (int64_t*)malloc(sz);
  int64_t *da = (int64_t*)malloc(sz), *db = (int64_t*)malloc(sz);
  for (int64_t e = 0; e < E; ++e) pr[e] = KNONE;
  for (int64_t e = 0; e < E; ++e)
    if (succ[e] != KNONE) pr[succ[e]] = e;
  int64_t *jump = ja, *jnext = jb, *dist = da, *dnext = db;
  for (int64_t e = 0; e < E; ++e) {
    jump[e] = pr[e];
    dist[e] = (pr[e] == KNONE) ? 0 : 1;
  }
  const int64_t max_rounds = ceil_log2(max64(E, 2)) + 2;
  int rc = 0;
  for (int64_t round = 0; E > 0; ++round) {
    if (round > max_rounds) {
      set_err("list ranking failed to converge: not a forest");
      rc = -1;
      break;
    }
    int done = 1;
    for (int64_t e = 0; e < E; ++e) {
      int64_t j = jump[e];
      if (j == KNONE) {
        jnext[e] = KNONE;
        dnext[e] = dist[e];
        continue;
      }
      jnext[e] = jump[j];
      dnext[e] = dist[e] + dist[j];
      if (jump[j] != KNONE) done = 0;
    }
    int64_t* t = jump;
    jump = jnext;
    jnext = t;
    t = dist;
    dist = dnext;
    dnext = t;
    if (done) break;
  }
  if (rc == 0)
    for (int64_t e = 0; e < E; ++e) rank[e] = dist[e];
  free(pr);
  free(ja);
  free(jb);
  free(da);
  free(db);
  return rc;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* euler_root_forest, euler_rooting.cpp:180-215, with compute_successor
 * (:76-87), break_cycles (:89-102), derive_parents (:155-178). */
int og_euler_root_forest(int64_t n, int64_t T, const int64_t* tu,
                         const int64_t* tv, const int64_t* labels,
                         int64_t designated_root, int64_t* parent,
                         int64_t* roots, int64_t* num_roots, int64_t* ranks_out) {
  if (designated_root != KNONE && (designated_root < 0 || designated_root >= n)) {
    set_err("designated root out of range");
    return -1;
  }
  int64_t* min_vertex = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  for (int64_t v = 0; v < max64(n, 1); ++v) min_vertex[v] = KEYINF;
  for (int64_t v = 0; v < n; ++v)
    if (v < min_vertex[labels[v]]) min_vertex[labels[v]] = v; /* :193-195 */
  if (designated_root != KNONE) min_vertex[labels[designated_root]] = designated_root;
  int64_t c = 0;
  for (int64_t v = 0; v < n; ++v)
    if (min_vertex[v] != KEYINF) roots[c++] = min_vertex[v]; /* :199-202 */
  free(min_vertex);
  if (T != n - c) {
    set_err("edge count does not match a spanning forest of the labeling");
    return -1;
  }
  const int64_t E = 2 * T;
  size_t sz = sizeof(int64_t) * (size_t)(E > 0 ? E : 1);
  size_t szn = sizeof(int64_t) * (size_t)(n > 0 ? n : 1);
  int64_t *from = (int64_t*)malloc(sz), *to = (int64_t*)malloc(sz);
  int64_t *next = (int64_t*)malloc(sz), *succ = (int64_t*)malloc(sz);
  int64_t *rank = (int64_t*)malloc(sz);
  int64_t *first = (int64_t*)malloc(szn), *last = (int64_t*)malloc(szn);
  og_build_euler(n, T, tu, tv, from, to, first, last, next);
  for (int64_t e = 0; e < E; ++e) { /* compute_successor :83-86 */
    int64_t r = (e + E / 2) % E;
    succ[e] = (next[r] != KNONE) ? next[r] : first[from[r]];
  }
  for (int64_t i = 0; i < c; ++i) { /* break_cycles :96-101 */
    int64_t l = last[roots[i]];
    if (l == KNONE) continue;
    succ[(l + E / 2) % E] = KNONE;
  }
  int rc = og_list_rank(E, succ, rank);
  if (rc == 0) {
    for (int64_t v = 0; v < n; ++v) parent[v] = v; /* derive_parents :167 */
    for (int64_t i = 0; i < T; ++i) {             /* :172-176 */
      int64_t ret = (rank[i] > rank[i + T]) ? i : i + T;
      parent[from[ret]] = to[ret];
    }
    qsort(roots, (size_t)c, sizeof(int64_t), cmp_i64); /* :163-164 */
    *num_roots = c;
    if (ranks_out) memcpy(ranks_out, rank, sz);
  }
  free(from);
  free(to);
  free(next);
  free(succ);
  free(rank);
  free(first);
  free(last);
  return rc;
}

/* cc_euler_rst, euler_rooting.cpp:217-226 */
int og_cc_euler_rst(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                    int64_t root, int64_t* parent, int64_t* roots,
                    int64_t* num_roots) {
  if (root < 0 || root >= n) {
    snprintf(g_err, sizeof g_err, "root %lld out of range", (long long)root);
    return -1;
  }
  int64_t* labels = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  uint8_t* flag = (uint8_t*)malloc((size_t)max64(m, 1));
  int64_t T = og_cc_spanning_forest(n, m, eu, ev, labels, flag, NULL);
  if (T < 0) {
    free(labels);
    free(flag);
    return -1;
  }
  int64_t* tu = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(T, 1));
  int64_t* tv = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(T, 1));
  int64_t k = 0;
  for (int64_t e = 0; e < m; ++e)
    if (flag[e]) {
      tu[k] = eu[e];
      tv[k++] = ev[e];
    }
  int rc = og_euler_root_forest(n, T, tu, tv, labels, root, parent, roots, num_roots, NULL);
  free(labels);
  free(flag);
  free(tu);
  free(tv);
  return rc;
}

/* ============================ pr_rst.cpp ============================== */
typedef struct {
  int64_t n, L;
  int64_t *parent, *rep, *scratch, *anc, *slot;
  uint8_t *on_path, *mark_buf;
  int64_t *graft_u, *graft_r;
  int64_t ngrafts;
} pr_state;

/* make_pr_state, pr_rst.cpp:40-70 */
static void pr_make(pr_state* st, int64_t n) {
  size_t nn = (size_t)max64(n, 1);
  st->n = n;
  st->L = ceil_log2(max64(n, 1));
  if (st->L < 1) st->L = 1;
  st->parent = (int64_t*)malloc(sizeof(int64_t) * nn);
  st->rep = (int64_t*)malloc(sizeof(int64_t) * nn);
  st->scratch = (int64_t*)malloc(sizeof(int64_t) * nn);
  st->slot = (int64_t*)malloc(sizeof(int64_t) * nn);
  st->anc = (int64_t*)malloc(sizeof(int64_t) * nn * (size_t)st->L);
  st->on_path = (uint8_t*)calloc(nn, 1);
  st->mark_buf = (uint8_t*)calloc(nn, 1);
  st->graft_u = (int64_t*)malloc(sizeof(int64_t) * nn);
  st->graft_r = (int64_t*)malloc(sizeof(int64_t) * nn);
  st->ngrafts = 0;
  for (int64_t v = 0; v < n; ++v) {
    st->parent[v] = st->rep[v] = v;
    st->scratch[v] = KNONE;
    for (int64_t k = 0; k < st->L; ++k) st->anc[v * st->L + k] = v;
    st->slot[v] = KEYINF;
  }
}
static void pr_free(pr_state* st) {
  free(st->parent);
  free(st->rep);
  free(st->scratch);
  free(st->slot);
  free(st->anc);
  free(st->on_path);
  free(st->mark_buf);
  free(st->graft_u);
  free(st->graft_r);
}

/* graft_round, pr_rst.cpp:72-133 */
static int pr_graft_round(pr_state* st, int64_t m, const int64_t* eu,
                          const int64_t* ev, int mode) {
  int64_t* rep = st->rep;
  int any = 0, uncompressed = 0;
  for (int64_t e = 0; e < m; ++e) {
    int64_t ru = rep[eu[e]], rv = rep[ev[e]];
    if (rep[ru] != ru || rep[rv] != rv) {
      uncompressed = 1;
      continue;
    }
    if (ru == rv) continue;
    int64_t winner = mode == 0 ? (ru < rv ? ru : rv) : (ru < rv ? rv : ru);
    int64_t loser = mode == 0 ? (ru < rv ? rv : ru) : (ru < rv ? ru : rv);
    int64_t key = pack_key(winner, e);
    if (key < st->slot[loser]) st->slot[loser] = key;
    any = 1;
  }
  if (uncompressed) {
    set_err("grafting ran on uncompressed reps");
    return -1;
  }
  st->ngrafts = 0;
  if (!any) return 0;
  for (int64_t v = 0; v < st->n; ++v) { /* resolve :112-122 */
    int64_t key = st->slot[v];
    if (key == KEYINF) continue;
    int64_t e = key & 0xffffffffLL;
    int64_t u = (rep[eu[e]] == v) ? eu[e] : ev[e];
    int64_t w = (u == eu[e]) ? ev[e] : eu[e];
    st->on_path[u] = 1;
    st->scratch[u] = w;
    st->graft_u[st->ngrafts] = u;
    st->graft_r[st->ngrafts++] = v; /* ascending v == sorted by r (:130) */
  }
  for (int64_t v = 0; v < st->n; ++v) { /* rep update :123-128 */
    int64_t key = st->slot[v];
    if (key == KEYINF) continue;
    rep[v] = key >> 32;
    st->slot[v] = KEYINF;
  }
  return 1;
}

/* mark_paths, pr_rst.cpp:135-164 */
static int64_t pr_mark_paths(pr_state* st) {
  const int64_t n = st->n, L = st->L;
  uint8_t *cur = st->on_path, *fresh = st->mark_buf;
  int64_t rounds = 0;
  for (int64_t k = 0; k < L; ++k) {
    int grew = 0;
    for (int64_t v = 0; v < n; ++v) {
      if (!cur[v]) continue;
      int64_t a = st->anc[v * L + k];
      if (!cur[a]) {
        fresh[a] = 1;
        grew = 1;
      }
    }
    ++rounds;
    if (!grew) break;
    for (int64_t v = 0; v < n; ++v)
      if (fresh[v]) {
        cur[v] = 1;
        fresh[v] = 0;
      }
  }
  return rounds;
}

/* reverse_paths, pr_rst.cpp:178-204 */
static int pr_reverse_paths(pr_state* st) {
  const int64_t n = st->n;
  for (int64_t v = 0; v < n; ++v) {
    if (!st->on_path[v]) continue;
    int64_t p = st->parent[v];
    if (p != v) st->scratch[p] = v;
  }
  int bad = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (!st->on_path[v]) continue;
    int64_t s = st->scratch[v];
    if (s == KNONE) {
      bad = 1;
      continue;
    }
    st->parent[v] = s;
    st->scratch[v] = KNONE;
    st->on_path[v] = 0;
  }
  if (bad) {
    set_err("reversal found a marked vertex with no source");
    return -1;
  }
  return 0;
}

/* batched_jump, pr_rst.cpp:216-252 (history snapshots are not kept). */
static int64_t pr_batched_jump(pr_state* st, int64_t batch) {
  if (batch < 1 || batch > 20) {
    set_err("jump batch out of range [1, 20]");
    return -1;
  }
  const int64_t n = st->n;
  const int64_t hops = (int64_t)1 << batch;
  int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  int64_t *snap = st->rep, *next = buf;
  const int64_t max_barriers = (ceil_log2(max64(n, 1)) + batch - 1) / batch + 2;
  int64_t barriers = 0;
  for (;;) {
    if (barriers > max_barriers) {
      if (snap != st->rep) memcpy(st->rep, snap, sizeof(int64_t) * (size_t)n);
      free(buf);
      set_err("pointer jumping detected a representative cycle");
      return -1;
    }
    int done = 1;
    for (int64_t v = 0; v < n; ++v) {
      int64_t x = snap[v];
      for (int64_t t = 1; t < hops; ++t) {
        int64_t nx = snap[x];
        if (nx == x) break;
        x = nx;
      }
      next[v] = x;
      if (snap[x] != x) done = 0;
    }
    int64_t* t = snap;
    snap = next;
    next = t;
    ++barriers;
    if (done) break;
  }
  if (snap != st->rep) memcpy(st->rep, snap, sizeof(int64_t) * (size_t)n);
  free(buf);
  return barriers;
}

/* rebuild_special_ancestors, pr_rst.cpp:254-265 */
static void pr_rebuild_anc(pr_state* st) {
  const int64_t n = st->n, L = st->L;
  for (int64_t v = 0; v < n; ++v) st->anc[v * L] = st->parent[v];
  for (int64_t k = 1; k < L; ++k)
    for (int64_t v = 0; v < n; ++v)
      st->anc[v * L + k] = st->anc[st->anc[v * L + (k - 1)] * L + (k - 1)];
}

/* pr_rst, pr_rst.cpp:267-314 */
int og_pr_rst(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
              int64_t root, int64_t jump_batch, int64_t* parent,
              int64_t* roots, int64_t* num_roots) {
  if (root < 0 || root >= n) {
    snprintf(g_err, sizeof g_err, "root %lld out of range", (long long)root);
    return -1;
  }
  pr_state st;
  pr_make(&st, n);
  int mode = 0;
  int rc = 0;
  for (int64_t round = 0;; ++round) {
    if (round > n + 1) {
      set_err("grafting failed to converge");
      rc = -1;
      break;
    }
    int g = pr_graft_round(&st, m, eu, ev, mode);
    if (g < 0) {
      rc = -1;
      break;
    }
    if (st.ngrafts == 0) break;
    pr_mark_paths(&st);
    for (int64_t i = 0; i < st.ngrafts && rc == 0; ++i) { /* :281-288 */
      int64_t r = st.graft_r[i];
      if (!st.on_path[r] || st.parent[r] != r) {
        snprintf(g_err, sizeof g_err, "path marking corrupted: %lld is not the root above %lld",
                 (long long)r, (long long)st.graft_u[i]);
        rc = -1;
      }
    }
    if (rc) break;
    if (pr_reverse_paths(&st) < 0 || pr_batched_jump(&st, jump_batch) < 0) {
      rc = -1;
      break;
    }
    pr_rebuild_anc(&st);
    mode = !mode;
  }
  if (rc == 0) {
    int64_t emergent = st.rep[root]; /* :298-303 */
    if (emergent != root) {
      st.on_path[root] = 1; /* mark_path :166-176 */
      pr_mark_paths(&st);
      if (!st.on_path[emergent] || st.parent[emergent] != emergent) {
        snprintf(g_err, sizeof g_err, "path marking corrupted: %lld is not the root above %lld",
                 (long long)emergent, (long long)root);
        rc = -1;
      } else {
        st.scratch[root] = root; /* reverse_path :206-214 */
        if (pr_reverse_paths(&st) < 0) rc = -1;
      }
    }
  }
  if (rc == 0) {
    int64_t c = 0;
    for (int64_t v = 0; v < n; ++v) {
      parent[v] = st.parent[v];
      if (parent[v] == v) roots[c++] = v; /* :305-313 */
    }
    *num_roots = c;
  }
  pr_free(&st);
  return rc;
}

/* ============================ bfs_rst.cpp ============================= */
/* bfs_rst.cpp:10-77, literal pull-based level-synchronous restatement. */
int og_bfs_rst(int64_t n, const int64_t* offsets, const int64_t* nbrs,
               int64_t root, int64_t* parent, int64_t* level, int64_t* roots,
               int64_t* num_roots) {
  if (root < 0 || root >= n) {
    snprintf(g_err, sizeof g_err, "root %lld out of range", (long long)root);
    return -1;
  }
  uint8_t* cur = (uint8_t*)calloc((size_t)n, 1);
  uint8_t* next = (uint8_t*)calloc((size_t)n, 1);
  int64_t seed = root, nr = 0;
  for (int64_t v = 0; v < n; ++v) {
    parent[v] = v;
    level[v] = (v == seed) ? 0 : KNONE;
    cur[v] = (v == seed);
  }
  roots[nr++] = seed;
  int rc = 0;
  for (;;) {
    int64_t guard = 0, next_seed = KNONE;
    for (int64_t d = 1;; ++d) {
      if (++guard > n + 1) {
        set_err("BFS failed to converge");
        rc = -1;
        break;
      }
      int changed = 0;
      int64_t restart = KEYINF;
      for (int64_t v = 0; v < n; ++v) {
        next[v] = 0;
        if (level[v] != KNONE) continue;
        int hit = 0;
        for (int64_t j = offsets[v]; j < offsets[v + 1]; ++j) {
          int64_t u = nbrs[j];
          if (cur[u]) {
            level[v] = d;
            parent[v] = u;
            next[v] = 1;
            changed = 1;
            hit = 1;
            break;
          }
        }
        if (!hit && v < restart) restart = v;
      }
      uint8_t* t = cur;
      cur = next;
      next = t;
      if (!changed) {
        if (restart != KEYINF) next_seed = restart;
        break;
      }
    }
    if (rc || next_seed == KNONE) break;
    seed = next_seed;
    roots[nr++] = seed;
    level[seed] = 0;
    cur[seed] = 1;
  }
  free(cur);
  free(next);
  *num_roots = nr;
  return rc;
}

/* O(n+m) restatement of bfs_rst: queue BFS from the
 * root, then from every smallest unvisited vertex in ascending order; the
 * parent is the smallest neighbour one level up (the first frontier hit of
 * the sorted pull scan at bfs_rst.cpp:49-55). */
int og_bfs_rst_fast(int64_t n, const int64_t* offsets, const int64_t* nbrs,
                    int64_t root, int64_t* parent, int64_t* level,
                    int64_t* roots, int64_t* num_roots) {
  if (root < 0 || root >= n) {
    snprintf(g_err, sizeof g_err, "root %lld out of range", (long long)root);
    return -1;
  }
  int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  for (int64_t v = 0; v < n; ++v) {
    parent[v] = v;
    level[v] = KNONE;
  }
  int64_t nr = 0, scan = 0;
  int64_t seed = root;
  for (;;) {
    roots[nr++] = seed;
    level[seed] = 0;
    int64_t head = 0, tail = 0;
    q[tail++] = seed;
    while (head < tail) {
      int64_t u = q[head++];
      for (int64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
        int64_t w = nbrs[j];
        if (level[w] != KNONE) continue;
        level[w] = level[u] + 1;
        q[tail++] = w;
      }
    }
    for (int64_t i = 1; i < tail; ++i) {
      int64_t v = q[i];
      for (int64_t j = offsets[v]; j < offsets[v + 1]; ++j)
        if (level[nbrs[j]] == level[v] - 1) {
          parent[v] = nbrs[j];
          break;
        }
    }
    while (scan < n && level[scan] != KNONE) ++scan;
    if (scan >= n) break;
    seed = scan;
  }
  free(q);
  *num_roots = nr;
  return 0;
}

/* ============================ validate.cpp ============================ */
static int64_t uf_find(int64_t* rep, int64_t v) { /* validate.cpp:21-31 */
  int64_t r = v;
  while (rep[r] != r) r = rep[r];
  while (rep[v] != r) {
    int64_t nx = rep[v];
    rep[v] = r;
    v = nx;
  }
  return r;
}

/* oracle_components, validate.cpp:46-53 */
void og_components(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                   int64_t* label) {
  for (int64_t v = 0; v < n; ++v) label[v] = v;
  for (int64_t e = 0; e < m; ++e) {
    int64_t a = uf_find(label, eu[e]), b = uf_find(label, ev[e]);
    if (a == b) continue;
    if (a > b) {
      int64_t t = a;
      a = b;
      b = t;
    }
    label[b] = a; /* smaller id stays representative (:33-41) */
  }
  for (int64_t v = 0; v < n; ++v) label[v] = uf_find(label, v);
}

static int has_edge(int64_t n, const int64_t* offsets, const int64_t* nbrs,
                    int64_t u, int64_t v) { /* graph.cpp:29-33 */
  if (u < 0 || u >= n || v < 0 || v >= n) return 0;
  int64_t lo = offsets[u], hi = offsets[u + 1];
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (nbrs[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < offsets[u + 1] && nbrs[lo] == v;
}

/* validate_rooted_forest, validate.cpp:108-211 */
int og_validate(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev,
                const int64_t* offsets, const int64_t* nbrs,
                const int64_t* parent, const int64_t* roots, int64_t num_roots,
                int64_t required_root) {
  int ok = 1;
  g_err[0] = 0;
  int64_t nself = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t p = parent[v];
    if (p < 0 || p >= n) {
      snprintf(g_err, sizeof g_err, "parent[%lld] = %lld out of range", (long long)v,
               (long long)p);
      return 0;
    }
    if (p == v) ++nself;
  }
  if (roots) { /* declared roots == self-parents (:118-135) */
    int64_t* d = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(num_roots, 1));
    memcpy(d, roots, sizeof(int64_t) * (size_t)num_roots);
    qsort(d, (size_t)num_roots, sizeof(int64_t), cmp_i64);
    int same = (num_roots == nself);
    int64_t k = 0;
    for (int64_t v = 0; v < n && same; ++v)
      if (parent[v] == v) same = (d[k++] == v);
    free(d);
    if (!same) {
      snprintf(g_err, sizeof g_err,
               "declared roots do not match self-parent vertices (%lld declared, %lld "
               "self-parents)",
               (long long)num_roots, (long long)nself);
      ok = 0;
    }
  }
  for (int64_t v = 0; v < n; ++v) { /* :137-145 */
    int64_t p = parent[v];
    if (p == v) continue;
    if (!has_edge(n, offsets, nbrs, v, p)) {
      if (ok)
        snprintf(g_err, sizeof g_err, "parent edge (%lld, %lld) is not a graph edge",
                 (long long)v, (long long)p);
      ok = 0;
    }
  }
  if (!ok) return 0;
  int64_t* chain_root = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  int64_t* stack = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  for (int64_t v = 0; v < n; ++v) chain_root[v] = KNONE;
  for (int64_t v = 0; v < n && ok; ++v) { /* :148-172 */
    if (chain_root[v] != KNONE) continue;
    int64_t cur = v, sp = 0;
    while (chain_root[cur] == KNONE) {
      int64_t p = parent[cur];
      if (p == cur) {
        chain_root[cur] = cur;
        break;
      }
      chain_root[cur] = -2;
      stack[sp++] = cur;
      cur = p;
      if (chain_root[cur] == -2) {
        snprintf(g_err, sizeof g_err, "parent chain cycle through vertex %lld",
                 (long long)cur);
        ok = 0;
        break;
      }
    }
    if (!ok) break;
    int64_t r = chain_root[cur];
    for (int64_t i = 0; i < sp; ++i) chain_root[stack[i]] = r;
  }
  if (ok) { /* :174-199 */
    int64_t* comp = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
    int64_t* root_of_comp = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
    og_components(n, m, eu, ev, comp);
    for (int64_t v = 0; v < n; ++v) root_of_comp[v] = KNONE;
    int64_t ncomp = 0, nroots_comp = 0;
    for (int64_t v = 0; v < n; ++v)
      if (comp[v] == v) ++ncomp;
    for (int64_t v = 0; v < n; ++v) {
      if (parent[v] != v) continue;
      int64_t c = comp[v];
      if (root_of_comp[c] != KNONE) {
        if (ok)
          snprintf(g_err, sizeof g_err, "component %lld has two roots: %lld and %lld",
                   (long long)c, (long long)root_of_comp[c], (long long)v);
        ok = 0;
      } else {
        root_of_comp[c] = v;
        ++nroots_comp;
      }
    }
    if (nroots_comp != ncomp) {
      if (ok)
        snprintf(g_err, sizeof g_err, "forest has %lld roots but graph has %lld components",
                 (long long)nroots_comp, (long long)ncomp);
      ok = 0;
    }
    for (int64_t v = 0; v < n; ++v) {
      if (comp[chain_root[v]] != comp[v]) {
        if (ok)
          snprintf(g_err, sizeof g_err, "vertex %lld reaches a root in a different component",
                   (long long)v);
        ok = 0;
        break;
      }
    }
    free(comp);
    free(root_of_comp);
  }
  free(chain_root);
  free(stack);
  if (ok && required_root != KNONE) { /* :201-209 */
    if (required_root < 0 || required_root >= n) {
      set_err("required root out of range");
      ok = 0;
    } else if (parent[required_root] != required_root) {
      snprintf(g_err, sizeof g_err, "vertex %lld was requested as root but is not one",
               (long long)required_root);
      ok = 0;
    }
  }
  return ok;
}

/* forest_depth, rooted_forest.cpp:12-95 (max depth only). */
int64_t og_forest_depth(int64_t n, const int64_t* parent) {
  int64_t* depth = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  int64_t* stack = (int64_t*)malloc(sizeof(int64_t) * (size_t)max64(n, 1));
  for (int64_t v = 0; v < n; ++v) depth[v] = -1;
  int64_t best = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (depth[v] >= 0) continue;
    int64_t cur = v, sp = 0;
    while (depth[cur] < 0) {
      if (depth[cur] == -2) {
        snprintf(g_err, sizeof g_err, "parent array contains a cycle at vertex %lld",
                 (long long)cur);
        free(depth);
        free(stack);
        return -1;
      }
      depth[cur] = -2;
      stack[sp++] = cur;
      int64_t p = parent[cur];
      if (p < 0 || p >= n) {
        snprintf(g_err, sizeof g_err, "parent out of range at vertex %lld", (long long)cur);
        free(depth);
        free(stack);
        return -1;
      }
      if (p == cur) {
        depth[cur] = 0;
        --sp;
        break;
      }
      cur = p;
    }
    while (sp > 0) {
      int64_t w = stack[--sp];
      depth[w] = depth[parent[w]] + 1;
    }
  }
  for (int64_t v = 0; v < n; ++v)
    if (depth[v] > best) best = depth[v];
  free(depth);
  free(stack);
  return best;
}
