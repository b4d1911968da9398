/* kron_uf.c -- TEST INFRASTRUCTURE ONLY (the checker for BASELINE config 5).
 *
 * Kronecker-28 (2^32 tuples, ~4.2e9 edges after normalize) is far beyond the
 * reference's host Graph (~200 GB), so its connectivity is
 * verified against an independent host computation in the spirit of
 * validate.cpp:46-53 (oracle_components), kept lean:
 *
 *   og_kron_uf    regenerates every tuple on the host with the same
 *                 generator as og_gen_kron (splitmix64
 *                 bits, (A,B,C) = (0.57,0.19,0.19), og_kron_perm) -- no edge
 *                 list is ever stored -- and unions its endpoints into an
 *                 int32 parent array (1 GiB at scale 28). Self-loops and
 *                 duplicate tuples are no-ops for a union-find, so normalize
 *                 (graph.cpp:39-46) is not needed for the partition.
 *   og_uf_edges   the same union-find over an explicit int32 edge list (the
 *                 GPU's tree edges): the list is a forest iff every union
 *                 merges two classes, i.e. iff roots == n - T.
 *
 * Both run on `threads` pthreads with a lock-free union-find: a union links
 * the larger root under the smaller with one CAS (ids only ever point to
 * smaller ids, so no cycle can form) and finds halve paths with CAS. The
 * final pass writes every vertex's root: the smallest id of its class.
 * Returns the number of classes.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

uint64_t og_splitmix64(uint64_t x);
uint64_t og_kron_perm(uint64_t x, int scale);

static inline int32_t uf_find(int32_t* p, int32_t x) {
  for (;;) {
    int32_t px = __atomic_load_n(&p[x], __ATOMIC_RELAXED);
    if (px == x) return x;
    int32_t gx = __atomic_load_n(&p[px], __ATOMIC_RELAXED);
    if (gx != px) __atomic_compare_exchange_n(&p[x], &px, gx, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED);
    x = gx;
  }
}

static inline void uf_unite(int32_t* p, int32_t a, int32_t b) {
  for (;;) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    if (a < b) {
      int32_t t = a;
      a = b;
      b = t;
    }
    int32_t expect = a;  /* a is still a root: link it under the smaller b */
    if (__atomic_compare_exchange_n(&p[a], &expect, b, 0, __ATOMIC_ACQ_REL, __ATOMIC_RELAXED))
      return;
  }
}

typedef struct {
  int kind; /* 0 init, 1 kron unions, 2 edge unions, 3 flatten + count */
  int scale;
  int64_t lo, hi;
  int32_t* parent;
  const int32_t* uv;
  int64_t count;
} uf_job;

static void* uf_worker(void* arg) {
  uf_job* j = (uf_job*)arg;
  int32_t* p = j->parent;
  if (j->kind == 0) {
    for (int64_t v = j->lo; v < j->hi; ++v) p[v] = (int32_t)v;
  } else if (j->kind == 1) {
    for (int64_t e = j->lo; e < j->hi; ++e) {
      uint64_t u = 0, v = 0;
      for (int b = 0; b < j->scale; ++b) {
        double r = (double)(og_splitmix64((uint64_t)e * 64ULL + (uint64_t)b) >> 11) *
                   (1.0 / 9007199254740992.0);
        int q = r < 0.57 ? 0 : r < 0.76 ? 1 : r < 0.95 ? 2 : 3;
        u = (u << 1) | (uint64_t)(q >> 1);
        v = (v << 1) | (uint64_t)(q & 1);
      }
      uf_unite(p, (int32_t)og_kron_perm(u, j->scale), (int32_t)og_kron_perm(v, j->scale));
    }
  } else if (j->kind == 2) {
    for (int64_t e = j->lo; e < j->hi; ++e) uf_unite(p, j->uv[2 * e], j->uv[2 * e + 1]);
  } else {
    int64_t c = 0;
    for (int64_t v = j->lo; v < j->hi; ++v) {
      int32_t r = uf_find(p, (int32_t)v);
      c += r == (int32_t)v;
      __atomic_store_n(&p[v], r, __ATOMIC_RELAXED);
    }
    j->count = c;
  }
  return NULL;
}

static int64_t run_jobs(int kind, int64_t total, int threads, int scale, int32_t* parent,
                        const int32_t* uv) {
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  uf_job* jobs = (uf_job*)calloc((size_t)threads, sizeof(uf_job));
  for (int t = 0; t < threads; ++t) {
    jobs[t].kind = kind;
    jobs[t].scale = scale;
    jobs[t].lo = total * t / threads;
    jobs[t].hi = total * (t + 1) / threads;
    jobs[t].parent = parent;
    jobs[t].uv = uv;
    pthread_create(&th[t], NULL, uf_worker, &jobs[t]);
  }
  int64_t sum = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    sum += jobs[t].count;
  }
  free(th);
  free(jobs);
  return sum;
}

/* Flatten: parent[v] = the smallest id of v's class (after all unions). */
static int64_t flatten(int64_t n, int threads, int32_t* parent) {
  return run_jobs(3, n, threads, 0, parent, NULL);
}

int64_t og_kron_uf(int scale, int edge_factor, int threads, int32_t* parent) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return -1;
  const int64_t n = (int64_t)1 << scale;
  run_jobs(0, n, threads, scale, parent, NULL);
  run_jobs(1, (int64_t)edge_factor << scale, threads, scale, parent, NULL);
  return flatten(n, threads, parent);
}

int64_t og_uf_edges(int64_t n, int64_t m, const int32_t* uv, int threads, int32_t* parent) {
  run_jobs(0, n, threads, 0, parent, NULL);
  run_jobs(2, m, threads, 0, parent, uv);
  return flatten(n, threads, parent);
}
