// graphgen.hpp -- synthetic graph shapes shared by the host C++ generators
// and the device generators.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define RSTG_HD __host__ __device__ __forceinline__
#else
#define RSTG_HD inline
#endif

namespace rstg {

RSTG_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Road mesh: vertical edge (id, id+R) kept iff splitmix64(0x5eed ^ id) < thr.
RSTG_HD uint64_t road_threshold(double p) { return (uint64_t)(p * 18446744073709551615.0); }
RSTG_HD bool road_vertical(uint64_t id, uint64_t thr) { return splitmix64(0x5eedULL ^ id) < thr; }

// Seeded bijection on [0, 2^scale) used to scatter Kronecker ids.
RSTG_HD uint64_t kron_perm(uint64_t x, int scale) {
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

// Graph500 Kronecker tuple e (A,B,C) = (0.57,0.19,0.19), before permutation.
RSTG_HD void kron_tuple(uint64_t e, int scale, uint64_t* u, uint64_t* v) {
  uint64_t a = 0, b = 0;
  for (int bit = 0; bit < scale; ++bit) {
    const double r = (double)(splitmix64(e * 64ULL + (uint64_t)bit) >> 11) * (1.0 / 9007199254740992.0);
    const int q = r < 0.57 ? 0 : r < 0.76 ? 1 : r < 0.95 ? 2 : 3;
    a = (a << 1) | (uint64_t)(q >> 1);
    b = (b << 1) | (uint64_t)(q & 1);
  }
  *u = a;
  *v = b;
}

}  // namespace rstg
