// common.cuh -- shared device/host plumbing for the B200 RST engine.
//
// Device data model: vertex ids int32, edge ids and CSR
// offsets uint32 (the reference caps n < 2^31, m <= 2^32; graph.cpp:17-18),
// hook keys uint64 packed (winner << 32) | edge, exactly pack_key
// (step_engine.hpp:137-141).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace rstg {

constexpr uint32_t kNone32 = 0xFFFFFFFFu;
// successor word of an arc whose slot holds no tree edge (never an arc id:
// 2N < 2^32 - 2; NONE is a tour's end)
constexpr uint32_t kEmptySlot = 0xFFFFFFFEu;
// kKeyInf = INT64_MAX exactly as the reference: every real key is below it
// (vertex ids < 2^31 - 1), so unsigned and signed order agree and an NCCL
// int64 MIN all-reduce combines slots like combine_min (multi-GPU CC).
constexpr unsigned long long kKeyInf = 0x7FFFFFFFFFFFFFFFull;
// Round-0 "has an edge" sentinel (graph.cu k_round0_keys): below empty,
// above every real key ((winner < 2^31) << 32 | e).
constexpr unsigned long long kKeyEdge = 0x7FFFFFFFFFFFFFFEull;
constexpr unsigned long long kAllOnes = 0xFFFFFFFFFFFFFFFFull;  // "no error yet" sentinels
constexpr int kBlock = 256;

// Algorithm-level failure carrying the reference's exception message.
struct AlgoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Input validation failure (reference: std::invalid_argument).
struct ArgError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                  cudaGetErrorString(e), file, line, what);
    throw std::runtime_error(buf);
  }
}
#define CK(x) ::rstg::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::rstg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

int num_sms();
// Raises a kernel's dynamic shared memory limit to `bytes` on the current
// device (the attribute is per device: one process may drive several GPUs).
// Thread-safe; a cheap lookup after the first call per (device, kernel).
void ensure_dyn_smem(const void* func, size_t bytes);
// Grid for a grid-stride loop over `work` items: enough CTAs to fill every SM
// (8 x 256 threads resident per SM), never more than the work needs.
inline unsigned grid_for(int64_t work, int block = kBlock) {
  int64_t need = (work + block - 1) / block;
  int64_t cap = (int64_t)num_sms() * (2048 / block) * 2;
  if (need < 1) need = 1;
  return (unsigned)(need < cap ? need : cap);
}

#ifdef __CUDACC__
// L1-bypassing loads for data other CTAs update within the same kernel
// (pointer-jumping shortcuts): any value ever stored is valid, fresher
// values only converge faster.
__device__ __forceinline__ int ld_cg(const int* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned ld_cg(const unsigned* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long* p) {
  return __ldcg(p);
}

__device__ __forceinline__ unsigned long long pack_key(uint32_t winner, uint32_t e) {
  return ((unsigned long long)winner << 32) | (unsigned long long)e;
}

// Block-level OR of a predicate, one global store per CTA that saw it.
__device__ __forceinline__ void block_flag(bool pred, int* flag) {
  if (__syncthreads_or(pred) && threadIdx.x == 0) *flag = 1;
}
#endif

}  // namespace rstg
