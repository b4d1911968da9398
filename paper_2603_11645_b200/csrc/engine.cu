// engine.cu -- Handle, workspace, phase timer, shared small kernels.
#include <map>
#include <mutex>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>

#include "engine.hpp"
#include "scan.cuh"

namespace rstg {

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

void ensure_dyn_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, func}];
  if (have >= bytes) return;
  CK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
}

// ---------------------------------------------------------------- timer
cudaEvent_t PhaseTimer::get() {
  if (used_ == pool_.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    pool_.push_back(e);
  }
  return pool_[used_++];
}
// Every phase is also an NVTX push/pop range (a no-op unless a tool is
// attached), so ncu --nvtx --print-nvtx-rename kernel attributes each
// launch to its phase (scripts/gpu_round.sh).
void PhaseTimer::begin(cudaStream_t s, const char* name, double bytes) {
  nvtxRangePushA(name);
  if (!enabled) return;
  Rec r{name, bytes, get(), nullptr};
  CK(cudaEventRecord(r.a, s));
  open_.push_back(recs_.size());
  recs_.push_back(r);
}
void PhaseTimer::end(cudaStream_t s) {
  nvtxRangePop();
  if (!enabled || open_.empty()) return;
  Rec& r = recs_[open_.back()];
  open_.pop_back();
  r.b = get();
  CK(cudaEventRecord(r.b, s));
}
std::vector<PhaseRec> PhaseTimer::collect() {
  std::vector<PhaseRec> out;
  for (auto& r : recs_) {
    if (!r.b) continue;
    CK(cudaEventSynchronize(r.b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    out.push_back(PhaseRec{r.name, (double)ms, r.bytes});
  }
  recs_.clear();
  open_.clear();
  used_ = 0;
  return out;
}

// --------------------------------------------------------------- handle
Handle::Handle(int dev) : device(dev) {
  CK(cudaSetDevice(dev));
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  CK(cudaMallocHost(&host_box, 64 * sizeof(int64_t)));
  CK(cudaMalloc(&dev_box, 256 * sizeof(int64_t)));
  // (defined contents: readbacks copy whole ranges of the box, some words of
  // which a given path never writes)
  memset(host_box, 0, 64 * sizeof(int64_t));
  CK(cudaMemset(dev_box, 0, 256 * sizeof(int64_t)));
  bufs_.assign(WS_COUNT, {nullptr, 0});
}

Handle::~Handle() {
  cudaSetDevice(device);
  cudaStreamSynchronize(stream);
  free_graph();
  for (auto& b : bufs_)
    if (b.first) cudaFree(b.first);
  cudaFree(dev_box);
  cudaFreeHost(host_box);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (own_stream) cudaStreamDestroy(stream);
}

void Handle::free_graph() {
  cudaFree(g.edges);
  cudaFree(g.offsets);
  cudaFree(g.nbrs);
  cudaFree(g.arc_edge);
  g = DeviceGraph{};
}

void* Handle::ws(int slot, size_t bytes) {
  auto& b = bufs_[slot];
  if (b.second < bytes) {
    // a new buffer (possibly at the old address) holds nothing known
    if (slot == WS_MINV) minv_clean = nullptr;
    if (slot == WS_RHEAD) rhead_clean = nullptr;
    if (slot == WS_XBITS) xbits_clean = nullptr;
    if (slot == WS_PR_SCRATCH || slot == WS_PR_ONPATH) pr_clean = nullptr;
    if (slot == WS_SLOT) slots_clean = nullptr;
    if (slot == WS_PR_BYL || slot == WS_PR_CBASE || slot == WS_PR_POS) pr_levels_n = -1;
    if (b.first) {
      CK(cudaStreamSynchronize(stream));
      CK(cudaFree(b.first));
    }
    size_t want = std::max(bytes, (size_t)256);
    CK(cudaMalloc(&b.first, want));
    b.second = want;
  }
  return b.first;
}

void Handle::release(int slot) {
  auto& b = bufs_[slot];
  if (slot == WS_MINV) minv_clean = nullptr;
  if (slot == WS_RHEAD) rhead_clean = nullptr;
  if (slot == WS_XBITS) xbits_clean = nullptr;
  if (slot == WS_PR_SCRATCH || slot == WS_PR_ONPATH) pr_clean = nullptr;
  if (slot == WS_SLOT) slots_clean = nullptr;
  if (slot == WS_PR_BYL || slot == WS_PR_CBASE || slot == WS_PR_POS) pr_levels_n = -1;
  if (b.first) {
    CK(cudaStreamSynchronize(stream));
    CK(cudaFree(b.first));
  }
  b = {nullptr, 0};
}

void Handle::read_box(const int64_t* dptr, int count) {
  CK(cudaMemcpyAsync(host_box, dptr, count * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
}

void Handle::set_stream(cudaStream_t s) {
  CK(cudaStreamSynchronize(stream));
  if (own_stream) CK(cudaStreamDestroy(stream));
  stream = s;
  own_stream = false;
}

// ------------------------------------------------------ scan partials
__global__ void k_scan_partials(uint32_t* partial, int64_t count) {
  // One CTA of 1024 threads walks the partials in chunks, carrying the sum.
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < count; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    uint32_t v = (i < count) ? partial[i] : 0u;
    uint32_t inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      uint32_t s = warp_sums[lane];
      uint32_t si = warp_incl_scan(s);
      warp_sums[lane] = si - s;
    }
    __syncthreads();
    uint32_t excl = carry_s + warp_sums[wid] + inc - v;
    if (i < count) partial[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[count] = carry_s;
}

// ------------------------------------------------------- roots ascending
namespace {
struct SelfParentFlag {
  const int32_t* parent;
  __device__ uint32_t operator()(int64_t v) const { return parent[v] == (int32_t)v ? 1u : 0u; }
};
}  // namespace

int64_t roots_ascending(Handle& h, const int32_t* parent, int32_t* roots) {
  return scan_emit(h, h.g.n, SelfParentFlag{parent},
                   EmitCompact{reinterpret_cast<uint32_t*>(roots)}, true);
}

}  // namespace rstg
