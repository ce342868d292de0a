// scratch.cu -- persistent per-(device, stream) attention scratch (attention.cuh Workspace)
// and the reference's scratch counter (scratch.hpp:14-21).
#include <atomic>
#include <map>
#include <memory>
#include <mutex>

#include "attention.cuh"

namespace kvb {

// Two scratch sets used alternately by consecutive calls on a stream: a layer's attention
// launch may overlap the previous layer's (programmatic dependent launch, attention_mma.cu),
// never the one before it, so neighbours never share scratch.
struct ScratchPool {
  std::mutex mu;          // held by the Workspace of the call in flight on this stream
  void* buf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [set][arena (uninitialised) / zeroed counters]
  size_t have[2][2] = {{0, 0}, {0, 0}};
  size_t want[2] = {0, 0};            // high-water marks seen (both sets grow to them)
  int parity = 0;                     // set of the next call
  int device = 0;
};

namespace {

std::atomic<uint64_t> g_scratch{0};
std::mutex g_pools_mu;
std::map<std::pair<int, cudaStream_t>, std::unique_ptr<ScratchPool>>& pools() {
  static auto* m = new std::map<std::pair<int, cudaStream_t>, std::unique_ptr<ScratchPool>>();
  return *m;  // leaked on purpose: freeing device memory after the driver shuts down fails
}

constexpr size_t kAlign = 256;

// The default memory pool returns freed memory to the driver at every synchronization unless
// a release threshold is set; the overflow allocations below would then be remapped per call.
void keep_pool(int dev) {
  static thread_local int done_dev = -1;
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  check_cuda(cudaDeviceGetDefaultMemPool(&pool, dev), "default mempool");
  uint64_t thr = 256ull << 20;
  check_cuda(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr), "mempool threshold");
  done_dev = dev;
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus s = cudaStreamCaptureStatusNone;
  check_cuda(cudaStreamIsCapturing(st, &s), "cudaStreamIsCapturing");
  return s != cudaStreamCaptureStatusNone;
}

}  // namespace

void scratch_add(size_t bytes) { g_scratch.fetch_add(bytes, std::memory_order_relaxed); }

Workspace::Workspace(cudaStream_t st) : st_(st) {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    auto& p = pools()[{dev, st}];
    if (!p) {
      p.reset(new ScratchPool());
      p->device = dev;
    }
    pool_ = p.get();
  }
  pool_->mu.lock();
  set_ = pool_->parity;
  pool_->parity ^= 1;
  try {
    grow();
  } catch (...) {
    pool_->mu.unlock();
    throw;
  }
}

// grow to the high-water mark of earlier calls (never inside a graph capture: the excess then
// stays on stream-ordered allocations)
void Workspace::grow() {
  cudaStream_t st = st_;
  const int k = set_;
  for (int z = 0; z < 2; ++z) {
    if (pool_->want[z] <= pool_->have[k][z] || capturing(st)) continue;
    check_cuda(cudaStreamSynchronize(st), "sync(scratch growth)");  // old buffer no longer in use
    if (pool_->buf[k][z]) check_cuda(cudaFree(pool_->buf[k][z]), "cudaFree(scratch)");
    pool_->buf[k][z] = nullptr;
    pool_->have[k][z] = 0;
    const size_t n = (pool_->want[z] + (pool_->want[z] >> 2) + kAlign - 1) / kAlign * kAlign;
    check_cuda(cudaMalloc(&pool_->buf[k][z], n), "cudaMalloc(scratch)");
    if (z == 1) check_cuda(cudaMemset(pool_->buf[k][z], 0, n), "cudaMemset(scratch)");
    pool_->have[k][z] = n;
  }
}

void* Workspace::take(size_t bytes, bool zero) {
  const int z = zero ? 1 : 0;
  bytes = (bytes + kAlign - 1) / kAlign * kAlign;
  bytes_ += bytes;
  scratch_add(bytes);
  const size_t off = off_[z];
  off_[z] += bytes;
  if (off_[z] > pool_->want[z]) pool_->want[z] = off_[z];
  if (off_[z] <= pool_->have[set_][z]) return static_cast<char*>(pool_->buf[set_][z]) + off;
  keep_pool(pool_->device);
  void* p = nullptr;
  check_cuda(cudaMallocAsync(&p, bytes, st_), "cudaMallocAsync(scratch)");
  extra_.push_back(p);
  if (zero) check_cuda(cudaMemsetAsync(p, 0, bytes, st_), "memset(scratch)");
  return p;
}

Workspace::~Workspace() {
  for (void* p : extra_) cudaFreeAsync(p, st_);
  pool_->mu.unlock();
}

}  // namespace kvb

using namespace kvb;

extern "C" {

void kvmix_scratch_reset(void) { g_scratch.store(0); }
uint64_t kvmix_scratch_allocated(void) { return g_scratch.load(); }

}  // extern "C"
