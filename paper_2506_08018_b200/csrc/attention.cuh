// attention.cuh -- decode attention entry points (attention.hpp:25-48).
#pragma once

#include <vector>

#include "cache.cuh"

namespace kvb {

// Stream-ordered scratch for split-K partials. Sizes depend on (B, H, rows, D) and the SM
// count only -- never on the cached token count (the reference's scratch contract,
// test_attention.cpp:182-205). Freed stream-ordered when the call returns, so concurrent
// readers on different streams never share scratch.
class Workspace {
 public:
  Workspace() = default;
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace() {
    for (auto& a : allocs_) cudaFreeAsync(a.first, a.second);
  }
  template <typename T>
  T* get(cudaStream_t st, size_t n) {
    keep_pool();
    void* p = nullptr;
    check_cuda(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st), "cudaMallocAsync(workspace)");
    allocs_.push_back({p, st});
    bytes_ += n * sizeof(T);
    return static_cast<T*>(p);
  }
  float2* ml(cudaStream_t st, size_t n) { return get<float2>(st, n); }
  float* acc(cudaStream_t st, size_t n) { return get<float>(st, n); }
  double* cs(cudaStream_t st, size_t n) { return get<double>(st, n); }
  size_t bytes() const { return bytes_; }

  // The default pool returns freed memory to the driver at every synchronization unless a
  // release threshold is set; a decode loop that synchronizes per step would then remap
  // its (tiny) scratch on every call (hundreds of microseconds). Keep it.
  static void keep_pool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (done_dev == dev) return;
    cudaMemPool_t pool;
    check_cuda(cudaDeviceGetDefaultMemPool(&pool, dev), "default mempool");
    uint64_t thr = 256ull << 20;
    check_cuda(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr), "mempool threshold");
    done_dev = dev;
  }

 private:
  std::vector<std::pair<void*, cudaStream_t>> allocs_;
  size_t bytes_ = 0;
};

void check_attend(const kvmix_cache* c, int q_heads, int t);
// split count used by every attention path: ~4 CTAs per SM, independent of T
int attend_splits(int BH);
void attend_generic(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
                    Workspace& ws, cudaStream_t st);
void attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
            Workspace& ws, cudaStream_t st);
void append_attend(kvmix_cache* c, const void* k, const void* v, kvmix_dtype kv_dt, int t, const void* q,
                   kvmix_dtype q_dt, int Hq, int tq, float* out, double* checksum, Workspace& ws, cudaStream_t st);
void fused_qk_scores(const kvmix_cache* c, const void* q, kvmix_dtype dt, int tq, float* scores, cudaStream_t st);
void softmax_rows(float* x, int64_t rows, int64_t cols, cudaStream_t st);
void fused_pv(const kvmix_cache* c, const float* probs, int tq, float* out, cudaStream_t st);
void reference_attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int tq, float* scratch, float* out,
                      double* checksum, Workspace& ws, cudaStream_t st);

__global__ void attend_combine_kernel(const float2* __restrict__ part_ml, const float* __restrict__ part_acc,
                                      int nsplit, int R, int H, int Hq, int tq, int D, float* __restrict__ out);
__global__ void checksum_kernel(const double* __restrict__ part, size_t n, double* out);

}  // namespace kvb
