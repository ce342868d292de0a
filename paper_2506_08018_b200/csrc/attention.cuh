// attention.cuh -- decode attention entry points (attention.hpp:25-48).
#pragma once

#include <vector>

#include "cache.cuh"

namespace kvb {

// Scratch for split-K partials, merge counters and append flags. Sizes depend on (B, H,
// rows, D) and the SM count only -- never on the cached token count (the reference's
// scratch contract, scratch.hpp:14-21, test_attention.cpp:182-205; kvmix_scratch_allocated
// reports the bytes requested).
//
// The memory is persistent per (device, stream): an arena for partials (uninitialised) and
// a zero-initialised buffer for arrival counters / flags, which the kernels return to zero
// before they exit -- so no call pays an allocation, a memset or a clearing launch, and
// calls on different streams never share scratch (concurrent readers). A call whose needs
// exceed the current buffers takes stream-ordered allocations for the excess and records
// the high-water mark; the next call on that stream grows the buffers (outside graph capture).
struct ScratchPool;
class Workspace {
 public:
  explicit Workspace(cudaStream_t st);
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace();
  template <typename T>
  T* get(cudaStream_t, size_t n) {
    return static_cast<T*>(take(std::max<size_t>(n, 1) * sizeof(T), false));
  }
  // zero on entry; the caller's kernels must leave it zero
  template <typename T>
  T* zeroed(size_t n) {
    return static_cast<T*>(take(std::max<size_t>(n, 1) * sizeof(T), true));
  }
  float2* ml(cudaStream_t st, size_t n) { return get<float2>(st, n); }
  float* acc(cudaStream_t st, size_t n) { return get<float>(st, n); }
  double* cs(cudaStream_t st, size_t n) { return get<double>(st, n); }
  size_t bytes() const { return bytes_; }

 private:
  void* take(size_t bytes, bool zero);
  void grow();
  cudaStream_t st_;
  ScratchPool* pool_;
  size_t off_[2] = {0, 0};  // bump offsets into the arena / the zeroed buffer
  int set_ = 0;             // scratch set of this call (alternates per stream)
  std::vector<void*> extra_;
  size_t bytes_ = 0;
};

// reference scratch counter (scratch.hpp:14-21): bytes of attention scratch requested
void scratch_add(size_t bytes);

void check_attend(const kvmix_cache* c, int q_heads, int t);
void check_query_shape(const kvmix_cache* c, int q_heads, int t);
// split count used by every attention path: ~4 CTAs per SM, independent of T
int attend_splits(int BH);
void attend_generic(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
                    Workspace& ws, cudaStream_t st);
void attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
            Workspace& ws, cudaStream_t st);
void append_attend(kvmix_cache* c, const void* k, const void* v, kvmix_dtype kv_dt, int t, const void* q,
                   kvmix_dtype q_dt, int Hq, int tq, float* out, double* checksum, Workspace& ws, cudaStream_t st);
// kvmix_*attend_layers on one device with distinct caches (k == nullptr: attention only):
// the layers the IMMA kernel serves share one launch per kernel instance
void attend_layers(kvmix_cache* const* caches, int n, const void* const* k, const void* const* v,
                   kvmix_dtype kv_dt, int t, const void* const* q, kvmix_dtype q_dt, int Hq, int tq,
                   float* const* out, cudaStream_t st);
void fused_qk_scores(const kvmix_cache* c, const void* q, kvmix_dtype dt, int tq, float* scores, cudaStream_t st);
void softmax_rows(float* x, int64_t rows, int64_t cols, cudaStream_t st);
void fused_pv(const kvmix_cache* c, const float* probs, int tq, float* out, cudaStream_t st);
void reference_attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int tq, float* scratch, float* out,
                      double* checksum, Workspace& ws, cudaStream_t st);

__global__ void attend_combine_kernel(const float2* __restrict__ part_ml, const float* __restrict__ part_acc,
                                      int nsplit, int R, int H, int Hq, int tq, int D, float* __restrict__ out);
__global__ void checksum_kernel(const double* __restrict__ part, size_t n, double* out);

}  // namespace kvb
