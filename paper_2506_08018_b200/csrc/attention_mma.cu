// attention_mma.cu -- tensor-core (mma.sync m16n8k16) fused decode attention (placeholder).
#include "attention.cuh"

namespace kvb {
bool attend_mma(const kvmix_cache*, const void*, kvmix_dtype, int, int, float*, double*, Workspace&, cudaStream_t) {
  return false;
}
}  // namespace kvb
