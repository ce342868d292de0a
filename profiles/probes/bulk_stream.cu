// bulk_stream.cu -- read-bandwidth probe for the attention kernel's memory pipeline:
// persistent warps each stream a contiguous range of fixed-size records with cp.async.bulk
// into an S-stage shared-memory ring (mbarrier complete_tx), touching one word per record --
// the data movement of attend_*_kernel without its arithmetic. Baseline: a grid-stride
// 16-byte-load kernel. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 bulk_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) bulk_kernel(const uint8_t* __restrict__ src, size_t nrec, uint32_t rec,
                                                          int S, int nwarps, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * WARPS + warp;
  if (gw >= nwarps) return;
  uint8_t* ring = sm + (size_t)warp * (S * rec + 128);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + S * rec);
  const size_t r0 = nrec * gw / nwarps, r1 = nrec * (gw + 1) / nwarps;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  size_t nxt = r0;
  auto issue = [&](int s) {
    if (nxt < r1) {
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(rec) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                smem_u32(ring + (size_t)s * rec)),
            "l"(src + nxt * rec), "r"(rec), "r"(smem_u32(&bars[s])), "l"(pol)
            : "memory");
      }
      ++nxt;
    }
  };
  for (int s = 0; s < S; ++s) issue(s);
  uint32_t acc = 0, phase = 0;
  int s = 0;
  for (size_t r = r0; r < r1; ++r) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(&bars[s])),
        "r"(phase)
        : "memory");
    acc ^= reinterpret_cast<const uint32_t*>(ring + (size_t)s * rec)[lane];
    __syncwarp();
    issue(s);
    if (++s == S) {
      s = 0;
      phase ^= 1u;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t bytes = 3ull << 30;  // 3 GiB >> L2
  uint8_t* buf;
  uint32_t* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(e0);
    ldg_kernel<<<sms * 8, 512>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("ldg  grid-stride 16B loads: %.0f GB/s\n", bytes / ms / 1e6);
  const uint32_t recs[] = {3072, 6144, 12288};
  const int stages[] = {2, 4, 8};
  const int wpsm[] = {8, 16, 24, 32};
  for (uint32_t rec : recs)
    for (int S : stages)
      for (int w : wpsm) {
        const size_t per_warp = (size_t)S * rec + 128;
        const int warps_cta = 4;
        const size_t smem = per_warp * warps_cta;
        if (smem > 227 * 1024 || smem * (w / warps_cta) > 227 * 1024) continue;
        cudaFuncSetAttribute(bulk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(bulk_kernel<4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        const int nwarps = sms * w;
        const size_t nrec = bytes / rec;
        float best = 1e9;
        for (int it = 0; it < 3; ++it) {
          cudaEventRecord(e0);
          bulk_kernel<4><<<(nwarps + 3) / 4, 128, smem>>>(buf, nrec, rec, S, nwarps, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("bulk rec %5u B  stages %d  warps/SM %2d : %.0f GB/s %s\n", rec, S, w, nrec * (double)rec / best / 1e6,
               err == cudaSuccess ? "" : cudaGetErrorString(err));
      }
  return 0;
}
