// Probe: latency of tcgen05.mma kind::i8 (M=128, A in TMEM, B in smem) + commit -> mbarrier,
// for 4 k-steps at N = 16 / 64, and of tcgen05.st 16x256b.x4 + wait::st, tcgen05.ld + wait::ld.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_latency tc_latency.cu && ./tc_latency
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 10) | (1u << 16) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

template <int N>
__global__ void lat(long long* out) {
  __shared__ __align__(1024) uint8_t bs[128 * 64];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 64; i += 128) bs[i] = 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = taddr_s;
  long long t_mma = 0, t_st = 0, t_ld = 0;
  const int IT = 64;
  uint32_t regs[16];
  for (int i = 0; i < 16; ++i) regs[i] = 0x01010101u * (i + tid);
  for (int it = 0; it < IT; ++it) {
    // tcgen05.st 16x256b.x4 + wait
    long long a = clock64();
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16};\n" ::"r"(tb + 128 + ((uint32_t)(32 * warp) << 16)),
        "r"(regs[0]), "r"(regs[1]), "r"(regs[2]), "r"(regs[3]), "r"(regs[4]), "r"(regs[5]), "r"(regs[6]), "r"(regs[7]),
        "r"(regs[8]), "r"(regs[9]), "r"(regs[10]), "r"(regs[11]), "r"(regs[12]), "r"(regs[13]), "r"(regs[14]),
        "r"(regs[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    long long b = clock64();
    t_st += b - a;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // MMA: 4 k-steps + commit -> mbarrier wait
    a = clock64();
    if (tid == 0) {
      for (int x = 0; x < 4; ++x)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tb),
            "r"(tb + 128 + 8 * x), "l"(desc_mn(smem_u32(bs) + 512 * x, 128, 2048)), "r"(idesc_i8(N)), "r"(x));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                   : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}\n" ::"r"(
            smem_u32(&bar)),
        "r"(it & 1)
        : "memory");
    b = clock64();
    t_mma += b - a;
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    a = clock64();
    uint32_t v0, v1, v2, v3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                 : "r"(tb + ((uint32_t)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    b = clock64();
    t_ld += b - a;
    regs[it & 15] += v0 + v1 + v2 + v3;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
  }
  if (tid == 0) {
    out[0] = t_st / IT;
    out[1] = t_mma / IT;
    out[2] = t_ld / IT;
    out[3] = regs[3];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tb));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  long long h[4];
  lat<16><<<1, 128>>>(d);
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("N=16: sttm 16x256b.x4 + wait %lld cyc, 4x mma + commit + mbarrier wait %lld cyc, ldtm x4 + wait %lld cyc\n",
         h[0], h[1], h[2]);
  lat<64><<<1, 128>>>(d);
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("N=64: sttm %lld cyc, mma round trip %lld cyc, ldtm %lld cyc (%s)\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
