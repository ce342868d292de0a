// Probe: tcgen05.mma kind::i8 with A from TMEM (written by tcgen05.st 32x32b or 16x256b),
// B from shared memory (MN-major, no swizzle), int32 accumulators in TMEM. Validates the
// descriptor bits and the TMEM fragment maps the tcgen05 attention kernel relies on.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_i8_probe tc_i8_probe.cu && ./tc_i8_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int M = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MN-major, no swizzle: element (k, n) at (k/8)*LBO + (k%8)*16 + (n/16)*SBO + n%16
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int n, bool bsigned, bool b_mn) {
  return (2u << 4) | (0u << 7) | ((bsigned ? 1u : 0u) << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <int N, bool FRAG>
__global__ void probe(const uint8_t* A, const int8_t* B, int K, int* D, int bsigned) {
  __shared__ __align__(1024) uint8_t bs[256 * 64];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B: MN-major, LBO = 128 (8 k rows of 16 B), SBO = K*16 (all k of one 16-column chunk)
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i % N;
    bs[(k / 8) * 128 + (k % 8) * 16 + (n / 16) * (K * 16) + n % 16] = (uint8_t)B[k * N + n];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = taddr_s;
  const uint32_t ta = tbase + 128;  // A at column 128, D at column 0
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  if (!FRAG) {
    // 32x32b: thread = row, columns c = 4 K bytes
    for (int c = 0; c < K / 4; ++c) {
      const uint32_t v = *reinterpret_cast<const uint32_t*>(A + (size_t)tid * K + 4 * c);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(ta + lane_base + c), "r"(v));
    }
  } else {
    // 16x256b: lane (g, t) of half u: r0, r1 -> row g, cols 8x + 2t (+1); r2, r3 -> row g + 8
    const int g = lane >> 2, t = lane & 3;
    for (int u = 0; u < 2; ++u)
      for (int x = 0; x < K / 32; ++x) {
        uint32_t r[4];
        for (int i = 0; i < 4; ++i) {
          const int row = 32 * warp + 16 * u + g + 8 * (i >> 1);
          const int col = 8 * x + 2 * t + (i & 1);
          r[i] = *reinterpret_cast<const uint32_t*>(A + (size_t)row * K + 4 * col);
        }
        asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(ta + lane_base + ((uint32_t)(16 * u) << 16) + 8 * x),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]));
      }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (tid == 0) {
    const uint32_t id = idesc_i8(N, bsigned, true);
    for (int s = 0; s < K / 32; ++s) {
      const uint64_t bd = desc_mn(smem_u32(bs) + s * 4 * 128, 128, K * 16);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase),
          "r"(ta + 8 * s), "l"(bd), "r"(id), "r"(s));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  for (int c = 0; c < N; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tbase + lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    D[tid * N + c] = (int)v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tbase));
}

template <int N, bool FRAG>
int run(int K, int bsigned) {
  std::vector<uint8_t> A(M * K);
  std::vector<int8_t> B(K * N);
  srand(1234 + N + K + FRAG);
  for (auto& a : A) a = (uint8_t)(rand() & 0xff);
  for (auto& b : B) b = (int8_t)(rand() & 0xff);
  uint8_t* dA;
  int8_t* dB;
  int* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  probe<N, FRAG><<<1, 128>>>(dA, dB, K, dD, bsigned);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int> Dh(M * N);
  CK(cudaMemcpy(Dh.data(), dD, Dh.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      long ref = 0;
      for (int k = 0; k < K; ++k)
        ref += (long)A[m * K + k] * (bsigned ? (long)B[k * N + n] : (long)(uint8_t)B[k * N + n]);
      if (ref != Dh[m * N + n]) {
        if (bad < 5) printf("  mismatch m=%d n=%d ref=%ld got=%d\n", m, n, ref, Dh[m * N + n]);
        ++bad;
      }
    }
  printf("N=%d K=%d frag=%d bsigned=%d: %s (%d bad)\n", N, K, (int)FRAG, bsigned, bad ? "FAIL" : "ok", bad);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad;
}

int main() {
  int bad = 0;
  bad += run<16, false>(64, 1);
  bad += run<16, false>(64, 0);
  bad += run<16, true>(128, 1);
  bad += run<32, true>(128, 1);
  bad += run<64, true>(64, 0);
  bad += run<64, false>(128, 1);
  printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad != 0;
}
