// Probe 3: the kernel's Key GEMV numerics. A = 2-bit codes (subnormal c*2^-24 or normal c),
// B = hi/lo fp16 split of x = q*s*sigma (max |x| in [2^14,2^15)), 8 chained k-steps (D=128).
// Reports max |(D_hi + D_lo) - exact| / sum|c x| over the 16 token rows.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <random>
#include <cuda_fp16.h>
__global__ void k(const uint32_t* A, const uint32_t* Bm, float* out, int sub) {
  const int lane = threadIdx.x;
  float d[4] = {0, 0, 0, 0};
  for (int ks = 0; ks < 8; ++ks) {
    uint32_t a[4];
    for (int i = 0; i < 4; ++i) {
      uint32_t x = A[(ks * 32 + lane) * 4 + i];
      if (!sub) { __half2 h = __floats2half2_rn((float)(x & 0xffff), (float)(x >> 16)); x = *reinterpret_cast<uint32_t*>(&h); }
      a[i] = x;
    }
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]),
                   "r"(Bm[(ks * 32 + lane) * 2]), "r"(Bm[(ks * 32 + lane) * 2 + 1]));
  }
  for (int i = 0; i < 4; ++i) out[lane * 4 + i] = d[i];
}
int main() {
  std::mt19937 rng(7); std::normal_distribution<float> nd(0.f, 1.f); std::uniform_int_distribution<int> ci(0, 3);
  static uint32_t hA[8 * 128], hB[8 * 64]; static double Am[16][128]; static double xs[128];
  float mx = 0; float raw[128];
  for (int d = 0; d < 128; ++d) { raw[d] = nd(rng) * (0.2f + 2.f * (d % 7) / 7.f); mx = fmaxf(mx, fabsf(raw[d])); }
  const float sig = ldexpf(1.f, 14 - (int)floorf(log2f(mx)));
  float hi[128], lo[128];
  for (int d = 0; d < 128; ++d) { float x = raw[d] * sig; xs[d] = x; __half h = __float2half_rn(x); hi[d] = __half2float(h); lo[d] = __half2float(__float2half_rn(x - hi[d])); }
  for (int ks = 0; ks < 8; ++ks)
    for (int lane = 0; lane < 32; ++lane) {
      int g = lane / 4, t = lane % 4;
      int rows[4] = {g, g + 8, g, g + 8}, kk[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
      for (int i = 0; i < 4; ++i) {
        int c0 = ci(rng), c1 = ci(rng);
        hA[(ks * 32 + lane) * 4 + i] = c0 | (c1 << 16);
        Am[rows[i]][ks * 16 + kk[i]] = c0; Am[rows[i]][ks * 16 + kk[i] + 1] = c1;
      }
      // B col 0 = hi, col 1 = lo, rest 0: b0 = (k 2t, 2t+1; n g), b1 = (k 2t+8, 2t+9; n g)
      float v[4] = {0, 0, 0, 0};
      int base = ks * 16;
      if (g == 0) { v[0] = hi[base + 2 * t]; v[1] = hi[base + 2 * t + 1]; v[2] = hi[base + 2 * t + 8]; v[3] = hi[base + 2 * t + 9]; }
      if (g == 1) { v[0] = lo[base + 2 * t]; v[1] = lo[base + 2 * t + 1]; v[2] = lo[base + 2 * t + 8]; v[3] = lo[base + 2 * t + 9]; }
      __half2 b0 = __floats2half2_rn(v[0], v[1]), b1 = __floats2half2_rn(v[2], v[3]);
      hB[(ks * 32 + lane) * 2] = *reinterpret_cast<uint32_t*>(&b0); hB[(ks * 32 + lane) * 2 + 1] = *reinterpret_cast<uint32_t*>(&b1);
    }
  uint32_t *dA, *dB; float* dO; cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dO, 512);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int sub = 0; sub < 2; ++sub) {
    k<<<1, 32>>>(dA, dB, dO, sub); float o[128]; cudaMemcpy(o, dO, 512, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int g = 0; g < 8; ++g) for (int h2 = 0; h2 < 2; ++h2) {
      int row = g + 8 * h2; int lane = g * 4;  // t = 0 holds cols 0 (hi), 1 (lo)
      double got = (double)o[lane * 4 + 2 * h2] + (double)o[lane * 4 + 2 * h2 + 1];
      if (sub) got *= ldexp(1.0, 24);
      double ref = 0, mag = 0; for (int d = 0; d < 128; ++d) { ref += Am[row][d] * xs[d]; mag += fabs(Am[row][d] * xs[d]); }
      worst = fmax(worst, fabs(got - ref) / mag);
    }
    printf("%s A: max |score - exact| / sum|c x| = %.3e\n", sub ? "subnormal" : "normal", worst);
  }
  return 0;
}
