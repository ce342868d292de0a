// Probe 2: precision of HMMA with fp16-subnormal A (codes * 2^-24) vs normal A (codes) for
// random fp16 B; reference in fp64. Prints max relative error of D for both encodings.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
__global__ void k(const uint32_t* A, const uint32_t* Bm, float* out, int sub) {
  const int lane = threadIdx.x;
  uint32_t a[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t x = A[lane * 4 + i];  // two codes (0..3) in the low bits of each half
    if (!sub) {  // normal encoding: exact fp16 integers
      __half2 h = __floats2half2_rn((float)(x & 0xffff), (float)(x >> 16));
      x = *reinterpret_cast<uint32_t*>(&h);
    }
    a[i] = x;
  }
  float d[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(Bm[lane * 2]), "r"(Bm[lane * 2 + 1]));
  for (int i = 0; i < 4; ++i) out[lane * 4 + i] = d[i];
}
int main() {
  uint32_t hA[128], hB[64];
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1103515245u + 12345u; return s >> 8; };
  for (int i = 0; i < 128; ++i) hA[i] = (rnd() % 4) | ((rnd() % 4) << 16);
  float bval[16][8];
  for (int kk = 0; kk < 16; ++kk) for (int n = 0; n < 8; ++n) bval[kk][n] = (float)((int)(rnd() % 60000) - 30000) * 0.5f;
  // B fragment: b0 = (k = 2t, 2t+1; n = g), b1 = (k = 2t+8, 2t+9; n = g)
  for (int lane = 0; lane < 32; ++lane) {
    int g = lane / 4, t = lane % 4;
    __half2 b0 = __floats2half2_rn(bval[2 * t][g], bval[2 * t + 1][g]);
    __half2 b1 = __floats2half2_rn(bval[2 * t + 8][g], bval[2 * t + 9][g]);
    hB[lane * 2] = *reinterpret_cast<uint32_t*>(&b0); hB[lane * 2 + 1] = *reinterpret_cast<uint32_t*>(&b1);
  }
  // A matrix from fragments: a0 = (row g, k 2t,2t+1), a1 = (row g+8, ...), a2 = (row g, k 2t+8..), a3
  double Am[16][16];
  for (int lane = 0; lane < 32; ++lane) {
    int g = lane / 4, t = lane % 4;
    int rows[4] = {g, g + 8, g, g + 8}, ks[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
    for (int i = 0; i < 4; ++i) { Am[rows[i]][ks[i]] = hA[lane * 4 + i] & 0xffff; Am[rows[i]][ks[i] + 1] = hA[lane * 4 + i] >> 16; }
  }
  uint32_t *dA, *dB; float* dO; cudaMalloc(&dA, 512); cudaMalloc(&dB, 256); cudaMalloc(&dO, 512);
  cudaMemcpy(dA, hA, 512, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  for (int sub = 0; sub < 2; ++sub) {
    k<<<1, 32>>>(dA, dB, dO, sub); float o[128]; cudaMemcpy(o, dO, 512, cudaMemcpyDeviceToHost);
    double maxrel = 0;
    for (int lane = 0; lane < 32; ++lane) {
      int g = lane / 4, t = lane % 4;
      int rr[4] = {g, g, g + 8, g + 8}, cc[4] = {2 * t, 2 * t + 1, 2 * t, 2 * t + 1};
      for (int i = 0; i < 4; ++i) {
        double ref = 0, mag = 0;
        for (int kk = 0; kk < 16; ++kk) { double bq = __half2float(__float2half_rn(bval[kk][cc[i]])); ref += Am[rr[i]][kk] * bq; mag += fabs(Am[rr[i]][kk] * bq); }
        if (sub) ref *= ldexp(1.0, -24), mag *= ldexp(1.0, -24);
        double e = fabs(o[lane * 4 + i] - ref) / (mag + 1e-300);
        if (e > maxrel) maxrel = e;
      }
    }
    printf("%s A: max |D - exact| / sum|products| = %.3e\n", sub ? "subnormal" : "normal", maxrel);
  }
  return 0;
}
