// Probe: does mma.sync.m16n8k16 f16->f32 consume fp16 subnormal A operands exactly?
// A = codes placed in the mantissa of zero-exponent halves (value c * 2^(off-24)), B = 2^k.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__global__ void k(float* out, int off) {
  const int lane = threadIdx.x;
  // every A element = code (lane % 4) at bit offset `off` in both halves
  const uint32_t c = (lane & 3) & 3;
  const uint32_t a = (c << off) | (c << (16 + off));
  const __half2 one = __floats2half2_rn(4096.f, 4096.f);  // B = 2^12
  const uint32_t b = *reinterpret_cast<const uint32_t*>(&one);
  float d[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
  out[lane * 4 + 0] = d[0]; out[lane * 4 + 1] = d[1]; out[lane * 4 + 2] = d[2]; out[lane * 4 + 3] = d[3];
}
int main() {
  float* o; cudaMalloc(&o, 128 * 4); float h[128];
  for (int off = 0; off <= 8; off += 2) {
    k<<<1, 32>>>(o, off); cudaMemcpy(h, o, 512, cudaMemcpyDeviceToHost);
    // row g, k: A[g][k] = code of lane (g*4 + k/2 % 4) ... just compare against the exact sum
    // every row sums 16 codes: sum over k of code(lane holding k) = 2*(0+1+2+3)*2 = 24 per row
    const double expect = 24.0 * (double)(1u << off) * 4096.0 / 16777216.0;  // *2^-24
    printf("off %d: D[0]=%.9g expect %.9g  %s\n", off, h[0], expect, h[0] == (float)expect ? "EXACT" : "MISMATCH");
  }
  return 0;
}
