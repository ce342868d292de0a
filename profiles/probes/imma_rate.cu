// Probe: legacy mma.sync throughput on sm_100a -- HMMA m16n8k16 f16->f32 vs IMMA m16n8k32
// u8 x s8 -> s32, per SM, with 8 independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int MODE>
__global__ void k(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  float f[8][4] = {};
  int i32[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (MODE == 0)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(f[c][0]), "+f"(f[c][1]), "+f"(f[c][2]), "+f"(f[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(i32[c][0]), "+r"(i32[c][1]), "+r"(i32[c][2]), "+r"(i32[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  uint32_t s = 0;
  for (int c = 0; c < 8; ++c)
    for (int e = 0; e < 4; ++e) s += __float_as_uint(f[c][e]) + (uint32_t)i32[c][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  uint32_t* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<148, warps * 32>>>(o, iters);
        else k<1><<<148, warps * 32>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double mma = 148.0 * warps * iters * 8;
        if (rep) printf("%s warps/SM %2d: %.3f ms, %.2f mma/clk/SM (at 1.965 GHz), %.1f cycles per mma per SMSP\n",
                        mode ? "IMMA.16832 u8.s8" : "HMMA.16816 f32", warps, ms, mma / 148 / (ms * 1e-3 * 1.965e9),
                        (ms * 1e-3 * 1.965e9) / (mma / 148 / 4));
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
