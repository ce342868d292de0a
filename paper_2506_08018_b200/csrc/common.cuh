// common.cuh -- shared device helpers for the B200 KVmix kernels (sm_100a).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/kvmix_b200.h"

namespace kvb {

// ---------------------------------------------------------------------------------------
// Error plumbing: internal code throws Error; the C ABI layer converts to kvmix_status.
// ---------------------------------------------------------------------------------------
struct Error : std::runtime_error {
  kvmix_status status;
  Error(kvmix_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(e == cudaErrorMemoryAllocation ? KVMIX_OUT_OF_MEMORY : KVMIX_CUDA_ERROR,
                std::string(what) + ": " + cudaGetErrorString(e));
  }
}

[[noreturn]] inline void invalid(const std::string& m) { throw Error(KVMIX_INVALID_ARGUMENT, m); }

void count_launch(int n = 1);
inline void after_launch(const char* what) {
  count_launch();
  check_cuda(cudaGetLastError(), what);
}

// ---------------------------------------------------------------------------------------
// Reference scalar semantics (bit-exact). IEEE fp32, no contraction: every mul/add that
// the reference rounds separately is spelled with __fmul_rn / __fadd_rn / __fdiv_rn.
// ---------------------------------------------------------------------------------------
// q_max_for_bits (quant.cpp:8-21)
__host__ __device__ inline int q_max_for_bits(int bits) {
  return bits == 1 ? 1 : bits == 2 ? 3 : bits == 3 ? 7 : 15;
}

// binary16 RNE == kvmix::half_from_float for every non-NaN float.
// NaN maps to sign|0x7e00 exactly like half.hpp:22-24 (cvt would emit 0x7fff).
__device__ inline uint16_t h16_bits(float x) {
  if (isnan(x)) return (uint16_t)((__float_as_uint(x) >> 16) & 0x8000u) | 0x7e00u;
  return __half_as_ushort(__float2half_rn(x));
}
__device__ inline float h16_float(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// make_group_meta (quant.hpp:93-98): packed {scale (lo 16), min (hi 16)} binary16 bits.
__device__ inline uint32_t make_meta(float mn, float mx, int q_max) {
  const uint16_t mh = h16_bits(mn);
  const uint16_t sh = h16_bits(__fdiv_rn(__fsub_rn(mx, mn), (float)q_max));
  return (uint32_t)sh | ((uint32_t)mh << 16);
}
__device__ inline float meta_scale(uint32_t m) { return h16_float((uint16_t)(m & 0xffffu)); }
__device__ inline float meta_min(uint32_t m) { return h16_float((uint16_t)(m >> 16)); }

// mixed3_wide_scale (quant.hpp:53): scale * (7.0f/3.0f), one rounded fp32 multiply.
__device__ inline float wide_scale(float s) { return __fmul_rn(s, 7.0f / 3.0f); }

// encode_element (quant.cpp:36-47). std::lround on x86-64 glibc returns LONG_MIN for NaN
// and |v| >= 2^63, which the clamp maps to 0; reproduce that instead of saturating.
__device__ inline uint32_t encode(float x, float scale, float minv, int bits, bool narrow) {
  int q_max = q_max_for_bits(bits);
  if (narrow) {
    scale = wide_scale(scale);
    q_max = 3;
  }
  if (scale == 0.0f) return 0u;
  const float v = __fdiv_rn(__fsub_rn(x, minv), scale);
  if (!(fabsf(v) < 0x1p63f)) return 0u;
  const float r = roundf(v);  // half away from zero == lround
  if (r <= 0.0f) return 0u;
  return r >= (float)q_max ? (uint32_t)q_max : (uint32_t)r;
}

// decode_code (quant.cpp:49-53): code*scale then +min, two rounded ops.
__device__ inline float decode(uint32_t code, float scale, float minv, bool narrow) {
  const float s = narrow ? wide_scale(scale) : scale;
  return __fadd_rn(__fmul_rn((float)code, s), minv);
}

// ---------------------------------------------------------------------------------------
// Reference word layout (bitpack.hpp:10-24): uniform b in {1,2,4} or Mixed3 (bits==3).
// ---------------------------------------------------------------------------------------
__host__ __device__ inline int codes_per_word(int bits) { return bits == 3 ? 11 : 32 / bits; }
__host__ __device__ inline uint32_t field_shift(int bits, uint32_t pos) {
  return bits == 3 ? (pos == 10 ? 30u : 3u * pos) : pos * (uint32_t)bits;
}
__host__ __device__ inline uint32_t field_mask(int bits, uint32_t pos) {
  return bits == 3 ? (pos == 10 ? 3u : 7u) : ((1u << bits) - 1u);
}
__host__ __device__ inline size_t words_for(size_t n, int bits) {
  return bits == 3 ? (n + 10) / 11 : (n * (size_t)bits + 31) / 32;
}

// ---------------------------------------------------------------------------------------
// Device cache tile layout ("fragment-native"). A tile is 16 tokens x D channels of
// b-bit codes, arranged so that each lane of a warp owns exactly the operands of an
// mma.sync m16n8k16 A fragment (rows g, g+8; cols 2t,2t+1, 2t+8,2t+9; g=lane/4,
// t=lane%4). Keys use A = [token][channel] (k-step kk = d/16), Values use
// A = [channel][token] (m-tile mt = d/16). Register r of the fragment holds the pair
// (lo half = first element, hi half = second element). Within a lane, fragment register
// r at slot s lives at virtual slot vs = r*(D/16) + s of a per-half bit stream with
// 16/b slots per 16-bit half. 3-bit codes are stored as a 2-bit plane (low bits) followed
// by a 1-bit plane (high bit). D must be a multiple of 64.
// ---------------------------------------------------------------------------------------
struct TileCoord {
  int lane, r, slot, half;
};

__host__ __device__ inline TileCoord key_coord(int i, int d) {
  const int kk = d >> 4, dc = d & 15;
  TileCoord c;
  c.half = dc & 1;
  c.r = (i >= 8 ? 1 : 0) + (dc >= 8 ? 2 : 0);
  c.lane = (i & 7) * 4 + ((dc & 7) >> 1);
  c.slot = kk;
  return c;
}

__host__ __device__ inline TileCoord value_coord(int i, int d) {
  const int mt = d >> 4, dc = d & 15;
  TileCoord c;
  c.half = i & 1;
  c.r = (dc >= 8 ? 1 : 0) + (i >= 8 ? 2 : 0);
  c.lane = (dc & 7) * 4 + ((i & 7) >> 1);
  c.slot = mt;
  return c;
}

// words per lane of one b-bit plane
__host__ __device__ inline int plane_wpl(int D, int b) { return D * b / 64; }
// total words of one tile at `bits` (3 -> 2-bit plane + 1-bit plane)
__host__ __device__ inline int tile_words(int D, int bits) {
  return bits == 3 ? 32 * (plane_wpl(D, 2) + plane_wpl(D, 1)) : 32 * plane_wpl(D, bits);
}
// word offset of (lane, w) inside a plane with `wpl` words per lane (chunks of <=4 words
// per lane so a warp's 128-bit loads are contiguous)
__host__ __device__ inline int plane_addr(int lane, int w, int wpl) {
  const int cw = wpl < 4 ? wpl : 4;
  return (w / cw) * (32 * cw) + lane * cw + (w % cw);
}

// Location (word offset within tile, bit shift) of a b-bit field of one plane.
__host__ __device__ inline void plane_field(const TileCoord& c, int D, int b, int* word, int* shift) {
  const int sph = 16 / b;
  const int vs = c.r * (D >> 4) + c.slot;
  const int w = vs / sph;
  *shift = c.half * 16 + (vs % sph) * b;
  *word = plane_addr(c.lane, w, plane_wpl(D, b));
}

// Read a code from a tile (bits in {2,3,4}).
__device__ inline uint32_t tile_get(const uint32_t* tile, const TileCoord& c, int D, int bits) {
  if (bits == 3) {
    int w, s;
    plane_field(c, D, 2, &w, &s);
    uint32_t lo = (tile[w] >> s) & 3u;
    plane_field(c, D, 1, &w, &s);
    uint32_t hi = (tile[32 * plane_wpl(D, 2) + w] >> s) & 1u;
    return lo | (hi << 2);
  }
  int w, s;
  plane_field(c, D, bits, &w, &s);
  return (tile[w] >> s) & ((1u << bits) - 1u);
}

// Mixed3 narrow-slot test from a segment-relative stream index (quant.cpp:39, :77-84).
__host__ __device__ inline bool is_narrow(int bits, uint64_t si) { return bits == 3 && si % 11 == 10; }

template <typename T>
__device__ inline float ld_f(const T* p);
template <>
__device__ inline float ld_f<float>(const float* p) { return *p; }
template <>
__device__ inline float ld_f<__half>(const __half* p) { return __half2float(*p); }

template <typename T>
__device__ inline T from_f(float x);
template <>
__device__ inline float from_f<float>(float x) { return x; }
template <>
__device__ inline __half from_f<__half>(float x) { return __float2half_rn(x); }

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    check_cuda(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
  }
  return n;
}

}  // namespace kvb
