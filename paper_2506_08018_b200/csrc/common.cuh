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
void count_kernel(const char* name);  // per-kernel-name tally (kvmix_launch_count_of)
inline void after_launch(const char* what) {
  count_launch();
  count_kernel(what);
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
// The reference's group fold (quant.hpp:128-139, :170-182): mn = x0, then mn = v < mn ? v : mn
// in stream order -- a NaN first element makes the meta NaN, a later NaN is skipped, and among
// equal extrema (-0 / +0) the first occurrence wins. fold_min / fold_max start from NaN and
// skip NaNs keeping first occurrences; segments combine in stream order; the NaN-first rule
// is applied by the caller.
__device__ __forceinline__ float fold_min(float a, float b) { return (isnan(a) || b < a) ? b : a; }
__device__ __forceinline__ float fold_max(float a, float b) { return (isnan(a) || b > a) ? b : a; }

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

// encode() without the IEEE division on the common path. va = RN(x - min) * rcp(s) is
// within 2 ulp of v = RN((x - min) / s) (rcp.approx: 1 ulp, the product 0.5), i.e. within
// 2^-19 for every v below 16, so the rounding of va and v can differ only when va lies
// within that distance of a half-integer: there (and for NaN, infinities and |va| >= 2^62)
// the exact encode() decides. s_eff / rc / qm are the slot's scale (wide for Mixed3 narrow
// slots), its approximate reciprocal and code range; bit-exact with encode(x, scale, ...).
__device__ inline float rcp_approx(float s) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
  return r;
}
__device__ inline uint32_t encode_fast(float x, float scale, float minv, float s_eff, float rc, int qm, int bits,
                                       bool narrow) {
  constexpr float kTie = 0x1p-14f;  // 32x the worst-case distance between va and v
  if (s_eff == 0.0f) return 0u;
  const float va = __fmul_rn(__fsub_rn(x, minv), rc);
  if (va < 0.5f - kTie) return 0u;  // v < 0.5: rounds to <= 0 (also -inf)
  if (va > (float)qm - 0.5f + kTie && va < 0x1p62f) return (uint32_t)qm;
  const float t = va + 0.5f;  // va in [0.5 - kTie, qm - 0.5 + kTie]: error <= 2^-20
  const float r = floorf(t);
  const float f = t - r;
  if (f >= kTie && f <= 1.0f - kTie) return (uint32_t)r;
  return encode(x, scale, minv, bits, narrow);  // near a tie, NaN or huge: exact path
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
// Device cache tile layouts. A tile is 16 tokens x D channels of b-bit codes (D % 64 == 0),
// stored as 32 lanes x wpl words (wpl = D*b/64), in chunks of <= 4 words per lane so a
// warp's 128-bit loads are contiguous (plane_addr). The layouts are "fragment-native": lane
// l of a warp reads exactly the tensor-core A operands it owns, with no shuffles.
//
// 2- and 4-bit codes (both sides) -- IMMA layout, mma.sync m16n8k32 u8 A fragments
// (g = lane/4, t = lane%4; a0 = row g, k 4t..4t+3; a1 = row g+8; a2/a3 = k 16+4t..16+4t+3).
// A fragment register holds 4 codes, one per byte; a byte holds C = 8/b codes of
// different registers at bit offsets b*class, so one AND with 0x03030303 << 2*class
// (0x0F0F0F0F << 4*class) yields a register of u8 values code * 2^(b*class).
//   Keys (A = [token][channel], one k-step per 32 channels, NK = D/32): token i, channel
//     d = 32 kk + 16 h + 4 t + e, i = g + 8 rb: lane 4g+t, q = kk + NK h, word (q/C)*2 + rb,
//     bit 8e + b (q%C). The class depends on the channel only (folded into the B operand).
//   Values (A = [channel][token], one k-step per 32-token block = tiles 2m, 2m+1, one
//     m-tile per 16 channels, NM = D/16): token i = 4t + e of the tile, channel
//     d = 16 mt + 8 rh + g: lane 4g+t, q = mt + NM rh, word q/C, bit 8e + b (q%C). Tile 2m
//     holds a0/a1 (tokens 0..15 of the block), tile 2m+1 holds a2/a3; the class depends on
//     the channel only (undone per accumulator row).
// 3-bit Keys -- two IMMA planes: the low 2 bits in the 2-bit Key layout above, then the high
// bit in a 1-bit plane (C = 8 classes per byte): z = q + 2 NK rb, word z / 8, bit 8e + z % 8
// (for D = 128 the class z % 8 = q depends on the channel only).
// 3-bit Values -- the 4-bit IMMA Value layout (codes 0..7 in 4-bit fields): the class of a
// Value code depends on its channel (the accumulator row), so a dense 1-bit high plane cannot
// share the low plane's accumulators; 4-bit fields keep the Value side a plain IMMA k-step.
// (The reference's Mixed3 words are rebuilt bit-exactly on export; its byte accounting --
// MemoryReport, the roofline's algorithmic bytes -- stays the 3-bit one.)
// ---------------------------------------------------------------------------------------

// storage bits of a Value code: 3-bit Values use 4-bit fields (see above)
__host__ __device__ constexpr int vstore_bits(int bits) { return bits == 3 ? 4 : bits; }

// words per lane of one b-bit plane
__host__ __device__ constexpr int plane_wpl(int D, int b) { return D * b / 64; }
// total words of one tile at `bits` (3 -> 2-bit plane + 1-bit plane)
__host__ __device__ constexpr int tile_words(int D, int bits) {
  return bits == 3 ? 32 * (plane_wpl(D, 2) + plane_wpl(D, 1)) : 32 * plane_wpl(D, bits);
}
// word offset of (lane, w) inside a plane with `wpl` words per lane (chunks of <=4 words
// per lane so a warp's 128-bit loads are contiguous)
__host__ __device__ inline int plane_addr(int lane, int w, int wpl) {
  const int cw = wpl < 4 ? wpl : 4;
  const int sh = cw == 4 ? 2 : cw == 2 ? 1 : cw == 1 ? 0 : -1;  // D in {64, 128}: shifts
  if (sh >= 0) return ((w >> sh) << (5 + sh)) + (lane << sh) + (w & (cw - 1));
  return (w / cw) * (32 * cw) + lane * cw + (w % cw);
}


// IMMA layout (b in {2, 4}): word offset / bit shift of (token-in-tile i, channel d).
__host__ __device__ inline void imma_field(bool key, int D, int b, int i, int d, int* word, int* shift) {
  const int C = 8 / b;
  int lane, w, bit;
  if (key) {
    const int NK = D >> 5, kk = d >> 5, dc = d & 31, h = dc >> 4, t = (dc & 15) >> 2, e = dc & 3;
    const int q = kk + NK * h;
    lane = 4 * (i & 7) + t;
    w = (q / C) * 2 + (i >> 3);
    bit = 8 * e + b * (q % C);
  } else {
    const int NM = D >> 4, mt = d >> 4, dc = d & 15, rh = dc >> 3, g = dc & 7, t = i >> 2, e = i & 3;
    const int q = mt + NM * rh;
    lane = 4 * g + t;
    w = q / C;
    bit = 8 * e + b * (q % C);
  }
  *word = plane_addr(lane, w, plane_wpl(D, b));
  *shift = bit;
}

// Inverse of imma_field: the (i, d) of field f (0 .. 32/b-1; byte e = f / C, class f % C)
// of word w of lane `lane`.
__host__ __device__ inline void imma_element(bool key, int D, int b, int lane, int w, int f, int* i, int* d,
                                             int* shift) {
  const int C = 8 / b, e = f / C, cls = f % C;
  const int g = lane >> 2, t = lane & 3;
  *shift = 8 * e + b * cls;
  if (key) {
    const int NK = D >> 5;
    const int q = (w >> 1) * C + cls, rb = w & 1;
    const int kk = q % NK, h = q / NK;
    *i = g + 8 * rb;
    *d = 32 * kk + 16 * h + 4 * t + e;
  } else {
    const int NM = D >> 4;
    const int q = w * C + cls;
    const int mt = q % NM, rh = q / NM;
    *i = 4 * t + e;
    *d = 16 * mt + 8 * rh + g;
  }
}

// Every code of a tile is one field (bits 2/4) or two (bits 3: low 2 bits, high bit).
struct CodeLoc {
  int w0, s0;       // field of the code (bits 2/4) or of its low 2 bits (bits 3)
  int w1, s1;       // bits 3: field of the high bit (word offset includes the 2-bit plane)
};

// 1-bit high plane of 3-bit Keys (IMMA): word offset / bit of (token-in-tile i, channel d)
__host__ __device__ inline void imma_key_hi_field(int D, int i, int d, int* word, int* shift) {
  const int NK = D >> 5, kk = d >> 5, dc = d & 31, h = dc >> 4, t = (dc & 15) >> 2, e = dc & 3;
  const int z = kk + NK * h + 2 * NK * (i >> 3);
  *word = plane_addr(4 * (i & 7) + t, z >> 3, plane_wpl(D, 1));
  *shift = 8 * e + (z & 7);
}

// Inverse of imma_key_hi_field for field f (0..31; byte e = f / 8, class f % 8) of word w.
__host__ __device__ inline void imma_key_hi_element(int D, int lane, int w, int f, int* i, int* d, int* shift) {
  const int NK = D >> 5, e = f >> 3, z = 8 * w + (f & 7);
  const int q = z % (2 * NK), rb = z / (2 * NK);
  const int kk = q % NK, h = q / NK;
  *i = (lane >> 2) + 8 * rb;
  *d = 32 * kk + 16 * h + 4 * (lane & 3) + e;
  *shift = 8 * e + (f & 7);
}

__host__ __device__ inline CodeLoc code_loc(bool key, int D, int bits, int i, int d) {
  CodeLoc c{0, 0, -1, 0};
  if (bits == 3 && key) {
    imma_field(true, D, 2, i, d, &c.w0, &c.s0);
    imma_key_hi_field(D, i, d, &c.w1, &c.s1);
    c.w1 += 32 * plane_wpl(D, 2);
  } else {
    imma_field(key, D, key ? bits : vstore_bits(bits), i, d, &c.w0, &c.s0);
  }
  return c;
}

// Read a code from a tile (bits in {2,3,4}).
__device__ inline uint32_t tile_get(const uint32_t* tile, bool key, int D, int bits, int i, int d) {
  const CodeLoc c = code_loc(key, D, bits, i, d);
  if (bits == 3 && key) return ((tile[c.w0] >> c.s0) & 3u) | (((tile[c.w1] >> c.s1) & 1u) << 2);
  const int sb = key ? bits : vstore_bits(bits);
  return (tile[c.w0] >> c.s0) & ((1u << sb) - 1u);
}

// OR a code into a zero-initialised field (global or shared memory).
__device__ inline void tile_or(uint32_t* tile, bool key, int D, int bits, int i, int d, uint32_t code) {
  if (code == 0) return;
  const CodeLoc c = code_loc(key, D, bits, i, d);
  if (bits == 3 && key) {
    if (code & 3u) atomicOr(tile + c.w0, (code & 3u) << c.s0);
    if (code >> 2) atomicOr(tile + c.w1, (code >> 2) << c.s1);
  } else {
    atomicOr(tile + c.w0, code << c.s0);
  }
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

// SM count of the current device (cached per device)
inline int num_sms() {
  static int n[64] = {};
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 0 || dev >= 64) invalid("device ordinal out of range");
  if (n[dev] == 0) check_cuda(cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev), "sm count");
  return n[dev];
}

// Switches to a cache's device for the duration of a C ABI call (restores the caller's).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace kvb
