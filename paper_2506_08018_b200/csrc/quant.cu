// quant.cu -- reference-layout quantize/pack, dequantize, pack/unpack kernels (sm_100a).
//
// Bit-exact with the reference's QuantizedGroups (quant.hpp:107-194, quant.cpp:36-124):
// the output words are the reference's PackedBuffer words for the whole tensor, in the
// reference stream order (Keys si = c*T + t, Values si = tok*D + d), including the Mixed3
// 11-per-word layout whose words straddle channel/token boundaries.
//
// Work decomposition (HBM-bound byte work; no tensor cores):
//  * Keys: one CTA per (b*H+h, span of n tokens, n a multiple of gs). The CTA stages the
//    contiguous [n][D] input slab in shared memory (coalesced 128-bit loads), computes the
//    per-(channel, group) metadata, and writes every output word whose FIRST code lies in
//    one of its D runs [c*T+t0, c*T+t0+n). The few trailing codes of such a word that
//    belong to the next run are encoded straight from global memory (their group meta is
//    recomputed from gs elements), so no word is shared between CTAs: no atomics, no
//    memset, one pass over the input.
//  * Values: the stream is the input order itself; one CTA per span of R rows (token
//    slots), thread-per-output-word, same ownership rule at the span end.
#include <algorithm>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace kvb {

namespace {

constexpr int kQThreads = 256;

template <typename T>
__device__ inline float gload(const T* x, size_t i) {
  return ld_f<T>(x + i);
}

// 16-byte vector of the input (8 halves / 4 floats) -> fp32
template <typename T>
struct Vec;
template <>
struct Vec<__half> {
  static constexpr int N = 8;
  __device__ static void unpack(const uint4& v, float* o) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(h[i]);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
  }
  __device__ static void load(const __half* p, float* o) { unpack(__ldg(reinterpret_cast<const uint4*>(p)), o); }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void unpack(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x);
    o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z);
    o[3] = __uint_as_float(v.w);
  }
  __device__ static void load(const float* p, float* o) { unpack(__ldg(reinterpret_cast<const uint4*>(p)), o); }
};

// One uniform 1/2/4-bit word of CPW codes sharing a group's (scale, min), bit-exact with
// encode(): va = RN(x - min) * rcp(scale) lies within 2^-19 of the reference quotient v, so
// clamp(va) rounded to the nearest integer (the 1.5 * 2^23 magic add: the integer lands in
// the low mantissa bits) is lround(v) unless va is within kTie of a half-integer; those codes
// (and, for fp32 inputs, NaN-free huge quotients the reference maps to 0) are redone by the
// exact encode() afterwards (rare). NaN -> 0 through the clamp, like the reference. fp16
// inputs cannot produce |v| >= 2^62 (|x - min| <= 2^17, scale >= 2^-24), so WIDE = false
// skips that check.
// sm_100 packed fp32 pairs (FADD2 / FMUL2): two IEEE round-to-nearest operations per
// instruction, bit-identical to two __fadd_rn / __fmul_rn
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  float2 r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return r;
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
  float2 r;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return r;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  float2 r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return r;
}

// (get(i): the word's i-th input as fp32, evaluated where used)
template <int BITS, int CPW, bool WIDE, typename Get>
__device__ __forceinline__ uint32_t encode_word_g(Get get, float sc, float mnv, int q_max) {
  constexpr float kTie = 0x1p-14f;
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  static_assert(CPW % 2 == 0, "codes in pairs");
  if (sc == 0.0f) return 0u;
  const float rc = rcp_approx(sc);
  const float qm = (float)q_max;
  const float2 mn2 = make_float2(mnv, mnv), rc2 = make_float2(rc, rc);
  const float2 mg2 = make_float2(kMagic, kMagic), nmg2 = make_float2(-kMagic, -kMagic);
  uint32_t word = 0;
  float far = 0.f;  // largest |vc - RN(vc)| of the word
  bool huge = false;
#pragma unroll
  for (int i = 0; i < CPW; i += 2) {
    const float2 va = f2_mul(f2_sub(make_float2(get(i), get(i + 1)), mn2), rc2);
    const float2 vc = make_float2(fminf(fmaxf(va.x, 0.f), qm), fminf(fmaxf(va.y, 0.f), qm));  // (NaN -> 0)
    const float2 u = f2_add(vc, mg2);
    const float2 dr = f2_sub(vc, f2_add(u, nmg2));  // vc - RN(vc), exact
    far = fmaxf(far, fmaxf(fabsf(dr.x), fabsf(dr.y)));
    if constexpr (WIDE) huge = huge || !(fabsf(va.x) < 0x1p62f) || !(fabsf(va.y) < 0x1p62f);
    word |= (__float_as_uint(u.x) & (uint32_t)q_max) << (BITS * i);
    word |= (__float_as_uint(u.y) & (uint32_t)q_max) << (BITS * (i + 1));
  }
  if (far > 0.5f - kTie || huge) {  // near a half-integer somewhere (rare): ties decide
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      const float va = __fmul_rn(__fsub_rn(get(i), mnv), rc);
      const float vc = fminf(fmaxf(va, 0.f), qm);
      const float dr = vc - __fsub_rn(__fadd_rn(vc, kMagic), kMagic);
      bool redo = fabsf(dr) > 0.5f - kTie;
      if constexpr (WIDE) redo = redo || !(fabsf(va) < 0x1p62f);
      if (redo)
        word = (word & ~((uint32_t)q_max << (BITS * i))) | (encode(get(i), sc, mnv, BITS, false) << (BITS * i));
    }
  }
  return word;
}

template <int BITS, int CPW, bool WIDE>
__device__ __forceinline__ uint32_t encode_word(const float (&v)[CPW], float sc, float mnv, int q_max) {
  return encode_word_g<BITS, CPW, WIDE>([&](int i) { return v[i]; }, sc, mnv, q_max);
}

// One interior Mixed3 word (quant.hpp:49-53): slots 0..9 3-bit with their group's scale,
// slot 10 the narrow 2-bit slot with the wide scale (scale * 7/3); slots k < kb belong to
// group a, k >= kb to group b (a word spans at most two groups). Branch-free like
// encode_word (the same 2^-19 bound: rcp.approx of the slot's scale, the magic-add rounding,
// a redo mask for near-ties; a zero scale gives a zero reciprocal, so its codes are 0 like
// encode()); flagged slots are redone by the exact encode() afterwards (rare).
template <bool WIDE>
__device__ __forceinline__ uint32_t encode_m3_word(const float (&v)[11], int kb, float sa, float na, float sb,
                                                   float nb) {
  constexpr float kTie = 0x1p-14f;
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  const float ra = sa == 0.0f ? 0.0f : rcp_approx(sa), rb = sb == 0.0f ? 0.0f : rcp_approx(sb);
  const float2 mg2 = make_float2(kMagic, kMagic);
  uint32_t word = 0;
  float far = 0.f;  // largest |vc - RN(vc)| of the word
  bool huge = false;
#pragma unroll
  for (int k = 0; k < 10; k += 2) {  // 3-bit slots in pairs (FADD2 / FMUL2)
    const float2 mn = make_float2(k >= kb ? nb : na, k + 1 >= kb ? nb : na);
    const float2 rc = make_float2(k >= kb ? rb : ra, k + 1 >= kb ? rb : ra);
    const float2 va = f2_mul(f2_sub(make_float2(v[k], v[k + 1]), mn), rc);
    const float2 vc = make_float2(fminf(fmaxf(va.x, 0.f), 7.f), fminf(fmaxf(va.y, 0.f), 7.f));  // (NaN -> 0)
    const float2 u = f2_add(vc, mg2);
    const float2 dr = f2_sub(vc, f2_sub(u, mg2));
    far = fmaxf(far, fmaxf(fabsf(dr.x), fabsf(dr.y)));
    if constexpr (WIDE) huge = huge || !(fabsf(va.x) < 0x1p62f) || !(fabsf(va.y) < 0x1p62f);
    word |= (__float_as_uint(u.x) & 7u) << (3 * k);
    word |= (__float_as_uint(u.y) & 7u) << (3 * k + 3);
  }
  {  // slot 10: the narrow slot (wide scale, codes 0..3)
    const bool hi = 10 >= kb;
    const float ws = wide_scale(hi ? sb : sa);
    const float rw = ws == 0.0f ? 0.0f : rcp_approx(ws);
    const float va = __fmul_rn(__fsub_rn(v[10], hi ? nb : na), rw);
    const float vc = fminf(fmaxf(va, 0.f), 3.f);
    const float u = __fadd_rn(vc, kMagic);
    far = fmaxf(far, fabsf(vc - __fsub_rn(u, kMagic)));
    if constexpr (WIDE) huge = huge || !(fabsf(va) < 0x1p62f);
    word |= (__float_as_uint(u) & 3u) << 30;
  }
  if (far > 0.5f - kTie || huge) {  // near a half-integer somewhere (rare): ties decide
#pragma unroll
    for (int k = 0; k < 11; ++k) {
      const bool hi = k >= kb;
      const float s = k == 10 ? wide_scale(hi ? sb : sa) : (hi ? sb : sa);
      const float rc = s == 0.0f ? 0.0f : rcp_approx(s);
      const float va = __fmul_rn(__fsub_rn(v[k], hi ? nb : na), rc);
      const float vc = fminf(fmaxf(va, 0.f), k == 10 ? 3.f : 7.f);
      const float dr = vc - __fsub_rn(__fadd_rn(vc, kMagic), kMagic);
      bool redo = fabsf(dr) > 0.5f - kTie;
      if constexpr (WIDE) redo = redo || !(fabsf(va) < 0x1p62f);
      if (redo) {
        const uint32_t sh = k == 10 ? 30u : 3u * k, mask = k == 10 ? 3u : 7u;
        word = (word & ~(mask << sh)) | (encode(v[k], hi ? sb : sa, hi ? nb : na, 3, k == 10) << sh);
      }
    }
  }
  return word;
}

// ---- Keys -------------------------------------------------------------------------------
// x: [B,H,T,D]; words/meta in reference order. Tile: n tokens (multiple of gs), all D.
// DT: compile-time head_dim (64 / 128: immediate shared-memory offsets; fp16 inputs fold and
// encode channel PAIRS from one 32-bit load) or 0 (runtime D).
template <typename T, int BITS, int DT>
__global__ void __launch_bounds__(kQThreads, BITS == 2 ? 5 : 6) quantize_key_kernel(const T* __restrict__ x, int H, int T_,
                                                                 int D_rt, int bits_rt, int gs, int n, int vec,
                                                                 uint32_t* __restrict__ words,
                                                                 uint32_t* __restrict__ meta,
                                                                 size_t n_total) {
  constexpr int bits = BITS;
  (void)bits_rt;
  const int D = DT ? DT : D_rt;
  constexpr bool PAIRS = DT != 0 && std::is_same<T, __half>::value;
  extern __shared__ __align__(16) uint8_t qsm[];
  // Mixed3 (gs >= 11): the last word of a channel's run holds up to 10 codes of the NEXT
  // run, all inside that run's first group; that group is staged too (rows nt .. nt+gs-1:
  // this channel's next span, or, at the end of the (b, kv-head), tokens 0 .. gs-1 for
  // channel d+1) so those codes and their group meta come from shared memory
  const int ext = (BITS == 3 && gs >= 11) ? 1 : 0;
  T* xs = reinterpret_cast<T*>(qsm);  // [n (+ gs)][D] in the input type (fp16 staging: 6 CTAs/SM)
  uint32_t* ms = reinterpret_cast<uint32_t*>(qsm + ((size_t)(n + ext * gs) * D * sizeof(T) + 15) / 16 * 16);  // [gst][D]
  const int bh = blockIdx.y;
  const int t0 = blockIdx.x * n;
  const int nt = min(n, T_ - t0);  // always a multiple of gs (T % gs == 0)
  const int gpt = nt / gs;
  const int gst = gpt + ext;       // meta columns per channel: [D][gst]
  const int gpc = T_ / gs;
  const int q_max = q_max_for_bits(bits);
  const T* src = x + ((size_t)bh * T_ + t0) * D;
  const bool next_span = t0 + nt < T_;

  auto stage = [&](T* dst, const T* from, int rows) {
    if (vec) {  // D % N == 0 and a 16-byte aligned input (host-checked): raw 16-byte copies,
                // 8 loads in flight per thread before the stores (one DRAM latency per batch)
      const int n16 = rows * D / Vec<T>::N;
      const uint4* s4 = reinterpret_cast<const uint4*>(from);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      const int nb = blockDim.x;
      int i = threadIdx.x;
      for (; i + 7 * nb < n16; i += 8 * nb) {
        uint4 r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __ldg(s4 + i + u * nb);
#pragma unroll
        for (int u = 0; u < 8; ++u) d4[i + u * nb] = r[u];
      }
      for (; i < n16; i += nb) d4[i] = __ldg(s4 + i);
    } else {
      for (int i = threadIdx.x; i < rows * D; i += blockDim.x) dst[i] = from[i];
    }
  };
  stage(xs, src, nt);
  if (ext) stage(xs + (size_t)nt * D, next_span ? src + (size_t)nt * D : x + (size_t)bh * T_ * D, gs);
  __syncthreads();

  // group meta: the reference's ordered fold (quant.hpp:128-139); fminf / fmaxf (and the fp16
  // __hmin2 / __hmax2, exact selections) skip NaN like it and differ from it only in the sign
  // of a zero extremum (the fold keeps the first of -0 / +0) and when the FIRST element is NaN
  // (the fold then stays NaN): those groups redo the ordered fold
  auto ordered = [&](int d, int g, float& mn, float& mx) {
    mn = mx = ld_f(&xs[(g * gs) * D + d]);
    for (int j = 1; j < gs; ++j) {
      const float v = ld_f(&xs[(g * gs + j) * D + d]);
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
  };
  if constexpr (PAIRS) {
    constexpr int DP = DT / 2;
    const __half2* xs2 = reinterpret_cast<const __half2*>(xs);
    // (uniform bits: the tile's meta offset once; Mixed3 keeps the per-store index, its 42-
    // register budget has no room for another live 64-bit value)
    const size_t mbase = BITS == 3 ? 0 : (size_t)bh * D * gpc + t0 / gs;
    for (int i = threadIdx.x; i < DP * gst; i += blockDim.x) {
      const int dp = i % DP, g = i / DP;
      const __half2* col = xs2 + (size_t)(g * gs) * DP + dp;
      const __half2 x0 = col[0];
      __half2 mn2 = x0, mx2 = x0;
      for (int j = 1; j < gs; ++j) {
        const __half2 v = col[j * DP];
        mn2 = __hmin2(mn2, v);
        mx2 = __hmax2(mx2, v);
      }
      const float2 fmn = __half22float2(mn2), fmx = __half22float2(mx2), f0 = __half22float2(x0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int d = 2 * dp + c;
        float mn = c ? fmn.y : fmn.x, mx = c ? fmx.y : fmx.x;
        if (mn == 0.f || mx == 0.f || isnan(c ? f0.y : f0.x)) ordered(d, g, mn, mx);
        const uint32_t m = make_meta(mn, mx, q_max);
        ms[g * D + d] = m;
        if (g < gpt)
          meta[BITS == 3 ? ((size_t)bh * D + d) * gpc + t0 / gs + g : mbase + (size_t)d * gpc + g] = m;
      }
    }
  } else
  for (int i = threadIdx.x; i < D * gst; i += blockDim.x) {
    const int d = i % D, g = i / D;  // d fastest: conflict-free smem columns
    const float x0 = ld_f(&xs[(g * gs) * D + d]);
    float mn = x0, mx = x0;
    for (int j = 1; j < gs; ++j) {
      const float v = ld_f(&xs[(g * gs + j) * D + d]);
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    if (mn == 0.f || mx == 0.f || isnan(x0)) ordered(d, g, mn, mx);
    const uint32_t m = make_meta(mn, mx, q_max);
    ms[g * D + d] = m;
    if (g < gpt) meta[((size_t)bh * D + d) * gpc + t0 / gs + g] = m;
  }
  __syncthreads();

  if constexpr (BITS != 3) {
    constexpr int CPW = 32 / BITS;
    if (gs % CPW == 0) {  // whole-group words (T % gs == 0): one meta per word, no run ends
      const int nwr = nt / CPW;
      const int nwr_sh = (nwr & (nwr - 1)) == 0 ? __ffs(nwr) - 1 : -1;
      const int gsh = (gs & (gs - 1)) == 0 ? __ffs(gs) - 1 : -1;  // (gs a power of two: shifts)
      if constexpr (PAIRS) {  // channels (2dp, 2dp+1): one 32-bit load per token, two words
        constexpr int DP = DT / 2;
        uint32_t* ow = ms + (size_t)gst * D;  // the tile's words [D][nwr + 1]
        const __half2* xs2 = reinterpret_cast<const __half2*>(xs);
        for (int i = threadIdx.x; i < DP * nwr; i += blockDim.x) {
          const int dp = i % DP, j = i / DP;
          __half2 hv[CPW];  // (kept packed: 16 registers for the two words' inputs)
#pragma unroll
          for (int k = 0; k < CPW; ++k) hv[k] = xs2[(j * CPW + k) * DP + dp];
          const int g = gsh >= 0 ? (j * CPW) >> gsh : (j * CPW) / gs;
          const uint2 m = *reinterpret_cast<const uint2*>(&ms[g * D + 2 * dp]);
          const size_t w = (((size_t)bh * D + 2 * dp) * (size_t)T_ + t0) / CPW + j;
          (void)w;
          ow[(2 * dp) * (nwr + 1) + j] = encode_word_g<BITS, CPW, false>([&](int k) { return __low2float(hv[k]); },
                                                                       meta_scale(m.x), meta_min(m.x), q_max);
          ow[(2 * dp + 1) * (nwr + 1) + j] = encode_word_g<BITS, CPW, false>(
              [&](int k) { return __high2float(hv[k]); }, meta_scale(m.y), meta_min(m.y), q_max);
        }
        // the tile's words leave channel by channel: a channel's run of nwr words is written by
        // consecutive threads (whole sectors per store instead of one word per channel row)
        __syncthreads();
        for (int i = threadIdx.x; i < D * nwr; i += blockDim.x) {
          const int d = nwr_sh >= 0 ? i >> nwr_sh : i / nwr, j = i - d * nwr;
          words[(((size_t)bh * D + d) * (size_t)T_ + t0) / CPW + j] = ow[d * (nwr + 1) + j];
        }
        return;
      }
      for (int i = threadIdx.x; i < D * nwr; i += blockDim.x) {
        const int d = i % D, j = i / D;  // a warp reads 32 consecutive channels of a token row
        float v[CPW];
#pragma unroll
        for (int k = 0; k < CPW; ++k) v[k] = ld_f(&xs[(j * CPW + k) * D + d]);
        const uint32_t m = ms[(j * CPW) / gs * D + d];
        const size_t w = (((size_t)bh * D + d) * (size_t)T_ + t0) / CPW + j;
        words[w] = encode_word<BITS, CPW, !std::is_same<T, __half>::value>(v, meta_scale(m), meta_min(m), q_max);
      }
      return;
    }
  }
  const int cpw = codes_per_word(bits);
  // every thread emits words: thread i -> channel d = i % D (a warp reads 32 consecutive
  // channels of one token row: conflict-free), word j = i / D of that channel's run. A
  // run's owned words are those whose FIRST code lies in it; trailing codes of the last
  // one that belong to the next run are encoded straight from global memory.
  // (gs a power of two: group index by shift)
  const int gsh = (gs & (gs - 1)) == 0 ? __ffs(gs) - 1 : -1;
  auto emit = [&](const int d, const size_t s0, const size_t w) {
    const size_t s1 = s0 + nt;
    const size_t p0 = w * cpw;
    uint32_t word = 0;
    if constexpr (BITS == 3) {
      if (gs >= 11 && p0 + 11 <= s1) {  // interior Mixed3 word: <= two groups, slot 10 narrow
        const int tt0 = (int)(p0 - s0);
        const int j0 = gsh >= 0 ? tt0 >> gsh : tt0 / gs, kb = (j0 + 1) * gs - tt0;  // first code of group j0 + 1
        const uint32_t ma = ms[j0 * D + d], mb = kb < 11 ? ms[(j0 + 1) * D + d] : ma;
        float xv[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) xv[k] = ld_f(&xs[(tt0 + k) * D + d]);
        words[w] = encode_m3_word<!std::is_same<T, __half>::value>(xv, kb, meta_scale(ma), meta_min(ma),
                                                                   meta_scale(mb), meta_min(mb));
        return;
      }
      // run-end word: codes of this run's last group, then (from slot kb = nt - tt0, 1..10)
      // of the next run's first group, staged at rows nt .. (channel d of the next span, or
      // channel d + 1 at the end of the (b, kv-head)); p0 % 11 == 0, so slot 10 is the narrow
      // one as in an interior word
      const int dn = next_span ? d : d + 1;
      if (ext && dn < D && p0 + 11 <= n_total) {
        const int tt0 = (int)(p0 - s0), kb = nt - tt0;
        const uint32_t ma = ms[(gpt - 1) * D + d], mb = ms[gpt * D + dn];
        float xv[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) xv[k] = k < kb ? ld_f(&xs[(tt0 + k) * D + d]) : ld_f(&xs[(nt + k - kb) * D + dn]);
        words[w] = encode_m3_word<!std::is_same<T, __half>::value>(xv, kb, meta_scale(ma), meta_min(ma),
                                                                   meta_scale(mb), meta_min(mb));
        return;
      }
    }
    int tt = (int)(p0 - s0);                                    // token of the first code
    int r11 = bits == 3 ? (int)(p0 % 11u) : 0;                  // stream index mod 11
    int g = tt / gs, gend = (g + 1) * gs;                       // current group and its end
    uint32_t m = ms[g * D + d];
    float sc = meta_scale(m), mnv = meta_min(m), rc = rcp_approx(sc);
    float ws = 0.f, rcw = 0.f;  // Mixed3 narrow slots: wide scale and its reciprocal
    if (bits == 3) {
      ws = wide_scale(sc);
      rcw = rcp_approx(ws);
    }
    int k = 0;
    for (; k < cpw && tt < nt; ++k, ++tt) {
      if (tt == gend) {
        ++g;
        gend += gs;
        m = ms[g * D + d];
        sc = meta_scale(m);
        mnv = meta_min(m);
        rc = rcp_approx(sc);
        if (bits == 3) {
          ws = wide_scale(sc);
          rcw = rcp_approx(ws);
        }
      }
      const bool nar = bits == 3 && r11 == 10;
      const uint32_t code = encode_fast(ld_f(&xs[tt * D + d]), sc, mnv, nar ? ws : sc, nar ? rcw : rc, nar ? 3 : q_max, bits, nar);
      word |= code << field_shift(bits, (uint32_t)k);
      if (++r11 == 11) r11 = 0;
    }
    if (ext && k < cpw) {  // codes of the next run: its first group, staged at rows nt ..
      const int dn = next_span ? d : d + 1;
      if (dn < D) {
        const uint32_t m2 = ms[gpt * D + dn];
        const float s2 = meta_scale(m2), n2 = meta_min(m2);
        for (int r = 0; k < cpw && p0 + k < n_total; ++k, ++r)
          word |= encode(ld_f(&xs[(nt + r) * D + dn]), s2, n2, bits, is_narrow(bits, p0 + k)) << field_shift(bits, (uint32_t)k);
      }
    }
    size_t cached = ~(size_t)0;  // codes of the next (b, kv-head): group meta once
    float sc2 = 0.f, mn2 = 0.f;
    for (; k < cpw; ++k) {
      const size_t p = p0 + k;
      if (p >= n_total) break;
      const size_t c2 = p / T_;
      const int t2 = (int)(p % T_);
      const size_t bh2 = c2 / D;
      const int d2 = (int)(c2 % D);
      const size_t grp = c2 * (size_t)gpc + (size_t)(t2 / gs);
      if (grp != cached) {
        const T* base = x + (bh2 * T_ + (size_t)(t2 / gs) * gs) * D + d2;
        float mn = gload(base, 0), mx = mn;
        for (int jj = 1; jj < gs; ++jj) {
          const float v = gload(base, (size_t)jj * D);
          mn = v < mn ? v : mn;
          mx = v > mx ? v : mx;
        }
        const uint32_t m2 = make_meta(mn, mx, q_max);
        sc2 = meta_scale(m2);
        mn2 = meta_min(m2);
        cached = grp;
      }
      const float xv = gload(x, (bh2 * T_ + t2) * D + d2);
      word |= encode(xv, sc2, mn2, bits, is_narrow(bits, p)) << field_shift(bits, (uint32_t)k);
    }
    words[w] = word;
  };
  if (blockDim.x % D == 0) {  // a thread keeps its channel: run bounds once per thread
    const int d = threadIdx.x % D;
    const size_t s0 = ((size_t)bh * D + d) * (size_t)T_ + t0, s1 = s0 + nt;
    const size_t w_begin = (s0 + cpw - 1) / cpw, w_end = (s1 + cpw - 1) / cpw;
    for (size_t w = w_begin + threadIdx.x / D; w < w_end; w += blockDim.x / D) emit(d, s0, w);
    return;
  }
  const int nwr_max = (nt + cpw - 1) / cpw + 1;  // owned words per run are at most this
  for (int i = threadIdx.x; i < D * nwr_max; i += blockDim.x) {
    const int d = i % D, j = i / D;
    const size_t s0 = ((size_t)bh * D + d) * (size_t)T_ + t0, s1 = s0 + nt;
    const size_t w_begin = (s0 + cpw - 1) / cpw, w_end = (s1 + cpw - 1) / cpw;
    const size_t w = w_begin + j;
    if (w < w_end) emit(d, s0, w);
  }
}

// ---- Values -----------------------------------------------------------------------------
// x: [rows][D] with rows = B*H*T token slots; groups along channels (partial last group).
template <typename T, int BITS>
__global__ void __launch_bounds__(kQThreads) quantize_value_kernel(const T* __restrict__ x, size_t rows,
                                                                   int D, int bits_rt, int gs, int R, int vec,
                                                                   uint32_t* __restrict__ words,
                                                                   uint32_t* __restrict__ meta) {
  constexpr int bits = BITS;
  (void)bits_rt;
  extern __shared__ float smem[];
  const int gpt = (D + gs - 1) / gs;
  const int Dp = D + 1;                                                // padded row stride
  float* xs = smem;                                                    // [R][Dp]
  uint32_t* ms = reinterpret_cast<uint32_t*>(xs + (size_t)R * Dp);     // [R][gpt]
  const size_t r0 = (size_t)blockIdx.x * R;
  const int nr = (int)min((size_t)R, rows - r0);
  const int q_max = q_max_for_bits(bits);
  const T* src = x + r0 * D;
  if (vec) {  // D % N == 0 and a 16-byte aligned input (host-checked)
    const int vpr = D / Vec<T>::N;  // vectors per row
    for (int i = threadIdx.x; i < nr * vpr; i += blockDim.x) {
      const int rr = i / vpr, c0 = (i - rr * vpr) * Vec<T>::N;
      float v[Vec<T>::N];
      Vec<T>::load(src + (size_t)rr * D + c0, v);
#pragma unroll
      for (int e = 0; e < Vec<T>::N; ++e) xs[rr * Dp + c0 + e] = v[e];
    }
  } else {
    for (int i = threadIdx.x; i < nr * D; i += blockDim.x) xs[(i / D) * Dp + i % D] = gload(src, i);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nr * gpt; i += blockDim.x) {
    const int rr = i / gpt, g = i % gpt;
    const int d0 = g * gs, d1 = min(d0 + gs, D);
    float mn = xs[rr * Dp + d0], mx = mn;
    for (int d = d0 + 1; d < d1; ++d) {
      const float v = xs[rr * Dp + d];
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
    const uint32_t m = make_meta(mn, mx, q_max);
    ms[i] = m;
    meta[(r0 + rr) * gpt + g] = m;
  }
  __syncthreads();
  const int cpw = codes_per_word(bits);
  const size_t n_total = rows * (size_t)D;
  const size_t s0 = r0 * D, s1 = s0 + (size_t)nr * D;
  const size_t w_begin = (s0 + cpw - 1) / cpw, w_end = (s1 + cpw - 1) / cpw;
  for (size_t w = w_begin + threadIdx.x; w < w_end; w += blockDim.x) {
    uint32_t word = 0;
    const size_t p0 = w * cpw;
    // row / channel / group / stream-index-mod-11 of the first code, then stepped per code
    const int off = (int)(p0 - s0);
    int rr = off / D, d = off - rr * D;
    int g = d / gs, gend = min((g + 1) * gs, D);
    int r11 = bits == 3 ? (int)(p0 % 11u) : 0;
    uint32_t m = rr < nr ? ms[rr * gpt + g] : 0u;
    float sc = meta_scale(m), mnv = meta_min(m), rc = rcp_approx(sc);
    float ws = 0.f, rcw = 0.f;  // Mixed3 narrow slots: wide scale and its reciprocal
    if (bits == 3) {
      ws = wide_scale(sc);
      rcw = rcp_approx(ws);
    }
    size_t cached = ~(size_t)0;
    float sc2 = 0.f, mn2 = 0.f;
    for (int k = 0; k < cpw; ++k) {
      const size_t p = p0 + k;
      if (p >= n_total) break;
      const bool nar = bits == 3 && r11 == 10;
      uint32_t code;
      if (p < s1) {
        code = encode_fast(xs[rr * Dp + d], sc, mnv, nar ? ws : sc, nar ? rcw : rc, nar ? 3 : q_max, bits, nar);
      } else {  // codes of the next span (only at span ends): group meta once per group
        const size_t row = p / D;
        const int dd = (int)(p % D);
        const int d0 = (dd / gs) * gs, d1 = min(d0 + gs, D);
        const size_t grp = row * (size_t)gpt + (size_t)(dd / gs);
        if (grp != cached) {
          float mn = gload(x, row * D + d0), mx = mn;
          for (int e = d0 + 1; e < d1; ++e) {
            const float v = gload(x, row * D + e);
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
          }
          const uint32_t m2 = make_meta(mn, mx, q_max);
          sc2 = meta_scale(m2);
          mn2 = meta_min(m2);
          cached = grp;
        }
        code = encode(gload(x, p), sc2, mn2, bits, nar);
      }
      word |= code << field_shift(bits, (uint32_t)k);
      if (++r11 == 11) r11 = 0;
      if (++d == gend) {  // next channel group (or next row)
        if (d == D) {
          d = 0;
          ++rr;
        }
        g = d / gs;
        gend = min((g + 1) * gs, D);
        if (rr < nr) {
          m = ms[rr * gpt + g];
          sc = meta_scale(m);
          mnv = meta_min(m);
          rc = rcp_approx(sc);
          if (bits == 3) {
            ws = wide_scale(sc);
            rcw = rcp_approx(ws);
          }
        }
      }
    }
    words[w] = word;
  }
}

// ---- Values, uniform 1/2/4-bit words inside whole groups --------------------------------
// When D % gs == 0 and a word's codes (32 / b channels) never leave their group, every word
// is independent: one thread per output word loads its 32/b inputs (16-byte vectors,
// consecutive threads -> consecutive bytes), the L = gs * b / 32 threads of a group reduce
// min/max with L-lane butterflies, and the word is encoded with the group's meta in
// registers. No shared memory, no run bookkeeping. The reference's sequential min/max
// (mn = v < mn ? v : mn from the first element, quant.hpp:93-98 callers) is reproduced
// exactly: lanes fold their values skipping NaN, segments combine in order keeping the
// earlier of equal values, and a NaN first element makes the result NaN.
// (fold_min / fold_max: common.cuh)

__host__ __device__ constexpr int value_words_per_thread(int bits) { return bits == 4 ? 2 : 1; }

template <typename T, int N>
__device__ __forceinline__ void load_n(const T* p, float (&o)[N]) {
#pragma unroll
  for (int i = 0; i < N; i += Vec<T>::N) Vec<T>::load(p + i, o + i);
}

// words of one slot: v = the word's inputs (zeros for idle lanes), w = its index
template <typename T, int BITS>
__device__ __forceinline__ void value_word(const float (&v)[32 / BITS], bool ok, size_t w, int lane, int L,
                                           uint32_t* __restrict__ words, uint32_t* __restrict__ meta) {
  constexpr int CPW = 32 / BITS;
  // fminf/fmaxf skip NaN like the fold; they differ from it only in the sign of a zero
  // extremum (the fold keeps the first of -0 / +0), so groups whose min or max is zero redo
  // the ordered fold
  float mn = v[0], mx = v[0];
#pragma unroll
  for (int i = 1; i < CPW; ++i) {
    mn = fminf(mn, v[i]);
    mx = fmaxf(mx, v[i]);
  }
  for (int o = 1; o < L; o <<= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (__any_sync(0xffffffffu, mn == 0.f || mx == 0.f)) {  // (every group of the warp redoes:
    mn = NAN;                                               //  same values where no zero)
    mx = NAN;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      mn = fold_min(mn, v[i]);
      mx = fold_max(mx, v[i]);
    }
    for (int o = 1; o < L; o <<= 1) {
      const float omn = __shfl_xor_sync(0xffffffffu, mn, o), omx = __shfl_xor_sync(0xffffffffu, mx, o);
      const bool hi = lane & o;  // the other lane holds the earlier segment
      const float fmn = hi ? fold_min(omn, mn) : fold_min(mn, omn);
      const float fmx = hi ? fold_max(omx, mx) : fold_max(mx, omx);
      mn = fmn;
      mx = fmx;
    }
  }
  const int lead = lane & ~(L - 1);
  if (__shfl_sync(0xffffffffu, isnan(v[0]) ? 1 : 0, lead)) mn = mx = NAN;  // NaN first element
  constexpr int q_max = BITS == 1 ? 1 : BITS == 2 ? 3 : 15;
  const uint32_t m = make_meta(mn, mx, q_max);
  if (!ok) return;  // (after the warp-wide shuffles)
  if (lane == lead) meta[w / L] = m;
  const float sc = meta_scale(m), mnv = meta_min(m), rc = rcp_approx(sc);
  const uint32_t word = encode_word<BITS, CPW, !std::is_same<T, __half>::value>(v, sc, mnv, q_max);
  words[w] = word;
}


// P words per thread (4-bit: two, so a thread keeps 32 bytes of loads in flight like the
// 2-bit words): slot p of the grid covers words [p S, (p + 1) S), S = threads in the grid (a
// multiple of 32, so every group stays inside one warp); all loads issue before the folds
template <typename T, int BITS>
__global__ void __launch_bounds__(kQThreads) quantize_value_words_kernel(const T* __restrict__ x, size_t nw, int L,
                                                                         uint32_t* __restrict__ words,
                                                                         uint32_t* __restrict__ meta) {
  constexpr int CPW = 32 / BITS;
  constexpr int P = value_words_per_thread(BITS);
  static_assert(CPW % Vec<T>::N == 0, "word = whole input vectors");
  const size_t S = (size_t)gridDim.x * blockDim.x;
  const size_t w0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  float v[P][CPW];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const size_t w = w0 + p * S;
    if (w < nw) load_n<T, CPW>(x + w * CPW, v[p]);  // groups are whole L-lane blocks: idle
    else {                                             // lanes form whole blocks
#pragma unroll
      for (int i = 0; i < CPW; ++i) v[p][i] = 0.f;
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) value_word<T, BITS>(v[p], w0 + p * S < nw, w0 + p * S, lane, L, words, meta);
}

// ---- Values, Mixed3 (3-bit), D % gs == 0 and gs % 32 == 0 ------------------------------
// A chunk of 11*gs stream elements holds exactly gs Mixed3 words (11 codes each) and 11
// groups, both aligned. One warp per chunk: the chunk is staged in shared memory (16-byte
// loads), lanes 0..10 fold one group each in stream order (the reference's sequential
// min/max, exactly), and every lane emits gs/32 words; a lane's 11 codes sit at stride 11
// in shared memory (odd: conflict-free). Slot 10 of every word is the narrow slot.
constexpr int kM3Warps = 8;
// gs 32: a warp takes two 11-group chunks (22 lanes make the metas at once, 64 words per warp)
__host__ __device__ constexpr int m3_groups_per_chunk(int gs) { return gs == 32 ? 22 : 11; }
__host__ __device__ constexpr int m3_warp_floats(int gs) {  // chunk + 6 per group, 16-byte aligned
  return (m3_groups_per_chunk(gs) * (gs + 6) + 3) / 4 * 4;
}

template <typename T, int GS>
__global__ void __launch_bounds__(kM3Warps * 32) quantize_value_m3_kernel(const T* __restrict__ x, size_t n,
                                                                         uint32_t* __restrict__ words,
                                                                         uint32_t* __restrict__ meta) {
  constexpr int gs = GS;
  extern __shared__ __align__(16) float m3s[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NG = m3_groups_per_chunk(gs);  // groups per chunk (gs 32: two 11-group chunks)
  constexpr int CE = NG * gs;                    // chunk elements
  constexpr int WPC = CE / 11;                   // words per chunk
  float* xs = m3s + (size_t)warp * m3_warp_floats(gs);
  float* gm = xs + CE;  // [NG] scale, [NG] min, [NG] rcp(scale), [NG] rcp(wide scale)
  float* gf = gm + 4 * NG;  // [NG][2] (fminf, fmaxf) folded from the registers of the staging loads
  const size_t chunk = (size_t)blockIdx.x * kM3Warps + warp;
  const size_t e0 = chunk * CE;
  if (e0 >= n) return;
  const int ne = (int)min((size_t)CE, n - e0);  // a multiple of gs (n % gs == 0)
  // stage (fp32 in shared memory)
  const bool full = ne == CE && (reinterpret_cast<uintptr_t>(x + e0) & 15) == 0;
  if (full) {
    // every 16-byte load of the chunk in flight before the first store (one DRAM latency)
    constexpr int NV = CE / Vec<T>::N, PER = (NV + 31) / 32;
    uint4 r[PER];
    const uint4* s4 = reinterpret_cast<const uint4*>(x + e0);
#pragma unroll
    for (int u = 0; u < PER; ++u)
      r[u] = lane + 32 * u < NV ? __ldg(s4 + lane + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
    // group min / max straight from the loaded vectors: a group is L = gs / N consecutive
    // vectors, i.e. L adjacent lanes of one load round (32 is a multiple of L)
    constexpr int L = gs / Vec<T>::N;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = lane + 32 * u;
      float v[Vec<T>::N];
      Vec<T>::unpack(r[u], v);
      if (i < NV) {
#pragma unroll
        for (int k = 0; k < Vec<T>::N; ++k) xs[i * Vec<T>::N + k] = v[k];
      }
      float mn = v[0], mx = v[0];
#pragma unroll
      for (int k = 1; k < Vec<T>::N; ++k) {
        mn = fminf(mn, v[k]);
        mx = fmaxf(mx, v[k]);
      }
#pragma unroll
      for (int o = 1; o < L; o <<= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (i < NV && (lane & (L - 1)) == 0) {
        gf[2 * (i / L)] = mn;
        gf[2 * (i / L) + 1] = mx;
      }
    }
  } else {
    for (int i = lane; i < ne; i += 32) xs[i] = ld_f(x + e0 + i);
  }
  __syncwarp();
  const int ng = ne / gs;
  if (lane < ng) {
    // fminf / fmaxf skip NaN like the ordered fold and differ from it only in the sign of a
    // zero extremum and for a NaN first element: those groups redo the fold (rare)
    float mn, mx;
    if (full) {
      mn = gf[2 * lane];
      mx = gf[2 * lane + 1];
    } else {
      const float4* g4 = reinterpret_cast<const float4*>(xs + lane * gs);
      mn = xs[lane * gs];
      mx = mn;
#pragma unroll 4
      for (int j = 0; j < gs / 4; ++j) {
        const float4 q = g4[j];
        mn = fminf(mn, fminf(fminf(q.x, q.y), fminf(q.z, q.w)));
        mx = fmaxf(mx, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
      }
    }
    if (mn == 0.f || mx == 0.f || isnan(xs[lane * gs])) {
      const float* g = xs + lane * gs;
      mn = mx = g[0];
      for (int j = 1; j < gs; ++j) {
        const float v = g[j];
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
      }
    }
    const uint32_t m = make_meta(mn, mx, 7);
    meta[chunk * NG + lane] = m;
    const float sc = meta_scale(m);
    gm[lane] = sc;
    gm[NG + lane] = meta_min(m);
    gm[2 * NG + lane] = rcp_approx(sc);
    gm[3 * NG + lane] = rcp_approx(wide_scale(sc));
  }
  __syncwarp();
  const size_t nw = (n + 10) / 11;
#pragma unroll
  for (int i = 0; i < WPC / 32; ++i) {
    const int wl = lane + 32 * i;
    const size_t w = chunk * WPC + wl;
    if (w >= nw) break;
    uint32_t word = 0;
    if (11 * wl + 11 <= ne) {  // every chunk but the stream's last
      // a word spans at most two groups: j0 for its first codes, j0 + 1 after the boundary
      const int j0 = (11 * wl) / gs, kb = (j0 + 1) * gs - 11 * wl;  // first code of group j0 + 1
      const int j1 = kb < 11 ? j0 + 1 : j0;
      float xv[11];
#pragma unroll
      for (int k = 0; k < 11; ++k) xv[k] = xs[11 * wl + k];
      word = encode_m3_word<!std::is_same<T, __half>::value>(xv, kb, gm[j0], gm[NG + j0], gm[j1], gm[NG + j1]);
    } else {
#pragma unroll
      for (int k = 0; k < 11; ++k) {
        const int e = 11 * wl + k;
        if (e < ne) {
          const int j = e / gs;
          const float sc = gm[j], mnv = gm[NG + j];
          const bool nar = k == 10;
          const uint32_t code = encode_fast(xs[e], sc, mnv, nar ? wide_scale(sc) : sc, gm[(nar ? 3 : 2) * NG + j],
                                            nar ? 3 : 7, 3, nar);
          word |= code << (nar ? 30u : 3u * k);
        }
      }
    }
    words[w] = word;
  }
}

// ---- dequantize (QuantizedGroups::value_at for every element) ----------------------------
__global__ void dequantize_kernel(int grouping, const uint32_t* __restrict__ words,
                                  const uint32_t* __restrict__ meta, int H, int T_, int D, int bits,
                                  int gs, size_t n, float* __restrict__ out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    const size_t rowi = e / D;  // (bh, t)
    const int t = (int)(rowi % T_);
    const size_t bh = rowi / T_;
    size_t si, mi;
    if (grouping == 0) {
      const size_t c = bh * D + d;
      si = c * T_ + t;
      mi = c * (size_t)(T_ / gs) + t / gs;
    } else {
      si = rowi * D + d;
      mi = rowi * (size_t)((D + gs - 1) / gs) + d / gs;
    }
    const int cpw = codes_per_word(bits);
    const uint32_t pos = (uint32_t)(si % cpw);
    const uint32_t code = (words[si / cpw] >> field_shift(bits, pos)) & field_mask(bits, pos);
    const uint32_t m = meta[mi];
    out[e] = decode(code, meta_scale(m), meta_min(m), is_narrow(bits, si));
  }
}

// ---- pack / unpack (PackedWriter::push, PackedBuffer::get) -------------------------------
__global__ void pack_kernel(const uint32_t* __restrict__ codes, size_t n, int bits,
                            uint32_t* __restrict__ words, unsigned long long* bad) {
  const int cpw = codes_per_word(bits);
  const size_t nw = words_for(n, bits);
  for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < nw; w += (size_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
    for (int k = 0; k < cpw; ++k) {
      const size_t i = w * cpw + k;
      if (i >= n) break;
      const uint32_t c = codes[i];
      if (c > field_mask(bits, (uint32_t)k)) {
        atomicMin(bad, (unsigned long long)i);
        continue;
      }
      word |= c << field_shift(bits, (uint32_t)k);
    }
    words[w] = word;
  }
}

__global__ void unpack_kernel(const uint32_t* __restrict__ words, size_t n, int bits,
                              uint32_t* __restrict__ codes) {
  const int cpw = codes_per_word(bits);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t pos = (uint32_t)(i % cpw);
    codes[i] = (words[i / cpw] >> field_shift(bits, pos)) & field_mask(bits, pos);
  }
}

int grid_for(size_t n, int threads) {
  const size_t b = (n + threads - 1) / threads;
  const size_t cap = (size_t)num_sms() * 16;
  return (int)std::max<size_t>(1, std::min(b, cap));
}

}  // namespace

void check_quant_args(int B, int H, int T, int D, int bits, int gs) {
  if (bits < 1 || bits > 4) invalid("unsupported bit width " + std::to_string(bits));
  if (gs <= 0) invalid("group_size must be positive");
  if (B < 0 || H < 0 || T < 0 || D < 0) invalid("tensor dimensions must be non-negative");
}

void quantize(kvmix_grouping grouping, const void* x, kvmix_dtype dt, int B, int H, int T, int D, int bits,
              int gs, uint32_t* words, uint16_t* meta, cudaStream_t st) {
  check_quant_args(B, H, T, D, bits, gs);
  if (grouping == KVMIX_PER_CHANNEL_KEY) {
    if (T % gs != 0) {
      invalid("key quantization needs T (" + std::to_string(T) + ") to be a multiple of group_size (" +
              std::to_string(gs) + ")");
    }
  } else if (grouping != KVMIX_PER_TOKEN_VALUE) {
    invalid("unknown grouping");
  }
  const size_t n = (size_t)B * H * T * D;
  if (n == 0) return;
  if (dt != KVMIX_F32 && dt != KVMIX_F16) invalid("unsupported dtype");
  auto* m32 = reinterpret_cast<uint32_t*>(meta);
  const int vec = (D % (dt == KVMIX_F16 ? 8 : 4) == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0) ? 1 : 0;
  const int max_smem = 96 * 1024;
  if (grouping == KVMIX_PER_CHANNEL_KEY) {
    // tile of k groups of gs tokens: aim for ~128 tokens, bounded by shared memory
    // uniform 1/2/4-bit words: 64-token tiles of 128 threads (more, smaller CTAs per SM, so
    // one CTA's fold / encode phases overlap other CTAs' tile loads); Mixed3 keeps 128-token
    // tiles (its next-group staging costs gs tokens per tile)
    // (KVMIX_QK_TOK / KVMIX_QK_THREADS: A/B overrides, read once)
    static const int env_tok = getenv("KVMIX_QK_TOK") ? std::max(8, atoi(getenv("KVMIX_QK_TOK"))) : 0;
    static const int env_thr = getenv("KVMIX_QK_THREADS") ? std::min(kQThreads, std::max(32, atoi(getenv("KVMIX_QK_THREADS")))) : 0;
    const int qk_tok = env_tok ? env_tok : (bits == 3 ? 128 : 64);
    const int qk_threads = env_thr ? env_thr : (bits == 3 ? kQThreads : 128);
    int k = std::max(1, qk_tok / gs);
    const size_t esz = dt == KVMIX_F16 ? 2 : 4;  // staged in the input type
    const int ext = (bits == 3 && gs >= 11) ? 1 : 0;  // + the next run's first group (kernel)
    auto smem_of = [&](int kk) {  // tile + group meta (+ the words of a uniform-bit tile)
      const size_t ow = bits == 3 ? 0 : (size_t)D * ((size_t)kk * gs / (32 / bits) + 1) * 4;
      return ((size_t)(kk + ext) * gs * D * esz + 15) / 16 * 16 + (size_t)D * (kk + ext) * 4 + ow;
    };
    while (k > 1 && smem_of(k) > (size_t)max_smem) --k;
    if (smem_of(k) > (size_t)227 * 1024) invalid("quantize: group_size * head_dim too large for one tile");
    const int n_tok = k * gs;
    const size_t smem = smem_of(k);
    dim3 grid((T + n_tok - 1) / n_tok, B * H);
    auto go = [&](auto kern, const auto* xp) {
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
      // the whole unified L1 as shared memory: as many staged tiles per SM as fit (the tile
      // loads of resident CTAs are what keeps HBM busy; L1 caching does not help here)
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
      kern<<<grid, qk_threads, smem, st>>>(xp, H, T, D, bits, gs, n_tok, vec, words, m32, n);
    };
    const float* xf = static_cast<const float*>(x);
    const __half* xh = static_cast<const __half*>(x);
    if (dt == KVMIX_F32) {
      if (bits == 1) go(quantize_key_kernel<float, 1, 0>, xf);
      else if (bits == 2) go(quantize_key_kernel<float, 2, 0>, xf);
      else if (bits == 3) go(quantize_key_kernel<float, 3, 0>, xf);
      else go(quantize_key_kernel<float, 4, 0>, xf);
    } else {
      // the common head_dims at compile time (fp16, 16-byte aligned rows: channel pairs)
#define KVB_QK_H(DD)                                                   \
      if (bits == 1) go(quantize_key_kernel<__half, 1, DD>, xh);       \
      else if (bits == 2) go(quantize_key_kernel<__half, 2, DD>, xh);  \
      else if (bits == 3) go(quantize_key_kernel<__half, 3, DD>, xh);  \
      else go(quantize_key_kernel<__half, 4, DD>, xh);
      if (vec && D == 128) { KVB_QK_H(128) }
      else if (vec && D == 64) { KVB_QK_H(64) }
      else { KVB_QK_H(0) }
#undef KVB_QK_H
    }
    after_launch("quantize_key_kernel");
  } else if (bits != 3 && vec && D % gs == 0 && gs % (32 / bits) == 0 && gs / (32 / bits) <= 32 &&
             ((gs / (32 / bits)) & (gs / (32 / bits) - 1)) == 0) {
    // whole-group words: one thread per word (the common KVmix shapes: gs 32/64/128)
    const int cpw = 32 / bits, L = gs / cpw;
    const size_t nw = n / cpw;
    const size_t per_block = (size_t)kQThreads * value_words_per_thread(bits);
    const unsigned grid = (unsigned)((nw + per_block - 1) / per_block);
    const float* xf = static_cast<const float*>(x);
    const __half* xh = static_cast<const __half*>(x);
#define KVB_QVW(TT, XP)                                                                             \
    if (bits == 1) quantize_value_words_kernel<TT, 1><<<grid, kQThreads, 0, st>>>(XP, nw, L, words, m32); \
    else if (bits == 2) quantize_value_words_kernel<TT, 2><<<grid, kQThreads, 0, st>>>(XP, nw, L, words, m32); \
    else quantize_value_words_kernel<TT, 4><<<grid, kQThreads, 0, st>>>(XP, nw, L, words, m32);
    if (dt == KVMIX_F32) {
      KVB_QVW(float, xf)
    } else {
      KVB_QVW(__half, xh)
    }
#undef KVB_QVW
    after_launch("quantize_value_words_kernel");
  } else if (bits == 3 && D % gs == 0 && (gs == 32 || gs == 64 || gs == 128)) {
    // Mixed3 chunks of 11 * gs elements, one warp each
    const size_t ce = (size_t)m3_groups_per_chunk(gs) * gs;
    const size_t chunks = (n + ce - 1) / ce;
    const unsigned grid = (unsigned)((chunks + kM3Warps - 1) / kM3Warps);
    const size_t smem = (size_t)kM3Warps * m3_warp_floats(gs) * 4;
    auto go = [&](auto kern, const auto* xp) {
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
      // the whole unified L1 as shared memory: as many staged tiles per SM as fit (the tile
      // loads of resident CTAs are what keeps HBM busy; L1 caching does not help here)
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
      kern<<<grid, kM3Warps * 32, smem, st>>>(xp, n, words, m32);
    };
    const float* xf = static_cast<const float*>(x);
    const __half* xh = static_cast<const __half*>(x);
    if (dt == KVMIX_F32) {
      if (gs == 32) go(quantize_value_m3_kernel<float, 32>, xf);
      else if (gs == 64) go(quantize_value_m3_kernel<float, 64>, xf);
      else go(quantize_value_m3_kernel<float, 128>, xf);
    } else {
      if (gs == 32) go(quantize_value_m3_kernel<__half, 32>, xh);
      else if (gs == 64) go(quantize_value_m3_kernel<__half, 64>, xh);
      else go(quantize_value_m3_kernel<__half, 128>, xh);
    }
    after_launch("quantize_value_m3_kernel");
  } else {
    const int gpt = (D + gs - 1) / gs;
    int R = std::max(1, 8192 / std::max(D, 1));
    auto smem_of = [&](int r) { return (size_t)r * (D + 1) * 4 + (size_t)r * gpt * 4; };
    while (R > 1 && smem_of(R) > (size_t)max_smem) --R;
    if (smem_of(R) > (size_t)227 * 1024) invalid("quantize: head_dim too large for one tile");
    const size_t rows = (size_t)B * H * T;
    const size_t smem = smem_of(R);
    const unsigned grid = (unsigned)((rows + R - 1) / R);
    auto go = [&](auto kern, const auto* xp) {
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
      // the whole unified L1 as shared memory: as many staged tiles per SM as fit (the tile
      // loads of resident CTAs are what keeps HBM busy; L1 caching does not help here)
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
      kern<<<grid, kQThreads, smem, st>>>(xp, rows, D, bits, gs, R, vec, words, m32);
    };
    const float* xf = static_cast<const float*>(x);
    const __half* xh = static_cast<const __half*>(x);
    if (dt == KVMIX_F32) {
      if (bits == 1) go(quantize_value_kernel<float, 1>, xf);
      else if (bits == 2) go(quantize_value_kernel<float, 2>, xf);
      else if (bits == 3) go(quantize_value_kernel<float, 3>, xf);
      else go(quantize_value_kernel<float, 4>, xf);
    } else {
      if (bits == 1) go(quantize_value_kernel<__half, 1>, xh);
      else if (bits == 2) go(quantize_value_kernel<__half, 2>, xh);
      else if (bits == 3) go(quantize_value_kernel<__half, 3>, xh);
      else go(quantize_value_kernel<__half, 4>, xh);
    }
    after_launch("quantize_value_kernel");
  }
}

void dequantize(kvmix_grouping grouping, const uint32_t* words, const uint16_t* meta, int B, int H, int T,
                int D, int bits, int gs, float* out, cudaStream_t st) {
  check_quant_args(B, H, T, D, bits, gs);
  if (grouping == KVMIX_PER_CHANNEL_KEY && T % gs != 0) invalid("key tensor needs T % group_size == 0");
  const size_t n = (size_t)B * H * T * D;
  if (n == 0) return;
  dequantize_kernel<<<grid_for(n, 256), 256, 0, st>>>((int)grouping, words,
                                                       reinterpret_cast<const uint32_t*>(meta), H, T, D,
                                                       bits, gs, n, out);
  after_launch("dequantize_kernel");
}

void pack(const uint32_t* codes, size_t n, int bits, uint32_t* words, cudaStream_t st) {
  if (bits != 1 && bits != 2 && bits != 3 && bits != 4) {
    invalid("feat_per_word: bits must be 1, 2 or 4, got " + std::to_string(bits));
  }
  if (n == 0) return;
  unsigned long long* bad = nullptr;
  check_cuda(cudaMallocAsync(&bad, sizeof(unsigned long long), st), "cudaMallocAsync");
  check_cuda(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st), "memset");
  const size_t nw = words_for(n, bits);
  pack_kernel<<<grid_for(nw, 256), 256, 0, st>>>(codes, n, bits, words, bad);
  after_launch("pack_kernel");
  unsigned long long first = 0;
  check_cuda(cudaMemcpyAsync(&first, bad, sizeof(first), cudaMemcpyDeviceToHost, st), "memcpy");
  check_cuda(cudaFreeAsync(bad, st), "cudaFreeAsync");
  check_cuda(cudaStreamSynchronize(st), "sync");
  if (first != ~0ull) {
    // same wording as PackedWriter::push (bitpack.cpp:26-41)
    uint32_t c = 0;
    check_cuda(cudaMemcpy(&c, codes + first, 4, cudaMemcpyDeviceToHost), "memcpy");
    if (bits == 3) {
      const size_t pos = first % 11;
      invalid("pack_mixed3: code " + std::to_string(c) + " in block " + std::to_string(first / 11) +
              " at intra-block index " + std::to_string(pos) + " exceeds " + std::to_string(pos == 10 ? 3 : 7));
    }
    invalid("pack_uniform: code " + std::to_string(c) + " at index " + std::to_string(first) + " exceeds " +
            std::to_string((1u << bits) - 1u) + " for " + std::to_string(bits) + "-bit fields");
  }
}

void unpack(const uint32_t* words, size_t n, int bits, uint32_t* codes, cudaStream_t st) {
  if (bits != 1 && bits != 2 && bits != 3 && bits != 4) invalid("unsupported bit width");
  if (n == 0) return;
  unpack_kernel<<<grid_for(n, 256), 256, 0, st>>>(words, n, bits, codes);
  after_launch("unpack_kernel");
}

}  // namespace kvb
