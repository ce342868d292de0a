/*
 * kvmix_oracle.c -- CPU restatement of the KVmix hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity checker for the B200 kernels. It is NOT part of the
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product path (paper_2506_08018_b200)
 * never links or calls it.
 *
 * Every function restates one reference function; the citation is the file:line
 * under /root/reference/proj it follows. Parity of this restatement is pinned
 * (tests/test_oracle.py) against
 *   (1) the reference's own known-answer tests (words 0xE4/0xFFFFFFFF, KVQG
 *       golden bytes, binary16 spot values, rpc_target values, formula cases), and
 *   (2) the reference library itself compiled from its sources into
 *       oracle/_ref/libkvmix_ref.so (oracle/Makefile), via committed golden
 *       fixtures in tests/golden/ (tests/golden/make_golden.py).
 *
 * Build flags matter: -O2 -ffp-contract=off, no -ffast-math, no -march=native.
 * The reference dequantize is "code * scale + min" as two rounded fp32 ops
 * (SURVEY.md 7.2 #2); contraction to FMA would change its last bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KO_OK 0
#define KO_INVALID 1
#define KO_OUT_OF_RANGE 2

/* ---- binary16 codec: include/kvmix/half.hpp:15-45 (encode), :47-68 (decode) ---- */
uint16_t ko_half_from_float(float f) {
  uint32_t bits;
  memcpy(&bits, &f, 4);
  const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
  const int32_t fexp = (int32_t)((bits >> 23) & 0xffu);
  const uint32_t mant = bits & 0x007fffffu;
  if (fexp == 0xff) return (uint16_t)(sign | 0x7c00u | (mant ? 0x0200u : 0u));
  const int32_t e = fexp - 127;
  if (e > 15) return (uint16_t)(sign | 0x7c00u);
  if (e >= -14) {
    /* round the 23-bit mantissa to 10 bits, nearest-even; a carry may bump the exponent */
    const uint32_t rounded = (mant + 0x00000fffu + ((mant >> 13) & 1u)) >> 13;
    const uint32_t h = ((uint32_t)(e + 15) << 10) + rounded;
    if (h >= 0x7c00u) return (uint16_t)(sign | 0x7c00u);
    return (uint16_t)(sign | h);
  }
  if (e < -25) return sign;
  /* subnormal result: integer multiple of 2^-24 */
  const uint32_t full = mant | 0x00800000u;
  const uint32_t sh = (uint32_t)(-e - 1);
  const uint32_t half_bit = 1u << (sh - 1);
  uint32_t q = full >> sh;
  const uint32_t rem = full & ((half_bit << 1) - 1u);
  if (rem > half_bit || (rem == half_bit && (q & 1u))) ++q;
  return (uint16_t)(sign | q);
}

float ko_float_from_half(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t ex = (h >> 10) & 0x1fu;
  uint32_t mant = h & 0x3ffu;
  uint32_t bits;
  if (ex == 0x1f) {
    bits = sign | 0x7f800000u | (mant << 13);
  } else if (ex != 0) {
    bits = sign | ((ex + 112u) << 23) | (mant << 13);
  } else if (mant != 0) {
    uint32_t e = 0;
    while (!(mant & 0x400u)) {
      mant <<= 1;
      ++e;
    }
    mant &= 0x3ffu;
    bits = sign | ((113u - e) << 23) | (mant << 13);
  } else {
    bits = sign;
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

/* half.hpp:71 */
float ko_round_through_half(float x) { return ko_float_from_half(ko_half_from_float(x)); }

/* ---- scalar helpers: src/quant.cpp:8-21, bitpack.hpp:31-33, quant.hpp:53, bitpack.cpp:8-14 ---- */
int ko_q_max_for_bits(int bits) {
  switch (bits) {
    case 1: return 1;
    case 2: return 3;
    case 3: return 7;
    case 4: return 15;
    default: return -1;
  }
}

int ko_feat_per_word(int bits) { return (bits == 1 || bits == 2 || bits == 4) ? 32 / bits : -1; }

static float mixed3_wide_scale(float s) { return s * (7.0f / 3.0f); }

/* ---- meta: quant.hpp:93-98 (make_group_meta) ---- */
void ko_make_meta(float mn, float mx, int q_max, float* scale, float* minv) {
  *minv = ko_round_through_half(mn);
  *scale = ko_round_through_half((mx - mn) / (float)q_max);
}

/* src/quant.cpp:23-32 (compute_meta) */
int ko_compute_meta(const float* g, size_t n, int q_max, float* scale, float* minv) {
  if (n == 0 || q_max < 1) return KO_INVALID;
  float mn = g[0], mx = g[0];
  for (size_t i = 0; i < n; ++i) {
    mn = g[i] < mn ? g[i] : mn;
    mx = g[i] > mx ? g[i] : mx;
  }
  ko_make_meta(mn, mx, q_max, scale, minv);
  return KO_OK;
}

/* ---- element codec: src/quant.cpp:36-47 (encode_element), :49-53 (decode_code) ---- */
uint32_t ko_encode(float x, float scale, float minv, int bits, uint64_t si) {
  long q_max = ko_q_max_for_bits(bits);
  if (bits == 3 && si % 11 == 10) {
    scale = mixed3_wide_scale(scale);
    q_max = 3;
  }
  if (scale == 0.0f) return 0;
  long q = lroundf((x - minv) / scale);
  q = q < 0 ? 0 : (q > q_max ? q_max : q);
  return (uint32_t)q;
}

float ko_decode(uint32_t code, float scale, float minv, int bits, uint64_t si) {
  const int narrow = bits == 3 && si % 11 == 10;
  const float s = narrow ? mixed3_wide_scale(scale) : scale;
  return (float)code * s + minv;
}

/* src/quant.cpp:57-67 */
void ko_quantize_group(const float* g, size_t n, float scale, float minv, int q_max, uint32_t* codes) {
  for (size_t i = 0; i < n; ++i) {
    if (scale == 0.0f) { codes[i] = 0; continue; }
    long q = lroundf((g[i] - minv) / scale);
    q = q < 0 ? 0 : (q > q_max ? q_max : q);
    codes[i] = (uint32_t)q;
  }
}

/* src/quant.cpp:69-75 */
void ko_dequantize_group(const uint32_t* codes, size_t n, float scale, float minv, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (float)codes[i] * scale + minv;
}

/* ---- bitpack: bitpack.hpp:10-24 layout, bitpack.cpp:23-46 push, :69-82 get ---- */
size_t ko_words_for(size_t n, int bits) {
  if (bits == 3) return (n + 10) / 11;
  return (n * (size_t)bits + 31) / 32;
}

/* Packs n codes. Returns KO_OK or KO_INVALID with *bad = offending index (bitpack.cpp:26-41). */
int ko_pack(const uint32_t* codes, size_t n, int bits, uint32_t* words, size_t* bad) {
  const size_t nw = ko_words_for(n, bits);
  memset(words, 0, nw * 4);
  for (size_t i = 0; i < n; ++i) {
    if (bits == 3) {
      const size_t pos = i % 11;
      const uint32_t qm = pos == 10 ? 3u : 7u;
      if (codes[i] > qm) { if (bad) *bad = i; return KO_INVALID; }
      words[i / 11] |= codes[i] << (pos == 10 ? 30u : 3u * (uint32_t)pos);
    } else {
      const uint32_t qm = (1u << bits) - 1u;
      const size_t fpw = 32u / (size_t)bits;
      if (codes[i] > qm) { if (bad) *bad = i; return KO_INVALID; }
      words[i / fpw] |= codes[i] << ((i % fpw) * (size_t)bits);
    }
  }
  return KO_OK;
}

uint32_t ko_get(const uint32_t* words, size_t idx, int bits) {
  if (bits == 3) {
    const size_t pos = idx % 11;
    const uint32_t w = words[idx / 11];
    return pos == 10 ? (w >> 30) & 3u : (w >> (3u * pos)) & 7u;
  }
  const size_t fpw = 32u / (size_t)bits;
  return (words[idx / fpw] >> ((idx % fpw) * (size_t)bits)) & ((1u << bits) - 1u);
}

/* ---- tensor quantizers ----
 * Keys:   quant.hpp:107-151 (quantize_key_stream) via quant.cpp:102-114.
 *         channel c=(b*H+h)*D+d, stream si=c*T+t, meta index c*(T/gs)+t/gs.
 * Values: quant.hpp:153-194 (quantize_value_stream) via quant.cpp:116-124.
 *         token slot tok=(b*H+h)*T+t, stream si=tok*D+d, meta tok*ceil(D/gs)+d/gs.
 * Input is the dense [B,H,T,D] fp32 tensor (tensor.hpp:24-27). `meta` receives
 * binary16 (scale, min) pairs exactly as the KVQG payload (quant.cpp:164-167). */
static int check_bits(int bits) { return bits >= 1 && bits <= 4; }

int ko_quantize_key(const float* x, int B, int H, int T, int D, int bits, int gs, uint32_t* words,
                    uint16_t* meta) {
  if (!check_bits(bits) || gs <= 0 || T % gs != 0) return KO_INVALID;
  const int q_max = ko_q_max_for_bits(bits);
  const size_t channels = (size_t)B * H * D;
  const int gpc = T / gs;
  float* ms = (float*)malloc(sizeof(float) * (channels * gpc + 1));
  float* mm = (float*)malloc(sizeof(float) * (channels * gpc + 1));
  for (size_t c = 0; c < channels; ++c) {
    const size_t bh = c / D, d = c % D;
    const float* base = x + bh * (size_t)T * D + d;
    for (int g = 0; g < gpc; ++g) {
      float mn = base[(size_t)g * gs * D], mx = mn;
      for (int j = 1; j < gs; ++j) {
        const float v = base[((size_t)g * gs + j) * D];
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
      }
      ko_make_meta(mn, mx, q_max, &ms[c * gpc + g], &mm[c * gpc + g]);
      meta[2 * (c * gpc + g)] = ko_half_from_float(ms[c * gpc + g]);
      meta[2 * (c * gpc + g) + 1] = ko_half_from_float(mm[c * gpc + g]);
    }
  }
  const size_t n = channels * (size_t)T;
  memset(words, 0, ko_words_for(n, bits) * 4);
  size_t si = 0;
  for (size_t c = 0; c < channels; ++c) {
    const size_t bh = c / D, d = c % D;
    for (int t = 0; t < T; ++t, ++si) {
      const size_t mi = c * gpc + t / gs;
      const uint32_t code = ko_encode(x[(bh * T + t) * D + d], ms[mi], mm[mi], bits, si);
      if (bits == 3) {
        const size_t pos = si % 11;
        words[si / 11] |= code << (pos == 10 ? 30u : 3u * (uint32_t)pos);
      } else {
        const size_t fpw = 32u / (size_t)bits;
        words[si / fpw] |= code << ((si % fpw) * (size_t)bits);
      }
    }
  }
  free(ms);
  free(mm);
  return KO_OK;
}

int ko_quantize_value(const float* x, int B, int H, int T, int D, int bits, int gs, uint32_t* words,
                      uint16_t* meta) {
  if (!check_bits(bits) || gs <= 0) return KO_INVALID;
  const int q_max = ko_q_max_for_bits(bits);
  const size_t tokens = (size_t)B * H * T;
  const int gpt = (D + gs - 1) / gs;
  const size_t n = tokens * (size_t)D;
  memset(words, 0, ko_words_for(n, bits) * 4);
  for (size_t tok = 0; tok < tokens; ++tok) {
    const float* row = x + tok * D;
    for (int g = 0; g < gpt; ++g) {
      const int d0 = g * gs, d1 = d0 + gs < D ? d0 + gs : D;
      float mn = row[d0], mx = mn;
      for (int d = d0 + 1; d < d1; ++d) {
        mn = row[d] < mn ? row[d] : mn;
        mx = row[d] > mx ? row[d] : mx;
      }
      float s, m;
      ko_make_meta(mn, mx, q_max, &s, &m);
      meta[2 * (tok * gpt + g)] = ko_half_from_float(s);
      meta[2 * (tok * gpt + g) + 1] = ko_half_from_float(m);
      for (int d = d0; d < d1; ++d) {
        const size_t si = tok * D + d;
        const uint32_t code = ko_encode(row[d], s, m, bits, si);
        if (bits == 3) {
          const size_t pos = si % 11;
          words[si / 11] |= code << (pos == 10 ? 30u : 3u * (uint32_t)pos);
        } else {
          const size_t fpw = 32u / (size_t)bits;
          words[si / fpw] |= code << ((si % fpw) * (size_t)bits);
        }
      }
    }
  }
  return KO_OK;
}

/* QuantizedGroups::value_at over a whole segment (quant.cpp:77-100): dense fp32 [B,H,T,D]. */
int ko_dequantize(const uint32_t* words, const uint16_t* meta, int grouping, int B, int H, int T,
                  int D, int bits, int gs, float* out) {
  if (!check_bits(bits) || gs <= 0) return KO_INVALID;
  const size_t bhn = (size_t)B * H;
  for (size_t bh = 0; bh < bhn; ++bh) {
    for (int t = 0; t < T; ++t) {
      for (int d = 0; d < D; ++d) {
        size_t si, mi;
        if (grouping == 0) {
          const size_t c = bh * D + d;
          si = c * T + t;
          mi = c * (size_t)(T / gs) + t / gs;
        } else {
          const size_t tok = bh * T + t;
          si = tok * D + d;
          mi = tok * (size_t)((D + gs - 1) / gs) + d / gs;
        }
        const float s = ko_float_from_half(meta[2 * mi]);
        const float m = ko_float_from_half(meta[2 * mi + 1]);
        out[(bh * T + t) * D + d] = ko_decode(ko_get(words, si, bits), s, m, bits, si);
      }
    }
  }
  return KO_OK;
}

/* ---- shrink rule: src/cache.cpp:30-34 (rpc_target), :65-79 (append), helpers.hpp:38-53 ---- */
int64_t ko_rpc_target(int64_t n, double r) { return (int64_t)floor(r * (double)n); }

/* One append of t tokens on one side. r is the config float promoted to double.
 * Returns the number of tokens aged out (Keys: whole groups only). */
int64_t ko_shrink(int64_t* tail, int64_t t, float r, int gs, int whole_groups) {
  *tail += t;
  const int64_t target = ko_rpc_target(*tail, (double)r);
  const int64_t excess = *tail - target;
  const int64_t aged = whole_groups ? excess / gs * gs : excess;
  if (aged > 0) {
    *tail -= aged;
    return aged;
  }
  return 0;
}

/* ---- attention on a dequantized snapshot ----
 * reference_attend, src/attention.cpp:168-211: scores in d order, * (1/sqrtf(D)),
 * double checksum, softmax_inplace (:83-94: max, expf, sum, * 1/sum), then P.V in j order.
 * q [B,H,t,D], keys/values [B,H,T,D]; out [B,H,t,D]. */
int ko_attend_f32(const float* q, const float* keys, const float* values, int B, int H, int tq,
                  int T, int D, float* out, double* checksum) {
  if (T < 1) return KO_INVALID;
  const float inv = 1.0f / sqrtf((float)D);
  float* srow = (float*)malloc(sizeof(float) * (size_t)T);
  double sum = 0.0;
  /* checksum is summed over the whole scores tensor before softmax, row-major */
  for (int b = 0; b < B; ++b)
    for (int h = 0; h < H; ++h)
      for (int i = 0; i < tq; ++i) {
        const float* qr = q + (((size_t)b * H + h) * tq + i) * D;
        const float* kb = keys + ((size_t)b * H + h) * (size_t)T * D;
        const float* vb = values + ((size_t)b * H + h) * (size_t)T * D;
        for (int j = 0; j < T; ++j) {
          float acc = 0.0f;
          for (int d = 0; d < D; ++d) acc += qr[d] * kb[(size_t)j * D + d];
          srow[j] = acc;
        }
        for (int j = 0; j < T; ++j) {
          srow[j] *= inv;
          sum += srow[j];
        }
        float mx = srow[0];
        for (int j = 0; j < T; ++j) mx = srow[j] > mx ? srow[j] : mx;
        float s = 0.0f;
        for (int j = 0; j < T; ++j) {
          srow[j] = expf(srow[j] - mx);
          s += srow[j];
        }
        const float is = 1.0f / s;
        for (int j = 0; j < T; ++j) srow[j] *= is;
        float* orow = out + (((size_t)b * H + h) * tq + i) * D;
        for (int d = 0; d < D; ++d) orow[d] = 0.0f;
        for (int j = 0; j < T; ++j)
          for (int d = 0; d < D; ++d) orow[d] += srow[j] * vb[(size_t)j * D + d];
      }
  free(srow);
  *checksum = sum;
  return KO_OK;
}

/* Same computation in double precision (the primary tolerance oracle). */
int ko_attend_f64(const float* q, const float* keys, const float* values, int B, int H, int tq,
                  int T, int D, double* out, double* checksum) {
  if (T < 1) return KO_INVALID;
  const double inv = 1.0 / sqrt((double)D);
  double* srow = (double*)malloc(sizeof(double) * (size_t)T);
  double sum = 0.0;
  for (int b = 0; b < B; ++b)
    for (int h = 0; h < H; ++h)
      for (int i = 0; i < tq; ++i) {
        const float* qr = q + (((size_t)b * H + h) * tq + i) * D;
        const float* kb = keys + ((size_t)b * H + h) * (size_t)T * D;
        const float* vb = values + ((size_t)b * H + h) * (size_t)T * D;
        double mx = -INFINITY;
        for (int j = 0; j < T; ++j) {
          double acc = 0.0;
          for (int d = 0; d < D; ++d) acc += (double)qr[d] * (double)kb[(size_t)j * D + d];
          srow[j] = acc * inv;
          sum += srow[j];
          mx = srow[j] > mx ? srow[j] : mx;
        }
        double s = 0.0;
        for (int j = 0; j < T; ++j) {
          srow[j] = exp(srow[j] - mx);
          s += srow[j];
        }
        double* orow = out + (((size_t)b * H + h) * tq + i) * D;
        for (int d = 0; d < D; ++d) orow[d] = 0.0;
        for (int j = 0; j < T; ++j)
          for (int d = 0; d < D; ++d) orow[d] += srow[j] / s * (double)vb[(size_t)j * D + d];
      }
  free(srow);
  *checksum = sum;
  return KO_OK;
}

/* ---- synthetic inputs: include/kvmix/rng.hpp:10-53 (splitmix64 + Box-Muller) ---- */
typedef struct {
  uint64_t state;
  int have_spare;
  double spare;
} ko_rng;

static uint64_t rng_next(ko_rng* r) {
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static double rng_double(ko_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_normal(ko_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_double(r);
  while (u1 <= 0.0) u1 = rng_double(r);
  const double u2 = rng_double(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

/* helpers.hpp:14-25 / harness.cpp:16-24: N(mu, sigma^2) rounded onto the binary16 grid.
 * Fills n values from a generator seeded with `seed` (fresh state). */
void ko_random_h16(uint64_t seed, size_t n, float sigma, float mu, float* out) {
  ko_rng r = {seed, 0, 0.0};
  for (size_t i = 0; i < n; ++i) out[i] = ko_round_through_half(mu + sigma * (float)rng_normal(&r));
}
