// cache.cu -- fused quantize-and-concatenate append (KVLayerCache::append, cache.cpp:45-117),
// bit-exact snapshot (cache.cpp:136-173) and reference-segment export/import.
//
// One append is ONE kernel launch in the common case (decode): CTAs are role-split into
//   * key age-out CTAs, one per (aged group of gs tokens, bh): min/max over the group per
//     channel, binary16 meta, encode with the segment's Mixed3 phase, then the group's
//     16-token tiles are assembled in shared memory and written with plain stores;
//   * value age-out CTAs, one per (16-token tile window, bh): per-token/per-channel-group
//     meta and codes; partial tiles are merged with atomicOr (fields of not-yet-aged
//     tokens are zero);
//   * tail CTAs copying the new tokens that stay in the full-precision window into the
//     ring buffer.
// The aged tokens are read straight from the old tail ring or from the new input, so the
// tail never has to be compacted (the reference erases from the front, cache.cpp:95).
// When the ring could wrap onto slots still being read (huge prefills), the tail copy is
// launched as a second kernel after the age-out kernel.
#include <algorithm>
#include <cmath>

#include "cache.cuh"

namespace kvb {

namespace {

constexpr int kAppendThreads = 128;

template <typename TT>
__device__ inline float round_to(float v);
template <>
__device__ inline float round_to<float>(float v) { return v; }
template <>
__device__ inline float round_to<__half>(float v) { return __half2float(__float2half_rn(v)); }

// Source of logical tail token j of one side for this append: old ring or new input.
template <typename TI, typename TT>
struct Src {
  const TT* tail;
  int64_t cap, start, L;
  const TI* in;  // [bh][t][D]
  int t;
  __device__ float at(int bh, int64_t j, int d, int D) const {
    if (j < L) return ld_f<TT>(tail + ((size_t)bh * cap + (size_t)((start + j) % cap)) * D + d);
    return round_to<TT>(ld_f<TI>(in + ((size_t)bh * t + (size_t)(j - L)) * D + d));
  }
};

// imma_element for a power-of-two channel count (D in {64, 128, 256}) with log2 arguments:
// shifts and masks instead of the generic divisions (the Key age-out assembles every field
// of two tiles per group; this keeps it a few instructions per field).
__device__ __forceinline__ void imma_element_p2(bool key, int ld, int b, int lc, int lane, int w, int f, int* i, int* d,
                                                int* shift) {
  const int C = 1 << lc, e = f >> lc, cls = f & (C - 1);
  const int g = lane >> 2, t = lane & 3;
  *shift = 8 * e + b * cls;
  if (key) {
    const int lnk = ld - 5;  // NK = D / 32
    const int q = ((w >> 1) << lc) + cls, rb = w & 1;
    *i = g + 8 * rb;
    *d = ((q & ((1 << lnk) - 1)) << 5) + ((q >> lnk) << 4) + 4 * t + e;
  } else {
    const int lnm = ld - 4;  // NM = D / 16
    const int q = (w << lc) + cls;
    *i = 4 * t + e;
    *d = ((q & ((1 << lnm) - 1)) << 4) + ((q >> lnm) << 3) + g;
  }
}

// Assemble one tile from codes[16][D] (u8, shared). For partial value tiles only rows in
// [i_lo, i_hi) contribute and words are OR-merged.
__device__ inline void emit_tile(bool key, int D, int bits, const uint8_t* codes, uint32_t* tile, bool atomic,
                                 int i_lo, int i_hi) {
  if (!key) bits = vstore_bits(bits);  // 3-bit Values: 4-bit fields
  const bool p2 = (D & (D - 1)) == 0;
  const int ld = 31 - __clz(D);
  if (bits != 3) {  // IMMA layout: 4 bytes x C classes per word
    const int wpl = plane_wpl(D, bits), cw = wpl < 4 ? wpl : 4;
    const int nf = 32 / bits;
    const int lc = bits == 1 ? 3 : bits == 2 ? 2 : 1;  // log2(8 / bits)
    for (int pw = threadIdx.x; pw < 32 * wpl; pw += blockDim.x) {
      const int chunk = pw / (32 * cw), within = pw % (32 * cw);
      const int lane = within / cw, w = chunk * cw + within % cw;
      uint32_t word = 0;
      for (int f = 0; f < nf; ++f) {
        int i, d, sh;
        if (p2) imma_element_p2(key, ld, bits, lc, lane, w, f, &i, &d, &sh);
        else imma_element(key, D, bits, lane, w, f, &i, &d, &sh);
        if (i < i_lo || i >= i_hi) continue;
        word |= (uint32_t)codes[i * D + d] << sh;
      }
      if (atomic) {
        if (word) atomicOr(tile + pw, word);
      } else {
        tile[pw] = word;
      }
    }
    return;
  }
  {  // 3-bit Keys: IMMA 2-bit plane of the low bits, then the 1-bit plane
    const int wpl2 = plane_wpl(D, 2), cw2 = wpl2 < 4 ? wpl2 : 4;
    for (int pw = threadIdx.x; pw < 32 * wpl2; pw += blockDim.x) {
      const int chunk = pw / (32 * cw2), within = pw % (32 * cw2);
      const int lane = within / cw2, w = chunk * cw2 + within % cw2;
      uint32_t word = 0;
      for (int f = 0; f < 16; ++f) {
        int i, d, sh;
        if (p2) imma_element_p2(true, ld, 2, 2, lane, w, f, &i, &d, &sh);
        else imma_element(true, D, 2, lane, w, f, &i, &d, &sh);
        if (i < i_lo || i >= i_hi) continue;
        word |= ((uint32_t)codes[i * D + d] & 3u) << sh;
      }
      if (atomic) {
        if (word) atomicOr(tile + pw, word);
      } else {
        tile[pw] = word;
      }
    }
    const int wpl1 = plane_wpl(D, 1), cw1 = wpl1 < 4 ? wpl1 : 4;
    uint32_t* t1 = tile + 32 * wpl2;
    for (int pw = threadIdx.x; pw < 32 * wpl1; pw += blockDim.x) {
      const int chunk = pw / (32 * cw1), within = pw % (32 * cw1);
      const int lane = within / cw1, w = chunk * cw1 + within % cw1;
      uint32_t word = 0;
      for (int f = 0; f < 32; ++f) {
        int i, d, sh;
        if (p2) {  // imma_key_hi_element with shifts (NK = D / 32 a power of two)
          const int lnk = ld - 5, e = f >> 3, z = 8 * w + (f & 7);
          const int q = z & ((2 << lnk) - 1), rb = z >> (lnk + 1);
          i = (lane >> 2) + 8 * rb;
          d = ((q & ((1 << lnk) - 1)) << 5) + ((q >> lnk) << 4) + 4 * (lane & 3) + e;
          sh = 8 * e + (f & 7);
        } else {
          imma_key_hi_element(D, lane, w, f, &i, &d, &sh);
        }
        if (i < i_lo || i >= i_hi) continue;
        word |= ((uint32_t)codes[i * D + d] >> 2) << sh;
      }
      if (atomic) {
        if (word) atomicOr(t1 + pw, word);
      } else {
        t1[pw] = word;
      }
    }
    return;
  }
}

struct AppendArgs {
  int H, D, gs, t;
  // keys
  int kbits, k_groups, k_blocks;
  int64_t k_q0, k_n;  // quantized count before, aged count
  uint32_t* k_tiles;
  uint32_t* k_meta;
  int2* k_info;
  SideView kv;  // addressing of the Key side (group records)
  // values
  int vbits, v_blocks, v_tile0;
  int v_warp;  // decode-sized age-out: one warp per (aged token, bh), lanes over channels
  int64_t v_q0, v_n;
  uint32_t* v_tiles;
  uint32_t* v_meta;
  int2* v_info;
  SideView vv;
  // tails: staying tokens of the input go to ring slots
  void* k_tail;
  void* v_tail;
  int64_t k_cap, k_start, k_L, v_cap, v_start, v_L;
  int64_t k_stay0, v_stay0;  // first input index that stays in each tail
  int tail_blocks;
  int BH;
  int phase;  // 0 = all roles, 1 = age-out only, 2 = tail only
};

template <typename TI, typename TT>
__global__ void __launch_bounds__(kAppendThreads) append_kernel(AppendArgs a, const TI* __restrict__ kin,
                                                                const TI* __restrict__ vin) {
  extern __shared__ uint8_t sm[];
  const int D = a.D, gs = a.gs;
  int blk = blockIdx.x;
  const int n_k_blocks = a.phase == 2 ? 0 : a.k_blocks;
  const int n_v_blocks = a.phase == 2 ? 0 : a.v_blocks;

  if (blk < n_k_blocks) {
    // ---- key age-out: one group of gs tokens for one bh --------------------------------
    const int bh = blk % a.BH, g = blk / a.BH;  // group index within this segment
    Src<TI, TT> src{static_cast<const TT*>(a.k_tail), a.k_cap, a.k_start, a.k_L, kin, a.t};
    const int Dl = a.kv.dl;
    uint8_t* codes = sm;  // [gs][Dl] (channels D..Dl-1 of the tile layout: zero codes)
    const int q_max = q_max_for_bits(a.kbits);
    const int64_t gglob = a.k_q0 / gs + g;
    float* xs = reinterpret_cast<float*>(sm + (size_t)gs * Dl);  // [gs][D] staged column values
    if (Dl != D) {
      for (int e = threadIdx.x; e < gs * (Dl - D); e += blockDim.x) codes[(e / (Dl - D)) * Dl + D + e % (Dl - D)] = 0;
    }
    const int64_t j0 = (int64_t)g * gs;
    // ring slot of logical token j0 (the group's tokens walk the ring incrementally)
    const int64_t slot0 = j0 < src.L ? (src.start + j0) % src.cap : 0;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      // stage the channel's gs values with the loads in flight together, then reduce
      int64_t slot = slot0;
#pragma unroll 8
      for (int jj = 0; jj < gs; ++jj) {
        const int64_t j = j0 + jj;
        float x;
        if (j < src.L) {
          x = ld_f<TT>(src.tail + ((size_t)bh * src.cap + (size_t)slot) * D + d);
          if (++slot == src.cap) slot = 0;
        } else {
          x = round_to<TT>(ld_f<TI>(src.in + ((size_t)bh * src.t + (size_t)(j - src.L)) * D + d));
        }
        xs[jj * D + d] = x;
      }
      float mn = xs[d], mx = mn;
      for (int jj = 1; jj < gs; ++jj) {
        const float x = xs[jj * D + d];
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
      }
      const uint32_t m = make_meta(mn, mx, q_max);
      a.k_meta[kmeta_index(a.kv, bh, gglob) + d] = m;
      const float sc = meta_scale(m), mnv = meta_min(m), rc = rcp_approx(sc);
      const float ws = wide_scale(sc), rcw = rcp_approx(ws);
      // reference stream index inside this segment [B,H,n,D]: (bh*D + d)*n + t_local
      const uint64_t sbase = ((uint64_t)a.kv.gbh(bh) * D + d) * (uint64_t)a.k_n + (uint64_t)j0;
      int r11 = (int)(sbase % 11u);
      for (int jj = 0; jj < gs; ++jj) {
        const float x = xs[jj * D + d];
        const bool nar = a.kbits == 3 && r11 == 10;
        codes[jj * Dl + d] = (uint8_t)encode_fast(x, sc, mnv, nar ? ws : sc, nar ? rcw : rc, nar ? 3 : q_max, a.kbits, nar);
        if (++r11 == 11) r11 = 0;
      }
    }
    if (bh == 0 && threadIdx.x == 0) a.k_info[gglob] = make_int2((int)a.k_n, g * gs);
    __syncthreads();
    const int64_t tile0 = (a.k_q0 + (int64_t)g * gs) / 16;
    for (int tt = 0; tt < gs / 16; ++tt) {
      uint32_t* tile = a.k_tiles + tile_index(a.kv, bh, tile0 + tt);
      emit_tile(true, Dl, a.kbits, codes + tt * 16 * Dl, tile, false, 0, 16);
    }
    return;
  }
  blk -= n_k_blocks;

  if (blk < n_v_blocks && a.v_warp) {
    // ---- value age-out, few tokens: one warp per (token, bh); lanes own D/32 channels,
    // channel-group min/max by shuffles over the group's lanes, codes OR-ed into the tile.
    constexpr int kW = kAppendThreads / 32;
    const int item = blk * kW + (int)(threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (item >= a.v_n * a.BH) return;
    const int bh = item % a.BH;
    const int64_t tl = item / a.BH;  // token index inside the segment
    const int64_t j = a.v_q0 + tl;   // global token index
    Src<TI, TT> src{static_cast<const TT*>(a.v_tail), a.v_cap, a.v_start, a.v_L, vin, a.t};
    const int LC = D / 32;           // 2 or 4 (host checks)
    const int q_max = q_max_for_bits(a.vbits);
    float x[4];
    for (int c = 0; c < LC; ++c) x[c] = src.at(bh, tl, lane * LC + c, D);
    const int glanes = min(gs, D) / LC;  // lanes per channel group (power of two)
    const uint32_t m = group_meta_warp(x, LC, glanes, lane, q_max);
    const int g0 = lane * LC / gs;
    if ((lane % glanes) == 0) a.v_meta[vmeta_at(a.vv, bh, j, g0)] = m;
    if (bh == 0 && lane == 0) a.v_info[j] = make_int2((int)a.v_n, (int)tl);
    const float sc = meta_scale(m), mnv = meta_min(m);
    uint32_t* tp = a.v_tiles + tile_index(a.vv, bh, j >> 4);
    for (int c = 0; c < LC; ++c) {
      const int d = lane * LC + c;
      const uint64_t si = ((uint64_t)a.vv.gbh(bh) * a.v_n + (uint64_t)tl) * D + d;
      tile_or(tp, false, a.vv.dl, a.vbits, (int)(j & 15), d, encode(x[c], sc, mnv, a.vbits, is_narrow(a.vbits, si)));
    }
    return;
  }
  if (blk < n_v_blocks) {
    // ---- value age-out: one 16-token tile window for one bh ---------------------------
    const int bh = blk % a.BH, w = blk / a.BH;
    const int64_t tile = a.v_tile0 + w;
    const int64_t g_lo = std::max<int64_t>(a.v_q0, tile * 16), g_hi = std::min<int64_t>(a.v_q0 + a.v_n, tile * 16 + 16);
    const int i_lo = (int)(g_lo - tile * 16), i_hi = (int)(g_hi - tile * 16);
    Src<TI, TT> src{static_cast<const TT*>(a.v_tail), a.v_cap, a.v_start, a.v_L, vin, a.t};
    uint8_t* codes = sm;                                       // [16][D]
    float* xs = reinterpret_cast<float*>(sm + 16 * D);         // [16][D+1]
    const int Dp = D + 1;
    const int cg = (D + gs - 1) / gs;
    const int q_max = q_max_for_bits(a.vbits);
    for (int e = threadIdx.x; e < 16 * D; e += blockDim.x) {
      const int i = e / D, d = e % D;
      codes[e] = 0;
      if (i >= i_lo && i < i_hi) xs[i * Dp + d] = src.at(bh, tile * 16 + i - a.v_q0, d, D);
    }
    __syncthreads();
    uint32_t* mrow = reinterpret_cast<uint32_t*>(xs + 16 * Dp);  // [16][cg]
    for (int e = threadIdx.x; e < (i_hi - i_lo) * cg; e += blockDim.x) {
      const int i = i_lo + e / cg, gi = e % cg;
      const int d0 = gi * gs, d1 = min(d0 + gs, D);
      float mn = xs[i * Dp + d0], mx = mn;
      for (int d = d0 + 1; d < d1; ++d) {
        const float x = xs[i * Dp + d];
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
      }
      const uint32_t m = make_meta(mn, mx, q_max);
      mrow[i * cg + gi] = m;
      a.v_meta[vmeta_at(a.vv, bh, tile * 16 + i, gi)] = m;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < (i_hi - i_lo) * D; e += blockDim.x) {
      const int i = i_lo + e / D, d = e % D;
      const uint32_t m = mrow[i * cg + d / gs];
      const int64_t tl = tile * 16 + i - a.v_q0;  // token index inside the segment
      const uint64_t si = ((uint64_t)a.vv.gbh(bh) * a.v_n + (uint64_t)tl) * D + d;
      codes[i * D + d] = (uint8_t)encode(xs[i * Dp + d], meta_scale(m), meta_min(m), a.vbits, is_narrow(a.vbits, si));
    }
    if (bh == 0) {
      for (int i = i_lo + threadIdx.x; i < i_hi; i += blockDim.x)
        a.v_info[tile * 16 + i] = make_int2((int)a.v_n, (int)(tile * 16 + i - a.v_q0));
    }
    __syncthreads();
    // only the aged rows' fields: one atomicOr per code into the (zero-initialised) tile
    uint32_t* tp = a.v_tiles + tile_index(a.vv, bh, tile);
    for (int e = threadIdx.x; e < (i_hi - i_lo) * D; e += blockDim.x) {
      const int i = i_lo + e / D, d = e % D;
      const uint32_t code = codes[i * D + d];
      tile_or(tp, false, a.vv.dl, a.vbits, i, d, code);
    }
    return;
  }
  blk -= n_v_blocks;
  if (a.phase == 1) return;

  // ---- tail CTAs: copy staying input tokens into both rings ------------------------------
  const size_t per_side = (size_t)a.BH * a.t * D;
  for (size_t e = (size_t)blk * blockDim.x + threadIdx.x; e < 2 * per_side; e += (size_t)a.tail_blocks * blockDim.x) {
    const bool is_k = e < per_side;
    const size_t r = is_k ? e : e - per_side;
    const int d = (int)(r % D);
    const size_t rowi = r / D;
    const int ti = (int)(rowi % a.t);
    const int bh = (int)(rowi / a.t);
    const int64_t stay0 = is_k ? a.k_stay0 : a.v_stay0;
    if (ti < stay0) continue;
    const int64_t L = is_k ? a.k_L : a.v_L, cap = is_k ? a.k_cap : a.v_cap, start = is_k ? a.k_start : a.v_start;
    const int64_t slot = (start + L + ti) % cap;  // logical index L + ti (before the shift)
    const TI* in = is_k ? kin : vin;
    TT* tail = static_cast<TT*>(is_k ? a.k_tail : a.v_tail);
    tail[((size_t)bh * cap + (size_t)slot) * D + d] = from_f<TT>(ld_f<TI>(in + r));
  }
}

// Decode-step append (t = 1, no Key group ages): one warp per (b, kv-head)
// (decode_append_warp, cache.cuh). A small kernel: the general append kernel's size costs
// instruction-cache misses that dominate a 1-token step.
__global__ void __launch_bounds__(kAppendThreads) append_decode_kernel(DecodeAppend a) {
  const int bh = blockIdx.x * (kAppendThreads / 32) + (int)(threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (bh >= a.BH) return;
  decode_append_warp(a, bh, lane);
}

// ---- snapshot / export / import --------------------------------------------------------

template <typename TT>
__global__ void snapshot_kernel(SideView s, bool key, int D, int gs, int64_t T, int BH, float* out) {
  const size_t n = (size_t)BH * T * D;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    const int64_t j = (int64_t)((e / D) % T);
    const int bh = (int)(e / ((size_t)D * T));
    out[e] = j < s.quantized ? packed_value(key, s, bh, j, d, D, gs) : tail_at<TT>(s, bh, j - s.quantized, d, D);
  }
}

// Rebuild a reference segment (QuantizedGroups of shape [B,H,n,D]) from the device store.
__global__ void export_words_kernel(SideView s, bool key, int D, int BH, int64_t S, int64_t n, uint32_t* words) {
  const int bits = s.bits;
  const int cpw = codes_per_word(bits);
  const size_t total = (size_t)BH * n * D;
  const size_t nw = words_for(total, bits);
  for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < nw; w += (size_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
    for (int k = 0; k < cpw; ++k) {
      const size_t p = w * cpw + k;
      if (p >= total) break;
      int bh, d;
      int64_t tl;
      if (key) {
        const size_t c = p / n;
        tl = (int64_t)(p % n);
        bh = (int)(c / D);
        d = (int)(c % D);
      } else {
        const size_t tok = p / D;
        d = (int)(p % D);
        bh = (int)(tok / n);
        tl = (int64_t)(tok % n);
      }
      const int64_t j = S + tl;
      const uint32_t* tile = s.tiles + tile_index(s, bh, j >> 4);
      const int i = (int)(j & 15);
      const uint32_t code = tile_get(tile, key, s.dl, bits, i, d);
      word |= code << field_shift(bits, (uint32_t)k);
    }
    words[w] = word;
  }
}

__global__ void export_meta_kernel(SideView s, bool key, int D, int gs, int BH, int64_t S, int64_t n, uint32_t* meta) {
  const int cg = (D + gs - 1) / gs;
  const size_t groups = key ? (size_t)BH * D * (n / gs) : (size_t)BH * n * cg;
  for (size_t mi = blockIdx.x * (size_t)blockDim.x + threadIdx.x; mi < groups; mi += (size_t)gridDim.x * blockDim.x) {
    if (key) {
      const int64_t gpc = n / gs;
      const size_t c = mi / gpc;
      const int64_t gl = (int64_t)(mi % gpc);
      const int bh = (int)(c / D), d = (int)(c % D);
      meta[mi] = s.meta[kmeta_index(s, bh, S / gs + gl) + d];
    } else {
      const size_t tok = mi / cg;
      const int g = (int)(mi % cg);
      const int bh = (int)(tok / n);
      const int64_t tl = (int64_t)(tok % n);
      meta[mi] = s.meta[vmeta_at(s, bh, S + tl, g)];
    }
  }
}

template <typename TT>
__global__ void export_tail_kernel(SideView s, int D, int BH, float* out) {
  const size_t n = (size_t)s.tail_len * BH * D;  // [j][bh][d]
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    const int bh = (int)((e / D) % BH);
    const int64_t j = (int64_t)(e / ((size_t)D * BH));
    out[e] = tail_at<TT>(s, bh, j, d, D);
  }
}

// Import one reference segment (words/meta as exported) at quantized position q0.
__global__ void import_kernel(SideView s, uint32_t* tiles, uint32_t* dmeta, int2* info, bool key,
                              int D, int gs, int BH, int64_t q0, int64_t n, const uint32_t* words,
                              const uint32_t* meta) {
  const int bits = s.bits;
  const int cpw = codes_per_word(bits);
  const size_t total = (size_t)BH * n * D;
  const int cg = (D + gs - 1) / gs;
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < total; p += (size_t)gridDim.x * blockDim.x) {
    int bh, d;
    int64_t tl;
    if (key) {
      const size_t c = p / n;
      tl = (int64_t)(p % n);
      bh = (int)(c / D);
      d = (int)(c % D);
    } else {
      const size_t tok = p / D;
      d = (int)(p % D);
      bh = (int)(tok / n);
      tl = (int64_t)(tok % n);
    }
    const uint32_t pos = (uint32_t)(p % cpw);
    const uint32_t code = (words[p / cpw] >> field_shift(bits, pos)) & field_mask(bits, pos);
    const int64_t j = q0 + tl;
    uint32_t* tile = tiles + tile_index(s, bh, j >> 4);
    tile_or(tile, key, s.dl, bits, (int)(j & 15), d, code);
    if (key) {
      if (tl % gs == 0) {
        dmeta[kmeta_index(s, bh, j / gs) + d] = meta[((size_t)bh * D + d) * (n / gs) + tl / gs];
        if (bh == 0 && d == 0) info[j / gs] = make_int2((int)n, (int)tl);
      }
    } else if (d % gs == 0) {
      dmeta[vmeta_at(s, bh, j, d / gs)] = meta[((size_t)bh * n + tl) * cg + d / gs];
      if (bh == 0 && d == 0) info[j] = make_int2((int)n, (int)tl);
    }
  }
}

template <typename TT>
__global__ void import_tail_kernel(void* tail, int64_t cap, int64_t start, int D, int BH, int64_t t, const float* src) {
  const size_t n = (size_t)t * BH * D;  // [j][bh][d]
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    const int bh = (int)((e / D) % BH);
    const int64_t j = (int64_t)(e / ((size_t)D * BH));
    static_cast<TT*>(tail)[((size_t)bh * cap + (size_t)((start + j) % cap)) * D + d] = from_f<TT>(src[e]);
  }
}

int grid_for(size_t n, int threads) {
  const size_t b = (n + threads - 1) / threads;
  const size_t cap = (size_t)num_sms() * 16;
  return (int)std::max<size_t>(1, std::min(b, cap));
}

template <typename TI, typename TT>
void launch_append(const AppendArgs& a, int blocks, size_t smem, const void* k, const void* v, cudaStream_t st) {
  auto kern = append_kernel<TI, TT>;
  if (smem > 48 * 1024) {
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  }
  kern<<<blocks, kAppendThreads, smem, st>>>(a, static_cast<const TI*>(k), static_cast<const TI*>(v));
  after_launch("append_kernel");
}

}  // namespace

void launch_decode_append(const DecodeAppend& da, cudaStream_t st) {
  const int blocks = (da.BH + kAppendThreads / 32 - 1) / (kAppendThreads / 32);
  append_decode_kernel<<<blocks, kAppendThreads, 0, st>>>(da);
  after_launch("append_decode_kernel");
}

bool cache_append_decode_plan(kvmix_cache* c, const void* k, const void* v, kvmix_dtype dt, int t, DecodeAppend* out) {
  if (t != 1 || (dt != KVMIX_F32 && dt != KVMIX_F16) || !k || !v) return false;
  if (c->total() + t > c->cap) return false;
  const int gs = c->cfg.group_size, D = c->D;
  auto& K = c->k;
  auto& V = c->v;
  const int64_t k_cur = K.tail_len + 1;
  const int64_t k_target = (int64_t)std::floor((double)K.ratio * (double)k_cur);
  const int64_t k_n = (k_cur - k_target) / gs * gs;
  const int64_t v_cur = V.tail_len + 1;
  const int64_t v_target = (int64_t)std::floor((double)V.ratio * (double)v_cur);
  const int64_t v_n = std::max<int64_t>(0, v_cur - v_target);
  const int gl = std::min(gs, D) / std::max(1, D / 32);
  if (k_n > 0 || v_n > 1 || !(D == 64 || D == 128) || (gl & (gl - 1)) != 0 || gs % (D / 32) != 0) return false;
  if (K.tail_len + 1 > K.tail_cap || V.tail_len + 1 > V.tail_cap) return false;
  DecodeAppend a{};
  a.D = D;
  a.gs = gs;
  a.BH = c->B * c->H;
  a.in16 = dt == KVMIX_F16;
  a.tail16 = c->tail_dtype == KVMIX_F16;
  a.kin = k;
  a.vin = v;
  a.k_tail = K.tail;
  a.k_cap = K.tail_cap;
  a.k_slot = (K.tail_start + K.tail_len) % K.tail_cap;
  a.v_age = (int)v_n;
  a.v_stay = V.tail_len + 1 - v_n > 0 ? 1 : 0;  // the new token stays unless it is the aged one
  a.vbits = V.bits;
  a.v_j = V.quantized;
  a.v_tail = V.tail;
  a.v_cap = V.tail_cap;
  a.v_start = V.tail_start;
  a.v_L = V.tail_len;
  a.v_slot = (V.tail_start + V.tail_len) % V.tail_cap;
  a.v_tiles = V.tiles;
  a.v_meta = V.meta;
  a.v_info = V.info;
  a.vv = view(V);
  *out = a;
  // host bookkeeping (cache.cpp:65-79): Key tail grows; one Value token may age
  K.tail_len += 1;
  if (v_n > 0) {
    V.segs.push_back(v_n);
    V.quantized += v_n;
    V.tail_start = (V.tail_start + v_n) % V.tail_cap;
  }
  V.tail_len = V.tail_len + 1 - v_n;
  return true;
}

void cache_append(kvmix_cache* c, const void* k, const void* v, kvmix_dtype dt, int t, cudaStream_t st) {
  {
    DecodeAppend da;
    if (cache_append_decode_plan(c, k, v, dt, t, &da)) {
      launch_decode_append(da, st);
      return;
    }
  }
  if (t < 1) invalid("KVLayerCache::append: need at least one token");
  if (dt != KVMIX_F32 && dt != KVMIX_F16) invalid("unsupported dtype");
  if (!k || !v) invalid("KVLayerCache::append: null tensor");
  if (c->total() + t > c->cap) {
    throw Error(KVMIX_OUT_OF_MEMORY, "KVLayerCache::append: capacity of " + std::to_string(c->cap) +
                                         " tokens exceeded (the device cache is sized at creation)");
  }
  const int gs = c->cfg.group_size, D = c->D, BH = c->B * c->H;
  auto& K = c->k;
  auto& V = c->v;
  // shrink rule (cache.cpp:65-79), host integer bookkeeping; rpc_target: floor(double(r) * n)
  const int64_t k_cur = K.tail_len + t;
  const int64_t k_target = (int64_t)std::floor((double)K.ratio * (double)k_cur);
  const int64_t k_n = (k_cur - k_target) / gs * gs;
  const int64_t v_cur = V.tail_len + t;
  const int64_t v_target = (int64_t)std::floor((double)V.ratio * (double)v_cur);
  const int64_t v_n = std::max<int64_t>(0, v_cur - v_target);
  const int64_t k_new_len = k_cur - std::max<int64_t>(0, k_n);
  const int64_t v_new_len = v_cur - v_n;
  if (k_new_len > K.tail_cap || v_new_len > V.tail_cap) {
    throw Error(KVMIX_RUNTIME_ERROR, "KVLayerCache::append: full-precision window exceeds its device ring");
  }

  AppendArgs a{};
  a.H = c->H;
  a.D = D;
  a.gs = gs;
  a.t = t;
  a.BH = BH;
  a.kbits = K.bits;
  a.k_q0 = K.quantized;
  a.k_n = std::max<int64_t>(0, k_n);
  a.k_groups = (int)(a.k_n / gs);
  a.k_blocks = a.k_groups * BH;
  a.k_tiles = K.tiles;
  a.k_meta = K.meta;
  a.k_info = K.info;
  a.kv = view(K);
  a.vbits = V.bits;
  a.v_q0 = V.quantized;
  a.v_n = v_n;
  if (v_n > 0) {
    a.v_tile0 = (int)(V.quantized / 16);
    const int64_t tile_end = (V.quantized + v_n + 15) / 16;
    a.v_blocks = (int)(tile_end - a.v_tile0) * BH;
    // decode-sized age-outs: warp per (token, bh) (channel groups of a power-of-two lane count)
    const int gl = std::min(gs, D) / std::max(1, D / 32);
    if (v_n <= 16 && (D == 64 || D == 128) && gl >= 1 && (gl & (gl - 1)) == 0 && gs % (D / 32) == 0) {
      a.v_warp = 1;
      a.v_blocks = (int)((v_n * BH + kAppendThreads / 32 - 1) / (kAppendThreads / 32));
    }
  }
  a.v_tiles = V.tiles;
  a.v_meta = V.meta;
  a.v_info = V.info;
  a.vv = view(V);
  a.k_tail = K.tail;
  a.v_tail = V.tail;
  a.k_cap = K.tail_cap;
  a.k_start = K.tail_start;
  a.k_L = K.tail_len;
  a.v_cap = V.tail_cap;
  a.v_start = V.tail_start;
  a.v_L = V.tail_len;
  // input token ti (logical L + ti) stays iff L + ti >= aged count
  a.k_stay0 = std::max<int64_t>(0, a.k_n - K.tail_len);
  a.v_stay0 = std::max<int64_t>(0, v_n - V.tail_len);
  const bool any_stay = a.k_stay0 < t || a.v_stay0 < t;
  a.tail_blocks = any_stay ? grid_for((size_t)2 * BH * t * D, kAppendThreads) : 0;

  const size_t smem_k = a.k_blocks ? (size_t)gs * c->Dl + (size_t)gs * D * 4 : 0;  // codes + staged values
  const size_t smem_v = a.v_blocks ? (size_t)16 * D + (size_t)16 * (D + 1) * 4 + (size_t)16 * c->cgroups() * 4 : 0;
  const size_t smem = std::max(smem_k, smem_v);
  // ring hazard: new tail slots could alias aged slots still being read only if L + t > cap
  const bool fused = (K.tail_len + t <= K.tail_cap) && (V.tail_len + t <= V.tail_cap);
  auto launch = [&](AppendArgs args, int blocks) {
    if (blocks == 0) return;
    const bool in16 = dt == KVMIX_F16, tail16 = c->tail_dtype == KVMIX_F16;
    if (!in16 && !tail16) launch_append<float, float>(args, blocks, smem, k, v, st);
    else if (!in16 && tail16) launch_append<float, __half>(args, blocks, smem, k, v, st);
    else if (in16 && !tail16) launch_append<__half, float>(args, blocks, smem, k, v, st);
    else launch_append<__half, __half>(args, blocks, smem, k, v, st);
  };
  if (fused) {
    a.phase = 0;
    launch(a, a.k_blocks + a.v_blocks + a.tail_blocks);
  } else {
    a.phase = 1;
    launch(a, a.k_blocks + a.v_blocks);
    a.phase = 2;
    launch(a, a.tail_blocks);
  }

  if (a.k_n > 0) {
    K.segs.push_back(a.k_n);
    K.quantized += a.k_n;
  }
  K.tail_start = (K.tail_start + a.k_n) % K.tail_cap;
  K.tail_len = k_new_len;
  if (v_n > 0) {
    V.segs.push_back(v_n);
    V.quantized += v_n;
  }
  V.tail_start = (V.tail_start + v_n) % V.tail_cap;
  V.tail_len = v_new_len;
}

void cache_snapshot(const kvmix_cache* c, float* keys, float* values, cudaStream_t st) {
  const int64_t T = c->total();
  const int BH = c->B * c->H;
  const size_t n = (size_t)BH * T * c->D;
  if (n == 0) return;
  const int grid = grid_for(n, 256);
  if (c->tail_dtype == KVMIX_F16) {
    snapshot_kernel<__half><<<grid, 256, 0, st>>>(view(c->k), true, c->D, c->cfg.group_size, T, BH, keys);
    snapshot_kernel<__half><<<grid, 256, 0, st>>>(view(c->v), false, c->D, c->cfg.group_size, T, BH, values);
  } else {
    snapshot_kernel<float><<<grid, 256, 0, st>>>(view(c->k), true, c->D, c->cfg.group_size, T, BH, keys);
    snapshot_kernel<float><<<grid, 256, 0, st>>>(view(c->v), false, c->D, c->cfg.group_size, T, BH, values);
  }
  count_launch();  // two launches above
  after_launch("snapshot_kernel");
}

static int64_t seg_start(const kvmix_cache::Side& s, int idx) {
  int64_t S = 0;
  for (int i = 0; i < idx; ++i) S += s.segs[i];
  return S;
}

static bool sharded(const kvmix_cache* c) { return c->k.Hg != c->H || c->k.b0 != 0 || c->k.h0 != 0; }

void cache_export_segment(const kvmix_cache* c, int side, int idx, uint32_t* words, uint16_t* meta, cudaStream_t st) {
  const auto& s = side == 0 ? c->k : c->v;
  if (s.bits == 3 && sharded(c) && words)
    invalid("export: the Mixed3 words of a sharded cache follow the global stream index; gather the shards");
  if (idx < 0 || idx >= (int)s.segs.size()) throw Error(KVMIX_OUT_OF_RANGE, "segment index out of range");
  const int64_t S = seg_start(s, idx), n = s.segs[idx];
  const int BH = c->B * c->H;
  const size_t nw = words_for((size_t)BH * n * c->D, s.bits);
  if (words) {
    export_words_kernel<<<grid_for(nw, 256), 256, 0, st>>>(view(s), side == 0, c->D, BH, S, n, words);
    after_launch("export_words_kernel");
  }
  if (meta) {
    const size_t groups = side == 0 ? (size_t)BH * c->D * (n / c->cfg.group_size) : (size_t)BH * n * c->cgroups();
    export_meta_kernel<<<grid_for(groups, 256), 256, 0, st>>>(view(s), side == 0, c->D, c->cfg.group_size, BH, S, n,
                                                              reinterpret_cast<uint32_t*>(meta));
    after_launch("export_meta_kernel");
  }
}

void cache_export_tail(const kvmix_cache* c, int side, float* out, cudaStream_t st) {
  const auto& s = side == 0 ? c->k : c->v;
  const int BH = c->B * c->H;
  const size_t n = (size_t)s.tail_len * BH * c->D;
  if (n == 0) return;
  if (c->tail_dtype == KVMIX_F16) export_tail_kernel<__half><<<grid_for(n, 256), 256, 0, st>>>(view(s), c->D, BH, out);
  else export_tail_kernel<float><<<grid_for(n, 256), 256, 0, st>>>(view(s), c->D, BH, out);
  after_launch("export_tail_kernel");
}

void cache_import_segment(kvmix_cache* c, int side, int t, const uint32_t* words, const uint16_t* meta, cudaStream_t st) {
  auto& s = side == 0 ? c->k : c->v;
  const int gs = c->cfg.group_size;
  if (s.bits == 3 && sharded(c)) invalid("import: Mixed3 segments cannot be imported into a sharded cache");
  if (t < 1) invalid("import: empty segment");
  if (side == 0 && (t % gs != 0)) invalid("import: key segment length must be a multiple of group_size");
  if (s.tail_len != 0) invalid("import: segments must be imported before the tail");
  if (s.quantized + t > c->cap) throw Error(KVMIX_OUT_OF_MEMORY, "import: capacity exceeded");
  if (side == 0 && s.quantized % gs != 0) invalid("import: key segments must stay group aligned");
  const int BH = c->B * c->H;
  const size_t total = (size_t)BH * t * c->D;
  import_kernel<<<grid_for(total, 256), 256, 0, st>>>(view(s), s.tiles, s.meta, s.info, side == 0, c->D, gs, BH,
                                                      s.quantized, t, words, reinterpret_cast<const uint32_t*>(meta));
  after_launch("import_kernel");
  s.segs.push_back(t);
  s.quantized += t;
}

void cache_import_tail(kvmix_cache* c, int side, const float* tail, int64_t t, cudaStream_t st) {
  auto& s = side == 0 ? c->k : c->v;
  if (t < 0 || t > s.tail_cap) invalid("import: tail longer than the device ring");
  if (s.quantized + t > c->cap) throw Error(KVMIX_OUT_OF_MEMORY, "import: capacity exceeded");
  const int BH = c->B * c->H;
  s.tail_start = 0;
  s.tail_len = t;
  const size_t n = (size_t)t * BH * c->D;
  if (n == 0) return;
  if (c->tail_dtype == KVMIX_F16)
    import_tail_kernel<__half><<<grid_for(n, 256), 256, 0, st>>>(s.tail, s.tail_cap, 0, c->D, BH, t, tail);
  else
    import_tail_kernel<float><<<grid_for(n, 256), 256, 0, st>>>(s.tail, s.tail_cap, 0, c->D, BH, t, tail);
  after_launch("import_tail_kernel");
}

void cache_reset(kvmix_cache* c, cudaStream_t st) {
  check_cuda(cudaMemsetAsync(c->rec, 0, c->rec_bytes, st), "memset records");
  for (auto* s : {&c->k, &c->v}) {
    s->segs.clear();
    s->quantized = 0;
    s->tail_len = 0;
    s->tail_start = 0;
  }
}

}  // namespace kvb
