// cache.cuh -- device-resident per-layer KV cache (KVLayerCache, cache.hpp:52-104).
#pragma once

#include <vector>

#include "common.cuh"

// HBM layout of one layer (bh = b*H + h, bh-major so one (b, kv-head) stream is contiguous
// -- the unit the attention work list and the multi-GPU shards partition). The packed store
// is ONE array of group records, so the attention kernel moves a whole group (Keys, Values
// and both metas) with a single bulk copy:
//   rec      [bh][group = token/gs] { K tiles [gs/16][tile_words(D, key_bits)]   fragment-native codes (common.cuh)
//                                     V tiles [gs/16][tile_words(D, value_bits)]
//                                     V meta  [ceil(D/gs)][gs]  u32 {scale_f16 | min_f16 << 16}
//                                     K meta  [D] }
//   K tail   [bh][ring slot][D]               fp32 or fp16 full-precision window (ring)
//   V tail   [bh][ring slot][D]
//   K info   [group] int2 {segment length, token offset in segment}  (Mixed3 narrow slots)
//   V info   [token] int2 {segment length, token offset in segment}
// Segments (one per age-out event, cache.cpp:82-117) are host bookkeeping only: the device
// store is flat, and export rebuilds each segment's reference words on demand.
struct kvmix_cache {
  struct Side {
    int bits = 2;
    float ratio = 0.1f;
    int64_t tail_cap = 0, tail_start = 0, tail_len = 0, quantized = 0;
    std::vector<int64_t> segs;
    uint32_t* tiles = nullptr;  // this side's tiles / meta inside the group records
    uint32_t* meta = nullptr;
    void* tail = nullptr;
    int2* info = nullptr;
    size_t tile_words = 0, bh_stride = 0, grp_stride = 0;  // words
    int tpg = 0, mrow = 0;  // tiles per group; meta words per Key group / per Value token
    int dl = 0;             // channels of the tile layout: head_dim rounded up to a multiple of 64
    // shard placement (kvmix_cache_set_shard): this cache holds heads [h0, h0 + H) of batch
    // rows [b0, b0 + B) of a [Bg, Hg] model batch; Mixed3 narrow slots follow the GLOBAL
    // (b, h) stream index, so a shard holds exactly the unsharded cache's slice
    int Hl = 1, Hg = 1, b0 = 0, h0 = 0;
  };
  kvmix_layer_config cfg{};
  int B = 0, H = 0, D = 0;
  int Dl = 0;  // tile-layout channels: D rounded up to a multiple of 64 (== D for 64 / 128)
  int64_t cap = 0;
  kvmix_dtype tail_dtype = KVMIX_F32;
  int device = 0;
  Side k, v;
  uint32_t* rec = nullptr;  // group records of both sides
  size_t rec_bytes = 0;
  int cgroups() const { return (D + cfg.group_size - 1) / cfg.group_size; }
  int64_t total() const { return k.quantized + k.tail_len; }
};

namespace kvb {

// Device view of one side, passed by value to kernels.
struct SideView {
  const uint32_t* tiles;
  const uint32_t* meta;
  const void* tail;
  const int2* info;
  int64_t tail_cap, tail_start, tail_len, quantized;
  int bits;
  size_t tile_words, bh_stride, grp_stride;
  int tpg, mrow;
  int dl;              // tile-layout channels (>= head_dim; the padded channels hold zero codes)
  int Hl, Hg, b0, h0;  // shard placement (Side)
  // global (b, kv-head) index of local bh: the one the reference's stream index uses
  __host__ __device__ int gbh(int bh) const { return (b0 + bh / Hl) * Hg + h0 + bh % Hl; }
};

inline SideView view(const kvmix_cache::Side& s) {
  return SideView{s.tiles, s.meta, s.tail, s.info, s.tail_cap, s.tail_start, s.tail_len, s.quantized,
                  s.bits, s.tile_words, s.bh_stride, s.grp_stride, s.tpg, s.mrow, s.dl, s.Hl, s.Hg, s.b0, s.h0};
}

// Word offsets into a side's tiles / meta (group-record layout above).
// (32-bit index math: tokens per (b, kv-head) < 2^31, enforced at cache creation)
__host__ __device__ inline size_t tile_index(const SideView& s, int bh, int64_t tile) {
  const unsigned t = (unsigned)tile, tp = (unsigned)s.tpg, gi = t / tp;
  return (size_t)bh * s.bh_stride + (size_t)gi * s.grp_stride + (size_t)(t - gi * tp) * s.tile_words;
}
// Key meta row of group grp (D words, one per channel)
__host__ __device__ inline size_t kmeta_index(const SideView& s, int bh, int64_t grp) {
  return (size_t)bh * s.bh_stride + (size_t)grp * s.grp_stride;
}
// Value meta word of token j, channel group g. Inside a group record the Value meta is
// [channel group][token] (gs words per channel group), so the metas of consecutive tokens of
// one channel group are contiguous (one 16-byte load for a token quad in the attention kernel).
__host__ __device__ inline size_t vmeta_at(const SideView& s, int bh, int64_t j, int g) {
  const unsigned gs = (unsigned)s.tpg * 16u, jj = (unsigned)j, gi = jj / gs;
  return (size_t)bh * s.bh_stride + (size_t)gi * s.grp_stride + (size_t)g * gs + (jj - gi * gs);
}

template <typename TT>
__device__ inline float tail_at(const SideView& s, int bh, int64_t j, int d, int D) {
  int64_t slot = s.tail_start + j;  // j < tail_len <= tail_cap
  if (slot >= s.tail_cap) slot -= s.tail_cap;
  return ld_f<TT>(static_cast<const TT*>(s.tail) + ((size_t)bh * s.tail_cap + (size_t)slot) * D + d);
}

// Narrow-slot test for the Mixed3 layout from the segment info, in mod-11 arithmetic
// (stream index = (bh*D + d)*n + t_local for Keys, (bh*n + t_local)*D + d for Values; bh is
// the GLOBAL (b, kv-head) index, SideView::gbh).
__device__ inline bool narrow_key(int bh, int d, int D, int2 info, int t_in_group) {
  const int c = (int)(((unsigned)bh * (unsigned)D + (unsigned)d) % 11u);
  return (c * (info.x % 11) + (info.y + t_in_group) % 11) % 11 == 10;
}
__device__ inline bool narrow_value(int bh, int d, int D, int2 info) {
  const int tok = (int)(((unsigned)bh % 11u) * (unsigned)(info.x % 11) % 11u + (unsigned)(info.y % 11)) % 11;
  return (tok * (D % 11) + d % 11) % 11 == 10;
}

// Dequantized value of quantized token j (j < s.quantized) of one side, bit-exact.
__device__ inline float packed_value(bool key, const SideView& s, int bh, int64_t j64, int d, int D, int gs) {
  const int j = (int)j64;
  const uint32_t* tile = s.tiles + tile_index(s, bh, j >> 4);
  const int i = j & 15;
  const uint32_t code = tile_get(tile, key, s.dl, s.bits, i, d);
  uint32_t m;
  bool narrow = false;
  if (key) {
    const int grp = j / gs;
    m = s.meta[kmeta_index(s, bh, grp) + d];
    if (s.bits == 3) narrow = narrow_key(s.gbh(bh), d, D, s.info[grp], j - grp * gs);
  } else {
    m = s.meta[vmeta_at(s, bh, j, d / gs)];
    if (s.bits == 3) narrow = narrow_value(s.gbh(bh), d, D, s.info[j]);
  }
  return decode(code, meta_scale(m), meta_min(m), narrow);
}

// ---- decode-step append (t = 1, no Key group ages) --------------------------------------
// Everything one warp needs to append one token of one (b, kv-head): the Key token goes to
// its ring slot; the Value side ages one token (the oldest window token or the new one) and/or
// stores the new token in its ring. Used by append_decode_kernel and, fused, by the
// attention kernel's prologue (kvmix_append_attend).
struct DecodeAppend {
  int D, gs, BH;
  int in16, tail16;          // input / window element types (fp16 or fp32)
  const void* kin;           // [B*H][D] new Key token
  const void* vin;           // [B*H][D] new Value token
  void* k_tail;              // Key ring
  int64_t k_cap, k_slot;     // ring capacity, slot of the new Key token
  int v_age;                 // 1: one Value token ages
  int v_stay;                // 1: the new Value token stays in the window
  int vbits;
  int64_t v_j;               // global index of the aged Value token
  void* v_tail;
  int64_t v_cap, v_start, v_L, v_slot;  // aged token: window slot v_start if v_L > 0, else the input
  uint32_t* v_tiles;
  uint32_t* v_meta;
  int2* v_info;
  SideView vv;
};

// Meta of one Value channel group spread over `glanes` consecutive lanes (power of two) with
// LC channels per lane in stream order: the ordered fold over the lanes' segments (the lower
// lane holds the earlier segment), then the leader's result broadcast so every lane of the
// group encodes with the stored meta.
template <int LCMAX>
__device__ inline uint32_t group_meta_warp(const float (&x)[LCMAX], int LC, int glanes, int lane, int q_max) {
  float mn = NAN, mx = NAN;
  for (int c = 0; c < LC; ++c) {
    mn = fold_min(mn, x[c]);
    mx = fold_max(mx, x[c]);
  }
  for (int o = 1; o < glanes; o <<= 1) {
    const float omn = __shfl_xor_sync(0xffffffffu, mn, o), omx = __shfl_xor_sync(0xffffffffu, mx, o);
    const bool hi = lane & o;  // the partner holds the earlier segment
    const float fmn = hi ? fold_min(omn, mn) : fold_min(mn, omn);
    const float fmx = hi ? fold_max(omx, mx) : fold_max(mx, omx);
    mn = fmn;
    mx = fmx;
  }
  const int lead = lane & ~(glanes - 1);
  if (__shfl_sync(0xffffffffu, isnan(x[0]) ? 1 : 0, lead)) mn = mx = NAN;  // NaN first element
  return __shfl_sync(0xffffffffu, make_meta(mn, mx, q_max), lead);
}

__device__ inline float da_load(const void* p, bool f16, size_t i) {
  return f16 ? __half2float(static_cast<const __half*>(p)[i]) : static_cast<const float*>(p)[i];
}
__device__ inline void da_store(void* p, bool f16, size_t i, float x) {
  if (f16) static_cast<__half*>(p)[i] = __float2half_rn(x);
  else static_cast<float*>(p)[i] = x;
}

// one warp, lanes over D/32 channels (D in {64, 128}, power-of-two channel-group lanes)
__device__ inline void decode_append_warp(const DecodeAppend& a, int bh, int lane) {
  const int D = a.D, gs = a.gs, LC = D / 32;
  {
    const size_t dst = ((size_t)bh * a.k_cap + (size_t)a.k_slot) * D;
    for (int c = 0; c < LC; ++c) {
      const int d = lane * LC + c;
      da_store(a.k_tail, a.tail16, dst + d, da_load(a.kin, a.in16, (size_t)bh * D + d));
    }
  }
  if (a.v_age) {
    const int q_max = q_max_for_bits(a.vbits);
    float x[4];
    for (int c = 0; c < LC; ++c) {
      const int d = lane * LC + c;
      // the window holds values already rounded to its element type; a new token is rounded
      // to it first (cache.cpp keeps one precision per side)
      x[c] = a.v_L > 0 ? da_load(a.v_tail, a.tail16, ((size_t)bh * a.v_cap + (size_t)a.v_start) * D + d)
                       : (a.tail16 ? __half2float(__float2half_rn(da_load(a.vin, a.in16, (size_t)bh * D + d)))
                                   : da_load(a.vin, a.in16, (size_t)bh * D + d));
    }
    const int glanes = min(gs, D) / LC;
    const uint32_t m = group_meta_warp(x, LC, glanes, lane, q_max);
    const int64_t j = a.v_j;
    if ((lane % glanes) == 0) a.v_meta[vmeta_at(a.vv, bh, j, lane * LC / gs)] = m;
    if (bh == 0 && lane == 0) a.v_info[j] = make_int2(1, 0);
    const float sc = meta_scale(m), mnv = meta_min(m);
    uint32_t* tp = a.v_tiles + tile_index(a.vv, bh, j >> 4);
    for (int c = 0; c < LC; ++c) {
      const int d = lane * LC + c;
      const uint64_t si = (uint64_t)a.vv.gbh(bh) * D + d;  // segment [B,H,1,D], global bh
      tile_or(tp, false, a.vv.dl, a.vbits, (int)(j & 15), d, encode(x[c], sc, mnv, a.vbits, is_narrow(a.vbits, si)));
    }
  }
  if (a.v_stay) {
    const size_t dst = ((size_t)bh * a.v_cap + (size_t)a.v_slot) * D;
    for (int c = 0; c < LC; ++c) {
      const int d = lane * LC + c;
      da_store(a.v_tail, a.tail16, dst + d, da_load(a.vin, a.in16, (size_t)bh * D + d));
    }
  }
}

// Host: if this append is a decode step the one-warp path handles, fill `out`, apply the
// host bookkeeping of the append (counters, segments, ring positions) and return true; the
// caller must then run decode_append_warp for every (b, kv-head) before the cache is read.
bool cache_append_decode_plan(kvmix_cache* c, const void* k, const void* v, kvmix_dtype dt, int t, DecodeAppend* out);
void launch_decode_append(const DecodeAppend& da, cudaStream_t st);

void cache_append(kvmix_cache* c, const void* k, const void* v, kvmix_dtype dt, int t, cudaStream_t st);
void cache_snapshot(const kvmix_cache* c, float* keys, float* values, cudaStream_t st);
void cache_export_segment(const kvmix_cache* c, int side, int idx, uint32_t* words, uint16_t* meta,
                          cudaStream_t st);
void cache_export_tail(const kvmix_cache* c, int side, float* out, cudaStream_t st);
void cache_import_segment(kvmix_cache* c, int side, int t, const uint32_t* words, const uint16_t* meta,
                          cudaStream_t st);
void cache_import_tail(kvmix_cache* c, int side, const float* tail, int64_t t, cudaStream_t st);
void cache_reset(kvmix_cache* c, cudaStream_t st);

}  // namespace kvb
