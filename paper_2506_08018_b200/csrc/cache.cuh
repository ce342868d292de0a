// cache.cuh -- device-resident per-layer KV cache (KVLayerCache, cache.hpp:52-104).
#pragma once

#include <vector>

#include "common.cuh"

// HBM layout of one layer (bh = b*H + h, all arrays bh-major so one (b, kv-head) stream is
// contiguous -- the unit attention CTAs and the multi-GPU shards partition):
//   K tiles  [bh][tile = token/16][tile_words(D, key_bits)]      packed codes, fragment-native
//   K meta   [bh][group = token/gs][D]        u32 {scale_f16 | min_f16 << 16}
//   K tail   [bh][ring slot][D]               fp32 or fp16 full-precision window (ring)
//   V tiles  [bh][tile][tile_words(D, value_bits)]
//   V meta   [bh][token][ceil(D/gs)]          u32
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
    uint32_t* tiles = nullptr;
    uint32_t* meta = nullptr;
    void* tail = nullptr;
    int2* info = nullptr;
    size_t tiles_per_bh = 0, tile_words = 0, meta_per_bh = 0;
  };
  kvmix_layer_config cfg{};
  int B = 0, H = 0, D = 0;
  int64_t cap = 0;
  kvmix_dtype tail_dtype = KVMIX_F32;
  int device = 0;
  Side k, v;
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
  size_t tiles_per_bh, tile_words, meta_per_bh;
};

inline SideView view(const kvmix_cache::Side& s) {
  return SideView{s.tiles, s.meta, s.tail, s.info, s.tail_cap, s.tail_start, s.tail_len, s.quantized,
                  s.bits, s.tiles_per_bh, s.tile_words, s.meta_per_bh};
}

template <typename TT>
__device__ inline float tail_at(const SideView& s, int bh, int64_t j, int d, int D) {
  int64_t slot = s.tail_start + j;  // j < tail_len <= tail_cap
  if (slot >= s.tail_cap) slot -= s.tail_cap;
  return ld_f<TT>(static_cast<const TT*>(s.tail) + ((size_t)bh * s.tail_cap + (size_t)slot) * D + d);
}

// Narrow-slot test for the Mixed3 layout from the segment info, in mod-11 arithmetic
// (stream index = (bh*D + d)*n + t_local for Keys, (bh*n + t_local)*D + d for Values).
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
  const uint32_t* tile = s.tiles + (size_t)bh * s.tiles_per_bh * s.tile_words + (size_t)(j >> 4) * s.tile_words;
  const int i = j & 15;
  const uint32_t code = tile_get(tile, key ? key_coord(i, d) : value_coord(i, d), D, s.bits);
  uint32_t m;
  bool narrow = false;
  if (key) {
    const int grp = j / gs;
    m = s.meta[(size_t)bh * s.meta_per_bh + (size_t)grp * D + d];
    if (s.bits == 3) narrow = narrow_key(bh, d, D, s.info[grp], j - grp * gs);
  } else {
    const int cg = (D + gs - 1) / gs;
    m = s.meta[(size_t)bh * s.meta_per_bh + (size_t)j * cg + d / gs];
    if (s.bits == 3) narrow = narrow_value(bh, d, D, s.info[j]);
  }
  return decode(code, meta_scale(m), meta_min(m), narrow);
}

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
