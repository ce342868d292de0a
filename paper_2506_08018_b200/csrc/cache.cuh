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
//                                     V meta  [gs][ceil(D/gs)]  u32 {scale_f16 | min_f16 << 16}
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
  };
  kvmix_layer_config cfg{};
  int B = 0, H = 0, D = 0;
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
};

inline SideView view(const kvmix_cache::Side& s) {
  return SideView{s.tiles, s.meta, s.tail, s.info, s.tail_cap, s.tail_start, s.tail_len, s.quantized,
                  s.bits, s.tile_words, s.bh_stride, s.grp_stride, s.tpg, s.mrow};
}

// Word offsets into a side's tiles / meta (group-record layout above).
__host__ __device__ inline size_t tile_index(const SideView& s, int bh, int64_t tile) {
  const int64_t gi = tile / s.tpg;
  return (size_t)bh * s.bh_stride + (size_t)gi * s.grp_stride + (size_t)(tile - gi * s.tpg) * s.tile_words;
}
// Key meta row of group grp (D words, one per channel)
__host__ __device__ inline size_t kmeta_index(const SideView& s, int bh, int64_t grp) {
  return (size_t)bh * s.bh_stride + (size_t)grp * s.grp_stride;
}
// Value meta row of token j (ceil(D/gs) words, one per channel group)
__host__ __device__ inline size_t vmeta_index(const SideView& s, int bh, int64_t j) {
  const int gs = s.tpg * 16;
  const int64_t gi = j / gs;
  return (size_t)bh * s.bh_stride + (size_t)gi * s.grp_stride + (size_t)(j - gi * gs) * s.mrow;
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
  const uint32_t* tile = s.tiles + tile_index(s, bh, j >> 4);
  const int i = j & 15;
  const uint32_t code = tile_get(tile, key, D, s.bits, i, d);
  uint32_t m;
  bool narrow = false;
  if (key) {
    const int grp = j / gs;
    m = s.meta[kmeta_index(s, bh, grp) + d];
    if (s.bits == 3) narrow = narrow_key(bh, d, D, s.info[grp], j - grp * gs);
  } else {
    m = s.meta[vmeta_index(s, bh, j) + d / gs];
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
