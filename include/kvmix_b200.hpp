// kvmix_b200.hpp -- C++ shim over the C ABI (kvmix_b200.h): the reference's hot-path C++
// API (namespace kvmix, /root/reference/proj/include/kvmix/{tensor,cache,quant,attention}.hpp)
// backed by the B200 kernels, so C++ callers written against the reference (e.g.
// CachedDecoder::step, toymodel.cpp:720-721; bench_attention, harness.cpp:101-120) switch
// by changing the include and linking libkvmix_b200 instead of kvmix_core.
//
// Host tensors (Tensor4f, row-major [B, nh, T, D] fp32) are copied to the device per call;
// the device-pointer performance API is the C ABI itself (kvmix_cache_handle()).
// Exceptions follow the reference: KVMIX_INVALID_ARGUMENT -> std::invalid_argument,
// KVMIX_OUT_OF_RANGE -> std::out_of_range, anything else -> std::runtime_error.
// Device constraints (kvmix_b200.h): head_dim % 64 == 0, head_dim <= 256, group_size % 16 == 0.
// The device cache reserves capacity; append() grows it (segments and tails re-imported)
// when a call would exceed it.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kvmix_b200.h"

namespace kvmix {

namespace b200 {

inline void check(kvmix_status st) {
  if (st == KVMIX_OK) return;
  const std::string m = kvmix_last_error();
  if (st == KVMIX_INVALID_ARGUMENT) throw std::invalid_argument(m);
  if (st == KVMIX_OUT_OF_RANGE) throw std::out_of_range(m);
  throw std::runtime_error(m);
}

inline void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t bytes) : n_(bytes) {
    if (bytes) cuda(cudaMalloc(&p_, bytes), "cudaMalloc");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  ~DevBuf() {
    if (p_) cudaFree(p_);
  }
  template <typename T = void>
  T* get() const { return static_cast<T*>(p_); }
  void upload(const void* src, size_t bytes) { cuda(cudaMemcpy(p_, src, bytes, cudaMemcpyHostToDevice), "H2D"); }
  void download(void* dst, size_t bytes) const { cuda(cudaMemcpy(dst, p_, bytes, cudaMemcpyDeviceToHost), "D2H"); }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

// binary16 -> float (meta values are binary16 bit patterns; half.hpp:44-71)
inline float half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16, exp = (h >> 10) & 0x1fu, man = h & 0x3ffu;
  uint32_t bits;
  if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else {  // subnormal: normalize
      int e = -1;
      uint32_t m = man;
      do {
        ++e;
        m <<= 1;
      } while ((m & 0x400u) == 0);
      bits = sign | (uint32_t)(127 - 15 - e) << 23 | (m & 0x3ffu) << 13;
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | man << 13;
  } else {
    bits = sign | (exp - 15 + 127) << 23 | man << 13;
  }
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

}  // namespace b200

// ---- tensor.hpp:12-41 --------------------------------------------------------------------
struct Tensor4f {
  int b = 0, nh = 0, t = 0, d = 0;
  std::vector<float> data;

  Tensor4f() = default;
  Tensor4f(int b_, int nh_, int t_, int d_) : b(b_), nh(nh_), t(t_), d(d_), data((size_t)b_ * nh_ * t_ * d_, 0.0f) {}
  size_t index(int bi, int hi, int ti, int di) const { return (((size_t)bi * nh + hi) * t + ti) * d + di; }
  float& at(int bi, int hi, int ti, int di) { return data[index(bi, hi, ti, di)]; }
  const float& at(int bi, int hi, int ti, int di) const { return data[index(bi, hi, ti, di)]; }
  float* row(int bi, int hi, int ti) { return data.data() + index(bi, hi, ti, 0); }
  const float* row(int bi, int hi, int ti) const { return data.data() + index(bi, hi, ti, 0); }
  size_t size() const { return data.size(); }
  bool same_shape(const Tensor4f& o) const { return b == o.b && nh == o.nh && t == o.t && d == o.d; }
};

// ---- cache.hpp:26-47 ---------------------------------------------------------------------
struct LayerQuantConfig {
  int layer_index = 0;
  int key_bits = 2;
  int value_bits = 2;
  float key_rpc_ratio = 0.1f;
  float value_rpc_ratio = 0.1f;
  int group_size = 32;

  static float default_rpc_for_bits(int bits) { return bits >= 3 ? 0.2f : 0.1f; }
  kvmix_layer_config c() const {
    return kvmix_layer_config{layer_index, key_bits, value_bits, key_rpc_ratio, value_rpc_ratio, group_size};
  }
  void validate() const {
    const kvmix_layer_config cc = c();
    b200::check(kvmix_config_validate(&cc));
  }
};

struct MemoryReport {
  uint64_t packed_payload_bits = 0;
  uint64_t metadata_bits = 0;
  uint64_t tail_bits = 0;
  uint64_t total_bits = 0;
  uint64_t fp16_baseline_bits = 0;
  double compression_ratio = 1.0;
};

inline int64_t rpc_target(int64_t current_rpc, double r) {
  int64_t out = 0;
  b200::check(kvmix_rpc_target(current_rpc, r, &out));
  return out;
}

// ---- quant.hpp:33-80 ---------------------------------------------------------------------
struct GroupMeta {
  float scale = 0.0f;
  float min_val = 0.0f;
};
enum class Grouping : uint8_t { kPerChannelKey = 0, kPerTokenValue = 1 };
struct QuantSpec {
  int bits = 4;
  Grouping grouping = Grouping::kPerChannelKey;
  int group_size = 32;
};
struct TensorShape {
  int b = 0, nh = 0, t = 0, d = 0;
  size_t elems() const { return (size_t)b * nh * t * d; }
};
// QuantizedGroups with the packed payload as its word vector (PackedBuffer::words,
// bitpack.hpp:35-46) and the binary16 meta pairs (the KVQG payload) alongside.
struct QuantizedGroups {
  std::vector<GroupMeta> meta;
  std::vector<uint32_t> words;
  std::vector<uint16_t> meta_half;  // {scale, min} pairs, KVQG order
  QuantSpec spec;
  TensorShape shape;
  size_t group_count() const { return meta.size(); }
};

namespace b200 {
inline QuantizedGroups quantize(const Tensor4f& x, const QuantSpec& spec) {
  const kvmix_grouping g = spec.grouping == Grouping::kPerChannelKey ? KVMIX_PER_CHANNEL_KEY : KVMIX_PER_TOKEN_VALUE;
  QuantizedGroups q;
  q.spec = spec;
  q.shape = TensorShape{x.b, x.nh, x.t, x.d};
  const size_t nw = kvmix_packed_word_count(x.size(), spec.bits);
  const size_t ng = kvmix_group_count(g, x.b, x.nh, x.t, x.d, spec.group_size);
  DevBuf dx(x.size() * 4), dw(std::max<size_t>(nw, 1) * 4), dm(std::max<size_t>(ng, 1) * 4);
  if (x.size()) dx.upload(x.data.data(), x.size() * 4);
  check(kvmix_quantize(g, dx.get(), KVMIX_F32, x.b, x.nh, x.t, x.d, spec.bits, spec.group_size, dw.get<uint32_t>(),
                       dm.get<uint16_t>(), nullptr));
  q.words.resize(nw);
  q.meta_half.resize(2 * ng);
  if (nw) dw.download(q.words.data(), nw * 4);
  if (ng) dm.download(q.meta_half.data(), ng * 4);
  q.meta.resize(ng);
  for (size_t i = 0; i < ng; ++i) q.meta[i] = GroupMeta{half_to_float(q.meta_half[2 * i]), half_to_float(q.meta_half[2 * i + 1])};
  return q;
}
}  // namespace b200

inline QuantizedGroups quantize_key_tensor(const Tensor4f& keys, const QuantSpec& spec) {
  QuantSpec s = spec;
  s.grouping = Grouping::kPerChannelKey;
  return b200::quantize(keys, s);
}
inline QuantizedGroups quantize_value_tensor(const Tensor4f& values, const QuantSpec& spec) {
  QuantSpec s = spec;
  s.grouping = Grouping::kPerTokenValue;
  return b200::quantize(values, s);
}

// ---- cache.hpp:52-104 --------------------------------------------------------------------
class KVLayerCache {
 public:
  KVLayerCache(const LayerQuantConfig& config, int batch, int heads, int head_dim, int64_t capacity_tokens = 4096,
               kvmix_dtype tail_dtype = KVMIX_F32)
      : cfg_(config), b_(batch), nh_(heads), d_(head_dim), tail_dtype_(tail_dtype) {
    create(capacity_tokens);
  }
  KVLayerCache(const KVLayerCache&) = delete;
  KVLayerCache& operator=(const KVLayerCache&) = delete;
  KVLayerCache(KVLayerCache&& o) noexcept
      : cfg_(o.cfg_), b_(o.b_), nh_(o.nh_), d_(o.d_), cap_(o.cap_), tail_dtype_(o.tail_dtype_), h_(o.h_) {
    o.h_ = nullptr;
  }
  ~KVLayerCache() {
    if (h_) kvmix_cache_destroy(h_);
  }

  void append(const Tensor4f& new_keys, const Tensor4f& new_values) {
    if (new_keys.b != b_ || new_keys.nh != nh_ || new_keys.d != d_ || !new_keys.same_shape(new_values))
      throw std::invalid_argument("KVLayerCache::append: tensor shape does not match cache");
    if (new_keys.t < 1) throw std::invalid_argument("KVLayerCache::append: need at least one token");
    if (total_tokens() + new_keys.t > cap_) grow(std::max<int64_t>(2 * cap_, total_tokens() + new_keys.t));
    b200::DevBuf k(new_keys.size() * 4), v(new_values.size() * 4);
    k.upload(new_keys.data.data(), new_keys.size() * 4);
    v.upload(new_values.data.data(), new_values.size() * 4);
    b200::check(kvmix_cache_append(h_, k.get(), v.get(), KVMIX_F32, new_keys.t, nullptr));
    b200::cuda(cudaDeviceSynchronize(), "append");
  }

  MemoryReport memory_usage() const {
    kvmix_memory_report r{};
    b200::check(kvmix_cache_memory_usage(h_, &r));
    return MemoryReport{r.packed_payload_bits, r.metadata_bits, r.tail_bits, r.total_bits, r.fp16_baseline_bits,
                        r.compression_ratio};
  }

  std::pair<Tensor4f, Tensor4f> snapshot_dequantized() const {
    const int T = (int)total_tokens();
    Tensor4f k(b_, nh_, T, d_), v(b_, nh_, T, d_);
    b200::DevBuf dk(std::max<size_t>(k.size(), 1) * 4), dv(std::max<size_t>(v.size(), 1) * 4);
    b200::check(kvmix_cache_snapshot(h_, dk.get<float>(), dv.get<float>(), nullptr));
    if (k.size()) {
      dk.download(k.data.data(), k.size() * 4);
      dv.download(v.data.data(), v.size() * 4);
    }
    return {std::move(k), std::move(v)};
  }

  int64_t total_tokens() const { return counter(0); }
  int64_t key_tail_tokens() const { return counter(1); }
  int64_t value_tail_tokens() const { return counter(2); }
  int64_t quantized_key_tokens() const { return counter(3); }
  int64_t quantized_value_tokens() const { return counter(4); }
  int batch() const { return b_; }
  int heads() const { return nh_; }
  int head_dim() const { return d_; }
  const LayerQuantConfig& config() const { return cfg_; }
  int64_t capacity_tokens() const { return cap_; }
  kvmix_cache* handle() const { return h_; }

 private:
  int64_t counter(int i) const {
    int64_t c[7];
    b200::check(kvmix_cache_counters(h_, c));
    return c[i];
  }
  void create(int64_t cap) {
    const kvmix_layer_config cc = cfg_.c();
    kvmix_cache* h = nullptr;
    b200::check(kvmix_cache_create(&cc, b_, nh_, d_, cap, tail_dtype_, &h));
    h_ = h;
    cap_ = cap;
  }
  // re-create with a larger reservation: segments re-imported in order, then the tails
  void grow(int64_t cap) {
    kvmix_cache* old = h_;
    int64_t c[7];
    b200::check(kvmix_cache_counters(old, c));
    create(cap);
    for (int side = 0; side < 2; ++side) {
      const int64_t nseg = c[5 + side];
      for (int64_t i = 0; i < nseg; ++i) {
        int64_t info[3];
        b200::check(kvmix_cache_segment_info(old, side, (int)i, info));
        b200::DevBuf w(std::max<int64_t>(info[1], 1) * 4), m(std::max<int64_t>(info[2], 1) * 4);
        b200::check(kvmix_cache_export_segment(old, side, (int)i, w.get<uint32_t>(), m.get<uint16_t>(), nullptr));
        b200::check(kvmix_cache_import_segment(h_, side, (int)info[0], w.get<uint32_t>(), m.get<uint16_t>(), nullptr));
      }
      const int64_t tl = c[1 + side];
      if (tl > 0) {
        b200::DevBuf tb((size_t)tl * b_ * nh_ * d_ * 4);
        b200::check(kvmix_cache_export_tail(old, side, tb.get<float>(), nullptr));
        b200::check(kvmix_cache_import_tail(h_, side, tb.get<float>(), tl, nullptr));
      }
    }
    b200::cuda(cudaDeviceSynchronize(), "grow");
    kvmix_cache_destroy(old);
  }

  LayerQuantConfig cfg_;
  int b_ = 1, nh_ = 1, d_ = 1;
  int64_t cap_ = 0;
  kvmix_dtype tail_dtype_ = KVMIX_F32;
  kvmix_cache* h_ = nullptr;
};

// ---- attention.hpp:25-48 -----------------------------------------------------------------
struct AttentionOutput {
  Tensor4f output;
  double scores_checksum = 0.0;
};

inline float attention_inv_scale(int head_dim) { return 1.0f / std::sqrt(static_cast<float>(head_dim)); }

namespace b200 {
inline AttentionOutput attend_impl(const Tensor4f& q, const KVLayerCache& cache, bool reference) {
  if (q.b != cache.batch() || q.d != cache.head_dim() || q.nh < 1 || q.nh % cache.heads() != 0 ||
      (reference && q.nh != cache.heads()))
    throw std::invalid_argument("attention: query shape does not match cache");
  AttentionOutput r;
  r.output = Tensor4f(q.b, q.nh, q.t, q.d);
  DevBuf dq(std::max<size_t>(q.size(), 1) * 4), dout(std::max<size_t>(r.output.size(), 1) * 4);
  if (q.size()) dq.upload(q.data.data(), q.size() * 4);
  if (reference) {
    DevBuf scratch(std::max<size_t>((size_t)2 * q.b * q.nh * std::max<int64_t>(cache.total_tokens(), 1) * q.d, 1) * 4);
    check(kvmix_reference_attend(cache.handle(), dq.get(), KVMIX_F32, q.t, scratch.get<float>(), dout.get<float>(),
                                 &r.scores_checksum, nullptr));
  } else {
    check(kvmix_attend(cache.handle(), dq.get(), KVMIX_F32, q.nh, q.t, dout.get<float>(), &r.scores_checksum, nullptr));
  }
  if (r.output.size()) dout.download(r.output.data.data(), r.output.size() * 4);
  return r;
}
}  // namespace b200

// attend (attention.cpp:161-166); q.nh may be a multiple G of the cache's heads (GQA)
inline AttentionOutput attend(const Tensor4f& query, const KVLayerCache& cache) {
  return b200::attend_impl(query, cache, false);
}
// reference_attend (attention.cpp:168-211)
inline AttentionOutput reference_attend(const Tensor4f& query, const KVLayerCache& cache) {
  return b200::attend_impl(query, cache, true);
}

// fused_qk_scores (attention.cpp:28-81): [B, nh, t, total], already * 1/sqrt(D)
inline Tensor4f fused_qk_scores(const Tensor4f& query, const KVLayerCache& cache) {
  const int T = (int)cache.total_tokens();
  Tensor4f s(query.b, query.nh, query.t, T);
  b200::DevBuf dq(std::max<size_t>(query.size(), 1) * 4), ds(std::max<size_t>(s.size(), 1) * 4);
  if (query.size()) dq.upload(query.data.data(), query.size() * 4);
  b200::check(kvmix_fused_qk_scores(cache.handle(), dq.get(), KVMIX_F32, query.t, ds.get<float>(), nullptr));
  if (s.size()) ds.download(s.data.data(), s.size() * 4);
  return s;
}

// softmax_rows (attention.cpp:96-105)
inline Tensor4f softmax_rows(Tensor4f scores) {
  if (scores.d == 0) throw std::invalid_argument("softmax over an empty row");
  b200::DevBuf d(std::max<size_t>(scores.size(), 1) * 4);
  if (scores.size()) d.upload(scores.data.data(), scores.size() * 4);
  b200::check(kvmix_softmax_rows(d.get<float>(), (int64_t)(scores.size() / scores.d), scores.d, nullptr));
  if (scores.size()) d.download(scores.data.data(), scores.size() * 4);
  return scores;
}

// fused_pv (attention.cpp:107-159): probs [B, nh, t, total] -> [B, nh, t, D]
inline Tensor4f fused_pv(const Tensor4f& probs, const KVLayerCache& cache) {
  Tensor4f out(probs.b, probs.nh, probs.t, cache.head_dim());
  b200::DevBuf dp(std::max<size_t>(probs.size(), 1) * 4), dout(std::max<size_t>(out.size(), 1) * 4);
  if (probs.size()) dp.upload(probs.data.data(), probs.size() * 4);
  b200::check(kvmix_fused_pv(cache.handle(), dp.get<float>(), probs.t, dout.get<float>(), nullptr));
  if (out.size()) dout.download(out.data.data(), out.size() * 4);
  return out;
}

}  // namespace kvmix
