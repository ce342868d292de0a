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
// Device constraints (kvmix_b200.h): head_dim <= 256, group_size % 16 == 0.
// The device cache reserves capacity; append() grows it (segments and tails re-imported)
// when a call would exceed it.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <istream>
#include <ostream>
#include <span>
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

// float -> binary16, round to nearest even, subnormals, inf; NaN -> sign | 0x7e00 (half.hpp:15-42)
inline uint16_t float_to_half(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  const uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
  const uint32_t a = u & 0x7fffffffu;
  if (a > 0x7f800000u) return sign | 0x7e00u;  // NaN
  if (a >= 0x477ff000u) return sign | 0x7c00u;  // >= 65520 rounds to inf (and inf)
  if (a < 0x33000001u) return sign;             // < 2^-25 (+tie) rounds to zero
  const int e = (int)(a >> 23) - 127;
  uint32_t man = (a & 0x7fffffu) | 0x800000u;
  if (e < -14) {  // subnormal result: shift so the LSB is 2^-24
    const int sh = -14 - e + 13;
    const uint32_t q = man >> sh, rem = man & ((1u << sh) - 1u), half = 1u << (sh - 1);
    const uint32_t r = q + ((rem > half || (rem == half && (q & 1u))) ? 1u : 0u);
    return sign | (uint16_t)r;
  }
  const uint32_t q = man >> 13, rem = man & 0x1fffu;
  uint32_t h = ((uint32_t)(e + 15) << 10) + (q & 0x3ffu);
  if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++h;  // (carry may reach the exponent: correct)
  return sign | (uint16_t)h;
}

}  // namespace b200

// ---- half.hpp:15-71 -----------------------------------------------------------------------
inline uint16_t half_from_float(float x) { return b200::float_to_half(x); }
inline float float_from_half(uint16_t h) { return b200::half_to_float(h); }
inline float round_through_half(float x) { return b200::half_to_float(b200::float_to_half(x)); }

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
// ---- bitpack.hpp:10-72 (PackedBuffer / PackedWriter; pack_* run on the device) -------------
enum class PackLayout : uint8_t { kUniform = 0, kMixed3 = 1 };
constexpr size_t kMixed3Block = 11;  // 10 x 3-bit + 1 x 2-bit fields per word
inline uint32_t mixed3_q_max(size_t stream_idx) { return stream_idx % kMixed3Block == kMixed3Block - 1 ? 3u : 7u; }

inline int feat_per_word(int bits) {
  if (bits != 1 && bits != 2 && bits != 4)
    throw std::invalid_argument("feat_per_word: bits must be 1, 2 or 4, got " + std::to_string(bits));
  return 32 / bits;
}

struct PackedBuffer {
  std::vector<uint32_t> words;
  PackLayout layout = PackLayout::kUniform;
  int bits = 0;
  size_t logical_len = 0;
  size_t word_count() const { return words.size(); }
  // bounds-checked read of code idx (LSB-first fields; Mixed3 slot 10 is the 2-bit field)
  uint32_t get(size_t idx) const {
    if (idx >= logical_len)
      throw std::out_of_range("PackedBuffer::get: index " + std::to_string(idx) + " out of bounds (logical_len " +
                              std::to_string(logical_len) + ")");
    if (layout == PackLayout::kMixed3) {
      const uint32_t w = words[idx / kMixed3Block];
      const size_t pos = idx % kMixed3Block;
      return pos == kMixed3Block - 1 ? w >> 30 : (w >> (3 * pos)) & 7u;
    }
    const size_t fpw = (size_t)(32 / bits);
    return (words[idx / fpw] >> (bits * (idx % fpw))) & ((1u << bits) - 1u);
  }
};

namespace b200 {
// codes -> words on the device (kvmix_pack: the reference's range errors, bitpack.cpp:23-46)
inline PackedBuffer device_pack(std::span<const uint32_t> codes, int bits) {
  PackedBuffer buf;
  buf.layout = bits == 3 ? PackLayout::kMixed3 : PackLayout::kUniform;
  buf.bits = bits;
  buf.logical_len = codes.size();
  const size_t nw = kvmix_packed_word_count(codes.size(), bits);
  DevBuf dc(std::max<size_t>(codes.size(), 1) * 4), dw(std::max<size_t>(nw, 1) * 4);
  if (!codes.empty()) dc.upload(codes.data(), codes.size() * 4);
  check(kvmix_pack(dc.get<uint32_t>(), codes.size(), bits, dw.get<uint32_t>(), nullptr));
  buf.words.resize(nw);
  if (nw) dw.download(buf.words.data(), nw * 4);
  return buf;
}
}  // namespace b200

inline PackedBuffer pack_uniform(std::span<const uint32_t> codes, int bits) {
  feat_per_word(bits);
  return b200::device_pack(codes, bits);
}
inline PackedBuffer pack_mixed3(std::span<const uint32_t> codes) { return b200::device_pack(codes, 3); }
inline uint32_t unpack_uniform(const PackedBuffer& buf, size_t idx) {
  if (buf.layout != PackLayout::kUniform)
    throw std::invalid_argument("unpack_uniform: buffer does not use a uniform layout");
  return buf.get(idx);
}
inline uint32_t unpack_mixed3(const PackedBuffer& buf, size_t idx) {
  if (buf.layout != PackLayout::kMixed3)
    throw std::invalid_argument("unpack_mixed3: buffer does not use the mixed 3-bit layout");
  return buf.get(idx);
}

// Streaming writer (host): codes straight into the word array, range-checked per field.
class PackedWriter {
 public:
  static PackedWriter uniform(int bits) {
    feat_per_word(bits);
    return PackedWriter(PackLayout::kUniform, bits);
  }
  static PackedWriter mixed3() { return PackedWriter(PackLayout::kMixed3, 3); }
  void push(uint32_t code) {
    if (layout_ == PackLayout::kUniform) {
      const uint32_t qm = (1u << bits_) - 1u;
      if (code > qm)
        throw std::invalid_argument("pack_uniform: code " + std::to_string(code) + " at index " + std::to_string(n_) +
                                    " exceeds " + std::to_string(qm) + " for " + std::to_string(bits_) +
                                    "-bit fields");
      const size_t f = n_ % (size_t)(32 / bits_);
      if (f == 0) words_.push_back(0u);
      words_.back() |= code << (bits_ * f);
    } else {
      const size_t pos = n_ % kMixed3Block;
      const uint32_t qm = mixed3_q_max(n_);
      if (code > qm)
        throw std::invalid_argument("pack_mixed3: code " + std::to_string(code) + " in block " +
                                    std::to_string(n_ / kMixed3Block) + " at intra-block index " +
                                    std::to_string(pos) + " exceeds " + std::to_string(qm));
      if (pos == 0) words_.push_back(0u);
      words_.back() |= code << (pos == kMixed3Block - 1 ? 30u : (uint32_t)(3 * pos));
    }
    ++n_;
  }
  size_t size() const { return n_; }
  PackedBuffer finish() && {
    PackedBuffer b;
    b.words = std::move(words_);
    b.layout = layout_;
    b.bits = bits_;
    b.logical_len = n_;
    return b;
  }

 private:
  PackedWriter(PackLayout l, int b) : layout_(l), bits_(b) {}
  std::vector<uint32_t> words_;
  PackLayout layout_;
  int bits_;
  size_t n_ = 0;
};

// ---- quant.cpp:8-75: scalar group helpers (host, bit-exact with the device kernels) --------
inline int q_max_for_bits(int bits) {
  if (bits < 1 || bits > 4) throw std::invalid_argument("unsupported bit width " + std::to_string(bits));
  return bits == 3 ? 7 : (1 << bits) - 1;
}
inline float mixed3_wide_scale(float scale) { return scale * (7.0f / 3.0f); }

// min / max in order from the first element; binary16 (scale, min) of the unrounded extrema
inline GroupMeta compute_meta(std::span<const float> group, int q_max) {
  if (group.empty()) throw std::invalid_argument("compute_meta: empty group");
  if (q_max < 1) throw std::invalid_argument("compute_meta: q_max must be >= 1");
  float mn = group[0], mx = group[0];
  for (float v : group) {
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  volatile float range = mx - mn;  // (no contraction with the division)
  return GroupMeta{round_through_half(range / (float)q_max), round_through_half(mn)};
}
namespace b200 {
// lround((x - min) / s) clamped to [0, q_max]; x86-64 lround gives LONG_MIN for NaN / huge
inline uint32_t encode_code(float x, float scale, float minv, long q_max) {
  if (scale == 0.0f) return 0u;
  volatile float d = x - minv;
  const float v = d / scale;
  if (!(std::fabs(v) < 0x1p63f)) return 0u;
  const long q = std::lround(v);
  return (uint32_t)(q < 0 ? 0 : q > q_max ? q_max : q);
}
inline float decode_code(uint32_t code, float scale, float minv) {
  volatile float p = (float)code * scale;  // rounded product, then the add (no FMA)
  return p + minv;
}
}  // namespace b200
inline std::vector<uint32_t> quantize_group(std::span<const float> group, const GroupMeta& meta, int q_max) {
  std::vector<uint32_t> codes(group.size());
  for (size_t i = 0; i < group.size(); ++i) codes[i] = b200::encode_code(group[i], meta.scale, meta.min_val, q_max);
  return codes;
}
inline std::vector<float> dequantize_group(std::span<const uint32_t> codes, const GroupMeta& meta) {
  std::vector<float> out(codes.size());
  for (size_t i = 0; i < codes.size(); ++i) out[i] = b200::decode_code(codes[i], meta.scale, meta.min_val);
  return out;
}

// QuantizedGroups (quant.hpp:64-77): meta + packed codes; meta_half keeps the binary16 pairs
// the device produced (the KVQG payload).
struct QuantizedGroups {
  std::vector<GroupMeta> meta;
  PackedBuffer codes;
  std::vector<uint16_t> meta_half;  // {scale, min} pairs, KVQG order
  QuantSpec spec;
  TensorShape shape;
  size_t group_count() const { return meta.size(); }
  // the normative address maps (quant.cpp:77-95)
  size_t stream_index(int bi, int hi, int ti, int di) const {
    if (spec.grouping == Grouping::kPerChannelKey)
      return (((size_t)bi * shape.nh + hi) * shape.d + di) * shape.t + ti;
    return (((size_t)bi * shape.nh + hi) * shape.t + ti) * shape.d + di;
  }
  size_t meta_index(int bi, int hi, int ti, int di) const {
    const int gs = spec.group_size;
    if (spec.grouping == Grouping::kPerChannelKey)
      return (((size_t)bi * shape.nh + hi) * shape.d + di) * (size_t)(shape.t / gs) + ti / gs;
    return (((size_t)bi * shape.nh + hi) * shape.t + ti) * (size_t)((shape.d + gs - 1) / gs) + di / gs;
  }
  // one element read back (quant.cpp:97-100): Mixed3 narrow slots decode with scale * 7/3
  float value_at(int bi, int hi, int ti, int di) const {
    const size_t si = stream_index(bi, hi, ti, di);
    const GroupMeta& m = meta[meta_index(bi, hi, ti, di)];
    const bool narrow = spec.bits == 3 && si % kMixed3Block == kMixed3Block - 1;
    return b200::decode_code(codes.get(si), narrow ? mixed3_wide_scale(m.scale) : m.scale, m.min_val);
  }
};

// KVQG (quant.hpp:82-89, quant.cpp:148-207), little-endian
namespace b200 {
template <typename T>
inline void put_le(std::vector<uint8_t>& o, T v) {
  uint8_t b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));
  o.insert(o.end(), b, b + sizeof(T));
}
template <typename T>
inline T take_le(std::span<const uint8_t> in, size_t& off, const char* who) {
  if (off + sizeof(T) > in.size()) throw std::runtime_error(std::string(who) + ": truncated buffer");
  T v;
  std::memcpy(&v, in.data() + off, sizeof(T));
  off += sizeof(T);
  return v;
}
}  // namespace b200

inline std::vector<uint8_t> serialize_quantized_groups(const QuantizedGroups& qg) {
  std::vector<uint8_t> o;
  o.reserve(48 + qg.meta.size() * 4 + qg.codes.words.size() * 4);
  o.insert(o.end(), {'K', 'V', 'Q', 'G'});
  b200::put_le<uint8_t>(o, 1);
  b200::put_le<uint8_t>(o, (uint8_t)qg.spec.bits);
  b200::put_le<uint8_t>(o, (uint8_t)qg.spec.grouping);
  b200::put_le<uint8_t>(o, (uint8_t)qg.codes.layout);
  for (uint32_t x : {(uint32_t)qg.spec.group_size, (uint32_t)qg.shape.b, (uint32_t)qg.shape.nh, (uint32_t)qg.shape.t,
                     (uint32_t)qg.shape.d})
    b200::put_le<uint32_t>(o, x);
  b200::put_le<uint64_t>(o, qg.meta.size());
  b200::put_le<uint64_t>(o, qg.codes.logical_len);
  b200::put_le<uint64_t>(o, qg.codes.words.size());
  for (const GroupMeta& m : qg.meta) {
    b200::put_le<uint16_t>(o, half_from_float(m.scale));
    b200::put_le<uint16_t>(o, half_from_float(m.min_val));
  }
  for (uint32_t w : qg.codes.words) b200::put_le<uint32_t>(o, w);
  return o;
}

inline QuantizedGroups deserialize_quantized_groups(std::span<const uint8_t> in) {
  static const char* who = "deserialize_quantized_groups";
  if (in.size() < 4 || std::memcmp(in.data(), "KVQG", 4) != 0) throw std::runtime_error(std::string(who) + ": bad magic");
  size_t off = 4;
  const uint8_t version = b200::take_le<uint8_t>(in, off, who);
  if (version != 1) throw std::runtime_error(std::string(who) + ": unsupported version " + std::to_string(version));
  QuantizedGroups qg;
  qg.spec.bits = b200::take_le<uint8_t>(in, off, who);
  qg.spec.grouping = (Grouping)b200::take_le<uint8_t>(in, off, who);
  qg.codes.layout = (PackLayout)b200::take_le<uint8_t>(in, off, who);
  qg.codes.bits = qg.spec.bits;
  qg.spec.group_size = (int)b200::take_le<uint32_t>(in, off, who);
  qg.shape.b = (int)b200::take_le<uint32_t>(in, off, who);
  qg.shape.nh = (int)b200::take_le<uint32_t>(in, off, who);
  qg.shape.t = (int)b200::take_le<uint32_t>(in, off, who);
  qg.shape.d = (int)b200::take_le<uint32_t>(in, off, who);
  const uint64_t ng = b200::take_le<uint64_t>(in, off, who);
  qg.codes.logical_len = b200::take_le<uint64_t>(in, off, who);
  const uint64_t nw = b200::take_le<uint64_t>(in, off, who);
  qg.meta.resize(ng);
  qg.meta_half.resize(2 * ng);
  for (uint64_t i = 0; i < ng; ++i) {
    qg.meta_half[2 * i] = b200::take_le<uint16_t>(in, off, who);
    qg.meta_half[2 * i + 1] = b200::take_le<uint16_t>(in, off, who);
    qg.meta[i] = GroupMeta{float_from_half(qg.meta_half[2 * i]), float_from_half(qg.meta_half[2 * i + 1])};
  }
  qg.codes.words.resize(nw);
  for (uint64_t i = 0; i < nw; ++i) qg.codes.words[i] = b200::take_le<uint32_t>(in, off, who);
  if (off != in.size()) throw std::runtime_error(std::string(who) + ": trailing bytes");
  return qg;
}

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
  q.codes.words.resize(nw);
  q.codes.layout = spec.bits == 3 ? PackLayout::kMixed3 : PackLayout::kUniform;
  q.codes.bits = spec.bits;
  q.codes.logical_len = x.size();
  q.meta_half.resize(2 * ng);
  if (nw) dw.download(q.codes.words.data(), nw * 4);
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

  // key_segments()/value_segments() (cache.hpp:75-76): one QuantizedGroups per age-out event,
  // exported from the device store in the reference's word order (by value: a host copy)
  std::vector<QuantizedGroups> key_segments() const { return segments(0); }
  std::vector<QuantizedGroups> value_segments() const { return segments(1); }

  // tail reads (cache.hpp:79-86); j indexes tail-local tokens, oldest first
  float key_tail_at(int bi, int hi, int64_t j, int di) const { return tail_at(0, bi, hi, j, di); }
  float value_tail_at(int bi, int hi, int64_t j, int di) const { return tail_at(1, bi, hi, j, di); }
  // whole tail, [token][b][h][d] fp32 (the KVCD tail payload)
  std::vector<float> tail(int side) const {
    const int64_t n = side ? value_tail_tokens() : key_tail_tokens();
    std::vector<float> out((size_t)n * b_ * nh_ * d_);
    if (!out.empty()) {
      b200::DevBuf d(out.size() * 4);
      b200::check(kvmix_cache_export_tail(h_, side, d.get<float>(), nullptr));
      b200::cuda(cudaDeviceSynchronize(), "export tail");
      d.download(out.data(), out.size() * 4);
    }
    return out;
  }

  // Versioned binary state dump (cache.cpp:190-249): byte-identical to the reference's
  void dump(std::ostream& os) const {
    auto pod = [&os](auto v) { os.write(reinterpret_cast<const char*>(&v), sizeof(v)); };
    os.write("KVCD", 4);
    pod((uint8_t)1);
    pod((int32_t)cfg_.layer_index);
    pod((uint8_t)cfg_.key_bits);
    pod((uint8_t)cfg_.value_bits);
    pod((float)cfg_.key_rpc_ratio);
    pod((float)cfg_.value_rpc_ratio);
    pod((uint32_t)cfg_.group_size);
    pod((uint32_t)b_);
    pod((uint32_t)nh_);
    pod((uint32_t)d_);
    pod((int64_t)key_tail_tokens());
    pod((int64_t)value_tail_tokens());
    pod((int64_t)quantized_key_tokens());
    pod((int64_t)quantized_value_tokens());
    for (int side = 0; side < 2; ++side) {
      const std::vector<QuantizedGroups> segs = segments(side);
      pod((uint32_t)segs.size());
      for (const QuantizedGroups& q : segs) {
        const std::vector<uint8_t> bytes = serialize_quantized_groups(q);
        pod((uint64_t)bytes.size());
        os.write(reinterpret_cast<const char*>(bytes.data()), (std::streamsize)bytes.size());
      }
    }
    for (int side = 0; side < 2; ++side) {
      const std::vector<float> t = tail(side);
      pod((uint64_t)t.size());
      os.write(reinterpret_cast<const char*>(t.data()), (std::streamsize)(t.size() * 4));
    }
  }

  // KVLayerCache::load (cache.cpp:251-281): segments imported in order, then the tails
  static KVLayerCache load(std::istream& is, int64_t capacity_tokens = 0, kvmix_dtype tail_dtype = KVMIX_F32) {
    auto pod = [&is](auto& v) {
      is.read(reinterpret_cast<char*>(&v), sizeof(v));
      if (!is) throw std::runtime_error("KVLayerCache::load: truncated stream");
    };
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "KVCD", 4) != 0) throw std::runtime_error("KVLayerCache::load: bad magic");
    uint8_t version = 0, kb = 0, vb = 0;
    pod(version);
    if (version != 1) throw std::runtime_error("KVLayerCache::load: unsupported version " + std::to_string(version));
    LayerQuantConfig cfg;
    int32_t layer = 0;
    uint32_t gs = 0, b = 0, nh = 0, d = 0;
    int64_t cnt[4];
    pod(layer);
    pod(kb);
    pod(vb);
    pod(cfg.key_rpc_ratio);
    pod(cfg.value_rpc_ratio);
    pod(gs);
    pod(b);
    pod(nh);
    pod(d);
    for (int64_t& c : cnt) pod(c);
    cfg.layer_index = layer;
    cfg.key_bits = kb;
    cfg.value_bits = vb;
    cfg.group_size = (int)gs;
    std::vector<QuantizedGroups> segs[2];
    for (int side = 0; side < 2; ++side) {
      uint32_t n = 0;
      pod(n);
      for (uint32_t i = 0; i < n; ++i) {
        uint64_t len = 0;
        pod(len);
        std::vector<uint8_t> bytes(len);
        is.read(reinterpret_cast<char*>(bytes.data()), (std::streamsize)len);
        if (!is) throw std::runtime_error("KVLayerCache::load: truncated segment");
        segs[side].push_back(deserialize_quantized_groups(bytes));
      }
    }
    std::vector<float> tails[2];
    for (int side = 0; side < 2; ++side) {
      uint64_t n = 0;
      pod(n);
      tails[side].resize(n);
      is.read(reinterpret_cast<char*>(tails[side].data()), (std::streamsize)(n * 4));
      if (!is) throw std::runtime_error("KVLayerCache::load: truncated tail");
    }
    const int64_t total = cnt[2] + cnt[0];
    KVLayerCache c(cfg, (int)b, (int)nh, (int)d, std::max<int64_t>(capacity_tokens, std::max<int64_t>(total, 1)),
                   tail_dtype);
    for (int side = 0; side < 2; ++side) {
      for (const QuantizedGroups& q : segs[side]) {
        b200::DevBuf w(std::max<size_t>(q.codes.words.size(), 1) * 4), m(std::max<size_t>(q.meta.size(), 1) * 4);
        std::vector<uint16_t> mh(2 * q.meta.size());
        for (size_t i = 0; i < q.meta.size(); ++i) {
          mh[2 * i] = half_from_float(q.meta[i].scale);
          mh[2 * i + 1] = half_from_float(q.meta[i].min_val);
        }
        if (!q.codes.words.empty()) w.upload(q.codes.words.data(), q.codes.words.size() * 4);
        if (!mh.empty()) m.upload(mh.data(), mh.size() * 2);
        b200::check(kvmix_cache_import_segment(c.h_, side, q.shape.t, w.get<uint32_t>(), m.get<uint16_t>(), nullptr));
      }
      const int64_t tl = cnt[side];
      if (tl > 0) {
        b200::DevBuf t(tails[side].size() * 4);
        t.upload(tails[side].data(), tails[side].size() * 4);
        b200::check(kvmix_cache_import_tail(c.h_, side, t.get<float>(), tl, nullptr));
      }
    }
    b200::cuda(cudaDeviceSynchronize(), "load");
    return c;
  }

 private:
  int64_t counter(int i) const {
    int64_t c[7];
    b200::check(kvmix_cache_counters(h_, c));
    return c[i];
  }
  std::vector<QuantizedGroups> segments(int side) const {
    std::vector<QuantizedGroups> out;
    const int64_t n = counter(5 + side);
    const int bits = side ? cfg_.value_bits : cfg_.key_bits;
    for (int64_t i = 0; i < n; ++i) {
      int64_t info[3];  // {t, words, groups}
      b200::check(kvmix_cache_segment_info(h_, side, (int)i, info));
      b200::DevBuf w(std::max<int64_t>(info[1], 1) * 4), m(std::max<int64_t>(info[2], 1) * 4);
      b200::check(kvmix_cache_export_segment(h_, side, (int)i, w.get<uint32_t>(), m.get<uint16_t>(), nullptr));
      b200::cuda(cudaDeviceSynchronize(), "export segment");
      QuantizedGroups q;
      q.spec = QuantSpec{bits, side ? Grouping::kPerTokenValue : Grouping::kPerChannelKey, cfg_.group_size};
      q.shape = TensorShape{b_, nh_, (int)info[0], d_};
      q.codes.layout = bits == 3 ? PackLayout::kMixed3 : PackLayout::kUniform;
      q.codes.bits = bits;
      q.codes.logical_len = q.shape.elems();
      q.codes.words.resize((size_t)info[1]);
      q.meta_half.resize(2 * (size_t)info[2]);
      if (info[1]) w.download(q.codes.words.data(), (size_t)info[1] * 4);
      if (info[2]) m.download(q.meta_half.data(), (size_t)info[2] * 4);
      q.meta.resize((size_t)info[2]);
      for (size_t g = 0; g < q.meta.size(); ++g)
        q.meta[g] = GroupMeta{b200::half_to_float(q.meta_half[2 * g]), b200::half_to_float(q.meta_half[2 * g + 1])};
      out.push_back(std::move(q));
    }
    return out;
  }
  float tail_at(int side, int bi, int hi, int64_t j, int di) const {
    const int64_t n = side ? value_tail_tokens() : key_tail_tokens();
    if (j < 0 || j >= n || bi < 0 || bi >= b_ || hi < 0 || hi >= nh_ || di < 0 || di >= d_)
      throw std::out_of_range("KVLayerCache: tail index out of range");
    return tail(side)[((size_t)j * b_ * nh_ + (size_t)bi * nh_ + hi) * d_ + di];
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
