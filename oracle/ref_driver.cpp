// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference library (TEST INFRASTRUCTURE).
//
// oracle/Makefile compiles this file together with the reference hot-path sources
// exactly where they lie (/root/reference/proj/src/{bitpack,quant,cache,attention}.cpp)
// into oracle/_ref/libkvmix_ref.so, using the reference's Release flags
// (-O3 -DNDEBUG, -fopenmp, no -march=native).
// Nothing here re-implements reference logic: every function forwards to the
// reference's public C++ API (include/kvmix/*.hpp) so Python tests and the bench
// CPU leg can call it through ctypes. Only tests/, smoke() and bench.py's
// cpu_baseline / --impl reference legs load this library.
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "kvmix/attention.hpp"
#include "kvmix/cache.hpp"
#include "kvmix/half.hpp"
#include "kvmix/quant.hpp"
#include "kvmix/rng.hpp"

using namespace kvmix;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  return 3;
}

Tensor4f make_tensor(const float* x, int b, int nh, int t, int d) {
  Tensor4f out(b, nh, t, d);
  if (x) std::memcpy(out.data.data(), x, out.data.size() * sizeof(float));
  return out;
}

void copy_groups(const QuantizedGroups& qg, uint32_t* words, uint16_t* meta) {
  if (words) std::memcpy(words, qg.codes.words.data(), qg.codes.words.size() * 4);
  if (meta) {
    for (size_t i = 0; i < qg.meta.size(); ++i) {
      meta[2 * i] = half_from_float(qg.meta[i].scale);
      meta[2 * i + 1] = half_from_float(qg.meta[i].min_val);
    }
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads() { return omp_get_max_threads(); }

uint16_t ref_half_from_float(float f) { return half_from_float(f); }
float ref_float_from_half(uint16_t h) { return float_from_half(h); }
int64_t ref_rpc_target(int64_t n, double r) { return rpc_target(n, r); }

// kvmix::Rng + round_through_half, as tests/helpers.hpp:14-18 and harness.cpp:16-24
void ref_random_h16(uint64_t seed, size_t n, float sigma, float mu, float* out) {
  Rng rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = round_through_half(mu + sigma * static_cast<float>(rng.normal()));
}

int ref_pack(const uint32_t* codes, size_t n, int bits, uint32_t* words, size_t* n_words) {
  try {
    std::span<const uint32_t> s(codes, n);
    PackedBuffer b = bits == 3 ? pack_mixed3(s) : pack_uniform(s, bits);
    std::memcpy(words, b.words.data(), b.words.size() * 4);
    *n_words = b.words.size();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// grouping 0 = per-channel Keys, 1 = per-token Values
int ref_quantize(int grouping, const float* x, int B, int H, int T, int D, int bits, int gs,
                 uint32_t* words, uint16_t* meta, uint64_t* n_words, uint64_t* n_groups) {
  try {
    Tensor4f t = make_tensor(x, B, H, T, D);
    QuantSpec spec{bits, grouping == 0 ? Grouping::kPerChannelKey : Grouping::kPerTokenValue, gs};
    QuantizedGroups qg = grouping == 0 ? quantize_key_tensor(t, spec) : quantize_value_tensor(t, spec);
    if (n_words) *n_words = qg.codes.words.size();
    if (n_groups) *n_groups = qg.meta.size();
    copy_groups(qg, words, meta);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// serialize_quantized_groups of the tensor quantizer's output (KVQG bytes, quant.cpp:148-170)
int ref_quantize_serialized(int grouping, const float* x, int B, int H, int T, int D, int bits,
                            int gs, uint8_t* out, uint64_t cap, uint64_t* len) {
  try {
    Tensor4f t = make_tensor(x, B, H, T, D);
    QuantSpec spec{bits, grouping == 0 ? Grouping::kPerChannelKey : Grouping::kPerTokenValue, gs};
    QuantizedGroups qg = grouping == 0 ? quantize_key_tensor(t, spec) : quantize_value_tensor(t, spec);
    std::vector<uint8_t> bytes = serialize_quantized_groups(qg);
    *len = bytes.size();
    if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- KVLayerCache ----
void* ref_cache_create(int kbits, int vbits, float rk, float rv, int gs, int B, int H, int D) {
  try {
    LayerQuantConfig c;
    c.key_bits = kbits;
    c.value_bits = vbits;
    c.key_rpc_ratio = rk;
    c.value_rpc_ratio = rv;
    c.group_size = gs;
    return new KVLayerCache(c, B, H, D);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_cache_destroy(void* h) { delete static_cast<KVLayerCache*>(h); }

int ref_cache_append(void* h, const float* k, const float* v, int t) {
  try {
    auto* c = static_cast<KVLayerCache*>(h);
    c->append(make_tensor(k, c->batch(), c->heads(), t, c->head_dim()),
              make_tensor(v, c->batch(), c->heads(), t, c->head_dim()));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// out: total, key_tail, value_tail, quant_keys, quant_values, n_key_segs, n_value_segs
void ref_cache_counters(void* h, int64_t* out) {
  auto* c = static_cast<KVLayerCache*>(h);
  out[0] = c->total_tokens();
  out[1] = c->key_tail_tokens();
  out[2] = c->value_tail_tokens();
  out[3] = c->quantized_key_tokens();
  out[4] = c->quantized_value_tokens();
  out[5] = static_cast<int64_t>(c->key_segments().size());
  out[6] = static_cast<int64_t>(c->value_segments().size());
}

// out: payload, meta, tail, total, baseline bits; ratio
void ref_cache_memory(void* h, uint64_t* out, double* ratio) {
  MemoryReport r = static_cast<KVLayerCache*>(h)->memory_usage();
  out[0] = r.packed_payload_bits;
  out[1] = r.metadata_bits;
  out[2] = r.tail_bits;
  out[3] = r.total_bits;
  out[4] = r.fp16_baseline_bits;
  *ratio = r.compression_ratio;
}

int ref_cache_snapshot(void* h, float* keys, float* values) {
  try {
    auto [k, v] = static_cast<KVLayerCache*>(h)->snapshot_dequantized();
    std::memcpy(keys, k.data.data(), k.data.size() * 4);
    std::memcpy(values, v.data.data(), v.data.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// segment export: side 0 = keys, 1 = values. info: t, n_words, n_groups
int ref_cache_segment(void* h, int side, int idx, int64_t* info, uint32_t* words, uint16_t* meta) {
  try {
    auto* c = static_cast<KVLayerCache*>(h);
    const auto& segs = side == 0 ? c->key_segments() : c->value_segments();
    const QuantizedGroups& qg = segs.at(static_cast<size_t>(idx));
    info[0] = qg.shape.t;
    info[1] = static_cast<int64_t>(qg.codes.words.size());
    info[2] = static_cast<int64_t>(qg.meta.size());
    copy_groups(qg, words, meta);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// KVCD dump (cache.cpp:229-249)
int ref_cache_dump(void* h, uint8_t* out, uint64_t cap, uint64_t* len) {
  try {
    std::ostringstream os;
    static_cast<KVLayerCache*>(h)->dump(os);
    const std::string s = os.str();
    *len = s.size();
    if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// fused attend (attention.cpp:161-166) or reference_attend (:168-211); q [B,H,t,D]
int ref_attend(void* h, const float* q, int t, int reference, float* out, double* checksum) {
  try {
    auto* c = static_cast<KVLayerCache*>(h);
    Tensor4f qt = make_tensor(q, c->batch(), c->heads(), t, c->head_dim());
    AttentionOutput o = reference ? reference_attend(qt, *c) : attend(qt, *c);
    std::memcpy(out, o.output.data.data(), o.output.data.size() * 4);
    *checksum = o.scores_checksum;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
