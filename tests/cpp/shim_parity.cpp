// C++ host parity through the shim (include/kvmix_b200.hpp): the reference's hot-path API
// (kvmix::KVLayerCache / attend / quantize_key_tensor, written exactly as the reference's
// callers write it) backed by the B200 kernels, checked against the reference library
// itself (oracle/_ref/libkvmix_ref.so, its extern "C" driver, loaded with dlopen so its own
// kvmix:: symbols stay private). Test infrastructure only. Exit code 0 = pass.
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <cstring>
#include <string>
#include <vector>

#include "kvmix_b200.hpp"

namespace {

struct Ref {
  void* so = nullptr;
  void (*random_h16)(uint64_t, size_t, float, float, float*);
  int (*quantize)(int, const float*, int, int, int, int, int, int, uint32_t*, uint16_t*, uint64_t*, uint64_t*);
  void* (*cache_create)(int, int, float, float, int, int, int, int);
  void (*cache_destroy)(void*);
  int (*cache_append)(void*, const float*, const float*, int);
  void (*cache_counters)(void*, int64_t*);
  void (*cache_memory)(void*, uint64_t*, double*);
  int (*cache_snapshot)(void*, float*, float*);
  int (*attend)(void*, const float*, int, int, float*, double*);
  int (*cache_segment)(void*, int, int, int64_t*, uint32_t*, uint16_t*);
  int (*cache_dump)(void*, uint8_t*, uint64_t, uint64_t*);
  int (*pack)(const uint32_t*, size_t, int, uint32_t*, size_t*) = nullptr;
  template <typename F>
  void sym(F& f, const char* n) {
    f = reinterpret_cast<F>(dlsym(so, n));
    if (!f) throw std::runtime_error(std::string("missing ") + n);
  }
  explicit Ref(const char* path) {
    so = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!so) throw std::runtime_error(dlerror());
    sym(random_h16, "ref_random_h16");
    sym(quantize, "ref_quantize");
    sym(cache_create, "ref_cache_create");
    sym(cache_destroy, "ref_cache_destroy");
    sym(cache_append, "ref_cache_append");
    sym(cache_counters, "ref_cache_counters");
    sym(cache_memory, "ref_cache_memory");
    sym(cache_snapshot, "ref_cache_snapshot");
    sym(attend, "ref_attend");
    sym(cache_segment, "ref_cache_segment");
    sym(cache_dump, "ref_cache_dump");
    sym(pack, "ref_pack");
  }
};

int failures = 0;
#define CHECK(cond, ...)                  \
  do {                                    \
    if (!(cond)) {                        \
      ++failures;                         \
      std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);           \
      std::printf("\n");                  \
    }                                     \
  } while (0)

kvmix::Tensor4f random_tensor(Ref& R, uint64_t seed, int b, int nh, int t, int d) {
  kvmix::Tensor4f x(b, nh, t, d);
  R.random_h16(seed, x.size(), 1.0f, 0.0f, x.data.data());
  return x;
}

void cache_case(Ref& R, int kb, int vb, float r, int B, int H, int D, const std::vector<int>& chunks) {
  kvmix::LayerQuantConfig cfg;
  cfg.key_bits = kb;
  cfg.value_bits = vb;
  cfg.key_rpc_ratio = r;
  cfg.value_rpc_ratio = r;
  kvmix::KVLayerCache dev(cfg, B, H, D, /*capacity_tokens=*/64);  // small: append() has to grow it
  void* ref = R.cache_create(kb, vb, r, r, 32, B, H, D);
  uint64_t seed = 1000 * kb + 10 * vb;
  for (int t : chunks) {
    kvmix::Tensor4f k = random_tensor(R, seed++, B, H, t, D), v = random_tensor(R, seed++, B, H, t, D);
    dev.append(k, v);
    R.cache_append(ref, k.data.data(), v.data.data(), t);
  }
  int64_t rc[7];
  R.cache_counters(ref, rc);
  CHECK(dev.total_tokens() == rc[0] && dev.key_tail_tokens() == rc[1] && dev.value_tail_tokens() == rc[2] &&
            dev.quantized_key_tokens() == rc[3] && dev.quantized_value_tokens() == rc[4],
        "K%dV%d counters differ", kb, vb);
  uint64_t rm[5];
  double ratio;
  R.cache_memory(ref, rm, &ratio);
  const kvmix::MemoryReport m = dev.memory_usage();
  CHECK(m.packed_payload_bits == rm[0] && m.metadata_bits == rm[1] && m.tail_bits == rm[2] && m.total_bits == rm[3],
        "K%dV%d MemoryReport differs", kb, vb);
  // snapshot_dequantized: bit-exact
  auto [ks, vs] = dev.snapshot_dequantized();
  std::vector<float> rk(ks.size()), rv(vs.size());
  R.cache_snapshot(ref, rk.data(), rv.data());
  CHECK(std::memcmp(ks.data.data(), rk.data(), rk.size() * 4) == 0, "K%dV%d key snapshot differs", kb, vb);
  CHECK(std::memcmp(vs.data.data(), rv.data(), rv.size() * 4) == 0, "K%dV%d value snapshot differs", kb, vb);
  float vmax = 0.f;
  for (float x : rv) vmax = std::fmax(vmax, std::fabs(x));
  // attend vs the reference's fused attend: |diff| <= 4e-5 max|V| (tests/test_attention_gpu.py)
  for (int tq : {1, 2}) {
    kvmix::Tensor4f q = random_tensor(R, 77 + tq, B, H, tq, D);
    const kvmix::AttentionOutput o = kvmix::attend(q, dev);
    std::vector<float> ro(o.output.size());
    double rcs = 0.0;
    R.attend(ref, q.data.data(), tq, 0, ro.data(), &rcs);
    float err = 0.f;
    for (size_t i = 0; i < ro.size(); ++i) err = std::fmax(err, std::fabs(o.output.data[i] - ro[i]));
    CHECK(err <= 4e-5f * vmax, "K%dV%d t=%d attend err %g (max|V| %g)", kb, vb, tq, err, vmax);
    CHECK(std::fabs(o.scores_checksum - rcs) <= 1e-4 * (1.0 + std::fabs(rcs)), "K%dV%d checksum %.9g vs %.9g", kb, vb,
          o.scores_checksum, rcs);
  }
  // key_segments / value_segments (cache.hpp:75-76): words and meta equal the reference's
  for (int side = 0; side < 2; ++side) {
    const std::vector<kvmix::QuantizedGroups> segs = side ? dev.value_segments() : dev.key_segments();
    CHECK((int64_t)segs.size() == (side ? rc[6] : rc[5]), "K%dV%d side %d segment count", kb, vb, side);
    int64_t t0 = 0;
    for (size_t i = 0; i < segs.size(); ++i) {
      int64_t info[3];
      std::vector<uint32_t> rw(segs[i].codes.words.size() + 8);
      std::vector<uint16_t> rm(2 * segs[i].meta.size() + 8);
      R.cache_segment(ref, side, (int)i, info, rw.data(), rm.data());
      CHECK(info[0] == segs[i].shape.t && info[1] == (int64_t)segs[i].codes.words.size() &&
                std::memcmp(rw.data(), segs[i].codes.words.data(), info[1] * 4) == 0 &&
                std::memcmp(rm.data(), segs[i].meta_half.data(), info[2] * 4) == 0,
            "K%dV%d side %d segment %zu differs", kb, vb, side, i);
      // QuantizedGroups::value_at == the snapshot's token (bit-exact)
      const kvmix::Tensor4f& snap = side ? vs : ks;
      for (int probe = 0; probe < 64; ++probe) {
        const int bi = probe % B, hi = (probe / 3) % H, ti = (int)((probe * 7919) % segs[i].shape.t), di = (probe * 31) % D;
        const float a = segs[i].value_at(bi, hi, ti, di), b = snap.at(bi, hi, (int)(t0 + ti), di);
        CHECK(std::memcmp(&a, &b, 4) == 0, "K%dV%d side %d value_at differs", kb, vb, side);
      }
      t0 += segs[i].shape.t;
    }
  }
  // tails: key_tail_at / value_tail_at are the snapshot's last tokens
  for (int64_t j = 0; j < dev.key_tail_tokens(); j += 7) {
    const float a = dev.key_tail_at(B - 1, H - 1, j, D / 2);
    const float b = ks.at(B - 1, H - 1, (int)(dev.quantized_key_tokens() + j), D / 2);
    CHECK(a == b, "K%dV%d key_tail_at(%lld)", kb, vb, (long long)j);
  }
  // dump (cache.cpp:190-249): byte-identical to the reference's; load restores the same state
  {
    std::ostringstream os;
    dev.dump(os);
    const std::string mine = os.str();
    uint64_t len = 0;
    R.cache_dump(ref, nullptr, 0, &len);
    std::string theirs(len, '\0');
    R.cache_dump(ref, reinterpret_cast<uint8_t*>(theirs.data()), len, &len);
    CHECK(mine == theirs, "K%dV%d KVCD dump differs (%zu vs %zu bytes)", kb, vb, mine.size(), theirs.size());
    std::istringstream is(mine);
    kvmix::KVLayerCache back = kvmix::KVLayerCache::load(is);
    std::ostringstream os2;
    back.dump(os2);
    CHECK(os2.str() == mine, "K%dV%d load(dump) round trip differs", kb, vb);
    kvmix::Tensor4f q = random_tensor(R, 99, B, H, 1, D);
    const kvmix::AttentionOutput a = kvmix::attend(q, dev), b = kvmix::attend(q, back);
    CHECK(std::memcmp(a.output.data.data(), b.output.data.data(), a.output.size() * 4) == 0,
          "K%dV%d attend after load differs", kb, vb);
  }
  R.cache_destroy(ref);
  std::printf("cache K%dV%d r=%.1f B%d H%d D%d: %lld tokens (capacity grown to %lld) ok\n", kb, vb, r, B, H, D,
              (long long)dev.total_tokens(), (long long)dev.capacity_tokens());
}

void quant_case(Ref& R, int bits, bool key) {
  const int B = 1, H = 4, T = 128, D = 128;
  kvmix::Tensor4f x = random_tensor(R, 5 + bits, B, H, T, D);
  const kvmix::QuantSpec spec{bits, key ? kvmix::Grouping::kPerChannelKey : kvmix::Grouping::kPerTokenValue, 32};
  const kvmix::QuantizedGroups q = key ? kvmix::quantize_key_tensor(x, spec) : kvmix::quantize_value_tensor(x, spec);
  std::vector<uint32_t> rw(q.codes.words.size() + 16);
  std::vector<uint16_t> rm(q.meta_half.size() + 16);
  uint64_t nw = 0, ng = 0;
  R.quantize(key ? 0 : 1, x.data.data(), B, H, T, D, bits, 32, rw.data(), rm.data(), &nw, &ng);
  CHECK(nw == q.codes.words.size() && ng == q.meta.size(), "quantize %d-bit counts", bits);
  CHECK(std::memcmp(rw.data(), q.codes.words.data(), nw * 4) == 0, "quantize %d-bit %s words differ", bits, key ? "key" : "value");
  CHECK(std::memcmp(rm.data(), q.meta_half.data(), ng * 4) == 0, "quantize %d-bit meta differ", bits);
  std::printf("quantize_%s_tensor %d-bit: %zu words, %zu groups bit-exact\n", key ? "key" : "value", bits, q.codes.words.size(),
              q.meta.size());
}

// bitpack / quant helpers of the reference API (bitpack.hpp, quant.hpp) through the shim
void bitpack_quant_case(Ref& R) {
  std::mt19937 rng(7);
  for (int bits : {1, 2, 3, 4}) {
    for (size_t n : {0u, 1u, 10u, 11u, 12u, 31u, 33u, 1000u}) {
      std::vector<uint32_t> codes(n);
      for (size_t i = 0; i < n; ++i) codes[i] = rng() % (bits == 3 ? kvmix::mixed3_q_max(i) + 1 : (1u << bits));
      kvmix::PackedWriter w = bits == 3 ? kvmix::PackedWriter::mixed3() : kvmix::PackedWriter::uniform(bits);
      for (uint32_t c : codes) w.push(c);
      const kvmix::PackedBuffer host = std::move(w).finish();
      const kvmix::PackedBuffer dev = bits == 3 ? kvmix::pack_mixed3(codes) : kvmix::pack_uniform(codes, bits);
      CHECK(host.words == dev.words && host.logical_len == n, "pack %d-bit n=%zu: device words differ", bits, n);
      std::vector<uint32_t> rw(dev.words.size() + 4);
      size_t rn = 0;
      if (n) R.pack(codes.data(), n, bits, rw.data(), &rn);
      CHECK(!n || (rn == dev.words.size() && std::memcmp(rw.data(), dev.words.data(), rn * 4) == 0),
            "pack %d-bit n=%zu differs from the reference", bits, n);
      for (size_t i = 0; i < n; ++i)
        CHECK((bits == 3 ? kvmix::unpack_mixed3(dev, i) : kvmix::unpack_uniform(dev, i)) == codes[i], "get %zu", i);
      bool threw = false;
      try {
        dev.get(n);
      } catch (const std::out_of_range&) {
        threw = true;
      }
      CHECK(threw, "PackedBuffer::get past the end must throw std::out_of_range");
    }
    bool threw = false;
    try {
      const std::vector<uint32_t> big{0u, bits == 3 ? 8u : (1u << bits)};
      if (bits == 3) kvmix::pack_mixed3(big);
      else kvmix::pack_uniform(big, bits);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw, "%d-bit code out of range must throw std::invalid_argument", bits);
  }
  // compute_meta / quantize_group / dequantize_group vs the device quantizer on one group
  for (int bits : {1, 2, 4}) {
    kvmix::Tensor4f x = random_tensor(R, 300 + bits, 1, 1, 32, 1);
    const kvmix::QuantizedGroups q = kvmix::quantize_key_tensor(x, kvmix::QuantSpec{bits, kvmix::Grouping::kPerChannelKey, 32});
    const kvmix::GroupMeta m = kvmix::compute_meta(x.data, kvmix::q_max_for_bits(bits));
    CHECK(m.scale == q.meta[0].scale && m.min_val == q.meta[0].min_val, "compute_meta %d-bit", bits);
    const std::vector<uint32_t> c = kvmix::quantize_group(x.data, m, kvmix::q_max_for_bits(bits));
    const std::vector<float> d = kvmix::dequantize_group(c, m);
    for (int i = 0; i < 32; ++i) {
      CHECK(c[i] == q.codes.get(i), "quantize_group %d-bit code %d", bits, i);
      const float v = q.value_at(0, 0, i, 0);
      CHECK(std::memcmp(&v, &d[i], 4) == 0, "dequantize_group %d-bit value %d", bits, i);
    }
  }
  // KVQG (quant.cpp:148-207): serialize -> deserialize -> serialize is the identity; bad input throws
  {
    kvmix::Tensor4f x = random_tensor(R, 400, 2, 3, 64, 32);
    for (int bits : {2, 3}) {
      const kvmix::QuantizedGroups q = kvmix::quantize_value_tensor(x, kvmix::QuantSpec{bits, kvmix::Grouping::kPerTokenValue, 32});
      const std::vector<uint8_t> bytes = kvmix::serialize_quantized_groups(q);
      const kvmix::QuantizedGroups back = kvmix::deserialize_quantized_groups(bytes);
      CHECK(kvmix::serialize_quantized_groups(back) == bytes && back.value_at(1, 2, 63, 31) == q.value_at(1, 2, 63, 31),
            "KVQG %d-bit round trip", bits);
      int errs = 0;
      std::vector<uint8_t> bad = bytes;
      bad[0] = 'X';
      try { kvmix::deserialize_quantized_groups(bad); } catch (const std::runtime_error&) { ++errs; }
      bad = bytes;
      bad.pop_back();
      try { kvmix::deserialize_quantized_groups(bad); } catch (const std::runtime_error&) { ++errs; }
      bad = bytes;
      bad.push_back(0);
      try { kvmix::deserialize_quantized_groups(bad); } catch (const std::runtime_error&) { ++errs; }
      CHECK(errs == 3, "KVQG bad magic / truncated / trailing must throw std::runtime_error");
    }
  }
  std::printf("bitpack / group helpers / KVQG through the shim: ok\n");
}

}  // namespace

int main(int argc, char** argv) {
  const char* ref_path = argc > 1 ? argv[1] : "oracle/_ref/libkvmix_ref.so";
  try {
    Ref R(ref_path);
    for (int bits : {2, 3, 4})
      for (bool key : {true, false}) quant_case(R, bits, key);
    bitpack_quant_case(R);
    cache_case(R, 2, 2, 0.1f, 2, 4, 128, {300, 1, 1, 97, 1, 1, 1, 40});
    cache_case(R, 3, 4, 0.2f, 1, 4, 128, {500, 1, 1, 1});
    cache_case(R, 4, 2, 0.1f, 2, 2, 64, {150, 33, 1, 1});
    // the reference's own small head dims (tests use 4..32; harness.hpp:50 / toymodel.hpp:40)
    cache_case(R, 2, 2, 0.2f, 1, 1, 4, {40, 1, 1, 30});
    cache_case(R, 3, 4, 0.2f, 2, 2, 16, {90, 1, 1, 40, 1});
    cache_case(R, 2, 3, 0.1f, 1, 2, 32, {200, 1, 7});
    // the reference's exception types through the shim
    bool threw = false;
    try {
      kvmix::KVLayerCache bad(kvmix::LayerQuantConfig{}, 1, 1, 128);
      bad.append(kvmix::Tensor4f(1, 2, 1, 128), kvmix::Tensor4f(1, 2, 1, 128));
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw, "shape mismatch must throw std::invalid_argument");
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 2;
  }
  std::printf(failures ? "shim parity: %d failure(s)\n" : "shim parity: all checks passed\n", failures);
  return failures ? 1 : 0;
}
