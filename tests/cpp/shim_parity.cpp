// C++ host parity through the shim (include/kvmix_b200.hpp): the reference's hot-path API
// (kvmix::KVLayerCache / attend / quantize_key_tensor, written exactly as the reference's
// callers write it) backed by the B200 kernels, checked against the reference library
// itself (oracle/_ref/libkvmix_ref.so, its extern "C" driver, loaded with dlopen so its own
// kvmix:: symbols stay private). Test infrastructure only. Exit code 0 = pass.
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
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
  R.cache_destroy(ref);
  std::printf("cache K%dV%d r=%.1f B%d H%d D%d: %lld tokens (capacity grown to %lld) ok\n", kb, vb, r, B, H, D,
              (long long)dev.total_tokens(), (long long)dev.capacity_tokens());
}

void quant_case(Ref& R, int bits, bool key) {
  const int B = 1, H = 4, T = 128, D = 128;
  kvmix::Tensor4f x = random_tensor(R, 5 + bits, B, H, T, D);
  const kvmix::QuantSpec spec{bits, key ? kvmix::Grouping::kPerChannelKey : kvmix::Grouping::kPerTokenValue, 32};
  const kvmix::QuantizedGroups q = key ? kvmix::quantize_key_tensor(x, spec) : kvmix::quantize_value_tensor(x, spec);
  std::vector<uint32_t> rw(q.words.size() + 16);
  std::vector<uint16_t> rm(q.meta_half.size() + 16);
  uint64_t nw = 0, ng = 0;
  R.quantize(key ? 0 : 1, x.data.data(), B, H, T, D, bits, 32, rw.data(), rm.data(), &nw, &ng);
  CHECK(nw == q.words.size() && ng == q.meta.size(), "quantize %d-bit counts", bits);
  CHECK(std::memcmp(rw.data(), q.words.data(), nw * 4) == 0, "quantize %d-bit %s words differ", bits, key ? "key" : "value");
  CHECK(std::memcmp(rm.data(), q.meta_half.data(), ng * 4) == 0, "quantize %d-bit meta differ", bits);
  std::printf("quantize_%s_tensor %d-bit: %zu words, %zu groups bit-exact\n", key ? "key" : "value", bits, q.words.size(),
              q.meta.size());
}

}  // namespace

int main(int argc, char** argv) {
  const char* ref_path = argc > 1 ? argv[1] : "oracle/_ref/libkvmix_ref.so";
  try {
    Ref R(ref_path);
    for (int bits : {2, 3, 4})
      for (bool key : {true, false}) quant_case(R, bits, key);
    cache_case(R, 2, 2, 0.1f, 2, 4, 128, {300, 1, 1, 97, 1, 1, 1, 40});
    cache_case(R, 3, 4, 0.2f, 1, 4, 128, {500, 1, 1, 1});
    cache_case(R, 4, 2, 0.1f, 2, 2, 64, {150, 33, 1, 1});
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
