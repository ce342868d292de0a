// capi.cu -- the extern "C" boundary (include/kvmix_b200.h): argument validation with the
// reference's error semantics, status codes + thread-local messages, cache lifecycle.
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>

#include <map>
#include <mutex>
#include <string>

#include "attention.cuh"

namespace kvb {

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

namespace {
std::mutex g_names_mu;
std::map<std::string, uint64_t>& kernel_names() {
  static std::map<std::string, uint64_t> m;
  return m;
}
}  // namespace

void count_kernel(const char* name) {
  std::lock_guard<std::mutex> lk(g_names_mu);
  ++kernel_names()[name];
}

void quantize(kvmix_grouping grouping, const void* x, kvmix_dtype dt, int B, int H, int T, int D, int bits, int gs,
              uint32_t* words, uint16_t* meta, cudaStream_t st);
void dequantize(kvmix_grouping grouping, const uint32_t* words, const uint16_t* meta, int B, int H, int T, int D,
                int bits, int gs, float* out, cudaStream_t st);
bool set_knob(const char* name, int v);
void request_pdl(bool on);
void pack(const uint32_t* codes, size_t n, int bits, uint32_t* words, cudaStream_t st);
void unpack(const uint32_t* words, size_t n, int bits, uint32_t* codes, cudaStream_t st);

namespace {
thread_local std::string g_err;

template <typename F>
kvmix_status guard(F&& f) {
  try {
    f();
    return KVMIX_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return KVMIX_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KVMIX_RUNTIME_ERROR;
  }
}

// LayerQuantConfig::validate (cache.cpp:14-28), same messages
void validate(const kvmix_layer_config& c) {
  const std::string L = "layer " + std::to_string(c.layer_index);
  if (c.key_bits < 2 || c.key_bits > 4 || c.value_bits < 2 || c.value_bits > 4)
    invalid(L + ": cache bit widths must be 2, 3 or 4");
  if (!(c.key_rpc_ratio >= 0.0f && c.key_rpc_ratio <= 1.0f && c.value_rpc_ratio >= 0.0f && c.value_rpc_ratio <= 1.0f))
    invalid(L + ": rpc ratios must lie in [0, 1]");
  if (c.group_size <= 0) invalid(L + ": group_size must be positive");
}

void alloc(void** p, size_t bytes) {
  check_cuda(cudaMalloc(p, std::max<size_t>(bytes, 16)), "cudaMalloc(cache)");
  check_cuda(cudaMemset(*p, 0, std::max<size_t>(bytes, 16)), "cudaMemset(cache)");
}

void free_cache(kvmix_cache* c) {
  if (!c) return;
  int prev = -1;  // (no throwing here: destroy is not status-returning)
  if (cudaGetDevice(&prev) == cudaSuccess && prev != c->device) cudaSetDevice(c->device);
  else prev = -1;
  for (auto* s : {&c->k, &c->v}) {
    cudaFree(s->tail);
    cudaFree(s->info);
  }
  cudaFree(c->rec);
  delete c;
  if (prev >= 0) cudaSetDevice(prev);
}

void check_cache(const kvmix_cache* c) {
  if (!c) invalid("null cache handle");
}

// kvmix_*attend_layers: one multi-layer launch per kernel instance when every cache is
// valid, on one device and distinct (a repeated cache needs its appends in order) and no
// layer's output overlaps another layer's output or any input (the layers of one launch
// run concurrently; the per-layer loop keeps the sequential semantics for such calls)
bool batchable(kvmix_cache* const* caches, int n, const void* const* q, size_t q_bytes, const void* const* k,
               const void* const* v, size_t kv_bytes, float* const* out, size_t out_bytes) {
  if (n < 2 || !caches || !q || !out) return false;
  for (int l = 0; l < n; ++l) {
    check_cache(caches[l]);
    const kvmix_cache* c = caches[l];
    if (c->device != caches[0]->device || c->B != caches[0]->B || c->H != caches[0]->H || c->D != caches[0]->D)
      return false;
    if (!q[l] || !out[l] || (k && (!k[l] || !v[l]))) return false;
    for (int j = 0; j < l; ++j)
      if (caches[j] == caches[l]) return false;
  }
  auto overlap = [](const void* a, size_t na, const void* b, size_t nb) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
  };
  for (int l = 0; l < n; ++l) {
    for (int j = 0; j < n; ++j) {
      if (j != l && overlap(out[l], out_bytes, out[j], out_bytes)) return false;
      if (overlap(out[l], out_bytes, q[j], q_bytes)) return false;
      if (k && (overlap(out[l], out_bytes, k[j], kv_bytes) || overlap(out[l], out_bytes, v[j], kv_bytes)))
        return false;
    }
  }
  return true;
}

// every cache entry point runs on the cache's device (the caller's current device is restored)
#define KVB_ON_CACHE_DEVICE(c) \
  check_cache(c);              \
  DeviceGuard dev_guard_((c)->device)
}  // namespace

}  // namespace kvb

using namespace kvb;

extern "C" {

const char* kvmix_last_error(void) { return g_err.c_str(); }
int kvmix_abi_version(void) { return KVMIX_B200_ABI_VERSION; }
uint64_t kvmix_launch_count(void) { return g_launches.load(); }

kvmix_status kvmix_set_knob(const char* name, int value) {
  return guard([&] {
    if (!set_knob(name, value)) invalid(std::string("unknown knob ") + (name ? name : "(null)"));
  });
}

uint64_t kvmix_launch_count_of(const char* kernel) {
  std::lock_guard<std::mutex> lk(kvb::g_names_mu);
  auto& m = kvb::kernel_names();
  auto it = m.find(kernel ? kernel : "");
  return it == m.end() ? 0 : it->second;
}

size_t kvmix_packed_word_count(size_t n, int bits) { return words_for(n, bits); }

kvmix_status kvmix_feat_per_word(int bits, int* out) {
  return guard([&] {
    if (bits != 1 && bits != 2 && bits != 4)
      invalid("feat_per_word: bits must be 1, 2 or 4, got " + std::to_string(bits));
    *out = 32 / bits;
  });
}

kvmix_status kvmix_pack(const uint32_t* codes, size_t n, int bits, uint32_t* words, void* stream) {
  return guard([&] { pack(codes, n, bits, words, as_stream(stream)); });
}

kvmix_status kvmix_unpack(const uint32_t* words, size_t n, int bits, uint32_t* codes, void* stream) {
  return guard([&] { unpack(words, n, bits, codes, as_stream(stream)); });
}

size_t kvmix_group_count(kvmix_grouping g, int B, int H, int T, int D, int gs) {
  if (gs <= 0) return 0;
  if (g == KVMIX_PER_CHANNEL_KEY) return (size_t)B * H * D * (T / gs);
  return (size_t)B * H * T * ((D + gs - 1) / gs);
}

kvmix_status kvmix_quantize(kvmix_grouping g, const void* x, kvmix_dtype dt, int B, int H, int T, int D, int bits,
                            int gs, uint32_t* words, uint16_t* meta, void* stream) {
  return guard([&] { quantize(g, x, dt, B, H, T, D, bits, gs, words, meta, as_stream(stream)); });
}

kvmix_status kvmix_dequantize(kvmix_grouping g, const uint32_t* words, const uint16_t* meta, int B, int H, int T, int D,
                              int bits, int gs, float* out, void* stream) {
  return guard([&] { dequantize(g, words, meta, B, H, T, D, bits, gs, out, as_stream(stream)); });
}

kvmix_status kvmix_config_validate(const kvmix_layer_config* cfg) {
  return guard([&] {
    if (!cfg) invalid("null config");
    validate(*cfg);
  });
}

kvmix_status kvmix_rpc_target(int64_t current, double r, int64_t* out) {
  return guard([&] {
    if (current < 0) invalid("rpc_target: negative token count");
    if (!(r >= 0.0 && r <= 1.0)) invalid("rpc_target: ratio outside [0, 1]");
    *out = (int64_t)std::floor(r * (double)current);
  });
}

kvmix_status kvmix_cache_create(const kvmix_layer_config* cfg, int batch, int heads, int head_dim,
                                int64_t capacity_tokens, kvmix_dtype tail_dtype, kvmix_cache** out) {
  kvmix_cache* c = nullptr;
  kvmix_status s = guard([&] {
    if (!cfg || !out) invalid("null argument");
    validate(*cfg);
    if (batch < 1 || heads < 1 || head_dim < 1) invalid("KVLayerCache: dimensions must be positive");
    if (head_dim > 256) invalid("device cache: head_dim must be <= 256 (got " + std::to_string(head_dim) + ")");
    if (cfg->group_size % 16 != 0)
      invalid("device cache: group_size must be a multiple of 16 (got " + std::to_string(cfg->group_size) + ")");
    if (capacity_tokens < 1) invalid("device cache: capacity_tokens must be positive");
    if (capacity_tokens >= (int64_t)1 << 31) invalid("device cache: capacity_tokens must be below 2^31");
    if (tail_dtype != KVMIX_F32 && tail_dtype != KVMIX_F16) invalid("unsupported tail dtype");
    c = new kvmix_cache();
    c->cfg = *cfg;
    c->B = batch;
    c->H = heads;
    c->D = head_dim;
    // tile layout over Dl = head_dim rounded up to a multiple of 64 channels (the IMMA fragment
    // maps need whole 64-channel blocks); the extra channels hold zero codes and are never read
    c->Dl = std::max(64, (head_dim + 63) / 64 * 64);
    c->cap = capacity_tokens;
    c->tail_dtype = tail_dtype;
    check_cuda(cudaGetDevice(&c->device), "cudaGetDevice");
    const int gs = cfg->group_size;
    const size_t BH = (size_t)batch * heads;
    const int64_t ngroups = (capacity_tokens + gs - 1) / gs;  // group records per (b, kv-head)
    const int tpg = gs / 16, cg = (head_dim + gs - 1) / gs;
    const size_t ktw = (size_t)tile_words(c->Dl, cfg->key_bits), vtw = (size_t)tile_words(c->Dl, vstore_bits(cfg->value_bits));
    const size_t kmw = ((size_t)head_dim + 3) / 4 * 4;  // Key meta row, padded so records stay 16-byte multiples
    const size_t rec_words = tpg * (ktw + vtw) + (size_t)gs * cg + kmw;
    c->rec_bytes = BH * (size_t)ngroups * rec_words * 4;
    alloc((void**)&c->rec, c->rec_bytes);
    const size_t esz = tail_dtype == KVMIX_F16 ? 2 : 4;
    struct Spec {
      kvmix_cache::Side* s;
      int bits;
      float r;
      bool key;
    } specs[2] = {{&c->k, cfg->key_bits, cfg->key_rpc_ratio, true}, {&c->v, cfg->value_bits, cfg->value_rpc_ratio, false}};
    for (auto& sp : specs) {
      auto& s = *sp.s;
      s.bits = sp.bits;
      s.ratio = sp.r;
      s.tile_words = sp.key ? ktw : vtw;
      s.tpg = tpg;
      s.grp_stride = rec_words;
      s.bh_stride = (size_t)ngroups * rec_words;
      s.tiles = c->rec + (sp.key ? 0 : tpg * ktw);
      s.meta = c->rec + tpg * (ktw + vtw) + (sp.key ? (size_t)gs * cg : 0);
      s.mrow = sp.key ? head_dim : cg;
      s.dl = c->Dl;
      // window bound: floor(r*cap) (+ gs-1 for whole-group key aging) plus decode slack
      const int64_t bound = (int64_t)std::floor((double)sp.r * (double)capacity_tokens) + (sp.key ? gs : 1);
      s.tail_cap = std::min<int64_t>(capacity_tokens, bound) + 64;
      s.Hl = s.Hg = heads;
      if (sp.key) alloc((void**)&s.info, sizeof(int2) * (size_t)ngroups);
      else alloc((void**)&s.info, sizeof(int2) * (size_t)capacity_tokens);
      alloc(&s.tail, BH * (size_t)s.tail_cap * head_dim * esz);
    }
    *out = c;
  });
  if (s != KVMIX_OK) {
    free_cache(c);
    if (out) *out = nullptr;
  }
  return s;
}

void kvmix_cache_destroy(kvmix_cache* c) { free_cache(c); }

kvmix_status kvmix_cache_set_shard(kvmix_cache* c, int global_batch, int global_heads, int batch_offset,
                                   int head_offset) {
  return guard([&] {
    check_cache(c);
    if (c->total() != 0 || !c->k.segs.empty() || !c->v.segs.empty())
      invalid("set_shard: the shard placement must be set before the first append");
    if (batch_offset < 0 || head_offset < 0 || batch_offset + c->B > global_batch || head_offset + c->H > global_heads)
      invalid("set_shard: shard [" + std::to_string(batch_offset) + ", " + std::to_string(batch_offset + c->B) + ") x [" +
              std::to_string(head_offset) + ", " + std::to_string(head_offset + c->H) + ") outside the global batch " +
              std::to_string(global_batch) + " x heads " + std::to_string(global_heads));
    for (auto* s : {&c->k, &c->v}) {
      s->Hl = c->H;
      s->Hg = global_heads;
      s->b0 = batch_offset;
      s->h0 = head_offset;
    }
  });
}

kvmix_status kvmix_cache_reset(kvmix_cache* c, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    cache_reset(c, as_stream(stream));
  });
}

kvmix_status kvmix_cache_append(kvmix_cache* c, const void* k, const void* v, kvmix_dtype dt, int t, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    cache_append(c, k, v, dt, t, as_stream(stream));
  });
}

kvmix_status kvmix_cache_counters(const kvmix_cache* c, int64_t out[7]) {
  return guard([&] {
    check_cache(c);
    out[0] = c->total();
    out[1] = c->k.tail_len;
    out[2] = c->v.tail_len;
    out[3] = c->k.quantized;
    out[4] = c->v.quantized;
    out[5] = (int64_t)c->k.segs.size();
    out[6] = (int64_t)c->v.segs.size();
  });
}

kvmix_status kvmix_cache_shape(const kvmix_cache* c, int64_t out[5]) {
  return guard([&] {
    check_cache(c);
    out[0] = c->B;
    out[1] = c->H;
    out[2] = c->D;
    out[3] = c->cap;
    out[4] = c->tail_dtype;
  });
}

kvmix_status kvmix_cache_config(const kvmix_cache* c, kvmix_layer_config* out) {
  return guard([&] {
    check_cache(c);
    *out = c->cfg;
  });
}

kvmix_status kvmix_cache_memory_usage(const kvmix_cache* c, kvmix_memory_report* r) {
  return guard([&] {
    check_cache(c);
    const uint64_t BH = (uint64_t)c->B * c->H, D = (uint64_t)c->D, gs = (uint64_t)c->cfg.group_size;
    std::memset(r, 0, sizeof(*r));
    for (int64_t n : c->k.segs) {
      r->packed_payload_bits += (uint64_t)words_for(BH * n * D, c->k.bits) * 32u;
      r->metadata_bits += BH * D * ((uint64_t)n / gs) * 32u;
    }
    const uint64_t cg = (D + gs - 1) / gs;
    for (int64_t n : c->v.segs) {
      r->packed_payload_bits += (uint64_t)words_for(BH * n * D, c->v.bits) * 32u;
      r->metadata_bits += BH * (uint64_t)n * cg * 32u;
    }
    r->tail_bits = (uint64_t)(c->k.tail_len + c->v.tail_len) * BH * D * 16u;
    r->total_bits = r->packed_payload_bits + r->metadata_bits + r->tail_bits;
    r->fp16_baseline_bits = (uint64_t)c->total() * BH * D * 16u * 2u;
    r->compression_ratio = r->total_bits == 0 ? 1.0 : (double)r->fp16_baseline_bits / (double)r->total_bits;
  });
}

kvmix_status kvmix_cache_algorithmic_bytes(const kvmix_cache* c, uint64_t* out) {
  kvmix_memory_report r;
  kvmix_status s = kvmix_cache_memory_usage(c, &r);
  if (s == KVMIX_OK) *out = r.total_bits / 8;
  return s;
}

kvmix_status kvmix_cache_snapshot(const kvmix_cache* c, float* keys, float* values, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    cache_snapshot(c, keys, values, as_stream(stream));
  });
}

kvmix_status kvmix_cache_segment_info(const kvmix_cache* c, int side, int idx, int64_t info[3]) {
  return guard([&] {
    check_cache(c);
    if (side != 0 && side != 1) invalid("side must be 0 (keys) or 1 (values)");
    const auto& s = side == 0 ? c->k : c->v;
    if (idx < 0 || idx >= (int)s.segs.size()) throw Error(KVMIX_OUT_OF_RANGE, "segment index out of range");
    const int64_t n = s.segs[idx];
    const size_t BH = (size_t)c->B * c->H;
    info[0] = n;
    info[1] = (int64_t)words_for(BH * n * c->D, s.bits);
    info[2] = side == 0 ? (int64_t)(BH * c->D * (n / c->cfg.group_size)) : (int64_t)(BH * n * c->cgroups());
  });
}

kvmix_status kvmix_cache_export_segment(const kvmix_cache* c, int side, int idx, uint32_t* words, uint16_t* meta,
                                        void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    if (side != 0 && side != 1) invalid("side must be 0 (keys) or 1 (values)");
    cache_export_segment(c, side, idx, words, meta, as_stream(stream));
  });
}

kvmix_status kvmix_cache_export_tail(const kvmix_cache* c, int side, float* out, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    if (side != 0 && side != 1) invalid("side must be 0 (keys) or 1 (values)");
    cache_export_tail(c, side, out, as_stream(stream));
  });
}

kvmix_status kvmix_cache_import_segment(kvmix_cache* c, int side, int t, const uint32_t* words, const uint16_t* meta,
                                        void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    if (side != 0 && side != 1) invalid("side must be 0 (keys) or 1 (values)");
    cache_import_segment(c, side, t, words, meta, as_stream(stream));
  });
}

kvmix_status kvmix_cache_import_tail(kvmix_cache* c, int side, const float* tail, int64_t t, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    if (side != 0 && side != 1) invalid("side must be 0 (keys) or 1 (values)");
    cache_import_tail(c, side, tail, t, as_stream(stream));
  });
}

kvmix_status kvmix_attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int q_heads, int t, float* out,
                          double* checksum, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    if (dt != KVMIX_F32 && dt != KVMIX_F16) invalid("unsupported dtype");
    Workspace ws(as_stream(stream));
    attend(c, q, dt, q_heads, t, out, checksum, ws, as_stream(stream));
  });
}

kvmix_status kvmix_append_attend(kvmix_cache* c, const void* k, const void* v, kvmix_dtype kv_dt, int t, const void* q,
                                 kvmix_dtype q_dt, int q_heads, int tq, float* out, double* checksum, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    if (q_dt != KVMIX_F32 && q_dt != KVMIX_F16) invalid("unsupported dtype");
    Workspace ws(as_stream(stream));
    append_attend(c, k, v, kv_dt, t, q, q_dt, q_heads, tq, out, checksum, ws, as_stream(stream));
  });
}

kvmix_status kvmix_attend_layers(kvmix_cache* const* caches, int n_layers, const void* const* q, kvmix_dtype dt,
                                 int q_heads, int t, float* const* out, void* stream) {
  return guard([&] {
    if (n_layers < 0) invalid("n_layers must be non-negative");
    const auto esz = [](kvmix_dtype d) { return d == KVMIX_F16 ? (size_t)2 : (size_t)4; };
    if (n_layers >= 2 && caches && caches[0] && (dt == KVMIX_F32 || dt == KVMIX_F16) && q_heads > 0 && t > 0 &&
        batchable(caches, n_layers, q, (size_t)caches[0]->B * q_heads * t * caches[0]->D * esz(dt), nullptr,
                  nullptr, 0, out, (size_t)caches[0]->B * q_heads * t * caches[0]->D * 4)) {
      DeviceGuard dev_guard_(caches[0]->device);
      attend_layers(const_cast<kvmix_cache* const*>(caches), n_layers, nullptr, nullptr, KVMIX_F32, 0, q, dt,
                    q_heads, t, out, as_stream(stream));
      return;
    }
    for (int l = 0; l < n_layers; ++l) {
      KVB_ON_CACHE_DEVICE(caches[l]);
      Workspace ws(as_stream(stream));
      // layers after the first may overlap the previous layer's drain (different caches;
      // every input was produced before this call)
      request_pdl(l > 0 && caches[l] != caches[l - 1] && caches[l]->device == caches[l - 1]->device);
      attend(caches[l], q[l], dt, q_heads, t, out[l], nullptr, ws, as_stream(stream));
    }
    request_pdl(false);
  });
}

kvmix_status kvmix_append_attend_layers(kvmix_cache* const* caches, int n_layers, const void* const* k,
                                        const void* const* v, kvmix_dtype kv_dt, int t, const void* const* q,
                                        kvmix_dtype q_dt, int q_heads, int tq, float* const* out, void* stream) {
  return guard([&] {
    if (n_layers < 0) invalid("n_layers must be non-negative");
    if (q_dt != KVMIX_F32 && q_dt != KVMIX_F16) invalid("unsupported dtype");
    const auto esz = [](kvmix_dtype d) { return d == KVMIX_F16 ? (size_t)2 : (size_t)4; };
    if (n_layers >= 2 && caches && caches[0] && k && v && q_heads > 0 && tq > 0 && t > 0 &&
        batchable(caches, n_layers, q, (size_t)caches[0]->B * q_heads * tq * caches[0]->D * esz(q_dt), k, v,
                  (size_t)caches[0]->B * caches[0]->H * t * caches[0]->D * esz(kv_dt), out,
                  (size_t)caches[0]->B * q_heads * tq * caches[0]->D * 4)) {
      DeviceGuard dev_guard_(caches[0]->device);
      attend_layers(caches, n_layers, k, v, kv_dt, t, q, q_dt, q_heads, tq, out, as_stream(stream));
      return;
    }
    for (int l = 0; l < n_layers; ++l) {
      KVB_ON_CACHE_DEVICE(caches[l]);
      Workspace ws(as_stream(stream));
      request_pdl(l > 0 && caches[l] != caches[l - 1] && caches[l]->device == caches[l - 1]->device);
      append_attend(caches[l], k[l], v[l], kv_dt, t, q[l], q_dt, q_heads, tq, out[l], nullptr, ws, as_stream(stream));
    }
    request_pdl(false);
  });
}

kvmix_status kvmix_fused_qk_scores(const kvmix_cache* c, const void* q, kvmix_dtype dt, int t, float* scores,
                                   void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    fused_qk_scores(c, q, dt, t, scores, as_stream(stream));
  });
}

kvmix_status kvmix_softmax_rows(float* scores, int64_t rows, int64_t cols, void* stream) {
  return guard([&] { softmax_rows(scores, rows, cols, as_stream(stream)); });
}

kvmix_status kvmix_fused_pv(const kvmix_cache* c, const float* probs, int t, float* out, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    fused_pv(c, probs, t, out, as_stream(stream));
  });
}

kvmix_status kvmix_reference_attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int t, float* scratch,
                                    float* out, double* checksum, void* stream) {
  return guard([&] {
    KVB_ON_CACHE_DEVICE(c);
    Workspace ws(as_stream(stream));
    reference_attend(c, q, dt, t, scratch, out, checksum, ws, as_stream(stream));
  });
}

}  // extern "C"
