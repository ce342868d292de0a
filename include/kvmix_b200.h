/*
 * kvmix_b200.h -- C ABI of the B200-native KVmix hot path (libkvmix_b200.so).
 *
 * Drop-in boundary for the reference's hot-path C++ API (/root/reference/proj):
 * every entry point below names the reference function it replaces. The reference
 * has no FFI of its own; these are the calls its C++ callers
 * (toymodel.cpp:720-721, harness.cpp:101-120) and any ctypes/cgo/JNI binding make.
 *
 * Conventions
 *  - Plain pointers and sizes only. Tensor pointers are DEVICE pointers (CUDA global
 *    memory of the current device) unless the name says "host". `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream); all device work is
 *    enqueued on it and returns without synchronizing unless stated.
 *  - Every function returns kvmix_status; on failure kvmix_last_error() (thread-local)
 *    holds the message. The C++ shim (kvmix_b200.hpp) rethrows invalid-argument as
 *    std::invalid_argument, out-of-range as std::out_of_range and the rest as
 *    std::runtime_error, matching the reference's exception types.
 *  - Dense tensors are row-major [B, H, T, D] like kvmix::Tensor4f (tensor.hpp:24-27).
 *  - Meta is the KVQG pair layout: per group two uint16 binary16 values
 *    {scale, min} (quant.cpp:164-167).
 *  - No CPU fallback: without a CUDA device every compute entry point fails with
 *    KVMIX_CUDA_ERROR.
 */
#ifndef KVMIX_B200_H_
#define KVMIX_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVMIX_B200_ABI_VERSION 1

typedef enum kvmix_status {
  KVMIX_OK = 0,
  KVMIX_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  KVMIX_OUT_OF_RANGE = 2,     /* std::out_of_range (PackedBuffer::get, bitpack.cpp:70-73) */
  KVMIX_RUNTIME_ERROR = 3,    /* std::runtime_error (deserialize/load, quant.cpp:174-205) */
  KVMIX_CUDA_ERROR = 4,
  KVMIX_OUT_OF_MEMORY = 5
} kvmix_status;

typedef enum kvmix_dtype { KVMIX_F32 = 0, KVMIX_F16 = 1 } kvmix_dtype;

/* quant.hpp:38 (Grouping) */
typedef enum kvmix_grouping { KVMIX_PER_CHANNEL_KEY = 0, KVMIX_PER_TOKEN_VALUE = 1 } kvmix_grouping;

const char* kvmix_last_error(void);
int kvmix_abi_version(void);

/* ---- bitpack (bitpack.hpp:35-72) ------------------------------------------------ */
/* words = ceil(n*bits/32) for bits in {1,2,4}; ceil(n/11) for the Mixed3 layout (bits==3). */
size_t kvmix_packed_word_count(size_t n_codes, int bits);
/* feat_per_word (bitpack.cpp:8-14): 32/bits; invalid for bits outside {1,2,4}. */
kvmix_status kvmix_feat_per_word(int bits, int* out);
/* pack_uniform / pack_mixed3 (bitpack.cpp:57-67). Range violations are detected on the
 * device; this call synchronizes `stream` to report the first offending index in the
 * message exactly like PackedWriter::push (bitpack.cpp:26-41). */
kvmix_status kvmix_pack(const uint32_t* codes, size_t n_codes, int bits, uint32_t* words, void* stream);
/* unpack_uniform / unpack_mixed3 over a whole buffer (bitpack.cpp:69-96). */
kvmix_status kvmix_unpack(const uint32_t* words, size_t n_codes, int bits, uint32_t* codes, void* stream);

/* ---- quantize / dequantize (quant.hpp:79-80, quant.cpp:102-124, :77-100) ------- */
/* Number of (scale,min) groups: Keys B*H*D*(T/gs); Values B*H*T*ceil(D/gs). */
size_t kvmix_group_count(kvmix_grouping grouping, int B, int H, int T, int D, int group_size);
/* quantize_key_tensor / quantize_value_tensor: x is [B,H,T,D] (f32 or f16). Writes
 * kvmix_packed_word_count(B*H*T*D, bits) words, bit-identical to
 * QuantizedGroups::codes.words, and kvmix_group_count(...) meta pairs. */
kvmix_status kvmix_quantize(kvmix_grouping grouping, const void* x, kvmix_dtype dtype, int B, int H,
                            int T, int D, int bits, int group_size, uint32_t* words, uint16_t* meta,
                            void* stream);
/* QuantizedGroups::value_at over the whole tensor, bit-exact (mul then add, no FMA). */
kvmix_status kvmix_dequantize(kvmix_grouping grouping, const uint32_t* words, const uint16_t* meta,
                              int B, int H, int T, int D, int bits, int group_size, float* out,
                              void* stream);

/* ---- per-layer cache (cache.hpp:26-104, quant_config.hpp:17-53) ---------------- */
typedef struct kvmix_layer_config {
  int layer_index;
  int key_bits;   /* 2..4 */
  int value_bits; /* 2..4 */
  float key_rpc_ratio;
  float value_rpc_ratio;
  int group_size;
} kvmix_layer_config;

typedef struct kvmix_memory_report {
  uint64_t packed_payload_bits;
  uint64_t metadata_bits;
  uint64_t tail_bits;
  uint64_t total_bits;
  uint64_t fp16_baseline_bits;
  double compression_ratio;
} kvmix_memory_report;

typedef struct kvmix_cache kvmix_cache;

/* LayerQuantConfig::validate (cache.cpp:14-28). */
kvmix_status kvmix_config_validate(const kvmix_layer_config* cfg);
/* rpc_target (cache.cpp:30-34): floor(r * n). */
kvmix_status kvmix_rpc_target(int64_t current, double r, int64_t* out);

/* KVLayerCache(config, batch, heads, head_dim) (cache.cpp:36-43). `capacity_tokens` is
 * the device reservation (total tokens the cache may ever hold); `tail_dtype` selects
 * the full-precision window storage (KVMIX_F32 keeps arbitrary fp32 inputs exact,
 * KVMIX_F16 matches the 16-bit accounting). Device constraints: head_dim <= 256 (any value:
 * the tile layout rounds it up to a multiple of 64 channels whose extra codes are zero;
 * the tensor-core attention kernels serve 64 / 128, the generic kernel the rest),
 * group_size % 16 == 0. Allocates on the current device. */
kvmix_status kvmix_cache_create(const kvmix_layer_config* cfg, int batch, int heads, int head_dim,
                                int64_t capacity_tokens, kvmix_dtype tail_dtype, kvmix_cache** out);
void kvmix_cache_destroy(kvmix_cache* cache);
/* Multi-GPU placement (batch x KV-head shards): this cache holds batch rows
 * [batch_offset, batch_offset + batch) and KV heads [head_offset, head_offset + heads) of a
 * global [global_batch, global_heads] cache. The reference's Mixed3 narrow slots are a
 * function of the GLOBAL stream index (quant.cpp:36-47, 77-95), so a placed shard holds
 * bit-for-bit the unsharded cache's slice. Must precede the first append. Segment
 * export/import of a 3-bit side of a sharded cache is refused (its words interleave with
 * the other shards'). */
kvmix_status kvmix_cache_set_shard(kvmix_cache* cache, int global_batch, int global_heads, int batch_offset,
                                   int head_offset);
/* Drops all tokens (device buffers are re-zeroed on `stream`). */
kvmix_status kvmix_cache_reset(kvmix_cache* cache, void* stream);
/* KVLayerCache::append (cache.cpp:45-80): k, v are [B,H,t,D] device tensors of `dtype`.
 * The shrink rule runs on the host (identical integer bookkeeping); the fused
 * quantize-and-concatenate of aged tokens and the tail update run on `stream`. */
kvmix_status kvmix_cache_append(kvmix_cache* cache, const void* k, const void* v, kvmix_dtype dtype,
                                int t, void* stream);
/* total, key_tail, value_tail, quantized_keys, quantized_values, key_segments, value_segments */
kvmix_status kvmix_cache_counters(const kvmix_cache* cache, int64_t out[7]);
/* batch, heads, head_dim, capacity_tokens, tail_dtype */
kvmix_status kvmix_cache_shape(const kvmix_cache* cache, int64_t out[5]);
kvmix_status kvmix_cache_config(const kvmix_cache* cache, kvmix_layer_config* out);
/* KVLayerCache::memory_usage (cache.cpp:119-134). Host-only bookkeeping. */
kvmix_status kvmix_cache_memory_usage(const kvmix_cache* cache, kvmix_memory_report* out);
/* Bytes one attention launch over this cache reads by the algorithm: payload + meta +
 * tails at 16 bits (== memory_usage().total_bits / 8). */
kvmix_status kvmix_cache_algorithmic_bytes(const kvmix_cache* cache, uint64_t* out);
/* KVLayerCache::snapshot_dequantized (cache.cpp:136-173), bit-exact; keys/values
 * [B,H,total,D] fp32 device buffers. */
kvmix_status kvmix_cache_snapshot(const kvmix_cache* cache, float* keys, float* values, void* stream);
/* key_segments()/value_segments() (cache.hpp:75-76): side 0 = Keys, 1 = Values.
 * info = {t, word_count, group_count}. export writes the segment's words/meta exactly
 * as the reference's QuantizedGroups for that age-out event. */
kvmix_status kvmix_cache_segment_info(const kvmix_cache* cache, int side, int index, int64_t info[3]);
kvmix_status kvmix_cache_export_segment(const kvmix_cache* cache, int side, int index, uint32_t* words,
                                        uint16_t* meta, void* stream);
/* key_tail_at / value_tail_at (cache.hpp:79-86): fp32 [tail_len][B][H][D]. */
kvmix_status kvmix_cache_export_tail(const kvmix_cache* cache, int side, float* out, void* stream);
/* KVLayerCache::load (cache.cpp:251-281) counterpart: appends one reference segment
 * (words/meta as exported) to a side, then restore_tail installs the tails. Used to
 * rebuild a device cache from a KVCD dump. */
kvmix_status kvmix_cache_import_segment(kvmix_cache* cache, int side, int t, const uint32_t* words,
                                        const uint16_t* meta, void* stream);
kvmix_status kvmix_cache_import_tail(kvmix_cache* cache, int side, const float* tail, int64_t t,
                                     void* stream);

/* ---- attention (attention.hpp:25-48) -------------------------------------------- */
/* attend (attention.cpp:161-166): q [B, Hq, t, D] (f32/f16), Hq = G * heads (G=1 is the
 * reference's case; G>1 is grouped-query attention, query head hq uses KV head hq/G).
 * out [B, Hq, t, D] fp32. If `checksum` (a HOST pointer) is non-NULL the call
 * synchronizes `stream` and stores the double sum of all scaled scores
 * (AttentionOutput::scores_checksum). Fused split-K dequant-in-the-loop kernel; no
 * full-precision K/V is materialized; scratch is independent of the token count. */
kvmix_status kvmix_attend(const kvmix_cache* cache, const void* q, kvmix_dtype dtype, int q_heads,
                          int t, float* out, double* checksum, void* stream);
/* One decode step of one layer: KVLayerCache::append(k, v) (t tokens, cache.cpp:45-80)
 * followed by attend(q) (attention.cpp:161-166), with the reference's semantics and errors.
 * When the append is a 1-token decode step that ages no Key group (the steady state), the
 * append runs inside the attention launch (one kernel instead of two); otherwise the two
 * calls run in order. Replaces the CachedDecoder::step pair `cache.append(); attend();`. */
kvmix_status kvmix_append_attend(kvmix_cache* cache, const void* k, const void* v, kvmix_dtype kv_dtype, int t,
                                 const void* q, kvmix_dtype q_dtype, int q_heads, int tq, float* out,
                                 double* checksum, void* stream);
/* attend over several layers' caches in one call: q[l], out[l] per layer. Results equal
 * n_layers kvmix_attend calls in order. Layers served by the same IMMA kernel instance share
 * ONE launch (attend_mma_layers_kernel) when the caches are distinct, on one device, of one
 * shape, and no out[l] overlaps another out[] or any q[]; otherwise one launch per layer. */
kvmix_status kvmix_attend_layers(kvmix_cache* const* caches, int n_layers, const void* const* q,
                                 kvmix_dtype dtype, int q_heads, int t, float* const* out,
                                 void* stream);
/* One decode step of a model stack in one call: kvmix_append_attend for every layer l
 * (k[l], v[l], q[l], out[l]) in order on `stream` -- the per-layer CachedDecoder::step pairs
 * (toymodel.cpp:720-721, 746) without a host round trip per layer. No checksum. Same shared
 * launch rule as kvmix_attend_layers (out[] must also not overlap k[] / v[]); the caches
 * after the call are bit-identical either way, the outputs equal up to fp32 merge order. */
kvmix_status kvmix_append_attend_layers(kvmix_cache* const* caches, int n_layers, const void* const* k,
                                        const void* const* v, kvmix_dtype kv_dtype, int t, const void* const* q,
                                        kvmix_dtype q_dtype, int q_heads, int tq, float* const* out, void* stream);
/* fused_qk_scores (attention.cpp:28-81): scores [B,H,t,total] fp32 (already * 1/sqrt(D)). */
kvmix_status kvmix_fused_qk_scores(const kvmix_cache* cache, const void* q, kvmix_dtype dtype, int t,
                                   float* scores, void* stream);
/* softmax_rows (attention.cpp:96-105): in place over rows x cols fp32. */
kvmix_status kvmix_softmax_rows(float* scores, int64_t rows, int64_t cols, void* stream);
/* fused_pv (attention.cpp:107-159): probs [B,H,t,total] -> out [B,H,t,D]. */
kvmix_status kvmix_fused_pv(const kvmix_cache* cache, const float* probs, int t, float* out, void* stream);
/* reference_attend (attention.cpp:168-211): dequantizes everything into `scratch`
 * (2*B*H*total*D floats, caller-provided) then dense attention. Oracle-style path. */
kvmix_status kvmix_reference_attend(const kvmix_cache* cache, const void* q, kvmix_dtype dtype, int t,
                                    float* scratch, float* out, double* checksum, void* stream);

/* scratch::reset / scratch::allocated (scratch.hpp:14-21): bytes of attention scratch the
 * library requested since the last reset (split-K partials, merge counters, flags). The
 * reference's contract is that the fused path's scratch does not depend on the cached token
 * count (test_attention.cpp:182-205); here it depends on (B, H, query rows, D, SM count) only.
 * The memory itself is persistent per (device, stream) and reused across calls. */
void kvmix_scratch_reset(void);
uint64_t kvmix_scratch_allocated(void);

/* Tuning / test hook: overrides one kernel knob for later launches ("KVMIX_TAIL_UNIT",
 * "KVMIX_GROUP_COST", "KVMIX_TEST_FLUSH_BLOCKS" (<= 0 restores the default), "KVMIX_MIN_COST",
 * "KVMIX_WS": 0 = single-warp tensor-core kernel only, 1 = warp-specialized kernel for 3-bit
 * Values (default), 2 = warp-specialized kernel for every tier; "KVMIX_R4": 1 = four query rows
 * per pass on the single-warp kernel when a KV head has more than two (default), 0 = two).
 * The same names are read once from the environment at the first launch. */
kvmix_status kvmix_set_knob(const char* name, int value);

/* Number of kernels this library has launched in this process (instrumentation for
 * the benchmark's gpu_launches count). */
uint64_t kvmix_launch_count(void);
/* Launches of one kernel by name ("attend_mma_kernel", "attend_generic_kernel", ...):
 * lets tests assert which device path served a call. */
uint64_t kvmix_launch_count_of(const char* kernel);

#ifdef __cplusplus
}
#endif
#endif /* KVMIX_B200_H_ */
