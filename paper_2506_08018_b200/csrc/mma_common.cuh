// mma_common.cuh -- shared pieces of the tensor-core decode-attention kernels
// (attention_mma.cu: one warp per unit range; attention_ws.cu: warp-specialized pairs):
// launch parameters, TMA / mbarrier / IMMA helpers, fragment layouts, the stream-K
// partition and the deterministic in-kernel merge.
#pragma once
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <string>

#include "attention.cuh"

namespace kvb {

namespace {

#ifndef KVB_WARPS
#define KVB_WARPS 4
#endif
constexpr int kMmaWarps = KVB_WARPS;  // independent warps per CTA (no CTA barriers)
#ifndef KVB_MIN_WARPS_N
#define KVB_MIN_WARPS_N 16
#endif
// resident warps per SM the register budget is sized for: 3-bit Keys with two query rows
// (GQA) get 12 (their B staging leaves shared memory for 12 warps with a two-stage ring anyway)
// four query rows (GQA G = 4: two IMMA column tiles, twice the accumulators) get KVB_MIN_WARPS_R4
#ifndef KVB_MIN_WARPS_R4
#define KVB_MIN_WARPS_R4 12
#endif
#ifndef KVB_MIN_WARPS_R4K3
#define KVB_MIN_WARPS_R4K3 8  // 3-bit Keys (a second B plane): 12 warps spill
#endif
#define KVB_MIN_WARPS(KB, R) \
  ((R) == 4 ? ((KB) == 3 ? KVB_MIN_WARPS_R4K3 : KVB_MIN_WARPS_R4) : (KB) == 3 && (R) == 2 ? 12 : KVB_MIN_WARPS_N)
#define KVB_MIN_CTAS(KB, R) (KVB_MIN_WARPS(KB, R) / KVB_WARPS)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kFlushBlocks = 1024;  // Value int32 accumulators: < 2^31 / (32 * 240 * 255)
// (KVMIX_TEST_FLUSH_BLOCKS lowers it so the parity tests reach the forced-fold path)
// Lazy online-softmax max (log2 units): the reference max m only moves when a block's max
// exceeds it by more than kLazy, so p = 2^(score - m) <= 2^kLazy and the Value accumulators
// are rescaled (folded) only a handful of times per segment.
constexpr int kLazy = 3;
constexpr int kEHead = 2;  // extra fixed-point headroom bits when the Value exponent is reset

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// binary16 pair {scale (lo), min (hi)} of a meta word -> fp32
__device__ __forceinline__ float2 meta_pair(uint32_t m) {
  return __half22float2(*reinterpret_cast<const __half2*>(&m));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA bulk copy global -> shared, completion counted on `bar`, evict-first in L2 (the
// packed cache is streamed once per step).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// D += A (u8, 16x32) * B (s8, 32x8), int32 (exact)
__device__ __forceinline__ void imma_us(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// D += A (u8, 16x32) * B (u8, 32x8), int32 (exact)
__device__ __forceinline__ void imma_uu(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float pow2i(int e) { return __int_as_float((127 + e) << 23); }

// 2^x via MUFU.EX2 without the denormal fix-up (x <= 0 here; 2^x < 2^-126 flushes to 0)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// inverse of n modulo 11 (n in 1..10)
__device__ __forceinline__ int inv11(int n) {
  // 1 1, 2 6, 3 4, 4 3, 5 9, 6 2, 7 8, 8 7, 9 5, 10 10
  return (int)((0xA578293461ull >> (4 * (n - 1))) & 0xFu);
}

// Four channels' balanced s8 digit words (byte n of uu[c] = digit n of channel c) -> digit
// planes: dst[n * stride] = {digit n of channels 0..3} (4x4 byte transpose).
__device__ __forceinline__ void store_digits(uint32_t* dst, int stride, const uint32_t (&uu)[4]) {
  const uint32_t lo01 = __byte_perm(uu[0], uu[1], 0x5140), hi01 = __byte_perm(uu[0], uu[1], 0x7362);
  const uint32_t lo23 = __byte_perm(uu[2], uu[3], 0x5140), hi23 = __byte_perm(uu[2], uu[3], 0x7362);
  dst[0] = __byte_perm(lo01, lo23, 0x5410);
  dst[stride] = __byte_perm(lo01, lo23, 0x7632);
  dst[2 * stride] = __byte_perm(hi01, hi23, 0x5410);
  dst[3 * stride] = __byte_perm(hi01, hi23, 0x7632);
}

// Lane's words of one tile in shared memory (layout: plane_addr in common.cuh).
template <int WPL>
__device__ __forceinline__ void lds_plane(const uint32_t* tile, int lane, uint32_t* w) {
  if constexpr (WPL >= 4) {
#pragma unroll
    for (int c = 0; c < WPL / 4; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(tile + c * 128 + lane * 4);
      w[4 * c] = v.x;
      w[4 * c + 1] = v.y;
      w[4 * c + 2] = v.z;
      w[4 * c + 3] = v.w;
    }
  } else if constexpr (WPL == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(tile + lane * 2);
    w[0] = v.x;
    w[1] = v.y;
  } else {
    w[0] = tile[lane];
  }
}

template <int D, int B>
__device__ __forceinline__ void lds_tile(const uint32_t* tile, int lane, uint32_t* w) {
  if constexpr (B == 3) {
    lds_plane<D * 2 / 64>(tile, lane, w);
    lds_plane<D / 64>(tile + 32 * (D * 2 / 64), lane, w + D * 2 / 64);
  } else {
    lds_plane<D * B / 64>(tile, lane, w);
  }
}

template <int D, int B>
constexpr int lane_words() {
  return B == 3 ? D * 3 / 64 : D * B / 64;
}



// Full-precision-window tokens per work unit. A window token costs several times a packed
// token (lane-parallel dequantization of partially aged Values, no TMA staging), so units
// are small to keep the stream-K ranges balanced (KVMIX_TAIL_UNIT overrides, for tuning).
constexpr int kTailUnit = 1;
constexpr int kGroupCost = 1;  // cost of one fast group in window-token units (KVMIX_GROUP_COST)
constexpr int kMaxPasses = 8;  // row passes per launch
constexpr int kMinCost = 8;    // minimum cost units per warp (KVMIX_MIN_COST overrides)

}  // namespace

// Tuning / test knobs, read from the environment once per process (attention_mma.cu).
struct Knobs {
  int tail_unit = kTailUnit, group_cost = kGroupCost, flush_blocks = kFlushBlocks, min_cost = kMinCost;
  int ws = 1;  // warp-specialized kernel (attention_ws.cu): 0 never, 1 for 3-bit Values, 2 always
  int tc = 0;  // tcgen05 kernel (attention_tc.cu) for the fast groups where it applies
  int pdl = 1;  // programmatic dependent launch between the layers of kvmix_*attend_layers
  int r4 = 1;      // four query rows per pass (two IMMA column tiles) on the single-warp kernel
  int layers = 1;  // kvmix_*attend_layers: one launch per kernel instance (else per layer)
  bool skip_tail = false, no_window = false;
};
Knobs& knobs();
bool take_pdl();

// Launch parameters shared by attend_mma_kernel and attend_ws_kernel.
struct MmaParams {
  SideView k, v;
  const void* q;
  int q16, tail16;
  int H, Hq, tq, rows, gs, cg;
  int row0;  // first query row of this launch; rows = query rows per pass (the slot stride)
  // passes: query rows [row0, row0 + rows_all) run as npass row passes of <= rows rows in one
  // launch, each unit range by npass adjacent warps (pass = global warp % npass) that stream
  // the same records at the same time (one DRAM read, the twins hit L2); pass x uses partial
  // slots x * pslots + (w + bh) and counters cnt[x * nbh + bh]
  int npass, rows_all, pslots, nbh;
  int64_t T, P;  // total tokens; fast-path limit (multiple of gs)
  int64_t Pw;    // window blocks cover tokens [P, Pw) (Keys fp16 in the ring, Values packed)
  int nwb;       // window blocks per (b, kv-head)
  // stream-K work list: per (b, kv-head) U = Gf fast groups + nwb window blocks +
  // ceil((T - Pw) / tail_unit) window-token units, N = BH * U units in bh-major order
  int Gf, U, N;  // 32-bit: the host falls back to the generic path beyond 2^31 units
  // cost-weighted split: a group costs Qc, a window token 1; (b, kv-head) cost cost_bh =
  // Qc Gf + (U - Gf), total Nc = BH cost_bh; warp w owns the units starting in cost range
  // [w Nc / W, (w+1) Nc / W)
  int Qc;
  int64_t cost_bh, Nc;
  int Grec;      // group records per (b, kv-head) (bh stride of the record array)
  int W;
  int stages;
  uint32_t kt_bytes, vt_bytes, vm_bytes, km_bytes;  // per-group copy sizes
  uint32_t stage_bytes;
  float inv;  // 1/sqrt(D)
  int want_cs;  // accumulate the double scores checksum (only when the caller asks)
  int fused;         // the call's 1-token append runs in the prologue (kvmix_append_attend)
  DecodeAppend da;
  // Arrival counters and flags live in zero-initialised scratch (Workspace::zeroed) and every
  // launch leaves them zero again: the last arriver of a counter resets it, the final writer of
  // a (pass, b, kv-head) resets its flag. No epochs or tags, so a launch is replayable.
  unsigned* flags;  // per (pass, b, kv-head) at pass * nbh + bh: 1 once the append is done
  unsigned* cnt;    // per (pass, b, kv-head): octets published (merge by the last)
  unsigned* cnt8;   // per (pass, warp octet k, bh) at slot pass * pslots + k + bh: partials published
  float* out;
  int flush_blocks;  // fold the int32 Value accumulators at least every this many blocks
  int tail_unit;     // window tokens per work unit
  int skip_tail;     // profiling only (KVMIX_PROF_SKIP_TAIL): leave the window out
  float2* part_ml;  // partial slot of (warp w, bh) = w + bh (unique along the staircase)
  float* part_acc;
  double* part_cs;
  // programmatic dependent launch (layer after layer inside kvmix_*attend_layers): the launch
  // may start while the previous layer's kernel drains; every warp waits for it to complete
  // (griddepcontrol.wait) before its first result / scratch write and only then lets the
  // next launch start (launch_dependents), so at most two launches are in flight and the
  // scratch sets they use alternate (Workspace)
  int pdl;
  // window-only launch (after attend_tc_kernel served the fast groups): warp = (pass, b,
  // kv-head), its window units only; the fast-group partials of attend_tc_kernel (slot c + bh
  // for the CTAs c whose tile ranges hold bh's tiles) are merged into the output here
  int wonly;
  const float2* ext_ml;
  const float* ext_acc;
  int ext_C;
  int64_t ext_NT;
  int ext_Tb, ext_R;
};

// Parameters of a multi-layer launch (attend_mma_layers_kernel): layer l's warps are
// [off[l], off[l + 1]). Passed by value in the kernel's parameter space (<= 32 KB).
constexpr int kMaxLayers = 32;
struct MmaLayers {
  int n;
  int off[kMaxLayers + 1];
  MmaParams l[kMaxLayers];
};
static_assert(sizeof(MmaLayers) <= 32000, "kernel parameter space");

// Partials of the fast groups written by attend_tc_kernel (attention_tc.cu).
struct TcExt {
  const float2* ml = nullptr;
  const float* acc = nullptr;
  const double* cs = nullptr;
  int C = 0;         // CTAs (tile ranges)
  int64_t NT = 0;    // tiles
  int Tb = 0;        // tiles per (b, kv-head)
  int R = 0;         // rows per partial slot
  size_t slots = 0;  // C + BH
};
bool attend_tc_launch(const kvmix_cache* c, const void* q, bool q16, int Hq, int tq, int Gf, bool want_cs,
                      Workspace& ws, cudaStream_t st, TcExt* ext);
bool attend_tc_eligible(const kvmix_cache* c, int rows);

namespace {

__device__ __forceinline__ void pdl_gate(const MmaParams& p) {
  if (p.pdl) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  }
}

// first unit whose start cost is >= c (units: Gf groups of cost Qc, then window units of 1)
__device__ __forceinline__ int unit_at_cost(const MmaParams& p, int64_t c) {
  const int bh = (int)(c / p.cost_bh);
  const int64_t cl = c - (int64_t)bh * p.cost_bh;
  const int64_t gcost = (int64_t)p.Qc * p.Gf;
  const int64_t local = cl <= gcost ? (cl + p.Qc - 1) / p.Qc : p.Gf + (cl - gcost);
  return bh * p.U + (int)local;
}

// Dequantized packed element (token j < quantized, channel d) with compile-time D.
template <int D, bool KEY, int BITS>
__device__ __forceinline__ float deq_lane(const SideView& s, int bh, int j, int d, int gs) {
  const uint32_t* tile = s.tiles + tile_index(s, bh, j >> 4);
  const uint32_t code = tile_get(tile, KEY, D, BITS, j & 15, d);
  uint32_t m;
  bool narrow = false;
  if (KEY) {
    const int grp = j / gs;
    m = s.meta[kmeta_index(s, bh, grp) + d];
    if (BITS == 3) narrow = narrow_key(s.gbh(bh), d, D, s.info[grp], j - grp * gs);
  } else {
    m = s.meta[vmeta_at(s, bh, j, d / gs)];
    if (BITS == 3) narrow = narrow_value(s.gbh(bh), d, D, s.info[j]);
  }
  return decode(code, meta_scale(m), meta_min(m), narrow);
}

__device__ __forceinline__ float tail_val(const SideView& s, bool f16, int bh, int64_t j, int d, int D) {
  return f16 ? tail_at<__half>(s, bh, j, d, D) : tail_at<float>(s, bh, j, d, D);
}

// warp owning the unit that starts at cost sx: floor(((sx + 1) W - 1) / Nc)
__device__ __forceinline__ int warp_at_cost(const MmaParams& p, int64_t sx) {
  return (int)(((sx + 1) * p.W - 1) / p.Nc);
}
// first and last warp whose ranges hold units of (b, kv-head) bh
__device__ __forceinline__ void bh_warps(const MmaParams& p, int bh, int& w0, int& w1) {
  const int64_t s0 = (int64_t)bh * p.cost_bh;
  const int ntail = p.U - p.Gf;
  const int64_t s1 = s0 + (ntail > 0 ? (int64_t)p.Qc * p.Gf + ntail - 1 : (int64_t)p.Qc * (p.Gf - 1));
  w0 = warp_at_cost(p, s0);
  w1 = warp_at_cost(p, s1);
}

// Arrival counter (zero at launch): returns true for the n-th arriver, which resets the word
// to zero for the next launch (every arrival of this launch has happened).
__device__ __forceinline__ bool count_arrival(unsigned* cw, int n) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;\n" : "=r"(old) : "l"(cw) : "memory");
  if ((int)old + 1 != n) return false;
  *reinterpret_cast<volatile unsigned*>(cw) = 0u;
  return true;
}

// Publish this warp's partial of bh; returns true for the last of the bh's warps to arrive.
// Two levels (warps in octets, then the octets) keep at most 8 warps retrying a CAS on one
// word: a (b, kv-head) split over dozens of warps would otherwise serialize on its counter.
// (the warp barrier orders every lane's partial before lane 0's release; the acquiring lane
// 0 of the last arriver passes the order on to its lanes through the next warp barrier)
__device__ __forceinline__ bool arrive_last(const MmaParams& p, int bh, int lane, int pass, int wg) {
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    int w0, w1;
    bh_warps(p, bh, w0, w1);
    const int k = wg >> 3;
    const int a = max(w0, 8 * k), z = min(w1, 8 * k + 7);
    last = z == a || count_arrival(p.cnt8 + (size_t)pass * p.pslots + k + bh, z - a + 1);
    const int nsub = (w1 >> 3) - (w0 >> 3) + 1;
    if (last && nsub > 1) last = count_arrival(p.cnt + (size_t)pass * p.nbh + bh, nsub);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  __syncwarp();
  return last != 0;
}

// Merge the partials of warps w0..w1 of bh (deterministic) -> out. A (b, kv-head) can be
// split over dozens of warps when there are few of them (B8 x 8 KV heads: ~37 per head), so
// the lanes read the partials' (m, l) in parallel and the accumulator rows are streamed with
// several loads in flight; the rows sum in warp order.
template <int D>
__device__ __forceinline__ float4 ld_part(const float* a) {
  if constexpr (D == 128) return __ldcg(reinterpret_cast<const float4*>(a));
  else {
    const float2 x = __ldcg(reinterpret_cast<const float2*>(a));
    return make_float4(x.x, x.y, 0.f, 0.f);
  }
}
template <int D>
__device__ __forceinline__ void merge_bh(const MmaParams& p, int bh, int lane, int pass, int prow0, int prows) {
  constexpr int LC = D / 32;
  static_assert(LC == 2 || LC == 4, "merge: D in {64, 128}");
  int w0, w1;
  bh_warps(p, bh, w0, w1);
  const int b = bh / p.H, h = bh % p.H, G = p.Hq / p.H;
  const size_t s0 = (size_t)pass * p.pslots + bh;
  for (int r = 0; r < prows; ++r) {
    float M = -INFINITY;
    for (int w = w0 + lane; w <= w1; w += 32) M = fmaxf(M, __ldcg(&p.part_ml[(s0 + w) * p.rows + r]).x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int wb = w0; wb <= w1; wb += 32) {
      float f = 0.f;
      if (wb + lane <= w1) {
        const float2 ml = __ldcg(&p.part_ml[(s0 + wb + lane) * p.rows + r]);
        if (ml.x != -INFINITY) {
          f = expf(ml.x - M);
          L += ml.y * f;
        }
      }
      const int nb = min(32, w1 - wb + 1);
      const float* base = p.part_acc + ((s0 + wb) * p.rows + r) * D + lane * LC;
      const size_t step = (size_t)p.rows * D;
      for (int i = 0; i < nb; i += 4) {
        float fi[4];
        float4 x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          fi[k] = __shfl_sync(0xffffffffu, f, (i + k) & 31);
          if (i + k >= nb) fi[k] = 0.f;
          // neutral partials (f = 0) never wrote their accumulator row: not read
          x[k] = fi[k] != 0.f ? ld_part<D>(base + (size_t)(i + k) * step) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a.x = fmaf(x[k].x, fi[k], a.x);
          a.y = fmaf(x[k].y, fi[k], a.y);
          a.z = fmaf(x[k].z, fi[k], a.z);
          a.w = fmaf(x[k].w, fi[k], a.w);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    const int gi = (prow0 + r) / p.tq, qi = (prow0 + r) % p.tq;
    float* o = p.out + (((size_t)b * p.Hq + h * G + gi) * p.tq + qi) * D + lane * LC;
    const float il = 1.0f / L;
    o[0] = a.x * il;
    o[1] = a.y * il;
    if constexpr (LC == 4) {
      o[2] = a.z * il;
      o[3] = a.w * il;
    }
  }
  // final writer of (pass, bh): every warp that waited on the append flag has arrived
  if (p.fused && lane == 0) p.flags[(size_t)pass * p.nbh + bh] = 0u;
}

// Per-warp dynamic shared layout (bytes):
//   ring[S][stage_bytes] | kstage | vbs[CGMAX][8 or 16 cols][32] u8 | bars[S] u64
// kstage: kbs[planes][4R cols][4 t][NK][2] u32 (digit words of the Key B fragments; 3-bit
//         Keys have a second plane), zeros[4 t][NK][2] (B columns without a query row),
//         then for 3-bit Keys ytab[R][D] f32 (narrow-slot factors per query row)
//         and ntab[D] u32 (word offset | shift << 16 of each channel's low 2 bits at row 0).
template <int D, int KB, int R>
struct WarpLayout {
  static constexpr int kKC = 4 * R;  // B columns that carry query rows (lanes g >= kKC read 0)
  static constexpr int kKB = kKC * 4 * (D / 32) * 2 * 4;
  static constexpr int kZ = (KB == 3 ? 2 : 1) * kKB;  // zero words read by the lanes g >= kKC
  static constexpr int kY = kZ + 4 * (D / 32) * 2 * 4;
  static constexpr int kK = KB == 3 ? kY + (R + 1) * D * 4 : kY;
  static constexpr int kV = (D / 32) * 8 * (R > 2 ? 2 : 1) * 32;  // [cg][4R cols][32 tokens] u8
  static constexpr int kQ = D * 4 + 32 * 8;  // q of all channels (window blocks), checksum slots
  __host__ __device__ static constexpr size_t bytes(int stages, uint32_t stage_bytes) {
    const size_t n = (size_t)stages * stage_bytes + kK + kV + kQ + (size_t)stages * 8;
    return (n + 127) / 128 * 128;  // keep every warp's ring 128-byte aligned
  }
};

// Compile-time stage geometry for a compile-time group size: record = K tiles | V tiles |
// V meta | K meta, ring depth chosen for 4 CTAs per SM (same rule as launch()).
template <int D, int KB, int VB, int R, int GS>
struct StageGeo {
  static constexpr uint32_t kKT = GS ? (uint32_t)((GS / 16) * tile_words(D, KB) * 4) : 0;
  static constexpr uint32_t kVT = GS ? (uint32_t)((GS / 16) * tile_words(D, vstore_bits(VB)) * 4) : 0;
  static constexpr uint32_t kVM = GS ? (uint32_t)(GS * ((D + (GS ? GS : 1) - 1) / (GS ? GS : 1)) * 4) : 0;
  static constexpr uint32_t kKM = (uint32_t)(D * 4);
  static constexpr uint32_t kStage = kKT + kVT + kVM + kKM;
  static constexpr long kStatic = (long)kMmaWarps * R * D * 4;  // s_acc
  // ring depth at `occ` resident CTAs per SM (the per-CTA reservation is 1 KB)
  static constexpr int stages_for(int occ) {
    return (int)(((227L * 1024 / occ - 1024 - kStatic) / kMmaWarps - (long)WarpLayout<D, KB, R>::bytes(0, 0) - 32 - 128) /
                 (long)(kStage ? kStage : 1));
  }
  static constexpr int kOcc = KVB_MIN_CTAS(KB, R);
  static constexpr int kStages = GS == 0 ? 0
                                 : stages_for(kOcc) >= 2 ? (stages_for(kOcc) < 4 ? stages_for(kOcc) : 4)
                                 : stages_for(kOcc * 3 / 4) >= 2 ? (stages_for(kOcc * 3 / 4) < 4 ? stages_for(kOcc * 3 / 4) : 4)
                                                                 : 2;
};

}  // namespace
}  // namespace kvb
