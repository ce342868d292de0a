// attention_mma.cu -- fused split-K decode attention on the tensor cores (mma.sync m16n8k16),
// fed by TMA bulk copies (cp.async.bulk + mbarrier) into a per-warp shared-memory ring.
//
// Decode is a GEMV per (b, kv-head): scores = K q, out = V^T p. At 2-bit gs32 a K+V element
// pair is 0.75 B of HBM traffic, so a CUDA-core loop (unpack + dequant + FMA per element)
// runs out of issue slots before HBM does. Here the codes go straight
// from shared memory into tensor-core A fragments: the device tile layout (common.cuh) is
// "fragment-native", so one 128-bit shared load per lane yields that lane's A operands.
// The dequantization is factored out of the dot products:
//     q.k_j  = sum_d (q_d s_gd) c_jd + sum_d q_d m_gd          (Keys, per channel group)
//     out_d  = sum_j (p_j s_jg) c_jd + sum_j p_j m_jg          (Values, per token group)
// The B operands (q*s, p*s, p) are split into an fp16 hi part and an fp16 lo remainder in
// two MMA columns, so products carry ~22 mantissa bits and accumulate in fp32. The Value
// min term is a second small MMA with A = the binary16 mins (exact in fp16).
//
// Unpack ("scale classes"): a fragment register holds two codes at the same bit offset of
// the two 16-bit halves. OR-ing the masked word into 0x6400 (fp16 1024) and subtracting
// 1024 gives the codes exactly, scaled by 2^offset -- so codes at offsets 0..9 need no
// shift at all. The slot -> offset map only depends on the k-step (Keys) / m-tile
// (Values), so the power of two is folded into the Key B operand per channel and into the
// Value accumulator of each m-tile at the end: one LOP3 + one HADD2 per register.
//
// Mixed3 (3-bit) Keys: the reference's narrow slots (stream index % 11 == 10) dequantize
// with scale*7/3. For channel d of a group the narrow tokens are t = tau_d (mod 11), so the
// correction sum_d [t == tau_d mod 11] c_td q_d (s'_d - s_d) is 11 extra B columns (one per
// residue class, hi/lo) in the same MMAs; each token picks the column of its residue.
//
// Memory pipeline: every unit of work (one Key group of gs tokens of one (b, kv-head))
// is four contiguous byte ranges in HBM -- Key tiles, Value tiles, Value meta, Key meta --
// copied by one elected lane with cp.async.bulk into a ring of S stages; the warp waits on
// the stage's mbarrier (complete_tx), computes, and refills the stage S groups ahead.
//
// CTA = 4 warps over one (b, kv-head) and a chunk of groups (warps interleave groups).
// Tokens past the last group whose Keys and Values are both packed (the full-precision
// window, a partially aged Value tile) are processed lane-parallel over channels (each
// lane owns D/32 channels) with the same online-softmax state. Partials (m, l, acc) go to
// the split-K combine kernel shared with the generic path.
#include <algorithm>
#include <cmath>

#include "attention.cuh"

namespace kvb {

namespace {

constexpr int kMmaWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

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

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x2_trans(uint32_t& b0, uint32_t& b1, const void* row_addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];\n"
               : "=r"(b0), "=r"(b1)
               : "r"(smem_u32(row_addr)));
}

// (a & MASK) | c in one LOP3 (MASK as the immediate, the magic in a register)
template <uint32_t MASK>
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(d) : "r"(a), "n"(MASK), "r"(c));
  return d;
}

// (2^10 + v_lo, 2^10 + v_hi) - 2^10 -> exact (v_lo, v_hi), normal fp16
__device__ __forceinline__ uint32_t sub_magic(uint32_t x) {
  __half2 v = *reinterpret_cast<__half2*>(&x);
  v = __hsub2(v, __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400)));
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- unpack ---------------------------------------------------------------------------
// Slots per 16-bit half: 16/B. With the class trick slot position p lives at bit offset
// off(p) of either w (low positions) or w >> SH (high positions), giving value c * 2^off.
template <int B>
struct Cls;
template <>
struct Cls<2> {  // positions 0..4 from w (offsets 0,2,..,8), 5..7 from w >> 10
  static constexpr int SPH = 8;
  __host__ __device__ static constexpr int split() { return 5; }
  __host__ __device__ static constexpr int sh() { return 10; }
  __host__ __device__ static constexpr int off(int p) { return 2 * (p < 5 ? p : p - 5); }
};
template <>
struct Cls<4> {  // positions 0,1 from w (offsets 0,4), 2,3 from w >> 8
  static constexpr int SPH = 4;
  __host__ __device__ static constexpr int split() { return 2; }
  __host__ __device__ static constexpr int sh() { return 8; }
  __host__ __device__ static constexpr int off(int p) { return 4 * (p < 2 ? p : p - 2); }
};
template <>
struct Cls<3> {  // 2-bit low plane at positions 0..3 of w / w >> 8 (hi bit lands at off+2 <= 8)
  static constexpr int SPH = 8;
  __host__ __device__ static constexpr int split() { return 4; }
  __host__ __device__ static constexpr int sh() { return 8; }
  __host__ __device__ static constexpr int off(int p) { return 2 * (p < 4 ? p : p - 4); }
};

template <int B, int NS>
struct Unpacker {
  // class trick valid iff the offset depends on the slot only: NS % SPH == 0
  static constexpr bool kClass = (NS % Cls<B>::SPH) == 0;
  // exponent of the power of two carried by slot s (the bit offset of its codes)
  __host__ __device__ static constexpr int exp_of_slot(int s) { return kClass ? Cls<B>::off(s % Cls<B>::SPH) : 0; }
  // Codes at offset >= kSubMin are handed to the tensor core as fp16 SUBNORMALS (exponent
  // field 0, value c * 2^(off-24), one LOP3): HMMA consumes subnormal inputs exactly but
  // aligns their products to the nominal 2^-14 exponent, so codes with many leading zeros
  // lose product bits (profiles/probes/hmma_hilo_prec.cu: 1e-6 vs 2e-8 relative). Low
  // offsets therefore use the exact magic form (OR 2^10, subtract 2^10 -> c * 2^off,
  // LOP3 + HADD2), high offsets (>= 4, at most 4 leading zeros) the subnormal form.
  static constexpr int kSubMin = 4;
  // power-of-two factor of the operand value relative to the code: 2^(off) or 2^(off-24)
  __host__ __device__ static constexpr bool is_sub(int s) { return kClass && B != 3 && exp_of_slot(s) >= kSubMin; }
  __host__ __device__ static constexpr int val_exp_of_slot(int s) { return exp_of_slot(s) - (is_sub(s) ? 24 : 0); }
  // some slot is subnormal (then the Key GEMV keeps magic and subnormal slots in separate
  // accumulator chains and joins them as chain_magic + 2^24 * chain_sub)
  static constexpr bool kHasSub = kClass && B != 3 && Cls<B>::off(Cls<B>::SPH - 1) >= kSubMin;

  __device__ __forceinline__ static uint32_t frag(const uint32_t* w, int r, int s) {
    const int vs = r * NS + s;
    if constexpr (B == 3) {
      // low 2 bits from the 2-bit plane w[0..NS/2), high bit from the 1-bit plane w[NS/2..)
      const uint32_t hw = w[NS / 2 + (vs >> 4)];
      const int hb = vs & 15;  // bit of the high plane in each half
      if constexpr (kClass) {
        const int p = vs & 7;
        const int o = Cls<3>::off(p);
        const uint32_t lw = p < Cls<3>::split() ? w[vs >> 3] : (w[vs >> 3] >> Cls<3>::sh());
        const int tgt = o + 2;
        const uint32_t hs = hb >= tgt ? (hw >> (hb - tgt)) : (hw << (tgt - hb));
        return sub_magic((lw & (0x00030003u << o)) | (hs & (0x00010001u << tgt)) | 0x64006400u);
      } else {
        const uint32_t lo = (w[vs >> 3] >> (2 * (vs & 7))) & 0x00030003u;
        const uint32_t hi = (hw >> hb) & 0x00010001u;
        return sub_magic(lo | (hi << 2) | 0x64006400u);
      }
    } else {
      constexpr int SPH = Cls<B>::SPH;
      constexpr uint32_t MASK = B == 2 ? 0x00030003u : 0x000F000Fu;
      const uint32_t word = w[vs / SPH];
      if constexpr (kClass) {
        const int p = vs % SPH;
        const uint32_t src = p < Cls<B>::split() ? word : (word >> Cls<B>::sh());
        const int o = Cls<B>::off(p);
        if (o >= kSubMin) return src & (MASK << o);  // subnormal operand
        const uint32_t magic = 0x64006400u;
        return sub_magic(o == 0 ? and_or<MASK>(src, magic) : and_or<(MASK << 2)>(src, magic));
      } else {
        return sub_magic(((word >> (B * (vs % SPH))) & MASK) | 0x64006400u);
      }
    }
  }
};

// Lane's words of one tile in shared memory (layout: plane_addr in common.cuh).
template <int B, int D>
__device__ __forceinline__ void lds_tile(const uint32_t* tile, int lane, uint32_t* w) {
  if constexpr (B == 3) {
    lds_tile<2, D>(tile, lane, w);
    lds_tile<1, D>(tile + 32 * (D / 32), lane, w + D / 32);
  } else {
    constexpr int WPL = D * B / 64;
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
}

template <int D, int B>
constexpr int lane_words() {
  return B == 3 ? D * 3 / 64 : D * B / 64;
}

__device__ __forceinline__ float pow2i(int e) { return __int_as_float((127 + e) << 23); }

// 2^x via MUFU.EX2 without the denormal fix-up (x <= 0 here; 2^x < 2^-126 flushes to 0)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// (hi, lo) fp16 split of x packed as {hi | lo << 16}: x ~= hi + lo to ~22 bits. Two values
// at a time through the packed converter (F2FP) instead of four scalar F2F on the XU pipe.
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& p0, uint32_t& p1) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  const uint32_t hu = *reinterpret_cast<const uint32_t*>(&h), lu = *reinterpret_cast<const uint32_t*>(&l);
  p0 = __byte_perm(hu, lu, 0x5410);
  p1 = __byte_perm(hu, lu, 0x7632);
}

struct MmaParams {
  SideView k, v;
  const void* q;
  int q16, tail16;
  int H, Hq, tq, rows, gs, cg;
  int64_t T, P;  // total tokens; fast-path limit (multiple of gs)
  // stream-K work list: per (b, kv-head) U = Gf fast groups + ceil((T - P) / kTailUnit)
  // tail units, N = BH * U units in bh-major order; warp w of W takes [w N / W, (w+1) N / W)
  int Gf, U, N;  // 32-bit: the host falls back to the generic path beyond 2^31 units
  int Grec;      // group records per (b, kv-head) (bh stride of the record array)
  int W;
  int stages;
  uint32_t kt_bytes, vt_bytes, vm_bytes, km_bytes;  // per-group copy sizes
  uint32_t stage_bytes;
  float inv;  // 1/sqrt(D)
  int want_cs;  // accumulate the double scores checksum (only when the caller asks)
  float2* part_ml;  // partial slot of (warp w, bh) = w + bh (unique along the staircase)
  float* part_acc;
  double* part_cs;
};

constexpr int kTailUnit = 8;  // full-precision-window tokens per work unit (~ one group's cost)

// Dequantized packed element (token j < quantized, channel d) with compile-time D (gs is a
// compile-time constant too when the kernel is instantiated with GS): the tail path's
// per-element cost without runtime divisions.
template <int D, bool KEY, int BITS>
__device__ __forceinline__ float deq_lane(const SideView& s, int bh, int j, int d, int gs) {
  const uint32_t* tile = s.tiles + tile_index(s, bh, j >> 4);
  const uint32_t code = tile_get(tile, KEY ? key_coord(j & 15, d) : value_coord(j & 15, d), D, BITS);
  uint32_t m;
  bool narrow = false;
  if (KEY) {
    const int grp = j / gs;
    m = s.meta[kmeta_index(s, bh, grp) + d];
    if (BITS == 3) narrow = narrow_key(bh, d, D, s.info[grp], j - grp * gs);
  } else {
    m = s.meta[vmeta_index(s, bh, j) + d / gs];
    if (BITS == 3) narrow = narrow_value(bh, d, D, s.info[j]);
  }
  return decode(code, meta_scale(m), meta_min(m), narrow);
}

__device__ __forceinline__ float tail_val(const SideView& s, bool f16, int bh, int64_t j, int d, int D) {
  return f16 ? tail_at<__half>(s, bh, j, d, D) : tail_at<float>(s, bh, j, d, D);
}

// Per-warp shared layout (bytes), dynamic:
//   ring[S][stage_bytes] | bk[D][NB*8] half | bv[2][CGMAX][16][8] half | bp[2][16][8] half |
//   bars[S] u64. B rows are 16 bytes (8 columns) so ldmatrix.trans yields the fragments.
template <int D, int NB, int CGMAX>
struct WarpLayout {
  static constexpr int kBk = D * NB * 8 * 2;
  static constexpr int kBv = 2 * CGMAX * 16 * 8 * 2;
  static constexpr int kBp = 2 * 16 * 8 * 2;
  static constexpr int kPV = kBv + kBp;
  __host__ __device__ static size_t bytes(int stages, uint32_t stage_bytes) {
    const size_t n = (size_t)stages * stage_bytes + kBk + kPV + (size_t)stages * 8;
    return (n + 127) / 128 * 128;  // keep every warp's ring 128-byte aligned
  }
};

// GS: 0 = runtime group size, else compile-time (32 is the KVmix default).
template <int D, int KB, int VB, int R, int GS>
__global__ void __launch_bounds__(kMmaWarps * 32, 4) attend_mma_kernel(MmaParams p) {
  constexpr int NS = D / 16;                   // k-steps (Keys) / m-tiles (Values)
  constexpr int KW = lane_words<D, KB>();      // words per lane, Key tile
  constexpr int VW = lane_words<D, VB>();      // words per lane, Value tile
  constexpr int LC = D / 32;                   // channels per lane for meta / q / tail
  constexpr bool K3 = KB == 3;
  constexpr int NCOL = 2 * R + (K3 ? 22 * R : 0);
  constexpr int NB = (NCOL + 7) / 8;           // 8-column MMA blocks for the Key GEMV
  constexpr int CGMAX = GS ? D / GS : 8;       // channel groups held in the P.V staging
  using WL = WarpLayout<D, NB, CGMAX>;
  using UK = Unpacker<KB, NS>;
  using UV = Unpacker<VB, NS>;
  static_assert(!K3 || R <= 2, "3-bit Keys support up to 2 query rows per KV head");
  // bias MMA A operand straight from the staged Value meta rows (16 B = 4 groups per token)
  constexpr bool kMetaRows = GS != 0 && D / (GS ? GS : 1) == 4;

  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ float s_acc[kMmaWarps][R][D];
  __shared__ float s_bias[kMmaWarps][R][8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wg = blockIdx.x * kMmaWarps + warp;  // warps are independent: no CTA barriers
  if (wg >= p.W) return;
  const int g = lane >> 2, t = lane & 3;
  const int G = p.Hq / p.H;
  const int gs = GS ? GS : p.gs;
  const int CG = GS ? D / GS : p.cg;
  const int TPG = gs / 16;  // tiles per group
  const int S = p.stages;
  const int u_beg = (int)((int64_t)wg * p.N / p.W), u_end = (int)((int64_t)(wg + 1) * p.N / p.W);

  uint8_t* wbase = dsm + (size_t)warp * WL::bytes(S, p.stage_bytes);
  uint8_t* ring = wbase;
  __half* bk = reinterpret_cast<__half*>(ring + (size_t)S * p.stage_bytes);            // [D][NB*8]
  uint8_t* pv = reinterpret_cast<uint8_t*>(bk) + WL::kBk;
  uint4(*bv)[CGMAX][16] = reinterpret_cast<uint4(*)[CGMAX][16]>(pv);          // [tile][cg][token] -> 8 cols
  uint4(*bp)[16] = reinterpret_cast<uint4(*)[16]>(pv + WL::kBv);              // [tile][token] -> 8 cols
  uint64_t* bars = reinterpret_cast<uint64_t*>(pv + WL::kPV);

  // zero the B staging (columns of absent query rows must stay 0)
  {
    uint4* z = reinterpret_cast<uint4*>(bk);
    for (int i = lane; i < (WL::kBk + WL::kPV) / 16; i += 32) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();

  const bool row_ok = t < p.rows;
  const uint64_t policy = evict_first_policy();

  // producer: this warp's fast groups in work-list order, issued S ahead of the consumer
  int i_bh = u_beg / p.U, i_g = u_beg - i_bh * p.U;
  if (i_g >= p.Gf) {
    ++i_bh;
    i_g = 0;
  }
  auto issue_next = [&](int s) {
    if (p.Gf > 0 && i_bh * p.U + i_g < u_end) {
      if (lane == 0) {
        // the group's record (K tiles | V tiles | V meta | K meta) is one contiguous range
        const uint32_t* src = p.k.tiles + ((size_t)i_bh * p.Grec + i_g) * (p.stage_bytes / 4);
        mbar_arrive_expect_tx(&bars[s], p.stage_bytes);
        bulk_g2s(ring + (size_t)s * p.stage_bytes, src, p.stage_bytes, &bars[s], policy);
      }
      if (++i_g == p.Gf) {
        ++i_bh;
        i_g = 0;
      }
    }
  };
  for (int s = 0; s < S; ++s) issue_next(s);

  float accv[NS][4];
  float accb[4];
  float m_run, l_run;  // row t (threads with t < rows)
  double cs;

  auto rescale = [&](float alpha) {
    if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        accv[i][0] *= alpha;
        accv[i][1] *= alpha;
        accv[i][2] *= alpha;
        accv[i][3] *= alpha;
      }
      accb[0] *= alpha;
      accb[1] *= alpha;
      accb[2] *= alpha;
      accb[3] *= alpha;
    }
  };

  // channel group of each Value m-tile
  int cg_of[NS];
#pragma unroll
  for (int mt = 0; mt < NS; ++mt) cg_of[mt] = (mt * 16) / gs;

  // the k-step of this lane's channels and the power of two its A codes carry
  float cls_scale = 1.f;
  {
    const int kk = (lane * LC) / 16;
#pragma unroll
    for (int x = 0; x < NS; ++x)
      if (x == kk) cls_scale = pow2i(-UK::exp_of_slot(x));
  }

  int s = 0;
  uint32_t phase = 0;
  for (int u = u_beg; u < u_end;) {
    // ---- one (b, kv-head) segment of the work list ----------------------------------------
    const int bh = u / p.U;
    const int lo = u - bh * p.U;
    const int hi = min(u_end - bh * p.U, p.U);
    u = bh * p.U + hi;
    const int b = bh / p.H, h = bh % p.H;

    // query rows: lane owns channels [lane*LC, lane*LC+LC)
    float qv[R][LC];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int rr = r < p.rows ? r : 0;
      const int gi = rr / p.tq, qi = rr % p.tq;
      const size_t off = (((size_t)b * p.Hq + h * G + gi) * p.tq + qi) * D + lane * LC;
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const float x = p.q16 ? __half2float(static_cast<const __half*>(p.q)[off + c]) : static_cast<const float*>(p.q)[off + c];
        qv[r][c] = r < p.rows ? x : 0.f;
      }
    }
    m_run = -INFINITY;
    l_run = 0.f;
#pragma unroll
    for (int i = 0; i < NS; ++i) accv[i][0] = accv[i][1] = accv[i][2] = accv[i][3] = 0.f;
    accb[0] = accb[1] = accb[2] = accb[3] = 0.f;
    cs = 0.0;

  const int g_stop = min(hi, p.Gf);
  for (int grp = lo; grp < g_stop; ++grp) {
    mbar_wait(&bars[s], phase);
    const uint8_t* st = ring + (size_t)s * p.stage_bytes;
    const uint32_t* kt = reinterpret_cast<const uint32_t*>(st);
    const uint32_t* vt = reinterpret_cast<const uint32_t*>(st + p.kt_bytes);
    const uint32_t* vm = reinterpret_cast<const uint32_t*>(st + p.kt_bytes + p.vt_bytes);
    const uint32_t* km = reinterpret_cast<const uint32_t*>(st + p.kt_bytes + p.vt_bytes + p.vm_bytes);

    // ---- Key group: B operand (q*s split hi/lo, pre-scaled by 2^(e - class) per row) ----
    float beta[R], inv_sig[R];
    {
      float sc[LC], mn[LC];
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const uint32_t m = km[lane * LC + c];
        sc[c] = meta_scale(m);
        mn[c] = meta_min(m);
      }
      int tau[LC];
      if constexpr (K3) {
        const int2 inf = __ldg(p.k.info + grp);  // {segment length, token offset of the group}
        const int nmod = inf.x % 11, omod = inf.y % 11;
#pragma unroll
        for (int c = 0; c < LC; ++c) {
          const int cmod = (int)(((unsigned)bh * D + lane * LC + c) % 11u);
          const int phi = (cmod * nmod + omod) % 11;  // stream index % 11 of the group's first token
          tau[c] = (21 - phi) % 11;                   // narrow tokens: t = tau (mod 11)
        }
      }
      uint32_t row[LC][NB * 4];  // this lane's B rows (channel-major), packed half2
#pragma unroll
      for (int c = 0; c < LC; ++c)
#pragma unroll
        for (int j = 0; j < NB * 4; ++j) row[c][j] = 0u;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float qs[LC], mx = 0.f, bt = 0.f;
#pragma unroll
        for (int c = 0; c < LC; ++c) {
          qs[c] = qv[r][c] * sc[c];
          mx = fmaxf(mx, fabsf(qs[c]));
          bt = fmaf(qv[r][c], mn[c], bt);
          if constexpr (K3) mx = fmaxf(mx, fabsf(qv[r][c] * (wide_scale(sc[c]) - sc[c])));
        }
        // max over the warp on the (non-negative) float bits: one REDUX
        const uint32_t mxu = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
        // sigma = 2^(14 - floor(log2 max|qs|)): max|qs*sigma| in [2^14, 2^15)
        const int e = (int)((mxu >> 23) & 0xffu);
        const int se = min(max(268 - e, 1), 254);
        inv_sig[r] = __int_as_float((254 - se) << 23);  // 1 / sigma
        const float sgc = __int_as_float(se << 23) * cls_scale;
#pragma unroll
        for (int c = 0; c < LC; c += 2) split2(qs[c] * sgc, qs[c + 1] * sgc, row[c][r], row[c + 1][r]);
        if constexpr (K3) {
#pragma unroll
          for (int c = 0; c < LC; ++c) {
            const float y = qv[r][c] * (wide_scale(sc[c]) - sc[c]) * sgc;
            const __half yh = __float2half_rn(y);
            const __half yl = __float2half_rn(y - __half2float(yh));
            const uint32_t yp = (uint32_t)__half_as_ushort(yh) | ((uint32_t)__half_as_ushort(yl) << 16);
#pragma unroll
            for (int xr = 0; xr < 11; ++xr) row[c][R + r * 11 + xr] = tau[c] == xr ? yp : 0u;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bt += __shfl_xor_sync(0xffffffffu, bt, o);
        beta[r] = bt;
      }
      __syncwarp();  // previous group's ldmatrix reads of bk are done
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(bk + (size_t)(lane * LC + c) * NB * 8);
        if constexpr (K3) {
#pragma unroll
          for (int j = 0; j < NB; ++j)
            reinterpret_cast<uint4*>(dst)[j] = make_uint4(row[c][4 * j], row[c][4 * j + 1], row[c][4 * j + 2], row[c][4 * j + 3]);
        } else {
          // columns of absent rows stay zero from the kernel prologue
#pragma unroll
          for (int j = 0; j < R; ++j) dst[j] = row[c][j];
        }
      }
    }
    __syncwarp();
    float my_beta = beta[0], my_isig = inv_sig[0];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      if (t == r) {
        my_beta = beta[r];
        my_isig = inv_sig[r];
      }
    }

    // ---- the group's tiles, two at a time (independent MMA chains, one softmax round) ----
    for (int tp = 0; tp < TPG; tp += 2) {
      uint32_t kw[2][KW], vw[2][VW];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        lds_tile<KB, D>(kt + (size_t)(tp + u) * tile_words(D, KB), lane, kw[u]);
        lds_tile<VB, D>(vt + (size_t)(tp + u) * tile_words(D, VB), lane, vw[u]);
      }
      // scores: K (16 tokens x D) . B, both tiles
      // NB == 1: two accumulator chains per tile (magic / subnormal slots, else even / odd
      // k-steps) halve the HMMA dependency chain; NB > 1 already has NB independent chains
      constexpr int NCH = NB == 1 ? 2 : 1;
      float dk[2][NB * NCH][4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int nb = 0; nb < NB * NCH; ++nb) dk[u][nb][0] = dk[u][nb][1] = dk[u][nb][2] = dk[u][nb][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < NS; ++kk) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          uint32_t b0, b1;
          ldmatrix_x2_trans(b0, b1, bk + (size_t)(16 * kk + (lane & 15)) * NB * 8 + nb * 8);
          const int acc = NCH == 2 ? (UK::kHasSub ? (UK::is_sub(kk) ? 1 : 0) : (kk & 1)) : nb;
#pragma unroll
          for (int u = 0; u < 2; ++u)
            mma16816(dk[u][acc], UK::frag(kw[u], 0, kk), UK::frag(kw[u], 1, kk), UK::frag(kw[u], 2, kk),
                     UK::frag(kw[u], 3, kk), b0, b1);
        }
      }
      if constexpr (NCH == 2) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int e = 0; e < 4; ++e) dk[u][0][e] = fmaf(UK::kHasSub ? 16777216.f : 1.f, dk[u][1][e], dk[u][0][e]);
      }
      float sa[2], sb[2];  // row t: token g / token g+8 of each tile
      if constexpr (K3) {
        // residue-class corrections without shared memory: for token row x the column pair
        // of residue class (tile*16 + row) % 11 lives in lane (row, t_src); every lane of
        // row `g` computes the same source, so the source lane itself knows which register
        // block to expose, and one shuffle per (row, query row) delivers it.
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
          for (int hlf = 0; hlf < 2; ++hlf) {  // token g, then token g+8
            const int x = ((tp + u) * 16 + g + 8 * hlf) % 11;
            float tot = 0.f;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int col = 2 * R + (r * 11 + x) * 2;     // even: hi, odd: lo
              const int nb = col >> 3, tsrc = (col & 7) >> 1;
              float mine = 0.f;                              // this lane's (hi+lo) in block nb
#pragma unroll
              for (int q = 0; q < NB; ++q)
                if (q == nb) mine = dk[u][q][2 * hlf] + dk[u][q][2 * hlf + 1];
              const float corr = __shfl_sync(0xffffffffu, mine, g * 4 + tsrc);
              if (r == t) tot = corr;
            }
            const float mainv = dk[u][0][2 * hlf] + dk[u][0][2 * hlf + 1];
            if (hlf == 0) sa[u] = mainv + tot;
            else sb[u] = mainv + tot;
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          sa[u] = dk[u][0][0] + dk[u][0][1];
          sb[u] = dk[u][0][2] + dk[u][0][3];
        }
      }
      float la[2], lb[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        sa[u] = (sa[u] * my_isig + my_beta) * p.inv;
        sb[u] = (sb[u] * my_isig + my_beta) * p.inv;
        la[u] = sa[u] * kLog2e;
        lb[u] = sb[u] * kLog2e;
      }
      if (p.want_cs && row_ok) cs += (double)((sa[0] + sb[0]) + (sa[1] + sb[1]));
      float tmax = fmaxf(fmaxf(la[0], lb[0]), fmaxf(la[1], lb[1]));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
      const float m_new = fmaxf(m_run, tmax);
      const float alpha = fast_exp2(m_run - m_new);
      float pa[2], pb[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        pa[u] = row_ok ? fast_exp2(la[u] - m_new) : 0.f;
        pb[u] = row_ok ? fast_exp2(lb[u] - m_new) : 0.f;
      }
      l_run = l_run * alpha + ((pa[0] + pb[0]) + (pa[1] + pb[1]));
      m_run = m_new;
      rescale(alpha);

      // ---- P.V B operands: lane j -> token j of the 32 (tile j/16, row-in-tile j%16) ----
      // each (token, group) row is 8 fp16 columns {hi_r, lo_r}: one 16-byte store per row
      {
        const int u = lane >> 4, i = lane & 15;
        const uint32_t* vmt = vm + (size_t)(tp * 16 + lane) * CG;  // this token's Value meta
        float vsc[CGMAX];
        if constexpr (kMetaRows) {
          const uint4 q4 = *reinterpret_cast<const uint4*>(vmt);
          vsc[0] = meta_scale(q4.x);
          vsc[1] = meta_scale(q4.y);
          vsc[2] = meta_scale(q4.z);
          vsc[3] = meta_scale(q4.w);
        } else {
#pragma unroll
          for (int c = 0; c < CGMAX; ++c) vsc[c] = (GS || c < CG) ? meta_scale(vmt[c]) : 0.f;
        }
        uint32_t prow[4] = {0u, 0u, 0u, 0u};
        uint32_t vrow[CGMAX][4];
#pragma unroll
        for (int c = 0; c < CGMAX; ++c) vrow[c][0] = vrow[c][1] = vrow[c][2] = vrow[c][3] = 0u;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int src = (i & 7) * 4 + r;
          const float x0 = __shfl_sync(0xffffffffu, pa[0], src);
          const float x1 = __shfl_sync(0xffffffffu, pb[0], src);
          const float x2 = __shfl_sync(0xffffffffu, pa[1], src);
          const float x3 = __shfl_sync(0xffffffffu, pb[1], src);
          const float pj = u == 0 ? (i < 8 ? x0 : x1) : (i < 8 ? x2 : x3);  // 0 for absent rows
          float xs[CGMAX + 1];
          xs[0] = pj;
#pragma unroll
          for (int c = 0; c < CGMAX; ++c) xs[c + 1] = pj * vsc[c];
          uint32_t pk[CGMAX + 2];
#pragma unroll
          for (int c = 0; c < CGMAX + 1; c += 2) split2(xs[c], c + 1 <= CGMAX ? xs[c + 1] : 0.f, pk[c], pk[c + 1]);
          prow[r] = pk[0];
#pragma unroll
          for (int c = 0; c < CGMAX; ++c) vrow[c][r] = pk[c + 1];
        }
        bp[u][i] = make_uint4(prow[0], prow[1], prow[2], prow[3]);
#pragma unroll
        for (int c = 0; c < CGMAX; ++c)
          if (GS || c < CG) bv[u][c][i] = make_uint4(vrow[c][0], vrow[c][1], vrow[c][2], vrow[c][3]);
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        uint32_t pb0, pb1;
        ldmatrix_x2_trans(pb0, pb1, &bp[u][lane & 15]);
        // bias MMA: A rows = per-token meta halves, B = p
        uint32_t a0 = 0u, a2 = 0u;
        if constexpr (kMetaRows) {
          // rows = {s0, m0, s1, m1, s2, m2, s3, m3} of the 16 tokens (ldmatrix.trans of the
          // staged 16-byte meta rows): odd rows give sum_j m_jg p_j, even rows sum_j s_jg p_j
          ldmatrix_x2_trans(a0, a2, vm + (size_t)((tp + u) * 16 + (lane & 15)) * CG);
        } else {
          const uint32_t* vmt = vm + (size_t)(tp + u) * 16 * CG;  // [16][CG]
          if (g < CG) {
            a0 = __byte_perm(vmt[(2 * t) * CG + g], vmt[(2 * t + 1) * CG + g], 0x7632);
            a2 = __byte_perm(vmt[(2 * t + 8) * CG + g], vmt[(2 * t + 9) * CG + g], 0x7632);
          }
        }
        mma16816(accb, a0, 0u, a2, 0u, pb0, pb1);
        if constexpr (GS != 0) {
          constexpr int CGC = D / GS;
          uint32_t bf0[CGC], bf1[CGC];
#pragma unroll
          for (int c = 0; c < CGC; ++c) ldmatrix_x2_trans(bf0[c], bf1[c], &bv[u][c][lane & 15]);
#pragma unroll
          for (int mt = 0; mt < NS; ++mt) {
            const int c = (mt * 16) / GS;
            mma16816(accv[mt], UV::frag(vw[u], 0, mt), UV::frag(vw[u], 1, mt), UV::frag(vw[u], 2, mt),
                     UV::frag(vw[u], 3, mt), bf0[c], bf1[c]);
          }
        } else {
#pragma unroll
          for (int mt = 0; mt < NS; ++mt) {
            uint32_t b0, b1;
            ldmatrix_x2_trans(b0, b1, &bv[u][cg_of[mt]][lane & 15]);
            mma16816(accv[mt], UV::frag(vw[u], 0, mt), UV::frag(vw[u], 1, mt), UV::frag(vw[u], 2, mt),
                     UV::frag(vw[u], 3, mt), b0, b1);
          }
        }
      }
      __syncwarp();
    }
    // refill this stage S groups ahead
    issue_next(s);
    if (++s == S) {
      s = 0;
      phase ^= 1u;
    }
  }

  // ---- tokens past the fast region: lane-parallel over channels ------------------------
  // Every lane tracks all R rows (identical values across lanes); the Value contribution
  // accumulates per lane for its LC channels and joins the fragments in the epilogue.
  float acct[R][LC];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < LC; ++c) acct[r][c] = 0.f;
  const int64_t j_lo = p.P + (int64_t)max(lo - p.Gf, 0) * kTailUnit;
  const int64_t j_hi = hi > p.Gf ? min(p.T, p.P + (int64_t)(hi - p.Gf) * kTailUnit) : j_lo;
  if (j_lo < j_hi) {
    float m_all[R], l_all[R];
    {
      float lr = l_run;
      lr += __shfl_xor_sync(0xffffffffu, lr, 4);
      lr += __shfl_xor_sync(0xffffffffu, lr, 8);
      lr += __shfl_xor_sync(0xffffffffu, lr, 16);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        m_all[r] = __shfl_sync(0xffffffffu, m_run, r);  // lane r = (g 0, t r)
        l_all[r] = __shfl_sync(0xffffffffu, lr, r);
      }
    }
    const int d0 = lane * LC;
    for (int64_t j = j_lo; j < j_hi; ++j) {
      float kx[LC], vx[LC];
      if (j >= p.k.quantized) {
#pragma unroll
        for (int c = 0; c < LC; ++c) kx[c] = tail_val(p.k, p.tail16, bh, j - p.k.quantized, d0 + c, D);
      } else {
#pragma unroll
        for (int c = 0; c < LC; ++c) kx[c] = deq_lane<D, true, KB>(p.k, bh, (int)j, d0 + c, gs);
      }
      if (j >= p.v.quantized) {
#pragma unroll
        for (int c = 0; c < LC; ++c) vx[c] = tail_val(p.v, p.tail16, bh, j - p.v.quantized, d0 + c, D);
      } else {
#pragma unroll
        for (int c = 0; c < LC; ++c) vx[c] = deq_lane<D, false, VB>(p.v, bh, (int)j, d0 + c, gs);
      }
      float alpha_mine = 1.f;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float x = 0.f;
#pragma unroll
        for (int c = 0; c < LC; ++c) x = fmaf(qv[r][c], kx[c], x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (r < p.rows) {
          const float sc = x * p.inv;
          if (p.want_cs && lane == 0) cs += (double)sc;
          const float ls = sc * kLog2e;
          const float m_new = fmaxf(m_all[r], ls);
          const float alpha = exp2f(m_all[r] - m_new);
          const float pj = exp2f(ls - m_new);
          l_all[r] = l_all[r] * alpha + pj;
          m_all[r] = m_new;
#pragma unroll
          for (int c = 0; c < LC; ++c) acct[r][c] = acct[r][c] * alpha + pj * vx[c];
          if (t == r) alpha_mine = alpha;
        }
      }
      rescale(alpha_mine);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (t == r) {
        m_run = m_all[r];
        l_run = g == 0 ? l_all[r] : 0.f;
      }
    }
  }

  // ---- segment epilogue: this warp's partial for (b, kv-head) -> slot wg + bh ----------
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 4);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 8);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
  if (row_ok && t < R) {
    // the Value fragments carry the per-m-tile power of two of their operands
#pragma unroll
    for (int mt = 0; mt < NS; ++mt) {
      const float f = pow2i(-UV::val_exp_of_slot(mt));
      s_acc[warp][t][mt * 16 + g] = (accv[mt][0] + accv[mt][1]) * f;
      s_acc[warp][t][mt * 16 + g + 8] = (accv[mt][2] + accv[mt][3]) * f;
    }
    if constexpr (kMetaRows) {
      if (g & 1) s_bias[warp][t][g >> 1] = accb[0] + accb[1];  // min rows
    } else {
      s_bias[warp][t][g] = accb[0] + accb[1];
    }
  }
  __syncwarp();
  const int64_t slot = (int64_t)wg + bh;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const float m_r = __shfl_sync(0xffffffffu, m_run, r);
    const float l_r = __shfl_sync(0xffffffffu, l_run, r);
    if (r < p.rows) {
      const size_t pi = (size_t)slot * p.rows + r;
      float o[LC];
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const int d = lane * LC + c;
        o[c] = s_acc[warp][r][d] + s_bias[warp][r][d / gs] + acct[r][c];
      }
      if constexpr (LC == 4) {
        *reinterpret_cast<float4*>(p.part_acc + pi * D + lane * LC) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
#pragma unroll
        for (int c = 0; c < LC; ++c) p.part_acc[pi * D + lane * LC + c] = o[c];
      }
      if (lane == 0) p.part_ml[pi] = make_float2(m_r == -INFINITY ? -INFINITY : m_r * kLn2, l_r);
    }
  }
  if (p.want_cs) {
    for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
    if (lane == 0) p.part_cs[slot] = cs;
  }
  __syncwarp();  // s_acc / s_bias are rewritten by the next segment
  }
}

// Combine the stream-K partials of each (b, kv-head): the warps whose unit ranges meet
// [bh U, (bh+1) U), slot w + bh, merged in warp order (deterministic).
__global__ void attend_combine_sk_kernel(const float2* __restrict__ part_ml, const float* __restrict__ part_acc,
                                         int N, int W, int U, int R, int H, int Hq, int tq, int D,
                                         float* __restrict__ out) {
  const int bh = blockIdx.x, r = blockIdx.y;
  const int b = bh / H, h = bh % H, G = Hq / H;
  const int gi = r / tq, qi = r % tq;
  const int hq = h * G + gi;
  const int w0 = (int)((((int64_t)bh * U + 1) * W - 1) / N);
  const int w1 = (int)((((int64_t)bh + 1) * U * W - 1) / N);  // 64-bit products
  float M = -INFINITY;
  for (int w = w0; w <= w1; ++w) M = fmaxf(M, part_ml[((size_t)w + bh) * R + r].x);
  float L = 0.f;
  for (int w = w0; w <= w1; ++w) {
    const float2 ml = part_ml[((size_t)w + bh) * R + r];
    if (ml.x != -INFINITY) L += ml.y * expf(ml.x - M);
  }
  const float invL = 1.0f / L;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float a = 0.f;
    for (int w = w0; w <= w1; ++w) {
      const float2 ml = part_ml[((size_t)w + bh) * R + r];
      if (ml.x != -INFINITY) a += part_acc[(((size_t)w + bh) * R + r) * D + d] * expf(ml.x - M);
    }
    out[(((size_t)b * Hq + hq) * tq + qi) * D + d] = a * invL;
  }
}

template <int D, int KB, int VB, int R, int GS>
int launch(MmaParams& p, int BH, Workspace& ws, cudaStream_t st) {
  constexpr int NCOL = 2 * R + (KB == 3 ? 22 * R : 0);
  constexpr int NB = (NCOL + 7) / 8;
  using WL = WarpLayout<D, NB, GS ? D / GS : 8>;
  auto kern = attend_mma_kernel<D, KB, VB, R, GS>;
  // ring depth: as many stages (2..4) as fit while keeping the highest CTA residency
  // the registers allow (4, else 3, else 2 CTAs per SM)
  static thread_local int static_smem = -1;
  if (static_smem < 0) {
    cudaFuncAttributes fa;
    check_cuda(cudaFuncGetAttributes(&fa, kern), "func attributes");
    static_smem = (int)fa.sharedSizeBytes;
  }
  const size_t fixed = WL::bytes(0, 0);
  int stages = 2;
  for (int occ_target = 4; occ_target >= 2; --occ_target) {
    const long per_cta = 227L * 1024 / occ_target - 1024 - static_smem;
    const long per_warp = per_cta / kMmaWarps - (long)fixed - 4 * 8 - 128;
    const long s_fit = per_warp / (long)p.stage_bytes;
    if (s_fit >= 2) {
      stages = (int)std::min<long>(4, s_fit);
      break;
    }
  }
  p.stages = stages;
  const size_t smem = (size_t)kMmaWarps * WL::bytes(p.stages, p.stage_bytes);
  check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  static thread_local size_t occ_smem = 0;
  static thread_local int occ = 0;
  if (occ_smem != smem) {  // residency of this instantiation at this ring size (cached)
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMmaWarps * 32, smem), "occupancy");
    occ_smem = smem;
  }
  // one resident wave of independent warps (persistent): equal unit ranges, no stragglers;
  // never more warps than units so every range is non-empty
  const int64_t wave = (int64_t)std::max(1, occ) * num_sms() * kMmaWarps;
  p.W = (int)std::max<int64_t>(1, std::min<int64_t>(p.N, wave));
  // partial slots w + bh < W + BH: scratch depends on (B, H, rows, D, SM count) only
  const size_t slots = (size_t)wave + BH;
  p.part_ml = ws.ml(st, slots * p.rows);
  p.part_acc = ws.acc(st, slots * p.rows * D);
  p.part_cs = ws.cs(st, slots + 1);
  if (p.want_cs) check_cuda(cudaMemsetAsync(p.part_cs, 0, (slots + 1) * sizeof(double), st), "memset");
  kern<<<(p.W + kMmaWarps - 1) / kMmaWarps, kMmaWarps * 32, smem, st>>>(p);
  return p.W;
}

template <int D, int KB, int VB, int R>
int dispatch_gs(MmaParams& p, int BH, Workspace& ws, cudaStream_t st) {
  if constexpr (KB == 3 && R > 2) {
    return 0;
  } else {
    return p.gs == 32 ? launch<D, KB, VB, R, 32>(p, BH, ws, st) : launch<D, KB, VB, R, 0>(p, BH, ws, st);
  }
}

template <int D, int R>
int dispatch_bits(MmaParams& p, int kb, int vb, int BH, Workspace& ws, cudaStream_t st) {
  switch (kb * 10 + vb) {
    case 22: return dispatch_gs<D, 2, 2, R>(p, BH, ws, st);
    case 24: return dispatch_gs<D, 2, 4, R>(p, BH, ws, st);
    case 42: return dispatch_gs<D, 4, 2, R>(p, BH, ws, st);
    case 44: return dispatch_gs<D, 4, 4, R>(p, BH, ws, st);
    case 32: return dispatch_gs<D, 3, 2, R>(p, BH, ws, st);
    case 34: return dispatch_gs<D, 3, 4, R>(p, BH, ws, st);
    default: return 0;
  }
}

}  // namespace


bool attend_mma(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
                Workspace& ws, cudaStream_t st) {
  const int rows = (Hq / c->H) * tq;
  if (rows > 4) return false;
  const int kb = c->k.bits, vb = c->v.bits;
  if (vb == 3 || (kb == 3 && rows > 2)) return false;
  const int D = c->D, gs = c->cfg.group_size;
  if (gs % 32 != 0) return false;  // groups are processed two tiles at a time
  if (D != 64 && D != 128) return false;
  const int BH = c->B * c->H;
  const int64_t T = c->total();
  MmaParams p{};
  p.k = view(c->k);
  p.v = view(c->v);
  p.q = q;
  p.q16 = dt == KVMIX_F16;
  p.tail16 = c->tail_dtype == KVMIX_F16;
  p.H = c->H;
  p.Hq = Hq;
  p.tq = tq;
  p.rows = rows;
  p.gs = gs;
  p.cg = c->cgroups();
  if (p.cg > 8) return false;
  p.T = T;
  p.P = (std::min(c->k.quantized, c->v.quantized) / gs) * gs;
  const int64_t U = p.P / gs + (T - p.P + kTailUnit - 1) / kTailUnit;
  if ((int64_t)BH * U >= (int64_t)1 << 31) return false;
  p.Gf = (int)(p.P / gs);
  p.U = (int)U;
  p.N = BH * p.U;
  p.kt_bytes = (uint32_t)((gs / 16) * c->k.tile_words * 4);
  p.vt_bytes = (uint32_t)((gs / 16) * c->v.tile_words * 4);
  p.vm_bytes = (uint32_t)(gs * p.cg * 4);
  p.km_bytes = (uint32_t)(D * 4);
  p.stage_bytes = p.kt_bytes + p.vt_bytes + p.vm_bytes + p.km_bytes;
  if ((size_t)p.stage_bytes != c->k.grp_stride * 4 || c->v.tiles != c->k.tiles + (gs / 16) * c->k.tile_words)
    return false;  // not the group-record layout this kernel streams
  if (c->k.bh_stride % c->k.grp_stride != 0 || c->k.bh_stride / c->k.grp_stride >= (1u << 31)) return false;
  p.Grec = (int)(c->k.bh_stride / c->k.grp_stride);
  if (p.vm_bytes % 16) return false;
  p.inv = 1.0f / sqrtf((float)D);
  p.want_cs = checksum != nullptr;
  const int R = rows <= 1 ? 1 : rows <= 2 ? 2 : 4;
  int W = 0;
#define KVB_DISPATCH_D(DD)                                                  \
  if (D == DD) {                                                            \
    if (R == 1) W = dispatch_bits<DD, 1>(p, kb, vb, BH, ws, st);           \
    else if (R == 2) W = dispatch_bits<DD, 2>(p, kb, vb, BH, ws, st);      \
    else W = dispatch_bits<DD, 4>(p, kb, vb, BH, ws, st);                  \
  }
  KVB_DISPATCH_D(64)
  KVB_DISPATCH_D(128)
#undef KVB_DISPATCH_D
  if (W == 0) return false;
  after_launch("attend_mma_kernel");
  attend_combine_sk_kernel<<<dim3(BH, rows), 128, 0, st>>>(p.part_ml, p.part_acc, p.N, p.W, p.U, rows, c->H, Hq, tq, D,
                                                           out);
  after_launch("attend_combine_sk_kernel");
  if (checksum) {
    const size_t nslot = (size_t)p.W + BH;
    checksum_kernel<<<1, 32, 0, st>>>(p.part_cs, nslot, p.part_cs + nslot);
    after_launch("checksum_kernel");
    check_cuda(cudaMemcpyAsync(checksum, p.part_cs + nslot, 8, cudaMemcpyDeviceToHost, st), "memcpy");
    check_cuda(cudaStreamSynchronize(st), "sync");
  }
  return true;
}

}  // namespace kvb
