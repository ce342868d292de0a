// attention_tc.cu -- decode attention over the packed groups on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, A operand in TMEM, B operand in shared memory, int32
// accumulators in TMEM), fed by TMA bulk copies. Serves the fast groups [0, Gf) of every
// (b, kv-head) of a D = 128, gs = 32 cache with 2/3/4-bit Keys and 2/4-bit Values and up to
// four query rows per KV head (GQA G <= 4) in ONE pass; the full-precision window and the
// merge of the split partials run in the window launch of attend_mma_kernel (attention_mma.cu,
// MmaParams::wonly), which reads this kernel's partials.
//
// Same factorization as attention_mma.cu (reference: attention.cpp:28-166):
//     q.k_j = sum_d (q_d s_gd) c_jd + sum_d q_d m_gd,   out_d = sum_j (p_j s_jg) c_jd + sum_j p_j m_jg
// with the codes as u8 A operands (one AND per 4 codes, carrying a per-channel power of two
// 2^(b*class), common.cuh) and the fp32 factors as B in fixed point, four base-256 digits in
// four MMA columns; integer products and int32 accumulation are exact.
//
// One CTA = 4 consumer warps (TMEM lane quarters) + an MMA-issue warp + a TMA warp; a TILE =
// 4 consecutive Key groups (128 tokens) of one (b, kv-head), one TMA bulk copy of the 4 group
// records into a ring stage.
//   * Scores: M = 128 tokens (warp w unpacks group w's Key codes into TMEM rows 32w..32w+31 with
//     tcgen05.st 16x256b -- the IMMA fragment layout of the cache maps onto it directly), K =
//     128 channels (+128 for the high-bit plane of 3-bit Keys), N = 4 groups x R rows x 4
//     digits: warp w writes the B digits of ITS group's q s into its own columns, so one MMA
//     scores the four groups (the cross-group columns are ignored). Thread = token reads its
//     R x 4 digit columns back (tcgen05.ld 32x32b).
//   * Values: M = 128 channels (warp w unpacks channels 32w..32w+31 of all four groups), K =
//     128 tokens (one k-step per group), N = R rows x 4 channel groups x 4 digits; the int32
//     accumulators persist in TMEM across tiles and are folded into fp32 registers (thread =
//     channel) only when the shared lazy reference max moves, the fixed-point exponent must
//     drop, or 256 tiles have accumulated.
//   * Online softmax: thread = token; the reference max / exponent are common to the CTA's
//     four warps (one accumulator), decided with ONE bar.red.or per tile on the common path
//     and a small exchange when it fires.
//   * Work: stream-K over the tiles of all (b, kv-head) in bh-major order, one contiguous tile
//     range per CTA (persistent, two CTAs per SM); every (CTA, bh) segment writes a partial
//     (m, l, acc) to slot CTA + bh.
#include "mma_common.cuh"

namespace kvb {

namespace {

constexpr int kTcCons = 4;              // consumer warps (TMEM lane quarters 0..3)
constexpr int kTcThreads = 6 * 32;      // + MMA warp (4) + TMA warp (5)
constexpr int kTcD = 128;
constexpr int kTcGS = 32;
constexpr int kTcFlushTiles = kFlushBlocks / 4;  // Value int32 accumulators (4 blocks per tile)

// ---- tcgen05 / TMEM primitives ---------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 16 lanes x 256 bits, 4 repetitions along the columns: register 4x + 2rb + y -> lane
// (lane/4) + 8 rb, column 8x + 2 (lane%4) + y (the m16n8 fragment map, probes/tc_i8_probe.cu)
__device__ __forceinline__ void sttm_16x256_x4(uint32_t ta, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16};\n" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// 32 lanes x 32 bits, 4 consecutive columns: thread = lane
__device__ __forceinline__ void ldtm_32x32_x4(uint32_t ta, int (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(ta)
               : "memory");
}

// shared-memory matrix descriptor, MN-major, no swizzle: element (k, n) at
// (k / 8) * lbo + (k % 8) * 16 + (n / 16) * sbo + n % 16 (bytes)
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// instruction descriptor, kind::i8: D s32, A u8 (K-major, TMEM), B u8 / s8 (MN-major), M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int n, bool b_signed) {
  return (2u << 4) | ((b_signed ? 1u : 0u) << 10) | (1u << 16) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"((int)acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// the consumer warps' named barrier (id 1, 128 threads); bar.red.or: any thread's predicate
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }
__device__ __forceinline__ bool cons_any(bool x) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, 1, 128, p;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
      : "=r"(r)
      : "r"((uint32_t)x)
      : "memory");
  return r != 0;
}

// order-preserving float <-> u32 (REDUX.MAX over signed floats, -inf included)
__device__ __forceinline__ uint32_t f2o(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t u) { return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u); }

struct TcParams {
  const uint8_t* rec;  // group records (kvmix_cache::rec): [bh][group] {K tiles | V tiles | V meta | K meta}
  SideView k;          // Key side (info, global bh for the Mixed3 narrow slots)
  const void* q;
  int q16;
  int H, Hq, tq, rows;  // rows = (Hq / H) * tq <= R
  int Gf, Tb, Grec;     // fast groups, tiles per (b, kv-head), records per (b, kv-head)
  int64_t NT;           // tiles
  int C;                // CTAs
  float inv;            // 1 / sqrt(D)
  int want_cs;
  int flush_tiles;
  float2* part_ml;  // [slot][R] (m in natural-log units, l)
  float* part_acc;  // [slot][R][D]
  double* part_cs;  // [slot]
};

template <int KB, int VB, int R>
struct TcGeo {
  static constexpr bool K3 = KB == 3;
  static constexpr int KT = K3 ? 256 : 128;  // K extent of the score MMA (3-bit Keys: two planes)
  static constexpr int NKS = KT / 32;        // score k-steps
  static constexpr int N = 16 * R;           // MMA N
  static constexpr uint32_t KTW = (uint32_t)tile_words(kTcD, KB);  // words per 16-token Key tile
  static constexpr uint32_t VTW = (uint32_t)tile_words(kTcD, VB);
  static constexpr uint32_t KTB = 2 * KTW * 4, VTB = 2 * VTW * 4;   // per group record
  static constexpr uint32_t VMB = kTcGS * 4 * 4, KMB = kTcD * 4;
  static constexpr uint32_t SB = KTB + VTB + VMB + KMB;  // group record bytes
  static constexpr uint32_t STAGE = 4 * SB;
  // TMEM columns of one team: D_V | D_K | A_K | A_V
  static constexpr int AKC = KT / 4;
  static constexpr int cDV = 0, cDK = N, cAK = 2 * N, cAV = 2 * N + AKC;
  static constexpr int kCols = cAV + 32;
#ifndef KVB_TC_TEAMS
#define KVB_TC_TEAMS 4
#endif
  static constexpr int TC = (kCols + 31) / 32 * 32;                          // columns per team
  static constexpr int T = 512 / TC < KVB_TC_TEAMS ? 512 / TC : KVB_TC_TEAMS;  // teams per CTA (one CTA per SM)
  static constexpr int NCOL = T * TC <= 128 ? 128 : T * TC <= 256 ? 256 : 512;  // (allocation: a power of two)
  static constexpr int THREADS = T * 128;
  // shared memory per team: ring | B_K | B_V | narrow tables | exchange | barriers
  static constexpr int BK = KT * N;   // row k = 16 B, N / 16 chunks of KT rows
  static constexpr int BV = 128 * N;  // group x at x * 32 * N
  static constexpr int YT = K3 ? kTcCons * R * kTcD * 4 : 0;  // narrow-slot factors [warp][row][d]
  static constexpr int XCH = 2048;  // words: [0, 128) reductions, [128, 136) f64 checksums, [256, 288) exchange, [320, 322) counters
  static constexpr int NBAR = 4 + 2;  // full[<=4], sfull, vdone
  static constexpr int TFIXED = BK + BV + YT + XCH + NBAR * 8 + 8;
  static constexpr int NTB = K3 ? kTcD * 4 : 0;  // channel -> field of the 2-bit plane (shared by the teams)
  static constexpr int stages() {
    const int avail = (226 * 1024 - NTB - 256) / T - TFIXED - 128;
    const int s = avail / (int)STAGE;
    return s >= 4 ? 4 : s < 2 ? 2 : s;
  }
  static constexpr int S = stages();
  static constexpr int TEAM = ((S * (int)STAGE + TFIXED) + 127) / 128 * 128;  // bytes per team
  static constexpr size_t smem() { return (size_t)T * TEAM + NTB + 256; }
};

// one named barrier per team (ids 1..4; 0 is __syncthreads)
__device__ __forceinline__ void team_sync(int id) { asm volatile("bar.sync %0, 128;\n" ::"r"(id) : "memory"); }
__device__ __forceinline__ bool team_any(int id, bool x) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %2, 0;\n\tbar.red.or.pred q, %1, 128, p;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
      : "=r"(r)
      : "r"(id), "r"((uint32_t)x)
      : "memory");
  return r != 0;
}

template <int KB, int VB, int R>
__global__ void __launch_bounds__(TcGeo<KB, VB, R>::THREADS, 1) attend_tc_kernel(TcParams p) {
  using G = TcGeo<KB, VB, R>;
  constexpr bool K3 = G::K3;
  constexpr int KB2 = K3 ? 2 : KB;                          // bits of the 2/4-bit Key plane
  constexpr int CK = 8 / KB2, CV = 8 / VB;                  // classes per byte
  constexpr uint32_t KMASK = KB2 == 4 ? 0x0F0F0F0Fu : 0x03030303u;
  constexpr uint32_t VMASK = VB == 4 ? 0x0F0F0F0Fu : 0x03030303u;
  constexpr int KW = lane_words<kTcD, KB>();
  constexpr int VWPL = plane_wpl(kTcD, VB);
  constexpr int S = G::S;

  extern __shared__ __align__(128) uint8_t dsm[];  // (no realignment: keeps the loads LDS, not generic)
  uint32_t* ntab = reinterpret_cast<uint32_t*>(dsm + (size_t)G::T * G::TEAM);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dsm + (size_t)G::T * G::TEAM + G::NTB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp >> 2, w = warp & 3;
  const int bar_id = 1 + team;
  // this team's worker index and tiles [t_beg, t_end) (32-bit: NT < 2^31)
  const int worker = blockIdx.x * G::T + team;
  const int t_beg = (int)((int64_t)worker * p.NT / p.C), t_end = (int)((int64_t)(worker + 1) * p.NT / p.C);
  const int n = worker < p.C ? t_end - t_beg : 0;  // (workers past C: no tiles)

  uint8_t* tb = dsm + (size_t)team * G::TEAM;
  uint8_t* ring = tb;
  uint8_t* bk = ring + (size_t)S * G::STAGE;
  uint8_t* bv = bk + G::BK;
  float* ytab = reinterpret_cast<float*>(bv + G::BV);
  uint32_t* xch = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ytab) + G::YT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + G::XCH);
  uint64_t* full = bars;       // [S] TMA -> team
  uint64_t* sfull = bars + 4;  // scores in D_K
  uint64_t* vdone = bars + 5;  // Value k-steps done (A_V, B_V, D_V free)
  uint32_t* cnt_k = xch + 320;  // arrival counters (zero between steps)
  uint32_t* cnt_v = xch + 321;

  if (w == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_init(sfull, 1);
    mbar_init(vdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {  // B buffers start zero (columns of absent groups / rows are never written)
    uint4* z = reinterpret_cast<uint4*>(bk);
    for (int i = threadIdx.x & 127; i < (G::BK + G::BV) / 16; i += 128) z[i] = make_uint4(0u, 0u, 0u, 0u);
    if ((threadIdx.x & 127) == 0) cnt_k[0] = cnt_v[0] = 0u;
  }
  if constexpr (K3) {
    for (int d = threadIdx.x; d < kTcD; d += G::THREADS) {
      int fw, sh;
      imma_field(true, kTcD, 2, 0, d, &fw, &sh);
      ntab[d] = (uint32_t)fw | ((uint32_t)sh << 16);
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "n"(G::NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot + (uint32_t)(team * G::TC);
  const uint32_t tq_w = tmem + ((uint32_t)(32 * w) << 16);  // this warp's TMEM lane quarter
  const bool leader = w == 0 && lane == 0;                  // issues this team's TMA and MMAs

  if (n > 0) {
    const int bh0 = t_beg / p.Tb, ti0 = t_beg - (t_beg / p.Tb) * p.Tb;
    const uint64_t pol = evict_first_policy();
    // next tile to fetch, tracked by every thread (whichever thread closes a tile refills its stage)
    int f_bh = bh0, f_ti = ti0;
    auto fetch_next = [&]() {
      if (++f_ti == p.Tb) {
        f_ti = 0;
        ++f_bh;
      }
    };
    auto fetch = [&](int i) {  // tile i (= (f_bh, f_ti)) -> stage i % S
      const int s = i % S;
      const int nv = min(4, p.Gf - 4 * f_ti);
      const uint32_t bytes = (uint32_t)nv * G::SB;
      mbar_arrive_expect_tx(&full[s], bytes);
      bulk_g2s(ring + (size_t)s * G::STAGE, p.rec + ((size_t)f_bh * p.Grec + 4 * (size_t)f_ti) * G::SB, bytes, &full[s],
               pol);
    };
    for (int i = 0; i < min(S, n); ++i) {
      if (leader) fetch(i);
      fetch_next();
    }
    // the last of the four warps to finish a step issues its MMAs (no team barrier): arrival
    // counters in shared memory, acq_rel so every warp's TMEM / shared writes happen before
    auto last_of_team = [&](uint32_t* cnt) {
      uint32_t old = 0;
      if (lane == 0) {
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(old) : "r"(smem_u32(cnt)) : "memory");
        if (old == kTcCons - 1) *reinterpret_cast<volatile uint32_t*>(cnt) = 0u;
      }
      return old == kTcCons - 1;  // (lane 0 only)
    };

    constexpr uint32_t idk = idesc_i8(G::N, true), idv = idesc_i8(G::N, false);
    const uint32_t bk_a = smem_u32(bk), bv_a = smem_u32(bv);
    // B_K rows k = lane + 32 i of this lane: k-step i, t = lane / 8, y = (lane / 4) % 2, e = lane % 4;
    // channel d = 32 (q % 4) + 16 (q / 4) + 4 t + e with q = 2 i + y (the A_K column map below)
    int dch[4];
    float clsL[4], clsH[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = 2 * i + ((lane >> 2) & 1);
      dch[i] = 32 * (q & 3) + 16 * (q >> 2) + 4 * (lane >> 3) + (lane & 3);
      clsL[i] = pow2i(-KB2 * (q % CK));
      clsH[i] = K3 ? 4.f * pow2i(-q) : 0.f;
    }
    // B_V row of this lane's token j = lane inside its group's k-step: tile half y = j / 16,
    // token 4 t + e of the tile -> k = 8 t + 4 y + e
    const int kv_row = 8 * ((lane & 15) >> 2) + 4 * (lane >> 4) + (lane & 3);
    // this thread as a Value accumulator row (TMEM lane 32 w + lane = 16 u + 8 rh + g). 2-bit
    // Values: warp w unpacks m-tiles w and w + 4 (all four words of a lane's 16-byte chunk, one
    // class w): channel d = 16 (w + 4 u) + 8 rh + g. 4-bit Values: m-tiles 2 w, 2 w + 1 (one
    // word, both classes): d = 32 w + lane.
    constexpr bool VALT = VB == 2;
    const int vchan = VALT ? 16 * w + 64 * (lane >> 4) + (lane & 15) : 32 * w + lane;
    const int vcg = vchan >> 5;  // its channel group (gs = 32)
    const int vq = VALT ? w : 2 * w + (lane >> 4) + 8 * ((lane >> 3) & 1);
    const float vcls = pow2i(-VB * (vq % CV));
    const int Gq = p.Hq / p.H;

    // per-segment state
    int cur_bh = -1, cb11 = 0;
    float qv[R][4], qc[R][4];
    float m_run[R], l_t[R], acc[R], bias[R][4];
    double cs = 0.0;
    int e_cur = 0, nacc = 0;
    bool dirty = false, fresh = true;

    auto fold = [&](const float (&alpha)[R]) {  // D_V (int32 digits) -> acc (fp32), then rescale
      const float wsc = pow2i(-e_cur) * vcls;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int v[4];
        if constexpr (VALT) {  // the two channel groups of this warp's rows: (w / 2) and 2 + (w / 2)
          int v2[4];
          ldtm_32x32_x4(tq_w + G::cDV + 16 * r + 4 * (w >> 1), v);
          ldtm_32x32_x4(tq_w + G::cDV + 16 * r + 4 * (2 + (w >> 1)), v2);
          tc_wait_ld();
          if (lane >> 4) {
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = v2[c];
          }
        } else {
          ldtm_32x32_x4(tq_w + G::cDV + 16 * r + 4 * w, v);
          tc_wait_ld();
        }
        const float f = fmaf((float)v[3], 16777216.f, fmaf((float)v[2], 65536.f, fmaf((float)v[1], 256.f, (float)v[0])));
        acc[r] = fmaf(f, wsc, acc[r]) * alpha[r];
      }
    };
    auto seg_begin = [&](int bh) {
      cur_bh = bh;
      const int b = bh / p.H, h = bh - (bh / p.H) * p.H;
      cb11 = (int)(((unsigned)p.k.gbh(bh) * (unsigned)kTcD) % 11u);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int rr = r < p.rows ? r : 0;
        const int gi = rr / p.tq, qi = rr % p.tq;
        const size_t off = (((size_t)b * p.Hq + (size_t)h * Gq + gi) * p.tq + qi) * kTcD;
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const float x = p.q16 ? __half2float(static_cast<const __half*>(p.q)[off + dch[ii]])
                                : static_cast<const float*>(p.q)[off + dch[ii]];
          qv[r][ii] = r < p.rows ? x : 0.f;
          qc[r][ii] = qv[r][ii] * clsL[ii];
        }
        m_run[r] = -INFINITY;
        l_t[r] = 0.f;
        acc[r] = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) bias[r][c] = 0.f;
      }
      cs = 0.0;
      e_cur = 0;
      nacc = 0;
      dirty = false;
      fresh = true;
    };
    auto seg_end = [&](int i_last) {
      if (dirty) {
        mbar_wait(vdone, i_last & 1);
        tc_fence_after();
        float one[R];
#pragma unroll
        for (int r = 0; r < R; ++r) one[r] = 1.f;
        fold(one);
      }
      // reductions over the 128 tokens: l, Value-min bias per channel group, checksum
      float* red = reinterpret_cast<float*>(xch);  // [w][R * 5]
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float x = l_t[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[w * R * 5 + r * 5 + 4] = x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float y = bias[r][c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
          if (lane == 0) red[w * R * 5 + r * 5 + c] = y;
        }
      }
      double* dred = reinterpret_cast<double*>(xch + 128);
      if (p.want_cs) {
        double x = cs;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) dred[w] = x;
      }
      team_sync(bar_id);
      const size_t slot = (size_t)worker + cur_bh;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float L = 0.f, bsum = 0.f;
#pragma unroll
        for (int ww = 0; ww < kTcCons; ++ww) {
          L += red[ww * R * 5 + r * 5 + 4];
          bsum += red[ww * R * 5 + r * 5 + vcg];  // channel group of this thread's channel
        }
        p.part_acc[(slot * R + r) * kTcD + vchan] = acc[r] + bsum;
        if (w == 0 && lane == 0)
          p.part_ml[slot * R + r] = make_float2(m_run[r] == -INFINITY ? -INFINITY : m_run[r] * kLn2, L);
      }
      if (p.want_cs && w == 0 && lane == 0) p.part_cs[slot] = (dred[0] + dred[1]) + (dred[2] + dred[3]);
      team_sync(bar_id);  // red / dred reused by the next segment
    };

    int bh = bh0, ti = ti0;
    for (int i = 0; i < n; ++i) {
      if (bh != cur_bh) {
        if (cur_bh >= 0) seg_end(i - 1);
        seg_begin(bh);
      }
      const int s = i % S;
      const int nv = min(4, p.Gf - 4 * ti);
      const bool gv = w < nv;  // this warp's group holds tokens
      const uint8_t* st = ring + (size_t)s * G::STAGE;
      const uint8_t* rec = st + (size_t)w * G::SB;
      const uint32_t* kt = reinterpret_cast<const uint32_t*>(rec);
      const uint32_t* vm = reinterpret_cast<const uint32_t*>(rec + G::KTB + G::VTB);
      const uint32_t* km = reinterpret_cast<const uint32_t*>(rec + G::KTB + G::VTB + G::VMB);
      mbar_wait(&full[s], (i / S) & 1);

      // ---- Keys of group w: B digits (fixed point q s), min-term, A codes -> TMEM ----
      float isig[R], beta[R];
      int nmod = 0, omod = 0;
      if (gv) {
        float sc[4], mn[4];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const float2 f = meta_pair(km[dch[ii]]);
          sc[ii] = f.x;
          mn[ii] = f.y;
        }
        if constexpr (K3) {
          const int2 inf = __ldg(p.k.info + 4 * ti + w);
          nmod = inf.x % 11;
          omod = inf.y % 11;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float x[4], xh[4], mx = 0.f, bt = 0.f;
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            x[ii] = qc[r][ii] * sc[ii];
            mx = fmaxf(mx, fabsf(x[ii]));
            if constexpr (K3) {
              xh[ii] = qv[r][ii] * clsH[ii] * sc[ii];
              mx = fmaxf(mx, fabsf(xh[ii]));
            }
            bt = fmaf(qv[r][ii], mn[ii], bt);
          }
          const uint32_t mxu = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
          const int e = (int)((mxu >> 23) & 0xffu);
          const int se = min(max(283 - e, 1), 254);  // sigma = 2^(29 - floor(log2 max))
          isig[r] = __int_as_float((254 - se) << 23);
          const float sg = __int_as_float(se << 23);
          // column n = (w R + r) * 4 + digit: byte (n / 16) * 16 KT + 16 k + n % 16
          const int n0 = (w * R + r) * 4;
          uint8_t* col = bk + (n0 >> 4) * 16 * G::KT + (n0 & 15) + 16 * lane;
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const uint32_t u = ((uint32_t)__float2int_rn(x[ii] * sg) + 0x80808080u) ^ 0x80808080u;
            *reinterpret_cast<uint32_t*>(col + 512 * ii) = u;
            if constexpr (K3) {
              const uint32_t uh = ((uint32_t)__float2int_rn(xh[ii] * sg) + 0x80808080u) ^ 0x80808080u;
              *reinterpret_cast<uint32_t*>(col + 16 * 128 + 512 * ii) = uh;
              ytab[(w * R + r) * kTcD + dch[ii]] = qv[r][ii] * (wide_scale(sc[ii]) - sc[ii]);
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) bt += __shfl_xor_sync(0xffffffffu, bt, o);
          beta[r] = bt;
        }
        // A: the group's two 16-token Key tiles -> TMEM rows 32 w + 16 u + (g, g + 8)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          uint32_t kw[KW];
          lds_tile<kTcD, KB>(kt + u * G::KTW, lane, kw);
          uint32_t ra[16];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int rb = 0; rb < 2; ++rb)
#pragma unroll
              for (int y = 0; y < 2; ++y) {
                const int q = 2 * x + y;
                ra[4 * x + 2 * rb + y] = kw[(q / CK) * 2 + rb] & (KMASK << (KB2 * (q % CK)));
              }
          const uint32_t ta = tq_w + ((uint32_t)(16 * u) << 16) + G::cAK;
          sttm_16x256_x4(ta, ra);
          if constexpr (K3) {
            constexpr int HW = kTcD * 2 / 64;  // first word of the 1-bit plane
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
              for (int rb = 0; rb < 2; ++rb)
#pragma unroll
                for (int y = 0; y < 2; ++y) ra[4 * x + 2 * rb + y] = kw[HW + rb] & (0x01010101u << (2 * x + y));
            sttm_16x256_x4(ta + 32, ra);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          isig[r] = 0.f;
          beta[r] = 0.f;
        }
      }
      tc_wait_st();
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (last_of_team(cnt_k)) {  // score MMAs: D_K = A_K (codes) x B_K (digits)
        tc_fence_after();
#pragma unroll
        for (int x = 0; x < G::NKS; ++x)
          mma_i8(tmem + G::cDK, tmem + G::cAK + 8 * x, desc_mn(bk_a + 512 * x, 128, 16 * G::KT), idk, x > 0);
        mma_commit(sfull);
      }

      // ---- Values of all four groups, channels 32 w .. 32 w + 31 -> A_V ----
      if (i >= 1) {  // the previous tile's Value k-steps are done with A_V / B_V / D_V
        mbar_wait(vdone, (i - 1) & 1);
        tc_fence_after();
      }
      if constexpr (VALT) {
        // 2-bit: q = mt + 8 rh with mt = w + 4 u -> word q / 4 = u + 2 rh, class w
        uint32_t ra0[16], ra1[16];
        const uint32_t msk = VMASK << (VB * w);
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            const uint32_t* vt = reinterpret_cast<const uint32_t*>(st + (size_t)x * G::SB + G::KTB) + y * G::VTW;
            const uint4 v4 = *reinterpret_cast<const uint4*>(vt + 4 * lane);
            ra0[4 * x + y] = v4.x & msk;      // u 0, rh 0
            ra0[4 * x + 2 + y] = v4.z & msk;  // u 0, rh 1
            ra1[4 * x + y] = v4.y & msk;      // u 1, rh 0
            ra1[4 * x + 2 + y] = v4.w & msk;  // u 1, rh 1
          }
        sttm_16x256_x4(tq_w + G::cAV, ra0);
        sttm_16x256_x4(tq_w + (16u << 16) + G::cAV, ra1);
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          uint32_t ra[16];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) {
              const uint32_t* vt = reinterpret_cast<const uint32_t*>(st + (size_t)x * G::SB + G::KTB) + y * G::VTW;
#pragma unroll
              for (int rh = 0; rh < 2; ++rh) {
                const int q = 2 * w + u + 8 * rh;
                const uint32_t word = vt[plane_addr(lane, q / CV, VWPL)];
                ra[4 * x + 2 * rh + y] = word & (VMASK << (VB * (q % CV)));
              }
            }
          sttm_16x256_x4(tq_w + ((uint32_t)(16 * u) << 16) + G::cAV, ra);
        }
      }

      // ---- scores of token j = lane of group w ----
      float scv[R];
      mbar_wait(sfull, i & 1);
      tc_fence_after();
      {
        int dg[R][4];
#pragma unroll
        for (int r = 0; r < R; ++r) ldtm_32x32_x4(tq_w + G::cDK + (w * R + r) * 4, dg[r]);
        tc_wait_ld();
        float corr[R], fac = 1.f;
#pragma unroll
        for (int r = 0; r < R; ++r) corr[r] = 0.f;
        if constexpr (K3) {
          if (gv) {
            // narrow slots of token j (stream index % 11 == 10): channels d = d0 + 11 k
            const int rres = ((10 - omod - lane) % 11 + 11) % 11;
            if (nmod != 0) {
              const int d0 = ((rres * inv11(nmod) - cb11) % 11 + 11) % 11;
              const uint32_t* tile = kt + (lane >> 4) * G::KTW;
              const int ib = lane & 15, rowoff = 16 * (ib & 7) + (ib >> 3);
              const float* yt = ytab + w * R * kTcD;
#pragma unroll
              for (int kk = 0; kk < (kTcD + 10) / 11; ++kk) {
                const int d = d0 + 11 * kk;
                if (d < kTcD) {
                  const uint32_t tbw = ntab[d];
                  const uint32_t code = (tile[(tbw & 0xffffu) + rowoff] >> (tbw >> 16)) & 3u;
#pragma unroll
                  for (int r = 0; r < R; ++r) corr[r] = fmaf((float)code, yt[r * kTcD + d], corr[r]);
                }
              }
            } else if ((omod + lane) % 11 == 10) {
              fac = 7.0f / 3.0f;  // every channel of this token is narrow
            }
          }
        }
        const float wl = p.inv * kLog2e;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int lo = dg[r][0] + (dg[r][1] << 8), hi = dg[r][2] + (dg[r][3] << 8);
          const float sum = fmaf((float)hi, 65536.f, (float)lo) * isig[r];
          const float scn = fmaf(sum, fac, beta[r]) + corr[r];  // natural units before 1/sqrt(D)
          scv[r] = gv ? scn * wl : -INFINITY;
          if (p.want_cs && gv && r < p.rows) cs += (double)(scn * p.inv);
        }
      }

      // ---- Value meta of this token, softmax bookkeeping (team-uniform max and exponent) ----
      float vs[4], vmn[4];
      int e_tok = 100;
      if (gv) {
        float smax = 0.f;
#pragma unroll
        for (int cg = 0; cg < 4; ++cg) {
          const float2 f = meta_pair(vm[cg * kTcGS + lane]);
          vs[cg] = f.x;
          vmn[cg] = f.y;
          smax = fmaxf(smax, f.x);
        }
        e_tok = min(156 - kLazy - (int)((__float_as_uint(smax) >> 23) & 0xffu), 100);
      } else {
#pragma unroll
        for (int cg = 0; cg < 4; ++cg) vs[cg] = vmn[cg] = 0.f;
      }

      bool need = nacc >= p.flush_tiles || (gv && e_cur > e_tok);
#pragma unroll
      for (int r = 0; r < R; ++r) need = need || scv[r] > m_run[r] + (float)kLazy;
      if (team_any(bar_id, need)) {
        // exchange the tile's per-row max and exponent bound over the four warps
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t mx = __reduce_max_sync(0xffffffffu, f2o(scv[r]));
          if (lane == 0) xch[256 + w * 8 + r] = mx;
        }
        const int emin = (int)__reduce_min_sync(0xffffffffu, (unsigned)(e_tok + 1024)) - 1024;
        if (lane == 0) xch[256 + w * 8 + 7] = (uint32_t)(emin + 1024);
        team_sync(bar_id);
        float alpha[R];
        bool moved = false;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          uint32_t mx = xch[256 + r];
#pragma unroll
          for (int ww = 1; ww < kTcCons; ++ww) mx = max(mx, xch[256 + ww * 8 + r]);
          const float tmax = o2f(mx);
          const float m_new = tmax > m_run[r] + (float)kLazy ? tmax : m_run[r];
          alpha[r] = m_new == m_run[r] ? 1.f : fast_exp2(m_run[r] - m_new);  // (0 from -inf)
          moved = moved || m_new != m_run[r];
          m_run[r] = m_new;
        }
        int e_blk = (int)xch[256 + 7];
#pragma unroll
        for (int ww = 1; ww < kTcCons; ++ww) e_blk = min(e_blk, (int)xch[256 + ww * 8 + 7]);
        e_blk -= 1024;
        if (dirty) {  // (the previous tile's Value k-steps are complete: waited above)
          fold(alpha);
          if (moved) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              l_t[r] *= alpha[r];
#pragma unroll
              for (int c = 0; c < 4; ++c) bias[r][c] *= alpha[r];
            }
          }
        }
        e_cur = e_blk - kEHead;
        nacc = 0;
        fresh = true;
      }

      // ---- p, l, Value-min bias, B digits of y = p s 2^E (u8) -> B_V ----
      {
        const float pe = pow2i(e_cur);
        uint8_t* dst = bv + (size_t)w * 32 * G::N + 16 * kv_row;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float pr = gv ? fast_exp2(scv[r] - m_run[r]) : 0.f;
          l_t[r] += pr;
          uint4 y;
          y.x = (uint32_t)__float2int_rn(pr * pe * vs[0]);
          y.y = (uint32_t)__float2int_rn(pr * pe * vs[1]);
          y.z = (uint32_t)__float2int_rn(pr * pe * vs[2]);
          y.w = (uint32_t)__float2int_rn(pr * pe * vs[3]);
#pragma unroll
          for (int c = 0; c < 4; ++c) bias[r][c] = fmaf(pr, vmn[c], bias[r][c]);
          *reinterpret_cast<uint4*>(dst + 512 * r) = y;  // chunk r: 32 rows x 16 B
        }
      }
      tc_wait_st();  // A_V stores of this tile
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (last_of_team(cnt_v)) {  // every read of this ring stage is done, A_V / B_V written
        tc_fence_after();
#pragma unroll
        for (int x = 0; x < 4; ++x)
          mma_i8(tmem + G::cDV, tmem + G::cAV + 8 * x, desc_mn(bv_a + x * 32 * G::N, 128, 512), idv, !(fresh && x == 0));
        mma_commit(vdone);
        if (i + S < n) fetch(i + S);  // refill this stage
      }
      if (i + S < n) fetch_next();
      fresh = false;
      dirty = true;
      ++nacc;
      if (++ti == p.Tb) {
        ti = 0;
        ++bh;
      }
    }
    seg_end(n - 1);
  }

  // teardown: every TMEM access (loads, the MMAs waited for) is complete
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(*tslot), "n"(G::NCOL));
}

template <int KB, int VB, int R>
bool launch_tc(const TcParams& p0, int BH, Workspace& ws, cudaStream_t st, TcExt* ext) {
  using G = TcGeo<KB, VB, R>;
  auto kern = attend_tc_kernel<KB, VB, R>;
  const size_t smem = G::smem();
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  static thread_local int attr_dev = -1;
  if (attr_dev != dev) {
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
    attr_dev = dev;
    if (getenv("KVMIX_TC_DEBUG"))
      fprintf(stderr, "attend_tc_kernel<%d,%d,%d>: %d teams, smem %zu B, %d stages, %d TMEM columns\n", KB, VB, R, G::T,
              smem, G::S, G::NCOL);
  }
  // one CTA per SM (the teams take all 512 TMEM columns), one tile range per team
  TcParams p = p0;
  const int64_t workers = (int64_t)num_sms() * G::T;
  p.C = (int)std::max<int64_t>(1, std::min<int64_t>(workers, p.NT));
  const int ctas = (p.C + G::T - 1) / G::T;
  // partial slots worker + bh for every possible worker: scratch depends on (B, H, rows, SM
  // count) only, never on the token count (scratch.hpp:14-21)
  const size_t slots = (size_t)workers + BH;
  p.part_ml = ws.ml(st, slots * R);
  p.part_acc = ws.acc(st, slots * R * kTcD);
  p.part_cs = ws.cs(st, slots + 1);
  if (p.want_cs) check_cuda(cudaMemsetAsync(p.part_cs, 0, (slots + 1) * sizeof(double), st), "memset");
  kern<<<ctas, G::THREADS, smem, st>>>(p);
  ext->ml = p.part_ml;
  ext->acc = p.part_acc;
  ext->cs = p.part_cs;
  ext->C = p.C;
  ext->NT = p.NT;
  ext->Tb = p.Tb;
  ext->R = R;
  ext->slots = slots;
  return true;
}

template <int KB, int R>
bool tc_vbits(const TcParams& p, int vb, int BH, Workspace& ws, cudaStream_t st, TcExt* ext) {
  if (vb == 2) return launch_tc<KB, 2, R>(p, BH, ws, st, ext);
  if (vb == 4) return launch_tc<KB, 4, R>(p, BH, ws, st, ext);
  return false;
}
template <int R>
bool tc_bits(const TcParams& p, int kb, int vb, int BH, Workspace& ws, cudaStream_t st, TcExt* ext) {
  if (kb == 2) return tc_vbits<2, R>(p, vb, BH, ws, st, ext);
  if (kb == 3) return tc_vbits<3, R>(p, vb, BH, ws, st, ext);
  if (kb == 4) return tc_vbits<4, R>(p, vb, BH, ws, st, ext);
  return false;
}

}  // namespace

// Whether attend_tc_launch serves this cache / query shape.
bool attend_tc_eligible(const kvmix_cache* c, int rows) {
  if (!knobs().tc) return false;
  if (c->D != kTcD || c->cfg.group_size != kTcGS) return false;
  if (c->v.bits != 2 && c->v.bits != 4) return false;
  if (rows < 1 || rows > 4) return false;
  return true;
}

// Launches attend_tc_kernel over the fast groups [0, Gf) of every (b, kv-head); fills `ext`
// with the partial slots the window launch merges. Returns false when nothing was launched
// (not eligible, or no fast group).
bool attend_tc_launch(const kvmix_cache* c, const void* q, bool q16, int Hq, int tq, int Gf, bool want_cs,
                      Workspace& ws, cudaStream_t st, TcExt* ext) {
  const int rows = (Hq / c->H) * tq;
  if (!attend_tc_eligible(c, rows) || Gf <= 0) return false;
  const int BH = c->B * c->H;
  TcParams p{};
  p.rec = reinterpret_cast<const uint8_t*>(c->k.tiles);
  p.k = view(c->k);
  p.q = q;
  p.q16 = q16;
  p.H = c->H;
  p.Hq = Hq;
  p.tq = tq;
  p.rows = rows;
  p.Gf = Gf;
  p.Tb = (Gf + 3) / 4;
  p.Grec = (int)(c->k.bh_stride / c->k.grp_stride);
  p.NT = (int64_t)BH * p.Tb;
  p.inv = 1.0f / sqrtf((float)kTcD);
  p.want_cs = want_cs;
  p.flush_tiles = std::max(1, std::min(kTcFlushTiles, knobs().flush_blocks / 4));
  const int kb = c->k.bits, vb = c->v.bits;
  bool ok = false;
  if (rows == 1) ok = tc_bits<1>(p, kb, vb, BH, ws, st, ext);
  else if (rows == 2) ok = tc_bits<2>(p, kb, vb, BH, ws, st, ext);
  else ok = tc_bits<4>(p, kb, vb, BH, ws, st, ext);
  if (ok) after_launch("attend_tc_kernel");
  return ok;
}

}  // namespace kvb
