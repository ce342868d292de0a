// attention_mma.cu -- fused split-K decode attention on the tensor cores, fed by TMA bulk
// copies (cp.async.bulk + mbarrier) into a per-warp shared-memory ring.
//
// Decode is a GEMV per (b, kv-head): scores = K q, out = V^T p. At 2-bit gs32 a K+V element
// pair is 0.75 B of HBM traffic, so a CUDA-core loop (unpack + dequant + FMA per element)
// runs out of issue slots before HBM does. The dequantization is
// factored out of the dot products
//     q.k_j  = sum_d (q_d s_gd) c_jd + sum_d q_d m_gd          (Keys, per channel group)
//     out_d  = sum_j (p_j s_jg) c_jd + sum_j p_j m_jg          (Values, per token group)
// and the code sums run on integer tensor cores: mma.sync m16n8k32 with the CODES as the
// u8 A operand straight from the packed words (IMMA layout, common.cuh: one AND per 4
// codes, each carrying a per-channel power of two 2^(b*class)) and the fp32 factors as the
// B operand in fixed point, split into four base-256 digits held in four MMA columns
// (digit n has weight 2^(8n)). Integer products and int32 accumulation are exact, so the
// only rounding is the fixed-point conversion of the B values (2^-29 of the largest one):
//   * Keys: B_d = round(q_d s_d 2^-(b class_d) sigma), sigma = 2^(29 - floor(log2 max)),
//     balanced s8 digits, per group; scores come back per 16-token tile.
//   * Values: B_j = round(p_j s_jg 2^E), unsigned u8 digits. p <= 1 and the running 2^E
//     only changes when the largest scale of a block would overflow 2^30, so int32
//     accumulators persist across blocks and are folded into fp32 (shared memory) only when
//     the online-softmax max moves, E changes, or 1024 blocks have accumulated.
//   * The min terms are fp32 FMAs (Keys: one dot product per group; Values: one FMA per
//     token and channel group).
// On sm_100a legacy mma.sync issues one MMA per ~8.5 cycles per SM sub-partition for both
// HMMA m16n8k16 and IMMA m16n8k32 (profiles/probes/imma_rate.cu), so k32 integer MMAs
// halve the tensor-pipe time as well as the unpack work of the fp16 formulation.
//
// Mixed3 (3-bit) Keys: the low 2 bits and the high bit are two IMMA planes whose B operands
// share sigma (4 q s 2^-class_hi for the high plane), so both accumulate into one int32
// score. The reference's narrow slots (stream index % 11 == 10) dequantize with scale*7/3:
// for a token the narrow channels are d = d0 + 11k, corrected on the CUDA cores (one token
// per lane, channel -> field table) with q_d (wide_scale(s_d) - s_d).
//
// Query rows: two per pass (one B column quadruple each); more rows (GQA with G > 2, several
// query tokens) run as row passes inside one launch.
//
// The full-precision Key window whose Values are already packed runs as 32-token "window
// blocks" (lane = token fp32 dot products from the ring, then the IMMA Value block).
//
// Memory pipeline: every unit of work (one Key group of gs tokens of one (b, kv-head)) is
// one contiguous record (Key tiles | Value tiles | Value meta | Key meta) copied by one
// elected lane with cp.async.bulk into a ring of S stages; the warp waits on the stage's
// mbarrier (complete_tx), computes, and refills the stage S groups ahead.
//
// Work distribution (stream-K): a list of per-(b, kv-head) units (fast groups, window
// blocks, then single window tokens) is cut into equal ranges over one resident wave of
// independent warps. A (b, kv-head) inside one warp's range is normalized and written by that
// warp; one split across warps is merged (in warp order: deterministic) by the last of its
// warps to publish a partial (tagged atomic counter) -- no separate combine launch.
#include "mma_common.cuh"

#include <cstdio>
#include <vector>

namespace kvb {
int attend_ws_launch(MmaParams& p, int D, int rows, int kb, int vb, int BH, Workspace& ws, cudaStream_t st);

// Tuning / test knobs, read from the environment once per process.
Knobs& knobs() {
  static Knobs k = [] {
    Knobs x;
    auto iv = [](const char* name, int lo, int hi, int dflt) {
      const char* e = getenv(name);
      return e ? std::max(lo, std::min(hi, atoi(e))) : dflt;
    };
    x.tail_unit = iv("KVMIX_TAIL_UNIT", 1, 64, kTailUnit);
    x.group_cost = iv("KVMIX_GROUP_COST", 1, 64, kGroupCost);
    x.flush_blocks = iv("KVMIX_TEST_FLUSH_BLOCKS", 1, kFlushBlocks, kFlushBlocks);
    x.min_cost = iv("KVMIX_MIN_COST", 1, 1 << 20, kMinCost);
    x.ws = iv("KVMIX_WS", 0, 2, 1);
    x.tc = iv("KVMIX_TC", 0, 1, 0);
    x.pdl = iv("KVMIX_PDL", 0, 1, 1);
    x.layers = iv("KVMIX_LAYERS", 0, 1, 1);
    x.r4 = iv("KVMIX_R4", 0, 1, 1);
    x.skip_tail = getenv("KVMIX_PROF_SKIP_TAIL") != nullptr;
    x.no_window = getenv("KVMIX_PROF_NO_WINDOW") != nullptr;
    return x;
  }();
  return k;
}


// One-shot request for a programmatic dependent launch of the next attention call on this
// host thread (set by kvmix_*attend_layers for layers after the first).
static thread_local bool g_pdl_next = false;
void request_pdl(bool on) { g_pdl_next = on && knobs().pdl; }
bool take_pdl() {
  const bool r = g_pdl_next;
  g_pdl_next = false;
  return r;
}

// kvmix_set_knob (test / tuning hook): overrides one knob for later launches
bool set_knob(const char* name, int v) {
  Knobs& k = knobs();
  const std::string n = name ? name : "";
  if (n == "KVMIX_TAIL_UNIT") k.tail_unit = std::max(1, std::min(64, v));
  else if (n == "KVMIX_GROUP_COST") k.group_cost = std::max(1, std::min(64, v));
  else if (n == "KVMIX_TEST_FLUSH_BLOCKS") k.flush_blocks = std::max(1, std::min(kFlushBlocks, v <= 0 ? kFlushBlocks : v));
  else if (n == "KVMIX_MIN_COST") k.min_cost = std::max(1, v);
  else if (n == "KVMIX_WS") k.ws = std::max(0, std::min(2, v));
  else if (n == "KVMIX_TC") k.tc = std::max(0, std::min(1, v));
  else if (n == "KVMIX_PDL") k.pdl = std::max(0, std::min(1, v));
  else if (n == "KVMIX_LAYERS") k.layers = std::max(0, std::min(1, v));
  else if (n == "KVMIX_R4") k.r4 = std::max(0, std::min(1, v));
  else return false;
  return true;
}


namespace {

// Window-only launch epilogue: this warp's window partial (m in log2 units, l, lane-parallel
// accumulators) merged with attend_tc_kernel's fast-group partials of (b, kv-head) bh -- the
// CTAs c0..c1 whose tile ranges hold bh's tiles, slot c + bh -- in CTA order (deterministic),
// normalized and written to the output.
template <int D, int R>
__device__ __forceinline__ void ext_merge_write(const MmaParams& p, int bh, int lane, int pass, int prow0, int prows,
                                                const float (&m_all)[R], const float (&l_all)[R],
                                                const float (&acct)[R][D / 32]) {
  constexpr int LC = D / 32;
  int c0 = 0, c1 = -1;
  if (p.ext_Tb > 0) {
    const int64_t x0 = (int64_t)bh * p.ext_Tb, x1 = x0 + p.ext_Tb - 1;
    c0 = (int)(((x0 + 1) * p.ext_C - 1) / p.ext_NT);
    c1 = (int)(((x1 + 1) * p.ext_C - 1) / p.ext_NT);
  }
  const int b = bh / p.H, h = bh % p.H, G = p.Hq / p.H;
  for (int r = 0; r < prows; ++r) {
    const int er = prow0 + r;
    const float mo = m_all[r] == -INFINITY ? -INFINITY : m_all[r] * kLn2;
    float M = mo;
    for (int c = c0; c <= c1; ++c) M = fmaxf(M, __ldcg(&p.ext_ml[((size_t)c + bh) * p.ext_R + er]).x);
    const float fo = mo == -INFINITY ? 0.f : expf(mo - M);
    float L = l_all[r] * fo;
    float a[LC];
#pragma unroll
    for (int k = 0; k < LC; ++k) a[k] = acct[r][k] * fo;
    for (int c = c0; c <= c1; ++c) {
      const size_t si = ((size_t)c + bh) * p.ext_R + er;
      const float2 ml = __ldcg(&p.ext_ml[si]);
      if (ml.x == -INFINITY) continue;
      const float f = expf(ml.x - M);
      L += ml.y * f;
      const float* src = p.ext_acc + si * D + lane * LC;
#pragma unroll
      for (int k = 0; k < LC; ++k) a[k] = fmaf(__ldcg(src + k), f, a[k]);
    }
    const int gi = er / p.tq, qi = er % p.tq;
    float* o = p.out + (((size_t)b * p.Hq + h * G + gi) * p.tq + qi) * D + lane * LC;
    const float il = 1.0f / L;
#pragma unroll
    for (int k = 0; k < LC; ++k) o[k] = a[k] * il;
  }
  if (p.fused && lane == 0) p.flags[(size_t)pass * p.nbh + bh] = 0u;  // final writer of (pass, bh)
}

// GS: 0 = runtime group size (a multiple of 32), else compile-time (32 is the KVmix default).
#ifdef KVB_TRACE
__device__ uint64_t* g_trace = nullptr;  // debug builds: per-warp timeline (KVMIX_TRACE_FILE)
#endif

// The kernel body: warp gw (of the layer whose parameters p are) runs its unit range.
// CS = false: the checksum is compiled out (multi-layer launches never ask for it).
template <int D, int KB, int VB, int R, int GS, bool CS>
__device__ __forceinline__ void attend_mma_body(const MmaParams& p, const int gw) {
  const bool want_cs = CS && p.want_cs;
  static_assert(D == 64 || D == 128, "IMMA attention handles D in {64, 128}");
  static_assert(VB == 2 || VB == 4, "Values: 2 or 4 bits");
  static_assert(R == 1 || R == 2 || R == 4, "one, two or four query rows per KV head");
  constexpr int NT = R == 4 ? 2 : 1;           // IMMA n8 column tiles (two rows x four digits each)
  constexpr bool K3 = KB == 3;
  static_assert(!K3 || D == 128, "3-bit Keys: D = 128");
  constexpr int NK = D / 32;                   // Key k-steps (32 channels)
  constexpr int NM = D / 16;                   // Value m-tiles (16 channels)
  constexpr int KW = lane_words<D, KB>();      // words per lane, Key tile
  constexpr int VW = lane_words<D, VB>();      // words per lane, Value tile
  constexpr int KB2 = K3 ? 2 : KB;             // bits of the Key plane in the 2/4-bit layout
  constexpr int CK = 8 / KB2;                  // classes per byte
  constexpr int CV = 8 / VB;
  constexpr uint32_t KMASK = KB2 == 4 ? 0x0F0F0F0Fu : 0x03030303u;
  constexpr uint32_t VMASK = VB == 4 ? 0x0F0F0F0Fu : 0x03030303u;
  constexpr int LC = D / 32;                   // channels per lane (tail path / epilogue)
  constexpr int QL = D / 4;                    // lanes with a distinct Key channel quad
  constexpr int CGMAX = D / 32;                // channel groups of a token (gs >= 32)
  using WL = WarpLayout<D, KB, R>;

  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ float s_acc[kMmaWarps][R][D];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warps are independent (no CTA barriers); npass adjacent warps share a unit range
#ifdef KVB_TRACE
  uint64_t tr_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_start));
#endif
  const int pass = gw % p.npass, wg = gw / p.npass;
  if (wg >= p.W) return;
  const int prow0 = p.row0 + pass * p.rows;                // this pass's query rows
  const int prows = min(p.rows, p.rows_all - pass * p.rows);
  const size_t pbase = (size_t)pass * p.pslots;            // this pass's partial slots
  const int g = lane >> 2, t = lane & 3;
  const int G = p.Hq / p.H;
  const int gs = GS ? GS : p.gs;
  const int CG = GS ? D / GS : p.cg;
  const int NBLK = gs / 32;  // 32-token blocks per group
  using SG = StageGeo<D, KB, VB, R, GS>;
  const int S = GS ? SG::kStages : p.stages;
  const uint32_t SB = GS ? SG::kStage : p.stage_bytes;            // bytes per group record
  const uint32_t KTB = GS ? SG::kKT : p.kt_bytes, VTB = GS ? SG::kVT : p.vt_bytes;
  const uint32_t VMB = GS ? SG::kVM : p.vm_bytes;
  const int64_t c_beg = p.wonly ? 0 : (int64_t)wg * p.Nc / p.W, c_end = p.wonly ? 0 : (int64_t)(wg + 1) * p.Nc / p.W;
  // window-only launch: warp wg = (b, kv-head) wg, its window units [Gf, U)
  const int u_beg = p.wonly ? wg * p.U + p.Gf : unit_at_cost(p, c_beg);
  const int u_end = p.wonly ? (wg + 1) * p.U : unit_at_cost(p, c_end);
  if (p.wonly && u_beg >= u_end) {  // no window: the fast-group partials alone
    float m0[R], l0[R], a0[R][D / 32];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      m0[r] = -INFINITY;
      l0[r] = 0.f;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) a0[r][c] = 0.f;
    }
    if (lane == 0 && want_cs) p.part_cs[pbase + wg + wg] = 0.0;
    ext_merge_write<D, R>(p, wg, lane, pass, prow0, prows, m0, l0, a0);
    return;
  }
  if (u_beg >= u_end) {  // no unit starts in this cost range: neutral partial
    const int bh = (int)(c_beg / p.cost_bh);
    int w0, w1;
    bh_warps(p, bh, w0, w1);
    if (wg < w0 || wg > w1) return;
    pdl_gate(p);
    if (lane < prows) p.part_ml[(pbase + wg + bh) * p.rows + lane] = make_float2(-INFINITY, 0.f);
    if (lane == 0 && want_cs) p.part_cs[pbase + wg + bh] = 0.0;
    if (arrive_last(p, bh, lane, pass, wg)) merge_bh<D>(p, bh, lane, pass, prow0, prows);
    return;
  }

  uint8_t* wbase = dsm + (size_t)warp * WL::bytes(S, SB);
  uint8_t* ring = wbase;
  uint8_t* kstage = ring + (size_t)S * SB;
  uint32_t* kbs = reinterpret_cast<uint32_t*>(kstage);
  float* ytab = reinterpret_cast<float*>(kstage + WL::kY);
  uint32_t* ntab = reinterpret_cast<uint32_t*>(kstage + WL::kY + R * D * 4);
  uint8_t* vbs = kstage + WL::kK;
  float* qbuf = reinterpret_cast<float*>(vbs + WL::kV);
  double* csm = reinterpret_cast<double*>(vbs + WL::kV + D * 4);  // per-lane checksum partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(vbs + WL::kV + WL::kQ);

  // zero the B staging (columns of absent query rows / digits must stay 0)
  {
    uint4* z = reinterpret_cast<uint4*>(kstage);
    for (int i = lane; i < (WL::kK + WL::kV) / 16; i += 32) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();

  // this lane's softmax rows: in column tile nt, lanes t = 2r, 2r+1 hold row 2 nt + r (IMMA
  // score columns 4r .. 4r+3 of the tile)
  const int my_r = t >> 1;
  bool row_ok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) row_ok[nt] = 2 * nt + my_r < prows;

  // producer: this warp's fast groups in work-list order, issued S ahead of the consumer
  // (running record pointer, groups left in the current (b, kv-head), groups left to issue)
  int rec_i;  // group record index (records of all (b, kv-head) are one array)
  int left_bh, left_all;
  {
    int i_bh = u_beg / p.U, i_g = u_beg - i_bh * p.U;
    if (i_g >= p.Gf) {
      ++i_bh;
      i_g = 0;
    }
    rec_i = i_bh * p.Grec + i_g;
    left_bh = p.Gf - i_g;
    // fast groups of [u_beg, u_end): whole (b, kv-head) ranges clipped at both ends
    const int bh0 = u_beg / p.U, bh1 = (u_end - 1) / p.U;
    int n = 0;
    for (int x = bh0; x <= bh1; ++x) {
      const int a = max(u_beg - x * p.U, 0), z = min(u_end - x * p.U, p.Gf);
      n += max(z - a, 0);
    }
    left_all = n;
  }
  auto issue_next = [&](int s) {
    if (left_all > 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&bars[s], SB);
        bulk_g2s(ring + (size_t)s * SB, reinterpret_cast<const uint8_t*>(p.k.tiles) + (size_t)rec_i * SB, SB, &bars[s],
                 evict_first_policy());
      }
      --left_all;
      ++rec_i;
      if (--left_bh == 0) {
        rec_i += p.Grec - p.Gf;
        left_bh = p.Gf;
      }
    }
  };
  for (int s = 0; s < S; ++s) issue_next(s);
  // (PDL: the gate -- wait for the previous layer's launch, then let the next one start -- sits
  // before the warp's first result write; gating right here, after the ring fill, measured
  // slower: 3.41 vs 3.26 ms per configs[1] step, the early warps stall on the previous layer)

  // fused 1-token append: the warp whose range holds a (b, kv-head)'s first window unit
  // appends its token (only the window path reads what the append writes), then publishes
  // (pass 0 only; the other passes' twins wait for the flag like later warps)
  if (p.fused && pass == 0) {
    for (int bh = u_beg / p.U; bh <= (u_end - 1) / p.U; ++bh) {
      const int x = bh * p.U + p.Gf;
      if (x >= u_beg && x < u_end) {
        decode_append_warp(p.da, bh, lane);
        if ((bh + 1) * p.U > u_end || p.npass > 1) {  // other warps read this window too: publish
          __threadfence();
          __syncwarp();
          if (lane < p.npass) st_release(p.flags + (size_t)lane * p.nbh + bh, 1u);  // one flag per pass
        }
      }
    }
  }

  // Key B-build mapping: lane owns channels 4*Lq .. 4*Lq+3 (IMMA: one B register's k rows)
  const int Lq = lane % QL;
  const bool qdup = lane >= QL;  // D = 64: lanes 16..31 mirror 0..15
  const int kkL = Lq >> 3, hL = (Lq & 7) >> 2, tL = Lq & 3;
  const float clsL = pow2i(-KB2 * ((kkL + NK * hL) % CK));
  // 3-bit Keys: 4 * 2^-class of the high-bit plane (class q for D = 128), channel offset
  // of this (b, kv-head) in the Mixed3 stream mod 11, and the channel -> field table
  const float clsH = K3 ? 4.f * pow2i(-((kkL + NK * hL) & 7)) : 0.f;
  const float invL = pow2i(KB2 * ((kkL + NK * hL) % CK));  // 1 / clsL
  const float clsHL = clsH * invL;                          // clsH / clsL
  if constexpr (K3) {
    for (int d = lane; d < D; d += 32) {
      int w, sh;
      imma_field(true, D, 2, 0, d, &w, &sh);
      ntab[d] = ((uint32_t)w << 5) | (uint32_t)sh;  // the funnel shift below reads sh = low 5 bits
    }
    __syncwarp();
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
    const int cb11 = (int)(((unsigned)p.k.gbh(bh) * (unsigned)D) % 11u);  // global (b, kv-head)
    (void)cb11;

    // query rows at this lane's Key channels
    float qv[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int rr = prow0 + (r < prows ? r : 0);
      const int gi = rr / p.tq, qi = rr % p.tq;
      const size_t off = (((size_t)b * p.Hq + h * G + gi) * p.tq + qi) * D + 4 * Lq;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float x = p.q16 ? __half2float(static_cast<const __half*>(p.q)[off + c]) : static_cast<const float*>(p.q)[off + c];
        qv[r][c] = r < prows ? x : 0.f;
      }
    }
    if constexpr (R == 1) {  // q of every channel for the window blocks' dot products
      if (p.nwb > 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) qbuf[4 * Lq + c] = qv[0][c];
      }
    }
    float qc[R][4];  // q * 2^-(b class) of this lane's Key channels (exact: power of two)
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) qc[r][c] = qv[r][c] * clsL;
    float m_run[NT], l_run[NT];  // row 2 nt + my_r (lazy reference max, log2 units)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      m_run[nt] = -INFINITY;
      l_run[nt] = 0.f;
    }
    if (want_cs) csm[lane] = 0.0;
    int accv[NT][NM][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < NM; ++i) accv[nt][i][0] = accv[nt][i][1] = accv[nt][i][2] = accv[nt][i][3] = 0;
    float bias[R];  // sum_j p_j m_jc of this lane's channel group cq = lane / 8 and token quads
#pragma unroll
    for (int r = 0; r < R; ++r) bias[r] = 0.f;
    int e_cur = 0;      // Value fixed-point exponent
    int nacc = 0;       // blocks in the int32 Value accumulators
    bool dirty = false;  // s_acc / accumulators / bias hold something
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < LC; ++c) s_acc[warp][r][lane * LC + c] = 0.f;
    __syncwarp();

    // Fold the int32 Value accumulators into s_acc (fp32): s_acc = (s_acc + acc 2^-E) alpha.
    // Lane (g, t) holds digit columns 2t, 2t+1 (row 2 nt + (t >> 1)) of channels 16 mt + g (+8).
    auto flush = [&](const float (&alpha)[NT]) {
      const float w0 = pow2i(16 * (t & 1) - e_cur);
      const float w1 = w0 * 256.f;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int mt = 0; mt < NM; ++mt) {
          const float c0 = pow2i(-VB * (mt % CV)), c1 = pow2i(-VB * ((mt + NM) % CV));
          float f0 = fmaf((float)accv[nt][mt][1], w1, (float)accv[nt][mt][0] * w0) * c0;
          float f1 = fmaf((float)accv[nt][mt][3], w1, (float)accv[nt][mt][2] * w0) * c1;
          f0 += __shfl_xor_sync(0xffffffffu, f0, 1);
          f1 += __shfl_xor_sync(0xffffffffu, f1, 1);
          if ((t & 1) == 0 && 2 * nt + my_r < R) {
            float* a = &s_acc[warp][2 * nt + my_r][16 * mt + g];
            a[0] = (a[0] + f0) * alpha[nt];  // accumulated with the old max
            a[8] = (a[8] + f1) * alpha[nt];
          }
          accv[nt][mt][0] = accv[nt][mt][1] = accv[nt][mt][2] = accv[nt][mt][3] = 0;
        }
      nacc = 0;
    };

    // Value k-step of one 32-token block: lane (g, t) owns token j = g + 8t (p of it for every
    // row in pr); fixed-point exponent / fold bookkeeping, B digits, 8 IMMA.
    auto value_block = [&](const uint32_t* vt2, const uint32_t* vm2, const float (&pr)[R], const float (&alpha)[NT],
                           int nvalid) {
      // lane (cq, tq) = (lane / 8, lane % 8) handles channel group cq of tokens 4tq .. 4tq+3
      const int cq = lane >> 3, tq = lane & 7;
      const bool cg_ok = cq < CG;
      float pq[R][4], sv[4], mv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int jj = 4 * tq + i;  // owned (p) by lane 4 (jj % 8) + jj / 8
#pragma unroll
        for (int r = 0; r < R; ++r) pq[r][i] = __shfl_sync(0xffffffffu, pr[r], 4 * (jj & 7) + (jj >> 3));
        const uint32_t w = (cg_ok && jj < nvalid) ? vm2[(size_t)cq * gs + jj] : 0u;  // [cg][token]; rows past nvalid never written
        const float2 f = meta_pair(w);
        sv[i] = f.x;
        mv[i] = f.y;
      }
      // fixed-point exponent: max scale of the block * 2^E < 2^30 (p <= 2^kLazy)
      const float smax = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
      const uint32_t smu = __reduce_max_sync(0xffffffffu, __float_as_uint(smax));
      const int e_blk = min(156 - kLazy - (int)((smu >> 23) & 0xffu), 100);
      if (!dirty) {
        e_cur = e_blk - kEHead;
      } else {
        bool mv_lane = false;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mv_lane |= row_ok[nt] && alpha[nt] != 1.0f;
        const bool moved = __any_sync(0xffffffffu, mv_lane);
        if (moved || e_cur > e_blk || nacc >= p.flush_blocks) {
          flush(alpha);
          if (moved) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const float ax = __shfl_xor_sync(0xffffffffu, alpha[nt], 2);
#pragma unroll
              for (int r = 2 * nt; r < 2 * nt + 2 && r < R; ++r) bias[r] *= (r - 2 * nt == my_r) ? alpha[nt] : ax;
            }
          }
          e_cur = e_blk - kEHead;
        }
      }
      dirty = true;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) bias[r] = fmaf(pq[r][i], mv[i], bias[r]);
      // B digits of y = p s 2^E (u8, four columns per row): one word per (digit, row) holds the
      // quad's four tokens -> vbs[cq][4r + n][pos(4tq) .. +3]
      if (cg_ok) {
        const float pe = pow2i(e_cur);
        const int pos = (tq & 3) * 8 + (tq >> 2) * 4;
        float se[4];  // s 2^E (exact: power-of-two factor), so (p s) 2^E == p (s 2^E)
#pragma unroll
        for (int i = 0; i < 4; ++i) se[i] = pe * sv[i];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          uint32_t uu[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) uu[i] = (uint32_t)__float2int_rn(pq[r][i] * se[i]);
          store_digits(reinterpret_cast<uint32_t*>(vbs + cq * (256 * NT) + (4 * r) * 32 + pos), 8, uu);
        }
      }
      __syncwarp();
      {
        uint32_t vw0[VW], vw1[VW];
        lds_tile<D, VB>(vt2, lane, vw0);
        lds_tile<D, VB>(vt2 + tile_words(D, VB), lane, vw1);
        uint32_t vb[NT][CGMAX][2];
        if constexpr (GS != 0) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < CGMAX; ++c) {
              if (c < D / (GS ? GS : 1)) {
                const uint2 x = *reinterpret_cast<const uint2*>(vbs + c * (256 * NT) + nt * 256 + g * 32 + 8 * t);
                vb[nt][c][0] = x.x;
                vb[nt][c][1] = x.y;
              }
            }
        }
#pragma unroll
        for (int mt = 0; mt < NM; ++mt) {
          const int q0 = mt, q1 = mt + NM;
          const uint32_t a0 = vw0[q0 / CV] & (VMASK << (VB * (q0 % CV)));
          const uint32_t a1 = vw0[q1 / CV] & (VMASK << (VB * (q1 % CV)));
          const uint32_t a2 = vw1[q0 / CV] & (VMASK << (VB * (q0 % CV)));
          const uint32_t a3 = vw1[q1 / CV] & (VMASK << (VB * (q1 % CV)));
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if constexpr (GS != 0) {
              const int c = (mt * 16) / (GS ? GS : 1);
              imma_uu(accv[nt][mt], a0, a1, a2, a3, vb[nt][c][0], vb[nt][c][1]);
            } else {
              const int c = (mt * 16) / gs;
              const uint2 x = *reinterpret_cast<const uint2*>(vbs + c * (256 * NT) + nt * 256 + g * 32 + 8 * t);
              imma_uu(accv[nt][mt], a0, a1, a2, a3, x.x, x.y);
            }
          }
        }
      }
      ++nacc;
      __syncwarp();  // vbs is rewritten by the next block
    };

    const int g_stop = min(hi, p.Gf);
    for (int grp = lo; grp < g_stop; ++grp) {
      mbar_wait(&bars[s], phase);
      const uint8_t* st = ring + (size_t)s * SB;
      const uint32_t* kt = reinterpret_cast<const uint32_t*>(st);
      const uint32_t* vt = reinterpret_cast<const uint32_t*>(st + KTB);
      const uint32_t* vm = reinterpret_cast<const uint32_t*>(st + KTB + VTB);
      const uint32_t* km = reinterpret_cast<const uint32_t*>(st + KTB + VTB + VMB);

      // ---- Key group: B operand ---------------------------------------------------------
      // Fixed-point B = round(q s 2^-(b class) sigma) in four balanced s8 digits; 3-bit Keys
      // add the high-bit plane's B = round(4 q s 2^-class_hi sigma) (same sigma, so both
      // planes accumulate into the same int32 scores) and the narrow-slot table
      // ytab[d] = q_d (wide_scale(s_d) - s_d) for the Mixed3 correction.
      float betaL[NT];   // sum_d q_d m_d of row 2 nt + my_r, scaled to log2 units
      float wsc0[NT];    // weight of this lane's score column pair (log2 units)
      uint32_t kb[NT][NK][2], kbh[NT][K3 ? NK : 1][2];
      int nmod = 0, omod = 0;  // 3-bit Keys: segment length / group offset mod 11
      {
        const uint4 m4 = *reinterpret_cast<const uint4*>(km + 4 * Lq);
        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
        float sc[4], mn[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float2 f = meta_pair(mw[c]);
          sc[c] = f.x;
          mn[c] = f.y;
        }
        if constexpr (K3) {
          const int2 inf = __ldg(p.k.info + grp);  // {segment length, token offset of the group}
          nmod = inf.x % 11;
          omod = inf.y % 11;
        }
        float beta[R], isig[R];
        float bsel[NT];  // R > 1: sum_d q_d m_d of row 2 nt + my_r
        __syncwarp();  // previous group's reads of kbs / ytab are done
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float x[4], xh[4], mx = 0.f, bt = 0.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            x[c] = qc[r][c] * sc[c];
            mx = fmaxf(mx, fabsf(x[c]));
            if constexpr (K3) {
              xh[c] = qc[r][c] * clsHL * sc[c];  // 4 q s 2^-class_hi
              mx = fmaxf(mx, fabsf(xh[c]));
            }
            bt = fmaf(qc[r][c], mn[c], bt);  // * 2^(b class) below
          }
          bt = qdup ? 0.f : bt * invL;  // sum_c q_c m_c of this lane (undo the class factor)
          // sigma = 2^(29 - floor(log2 max|x|)): max|x sigma| in [2^29, 2^30)
          const uint32_t mxu = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
          const int e = (int)((mxu >> 23) & 0xffu);
          const int se = min(max(283 - e, 1), 254);
          isig[r] = __int_as_float((254 - se) << 23);
          const float sg = __int_as_float(se << 23);
          uint32_t uu[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) uu[c] = ((uint32_t)__float2int_rn(x[c] * sg) + 0x80808080u) ^ 0x80808080u;
          if (!qdup) store_digits(kbs + ((4 * r) * 4 + tL) * (2 * NK) + kkL * 2 + hL, 4 * 2 * NK, uu);
          if constexpr (K3) {
#pragma unroll
            for (int c = 0; c < 4; ++c) uu[c] = ((uint32_t)__float2int_rn(xh[c] * sg) + 0x80808080u) ^ 0x80808080u;
            store_digits(kbs + WL::kKC * 4 * 2 * NK + ((4 * r) * 4 + tL) * (2 * NK) + kkL * 2 + hL, 4 * 2 * NK, uu);
            {  // narrow-slot correction table of this row
              float4 y;
              y.x = qc[r][0] * invL * (wide_scale(sc[0]) - sc[0]);
              y.y = qc[r][1] * invL * (wide_scale(sc[1]) - sc[1]);
              y.z = qc[r][2] * invL * (wide_scale(sc[2]) - sc[2]);
              y.w = qc[r][3] * invL * (wide_scale(sc[3]) - sc[3]);
              *reinterpret_cast<float4*>(ytab + r * D + 4 * lane) = y;
            }
          }
          if constexpr (R == 1) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bt += __shfl_xor_sync(0xffffffffu, bt, o);
          }
          beta[r] = bt;  // R > 1: this lane's term, reduced below
        }
        if constexpr (R > 1) {
          // transposed butterfly: the xor-16 (and, R = 4, xor-8) steps halve the rows a lane
          // carries, so lane L ends with the total of row 2 b4 + b3 (R = 4) / b4 (R = 2)
          const bool hi16 = lane & 16;
          float x;
          if constexpr (R == 4) {
            const float s0 = hi16 ? beta[0] : beta[2], s1 = hi16 ? beta[1] : beta[3];
            const float k0 = hi16 ? beta[2] : beta[0], k1 = hi16 ? beta[3] : beta[1];
            const float y0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
            const float y1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
            const bool hi8 = lane & 8;
            x = (hi8 ? y1 : y0) + __shfl_xor_sync(0xffffffffu, hi8 ? y0 : y1, 8);
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) bsel[nt] = __shfl_sync(0xffffffffu, x, 16 * nt + 8 * my_r);
          } else {
            x = (hi16 ? beta[1] : beta[0]) + __shfl_xor_sync(0xffffffffu, hi16 ? beta[0] : beta[1], 16);
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            bsel[0] = __shfl_sync(0xffffffffu, x, 16 * my_r);  // (my_r = 1 without a second row: unused)
          }
        }
        __syncwarp();
        // B fragments: b0 = k rows 4t..4t+3, b1 = 16+4t.., column 8 nt + g (digit g%4 of row
        // (8 nt + g)/4)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int col = 8 * nt + g;
          const bool has_col = col < WL::kKC;
          const uint32_t* zsrc = reinterpret_cast<const uint32_t*>(kstage + WL::kZ) + t * (2 * NK);
          const uint32_t* src = has_col ? kbs + (col * 4 + t) * (2 * NK) : zsrc;
#pragma unroll
          for (int kk = 0; kk < NK; kk += 2) {
            const uint4 v = *reinterpret_cast<const uint4*>(src + 2 * kk);
            kb[nt][kk][0] = v.x;
            kb[nt][kk][1] = v.y;
            kb[nt][kk + 1][0] = v.z;
            kb[nt][kk + 1][1] = v.w;
          }
          if constexpr (K3) {
#pragma unroll
            for (int kk = 0; kk < NK; kk += 2) {
              const uint32_t* srch = has_col ? src + WL::kKC * 4 * 2 * NK : zsrc;
              const uint4 v = *reinterpret_cast<const uint4*>(srch + 2 * kk);
              kbh[nt][kk][0] = v.x;
              kbh[nt][kk][1] = v.y;
              kbh[nt][kk + 1][0] = v.z;
              kbh[nt][kk + 1][1] = v.w;
            }
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int rr = 2 * nt + my_r < R ? 2 * nt + my_r : 0;
          float is = isig[0], bb = R > 1 ? bsel[nt] : beta[0];
#pragma unroll
          for (int r = 1; r < R; ++r)
            if (rr == r) is = isig[r];
          wsc0[nt] = pow2i(16 * (t & 1)) * is * p.inv * kLog2e;
          betaL[nt] = bb * p.inv * kLog2e;
        }
      }

      // ---- the group's 32-token blocks: 2 Key tiles + one Value k-step each ---------------
      for (int blk = 0; blk < NBLK; ++blk) {
        const uint32_t* kt2 = kt + (size_t)(2 * blk) * tile_words(D, KB);
        const uint32_t* vt2 = vt + (size_t)(2 * blk) * tile_words(D, VB);
        const uint32_t* vm2 = vm + 32 * blk;  // V meta [cg][gs]
        float la[NT][2], lb[NT][2];  // scores (log2 units) of tokens g / g+8 of tile u, row 2 nt + my_r
        {
          uint32_t kw[2][KW];
          lds_tile<D, KB>(kt2, lane, kw[0]);
          lds_tile<D, KB>(kt2 + tile_words(D, KB), lane, kw[1]);
          int dk[NT][2][4];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) dk[nt][u2][0] = dk[nt][u2][1] = dk[nt][u2][2] = dk[nt][u2][3] = 0;
#pragma unroll
          for (int kk = 0; kk < NK; ++kk) {
            const int q0 = kk, q1 = kk + NK;  // channel halves h = 0 / 1
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) {
              const uint32_t a0 = kw[u2][(q0 / CK) * 2 + 0] & (KMASK << (KB2 * (q0 % CK)));
              const uint32_t a1 = kw[u2][(q0 / CK) * 2 + 1] & (KMASK << (KB2 * (q0 % CK)));
              const uint32_t a2 = kw[u2][(q1 / CK) * 2 + 0] & (KMASK << (KB2 * (q1 % CK)));
              const uint32_t a3 = kw[u2][(q1 / CK) * 2 + 1] & (KMASK << (KB2 * (q1 % CK)));
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) imma_us(dk[nt][u2], a0, a1, a2, a3, kb[nt][kk][0], kb[nt][kk][1]);
              if constexpr (K3) {  // high-bit plane: words (q + 2 NK rb) / 8, class q (D = 128)
                constexpr int HW = D * 2 / 64;  // first word of the 1-bit plane
                const uint32_t h0 = kw[u2][HW + 0] & (0x01010101u << q0);
                const uint32_t h1 = kw[u2][HW + 1] & (0x01010101u << q0);
                const uint32_t h2 = kw[u2][HW + 0] & (0x01010101u << q1);
                const uint32_t h3 = kw[u2][HW + 1] & (0x01010101u << q1);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) imma_us(dk[nt][u2], h0, h1, h2, h3, kbh[nt][kk][0], kbh[nt][kk][1]);
              }
            }
          }
          float corr[NT][4];  // Mixed3 narrow corrections of tokens g, g+8, 16+g, 24+g (row 2 nt + my_r)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) corr[nt][0] = corr[nt][1] = corr[nt][2] = corr[nt][3] = 0.f;
          float fac[4] = {1.f, 1.f, 1.f, 1.f};
          if constexpr (K3) {
            // lane (g, t) corrects token jt = g + 8t of the block: narrow channels d = d0 + 11k
            const int jt = g + 8 * t, tg = 32 * blk + jt;
            const int rres = ((10 - omod - tg) % 11 + 11) % 11;
            float dlt[R];
#pragma unroll
            for (int r = 0; r < R; ++r) dlt[r] = 0.f;
            if (nmod != 0) {
              const int d0 = ((rres * inv11(nmod) - cb11) % 11 + 11) % 11;
              const uint32_t* tile = kt2 + (t >> 1) * tile_words(D, KB);
              const int ib = jt & 15, rowoff = 16 * (ib & 7) + (ib >> 3);
#pragma unroll
              for (int k = 0; k < (D + 10) / 11; ++k) {
                const int d = d0 + 11 * k;
                if (d < D) {
                  const uint32_t tb = ntab[d];  // {word offset at row 0 << 5 | shift}
                  const uint32_t code = __funnelshift_r(tile[(tb >> 5) + rowoff], 0u, tb) & 3u;
#pragma unroll
                  for (int r = 0; r < R; ++r) dlt[r] = fmaf((float)code, ytab[r * D + d], dlt[r]);
                }
              }
            }
            const float wsn = p.inv * kLog2e;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int x = 0; x < 4; ++x) {  // row 2 nt + my_r of token g + 8x (lane 4g + x made it)
                float c = __shfl_sync(0xffffffffu, dlt[2 * nt], 4 * g + x);
                if constexpr (R >= 2) {
                  const float c1 = __shfl_sync(0xffffffffu, dlt[2 * nt + 1], 4 * g + x);
                  c = my_r ? c1 : c;
                }
                corr[nt][x] = c * wsn;
              }
            if (nmod == 0) {  // every channel of the tokens with (omod + tg) % 11 == 10 is narrow
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                const int tgx = 32 * blk + g + 8 * x;
                if ((omod + tgx) % 11 == 10) fac[x] = 7.0f / 3.0f;
              }
            }
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) {
              // digits n0, n0+1 of this lane's columns: dk0 + 256 dk1 fits int32 (|dk| < 2^23)
              float pa = (float)(dk[nt][u2][0] + (dk[nt][u2][1] << 8)) * wsc0[nt];
              float pb = (float)(dk[nt][u2][2] + (dk[nt][u2][3] << 8)) * wsc0[nt];
              pa += __shfl_xor_sync(0xffffffffu, pa, 1);
              pb += __shfl_xor_sync(0xffffffffu, pb, 1);
              la[nt][u2] = fmaf(pa, fac[2 * u2], betaL[nt]) + corr[nt][2 * u2];
              lb[nt][u2] = fmaf(pb, fac[2 * u2 + 1], betaL[nt]) + corr[nt][2 * u2 + 1];
            }
        }
        if (want_cs && (t & 1) == 0) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            if (row_ok[nt]) csm[lane] += (double)(((la[nt][0] + lb[nt][0]) + (la[nt][1] + lb[nt][1])) * kLn2);
        }

        // ---- online softmax (rows 2 nt + my_r) ---------------------------------------------
        float alpha[NT], pa[NT][2], pb[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float tmax = fmaxf(fmaxf(la[nt][0], lb[nt][0]), fmaxf(la[nt][1], lb[nt][1]));
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
          const float m_new = tmax > m_run[nt] + (float)kLazy ? tmax : m_run[nt];
          alpha[nt] = fast_exp2(m_run[nt] - m_new);
#pragma unroll
          for (int u2 = 0; u2 < 2; ++u2) {
            pa[nt][u2] = row_ok[nt] ? fast_exp2(la[nt][u2] - m_new) : 0.f;
            pb[nt][u2] = row_ok[nt] ? fast_exp2(lb[nt][u2] - m_new) : 0.f;
          }
          l_run[nt] = l_run[nt] * alpha[nt] + ((pa[nt][0] + pb[nt][0]) + (pa[nt][1] + pb[nt][1]));
          m_run[nt] = m_new;
        }

        // ---- Value block: lane (g, t) owns token g + 8t of the 32 -------------------------
        float pr[R];  // p of token j for every row
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const float mine = (t & 1) ? ((t >> 1) ? pb[nt][1] : pb[nt][0]) : ((t >> 1) ? pa[nt][1] : pa[nt][0]);
          const float other = (t & 1) ? ((t >> 1) ? pb[nt][0] : pb[nt][1]) : ((t >> 1) ? pa[nt][0] : pa[nt][1]);
          const float recv = __shfl_xor_sync(0xffffffffu, other, 2);  // partner t^2's token, my row
#pragma unroll
          for (int r = 2 * nt; r < 2 * nt + 2 && r < R; ++r) pr[r] = (r - 2 * nt == my_r) ? mine : recv;
        }
        value_block(vt2, vm2, pr, alpha, 32);
      }
      // refill this stage S groups ahead
      issue_next(s);
      if (++s == S) {
        s = 0;
        phase ^= 1u;
      }
    }

    // ---- window blocks: 32 tokens of the full-precision Key window whose Values are packed
    // (Keys: lane = token fp32 dot products from the ring; Values: the IMMA block path on the
    // partial group's tiles). Waits for the fused append when an earlier warp made it.
    if (p.fused && (lo > p.Gf || pass != 0) && hi > p.Gf) {
      while (ld_acquire(p.flags + (size_t)pass * p.nbh + bh) == 0u) __nanosleep(32);
    }
    if constexpr (R == 1) {
      const int wb_lo = max(lo, p.Gf) - p.Gf, wb_hi = min(hi, p.Gf + p.nwb) - p.Gf;
      if (wb_lo < wb_hi) {
        __syncwarp();  // qbuf (filled at the segment start) visible
      }
      for (int wb = wb_lo; wb < wb_hi; ++wb) {
        const int64_t j0 = p.P + 32 * (int64_t)wb;
        const int jt = g + 8 * t;
        const int64_t jj = j0 + jt;
        const bool valid = jj < p.Pw;
        float sl = -INFINITY;
        if (valid) {
          int64_t slot = p.k.tail_start + (jj - p.k.quantized);
          if (slot >= p.k.tail_cap) slot -= p.k.tail_cap;
          float acc = 0.f;
          if (p.tail16) {
            const uint4* row = reinterpret_cast<const uint4*>(static_cast<const __half*>(p.k.tail) +
                                                              ((size_t)bh * p.k.tail_cap + (size_t)slot) * D);
#pragma unroll 4
            for (int ch = 0; ch < D / 8; ++ch) {
              const uint4 hv = __ldcg(row + ch);
              const float4 qa = *reinterpret_cast<const float4*>(qbuf + 8 * ch);
              const float4 qb = *reinterpret_cast<const float4*>(qbuf + 8 * ch + 4);
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&hv.x));
              const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&hv.y));
              const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&hv.z));
              const float2 f3 = __half22float2(*reinterpret_cast<const __half2*>(&hv.w));
              acc = fmaf(qa.x, f0.x, acc);
              acc = fmaf(qa.y, f0.y, acc);
              acc = fmaf(qa.z, f1.x, acc);
              acc = fmaf(qa.w, f1.y, acc);
              acc = fmaf(qb.x, f2.x, acc);
              acc = fmaf(qb.y, f2.y, acc);
              acc = fmaf(qb.z, f3.x, acc);
              acc = fmaf(qb.w, f3.y, acc);
            }
          } else {
            const float4* row = reinterpret_cast<const float4*>(static_cast<const float*>(p.k.tail) +
                                                                ((size_t)bh * p.k.tail_cap + (size_t)slot) * D);
#pragma unroll 4
            for (int ch = 0; ch < D / 4; ++ch) {
              const float4 kv4 = __ldcg(row + ch);
              const float4 qa = *reinterpret_cast<const float4*>(qbuf + 4 * ch);
              acc = fmaf(qa.x, kv4.x, acc);
              acc = fmaf(qa.y, kv4.y, acc);
              acc = fmaf(qa.z, kv4.z, acc);
              acc = fmaf(qa.w, kv4.w, acc);
            }
          }
          const float scn = acc * p.inv;
          if (want_cs) csm[lane] += (double)scn;
          sl = scn * kLog2e;
        }
        float tmax = sl;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        // every lane scores a token of row 0: use row 0's reference max (lanes t >= 2 carry
        // the unused row 1 of the fast blocks)
        const float m_ref = __shfl_sync(0xffffffffu, m_run[0], 0);
        const float m_new = tmax > m_ref + (float)kLazy ? tmax : m_ref;
        const float alpha[NT] = {fast_exp2(m_ref - m_new)};
        const float pj = valid ? fast_exp2(sl - m_new) : 0.f;
        // l of row 0 in the lanes t = 0, 1 convention: the quad (g, 0..3) holds tokens g, g+8, 16+g, 24+g
        float quad = pj + __shfl_xor_sync(0xffffffffu, pj, 1);
        quad += __shfl_xor_sync(0xffffffffu, quad, 2);
        l_run[0] = l_run[0] * alpha[0] + quad;
        m_run[0] = m_new;
        const int gi = (int)(j0 / gs), bi = (int)((j0 - (int64_t)gi * gs) / 32);
        const uint8_t* rec = reinterpret_cast<const uint8_t*>(p.k.tiles) + ((size_t)bh * p.Grec + gi) * SB;
        const uint32_t* vt2 = reinterpret_cast<const uint32_t*>(rec + KTB) + (size_t)(2 * bi) * tile_words(D, VB);
        const uint32_t* vm2 = reinterpret_cast<const uint32_t*>(rec + KTB + VTB) + 32 * bi;
        const float pr[R] = {pj};
        value_block(vt2, vm2, pr, alpha, (int)(p.Pw - j0 < 32 ? p.Pw - j0 : 32));
      }
    }

    // ---- end of the fast region: fold accumulators, gather the softmax state ------------
    if (dirty) {
      float one[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) one[nt] = 1.0f;
      flush(one);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {  // channel group cq's total over its 8 token-quad lanes
      bias[r] += __shfl_xor_sync(0xffffffffu, bias[r], 1);
      bias[r] += __shfl_xor_sync(0xffffffffu, bias[r], 2);
      bias[r] += __shfl_xor_sync(0xffffffffu, bias[r], 4);
    }
    float m_all[R], l_all[R];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float lr = l_run[nt];
      lr += __shfl_xor_sync(0xffffffffu, lr, 4);
      lr += __shfl_xor_sync(0xffffffffu, lr, 8);
      lr += __shfl_xor_sync(0xffffffffu, lr, 16);
#pragma unroll
      for (int r = 2 * nt; r < 2 * nt + 2 && r < R; ++r) {
        m_all[r] = __shfl_sync(0xffffffffu, m_run[nt], 2 * (r - 2 * nt));  // lane (g 0, t 2r')
        l_all[r] = __shfl_sync(0xffffffffu, lr, 2 * (r - 2 * nt));
      }
    }
    __syncwarp();
    // lane-parallel accumulators over channels lane*LC .. lane*LC+LC-1
    float acct[R][LC];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const int d = lane * LC + c;
        const float bsel = __shfl_sync(0xffffffffu, bias[r], 8 * (d / gs));  // group d / gs: lanes 8 cg ..
        acct[r][c] = s_acc[warp][r][d] + bsel;
      }

    // ---- tokens past the fast region: lane-parallel over channels ------------------------
    const int tb0 = p.Gf + p.nwb;  // first lane-parallel window unit
    const int64_t j_lo = p.Pw + (int64_t)max(lo - tb0, 0) * p.tail_unit;
    const int64_t j_hi = hi > tb0 && !p.skip_tail ? min(p.T, p.Pw + (int64_t)(hi - tb0) * p.tail_unit) : j_lo;
    if (j_lo < j_hi) {
      const int d0 = lane * LC;
      float qt[R][LC];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int rr = prow0 + (r < prows ? r : 0);
        const int gi = rr / p.tq, qi = rr % p.tq;
        const size_t off = (((size_t)b * p.Hq + h * G + gi) * p.tq + qi) * D + d0;
#pragma unroll
        for (int c = 0; c < LC; ++c)
          qt[r][c] = p.q16 ? __half2float(static_cast<const __half*>(p.q)[off + c]) : static_cast<const float*>(p.q)[off + c];
      }
      // IMMA Value layout of this lane's channels: word offset at t = 0 and bit shift at e = 0
      constexpr int VWPL = D * VB / 64, VCW = VWPL < 4 ? VWPL : 4;
      int vbase[LC], vsh[LC];
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const int d = d0 + c, dc = d & 15;
        const int q = (d >> 4) + NM * (dc >> 3);
        vbase[c] = plane_addr(4 * (dc & 7), q / CV, VWPL);
        vsh[c] = VB * (q % CV);
      }
      // four tokens per round: all loads issued first, the four reductions interleaved
      constexpr int TB = 4;
      for (int64_t j0 = j_lo; j0 < j_hi; j0 += TB) {
        float kx[TB][LC], vx[TB][LC];
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          const int64_t jj = min(j0 + i, j_hi - 1);
          if (jj >= p.k.quantized) {
            if (p.tail16 && LC == 4) {  // this lane's 4 channels: one 8-byte load from the ring
              int64_t slot = p.k.tail_start + (jj - p.k.quantized);
              if (slot >= p.k.tail_cap) slot -= p.k.tail_cap;
              const uint2 hv = __ldcg(reinterpret_cast<const uint2*>(static_cast<const __half*>(p.k.tail) +
                                                                    ((size_t)bh * p.k.tail_cap + (size_t)slot) * D + d0));
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&hv.x));
              const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&hv.y));
              kx[i][0] = f0.x;
              kx[i][1] = f0.y;
              kx[i][2 % LC] = f1.x;
              kx[i][3 % LC] = f1.y;
            } else {
#pragma unroll
              for (int c = 0; c < LC; ++c) kx[i][c] = tail_val(p.k, p.tail16, bh, jj - p.k.quantized, d0 + c, D);
            }
          } else {
#pragma unroll
            for (int c = 0; c < LC; ++c) kx[i][c] = deq_lane<D, true, KB>(p.k, bh, (int)jj, d0 + c, gs);
          }
          if (jj >= p.v.quantized) {
#pragma unroll
            for (int c = 0; c < LC; ++c) vx[i][c] = tail_val(p.v, p.tail16, bh, jj - p.v.quantized, d0 + c, D);
          } else {
            // packed Value of a window token (IMMA layout): shared token address math, one
            // meta word for the lane's channels (same channel group), per-channel word/shift
            const int j32 = (int)jj;
            const uint32_t* tile = p.v.tiles + tile_index(p.v, bh, j32 >> 4);
            const int ti = (j32 & 15) >> 2, te = j32 & 3;
            const float2 sm = meta_pair(__ldcg(p.v.meta + vmeta_at(p.v, bh, j32, d0 / gs)));
#pragma unroll
            for (int c = 0; c < LC; ++c) {
              const uint32_t w = __ldcg(tile + vbase[c] + ti * VCW);
              const uint32_t code = (w >> (vsh[c] + 8 * te)) & ((1u << VB) - 1u);
              vx[i][c] = fmaf((float)code, sm.x, sm.y);
            }
          }
        }
        float x[TB][R];
#pragma unroll
        for (int i = 0; i < TB; ++i)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float a = 0.f;
#pragma unroll
            for (int c = 0; c < LC; ++c) a = fmaf(qt[r][c], kx[i][c], a);
            x[i][r] = a;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < TB; ++i)
#pragma unroll
            for (int r = 0; r < R; ++r) x[i][r] += __shfl_xor_sync(0xffffffffu, x[i][r], o);
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          if (j0 + i >= j_hi) break;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (r < prows) {
              const float sc = x[i][r] * p.inv;
              if (want_cs && lane == 0) csm[0] += (double)sc;
              const float ls = sc * kLog2e;
              const float m_new = fmaxf(m_all[r], ls);
              const float alpha = exp2f(m_all[r] - m_new);
              const float pj = exp2f(ls - m_new);
              l_all[r] = l_all[r] * alpha + pj;
              m_all[r] = m_new;
#pragma unroll
              for (int c = 0; c < LC; ++c) acct[r][c] = acct[r][c] * alpha + pj * vx[i][c];
            }
          }
        }
      }
    }

    // ---- segment epilogue ----------------------------------------------------------------
    pdl_gate(p);
    // A (b, kv-head) inside this warp's range is normalized and written directly; otherwise
    // the partial goes to slot wg + bh and the last of its warps to arrive merges them.
    const size_t slot = pbase + wg + bh;
    if (want_cs) {
      double csl = csm[lane];
      for (int o = 16; o > 0; o >>= 1) csl += __shfl_xor_sync(0xffffffffu, csl, o);
      if (lane == 0) p.part_cs[slot] = csl;
    }
    if (p.wonly) {
      ext_merge_write<D, R>(p, bh, lane, pass, prow0, prows, m_all, l_all, acct);
    } else if (lo == 0 && hi == p.U) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r < prows) {
          const int gi = (prow0 + r) / p.tq, qi = (prow0 + r) % p.tq;
          float* o = p.out + (((size_t)b * p.Hq + h * G + gi) * p.tq + qi) * D + lane * LC;
          const float il = 1.0f / l_all[r];
#pragma unroll
          for (int c = 0; c < LC; ++c) o[c] = acct[r][c] * il;
        }
      }
      if (p.fused && lane == 0) p.flags[(size_t)pass * p.nbh + bh] = 0u;  // final writer of (pass, bh)
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r < prows) {
          const size_t pi = slot * p.rows + r;
          if constexpr (LC == 4) {
            *reinterpret_cast<float4*>(p.part_acc + pi * D + lane * LC) =
                make_float4(acct[r][0], acct[r][1], acct[r][2], acct[r][3]);
          } else {
#pragma unroll
            for (int c = 0; c < LC; ++c) p.part_acc[pi * D + lane * LC + c] = acct[r][c];
          }
          if (lane == 0) p.part_ml[pi] = make_float2(m_all[r] == -INFINITY ? -INFINITY : m_all[r] * kLn2, l_all[r]);
        }
      }
      if (arrive_last(p, bh, lane, pass, wg)) merge_bh<D>(p, bh, lane, pass, prow0, prows);
    }
    __syncwarp();  // s_acc is rewritten by the next segment
  }
#ifdef KVB_TRACE
  if (lane == 0 && g_trace) {  // (start, end, SM, unit range) per warp
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_trace[4 * gw] = tr_start;
    g_trace[4 * gw + 1] = t1;
    g_trace[4 * gw + 2] = sm;
    g_trace[4 * gw + 3] = ((uint64_t)u_beg << 32) | (uint32_t)u_end;
  }
#endif
}

template <int D, int KB, int VB, int R, int GS>
__global__ void __launch_bounds__(kMmaWarps * 32, KVB_MIN_CTAS(KB, R)) attend_mma_kernel(MmaParams p) {
  attend_mma_body<D, KB, VB, R, GS, true>(p, blockIdx.x * kMmaWarps + (threadIdx.x >> 5));
}

// Several layers of a decode step in one launch: warps [off[l], off[l+1]) run layer l with
// its own parameters, scratch and unit ranges (each layer exactly as its own launch would,
// with fewer warps), so the launch ramp and drain are paid once per step instead of once
// per layer. The parameter block lives in the kernel's constant bank (__grid_constant__:
// the layer's fields are read in place, not copied).
template <int D, int KB, int VB, int R, int GS>
__global__ void __launch_bounds__(kMmaWarps * 32, KVB_MIN_CTAS(KB, R))
    attend_mma_layers_kernel(const __grid_constant__ MmaLayers mp) {
  const int gw = blockIdx.x * kMmaWarps + (threadIdx.x >> 5);
  int li = 0;
  while (li + 1 < mp.n && gw >= mp.off[li + 1]) ++li;
  if (gw >= mp.off[li + 1]) return;
  attend_mma_body<D, KB, VB, R, GS, false>(mp.l[li], gw - mp.off[li]);
}

// Ring depth, dynamic shared memory and the resident wave (warps) of kernel `kern`.
template <int D, int KB, int VB, int R, int GS, typename Kern>
void mma_geometry(Kern kern, uint32_t stage_bytes, int& stages_out, size_t& smem, int64_t& wave) {
  using WL = WarpLayout<D, KB, R>;
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
  for (int occ_target = KVB_MIN_CTAS(KB, R); occ_target >= 1; occ_target = occ_target * 3 / 4) {
    const long per_cta = 227L * 1024 / occ_target - 1024 - static_smem;
    const long per_warp = per_cta / kMmaWarps - (long)fixed - 4 * 8 - 128;
    const long s_fit = per_warp / (long)stage_bytes;
    if (s_fit >= 2) {
      stages = (int)std::min<long>(4, s_fit);
      break;
    }
  }
  if constexpr (GS != 0) {
    using SG = StageGeo<D, KB, VB, R, GS>;
    static_assert(SG::kStages >= 2, "stage geometry");
    if (stage_bytes != SG::kStage) throw Error(KVMIX_RUNTIME_ERROR, "attend: record geometry mismatch");
    stages = SG::kStages;
  }
  stages_out = stages;
  smem = (size_t)kMmaWarps * WL::bytes(stages, stage_bytes);
  // per device: the dynamic shared memory attribute and the residency at this ring size are
  // set / queried once (host cost per call is a few table lookups)
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  static thread_local int occ_dev = -1;
  static thread_local size_t occ_smem = 0;
  static thread_local int occ = 0;
  if (occ_smem != smem || occ_dev != dev) {
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMmaWarps * 32, smem), "occupancy");
    occ_smem = smem;
    occ_dev = dev;
  }
  // one resident wave of independent warps (persistent): equal unit ranges, no stragglers
  wave = (int64_t)std::max(1, occ) * num_sms() * kMmaWarps;
}

// Partial slots, merge counters and append flags of one layer's launch parameters.
template <int D>
void mma_scratch(MmaParams& p, int BH, Workspace& ws, cudaStream_t st) {
  p.nbh = BH;
  const size_t slots = (size_t)p.npass * p.pslots;
  p.part_ml = ws.ml(st, slots * p.rows);
  p.part_acc = ws.acc(st, slots * p.rows * D);
  p.part_cs = ws.cs(st, slots + 1);
  p.cnt = ws.zeroed<unsigned>((size_t)p.npass * BH);
  p.cnt8 = ws.zeroed<unsigned>(slots);
  p.flags = p.fused ? ws.zeroed<unsigned>((size_t)p.npass * BH) : nullptr;
  if (p.want_cs) check_cuda(cudaMemsetAsync(p.part_cs, 0, (slots + 1) * sizeof(double), st), "memset");
}

template <typename Kern, typename Arg>
void launch_ex(Kern kern, unsigned grid, size_t smem, cudaStream_t st, bool pdl, const Arg& arg) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kMmaWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  check_cuda(cudaLaunchKernelEx(&cfg, kern, arg), pdl ? "attend launch (PDL)" : "attend launch");
}

template <int D, int KB, int VB, int R, int GS>
int launch(MmaParams& p, int BH, Workspace& ws, cudaStream_t st) {
  auto kern = attend_mma_kernel<D, KB, VB, R, GS>;
  size_t smem = 0;
  int64_t wave = 0;
  mma_geometry<D, KB, VB, R, GS>(kern, p.stage_bytes, p.stages, smem, wave);
  // small problems: at least kMinCost cost units per warp (a warp's prologue and the merge
  // of a head split over many warps cost more than a few groups)
  const int64_t min_cost = knobs().min_cost;
  const int64_t w_cap = std::max<int64_t>(1, p.Nc / min_cost);
  p.W = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(p.N, wave / p.npass), w_cap));
  if (p.wonly) p.W = BH;  // one warp per (pass, b, kv-head)
  // partial slots x * pslots + w + bh (w + bh < W + BH): scratch depends on (B, H, rows, D,
  // SM count) only
  p.pslots = (int)(std::max<int64_t>(wave, p.W) + BH);
  mma_scratch<D>(p, BH, ws, st);
  const int64_t warps = (int64_t)p.W * p.npass;
  const unsigned grid = (unsigned)((warps + kMmaWarps - 1) / kMmaWarps);
  if (p.pdl) {
    launch_ex(kern, grid, smem, st, true, p);
  } else {
#ifdef KVB_TRACE
    static uint64_t* tbuf = nullptr;
    static size_t tcap = 0;
    const size_t need = (size_t)grid * kMmaWarps * 4;
    if (getenv("KVMIX_TRACE_FILE")) {
      if (need > tcap) {
        if (tbuf) cudaFree(tbuf);
        check_cuda(cudaMalloc(&tbuf, need * 8), "trace");
        tcap = need;
      }
      check_cuda(cudaMemset(tbuf, 0, need * 8), "trace");
      check_cuda(cudaMemcpyToSymbol(g_trace, &tbuf, sizeof(tbuf)), "trace symbol");
    }
#endif
    kern<<<grid, kMmaWarps * 32, smem, st>>>(p);
#ifdef KVB_TRACE
    if (getenv("KVMIX_TRACE_FILE")) {  // (debug builds) append this launch's timeline
      std::vector<uint64_t> h(need);
      check_cuda(cudaMemcpy(h.data(), tbuf, need * 8, cudaMemcpyDeviceToHost), "trace copy");
      if (FILE* fp = fopen(getenv("KVMIX_TRACE_FILE"), "ab")) {
        const uint64_t hdr[4] = {0x5452414345ull, need / 4, (uint64_t)p.U, (uint64_t)p.Gf};
        fwrite(hdr, 8, 4, fp);
        fwrite(h.data(), 8, need, fp);
        fclose(fp);
      }
    }
#endif
  }
  return p.W;
}

template <int D, int KB, int VB, int R>
int dispatch_gs(MmaParams& p, int BH, Workspace& ws, cudaStream_t st) {
  if constexpr (KB == 3 && D != 128) {
    return 0;  // 3-bit Keys: D = 128 (attend_mma never asks for another)
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



// One launch for the layers L[0, n) (all on this kernel instance): the resident wave is
// shared among the layers in proportion to their cost, each layer keeps its own unit
// ranges, partial slots, counters and merges.
template <int D, int KB, int VB, int R, int GS>
void launch_layers(MmaParams* L, const int* BHs, int n, Workspace& ws, cudaStream_t st, bool pdl) {
  auto kern = attend_mma_layers_kernel<D, KB, VB, R, GS>;
  size_t smem = 0;
  int64_t wave = 0;
  int stages = 0;
  mma_geometry<D, KB, VB, R, GS>(kern, L[0].stage_bytes, stages, smem, wave);
  double tot = 0.0;
  for (int l = 0; l < n; ++l) tot += (double)L[l].Nc * L[l].npass;
  thread_local MmaLayers mp;  // (host staging; the launch copies it)
  mp.n = n;
  int64_t off = 0;
  const int64_t min_cost = knobs().min_cost;
  for (int l = 0; l < n; ++l) {
    MmaParams& p = L[l];
    p.stages = stages;
    const double share = tot > 0.0 ? (double)wave * (double)p.Nc * p.npass / tot : 1.0;
    const int64_t w_cap = std::max<int64_t>(1, std::min<int64_t>(p.N, p.Nc / min_cost));
    p.W = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)(share / p.npass), w_cap));
    // partial slots: as the single-layer launch (a wave + BH), so scratch does not depend on T
    p.pslots = (int)(std::max<int64_t>(wave, p.W) + BHs[l]);
    p.pdl = 1;  // the gate also lets the next launch start early (griddepcontrol.wait is a
                // no-op in a launch without the PDL attribute)
    mma_scratch<D>(p, BHs[l], ws, st);
    mp.off[l] = (int)off;
    mp.l[l] = p;
    off += (int64_t)p.W * p.npass;
  }
  mp.off[n] = (int)off;
  const unsigned grid = (unsigned)((off + kMmaWarps - 1) / kMmaWarps);
  launch_ex(kern, grid, smem, st, pdl, mp);
}

template <int D, int R>
bool dispatch_layers(MmaParams* L, const int* BHs, int n, int kb, int vb, Workspace& ws, cudaStream_t st, bool pdl) {
  switch (kb * 10 + vb) {
    case 22: launch_layers<D, 2, 2, R, 32>(L, BHs, n, ws, st, pdl); return true;
    case 24: launch_layers<D, 2, 4, R, 32>(L, BHs, n, ws, st, pdl); return true;
    case 42: launch_layers<D, 4, 2, R, 32>(L, BHs, n, ws, st, pdl); return true;
    case 44: launch_layers<D, 4, 4, R, 32>(L, BHs, n, ws, st, pdl); return true;
    case 32:
    case 34:
      if constexpr (D == 128) {
        if (vb == 2) launch_layers<D, 3, 2, R, 32>(L, BHs, n, ws, st, pdl);
        else launch_layers<D, 3, 4, R, 32>(L, BHs, n, ws, st, pdl);
        return true;
      }
      return false;
    default: return false;
  }
}

// unit list of a pass: window blocks only with one query row; returns units per (b, kv-head)
int64_t mma_layout(MmaParams& p, const kvmix_cache* c, int nrows) {
  const int64_t T = p.T;
  p.Pw = p.P;
  p.nwb = 0;
  if (nrows == 1 && c->k.quantized == p.P && !knobs().no_window) {
    p.Pw = std::min(T, c->v.quantized);
    if (p.Pw > p.P) p.nwb = (int)((p.Pw - p.P + 31) / 32);
    else p.Pw = p.P;
  }
  return (int64_t)p.Gf + p.nwb + (T - p.Pw + p.tail_unit - 1) / p.tail_unit;
}

struct MmaGeo {
  int per_pass, npass_all, chunk, rows, kb, vb, D, BH;
};

// The layer fields of the launch parameters (everything but the pass split, the warp
// count and the scratch); false when the IMMA kernels do not serve this call.
bool mma_setup(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, bool want_cs,
               const DecodeAppend* da, MmaParams& p, MmaGeo& g) {
  const int rows = (Hq / c->H) * tq;
  const int kb = c->k.bits, vb = c->v.bits;
  if (vb == 3 && !knobs().ws) return false;  // 3-bit Values: the warp-specialized kernel only
  const int D = c->D, gs = c->cfg.group_size;
  if (gs % 32 != 0) return false;  // groups are processed in 32-token blocks
  if (D != 64 && D != 128) return false;
  if (kb == 3 && D != 128) return false;
  // query rows per pass: 2 (one n8 B tile holds two rows' four digits), 4 on the single-warp
  // kernel when there are more (two n8 tiles share every unpacked A fragment: GQA G = 4 reads
  // and unpacks each record once); more rows (G = 8, several query tokens) run as row passes
  // inside one launch, up to kMaxPasses per launch (their warps stream the same records
  // together, so the cache is read from DRAM about once per launch)
  const bool ws_path = knobs().ws == 2 || (knobs().ws == 1 && vb == 3);
  const int per_pass = rows == 1 ? 1 : (rows == 2 || ws_path || knobs().tc || !knobs().r4) ? 2 : 4;
  const int npass_all = (rows + per_pass - 1) / per_pass;
  const int chunk = std::min(npass_all, kMaxPasses);
  const int BH = c->B * c->H;
  const int64_t T = c->total();
  p = MmaParams{};
  p.k = view(c->k);
  p.v = view(c->v);
  p.q = q;
  p.q16 = dt == KVMIX_F16;
  p.tail16 = c->tail_dtype == KVMIX_F16;
  p.H = c->H;
  p.Hq = Hq;
  p.tq = tq;
  p.gs = gs;
  p.cg = c->cgroups();
  p.T = T;
  p.P = (std::min(c->k.quantized, c->v.quantized) / gs) * gs;
  p.Gf = (int)(p.P / gs);
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
  p.want_cs = want_cs;
  p.out = out;
  const Knobs kn = knobs();
  p.tail_unit = kn.tail_unit;
  p.skip_tail = kn.skip_tail;
  p.Qc = kn.group_cost;
  p.flush_blocks = kn.flush_blocks;
  if (da) {  // fused append: only if the aged Value token is outside the fast groups
    if (da->v_age && da->v_j < p.P) return false;
    if (T <= p.P) return false;  // (cannot happen after an append: the new Key is in the window)
  }
  if ((int64_t)BH * mma_layout(p, c, per_pass) >= (int64_t)1 << 31) return false;
  g.per_pass = per_pass;
  g.npass_all = npass_all;
  g.chunk = chunk;
  g.rows = rows;
  g.kb = kb;
  g.vb = vb;
  g.D = D;
  g.BH = BH;
  return true;

}

// the pass fields of launch x0 (row passes [x0, x0 + chunk))
void mma_pass(MmaParams& p, const kvmix_cache* c, const MmaGeo& g, int x0, const DecodeAppend* da) {
  const int r0 = x0 * g.per_pass;
  p.row0 = r0;
  p.rows = g.per_pass;  // rows per pass (the last pass of a launch may hold fewer)
  p.npass = std::min(g.chunk, g.npass_all - x0);
  p.rows_all = std::min(g.rows - r0, p.npass * g.per_pass);
  p.U = (int)mma_layout(p, c, g.per_pass);
  p.N = g.BH * p.U;
  p.cost_bh = (int64_t)p.Qc * p.Gf + (p.U - p.Gf);
  p.Nc = (int64_t)g.BH * p.cost_bh;
  p.fused = 0;
  if (da && r0 == 0) {  // the first launch runs the append; later launches follow in stream order
    p.fused = 1;
    p.da = *da;
  }
}

}  // namespace

bool attend_mma(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
                Workspace& ws, cudaStream_t st, const DecodeAppend* da) {
  MmaParams p;
  MmaGeo g;
  if (!mma_setup(c, q, dt, Hq, tq, out, checksum != nullptr, da, p, g)) return false;
  const int per_pass = g.per_pass, npass_all = g.npass_all, chunk = g.chunk, rows = g.rows;
  const int kb = g.kb, vb = g.vb, D = g.D, BH = g.BH;
  // tcgen05 kernel over the fast groups (all query rows in one pass), then ONE window launch
  // (warp per (pass, b, kv-head)) that runs the fused append and the window and merges
  TcExt ext;
  (void)rows;
  const bool use_tc = npass_all <= kMaxPasses && p.Gf > 0 && attend_tc_eligible(c, rows) &&
                      attend_tc_launch(c, q, dt == KVMIX_F16, Hq, tq, p.Gf, checksum != nullptr, ws, st, &ext);
  double cs_total = 0.0;
  if (use_tc && checksum) {
    checksum_kernel<<<1, 32, 0, st>>>(ext.cs, ext.slots, const_cast<double*>(ext.cs) + ext.slots);
    after_launch("checksum_kernel");
    double part = 0.0;
    check_cuda(cudaMemcpyAsync(&part, ext.cs + ext.slots, 8, cudaMemcpyDeviceToHost, st), "memcpy");
    check_cuda(cudaStreamSynchronize(st), "sync");
    cs_total += part;
  }
  // programmatic dependent launch: only when the caller (kvmix_*attend_layers) asked for it
  // for this call, a single IMMA launch serves it and no checksum round trip follows
  p.pdl = (take_pdl() && !use_tc && !checksum && npass_all <= chunk) ? 1 : 0;
  if (use_tc) {
    p.wonly = 1;
    p.ext_ml = ext.ml;
    p.ext_acc = ext.acc;
    p.ext_C = ext.C;
    p.ext_NT = ext.NT;
    p.ext_Tb = ext.Tb;
    p.ext_R = ext.R;
  }
  for (int x0 = 0; x0 < npass_all; x0 += chunk) {
    const int r0 = x0 * per_pass;
    const int nrows = per_pass;
    mma_pass(p, c, g, x0, da);
    int W = 0;
    const char* kname = "attend_mma_kernel";
    // the warp-specialized kernel serves 3-bit Values (KVMIX_WS = 1, default) or every tier
    // (KVMIX_WS = 2); the single-warp kernel is ~5% faster on the 2/4-bit tiers (profiles/r2)
    if (!use_tc && (knobs().ws == 2 || (knobs().ws == 1 && vb == 3))) {
      p.pdl = 0;
      W = attend_ws_launch(p, D, nrows, kb, vb, BH, ws, st);
      kname = "attend_ws_kernel";
    }
    if (W == 0) {
      kname = "attend_mma_kernel";
#define KVB_DISPATCH_D(DD)                                                  \
      if (D == DD) {                                                        \
        if (nrows == 1) W = dispatch_bits<DD, 1>(p, kb, vb, BH, ws, st);   \
        else if (nrows == 2) W = dispatch_bits<DD, 2>(p, kb, vb, BH, ws, st); \
        else W = dispatch_bits<DD, 4>(p, kb, vb, BH, ws, st);              \
      }
      KVB_DISPATCH_D(64)
      KVB_DISPATCH_D(128)
#undef KVB_DISPATCH_D
    }
    if (W == 0) {
      if (r0 == 0 && !use_tc) return false;  // nothing launched yet: the caller takes the generic path
      throw Error(KVMIX_RUNTIME_ERROR, "attend: tensor-core pass unavailable after the first");
    }
    after_launch(kname);
    if (checksum) {
      const size_t nslot = (size_t)p.npass * p.pslots;
      checksum_kernel<<<1, 32, 0, st>>>(p.part_cs, nslot, p.part_cs + nslot);
      after_launch("checksum_kernel");
      double part = 0.0;
      check_cuda(cudaMemcpyAsync(&part, p.part_cs + nslot, 8, cudaMemcpyDeviceToHost, st), "memcpy");
      check_cuda(cudaStreamSynchronize(st), "sync");
      cs_total += part;
    }
  }
  if (checksum) *checksum = cs_total;
  return true;
}

// The layers of one decode step (kvmix_*attend_layers; distinct caches on the current
// device; k == nullptr: attention only). Every layer the single IMMA launch serves is
// queued with its decode append and launched together with the other layers of the same
// kernel instance (KVmix tiers: two launches per step); the rest run alone, in order.
// Layers are independent, so only each layer's own order (append, then attention) matters.
void attend_layers(kvmix_cache* const* caches, int n, const void* const* k, const void* const* v,
                   kvmix_dtype kv_dt, int t, const void* const* q, kvmix_dtype q_dt, int Hq, int tq,
                   float* const* out, cudaStream_t st) {
  struct Group {
    int D, kb, vb, R;
    std::vector<MmaParams> p;
    std::vector<int> bh;
  };
  std::vector<Group> groups;
  int launched = 0;
  auto flush = [&](Group& g) {
    if (g.p.empty()) return;
    Workspace ws(st);
    const bool pdl = launched > 0 && knobs().pdl;  // after the call's first launch
    const int n = (int)g.p.size();
    bool ok = false;
    if (g.D == 64) ok = g.R == 1   ? dispatch_layers<64, 1>(g.p.data(), g.bh.data(), n, g.kb, g.vb, ws, st, pdl)
                        : g.R == 2 ? dispatch_layers<64, 2>(g.p.data(), g.bh.data(), n, g.kb, g.vb, ws, st, pdl)
                                   : dispatch_layers<64, 4>(g.p.data(), g.bh.data(), n, g.kb, g.vb, ws, st, pdl);
    else ok = g.R == 1   ? dispatch_layers<128, 1>(g.p.data(), g.bh.data(), n, g.kb, g.vb, ws, st, pdl)
              : g.R == 2 ? dispatch_layers<128, 2>(g.p.data(), g.bh.data(), n, g.kb, g.vb, ws, st, pdl)
                         : dispatch_layers<128, 4>(g.p.data(), g.bh.data(), n, g.kb, g.vb, ws, st, pdl);
    if (!ok) throw Error(KVMIX_RUNTIME_ERROR, "attend: multi-layer launch unavailable");
    after_launch("attend_mma_layers_kernel");
    ++launched;
    g.p.clear();
    g.bh.clear();
  };
  auto try_add = [&](const kvmix_cache* c, const void* ql, float* o, const DecodeAppend* da) {
    const Knobs& kn = knobs();
    if (kn.tc || !kn.layers || c->cfg.group_size != 32) return false;
    MmaParams p;
    MmaGeo g;
    if (!mma_setup(c, ql, q_dt, Hq, tq, o, false, da, p, g)) return false;
    if (g.npass_all > g.chunk) return false;                       // several launches per layer
    if (kn.ws == 2 || (kn.ws == 1 && g.vb == 3)) return false;    // warp-specialized kernel
    mma_pass(p, c, g, 0, da);
    const int R = g.per_pass;
    Group* gr = nullptr;
    for (Group& x : groups)
      if (x.D == g.D && x.kb == g.kb && x.vb == g.vb && x.R == R) gr = &x;
    if (!gr) {
      groups.push_back(Group{g.D, g.kb, g.vb, R, {}, {}});
      gr = &groups.back();
    }
    if ((int)gr->p.size() == kMaxLayers) flush(*gr);
    gr->p.push_back(p);
    gr->bh.push_back(g.BH);
    return true;
  };
  // a layer that raises (shape / capacity errors) leaves the layers before it complete, as
  // the per-layer loop does: their queued launches (which hold their committed appends) run
  // before the error propagates
  try {
  for (int l = 0; l < n; ++l) {
    kvmix_cache* c = caches[l];
    if (k) {
      if (c->total() + t > c->cap || t < 1) {
        cache_append(c, k[l], v[l], kv_dt, t, st);  // raises the reference's errors
      } else {
        check_query_shape(c, Hq, tq);
        DecodeAppend da;
        if (cache_append_decode_plan(c, k[l], v[l], kv_dt, t, &da)) {
          if (try_add(c, q[l], out[l], &da)) continue;
          launch_decode_append(da, st);
        } else {
          cache_append(c, k[l], v[l], kv_dt, t, st);
        }
      }
    }
    check_attend(c, Hq, tq);
    if (try_add(c, q[l], out[l], nullptr)) continue;
    Workspace ws(st);
    attend(c, q[l], q_dt, Hq, tq, out[l], nullptr, ws, st);
  }
  } catch (...) {
    for (Group& g : groups) flush(g);
    throw;
  }
  for (Group& g : groups) flush(g);
}

}  // namespace kvb

