// attention_ws.cuh -- warp-specialized variant of the fused decode-attention kernel
// (included by attention_mma.cu inside its anonymous namespace; shares MmaParams, the record
// geometry, the IMMA fragment layouts and the stream-K partition / merge with
// attend_mma_kernel).
//
// Why: the single-warp kernel issues ~450 instructions per 32-token group (K2V2) with 16
// warps per SM at ~125 registers; ncu shows it latency/issue bound (59% issue-active,
// `wait` / `short_scoreboard` stalls) at 0.60 of HBM. Here every unit range is worked by a
// PAIR of warps with disjoint roles and register sets, so two independent instruction
// streams overlap and each warp carries fewer live registers:
//   * the K-warp (Keys): per group the fixed-point B digits of q * scale (IMMA s8 B operand),
//     the code x digit IMMAs of the two 16-token Key tiles per 32-token block, the min-term
//     dot product and the Mixed3 narrow-slot correction -> 32 scores per block and query row
//     (log2 units) into a shared-memory score ring;
//   * the V-warp (Values): online softmax over the scores (lazy reference max), the u8 Value
//     digits of p * scale * 2^E and the Value IMMAs into int32 accumulators that persist
//     across blocks, the folds, the full-precision window tokens and the epilogue / merge.
// Synchronization is per pair and asynchronous: mbarriers for the TMA ring (complete_tx),
// for "score block full" (K -> V) and "score block free" (V -> K). The V-warp is the last
// reader of a ring stage, so it refills it. Roles alternate per CTA so both roles land on
// every SM sub-partition.

#ifndef KVB_WS_PAIRS
#define KVB_WS_PAIRS 2  // warp pairs per CTA
#endif
#ifndef KVB_WS_MIN_CTAS
#define KVB_WS_MIN_CTAS 5  // CTAs per SM the registers are sized for (20 warps: <= 96 registers)
#endif
constexpr int kWsPairs = KVB_WS_PAIRS;
constexpr int kScoreSlots = 8;  // score-ring depth (>= stages x blocks per group: no free-slot waits)

// Per-pair dynamic shared layout (bytes):
//   ring[S][SB] | sc[SR][R][32] f32 | pb[R][32] f32 | kstage (WarpLayout::kK) | vbs (kV)
//   | qbuf[D] f32 | csm[32] f64 | sacc[R][D] f32 | vtab[D] u32 | bars: full[S], sfull[SR], sempty[SR]
template <int D, int KB, int R>
struct PairLayout {
  using WL = WarpLayout<D, KB, R>;
  static constexpr int kSc = kScoreSlots * R * 32 * 4;
  static constexpr int kPb = R * 32 * 4;
  static constexpr int kQb = D * 4;
  static constexpr int kCs = 32 * 8;
  static constexpr int kAcc = R * D * 4;
  static constexpr int kVtab = D * 4 + R * (D / 32) * 32 * 4;  // vtab + nw (3-bit Values)
  static constexpr int kFixed = kSc + kPb + WL::kK + WL::kV + kQb + kCs + kAcc + kVtab;
  __host__ __device__ static constexpr size_t bytes(int stages, uint32_t stage_bytes) {
    const size_t n = (size_t)stages * stage_bytes + kFixed + (size_t)(stages + 2 * kScoreSlots) * 8;
    return (n + 127) / 128 * 128;
  }
};

template <int D, int KB, int VB, int R, int GS>
struct WsGeo {
  using SG = StageGeo<D, KB, VB, R, GS>;
  // ring stage: the group record, plus the Value tokens' segment info for 3-bit Values
  static constexpr uint32_t kStageX = SG::kStage + (VB == 3 ? (uint32_t)GS * 8u : 0u);
  static constexpr int stages_for(int occ) {
    return (int)(((227L * 1024 / occ - 1024) / kWsPairs - (long)PairLayout<D, KB, R>::bytes(0, 0) - 128) /
                 (long)(kStageX ? kStageX : 1));
  }
  static constexpr int kStages = GS == 0 ? 0
                                 : stages_for(KVB_WS_MIN_CTAS) >= 2 ? (stages_for(KVB_WS_MIN_CTAS) < 4 ? stages_for(KVB_WS_MIN_CTAS) : 4)
                                                                     : 2;
};

// mbarrier ops on precomputed shared-memory addresses (no generic-to-shared conversion per call)
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// order-preserving float <-> u32 (for REDUX.MAX over signed floats, -inf included)
__device__ __forceinline__ uint32_t f2ord(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// named barrier of one warp pair (immediate ids: a register id makes ptxas reserve all 16
// barriers per CTA, which caps the CTAs per SM)
__device__ __forceinline__ void pair_sync(int pl) {
  static_assert(kWsPairs <= 4, "pair barriers 1..4");
  switch (pl) {
    case 0: asm volatile("bar.sync 1, 64;\n" ::: "memory"); break;
    case 1: asm volatile("bar.sync 2, 64;\n" ::: "memory"); break;
    case 2: asm volatile("bar.sync 3, 64;\n" ::: "memory"); break;
    default: asm volatile("bar.sync 4, 64;\n" ::: "memory"); break;
  }
}

template <int D, int KB, int VB, int R, int GS>
__global__ void __launch_bounds__(kWsPairs * 64, KVB_WS_MIN_CTAS) attend_ws_kernel(MmaParams p) {
  static_assert(D == 64 || D == 128, "IMMA attention handles D in {64, 128}");
  static_assert(VB >= 2 && VB <= 4, "Values: 2, 3 or 4 bits");
  constexpr bool V3 = VB == 3;
  constexpr int VBS = vstore_bits(VB);  // 3-bit Values: 4-bit fields
  static_assert(R == 1 || R == 2, "one or two query rows per pass");
  constexpr bool K3 = KB == 3;
  static_assert(!K3 || D == 128, "3-bit Keys: D = 128");
  constexpr int NK = D / 32, NM = D / 16;
  constexpr int KW = lane_words<D, KB>(), VW = lane_words<D, VBS>();
  constexpr int KB2 = K3 ? 2 : KB;
  constexpr int CK = 8 / KB2, CV = 8 / VBS;
  constexpr uint32_t KMASK = KB2 == 4 ? 0x0F0F0F0Fu : 0x03030303u;
  constexpr uint32_t VMASK = VBS == 4 ? 0x0F0F0F0Fu : 0x03030303u;
  constexpr int LC = D / 32, QL = D / 4, CGMAX = D / 32;
  using WL = WarpLayout<D, KB, R>;
  using PL = PairLayout<D, KB, R>;
  using SG = StageGeo<D, KB, VB, R, GS>;
  using WG = WsGeo<D, KB, VB, R, GS>;

  extern __shared__ __align__(128) uint8_t dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pl = warp >> 1;
  // roles alternate [K, V, V, K] / [V, K, K, V] per CTA: both roles on every sub-partition
  const bool kwarp = (((warp & 1) ^ (warp >> 1) ^ (int)(blockIdx.x & 1)) & 1) == 0;
  const int gp = blockIdx.x * kWsPairs + pl;
  const int pass = gp % p.npass, wg = gp / p.npass;
  if (wg >= p.W) return;  // (both warps of the pair)
  const int prow0 = p.row0 + pass * p.rows;
  const int prows = min(p.rows, p.rows_all - pass * p.rows);
  const size_t pbase = (size_t)pass * p.pslots;
  const int g = lane >> 2, t = lane & 3;
  const int G = p.Hq / p.H;
  const int gs = GS ? GS : p.gs;
  const int CG = GS ? D / GS : p.cg;
  const int NBLK = gs / 32;
  const int S = GS ? WG::kStages : p.stages;
  const uint32_t SB = GS ? SG::kStage : p.stage_bytes;  // group record bytes
  const uint32_t IB = V3 ? (uint32_t)gs * 8u : 0u;       // + the Value info of its tokens (3-bit Values)
  const uint32_t SBX = SB + IB;                          // ring stage stride
  const uint32_t KTB = GS ? SG::kKT : p.kt_bytes, VTB = GS ? SG::kVT : p.vt_bytes;
  const uint32_t VMB = GS ? SG::kVM : p.vm_bytes;
  const int64_t c_beg = (int64_t)wg * p.Nc / p.W, c_end = (int64_t)(wg + 1) * p.Nc / p.W;
  const int u_beg = unit_at_cost(p, c_beg), u_end = unit_at_cost(p, c_end);
  if (u_beg >= u_end) {  // no unit starts in this cost range: neutral partial (V-warp only)
    if (kwarp) return;
    const int bh = (int)(c_beg / p.cost_bh);
    int w0, w1;
    bh_warps(p, bh, w0, w1);
    if (wg < w0 || wg > w1) return;
    if (lane < prows) p.part_ml[(pbase + wg + bh) * p.rows + lane] = make_float2(-INFINITY, 0.f);
    if (arrive_last(p, bh, lane, pass, wg)) merge_bh<D>(p, bh, lane, pass, prow0, prows);
    return;
  }

  uint8_t* base = dsm + (size_t)pl * PL::bytes(S, SBX);
  uint8_t* ring = base;
  float* sc = reinterpret_cast<float*>(ring + (size_t)S * SBX);  // [SR][R][32]
  float* pb = sc + kScoreSlots * R * 32;                         // [R][32]
  uint8_t* kstage = reinterpret_cast<uint8_t*>(pb + R * 32);
  uint32_t* kbs = reinterpret_cast<uint32_t*>(kstage);
  float* ytab = reinterpret_cast<float*>(kstage + WL::kY);
  uint32_t* ntab = reinterpret_cast<uint32_t*>(kstage + WL::kY + R * D * 4);
  uint8_t* vbs = kstage + WL::kK;
  float* qbuf = reinterpret_cast<float*>(vbs + WL::kV);
  double* csm = reinterpret_cast<double*>(qbuf + D);
  float* sacc = reinterpret_cast<float*>(csm + 32);  // [R][D]
  uint32_t* vtab = reinterpret_cast<uint32_t*>(sacc + R * D);  // [D] 3-bit Values: field of row 0
  float* nw = reinterpret_cast<float*>(vtab + D);                // [R][D/32][32] 3-bit Values: p (ws - s) per token
  uint64_t* full = reinterpret_cast<uint64_t*>(nw + R * (D / 32) * 32);
  uint64_t* sfull = full + S;
  uint64_t* sempty = sfull + kScoreSlots;
  const uint32_t full_a = smem_u32(full), sfull_a = smem_u32(sfull), sempty_a = smem_u32(sempty);
  // The TMA ring bounds the K-warp's lead: it waits for stage s, which the V-warp refills only
  // after consuming all blocks of the group S earlier, so when the range has no window blocks
  // (score blocks outside the ring's flow control) and S * NBLK <= kScoreSlots, a fast group's
  // score slot is always free (the V-warp still arrives on "free" after every block).
  bool slot_free = S * NBLK <= kScoreSlots;
  if (R == 1 && p.nwb > 0) {
    for (int u = u_beg; u < u_end && slot_free;) {
      const int bh = u / p.U, lo = u - bh * p.U, hi = min(u_end - bh * p.U, p.U);
      if (hi > p.Gf && lo < p.Gf + p.nwb) slot_free = false;
      u = bh * p.U + hi;
    }
  }

  if (!kwarp) {
    // zero the B staging (columns of absent query rows / digits stay 0); barriers
    uint4* z = reinterpret_cast<uint4*>(kstage);
    for (int i = lane; i < (WL::kK + WL::kV) / 16; i += 32) z[i] = make_uint4(0u, 0u, 0u, 0u);
    if constexpr (V3) {  // channel -> {word offset | shift << 16} of token 0 in a 4-bit Value tile
      for (int d = lane; d < D; d += 32) {
        int w, sh;
        imma_field(false, D, 4, 0, d, &w, &sh);
        vtab[d] = (uint32_t)w | ((uint32_t)sh << 16);
      }
    }
    if (lane == 0) {
      for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
      for (int s = 0; s < kScoreSlots; ++s) {
        mbar_init(&sfull[s], 1);
        mbar_init(&sempty[s], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
  }
  pair_sync(pl);

  // shared walk over the unit range: (b, kv-head) segments [lo, hi) of units
  // ---------------------------------------------------------------------------------------
  if (kwarp) {
    // ======================================= K-warp =======================================
    // fused 1-token append (pass 0): the pair whose range holds a (b, kv-head)'s first window
    // unit appends its token, then publishes it to every pass (the partner V-warp and later
    // pairs wait on the flag before reading the window)
    if (p.fused && pass == 0) {
      for (int bh = u_beg / p.U; bh <= (u_end - 1) / p.U; ++bh) {
        const int x = bh * p.U + p.Gf;
        if (x >= u_beg && x < u_end) {
          decode_append_warp(p.da, bh, lane);
          __threadfence();
          __syncwarp();
          if (lane < p.npass) st_release(p.flags + (size_t)lane * p.nbh + bh, 1u);
        }
      }
    }
    const int Lq = lane % QL;
    const bool qdup = lane >= QL;
    const int kkL = Lq >> 3, hL = (Lq & 7) >> 2, tL = Lq & 3;
    const float clsL = pow2i(-KB2 * ((kkL + NK * hL) % CK));
    const float clsH = K3 ? 4.f * pow2i(-((kkL + NK * hL) & 7)) : 0.f;
    const float invL = pow2i(KB2 * ((kkL + NK * hL) % CK));
    const float clsHL = clsH * invL;
    if constexpr (K3) {
      for (int d = lane; d < D; d += 32) {
        int w, sh;
        imma_field(true, D, 2, 0, d, &w, &sh);
        ntab[d] = (uint32_t)w | ((uint32_t)sh << 16);
      }
      __syncwarp();
    }
    const int my_r = t >> 1;
    int s = 0, sl = 0;
    uint32_t phase = 0, sphase = 0;
    // publish one score block (lane (g, t even) holds tokens g, g+8, 16+g, 24+g of row my_r)
    auto put_scores = [&](float a0, float b0, float a1, float b1) {
      if (!slot_free) mbar_wait_a(sempty_a + 8 * sl, sphase ^ 1u);
      if ((t & 1) == 0 && my_r < prows) {
        float* o = sc + (sl * R + my_r) * 32;
        o[g] = a0;
        o[g + 8] = b0;
        o[16 + g] = a1;
        o[24 + g] = b1;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_a(sfull_a + 8 * sl);
      if (++sl == kScoreSlots) {
        sl = 0;
        sphase ^= 1u;
      }
    };
    for (int u = u_beg; u < u_end;) {
      const int bh = u / p.U;
      const int lo = u - bh * p.U;
      const int hi = min(u_end - bh * p.U, p.U);
      u = bh * p.U + hi;
      const int b = bh / p.H, h = bh % p.H;
      const int cb11 = (int)(((unsigned)p.k.gbh(bh) * (unsigned)D) % 11u);
      (void)cb11;
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
      if constexpr (R == 1) {
        if (p.nwb > 0) {
          __syncwarp();  // the previous segment's window reads of qbuf are done
#pragma unroll
          for (int c = 0; c < 4; ++c) qbuf[4 * Lq + c] = qv[0][c];
        }
      }
      float qc[R][4];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) qc[r][c] = qv[r][c] * clsL;
      if (p.want_cs) csm[lane] = 0.0;

      const int g_stop = min(hi, p.Gf);
      for (int grp = lo; grp < g_stop; ++grp) {
        mbar_wait_a(full_a + 8 * s, phase);
#ifdef KVB_DIAG_MEMONLY  // diagnostic build: the data movement and the pair protocol only
        for (int blk = 0; blk < NBLK; ++blk) put_scores(0.f, 0.f, 0.f, 0.f);
        if (++s == S) {
          s = 0;
          phase ^= 1u;
        }
        continue;
#endif
        const uint8_t* st = ring + (size_t)s * SBX;
        const uint32_t* kt = reinterpret_cast<const uint32_t*>(st);
        const uint32_t* km = reinterpret_cast<const uint32_t*>(st + KTB + VTB + VMB);
        float betaL, wsc0;
        uint32_t kb[NK][2], kbh[K3 ? NK : 1][2];
        int nmod = 0, omod = 0;
        {
          const uint4 m4 = *reinterpret_cast<const uint4*>(km + 4 * Lq);
          const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
          float scl[4], mn[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float2 f = meta_pair(mw[c]);
            scl[c] = f.x;
            mn[c] = f.y;
          }
          if constexpr (K3) {
            const int2 inf = __ldg(p.k.info + grp);
            nmod = inf.x % 11;
            omod = inf.y % 11;
          }
          float beta[R], isig[R];
          __syncwarp();  // previous group's reads of kbs / ytab are done
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float x[4], xh[4], mx = 0.f, bt = 0.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              x[c] = qc[r][c] * scl[c];
              mx = fmaxf(mx, fabsf(x[c]));
              if constexpr (K3) {
                xh[c] = qc[r][c] * clsHL * scl[c];
                mx = fmaxf(mx, fabsf(xh[c]));
              }
              bt = fmaf(qc[r][c], mn[c], bt);
            }
            bt = qdup ? 0.f : bt * invL;
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
              float4 y;
              y.x = qc[r][0] * invL * (wide_scale(scl[0]) - scl[0]);
              y.y = qc[r][1] * invL * (wide_scale(scl[1]) - scl[1]);
              y.z = qc[r][2] * invL * (wide_scale(scl[2]) - scl[2]);
              y.w = qc[r][3] * invL * (wide_scale(scl[3]) - scl[3]);
              *reinterpret_cast<float4*>(ytab + r * D + 4 * lane) = y;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bt += __shfl_xor_sync(0xffffffffu, bt, o);
            beta[r] = bt;
          }
          __syncwarp();
          {
            const bool has_col = g < WL::kKC;
            const uint32_t* zsrc = reinterpret_cast<const uint32_t*>(kstage + WL::kZ) + t * (2 * NK);
            const uint32_t* src = has_col ? kbs + (g * 4 + t) * (2 * NK) : zsrc;
#pragma unroll
            for (int kk = 0; kk < NK; kk += 2) {
              const uint4 v = *reinterpret_cast<const uint4*>(src + 2 * kk);
              kb[kk][0] = v.x;
              kb[kk][1] = v.y;
              kb[kk + 1][0] = v.z;
              kb[kk + 1][1] = v.w;
            }
            if constexpr (K3) {
#pragma unroll
              for (int kk = 0; kk < NK; kk += 2) {
                const uint32_t* srch = has_col ? src + WL::kKC * 4 * 2 * NK : zsrc;
                const uint4 v = *reinterpret_cast<const uint4*>(srch + 2 * kk);
                kbh[kk][0] = v.x;
                kbh[kk][1] = v.y;
                kbh[kk + 1][0] = v.z;
                kbh[kk + 1][1] = v.w;
              }
            }
          }
          const int rr = my_r < R ? my_r : 0;
          float is = isig[0], bb = beta[0];
#pragma unroll
          for (int r = 1; r < R; ++r)
            if (rr == r) {
              is = isig[r];
              bb = beta[r];
            }
          wsc0 = pow2i(16 * (t & 1)) * is * p.inv * kLog2e;
          betaL = bb * p.inv * kLog2e;
        }

        for (int blk = 0; blk < NBLK; ++blk) {
          const uint32_t* kt2 = kt + (size_t)(2 * blk) * tile_words(D, KB);
          float la[2], lb[2];
          uint32_t kw[2][KW];
          lds_tile<D, KB>(kt2, lane, kw[0]);
          lds_tile<D, KB>(kt2 + tile_words(D, KB), lane, kw[1]);
          int dk[2][4];
#pragma unroll
          for (int u2 = 0; u2 < 2; ++u2) dk[u2][0] = dk[u2][1] = dk[u2][2] = dk[u2][3] = 0;
#pragma unroll
          for (int kk = 0; kk < NK; ++kk) {
            const int q0 = kk, q1 = kk + NK;
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) {
              const uint32_t a0 = kw[u2][(q0 / CK) * 2 + 0] & (KMASK << (KB2 * (q0 % CK)));
              const uint32_t a1 = kw[u2][(q0 / CK) * 2 + 1] & (KMASK << (KB2 * (q0 % CK)));
              const uint32_t a2 = kw[u2][(q1 / CK) * 2 + 0] & (KMASK << (KB2 * (q1 % CK)));
              const uint32_t a3 = kw[u2][(q1 / CK) * 2 + 1] & (KMASK << (KB2 * (q1 % CK)));
              imma_us(dk[u2], a0, a1, a2, a3, kb[kk][0], kb[kk][1]);
              if constexpr (K3) {
                constexpr int HW = D * 2 / 64;
                const uint32_t h0 = kw[u2][HW + 0] & (0x01010101u << q0);
                const uint32_t h1 = kw[u2][HW + 1] & (0x01010101u << q0);
                const uint32_t h2 = kw[u2][HW + 0] & (0x01010101u << q1);
                const uint32_t h3 = kw[u2][HW + 1] & (0x01010101u << q1);
                imma_us(dk[u2], h0, h1, h2, h3, kbh[kk][0], kbh[kk][1]);
              }
            }
          }
          float corr[4] = {0.f, 0.f, 0.f, 0.f};
          float fac[4] = {1.f, 1.f, 1.f, 1.f};
          if constexpr (K3) {
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
                  const uint32_t tb = ntab[d];
                  const uint32_t code = (tile[(tb & 0xffffu) + rowoff] >> (tb >> 16)) & 3u;
#pragma unroll
                  for (int r = 0; r < R; ++r) dlt[r] = fmaf((float)code, ytab[r * D + d], dlt[r]);
                }
              }
            }
            const float wsn = p.inv * kLog2e;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              float c = __shfl_sync(0xffffffffu, dlt[0], 4 * g + x);
              if constexpr (R == 2) {
                const float c1 = __shfl_sync(0xffffffffu, dlt[1], 4 * g + x);
                c = my_r ? c1 : c;
              }
              corr[x] = c * wsn;
            }
            if (nmod == 0) {
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                const int tgx = 32 * blk + g + 8 * x;
                if ((omod + tgx) % 11 == 10) fac[x] = 7.0f / 3.0f;
              }
            }
          }
#pragma unroll
          for (int u2 = 0; u2 < 2; ++u2) {
            float pa = (float)(dk[u2][0] + (dk[u2][1] << 8)) * wsc0;
            float pbb = (float)(dk[u2][2] + (dk[u2][3] << 8)) * wsc0;
            pa += __shfl_xor_sync(0xffffffffu, pa, 1);
            pbb += __shfl_xor_sync(0xffffffffu, pbb, 1);
            if constexpr (K3) {
              la[u2] = fmaf(pa, fac[2 * u2], betaL) + corr[2 * u2];
              lb[u2] = fmaf(pbb, fac[2 * u2 + 1], betaL) + corr[2 * u2 + 1];
            } else {
              la[u2] = pa + betaL;
              lb[u2] = pbb + betaL;
            }
          }
          if (p.want_cs && my_r < prows && (t & 1) == 0) csm[lane] += (double)(((la[0] + lb[0]) + (la[1] + lb[1])) * kLn2);
          put_scores(la[0], lb[0], la[1], lb[1]);
        }
        if (++s == S) {
          s = 0;
          phase ^= 1u;
        }
      }

      // window blocks (one query row): the fp16 / fp32 Key ring, lane = token
      if (p.fused && hi > p.Gf && !(pass == 0 && lo <= p.Gf)) {
        while (ld_acquire(p.flags + (size_t)pass * p.nbh + bh) == 0u) __nanosleep(32);
      }
      if constexpr (R == 1) {
        const int wb_lo = max(lo, p.Gf) - p.Gf, wb_hi = min(hi, p.Gf + p.nwb) - p.Gf;
        if (wb_lo < wb_hi) __syncwarp();
        for (int wb = wb_lo; wb < wb_hi; ++wb) {
          const int64_t j0 = p.P + 32 * (int64_t)wb;
          const int jt = g + 8 * t;
          const int64_t jj = j0 + jt;
          float slv = -INFINITY;
          if (jj < p.Pw) {
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
            if (p.want_cs) csm[lane] += (double)scn;
            slv = scn * kLog2e;
          }
          mbar_wait_a(sempty_a + 8 * sl, sphase ^ 1u);
          sc[sl * R * 32 + jt] = slv;
          __syncwarp();
          if (lane == 0) mbar_arrive_a(sfull_a + 8 * sl);
          if (++sl == kScoreSlots) {
            sl = 0;
            sphase ^= 1u;
          }
        }
      }
      if (p.want_cs) {
        double csl = csm[lane];
        for (int o = 16; o > 0; o >>= 1) csl += __shfl_xor_sync(0xffffffffu, csl, o);
        if (lane == 0) atomicAdd(p.part_cs + pbase + wg + bh, csl);
      }
    }
    return;
  }

  // ========================================= V-warp ========================================
  int rec_i, rec_g, left_bh, left_all;
  {
    int i_bh = u_beg / p.U, i_g = u_beg - i_bh * p.U;
    if (i_g >= p.Gf) {
      ++i_bh;
      i_g = 0;
    }
    rec_i = i_bh * p.Grec + i_g;
    rec_g = i_g;
    left_bh = p.Gf - i_g;
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
        mbar_arrive_expect_tx(&full[s], SBX);
        bulk_g2s(ring + (size_t)s * SBX, reinterpret_cast<const uint8_t*>(p.k.tiles) + (size_t)rec_i * SB, SB, &full[s],
                 evict_first_policy());
        if constexpr (V3)  // (b, kv-head independent: the shrink rule is uniform)
          bulk_g2s(ring + (size_t)s * SBX + SB, p.v.info + (size_t)rec_g * gs, IB, &full[s], evict_first_policy());
      }
      --left_all;
      ++rec_i;
      ++rec_g;
      if (--left_bh == 0) {
        rec_i += p.Grec - p.Gf;
        rec_g = 0;
        left_bh = p.Gf;
      }
    }
  };
  for (int s = 0; s < S; ++s) issue_next(s);

  const int my_r = t >> 1;  // accumulator fragment row of this lane (digit columns 2t, 2t+1)
  const int cq = lane >> 3, tq = lane & 7;  // Value B build: channel group cq, token quad tq
  const bool cg_ok = cq < CG;
  int s = 0, sl = 0;
  uint32_t phase = 0, sphase = 0;
  for (int u = u_beg; u < u_end;) {
    const int bh = u / p.U;
    const int lo = u - bh * p.U;
    const int hi = min(u_end - bh * p.U, p.U);
    u = bh * p.U + hi;
    const int b = bh / p.H, h = bh % p.H;

    float m_run[R], l_lane[R], bias[R];
    float corr[V3 ? R : 1][V3 ? LC : 1];  // 3-bit Values: narrow-slot corrections of this lane's channels
#pragma unroll
    for (int r = 0; r < R; ++r) {
      m_run[r] = -INFINITY;
      l_lane[r] = 0.f;
      bias[r] = 0.f;
      if constexpr (V3) {
#pragma unroll
        for (int c = 0; c < LC; ++c) corr[r][c] = 0.f;
      }
    }
    int accv[NM][4];
#pragma unroll
    for (int i = 0; i < NM; ++i) accv[i][0] = accv[i][1] = accv[i][2] = accv[i][3] = 0;
    int e_cur = 0, nacc = 0;
    bool dirty = false;
    __syncwarp();  // the previous segment's reads of sacc are done
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < LC; ++c) sacc[r * D + lane * LC + c] = 0.f;
    __syncwarp();

    // fold the int32 accumulators into sacc (fp32): sacc = (sacc + acc 2^-E) alpha_row
    auto flush = [&](const float (&alpha)[R]) {
      const float w0 = pow2i(16 * (t & 1) - e_cur);
      const float w1 = w0 * 256.f;
      float al = alpha[0];
#pragma unroll
      for (int r = 1; r < R; ++r)
        if (my_r == r) al = alpha[r];
#pragma unroll
      for (int mt = 0; mt < NM; ++mt) {
        const float c0 = pow2i(-VBS * (mt % CV)), c1 = pow2i(-VBS * ((mt + NM) % CV));
        float f0 = fmaf((float)accv[mt][1], w1, (float)accv[mt][0] * w0) * c0;
        float f1 = fmaf((float)accv[mt][3], w1, (float)accv[mt][2] * w0) * c1;
        f0 += __shfl_xor_sync(0xffffffffu, f0, 1);
        f1 += __shfl_xor_sync(0xffffffffu, f1, 1);
        if ((t & 1) == 0 && my_r < R) {
          float* a = sacc + my_r * D + 16 * mt + g;
          a[0] = (a[0] + f0) * al;
          a[8] = (a[8] + f1) * al;
        }
        accv[mt][0] = accv[mt][1] = accv[mt][2] = accv[mt][3] = 0;
      }
      nacc = 0;
    };

    // one 32-token block: scores (lane j = token j) -> p; Value digits; IMMA
    auto value_block = [&](const uint32_t* vt2, const uint32_t* vm2, int64_t jb, const int2* vinf2) {
      mbar_wait_a(sfull_a + 8 * sl, sphase);
      float x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = r < prows ? sc[(sl * R + r) * 32 + lane] : -INFINITY;
      __syncwarp();
      if (lane == 0 && !slot_free) mbar_arrive_a(sempty_a + 8 * sl);  // (slot_free: nobody waits; see above)
      if (++sl == kScoreSlots) {
        sl = 0;
        sphase ^= 1u;
      }
#ifdef KVB_DIAG_MEMONLY
      if (vt2) return;
#endif
      float alpha[R], pj[R];
      bool moved = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float bmax = ord2f(__reduce_max_sync(0xffffffffu, f2ord(x[r])));
        const float m_new = bmax > m_run[r] + (float)kLazy ? bmax : m_run[r];
        alpha[r] = fast_exp2(m_run[r] - m_new);  // (-inf - -inf = NaN only while the row is empty)
        if (m_run[r] == m_new) alpha[r] = 1.0f;
        pj[r] = fast_exp2(x[r] - m_new);
        l_lane[r] = l_lane[r] * alpha[r] + pj[r];
        m_run[r] = m_new;
        moved |= alpha[r] != 1.0f;
      }
      // Value metas of this lane's token quad and channel group ([cg][token] in the record)
      float sv[4], mv[4];
      {
        const uint4 w4 = cg_ok ? *reinterpret_cast<const uint4*>(vm2 + (size_t)cq * gs + 4 * tq) : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = meta_pair(w[i]);
          sv[i] = f.x;
          mv[i] = f.y;
        }
      }
      const float smax = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
      const uint32_t smu = __reduce_max_sync(0xffffffffu, __float_as_uint(smax));
      const int e_blk = min(156 - kLazy - (int)((smu >> 23) & 0xffu), 100);
      if (!dirty) {
        e_cur = e_blk - kEHead;
      } else if (moved || e_cur > e_blk || nacc >= p.flush_blocks) {
        flush(alpha);
        if (moved) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            bias[r] *= alpha[r];
            if constexpr (V3) {
#pragma unroll
              for (int c = 0; c < LC; ++c) corr[r][c] *= alpha[r];
            }
          }
        }
        e_cur = e_blk - kEHead;
      }
      dirty = true;
      // p of every token to the token-quad lanes
#pragma unroll
      for (int r = 0; r < R; ++r) pb[r * 32 + lane] = pj[r];
      __syncwarp();
      const float pe = pow2i(e_cur);
      const int pos = (tq & 3) * 8 + (tq >> 2) * 4;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float4 p4 = *reinterpret_cast<const float4*>(pb + r * 32 + 4 * tq);
        const float pq[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) bias[r] = fmaf(pq[i], mv[i], bias[r]);
        if (cg_ok) {
          uint32_t uu[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) uu[i] = (uint32_t)__float2int_rn(pq[i] * pe * sv[i]);
          store_digits(reinterpret_cast<uint32_t*>(vbs + cq * 256 + (4 * r) * 32 + pos), 8, uu);
        }
      }
      if constexpr (V3) {
        // Mixed3 narrow slots (stream index % 11 == 10, quant.cpp:36-53) decode with
        // wide_scale(s) = s * 7/3: the IMMA sums code * s, so p (wide_scale(s) - s) code is
        // added on the CUDA cores. Token j (= lane) is narrow at channels d = rho_j + 11 k,
        // rho_j = 10 - tok_j * D (mod 11), tok_j its index in its segment's stream (global
        // (b, kv-head)). Gathered per OUTPUT channel (no shared atomics: they are CAS loops):
        // the lane owning channel d sums over the tokens of residue d % 11 (a ballot mask)
        // into registers that are rescaled with the softmax like the min-term bias.
        const bool vq = jb + lane < p.v.quantized;  // (window blocks: unpacked tokens have no codes)
        const int2 inf = vq ? vinf2[lane] : make_int2(1, 0);  // (ring stage, or global for window blocks)
        const int tok = (int)((((unsigned)p.v.gbh(bh) % 11u) * (unsigned)(inf.x % 11) + (unsigned)(inf.y % 11)) % 11u);
        const int rho = vq ? ((10 - tok * (D % 11)) % 11 + 11) % 11 : 11;
#pragma unroll
        for (int c = 0; c < CGMAX; ++c) {
          if (c < CG) {
            const float sc0 = meta_pair(vm2[(size_t)c * gs + lane]).x;
            const float dsc = wide_scale(sc0) - sc0;
#pragma unroll
            for (int r = 0; r < R; ++r) nw[(r * CGMAX + c) * 32 + lane] = pj[r] * dsc;
          }
        }
        // one code of token j at channel d (tb = vtab[d]) times its weight, into corr[.][c]
        auto narrow_fma = [&](int j, int c, uint32_t tb, const float* wg) {
          const uint32_t code =
              (vt2[(j >> 4) * tile_words(D, VBS) + (tb & 0xffffu) + 4 * ((j & 15) >> 2)] >> ((tb >> 16) + 8 * (j & 3))) & 7u;
#pragma unroll
          for (int r = 0; r < R; ++r) corr[r][c] = fmaf((float)code, wg[r * CGMAX * 32 + j], corr[r][c]);
        };
        const int2 inf0 = make_int2(__shfl_sync(0xffffffffu, inf.x, 0), __shfl_sync(0xffffffffu, inf.y, 0));
        const int rho0 = __shfl_sync(0xffffffffu, rho, 0);
        __syncwarp();
        if (__all_sync(0xffffffffu, vq && inf.x == inf0.x && inf.y == inf0.y + lane)) {
          // the block is one run of consecutive stream tokens (prefill segments): the tokens of
          // residue rho are j = (rho0 - rho) / (D mod 11) + 11 m, no masks, no divergence
          constexpr int kInvD = D % 11 == 7 ? 8 : 5;  // (D mod 11)^-1 mod 11 for D = 128 / 64
#pragma unroll
          for (int c = 0; c < LC; ++c) {
            const int d = lane * LC + c;
            const int j0 = ((rho0 - d % 11 + 11) * kInvD) % 11;
            const uint32_t tb = vtab[d];
            const float* wg = nw + (d / gs) * 32;
            narrow_fma(j0, c, tb, wg);
            narrow_fma(j0 + 11, c, tb, wg);
            if (j0 + 22 < 32) narrow_fma(j0 + 22, c, tb, wg);
          }
        } else {
          // general blocks (segment boundaries, one-token decode segments): per residue class a
          // ballot mask of its tokens, gathered by the owners of the class's channels
          uint32_t mk = 0;
#pragma unroll
          for (int x = 0; x < 11; ++x) {
            const uint32_t bm = __ballot_sync(0xffffffffu, rho == x);
            if (lane == x) mk = bm;
          }
#pragma unroll
          for (int c = 0; c < LC; ++c) {
            const int d = lane * LC + c;
            uint32_t m = __shfl_sync(0xffffffffu, mk, d % 11);
            const uint32_t tb = vtab[d];
            const float* wg = nw + (d / gs) * 32;
            while (m) {
              const int j = __ffs(m) - 1;
              m &= m - 1;
              narrow_fma(j, c, tb, wg);
            }
          }
        }
      }
      __syncwarp();
      {
        uint32_t vw0[VW], vw1[VW];
        lds_tile<D, VBS>(vt2, lane, vw0);
        lds_tile<D, VBS>(vt2 + tile_words(D, VBS), lane, vw1);
        uint32_t vb[CGMAX][2];
        if constexpr (GS != 0) {
#pragma unroll
          for (int c = 0; c < CGMAX; ++c) {
            if (c < D / (GS ? GS : 1)) {
              const uint2 xx = *reinterpret_cast<const uint2*>(vbs + c * 256 + g * 32 + 8 * t);
              vb[c][0] = xx.x;
              vb[c][1] = xx.y;
            }
          }
        }
#pragma unroll
        for (int mt = 0; mt < NM; ++mt) {
          const int q0 = mt, q1 = mt + NM;
          const uint32_t a0 = vw0[q0 / CV] & (VMASK << (VBS * (q0 % CV)));
          const uint32_t a1 = vw0[q1 / CV] & (VMASK << (VBS * (q1 % CV)));
          const uint32_t a2 = vw1[q0 / CV] & (VMASK << (VBS * (q0 % CV)));
          const uint32_t a3 = vw1[q1 / CV] & (VMASK << (VBS * (q1 % CV)));
          if constexpr (GS != 0) {
            const int c = (mt * 16) / (GS ? GS : 1);
            imma_uu(accv[mt], a0, a1, a2, a3, vb[c][0], vb[c][1]);
          } else {
            const int c = (mt * 16) / gs;
            const uint2 xx = *reinterpret_cast<const uint2*>(vbs + c * 256 + g * 32 + 8 * t);
            imma_uu(accv[mt], a0, a1, a2, a3, xx.x, xx.y);
          }
        }
      }
      ++nacc;
      __syncwarp();  // pb / vbs are rewritten by the next block
    };

    const int g_stop = min(hi, p.Gf);
    for (int grp = lo; grp < g_stop; ++grp) {
      mbar_wait_a(full_a + 8 * s, phase);  // (completed already: the K-warp consumed it) -- async-proxy visibility
      const uint8_t* st = ring + (size_t)s * SBX;
      const uint32_t* vt = reinterpret_cast<const uint32_t*>(st + KTB);
      const int2* vinf = reinterpret_cast<const int2*>(st + SB);  // (3-bit Values)
      const uint32_t* vm = reinterpret_cast<const uint32_t*>(st + KTB + VTB);
      for (int blk = 0; blk < NBLK; ++blk)
        value_block(vt + (size_t)(2 * blk) * tile_words(D, VBS), vm + 32 * blk, (int64_t)grp * gs + 32 * blk,
                    vinf + 32 * blk);
      __syncwarp();
      issue_next(s);  // this warp was the stage's last reader: refill it S groups ahead
      if (++s == S) {
        s = 0;
        phase ^= 1u;
      }
    }
    if (p.fused && hi > p.Gf) {
      while (ld_acquire(p.flags + (size_t)pass * p.nbh + bh) == 0u) __nanosleep(32);
    }
    if constexpr (R == 1) {
      const int wb_lo = max(lo, p.Gf) - p.Gf, wb_hi = min(hi, p.Gf + p.nwb) - p.Gf;
      for (int wb = wb_lo; wb < wb_hi; ++wb) {
        const int64_t j0 = p.P + 32 * (int64_t)wb;
        const int gi = (int)(j0 / gs), bi = (int)((j0 - (int64_t)gi * gs) / 32);
        const uint8_t* rec = reinterpret_cast<const uint8_t*>(p.k.tiles) + ((size_t)bh * p.Grec + gi) * SB;
        // the partial group's Value tiles / metas in global memory (tokens past Pw: p = 0;
        // their codes and metas are zero: fields of not-yet-aged tokens are never written)
        value_block(reinterpret_cast<const uint32_t*>(rec + KTB) + (size_t)(2 * bi) * tile_words(D, VBS),
                    reinterpret_cast<const uint32_t*>(rec + KTB + VTB) + 32 * bi, j0, p.v.info + j0);
      }
    }

    // ---- end of the fast region: fold accumulators, gather the softmax state ------------
    if (dirty) {
      float one[R];
#pragma unroll
      for (int r = 0; r < R; ++r) one[r] = 1.0f;
      flush(one);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      bias[r] += __shfl_xor_sync(0xffffffffu, bias[r], 1);
      bias[r] += __shfl_xor_sync(0xffffffffu, bias[r], 2);
      bias[r] += __shfl_xor_sync(0xffffffffu, bias[r], 4);
    }
    float m_all[R], l_all[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float lr = l_lane[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lr += __shfl_xor_sync(0xffffffffu, lr, o);
      m_all[r] = m_run[r];
      l_all[r] = lr;
    }
    __syncwarp();
    float acct[R][LC];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const int d = lane * LC + c;
        const float bsel = __shfl_sync(0xffffffffu, bias[r], 8 * (d / gs));
        acct[r][c] = sacc[r * D + d] + bsel;
        if constexpr (V3) acct[r][c] += corr[r][c];
      }

    // ---- tokens past the fast region: lane-parallel over channels ------------------------
    const int tb0 = p.Gf + p.nwb;
    const int64_t j_lo = p.Pw + (int64_t)max(lo - tb0, 0) * p.tail_unit;
    const int64_t j_hi = hi > tb0 && !p.skip_tail ? min(p.T, p.Pw + (int64_t)(hi - tb0) * p.tail_unit) : j_lo;
    double cs_tail = 0.0;
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
      constexpr int VWPL = D * VBS / 64, VCW = VWPL < 4 ? VWPL : 4;
      int vbase[LC], vsh[LC];
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const int d = d0 + c, dc = d & 15;
        const int q = (d >> 4) + NM * (dc >> 3);
        vbase[c] = plane_addr(4 * (dc & 7), q / CV, VWPL);
        vsh[c] = VBS * (q % CV);
      }
      constexpr int TB = 4;
      for (int64_t j0 = j_lo; j0 < j_hi; j0 += TB) {
        float kx[TB][LC], vx[TB][LC];
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          const int64_t jj = min(j0 + i, j_hi - 1);
          if (jj >= p.k.quantized) {
            if (p.tail16 && LC == 4) {
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
            const int j32 = (int)jj;
            if constexpr (V3) {  // Mixed3 narrow slots: the exact decode (rare: window tokens)
#pragma unroll
              for (int c = 0; c < LC; ++c) vx[i][c] = deq_lane<D, false, 3>(p.v, bh, j32, d0 + c, gs);
            } else {
              const uint32_t* tile = p.v.tiles + tile_index(p.v, bh, j32 >> 4);
              const int ti = (j32 & 15) >> 2, te = j32 & 3;
              const float2 smf = meta_pair(__ldcg(p.v.meta + vmeta_at(p.v, bh, j32, d0 / gs)));
#pragma unroll
              for (int c = 0; c < LC; ++c) {
                const uint32_t w = __ldcg(tile + vbase[c] + ti * VCW);
                const uint32_t code = (w >> (vsh[c] + 8 * te)) & ((1u << VBS) - 1u);
                vx[i][c] = fmaf((float)code, smf.x, smf.y);
              }
            }
          }
        }
        float xs[TB][R];
#pragma unroll
        for (int i = 0; i < TB; ++i)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float a = 0.f;
#pragma unroll
            for (int c = 0; c < LC; ++c) a = fmaf(qt[r][c], kx[i][c], a);
            xs[i][r] = a;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < TB; ++i)
#pragma unroll
            for (int r = 0; r < R; ++r) xs[i][r] += __shfl_xor_sync(0xffffffffu, xs[i][r], o);
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          if (j0 + i >= j_hi) break;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (r < prows) {
              const float scv = xs[i][r] * p.inv;
              if (p.want_cs) cs_tail += (double)scv;
              const float ls = scv * kLog2e;
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
    const size_t slot = pbase + wg + bh;
    if (p.want_cs && lane == 0 && cs_tail != 0.0) atomicAdd(p.part_cs + slot, cs_tail);
    if (lo == 0 && hi == p.U) {
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
      if (p.fused && lane == 0) p.flags[(size_t)pass * p.nbh + bh] = 0u;
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
  }
}

template <int D, int KB, int VB, int R, int GS>
int launch_ws(MmaParams& p, int BH, Workspace& ws, cudaStream_t st) {
  using PL = PairLayout<D, KB, R>;
  auto kern = attend_ws_kernel<D, KB, VB, R, GS>;
  int stages = 2;
  const uint32_t sbx = p.stage_bytes + (VB == 3 ? (uint32_t)p.gs * 8u : 0u);  // ring stage (record + info)
  for (int occ = KVB_WS_MIN_CTAS; occ >= 1; --occ) {
    const long per_pair = (227L * 1024 / occ - 1024) / kWsPairs - (long)PL::bytes(0, 0) - 128;
    const long s_fit = per_pair / (long)sbx;
    if (s_fit >= 2) {
      stages = (int)std::min<long>(4, s_fit);
      break;
    }
  }
  if constexpr (GS != 0) {
    using SG = StageGeo<D, KB, VB, R, GS>;
    using WG = WsGeo<D, KB, VB, R, GS>;
    static_assert(WG::kStages >= 2, "stage geometry");
    if (p.stage_bytes != SG::kStage) throw Error(KVMIX_RUNTIME_ERROR, "attend: record geometry mismatch");
    stages = WG::kStages;
  }
  p.stages = stages;
  const size_t smem = (size_t)kWsPairs * PL::bytes(p.stages, sbx);
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  static thread_local int occ_dev = -1;
  static thread_local size_t occ_smem = 0;
  static thread_local int occ = 0;
  if (occ_smem != smem || occ_dev != dev) {
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
    // all of the unified L1 / shared storage as shared memory: the ring and score buffers of
    // every resident pair (the default carveout would cap the residency below the registers')
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWsPairs * 64, smem), "occupancy");
    occ_smem = smem;
    occ_dev = dev;
  }
  if (occ < 1) throw Error(KVMIX_RUNTIME_ERROR, "attend: warp-specialized kernel does not fit on an SM");
  const int64_t wave = (int64_t)occ * num_sms() * kWsPairs;  // resident pairs
  const int64_t min_cost = knobs().min_cost;
  const int64_t w_cap = std::max<int64_t>(1, p.Nc / min_cost);
  p.W = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(p.N, wave / p.npass), w_cap));
  p.pslots = (int)(wave + BH);
  p.nbh = BH;
  const size_t slots = (size_t)p.npass * p.pslots;
  p.part_ml = ws.ml(st, slots * p.rows);
  p.part_acc = ws.acc(st, slots * p.rows * D);
  p.part_cs = ws.cs(st, slots + 1);
  p.cnt = ws.zeroed<unsigned>((size_t)p.npass * BH);
  p.cnt8 = ws.zeroed<unsigned>(slots);
  p.flags = p.fused ? ws.zeroed<unsigned>((size_t)p.npass * BH) : nullptr;
  if (p.want_cs) check_cuda(cudaMemsetAsync(p.part_cs, 0, (slots + 1) * sizeof(double), st), "memset");
  const int64_t pairs = (int64_t)p.W * p.npass;
  kern<<<(unsigned)((pairs + kWsPairs - 1) / kWsPairs), kWsPairs * 64, smem, st>>>(p);
  return p.W;
}
