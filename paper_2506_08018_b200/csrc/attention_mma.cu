// attention_mma.cu -- fused split-K decode attention on the tensor cores (mma.sync m16n8k16).
//
// Decode is a GEMV per (b, kv-head): scores = K q, out = V^T p. At 2-bit gs32 a K+V element
// pair is 0.75 B of HBM traffic, so a CUDA-core loop (unpack + dequant + FMA per element)
// runs out of issue slots before HBM does. Here the codes go straight
// from registers into tensor-core A fragments: the device tile layout (common.cuh) is
// "fragment-native", so one 128-bit load per lane yields that lane's A operands and each
// fragment register is unpacked with shift/LOP3/HSUB2 into exact fp16 integers. The
// dequantization is factored out of the dot products:
//     q.k_j  = sum_d (q_d s_gd) c_jd + sum_d q_d m_gd          (Keys, per channel group)
//     out_d  = sum_j (p_j s_jg) c_jd + sum_j p_j m_jg          (Values, per token group)
// The B operands (q*s, p*s, p) are split into an fp16 hi part and an fp16 lo remainder in
// two MMA columns, so products carry ~22 mantissa bits and accumulate in fp32. The Value
// min term is a second small MMA with A = the binary16 mins (exact in fp16).
//
// CTA = 4 warps over one (b, kv-head) and a chunk of Key groups; warps own whole groups
// (interleaved). Per 16-token tile a warp: K MMA (D/16 k-steps) -> scores -> online
// softmax (log2 domain) -> builds the P.V B fragments in shared memory -> V MMA (D/16
// m-tiles). Tokens past the last fully packed group (the ragged tail and the
// full-precision window) use a per-token CUDA-core loop updating the same state. Partials
// (m, l, acc) go to the split-K combine kernel shared with the generic path.
#include <algorithm>
#include <cmath>

#include "attention.cuh"

namespace kvb {

namespace {

constexpr int kMmaWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t h2_sub_magic(uint32_t x) {
  // (1024 + c_lo, 1024 + c_hi) - 1024 -> exact (c_lo, c_hi)
  __half2 v = *reinterpret_cast<__half2*>(&x);
  const __half2 m = __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400));
  v = __hsub2(v, m);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Unpack fragment register r at slot s from a lane's words of a b-bit plane.
template <int B, int NS>
__device__ __forceinline__ uint32_t frag(const uint32_t* w, int r, int s) {
  constexpr int SPH = 16 / B;
  constexpr uint32_t MASK = B == 2 ? 0x00030003u : B == 4 ? 0x000F000Fu : 0x00010001u;
  const int vs = r * NS + s;
  const uint32_t x = ((w[vs / SPH] >> (B * (vs % SPH))) & MASK) | 0x64006400u;
  return h2_sub_magic(x);
}

template <int WPL>
__device__ __forceinline__ void load_plane(const uint32_t* __restrict__ tile, int lane, uint32_t (&w)[WPL]) {
  if constexpr (WPL >= 4) {
#pragma unroll
    for (int c = 0; c < WPL / 4; ++c) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(tile + c * 128 + lane * 4));
      w[4 * c] = v.x;
      w[4 * c + 1] = v.y;
      w[4 * c + 2] = v.z;
      w[4 * c + 3] = v.w;
    }
  } else if constexpr (WPL == 2) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(tile + lane * 2));
    w[0] = v.x;
    w[1] = v.y;
  } else {
    w[0] = __ldg(tile + lane);
  }
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

struct MmaParams {
  SideView k, v;
  const void* q;
  int H, Hq, tq, rows, gs, cg;
  int64_t T, P;          // total tokens; fast-path limit (multiple of gs)
  int64_t groups_total;  // ceil(T / gs)
  int chunk_groups;
  float inv;             // 1/sqrt(D)
  float2* part_ml;
  float* part_acc;
  double* part_cs;
};

// Per-warp shared memory (halves unless noted).
template <int D>
struct WarpSmem {
  static constexpr int KST = D + 8;  // padded row stride: conflict-free B fragment reads
  static constexpr int VST = 24;     // padded token stride (16 tokens)
  __half bk[8][KST];                 // K B operand: [column][channel]
  __half bv[8][8][VST];              // V B operand: [channel group][column][token]
  __half bp[8][VST];                 // P (bias MMA) B operand: [column][token]
  uint32_t vm[16][8];                // staged Value meta of the tile: [token][channel group]
};

template <int D, int KB, int VB, int R, typename TT, typename TQ>
__global__ void __launch_bounds__(kMmaWarps * 32, 3) attend_mma_kernel(MmaParams p) {
  constexpr int NS = D / 16;        // k-steps (Keys) / m-tiles (Values)
  constexpr int KW = D * KB / 64;   // words per lane, Key tile
  constexpr int VW = D * VB / 64;   // words per lane, Value tile
  constexpr int LC = D / 32;        // channels per lane for meta / q
  __shared__ WarpSmem<D> wsm[kMmaWarps];
  __shared__ float s_m[kMmaWarps][R], s_l[kMmaWarps][R];
  __shared__ float s_acc[kMmaWarps][R][D];
  __shared__ float s_bias[kMmaWarps][R][8];
  __shared__ double s_cs[kMmaWarps];

  const int split = blockIdx.x, bh = blockIdx.y, nsplit = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int b = bh / p.H, h = bh % p.H, G = p.Hq / p.H;
  const int gs = p.gs, CG = p.cg;
  WarpSmem<D>& sm = wsm[warp];

  // zero this warp's B operand staging (unused columns must stay 0)
  {
    uint32_t* z = reinterpret_cast<uint32_t*>(&sm);
    for (int i = lane; i < (int)(sizeof(WarpSmem<D>) / 4); i += 32) z[i] = 0u;
  }
  // query rows: lane owns channels [lane*LC, lane*LC+LC)
  float qv[R][LC];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int rr = r < p.rows ? r : 0;
    const int gi = rr / p.tq, qi = rr % p.tq;
    const TQ* qp = static_cast<const TQ*>(p.q) + (((size_t)b * p.Hq + h * G + gi) * p.tq + qi) * D + lane * LC;
#pragma unroll
    for (int c = 0; c < LC; ++c) qv[r][c] = r < p.rows ? ld_f<TQ>(qp + c) : 0.f;
  }
  __syncwarp();

  float m_run = -INFINITY, l_run = 0.f;  // row t (threads with t < rows)
  float accv[NS][4];
#pragma unroll
  for (int i = 0; i < NS; ++i) accv[i][0] = accv[i][1] = accv[i][2] = accv[i][3] = 0.f;
  float accb[4] = {0.f, 0.f, 0.f, 0.f};
  double cs = 0.0;
  const bool row_ok = t < p.rows;

  const int64_t g_beg = (int64_t)split * p.chunk_groups;
  const int64_t g_end = min(g_beg + p.chunk_groups, p.groups_total);
  const int64_t g_fast_end = min(g_end, p.P / gs);
  const size_t ktile_base = (size_t)bh * p.k.tiles_per_bh * p.k.tile_words;
  const size_t vtile_base = (size_t)bh * p.v.tiles_per_bh * p.v.tile_words;
  const uint32_t* kmeta_bh = p.k.meta + (size_t)bh * p.k.meta_per_bh;
  const uint32_t* vmeta_bh = p.v.meta + (size_t)bh * p.v.meta_per_bh;

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

  for (int64_t grp = g_beg + warp; grp < g_fast_end; grp += kMmaWarps) {
    // ---- Key group: B operand (q*s split hi/lo, pre-scaled by 2^e per row) and beta ----
    float beta[R], inv_sig[R];
    {
      uint32_t km[LC];
      const uint32_t* mp = kmeta_bh + (size_t)grp * D + lane * LC;
      if constexpr (LC == 4) {
        const uint4 v4 = __ldg(reinterpret_cast<const uint4*>(mp));
        km[0] = v4.x; km[1] = v4.y; km[2] = v4.z; km[3] = v4.w;
      } else {
#pragma unroll
        for (int c = 0; c < LC; ++c) km[c] = __ldg(mp + c);
      }
      float sc[LC], mn[LC];
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        sc[c] = meta_scale(km[c]);
        mn[c] = meta_min(km[c]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float qs[LC], mx = 0.f, bt = 0.f;
#pragma unroll
        for (int c = 0; c < LC; ++c) {
          qs[c] = qv[r][c] * sc[c];
          mx = fmaxf(mx, fabsf(qs[c]));
          bt = fmaf(qv[r][c], mn[c], bt);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          bt += __shfl_xor_sync(0xffffffffu, bt, o);
        }
        // sigma = 2^(14 - floor(log2 max|qs|)): max|qs*sigma| in [2^14, 2^15)
        const int e = (__float_as_int(mx) >> 23) & 0xff;
        const int se = min(max(268 - e, 1), 254);
        const float sig = __int_as_float(se << 23);
        inv_sig[r] = __int_as_float((254 - se) << 23);
        beta[r] = bt;
#pragma unroll
        for (int c = 0; c < LC; ++c) {
          const float x = qs[c] * sig;
          const __half hi = __float2half_rn(x);
          const __half lo = __float2half_rn(x - __half2float(hi));
          sm.bk[2 * r][lane * LC + c] = hi;
          sm.bk[2 * r + 1][lane * LC + c] = lo;
        }
      }
    }
    __syncwarp();
    uint32_t bk0[NS], bk1[NS];
#pragma unroll
    for (int kk = 0; kk < NS; ++kk) {
      bk0[kk] = *reinterpret_cast<const uint32_t*>(&sm.bk[g][16 * kk + 2 * t]);
      bk1[kk] = *reinterpret_cast<const uint32_t*>(&sm.bk[g][16 * kk + 2 * t + 8]);
    }
    float my_beta = beta[0], my_isig = inv_sig[0];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      if (t == r) {
        my_beta = beta[r];
        my_isig = inv_sig[r];
      }
    }

    for (int tt = 0; tt < gs / 16; ++tt) {
      const int64_t tile = grp * (gs / 16) + tt;
      uint32_t kw[KW], vw[VW];
      load_plane<KW>(p.k.tiles + ktile_base + (size_t)tile * p.k.tile_words, lane, kw);
      load_plane<VW>(p.v.tiles + vtile_base + (size_t)tile * p.v.tile_words, lane, vw);
      // stage the tile's Value meta [16 tokens][CG]
      for (int i = lane; i < 16 * CG; i += 32) sm.vm[i / CG][i % CG] = __ldg(vmeta_bh + (size_t)tile * 16 * CG + i);

      // ---- scores: K (16 tokens x D) . B ----
      float dk[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < NS; ++kk) {
        mma16816(dk, frag<KB, NS>(kw, 0, kk), frag<KB, NS>(kw, 1, kk), frag<KB, NS>(kw, 2, kk),
                 frag<KB, NS>(kw, 3, kk), bk0[kk], bk1[kk]);
      }
      // row t: token g -> dk[0] + dk[1]; token g+8 -> dk[2] + dk[3]
      const float sa = ((dk[0] + dk[1]) * my_isig + my_beta) * p.inv;
      const float sb = ((dk[2] + dk[3]) * my_isig + my_beta) * p.inv;
      if (row_ok) cs += (double)(sa + sb);
      const float la = sa * kLog2e, lb = sb * kLog2e;
      float tmax = fmaxf(la, lb);
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
      const float m_new = fmaxf(m_run, tmax);
      const float alpha = exp2f(m_run - m_new);
      const float pa = row_ok ? exp2f(la - m_new) : 0.f;
      const float pb = row_ok ? exp2f(lb - m_new) : 0.f;
      l_run = l_run * alpha + pa + pb;
      m_run = m_new;
      rescale(alpha);

      // ---- P.V B operands: lane -> token j = lane % 16 ----
      __syncwarp();
      {
        const int j = lane & 15, hh = lane >> 4;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int src = (j & 7) * 4 + r;
          const float xa = __shfl_sync(0xffffffffu, pa, src);
          const float xb = __shfl_sync(0xffffffffu, pb, src);
          const float pj = j < 8 ? xa : xb;
          if (r < p.rows) {
            if (hh == 0) {
              const __half hi = __float2half_rn(pj);
              sm.bp[2 * r][j] = hi;
              sm.bp[2 * r + 1][j] = __float2half_rn(pj - __half2float(hi));
            }
            for (int c = hh; c < CG; c += 2) {
              const float x = pj * meta_scale(sm.vm[j][c]);
              const __half hi = __float2half_rn(x);
              sm.bv[c][2 * r][j] = hi;
              sm.bv[c][2 * r + 1][j] = __float2half_rn(x - __half2float(hi));
            }
          }
        }
      }
      __syncwarp();
      // bias MMA: A = Value mins [group][token] (rows >= CG are zero), B = p
      {
        uint32_t a0 = 0u, a2 = 0u;
        if (g < CG) {
          a0 = __byte_perm(sm.vm[2 * t][g], sm.vm[2 * t + 1][g], 0x7632);
          a2 = __byte_perm(sm.vm[2 * t + 8][g], sm.vm[2 * t + 9][g], 0x7632);
        }
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&sm.bp[g][2 * t]);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&sm.bp[g][2 * t + 8]);
        mma16816(accb, a0, 0u, a2, 0u, b0, b1);
      }
#pragma unroll
      for (int mt = 0; mt < NS; ++mt) {
        const int c = (mt * 16) / gs;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&sm.bv[c][g][2 * t]);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&sm.bv[c][g][2 * t + 8]);
        mma16816(accv[mt], frag<VB, NS>(vw, 0, mt), frag<VB, NS>(vw, 1, mt), frag<VB, NS>(vw, 2, mt),
                 frag<VB, NS>(vw, 3, mt), b0, b1);
      }
      __syncwarp();
    }
  }

  // ---- tokens past the fast region: per-token CUDA-core path --------------------------
  {
    const int64_t j_lo = max(g_beg * gs, p.P), j_hi = min(g_end * (int64_t)gs, p.T);
    for (int64_t j = j_lo + warp; j < j_hi; j += kMmaWarps) {
      float part[R];
#pragma unroll
      for (int r = 0; r < R; ++r) part[r] = 0.f;
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const int d = lane * LC + c;
        const float kx = j < p.k.quantized ? packed_value(true, p.k, bh, j, d, D, gs)
                                           : tail_at<TT>(p.k, bh, j - p.k.quantized, d, D);
#pragma unroll
        for (int r = 0; r < R; ++r) part[r] = fmaf(qv[r][c], kx, part[r]);
      }
      float s_mine = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float x = part[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (r == t) s_mine = x * p.inv;
      }
      if (row_ok && g == 0) cs += (double)s_mine;
      const float ls = s_mine * kLog2e;
      const float m_new = row_ok ? fmaxf(m_run, ls) : m_run;
      const float alpha = row_ok ? exp2f(m_run - m_new) : 1.f;
      const float pj = row_ok ? exp2f(ls - m_new) : 0.f;
      l_run = l_run * alpha + (g == 0 ? pj : 0.f);
      m_run = m_new;
      rescale(alpha);
#pragma unroll
      for (int mt = 0; mt < NS; ++mt) {
        const int d0 = mt * 16 + g, d1 = d0 + 8;
        const float v0 = j < p.v.quantized ? packed_value(false, p.v, bh, j, d0, D, gs)
                                           : tail_at<TT>(p.v, bh, j - p.v.quantized, d0, D);
        const float v1 = j < p.v.quantized ? packed_value(false, p.v, bh, j, d1, D, gs)
                                           : tail_at<TT>(p.v, bh, j - p.v.quantized, d1, D);
        accv[mt][0] = fmaf(pj, v0, accv[mt][0]);
        accv[mt][2] = fmaf(pj, v1, accv[mt][2]);
      }
    }
  }

  // ---- warp epilogue -> shared ----------------------------------------------------------
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 4);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 8);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
  if (row_ok && t < R) {
    if (g == 0) {
      s_m[warp][t] = m_run;
      s_l[warp][t] = l_run;
    }
#pragma unroll
    for (int mt = 0; mt < NS; ++mt) {
      s_acc[warp][t][mt * 16 + g] = accv[mt][0] + accv[mt][1];
      s_acc[warp][t][mt * 16 + g + 8] = accv[mt][2] + accv[mt][3];
    }
    if (g < 8) s_bias[warp][t][g] = accb[0] + accb[1];
  }
  // checksum: reduce the warp's doubles
  for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
  if (lane == 0) s_cs[warp] = cs;
  __syncthreads();

  // ---- CTA merge (fixed warp order) and split partial -----------------------------------
  for (int e = threadIdx.x; e < p.rows * D; e += blockDim.x) {
    const int r = e / D, d = e % D;
    const int c = d / gs;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kMmaWarps; ++w) M = fmaxf(M, s_m[w][r]);
    float a = 0.f, L = 0.f;
#pragma unroll
    for (int w = 0; w < kMmaWarps; ++w) {
      const float mw = s_m[w][r];
      if (mw != -INFINITY) {
        const float f = exp2f(mw - M);
        a += (s_acc[w][r][d] + s_bias[w][r][c]) * f;
        L += s_l[w][r] * f;
      }
    }
    const size_t pi = ((size_t)bh * nsplit + split) * p.rows + r;
    p.part_acc[pi * D + d] = a;
    if (d == 0) p.part_ml[pi] = make_float2(M == -INFINITY ? -INFINITY : M * kLn2, L);
  }
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < kMmaWarps; ++w) tot += s_cs[w];
    p.part_cs[(size_t)bh * nsplit + split] = tot;
  }
}

template <int D, int KB, int VB, int R, typename TT, typename TQ>
void launch(const MmaParams& p, int nsplit, int BH, cudaStream_t st) {
  attend_mma_kernel<D, KB, VB, R, TT, TQ><<<dim3(nsplit, BH), kMmaWarps * 32, 0, st>>>(p);
}

template <int D, int KB, int VB, int R>
bool dispatch_types(const MmaParams& p, int nsplit, int BH, bool tail16, bool q16, cudaStream_t st) {
  if (tail16) {
    if (q16) launch<D, KB, VB, R, __half, __half>(p, nsplit, BH, st);
    else launch<D, KB, VB, R, __half, float>(p, nsplit, BH, st);
  } else {
    if (q16) launch<D, KB, VB, R, float, __half>(p, nsplit, BH, st);
    else launch<D, KB, VB, R, float, float>(p, nsplit, BH, st);
  }
  return true;
}

template <int D, int R>
bool dispatch_bits(const MmaParams& p, int kb, int vb, int nsplit, int BH, bool tail16, bool q16, cudaStream_t st) {
  if (kb == 2 && vb == 2) return dispatch_types<D, 2, 2, R>(p, nsplit, BH, tail16, q16, st);
  if (kb == 2 && vb == 4) return dispatch_types<D, 2, 4, R>(p, nsplit, BH, tail16, q16, st);
  if (kb == 4 && vb == 2) return dispatch_types<D, 4, 2, R>(p, nsplit, BH, tail16, q16, st);
  if (kb == 4 && vb == 4) return dispatch_types<D, 4, 4, R>(p, nsplit, BH, tail16, q16, st);
  return false;
}

}  // namespace

int mma_splits(int BH, int64_t groups_total) {
  // ~8 waves of (148 SMs x 3 CTAs), at least one Key group per warp; the cap depends on
  // (B, H) only so the scratch size never depends on the token count.
  const int cap = std::max(1, std::min(512, (8 * 3 * num_sms() + BH - 1) / std::max(1, BH)));
  const int64_t by_len = std::max<int64_t>(1, (groups_total + kMmaWarps - 1) / kMmaWarps);
  return (int)std::min<int64_t>(cap, by_len);
}

bool attend_mma(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
                Workspace& ws, cudaStream_t st) {
  const int rows = (Hq / c->H) * tq;
  if (rows > 4) return false;
  const int kb = c->k.bits, vb = c->v.bits;
  if (kb == 3 || vb == 3) return false;
  const int D = c->D, gs = c->cfg.group_size;
  const int BH = c->B * c->H;
  const int64_t T = c->total();
  MmaParams p{};
  p.k = view(c->k);
  p.v = view(c->v);
  p.q = q;
  p.H = c->H;
  p.Hq = Hq;
  p.tq = tq;
  p.rows = rows;
  p.gs = gs;
  p.cg = c->cgroups();
  if (p.cg > 8) return false;
  p.T = T;
  p.P = (std::min(c->k.quantized, c->v.quantized) / gs) * gs;
  p.groups_total = (T + gs - 1) / gs;
  const int nsplit = mma_splits(BH, p.groups_total);
  p.chunk_groups = (int)((p.groups_total + nsplit - 1) / nsplit);
  p.inv = 1.0f / sqrtf((float)D);
  const int cap_splits = mma_splits(BH, (int64_t)1 << 40);
  p.part_ml = ws.ml(st, (size_t)BH * cap_splits * rows);
  p.part_acc = ws.acc(st, (size_t)BH * cap_splits * rows * D);
  p.part_cs = ws.cs(st, (size_t)BH * cap_splits + 1);
  const bool tail16 = c->tail_dtype == KVMIX_F16, q16 = dt == KVMIX_F16;
  const int R = rows <= 1 ? 1 : rows <= 2 ? 2 : 4;
  bool ok = false;
#define KVB_DISPATCH_D(DD)                                                                     \
  if (D == DD) {                                                                               \
    if (R == 1) ok = dispatch_bits<DD, 1>(p, kb, vb, nsplit, BH, tail16, q16, st);             \
    else if (R == 2) ok = dispatch_bits<DD, 2>(p, kb, vb, nsplit, BH, tail16, q16, st);        \
    else ok = dispatch_bits<DD, 4>(p, kb, vb, nsplit, BH, tail16, q16, st);                    \
  }
  KVB_DISPATCH_D(64)
  KVB_DISPATCH_D(128)
#undef KVB_DISPATCH_D
  if (!ok) return false;
  after_launch("attend_mma_kernel");
  attend_combine_kernel<<<dim3(BH, rows), 128, 0, st>>>(p.part_ml, p.part_acc, nsplit, rows, c->H, Hq, tq, D, out);
  after_launch("attend_combine_kernel");
  if (checksum) {
    checksum_kernel<<<1, 32, 0, st>>>(p.part_cs, (size_t)BH * nsplit, p.part_cs + (size_t)BH * cap_splits);
    after_launch("checksum_kernel");
    check_cuda(cudaMemcpyAsync(checksum, p.part_cs + (size_t)BH * cap_splits, 8, cudaMemcpyDeviceToHost, st), "memcpy");
    check_cuda(cudaStreamSynchronize(st), "sync");
  }
  return true;
}

}  // namespace kvb
