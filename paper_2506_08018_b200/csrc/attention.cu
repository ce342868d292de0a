// attention.cu -- decode attention over the packed cache: generic split-K kernel,
// fused_qk_scores / softmax_rows / fused_pv (attention.cpp:28-159) and the
// dequantize-everything reference_attend (attention.cpp:168-211).
//
// This file holds the GENERIC CUDA-core path: one warp per token, lanes over channels,
// dequantization inside the dot products (no K/V materialization), online softmax per
// query row, split-K over the token axis with a deterministic combine kernel. It handles
// every shape the device cache accepts (any G = Hq/H, any number of query rows, all bit
// widths, any head_dim up to 256, tokens in the full-precision tail). The tensor-core paths
// (attention_mma.cu, attention_ws.cu, attention_tc.cu) serve D in {64, 128}; this kernel the rest.
#include <algorithm>
#include <cmath>

#include "attention.cuh"

namespace kvb {

namespace {

template <typename TT>
struct PackedKV {
  SideView k, v;
  int D, gs;
  __device__ float key(int bh, int64_t j, int d) const {
    return j < k.quantized ? packed_value(true, k, bh, j, d, D, gs) : tail_at<TT>(k, bh, j - k.quantized, d, D);
  }
  __device__ float val(int bh, int64_t j, int d) const {
    return j < v.quantized ? packed_value(false, v, bh, j, d, D, gs) : tail_at<TT>(v, bh, j - v.quantized, d, D);
  }
};

struct DenseKV {
  const float* keys;
  const float* values;
  int64_t T;
  int D;
  __device__ float key(int bh, int64_t j, int d) const { return keys[((size_t)bh * T + j) * D + d]; }
  __device__ float val(int bh, int64_t j, int d) const { return values[((size_t)bh * T + j) * D + d]; }
};

constexpr int kWarps = 4;
constexpr int kMaxLaneCh = 8;  // D <= 256

__device__ inline float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// One CTA = one (token chunk, b, kv-head); rows = G * tq query rows share the K/V reads.
// Writes the un-normalized partial (m, l, acc[D]) per (split, bh, row) and a double
// checksum partial per (split, bh).
template <typename KV, typename TQ>
__global__ void __launch_bounds__(kWarps * 32) attend_generic_kernel(KV kv, const TQ* __restrict__ q, int H, int Hq,
                                                                     int tq, int D, int64_t T, int64_t chunk,
                                                                     int R, float2* __restrict__ part_ml,
                                                                     float* __restrict__ part_acc,
                                                                     double* __restrict__ part_cs, float inv) {
  extern __shared__ float smem[];
  const int split = blockIdx.x, bh = blockIdx.y;
  const int nsplit = gridDim.x;
  const int b = bh / H, h = bh % H;
  const int G = Hq / H;
  float* qs = smem;                       // [R][D]
  float* wm = qs + R * D;                 // [kWarps][R]
  float* wl = wm + kWarps * R;            // [kWarps][R]
  float* wacc = wl + kWarps * R;          // [kWarps][R][D]
  double* wcs = reinterpret_cast<double*>(wacc + kWarps * R * D);  // [kWarps]
  for (int e = threadIdx.x; e < R * D; e += blockDim.x) {
    const int r = e / D, d = e % D;
    const int gi = r / tq, qi = r % tq;
    const int hq = h * G + gi;
    qs[e] = ld_f<TQ>(q + (((size_t)b * Hq + hq) * tq + qi) * D + d);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (D + 31) / 32;  // channels d = lane + 32 c < D per lane (any head_dim <= 256)
  const int64_t j0 = (int64_t)split * chunk, j1 = min(T, j0 + chunk);
  double cs = 0.0;
  for (int r = 0; r < R; ++r) {
    float m = -INFINITY, l = 0.f;
    float acc[kMaxLaneCh];
#pragma unroll
    for (int c = 0; c < kMaxLaneCh; ++c) acc[c] = 0.f;
    for (int64_t j = j0 + warp; j < j1; j += kWarps) {
      float part = 0.f;
      for (int c = 0; c < nch; ++c) {
        const int d = lane + 32 * c;
        if (d < D) part = fmaf(qs[r * D + d], kv.key(bh, j, d), part);
      }
      const float s = warp_sum(part) * inv;
      cs += (double)s;
      const float mn = fmaxf(m, s);
      const float alpha = expf(m - mn);  // exp(-inf) = 0 on the first token
      const float p = expf(s - mn);
      l = l * alpha + p;
#pragma unroll
      for (int c = 0; c < kMaxLaneCh; ++c) {
        if (c < nch && lane + 32 * c < D) acc[c] = acc[c] * alpha + p * kv.val(bh, j, lane + 32 * c);
      }
      m = mn;
    }
    if (lane == 0) {
      wm[warp * R + r] = m;
      wl[warp * R + r] = l;
    }
    for (int c = 0; c < nch; ++c)
      if (lane + 32 * c < D) wacc[(warp * R + r) * D + lane + 32 * c] = acc[c];
  }
  if (lane == 0) wcs[warp] = cs;  // lane 0 saw every score of its warp
  __syncthreads();
  // merge warps (fixed order), write partials
  for (int e = threadIdx.x; e < R * D; e += blockDim.x) {
    const int r = e / D, d = e % D;
    float M = -INFINITY;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, wm[w * R + r]);
    float a = 0.f;
    for (int w = 0; w < kWarps; ++w) {
      const float mw = wm[w * R + r];
      if (mw != -INFINITY) a += wacc[(w * R + r) * D + d] * expf(mw - M);
    }
    part_acc[(((size_t)bh * nsplit + split) * R + r) * D + d] = a;
    if (d == 0) {
      float L = 0.f;
      for (int w = 0; w < kWarps; ++w) {
        const float mw = wm[w * R + r];
        if (mw != -INFINITY) L += wl[w * R + r] * expf(mw - M);
      }
      part_ml[((size_t)bh * nsplit + split) * R + r] = make_float2(M, L);
    }
  }
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += wcs[w];
    part_cs[(size_t)bh * nsplit + split] = t;
  }
}

}  // namespace

// Combine split partials into out [B, Hq, tq, D] (fixed split order: deterministic).
__global__ void attend_combine_kernel(const float2* __restrict__ part_ml, const float* __restrict__ part_acc, int nsplit,
                                      int R, int H, int Hq, int tq, int D, float* __restrict__ out) {
  const int bh = blockIdx.x, r = blockIdx.y;
  const int b = bh / H, h = bh % H, G = Hq / H;
  const int gi = r / tq, qi = r % tq;
  const int hq = h * G + gi;
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, part_ml[((size_t)bh * nsplit + s) * R + r].x);
  float L = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float2 ml = part_ml[((size_t)bh * nsplit + s) * R + r];
    if (ml.x != -INFINITY) L += ml.y * expf(ml.x - M);
  }
  const float invL = 1.0f / L;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < nsplit; ++s) {
      const float2 ml = part_ml[((size_t)bh * nsplit + s) * R + r];
      if (ml.x != -INFINITY) a += part_acc[(((size_t)bh * nsplit + s) * R + r) * D + d] * expf(ml.x - M);
    }
    out[(((size_t)b * Hq + hq) * tq + qi) * D + d] = a * invL;
  }
}

__global__ void checksum_kernel(const double* __restrict__ part, size_t n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

namespace {

// scores[b][h][qi][j] = (q . k_j) * inv, reference order of operations per element.
template <typename KV, typename TQ>
__global__ void qk_scores_kernel(KV kv, const TQ* __restrict__ q, int H, int tq, int D, int64_t T, float inv,
                                 float* __restrict__ scores) {
  const int bh = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= T) return;
  for (int qi = 0; qi < tq; ++qi) {
    float part = 0.f;
    for (int d = lane; d < D; d += 32) part = fmaf(ld_f<TQ>(q + ((size_t)bh * tq + qi) * D + d), kv.key(bh, j, d), part);
    const float s = warp_sum(part) * inv;
    if (lane == 0) scores[((size_t)bh * tq + qi) * T + j] = s;
  }
}

__global__ void softmax_rows_kernel(float* __restrict__ x, int64_t cols) {
  float* row = x + (size_t)blockIdx.x * cols;
  __shared__ float red[32];
  float m = -INFINITY;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) m = fmaxf(m, row[j]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  float s = 0.f;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    const float e = expf(row[j] - m);
    row[j] = e;
    s += e;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    s = warp_sum(s);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  const float is = 1.0f / red[0];
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) row[j] *= is;
}

// out[b][h][qi][d] = sum_j p_j * v_j[d]; one CTA per (bh, qi), threads over d, token loop.
template <typename KV>
__global__ void pv_kernel(KV kv, const float* __restrict__ probs, int tq, int D, int64_t T, float* __restrict__ out) {
  const int bh = blockIdx.x, qi = blockIdx.y;
  const float* p = probs + ((size_t)bh * tq + qi) * T;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float a = 0.f;
    for (int64_t j = 0; j < T; ++j) a = fmaf(p[j], kv.val(bh, j, d), a);
    out[((size_t)bh * tq + qi) * D + d] = a;
  }
}


template <typename KV, typename TQ>
void run_generic(const KV& kv, const TQ* q, int B, int H, int Hq, int tq, int D, int64_t T, float* out,
                 Workspace& ws, double* checksum, cudaStream_t st) {
  const int BH = B * H;
  const int R = (Hq / H) * tq;
  const int nsplit = attend_splits(BH);
  const int64_t chunk = (T + nsplit - 1) / nsplit;
  float2* ml = ws.ml(st, (size_t)BH * nsplit * R);
  float* acc = ws.acc(st, (size_t)BH * nsplit * R * D);
  double* cs = ws.cs(st, (size_t)BH * nsplit + 1);
  const size_t smem = (size_t)R * D * 4 + 2 * kWarps * R * 4 + (size_t)kWarps * R * D * 4 + kWarps * 8 + 8;
  if (smem > 227 * 1024) invalid("attention: too many query rows per KV head for one CTA");
  auto kern = attend_generic_kernel<KV, TQ>;
  check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  const float inv = 1.0f / sqrtf((float)D);
  kern<<<dim3(nsplit, BH), kWarps * 32, smem, st>>>(kv, q, H, Hq, tq, D, T, chunk, R, ml, acc, cs, inv);
  after_launch("attend_generic_kernel");
  attend_combine_kernel<<<dim3(BH, R), 128, 0, st>>>(ml, acc, nsplit, R, H, Hq, tq, D, out);
  after_launch("attend_combine_kernel");
  if (checksum) {
    checksum_kernel<<<1, 32, 0, st>>>(cs, (size_t)BH * nsplit, cs + (size_t)BH * nsplit);
    after_launch("checksum_kernel");
    check_cuda(cudaMemcpyAsync(checksum, cs + (size_t)BH * nsplit, 8, cudaMemcpyDeviceToHost, st), "memcpy");
    check_cuda(cudaStreamSynchronize(st), "sync");
  }
}

}  // namespace

int attend_splits(int BH) {
  // ~4 CTAs per SM over the (b, kv-head) x split grid; independent of the token count
  const int sms = num_sms();
  return std::max(1, std::min(64, (4 * sms + BH - 1) / std::max(1, BH)));
}

void check_query_shape(const kvmix_cache* c, int q_heads, int t) {
  if (t < 1) invalid("attention: need at least one query row");
  if (q_heads < c->H || q_heads % c->H != 0) invalid("attention: query shape does not match cache");
}

void check_attend(const kvmix_cache* c, int q_heads, int t) {
  check_query_shape(c, q_heads, t);
  if (c->total() < 1) invalid("softmax over an empty row");
}

void attend_generic(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out,
                    double* checksum, Workspace& ws, cudaStream_t st) {
  check_attend(c, Hq, tq);
  const int64_t T = c->total();
  auto go = [&](auto tag) {
    using TT = decltype(tag);
    PackedKV<TT> kv{view(c->k), view(c->v), c->D, c->cfg.group_size};
    if (dt == KVMIX_F16) run_generic(kv, static_cast<const __half*>(q), c->B, c->H, Hq, tq, c->D, T, out, ws, checksum, st);
    else run_generic(kv, static_cast<const float*>(q), c->B, c->H, Hq, tq, c->D, T, out, ws, checksum, st);
  };
  if (c->tail_dtype == KVMIX_F16) go(__half{});
  else go(float{});
}

void fused_qk_scores(const kvmix_cache* c, const void* q, kvmix_dtype dt, int tq, float* scores, cudaStream_t st) {
  check_attend(c, c->H, tq);
  const int64_t T = c->total();
  const float inv = 1.0f / sqrtf((float)c->D);
  dim3 grid((unsigned)((T + 3) / 4), c->B * c->H);
  auto go = [&](auto tag) {
    using TT = decltype(tag);
    PackedKV<TT> kv{view(c->k), view(c->v), c->D, c->cfg.group_size};
    if (dt == KVMIX_F16) qk_scores_kernel<<<grid, 128, 0, st>>>(kv, static_cast<const __half*>(q), c->H, tq, c->D, T, inv, scores);
    else qk_scores_kernel<<<grid, 128, 0, st>>>(kv, static_cast<const float*>(q), c->H, tq, c->D, T, inv, scores);
  };
  if (c->tail_dtype == KVMIX_F16) go(__half{});
  else go(float{});
  after_launch("qk_scores_kernel");
}

void softmax_rows(float* x, int64_t rows, int64_t cols, cudaStream_t st) {
  if (cols < 1) invalid("softmax over an empty row");
  if (rows < 1) return;
  softmax_rows_kernel<<<(unsigned)rows, 256, 0, st>>>(x, cols);
  after_launch("softmax_rows_kernel");
}

void fused_pv(const kvmix_cache* c, const float* probs, int tq, float* out, cudaStream_t st) {
  if (tq < 1) invalid("fused_pv: need at least one row");
  const int64_t T = c->total();
  auto go = [&](auto tag) {
    using TT = decltype(tag);
    PackedKV<TT> kv{view(c->k), view(c->v), c->D, c->cfg.group_size};
    pv_kernel<<<dim3(c->B * c->H, tq), 128, 0, st>>>(kv, probs, tq, c->D, T, out);
  };
  if (c->tail_dtype == KVMIX_F16) go(__half{});
  else go(float{});
  after_launch("pv_kernel");
}

void reference_attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int tq, float* scratch, float* out,
                      double* checksum, Workspace& ws, cudaStream_t st) {
  check_attend(c, c->H, tq);
  const int64_t T = c->total();
  float* keys = scratch;
  float* values = scratch + (size_t)c->B * c->H * T * c->D;
  cache_snapshot(c, keys, values, st);
  DenseKV kv{keys, values, T, c->D};
  if (dt == KVMIX_F16) run_generic(kv, static_cast<const __half*>(q), c->B, c->H, c->H, tq, c->D, T, out, ws, checksum, st);
  else run_generic(kv, static_cast<const float*>(q), c->B, c->H, c->H, tq, c->D, T, out, ws, checksum, st);
}

}  // namespace kvb

namespace kvb {
// Dispatcher: the tensor-core kernel (attention_mma.cu) when it supports the shape, the
// generic kernel otherwise.
bool attend_mma(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
                Workspace& ws, cudaStream_t st, const DecodeAppend* da);
void launch_decode_append(const DecodeAppend& da, cudaStream_t st);
void attend(const kvmix_cache* c, const void* q, kvmix_dtype dt, int Hq, int tq, float* out, double* checksum,
            Workspace& ws, cudaStream_t st) {
  check_attend(c, Hq, tq);
  if (attend_mma(c, q, dt, Hq, tq, out, checksum, ws, st, nullptr)) return;
  attend_generic(c, q, dt, Hq, tq, out, checksum, ws, st);
}

// append(k, v) then attend(q) in one launch when the append is a decode step the
// attention kernel can run in its prologue; otherwise the two calls in order.
void append_attend(kvmix_cache* c, const void* k, const void* v, kvmix_dtype kv_dt, int t, const void* q,
                   kvmix_dtype q_dt, int Hq, int tq, float* out, double* checksum, Workspace& ws, cudaStream_t st) {
  if (c->total() + t > c->cap || t < 1) {
    cache_append(c, k, v, kv_dt, t, st);  // raises the reference's errors
  } else {
    check_query_shape(c, Hq, tq);  // shape errors before any state changes (the append makes
                                   // the cache non-empty)
    DecodeAppend da;
    if (cache_append_decode_plan(c, k, v, kv_dt, t, &da)) {
      if (attend_mma(c, q, q_dt, Hq, tq, out, checksum, ws, st, &da)) return;
      launch_decode_append(da, st);
    } else {
      cache_append(c, k, v, kv_dt, t, st);
    }
  }
  attend(c, q, q_dt, Hq, tq, out, checksum, ws, st);
}
}  // namespace kvb
