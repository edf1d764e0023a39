// Chunk-level quantization search (Module I):
//   score_chunks        retrieval.py:199-219  (cosine, zero-norm substitution)
//   compute_thresholds  retrieval.py:222-237  (two roundings each, no FMA)
//   assign_tiers        retrieval.py:240-250  (strict rule, ties -> INT4)
//   stable grouping     kv_store.py:190-192,204-206 (perm = INT2 || INT4 || FP16)
// Scores: a grid over (chunk blocks, sequences), four chunks per warp with all their loads in
// flight (the embeddings are the only sizeable input).  Thresholds, tiers and the stable
// partition: one CTA per sequence.  Everything stays on the device.
#include <math.h>

#include "ckv_common.cuh"

namespace ckv {

constexpr int kSearchThreads = 512;

__device__ __forceinline__ double block_reduce(double v, bool is_min, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_min ? fmin(v, w) : fmax(v, w);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (blockDim.x >> 5) ? red[lane] : (is_min ? INFINITY : -INFINITY);
    for (int o = 16; o > 0; o >>= 1) {
      double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_min ? fmin(v, w) : fmax(v, w);
    }
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

constexpr int kScoreWarps = 8, kScorePerWarp = 4;

// raw cosine per chunk: q . c / (|q| |c|)  (retrieval.py:202); NaN marks zero-norm chunks
__global__ void __launch_bounds__(kScoreWarps * 32)
score_kernel(const double* __restrict__ emb, const double* __restrict__ emb_norm,
             const double* __restrict__ q, const double* __restrict__ q_norm,
             const int32_t* __restrict__ seq_chunks, int n_max, int dim, double* __restrict__ scores) {
  const int b = blockIdx.y;
  const int n = seq_chunks ? min(seq_chunks[b], n_max) : n_max;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = (blockIdx.x * kScoreWarps + warp) * kScorePerWarp;
  if (i0 >= n) return;
  const double* Q = q + (int64_t)b * dim;
  const double* E = emb + ((int64_t)b * n_max + i0) * dim;
  double s[kScorePerWarp];
#pragma unroll
  for (int k = 0; k < kScorePerWarp; ++k) s[k] = 0.0;
#pragma unroll 4
  for (int d = lane; d < dim; d += 32) {
    const double qd = __ldg(Q + d);
#pragma unroll
    for (int k = 0; k < kScorePerWarp; ++k)
      if (i0 + k < n) s[k] = fma(qd, __ldg(E + (int64_t)k * dim + d), s[k]);
  }
#pragma unroll
  for (int k = 0; k < kScorePerWarp; ++k)
    for (int o = 16; o > 0; o >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o);
  if (lane < kScorePerWarp && i0 + lane < n) {
    double v = s[0];
#pragma unroll
    for (int k = 1; k < kScorePerWarp; ++k) if (lane == k) v = s[k];
    const double cn = emb_norm[(int64_t)b * n_max + i0 + lane];
    scores[(int64_t)b * n_max + i0 + lane] = cn > 0.0 ? __ddiv_rn(v, __dmul_rn(q_norm[b], cn)) : NAN;
  }
}

// scored != 0: `scores` holds score_kernel's raw cosines (zero-norm substitution still to do);
// scored == 0: `scores` is caller input (compute_thresholds / assign_tiers entries).
__global__ void __launch_bounds__(kSearchThreads)
search_kernel(int scored, const double* __restrict__ q_norm,
              const int32_t* __restrict__ seq_chunks, int n_max, double alpha,
              double beta, int ab_gt_1, const double* __restrict__ t_in,
              double* __restrict__ scores, double* __restrict__ stats,
              uint8_t* __restrict__ tiers, uint32_t* __restrict__ perm,
              int32_t* __restrict__ seg_counts, int32_t* __restrict__ flags) {
  __shared__ double red[32];
  __shared__ int cnt[kSearchThreads][3];
  __shared__ int tot[3];
  const int b = blockIdx.x;
  const int n = seq_chunks ? min(seq_chunks[b], n_max) : n_max;
  const double qn = scored ? q_norm[b] : 1.0;
  double* S = scores + (int64_t)b * n_max;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t flag = 0;
  if (qn == 0.0) flag |= CKV_FLAG_ZERO_QUERY;
  if (n == 0) flag |= CKV_FLAG_EMPTY_SCORES;

  double lo = INFINITY, hi = -INFINITY;
  if (scored) {
    __syncthreads();
    // zero-norm chunks score min(valid), 0.0 if none valid (retrieval.py:217-219)
    double lmin = INFINITY;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double s = S[i];
      if (!isnan(s)) lmin = fmin(lmin, s);
    }
    const double vmin = block_reduce(lmin, true, red);
    const double floor_v = isinf(vmin) ? 0.0 : vmin;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double s = S[i];
      if (isnan(s)) S[i] = s = floor_v;
      lo = fmin(lo, s);
      hi = fmax(hi, s);
    }
  } else {
    // scores supplied by the caller (compute_thresholds / assign_tiers entry)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double s = S[i];
      lo = fmin(lo, s);
      hi = fmax(hi, s);
    }
  }
  const double s_min = block_reduce(lo, true, red);
  const double s_max = block_reduce(hi, false, red);
  if (ab_gt_1 && s_max > s_min) flag |= CKV_FLAG_CROSSING;  // retrieval.py:231-234
  const double range = __dsub_rn(s_max, s_min);
  // retrieval.py:235-236, or caller-given thresholds (assign_tiers, retrieval.py:240)
  const double t_low = t_in ? t_in[2 * b] : __dadd_rn(s_min, __dmul_rn(range, alpha));
  const double t_high = t_in ? t_in[2 * b + 1] : __dsub_rn(s_max, __dmul_rn(range, beta));

  // tier per chunk + stable three-way partition.  Thread t owns a contiguous slice so
  // per-tier order inside the permutation is the original chunk order (kv_store.py:190-192).
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int i0 = min(n, (int)threadIdx.x * per), i1 = min(n, i0 + per);
  int c0 = 0, c1 = 0, c2 = 0;
  uint8_t* T = tiers + (int64_t)b * n_max;
  for (int i = i0; i < i1; ++i) {
    const double s = S[i];
    const uint8_t t = s < t_low ? CKV_TIER_INT2 : (s > t_high ? CKV_TIER_FP16 : CKV_TIER_INT4);
    T[i] = t;
    c0 += t == CKV_TIER_INT2;
    c1 += t == CKV_TIER_INT4;
    c2 += t == CKV_TIER_FP16;
  }
  cnt[threadIdx.x][0] = c0;
  cnt[threadIdx.x][1] = c1;
  cnt[threadIdx.x][2] = c2;
  __syncthreads();
  // exclusive scan over threads (serial per tier by 3 threads; n_threads <= 512)
  if (threadIdx.x < 3) {
    int acc = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      int v = cnt[t][threadIdx.x];
      cnt[t][threadIdx.x] = acc;
      acc += v;
    }
    tot[threadIdx.x] = acc;
  }
  __syncthreads();
  const int n2 = tot[0], n4 = tot[1];
  int p0 = cnt[threadIdx.x][0], p1 = n2 + cnt[threadIdx.x][1], p2 = n2 + n4 + cnt[threadIdx.x][2];
  uint32_t* P = perm + (int64_t)b * n_max;
  for (int i = i0; i < i1; ++i) {
    const uint8_t t = T[i];
    const int pos = t == CKV_TIER_INT2 ? p0++ : (t == CKV_TIER_INT4 ? p1++ : p2++);
    P[pos] = (uint32_t)i;
  }
  if (threadIdx.x == 0) {
    seg_counts[b * 3 + 0] = n2;
    seg_counts[b * 3 + 1] = n4;
    seg_counts[b * 3 + 2] = tot[2];
    double* st = stats + (int64_t)b * 4;
    st[0] = s_min;
    st[1] = s_max;
    st[2] = t_low;
    st[3] = t_high;
    flags[b] = flag;
  }
}

}  // namespace ckv

using namespace ckv;

extern "C" int32_t ckv_search(const double* emb, const double* emb_norm, const double* q,
                              const double* q_norm, const int32_t* seq_chunks, int32_t batch,
                              int32_t n_chunks, int32_t dim, double alpha, double beta,
                              double* scores, double* stats, uint8_t* tiers, uint32_t* perm,
                              int32_t* seg_counts, int32_t* flags, void* stream) {
  if (batch < 0 || n_chunks < 0 || (emb && dim < 1)) return CKV_ERR_ARG;
  if (emb && (!emb_norm || !q || !q_norm)) return CKV_ERR_ARG;
  if (!(alpha >= 0.0 && alpha <= 1.0 && beta >= 0.0 && beta <= 1.0)) return CKV_ERR_ARG;
  if (batch == 0) return CKV_OK;
  const int ab_gt_1 = (alpha + beta) > 1.0;
  if (emb && n_chunks > 0) {
    const int per_cta = kScoreWarps * kScorePerWarp;
    score_kernel<<<dim3((unsigned)cdiv(n_chunks, per_cta), (unsigned)batch), kScoreWarps * 32, 0,
                   as_stream(stream)>>>(emb, emb_norm, q, q_norm, seq_chunks, n_chunks, dim, scores);
    CKV_LAUNCH_CHECK();
  }
  search_kernel<<<batch, kSearchThreads, 0, as_stream(stream)>>>(
      emb ? 1 : 0, q_norm, seq_chunks, n_chunks, alpha, beta, ab_gt_1, nullptr, scores, stats,
      tiers, perm, seg_counts, flags);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

extern "C" int32_t ckv_assign_tiers(const double* scores, const double* thresholds,
                                    const int32_t* seq_chunks, int32_t batch, int32_t n_chunks,
                                    uint8_t* tiers, uint32_t* perm, int32_t* seg_counts,
                                    double* stats, int32_t* flags, void* stream) {
  if (batch < 0 || n_chunks < 0 || !scores || !thresholds) return CKV_ERR_ARG;
  if (batch == 0) return CKV_OK;
  search_kernel<<<batch, kSearchThreads, 0, as_stream(stream)>>>(
      0, nullptr, seq_chunks, n_chunks, 0.0, 0.0, 0, thresholds, const_cast<double*>(scores), stats,
      tiers, perm, seg_counts, flags);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}
