// Chunk-level KV cache computation (Module II, decode side):
//   attention.mixed_decode_attention   attention.py:63-90
//     per-tier q.K^T (fqm, transpose)    attention.py:75-77 -> quantizer.fqm -> _core.pyx:148-192
//     concat, *= scale, one softmax      attention.py:78-82, stable_softmax attention.py:24-31
//     per-tier P.V summed                attention.py:84-90
// for every (layer, sequence, kv-head) unit in one launch.  One global softmax over the
// concatenated INT2 || INT4 || FP16 sequence is computed as an online (m, l, acc) softmax
// walked tile by tile; split-KV partials are merged by log-sum-exp.  Mathematically the
// same result; numerically fp16 operands with fp32 accumulation.
//
// Tile = 16 tokens.  Per warp and tile:
//   S^T[16 tok x 8 q] = K_tile[16 x 128] . Q^T          mma.m16n8k16 x 8  (+1 for the lo term)
//   P = exp2(S - m) (online, lazy rescale), P^T -> P via movmatrix
//   O^T[128 d x 8 q] += V_tile^T[128 x 16] . P^T        mma.m16n8k16 x 8  (+1 for the lo term)
// Quantized operands are rebuilt in registers from the reference-format packed words:
//   fp16 magic: (code << j) | exp(2^(10-j)) == 2^(10-j) + code exactly, then
//   v = fma(x, sc, -2^(10-j) sc) = sc * code  (one rounding); the per-(token, group) zero point
//   lo is applied through an extra MMA (K side: lo x sum_g(q); V side: sum_t p_t lo_t).
#include <math.h>

#include "ckv_common.cuh"

namespace ckv {

constexpr int kDecWarps = 4;
constexpr int kTile = 16;
constexpr int kPartStride = kHeadDim + 2;  // acc[128], m, l
constexpr float kRescaleThresh = 8.0f;     // lazy rescale: p <= 2^8 in fp16

struct DecArgs {
  const uint16_t* q;
  int64_t q_sl, q_sb;
  ckv_arena K, V;
  const int32_t* seq;
  int L, B, H, m, splits;
  float scale_log2;
  float* ws;  // [L][B][H*m][splits][130]
  uint16_t* out;
  int64_t o_sl, o_sb;
  float* partial_out;  // [L][B][H*m][130] or null
};

struct Seq8 {
  int off2, len2, off4, len4, off_fp, len_fp, tail_src, ctx;
};

__device__ __forceinline__ Seq8 ld_seq(const int32_t* seq, int b) {
  const int4 a = reinterpret_cast<const int4*>(seq)[2 * b];
  const int4 c = reinterpret_cast<const int4*>(seq)[2 * b + 1];
  return Seq8{a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// half2 (lo, hi) metadata -> scale (hi - lo)/qmax as fp16 and lo as fp16
__device__ __forceinline__ float meta_scale(uint32_t meta, float inv_qmax) {
  const float2 lh = __half22float2(u32_as_h2(meta));
  return (lh.y - lh.x) * inv_qmax;
}
__device__ __forceinline__ uint32_t meta_lo_pair(uint32_t m0, uint32_t m1) {
  return prmt(m0, m1, 0x5410);  // (lo0, lo1)
}

// Per pair-register dequant constants for one (sc_lo_half, sc_hi_half) pair.
// negB[k] = -2^(10-2k) * sc  for magic exponents j = 2k (k = 0..4).
struct DeqC {
  __half2 sc;
  __half2 negB[5];
};
__device__ __forceinline__ DeqC make_deq(float s0, float s1) {
  DeqC d;
  d.sc = __floats2half2_rn(s0, s1);
#pragma unroll
  for (int k = 0; k < 5; ++k) d.negB[k] = __hmul2(d.sc, __float2half2_rn(-(float)(1 << (10 - 2 * k))));
  return d;
}

// INT2: 2-bit codes at bits (2i, 16 + 2i) of x; pair index i in 0..7 (i >= 5 uses x >> 10).
template <int I>
__device__ __forceinline__ uint32_t deq2(uint32_t c, const DeqC& d) {
  constexpr int j = I <= 4 ? 2 * I : 2 * (I - 5);
  const uint32_t x = I <= 4 ? c : (c >> 10);
  const uint32_t raw = (x & (0x00030003u << j)) | (((uint32_t)(25 - j) << 10) * 0x10001u);
  return h2_as_u32(__hfma2(u32_as_h2(raw), d.sc, d.negB[j / 2]));
}
// INT4: 4-bit codes at bits (4i, 16 + 4i) of x; i in 0..3 (i >= 2 uses x >> 8).
template <int I>
__device__ __forceinline__ uint32_t deq4(uint32_t c, const DeqC& d) {
  constexpr int j = 4 * (I & 1);
  const uint32_t x = I < 2 ? c : (c >> 8);
  const uint32_t raw = (x & (0x000F000Fu << j)) | (((uint32_t)(25 - j) << 10) * 0x10001u);
  return h2_as_u32(__hfma2(u32_as_h2(raw), d.sc, d.negB[j / 2]));
}
// Slow path (scale too large for the magic bias): exact code via subtraction, full affine.
template <int BITS>
__device__ __forceinline__ uint32_t deq_slow(uint32_t c, int i, __half2 sc, __half2 lo) {
  const int j = BITS == 2 ? (i <= 4 ? 2 * i : 2 * (i - 5)) : 4 * (i & 1);
  const uint32_t x = BITS == 2 ? (i <= 4 ? c : c >> 10) : (i < 2 ? c : c >> 8);
  const uint32_t mask = (BITS == 2 ? 0x00030003u : 0x000F000Fu) << j;
  const uint32_t raw = (x & mask) | (((uint32_t)(25 - j) << 10) * 0x10001u);
  const __half2 bias = __float2half2_rn((float)(1 << (10 - j)));
  const __half2 code = __hsub2(u32_as_h2(raw), bias);  // exact small integer
  return h2_as_u32(__hfma2(code, sc, lo));
}

struct WarpState {
  float acc[8][4];  // O^T C-fragments, m-tile mt: rows d = 16g+mt (c0,c1), 16g+8+mt (c2,c3)
  float lacc[4];    // sum_t p_t * lo_t per (group of row g, col)
  float mrun[2];    // running max (log2 domain) for cols 2c, 2c+1
  float lsum[2];
};

// Online softmax on one S^T tile and P^T -> P B-fragments for the PV MMA.
__device__ __forceinline__ void softmax_tile(float (&s)[4], WarpState& st, uint32_t& bp0,
                                             uint32_t& bp1) {
  float t0 = fmaxf(s[0], s[2]), t1 = fmaxf(s[1], s[3]);
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, o));
    t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, o));
  }
  const bool need = (t0 > st.mrun[0] + kRescaleThresh) || (t1 > st.mrun[1] + kRescaleThresh);
  if (__any_sync(0xffffffffu, need)) {
    const float n0 = fmaxf(st.mrun[0], t0), n1 = fmaxf(st.mrun[1], t1);
    const float f0 = st.mrun[0] == -INFINITY ? 0.0f : fast_exp2(st.mrun[0] - n0);
    const float f1 = st.mrun[1] == -INFINITY ? 0.0f : fast_exp2(st.mrun[1] - n1);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      st.acc[mt][0] *= f0; st.acc[mt][1] *= f1; st.acc[mt][2] *= f0; st.acc[mt][3] *= f1;
    }
    st.lacc[0] *= f0; st.lacc[1] *= f1; st.lacc[2] *= f0; st.lacc[3] *= f1;
    st.lsum[0] *= f0; st.lsum[1] *= f1;
    st.mrun[0] = n0; st.mrun[1] = n1;
  }
  const float p0 = fast_exp2(s[0] - st.mrun[0]), p1 = fast_exp2(s[1] - st.mrun[1]);
  const float p2 = fast_exp2(s[2] - st.mrun[0]), p3 = fast_exp2(s[3] - st.mrun[1]);
  st.lsum[0] += p0 + p2;
  st.lsum[1] += p1 + p3;
  bp0 = movmatrix_trans(h2_as_u32(__floats2half2_rn(p0, p1)));  // (P[g][2c], P[g][2c+1])
  bp1 = movmatrix_trans(h2_as_u32(__floats2half2_rn(p2, p3)));  // (P[g][8+2c], P[g][9+2c])
}

// ---- INT2 tile ------------------------------------------------------------------
__device__ __forceinline__ void tile_int2(const DecArgs& a, const uint32_t* kc, const uint32_t* km,
                                          const uint32_t* vc, const uint32_t* vm,
                                          const uint32_t (&qb)[8][2], uint32_t qaug, WarpState& st,
                                          int g, int c) {
  // K: tokens g, g+8; group c = words 2c, 2c+1 (d 32c .. 32c+31)
  const uint2 kw0 = *reinterpret_cast<const uint2*>(kc + g * 8 + 2 * c);
  const uint2 kw1 = *reinterpret_cast<const uint2*>(kc + (g + 8) * 8 + 2 * c);
  const uint32_t km0 = km[g * 4 + c], km1 = km[(g + 8) * 4 + c];
  // V: tokens 2c, 2c+1, 2c+8, 2c+9; word g (d 16g .. 16g+15), group g/2
  const uint32_t v0 = vc[(2 * c) * 8 + g], v1 = vc[(2 * c + 1) * 8 + g];
  const uint32_t v2 = vc[(2 * c + 8) * 8 + g], v3 = vc[(2 * c + 9) * 8 + g];
  const uint32_t vm0 = vm[(2 * c) * 4 + (g >> 1)], vm1 = vm[(2 * c + 1) * 4 + (g >> 1)];
  const uint32_t vm2 = vm[(2 * c + 8) * 4 + (g >> 1)], vm3 = vm[(2 * c + 9) * 4 + (g >> 1)];
  constexpr float iq = 1.0f / 3.0f;
  const float sk0 = meta_scale(km0, iq), sk1 = meta_scale(km1, iq);
  const float sv0 = meta_scale(vm0, iq), sv1 = meta_scale(vm1, iq);
  const float sv2 = meta_scale(vm2, iq), sv3 = meta_scale(vm3, iq);
  const float smax = fmaxf(fmaxf(fmaxf(sk0, sk1), fmaxf(sv0, sv1)), fmaxf(sv2, sv3));
  const bool slow = __any_sync(0xffffffffu, smax > 63.0f);

  float s[4] = {0.f, 0.f, 0.f, 0.f};
  if (!slow) {
    const DeqC dk0 = make_deq(sk0, sk0), dk1 = make_deq(sk1, sk1);
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t w0 = blk ? kw0.y : kw0.x, w1 = blk ? kw1.y : kw1.x;
      mma_16816(s, deq2<0>(w0, dk0), deq2<0>(w1, dk1), deq2<1>(w0, dk0), deq2<1>(w1, dk1), qb[4 * blk + 0][0], qb[4 * blk + 0][1]);
      mma_16816(s, deq2<2>(w0, dk0), deq2<2>(w1, dk1), deq2<3>(w0, dk0), deq2<3>(w1, dk1), qb[4 * blk + 1][0], qb[4 * blk + 1][1]);
      mma_16816(s, deq2<4>(w0, dk0), deq2<4>(w1, dk1), deq2<5>(w0, dk0), deq2<5>(w1, dk1), qb[4 * blk + 2][0], qb[4 * blk + 2][1]);
      mma_16816(s, deq2<6>(w0, dk0), deq2<6>(w1, dk1), deq2<7>(w0, dk0), deq2<7>(w1, dk1), qb[4 * blk + 3][0], qb[4 * blk + 3][1]);
    }
    // zero points: lo_{tok, c} * (Qhi + Qlo)_c
    const uint32_t lo0 = prmt(km0, km0, 0x1010), lo1 = prmt(km1, km1, 0x1010);
    mma_16816(s, lo0, lo1, 0u, 0u, qaug, 0u);
  } else {
    const __half2 sc0 = __float2half2_rn(sk0), sc1 = __float2half2_rn(sk1);
    const __half2 lo0 = u32_as_h2(prmt(km0, km0, 0x1010)), lo1 = u32_as_h2(prmt(km1, km1, 0x1010));
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int blk = ks >> 2, i0 = 2 * (ks & 3);
      const uint32_t w0 = blk ? kw0.y : kw0.x, w1 = blk ? kw1.y : kw1.x;
      mma_16816(s, deq_slow<2>(w0, i0, sc0, lo0), deq_slow<2>(w1, i0, sc1, lo1),
                deq_slow<2>(w0, i0 + 1, sc0, lo0), deq_slow<2>(w1, i0 + 1, sc1, lo1), qb[ks][0], qb[ks][1]);
    }
  }
  uint32_t bp0, bp1;
  softmax_tile(s, st, bp0, bp1);
  const uint32_t c01lo = prmt(v0, v1, 0x5410), c01hi = prmt(v0, v1, 0x7632);
  const uint32_t c23lo = prmt(v2, v3, 0x5410), c23hi = prmt(v2, v3, 0x7632);
  if (!slow) {
    const DeqC d01 = make_deq(sv0, sv1), d23 = make_deq(sv2, sv3);
#define PV2(I)                                                                                     \
  mma_16816(st.acc[I], deq2<I>(c01lo, d01), deq2<I>(c01hi, d01), deq2<I>(c23lo, d23),            \
            deq2<I>(c23hi, d23), bp0, bp1);
    PV2(0) PV2(1) PV2(2) PV2(3) PV2(4) PV2(5) PV2(6) PV2(7)
#undef PV2
    mma_16816(st.lacc, meta_lo_pair(vm0, vm1), 0u, meta_lo_pair(vm2, vm3), 0u, bp0, bp1);
  } else {
    const __half2 sc01 = __floats2half2_rn(sv0, sv1), sc23 = __floats2half2_rn(sv2, sv3);
    const __half2 lo01 = u32_as_h2(meta_lo_pair(vm0, vm1)), lo23 = u32_as_h2(meta_lo_pair(vm2, vm3));
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
      mma_16816(st.acc[mt], deq_slow<2>(c01lo, mt, sc01, lo01), deq_slow<2>(c01hi, mt, sc01, lo01),
                deq_slow<2>(c23lo, mt, sc23, lo23), deq_slow<2>(c23hi, mt, sc23, lo23), bp0, bp1);
  }
}

// ---- INT4 tile ------------------------------------------------------------------
__device__ __forceinline__ void tile_int4(const DecArgs& a, const uint32_t* kc, const uint32_t* km,
                                          const uint32_t* vc, const uint32_t* vm,
                                          const uint32_t (&qb)[8][2], uint32_t qaug, WarpState& st,
                                          int g, int c) {
  // K: tokens g, g+8; group c = words 4c .. 4c+3
  const uint4 kw0 = *reinterpret_cast<const uint4*>(kc + g * 16 + 4 * c);
  const uint4 kw1 = *reinterpret_cast<const uint4*>(kc + (g + 8) * 16 + 4 * c);
  const uint32_t km0 = km[g * 4 + c], km1 = km[(g + 8) * 4 + c];
  // V: tokens 2c, 2c+1, 2c+8, 2c+9; words 2g, 2g+1 (d 16g .. 16g+15)
  const uint2 v0 = *reinterpret_cast<const uint2*>(vc + (2 * c) * 16 + 2 * g);
  const uint2 v1 = *reinterpret_cast<const uint2*>(vc + (2 * c + 1) * 16 + 2 * g);
  const uint2 v2 = *reinterpret_cast<const uint2*>(vc + (2 * c + 8) * 16 + 2 * g);
  const uint2 v3 = *reinterpret_cast<const uint2*>(vc + (2 * c + 9) * 16 + 2 * g);
  const uint32_t vm0 = vm[(2 * c) * 4 + (g >> 1)], vm1 = vm[(2 * c + 1) * 4 + (g >> 1)];
  const uint32_t vm2 = vm[(2 * c + 8) * 4 + (g >> 1)], vm3 = vm[(2 * c + 9) * 4 + (g >> 1)];
  constexpr float iq = 1.0f / 15.0f;
  const float sk0 = meta_scale(km0, iq), sk1 = meta_scale(km1, iq);
  const float sv0 = meta_scale(vm0, iq), sv1 = meta_scale(vm1, iq);
  const float sv2 = meta_scale(vm2, iq), sv3 = meta_scale(vm3, iq);
  const float smax = fmaxf(fmaxf(fmaxf(sk0, sk1), fmaxf(sv0, sv1)), fmaxf(sv2, sv3));
  const bool slow = __any_sync(0xffffffffu, smax > 63.0f);

  float s[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t kwa[4] = {kw0.x, kw0.y, kw0.z, kw0.w}, kwb[4] = {kw1.x, kw1.y, kw1.z, kw1.w};
  if (!slow) {
    const DeqC dk0 = make_deq(sk0, sk0), dk1 = make_deq(sk1, sk1);
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      // pairs (d0, d0+8) = (word 2blk code i, word 2blk+1 code i)
      const uint32_t a_lo = prmt(kwa[2 * blk], kwa[2 * blk + 1], 0x5410), a_hi = prmt(kwa[2 * blk], kwa[2 * blk + 1], 0x7632);
      const uint32_t b_lo = prmt(kwb[2 * blk], kwb[2 * blk + 1], 0x5410), b_hi = prmt(kwb[2 * blk], kwb[2 * blk + 1], 0x7632);
      mma_16816(s, deq4<0>(a_lo, dk0), deq4<0>(b_lo, dk1), deq4<1>(a_lo, dk0), deq4<1>(b_lo, dk1), qb[4 * blk + 0][0], qb[4 * blk + 0][1]);
      mma_16816(s, deq4<2>(a_lo, dk0), deq4<2>(b_lo, dk1), deq4<3>(a_lo, dk0), deq4<3>(b_lo, dk1), qb[4 * blk + 1][0], qb[4 * blk + 1][1]);
      mma_16816(s, deq4<0>(a_hi, dk0), deq4<0>(b_hi, dk1), deq4<1>(a_hi, dk0), deq4<1>(b_hi, dk1), qb[4 * blk + 2][0], qb[4 * blk + 2][1]);
      mma_16816(s, deq4<2>(a_hi, dk0), deq4<2>(b_hi, dk1), deq4<3>(a_hi, dk0), deq4<3>(b_hi, dk1), qb[4 * blk + 3][0], qb[4 * blk + 3][1]);
    }
    const uint32_t lo0 = prmt(km0, km0, 0x1010), lo1 = prmt(km1, km1, 0x1010);
    mma_16816(s, lo0, lo1, 0u, 0u, qaug, 0u);
  } else {
    const __half2 sc0 = __float2half2_rn(sk0), sc1 = __float2half2_rn(sk1);
    const __half2 lo0 = u32_as_h2(prmt(km0, km0, 0x1010)), lo1 = u32_as_h2(prmt(km1, km1, 0x1010));
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t a_lo = prmt(kwa[2 * blk], kwa[2 * blk + 1], 0x5410), a_hi = prmt(kwa[2 * blk], kwa[2 * blk + 1], 0x7632);
      const uint32_t b_lo = prmt(kwb[2 * blk], kwb[2 * blk + 1], 0x5410), b_hi = prmt(kwb[2 * blk], kwb[2 * blk + 1], 0x7632);
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const uint32_t ca = q2 < 2 ? a_lo : a_hi, cb = q2 < 2 ? b_lo : b_hi;
        const int i = 2 * (q2 & 1);
        mma_16816(s, deq_slow<4>(ca, i, sc0, lo0), deq_slow<4>(cb, i, sc1, lo1),
                  deq_slow<4>(ca, i + 1, sc0, lo0), deq_slow<4>(cb, i + 1, sc1, lo1), qb[4 * blk + q2][0], qb[4 * blk + q2][1]);
      }
    }
  }
  uint32_t bp0, bp1;
  softmax_tile(s, st, bp0, bp1);
  // V pairs (tok 2c, 2c+1) / (2c+8, 2c+9) for d = 16g + mt (word 2g) and 16g + 8 + mt (word 2g+1)
  const uint32_t x01[4] = {prmt(v0.x, v1.x, 0x5410), prmt(v0.x, v1.x, 0x7632),
                           prmt(v0.y, v1.y, 0x5410), prmt(v0.y, v1.y, 0x7632)};
  const uint32_t x23[4] = {prmt(v2.x, v3.x, 0x5410), prmt(v2.x, v3.x, 0x7632),
                           prmt(v2.y, v3.y, 0x5410), prmt(v2.y, v3.y, 0x7632)};
  if (!slow) {
    const DeqC d01 = make_deq(sv0, sv1), d23 = make_deq(sv2, sv3);
    // mt in 0..3 -> x[0] pairs mt; mt in 4..7 -> x[1] pairs mt-4; rows g+8 use x[2], x[3]
#define PV4(MT)                                                                                    \
  mma_16816(st.acc[MT], deq4<(MT) & 3>(x01[(MT) >> 2], d01), deq4<(MT) & 3>(x01[2 + ((MT) >> 2)], d01), \
            deq4<(MT) & 3>(x23[(MT) >> 2], d23), deq4<(MT) & 3>(x23[2 + ((MT) >> 2)], d23), bp0, bp1);
    PV4(0) PV4(1) PV4(2) PV4(3) PV4(4) PV4(5) PV4(6) PV4(7)
#undef PV4
    mma_16816(st.lacc, meta_lo_pair(vm0, vm1), 0u, meta_lo_pair(vm2, vm3), 0u, bp0, bp1);
  } else {
    const __half2 sc01 = __floats2half2_rn(sv0, sv1), sc23 = __floats2half2_rn(sv2, sv3);
    const __half2 lo01 = u32_as_h2(meta_lo_pair(vm0, vm1)), lo23 = u32_as_h2(meta_lo_pair(vm2, vm3));
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
      mma_16816(st.acc[mt], deq_slow<4>(x01[mt >> 2], mt & 3, sc01, lo01),
                deq_slow<4>(x01[2 + (mt >> 2)], mt & 3, sc01, lo01),
                deq_slow<4>(x23[mt >> 2], mt & 3, sc23, lo23),
                deq_slow<4>(x23[2 + (mt >> 2)], mt & 3, sc23, lo23), bp0, bp1);
  }
}

// ---- FP16 tile (FP16-tier chunks, tail, decode tokens) ----------------------------
__device__ __forceinline__ void tile_fp16(const uint16_t* kf, const uint16_t* vf, int valid,
                                          const uint32_t (&qb)[8][2], WarpState& st, int g, int c) {
  // K: tokens g, g+8, d 32c .. 32c+31 (16 words each)
  uint32_t ka[16], kb[16];
  {
    const uint4* p0 = reinterpret_cast<const uint4*>(kf + g * kHeadDim + 32 * c);
    const uint4* p1 = reinterpret_cast<const uint4*>(kf + (g + 8) * kHeadDim + 32 * c);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint4 x = p0[u], y = p1[u];
      ka[4 * u] = x.x; ka[4 * u + 1] = x.y; ka[4 * u + 2] = x.z; ka[4 * u + 3] = x.w;
      kb[4 * u] = y.x; kb[4 * u + 1] = y.y; kb[4 * u + 2] = y.z; kb[4 * u + 3] = y.w;
    }
  }
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    // pair (d0, d0+8), d0 = 32c + 16blk + 2(ks&3): words 8blk + (ks&3) and 8blk + 4 + (ks&3)
    const int wa = 8 * (ks >> 2) + (ks & 3), wb = wa + 4;
    mma_16816(s, prmt(ka[wa], ka[wb], 0x5410), prmt(kb[wa], kb[wb], 0x5410),
              prmt(ka[wa], ka[wb], 0x7632), prmt(kb[wa], kb[wb], 0x7632), qb[ks][0], qb[ks][1]);
  }
  if (g >= valid) { s[0] = -INFINITY; s[1] = -INFINITY; }
  if (g + 8 >= valid) { s[2] = -INFINITY; s[3] = -INFINITY; }
  uint32_t bp0, bp1;
  softmax_tile(s, st, bp0, bp1);
  // V: tokens 2c, 2c+1, 2c+8, 2c+9, d 16g .. 16g+15 (8 words each)
  uint32_t vw[4][8];
  const int toks[4] = {2 * c, 2 * c + 1, 2 * c + 8, 2 * c + 9};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint4* p = reinterpret_cast<const uint4*>(vf + toks[t] * kHeadDim + 16 * g);
    const uint4 x = p[0], y = p[1];
    vw[t][0] = x.x; vw[t][1] = x.y; vw[t][2] = x.z; vw[t][3] = x.w;
    vw[t][4] = y.x; vw[t][5] = y.y; vw[t][6] = y.z; vw[t][7] = y.w;
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const uint32_t sel = (mt & 1) ? 0x7632 : 0x5410;
    const int w0 = mt >> 1, w1 = 4 + (mt >> 1);
    mma_16816(st.acc[mt], prmt(vw[0][w0], vw[1][w0], sel), prmt(vw[0][w1], vw[1][w1], sel),
              prmt(vw[2][w0], vw[3][w0], sel), prmt(vw[2][w1], vw[3][w1], sel), bp0, bp1);
  }
}

__global__ void __launch_bounds__(kDecWarps * 32, 4) decode_kernel(const DecArgs a) {
  __shared__ float s_acc[kDecWarps][8][kHeadDim];
  __shared__ float s_ml[kDecWarps][8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int split = blockIdx.x, h = blockIdx.y;
  const int l = blockIdx.z / a.B, b = blockIdx.z % a.B;
  const Seq8 sq = ld_seq(a.seq, b);
  const int n2t = sq.len2 / kTile, n4t = sq.len4 / kTile;
  const int nft = (sq.len_fp + kTile - 1) / kTile;
  // byte-balanced split of the virtual tile sequence (INT2 || INT4 || FP16)
  const int64_t c2 = 96, c4 = 160, cf = 512;
  const int64_t tot = n2t * c2 + n4t * c4 + nft * cf;
  auto tile_at = [&](int64_t x) -> int {  // first tile whose start cost >= x
    if (x <= n2t * c2) return (int)((x + c2 - 1) / c2);
    x -= n2t * c2;
    if (x <= n4t * c4) return n2t + (int)((x + c4 - 1) / c4);
    x -= n4t * c4;
    return n2t + n4t + (int)min((int64_t)nft, (x + cf - 1) / cf);
  };
  const int t_begin = tile_at(tot * split / a.splits);
  const int t_end = tile_at(tot * (split + 1) / a.splits);

  // Q B-fragments (scaled to log2 units), q-row i = g (zero if g >= m)
  uint32_t qb[8][2], qaug;
  {
    float qv[32];
    const uint16_t* qrow = a.q + l * a.q_sl + b * a.q_sb + (int64_t)(h * a.m + g) * kHeadDim + 32 * c;
    if (g < a.m) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 x = reinterpret_cast<const uint4*>(qrow)[u];
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(u32_as_h2(w[e]));
          qv[8 * u + 2 * e] = f.x * a.scale_log2;
          qv[8 * u + 2 * e + 1] = f.y * a.scale_log2;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) qv[e] = 0.f;
    }
    float qsum = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      qv[e] = __half2float(__float2half_rn(qv[e]));  // exactly the fp16 operand the MMA sees
      qsum += qv[e];
    }
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int d0 = 16 * (ks >> 2) + 2 * (ks & 3);  // lane-local index within group c
      qb[ks][0] = h2_as_u32(__floats2half2_rn(qv[d0], qv[d0 + 8]));
      qb[ks][1] = h2_as_u32(__floats2half2_rn(qv[d0 + 1], qv[d0 + 9]));
    }
    const __half qhi = __float2half_rn(qsum);
    const __half qlo = __float2half_rn(qsum - __half2float(qhi));
    qaug = h2_as_u32(__halves2half2(qhi, qlo));
  }

  WarpState st;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) st.acc[mt][0] = st.acc[mt][1] = st.acc[mt][2] = st.acc[mt][3] = 0.f;
  st.lacc[0] = st.lacc[1] = st.lacc[2] = st.lacc[3] = 0.f;
  st.mrun[0] = st.mrun[1] = -INFINITY;
  st.lsum[0] = st.lsum[1] = 0.f;

  const int64_t unit = (int64_t)l * a.H + h;
  const uint32_t* k2 = a.K.codes2 + (unit * a.K.rows2 + sq.off2) * 8;
  const uint32_t* k2m = a.K.meta2 + (unit * a.K.rows2 + sq.off2) * 4;
  const uint32_t* v2 = a.V.codes2 + (unit * a.V.rows2 + sq.off2) * 8;
  const uint32_t* v2m = a.V.meta2 + (unit * a.V.rows2 + sq.off2) * 4;
  const uint32_t* k4 = a.K.codes4 + (unit * a.K.rows4 + sq.off4) * 16;
  const uint32_t* k4m = a.K.meta4 + (unit * a.K.rows4 + sq.off4) * 4;
  const uint32_t* v4 = a.V.codes4 + (unit * a.V.rows4 + sq.off4) * 16;
  const uint32_t* v4m = a.V.meta4 + (unit * a.V.rows4 + sq.off4) * 4;
  const uint16_t* kf = a.K.fp + (unit * a.K.rows_fp + sq.off_fp) * kHeadDim;
  const uint16_t* vf = a.V.fp + (unit * a.V.rows_fp + sq.off_fp) * kHeadDim;

  for (int t = t_begin + warp; t < t_end; t += kDecWarps) {
    if (t < n2t) {
      const int r = t * kTile;
      tile_int2(a, k2 + r * 8, k2m + r * 4, v2 + r * 8, v2m + r * 4, qb, qaug, st, g, c);
    } else if (t < n2t + n4t) {
      const int r = (t - n2t) * kTile;
      tile_int4(a, k4 + r * 16, k4m + r * 4, v4 + r * 16, v4m + r * 4, qb, qaug, st, g, c);
    } else {
      const int r = (t - n2t - n4t) * kTile;
      tile_fp16(kf + (int64_t)r * kHeadDim, vf + (int64_t)r * kHeadDim, sq.len_fp - r, qb, st, g, c);
    }
  }

  // finish the warp: fold zero-point term, reduce row sums over the 8 row-groups
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    st.acc[mt][0] += st.lacc[0]; st.acc[mt][1] += st.lacc[1];
    st.acc[mt][2] += st.lacc[0]; st.acc[mt][3] += st.lacc[1];
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    st.lsum[0] += __shfl_xor_sync(0xffffffffu, st.lsum[0], o);
    st.lsum[1] += __shfl_xor_sync(0xffffffffu, st.lsum[1], o);
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    s_acc[warp][2 * c][16 * g + mt] = st.acc[mt][0];
    s_acc[warp][2 * c + 1][16 * g + mt] = st.acc[mt][1];
    s_acc[warp][2 * c][16 * g + 8 + mt] = st.acc[mt][2];
    s_acc[warp][2 * c + 1][16 * g + 8 + mt] = st.acc[mt][3];
  }
  if (g == 0) {
    s_ml[warp][2 * c][0] = st.mrun[0]; s_ml[warp][2 * c][1] = st.lsum[0];
    s_ml[warp][2 * c + 1][0] = st.mrun[1]; s_ml[warp][2 * c + 1][1] = st.lsum[1];
  }
  __syncthreads();
  // merge the 4 warps: thread -> d
  const int d = threadIdx.x;
  const int hq0 = h * a.m;
  for (int i = 0; i < a.m; ++i) {
    float ms = -INFINITY;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) ms = fmaxf(ms, s_ml[w][i][0]);
    float acc = 0.f, lsum = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) {
      const float mw = s_ml[w][i][0];
      const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
      acc += f * s_acc[w][i][d];
      lsum += f * s_ml[w][i][1];
    }
    const int64_t row = ((int64_t)l * a.B + b) * (a.H * a.m) + hq0 + i;
    if (a.splits == 1 && a.partial_out == nullptr) {
      a.out[l * a.o_sl + b * a.o_sb + (int64_t)(hq0 + i) * kHeadDim + d] = __half_as_ushort(__float2half_rn(acc / lsum));
    } else {
      float* dst = a.splits == 1 ? a.partial_out + row * kPartStride
                                 : a.ws + (row * a.splits + split) * kPartStride;
      dst[d] = acc;
      if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
    }
  }
}

// Merge split partials: [rows][splits][130] -> out fp16 (or a [rows][130] partial for the
// cross-rank exchange when partial_out is set).
__global__ void merge_splits_kernel(const float* __restrict__ ws, int splits, int64_t rows,
                                    int B, int Hq, uint16_t* __restrict__ out, int64_t o_sl,
                                    int64_t o_sb, float* __restrict__ partial_out) {
  const int64_t row = blockIdx.x;
  const int d = threadIdx.x;
  const float* p = ws + row * splits * kPartStride;
  float ms = -INFINITY;
  for (int s = 0; s < splits; ++s) ms = fmaxf(ms, p[s * kPartStride + kHeadDim]);
  float acc = 0.f, lsum = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float mw = p[s * kPartStride + kHeadDim];
    const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
    acc += f * p[s * kPartStride + d];
    lsum += f * p[s * kPartStride + kHeadDim + 1];
  }
  if (partial_out) {
    float* dst = partial_out + row * kPartStride;
    dst[d] = acc;
    if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
  } else {
    const int hq = (int)(row % Hq);
    const int b = (int)((row / Hq) % B);
    const int64_t l = row / ((int64_t)Hq * B);
    out[l * o_sl + b * o_sb + (int64_t)hq * kHeadDim + d] = __half_as_ushort(__float2half_rn(acc / lsum));
  }
}

// Cross-rank merge of gathered partials [P][rows][130] -> out fp16 [rows][128].
__global__ void lse_merge_kernel(const float* __restrict__ parts, int P, int64_t rows,
                                 uint16_t* __restrict__ out) {
  const int64_t row = blockIdx.x;
  const int d = threadIdx.x;
  float ms = -INFINITY;
  for (int p = 0; p < P; ++p) ms = fmaxf(ms, parts[((int64_t)p * rows + row) * kPartStride + kHeadDim]);
  float acc = 0.f, lsum = 0.f;
  for (int p = 0; p < P; ++p) {
    const float* q = parts + ((int64_t)p * rows + row) * kPartStride;
    const float f = q[kHeadDim] == -INFINITY ? 0.f : fast_exp2(q[kHeadDim] - ms);
    acc += f * q[d];
    lsum += f * q[kHeadDim + 1];
  }
  out[row * kHeadDim + d] = __half_as_ushort(__float2half_rn(acc / lsum));
}

}  // namespace ckv

using namespace ckv;

extern "C" {

int64_t ckv_decode_workspace_bytes(int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                                   int32_t splits) {
  if (splits <= 1) return 0;
  return (int64_t)layers * batch * kv_heads * m * splits * kPartStride * (int64_t)sizeof(float);
}

int32_t ckv_decode_attention(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                             ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                             int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                             float scale, int32_t splits, void* workspace, uint16_t* out,
                             int64_t o_s_layer, int64_t o_s_batch, float* partial_out,
                             void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0 || splits < 1) return CKV_ERR_ARG;
  if (m < 1 || m > 8) return CKV_ERR_UNSUPPORTED;
  if (!q || !seq || (!out && !partial_out)) return CKV_ERR_ARG;
  if (splits > 1 && !workspace) return CKV_ERR_ARG;
  if ((q_s_layer % 8) || (q_s_batch % 8)) return CKV_ERR_UNSUPPORTED;
  if (layers * batch * kv_heads == 0) return CKV_OK;
  DecArgs a;
  a.q = q; a.q_sl = q_s_layer; a.q_sb = q_s_batch;
  a.K = k_arena; a.V = v_arena; a.seq = seq;
  a.L = layers; a.B = batch; a.H = kv_heads; a.m = m; a.splits = splits;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.ws = reinterpret_cast<float*>(workspace);
  a.out = out; a.o_sl = o_s_layer; a.o_sb = o_s_batch;
  a.partial_out = partial_out;
  dim3 grid((unsigned)splits, (unsigned)kv_heads, (unsigned)(layers * batch));
  decode_kernel<<<grid, kDecWarps * 32, 0, as_stream(stream)>>>(a);
  CKV_LAUNCH_CHECK();
  if (splits > 1) {
    const int64_t rows = (int64_t)layers * batch * kv_heads * m;
    merge_splits_kernel<<<(unsigned)rows, kHeadDim, 0, as_stream(stream)>>>(
        a.ws, splits, rows, batch, kv_heads * m, out, o_s_layer, o_s_batch, partial_out);
    CKV_LAUNCH_CHECK();
  }
  return CKV_OK;
}

int32_t ckv_lse_merge(const float* partials, int32_t n_parts, int64_t rows, uint16_t* out,
                      void* stream) {
  if (n_parts < 1 || rows < 0 || !partials || !out) return CKV_ERR_ARG;
  if (rows == 0) return CKV_OK;
  lse_merge_kernel<<<(unsigned)rows, kHeadDim, 0, as_stream(stream)>>>(partials, n_parts, rows, out);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

}  // extern "C"
