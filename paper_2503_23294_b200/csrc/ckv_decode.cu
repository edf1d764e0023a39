// Chunk-level KV cache computation (Module II, decode side):
//   attention.mixed_decode_attention   attention.py:63-90
//     per-tier q.K^T (fqm, transpose)    attention.py:75-77 -> quantizer.fqm -> _core.pyx:148-192
//     concat, *= scale, one softmax      attention.py:78-82, stable_softmax attention.py:24-31
//     per-tier P.V summed                attention.py:84-90
// for every (layer, sequence, kv-head) unit in one launch.  The one global softmax over the
// concatenated INT2 || INT4 || FP16 sequence is computed as an online (m, l, acc) softmax
// walked tile by tile; split-KV partials are merged by log-sum-exp in the same launch (the
// last CTA of a unit merges).  fp16 operands, fp32 accumulation.
//
// Tile = 16 tokens.  Per warp and tile:
//   S^T[16 tok x 8 q] = K_tile[16 x 128] . Q^T          mma.m16n8k16 x 8  (+1 for the lo term)
//   P = exp2(S - m) (online, lazy rescale), P^T -> P via movmatrix
//   O^T[128 d x 8 q] += V_tile^T[128 x 16] . P^T        mma.m16n8k16 x 8  (+1 for the lo term)
// Quantized tiles stream through a per-warp 4-stage cp.async ring in shared memory (rows
// permuted inside the tile so every fragment read is bank-conflict free); FP16 tiles (<4% of
// bytes) are read straight from global memory.  Operands are rebuilt in registers from the
// reference-format packed words:
//   fp16 magic: (code << j) | exp(16)  ==  16 + code * 2^(j-6)  exactly, then
//   v = fma(x, sc, -16 sc) = sc * code * 2^(j-6)  (one rounding, one constant per scale).
//   The per-slot power-of-two weight 2^(j-6) is folded into q (K side: q' = q 2^(6-j) per
//   d-slot) and into the output rows (V side: j depends only on the m-tile, undone once at
//   the end).  The per-(token, group) zero point lo goes through one extra MMA per side
//   (K: lo x sum_g(q); V: sum_t p_t lo_t).  Units whose scales (or q) are too wide for the
//   weighted form run an unweighted exact mode (code by subtraction, full affine).
#include <math.h>

#include <cuda/atomic>
#include <type_traits>

#include "ckv_common.cuh"

namespace ckv {

constexpr int kDecWarps = 4;
constexpr int kTile = 16;
// Per-warp cp.async ring.  A stage holds one 16-token tile of the tile-native arenas verbatim
// (see the tile functions below): INT2 1536 B, INT4 2560 B.  The INT2 and INT4 phases reuse
// the same per-warp region, each with its own stage count.
#ifndef CKV_DEC_MIN_CTAS
#define CKV_DEC_MIN_CTAS 4
#endif
#ifndef CKV_DEC_STAGES2
#define CKV_DEC_STAGES2 4
#endif
#ifndef CKV_DEC_STAGES4
#define CKV_DEC_STAGES4 4
#endif
constexpr int kMinCtas = CKV_DEC_MIN_CTAS;
template <int BITS> struct Ring {
  static constexpr int stages = BITS == 2 ? CKV_DEC_STAGES2 : CKV_DEC_STAGES4;
  static constexpr int bytes = BITS == 2 ? 1536 : 2560;
};
constexpr int kWarpRing = Ring<2>::stages * Ring<2>::bytes > Ring<4>::stages * Ring<4>::bytes
                              ? Ring<2>::stages * Ring<2>::bytes : Ring<4>::stages * Ring<4>::bytes;
constexpr int kDynSmem = kDecWarps * kWarpRing;  // 40 KB per CTA (4 x 2560 B per warp)
constexpr int kPartStride = kHeadDim + 2;  // acc[128], m, l (partial_out / cross-rank format)
constexpr int kWsStride = kHeadDim + 4;    // split workspace rows: acc[128], m, l, pad (16-B rows)
constexpr float kRescaleThresh = 8.0f;     // lazy rescale: p <= 2^8 in fp16

struct DecArgs {
  const uint16_t* q;
  int64_t q_sl, q_sb;
  ckv_arena K, V;
  const int32_t* seq;
  int L, B, H, m, splits;
  int b0, Bc;           // this launch's sequences [b0, b0 + Bc) of the B in the cache
  float scale_log2;
  float* ws;            // [L*B*H*m][splits][130] partials
  uint32_t* counters;   // [L*B*H] arrival counters (self-resetting)
  uint16_t* out;
  int64_t o_sl, o_sb;
  float* partial_out;   // [L][B][H*m][130] or null
  uint32_t zero;        // runtime 0: keeps the fp16 magic exponents in registers (see Magic)
};

// Optional per-CTA timeline (tuning aid, not part of the ABI): when set, every CTA appends 16
// int64: globaltimer at start, after the PDL wait, after q staging, after warp 0's tiles, at
// exit; smid, linear block index, q pointer (launch id); after all warps' tiles, before the
// arrival atomic, after it, is-last; per-warp tile end times.
__device__ int64_t* g_trace = nullptr;
__device__ unsigned long long g_trace_n = 0;
__device__ __forceinline__ int64_t gtime() {
  int64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Probe points write shared memory and re-read g_trace each time, so nothing of the tracing
// stays live in registers across the tile loop.
__device__ __forceinline__ bool tracing() { return *reinterpret_cast<int64_t* volatile*>(&g_trace) != nullptr; }
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// (split, kv head, layer, sequence) of this CTA, re-read from the special registers at each
// call (volatile) so nothing derived from them stays live in registers across the tile loop.
struct CtaIds {
  int split, h, l, b;
};
__device__ __forceinline__ CtaIds cta_ids(int Bc, int b0) {
  uint32_t x, y, z;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(x));
  asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(y));
  asm volatile("mov.u32 %0, %%ctaid.z;" : "=r"(z));
  return CtaIds{(int)x, (int)y, (int)z / Bc, b0 + (int)z % Bc};
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N)); }

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}


constexpr uint32_t kMagic16 = 0x4C004C00u;  // fp16 16.0 in both halves
constexpr float kWideQ = 1000.0f;           // and |q| 2^6 in fp16 range
// precise K path when (largest K group span) x max|q| (log2-scaled q) exceeds this: the normal
// path's score error is ~2^-12 span |q| per group element (measured ~1.5e-3 relative output
// error at a product of ~3 on N(0,1) data, 1.8e-2 at ~55 on SURVEY's outlier variant)
constexpr float kPreciseSpanQ = 8.0f;

// scale (hi - lo) / qmax of one (lo, hi) half2 metadata word (hi - lo via mixed f16/f32 add)
__device__ __forceinline__ float meta_scale(uint32_t meta, float inv_qmax) {
  float d;
  asm("{.reg .f16 lo, hi; .reg .f32 a; mov.b32 {lo, hi}, %1; cvt.f32.f16 a, lo; sub.rn.f32.f16 %0, hi, a;}"
      : "=f"(d) : "r"(meta));
  return d * inv_qmax;
}

struct DeqC {
  __half2 sc;  // (sc_lo_half, sc_hi_half)
  __half2 nm;  // -16 * sc  (exact: power-of-two multiple)
};

// Scale constants straight from fp16 metadata with half2 arithmetic: span = hi - lo (one
// rounding), nm = -16 sc (exact).  The rounding of fp16(1/qmax) would bias every scale by the
// same relative amount (2.4e-4 for 1/3), and a constant bias does not average out over a long
// context.  K: sc = span * fp16(1/qmax), and the constant factor 1 / (qmax fp16(1/qmax)) is
// folded into that tier's q fragments.  V: sc = span * c_hi + span * c_lo (c_hi + c_lo = 1/qmax
// to 2^-22), one rounding.  K: one (lo, hi) word -> that token's constants in both halves;
// V: two words (tokens t0, t1) -> (t0, t1) constants.
__device__ __forceinline__ float kscale_fold(float inv_q) {  // 1 / (qmax * fp16(1/qmax))
  return inv_q / __half2float(__float2half_rn(inv_q));
}
__device__ __forceinline__ DeqC kdeq(uint32_t meta, __half2 inv_q) {
  const __half2 h = u32_as_h2(meta);
  DeqC d;
  d.sc = __hmul2(__hsub2(__high2half2(h), __low2half2(h)), inv_q);
  d.nm = __hmul2(d.sc, __float2half2_rn(-16.0f));
  return d;
}
__device__ __forceinline__ DeqC vdeq(uint32_t lo01, uint32_t hi01, float inv_q) {
  const __half c_hi = __float2half_rn(inv_q);
  const __half c_lo = __float2half_rn(inv_q - __half2float(c_hi));
  const __half2 span = __hsub2(u32_as_h2(hi01), u32_as_h2(lo01));
  DeqC d;
  d.sc = __hfma2(span, __half2half2(c_hi), __hmul2(span, __half2half2(c_lo)));
  d.nm = __hmul2(d.sc, __float2half2_rn(-16.0f));
  return d;
}

// weighted dequant of a pair of codes at bits (j, 16 + j) of x (mask = code mask << j)
__device__ __forceinline__ uint32_t wdeq(uint32_t x, uint32_t mask, uint32_t magic, const DeqC& d) {
  const uint32_t raw = (x & mask) | magic;
  return h2_as_u32(__hfma2(u32_as_h2(raw), d.sc, d.nm));
}
// exact (unweighted) dequant: code by subtraction, full affine v = code * sc + lo
__device__ __forceinline__ uint32_t edeq(uint32_t x, int j, uint32_t cmask, __half2 sc, __half2 lo) {
  const uint32_t raw = (x & (cmask << j)) | (((uint32_t)(25 - j) << 10) * 0x10001u);
  const __half2 code = __hsub2(u32_as_h2(raw), __float2half2_rn((float)(1 << (10 - j))));
  return h2_as_u32(__hfma2(code, sc, lo));
}

// INT2 K pair i of a word: bits (2i, 16+2i) for i <= 4, (2(i-5), ...) of w >> 10 for i >= 5
template <int I> struct K2 {
  static constexpr int j = I <= 4 ? 2 * I : 2 * (I - 5);
  static constexpr bool hi = I >= 5;
};
// INT4 K pair i (of a 4-pair PRMT word): bits (4(i&1), ...) of x or x >> 8
template <int I> struct K4 {
  static constexpr int j = 4 * (I & 1);
  static constexpr bool hi = (I & 3) >= 2;
};

struct WarpState {
  float acc[8][4];  // O^T C-fragments, m-tile mt: rows d = 16g+mt (c0,c1), 16g+8+mt (c2,c3)
  float lacc[2];    // sum_t p_t * lo_t for the group of row g, cols 2c, 2c+1
  float lsq[2];     // sum_t p_t over the quantized tiles (complete, from the lo MMA's ones rows)
  float mrun[2];    // running max (log2 domain) for cols 2c, 2c+1
  float lsum[2];
};

template <bool FADD_SUM>
__device__ __forceinline__ void softmax_tile(float (&s)[4], WarpState& st, uint32_t& bp0,
                                             uint32_t& bp1) {
  // Lazy online softmax: keep the running max unless a score exceeds it by more than the
  // threshold (then P <= 2^8 still fits fp16).  Only then reduce the tile max across the
  // 8 row-groups and rescale; the common case needs no shuffles.
  // scores relative to the running max (the exp2 arguments; the threshold test reuses them)
  float d0 = s[0] - st.mrun[0], d1 = s[1] - st.mrun[1], d2 = s[2] - st.mrun[0], d3 = s[3] - st.mrun[1];
  const bool need = (fmaxf(d0, d2) > kRescaleThresh) || (fmaxf(d1, d3) > kRescaleThresh);
  if (__any_sync(0xffffffffu, need)) {
    float t0 = fmaxf(s[0], s[2]), t1 = fmaxf(s[1], s[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, o));
      t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, o));
    }
    const float n0 = fmaxf(st.mrun[0], t0), n1 = fmaxf(st.mrun[1], t1);
    const float f0 = st.mrun[0] == -INFINITY ? 0.0f : fast_exp2(st.mrun[0] - n0);
    const float f1 = st.mrun[1] == -INFINITY ? 0.0f : fast_exp2(st.mrun[1] - n1);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      st.acc[mt][0] *= f0; st.acc[mt][1] *= f1; st.acc[mt][2] *= f0; st.acc[mt][3] *= f1;
    }
    st.lacc[0] *= f0; st.lacc[1] *= f1;
    st.lsq[0] *= f0; st.lsq[1] *= f1;
    st.lsum[0] *= f0; st.lsum[1] *= f1;
    st.mrun[0] = n0; st.mrun[1] = n1;
    d0 = s[0] - n0; d1 = s[1] - n1; d2 = s[2] - n0; d3 = s[3] - n1;
  }
  const float p0 = fast_exp2(d0), p1 = fast_exp2(d1), p2 = fast_exp2(d2), p3 = fast_exp2(d3);
  if (FADD_SUM) {  // else the lo MMA of the tile's P.V sums P (rows g+8 of its A are ones)
    st.lsum[0] += p0 + p2;
    st.lsum[1] += p1 + p3;
  }
  bp0 = movmatrix_trans(h2_as_u32(__floats2half2_rn(p0, p1)));  // (P[g][2c], P[g][2c+1])
  bp1 = movmatrix_trans(h2_as_u32(__floats2half2_rn(p2, p3)));  // (P[g][8+2c], P[g][9+2c])
}

// Q B-fragments live in shared memory as three sets ([set][k-step pair][32 lanes] x 16 B, one
// copy per CTA: k-steps 2kp, 2kp+1 of a lane side by side, so a pair is one conflict-free
// 128-bit load): 0 = INT2 slot weights, 1 = INT4 slot weights, 2 = unweighted (FP16 tiles and
// the exact mode).  After the sets, [32 lanes] x 4 B: the (hi, lo) split of sum_g(q) for the
// zero-point MMA.
constexpr int kQSet = 4 * 32 * 16;
constexpr int kQBytes = 3 * kQSet + 32 * 4;
struct QS {
  uint32_t base;  // s_q + 16 * lane
  uint32_t aug_addr;
  __device__ __forceinline__ uint2 ld(int set, int ks) const {
    return lds64(base + set * kQSet + 512 * (ks >> 1) + 8 * (ks & 1));
  }
  __device__ __forceinline__ uint4 ld2(int set, int kp) const { return lds128(base + set * kQSet + 512 * kp); }
  __device__ __forceinline__ uint32_t aug() const { return lds32(aug_addr); }
};
__device__ __forceinline__ uint2 lo2(const uint4& v) { return make_uint2(v.x, v.y); }
__device__ __forceinline__ uint2 hi2(const uint4& v) { return make_uint2(v.z, v.w); }

__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint2 b) {
  mma_16816(d, a0, a1, a2, a3, b.x, b.y);
}

// The V zero-point term sum_t p_t lo_t (A rows g) and, on the A rows g+8 set to fp16 ones, the
// tile's row sums sum_t p_t of the same fp16 P the P.V MMAs use.
__device__ __forceinline__ void lo_mma(WarpState& st, uint32_t a0, uint32_t a2, uint32_t bp0, uint32_t bp1) {
  constexpr uint32_t kOnes = 0x3C003C00u;
  float t[4] = {st.lacc[0], st.lacc[1], st.lsq[0], st.lsq[1]};
  mma_16816(t, a0, kOnes, a2, kOnes, bp0, bp1);
  st.lacc[0] = t[0];
  st.lacc[1] = t[1];
  st.lsq[0] = t[2];
  st.lsq[1] = t[3];
}

// ---- quantized tiles from a shared-memory stage ---------------------------------------
// A stage holds one tile in the tile-native arena layout (ckv_common.cuh), copied verbatim:
//   INT2: KC @0 (512 B), VC @512 (512 B), KM @1024 (256 B), VM @1280 (256 B)
//   INT4: KC @0 (1024 B), VC @1024 (1024 B), KM @2048, VM @2304
// `sl` = stage + 16 * lane (this lane's code slots); metadata addresses add the per-lane
// deltas of MetaOff (K: 8-byte entry per lane; V: 16-byte entry (g/2, c), shared by lane pairs).
struct MetaOff {
  int32_t k, v;  // k = -8 lane, v = 16 ((g >> 1) * 4 + c) - 16 lane
};

// exact-mode scales (f32, then fp16) of two tokens from (lo0, lo1) and (hi0, hi1) half2 words
__device__ __forceinline__ __half2 exact_sc2(uint32_t lo01, uint32_t hi01, float inv_q) {
  const float2 l = __half22float2(u32_as_h2(lo01)), h = __half22float2(u32_as_h2(hi01));
  return __floats2half2_rn((h.x - l.x) * inv_q, (h.y - l.y) * inv_q);
}

template <bool EXACT>
__device__ __forceinline__ void qk_int2(uint32_t sl, const MetaOff& mo, const QS& qs, uint32_t mg, float (&s)[4]) {
  const uint4 kk = lds128(sl);  // (tok g: words 2c, 2c+1), (tok g+8: words 2c, 2c+1)
  const uint2 kmm = lds64(sl + 1024 + mo.k);
  constexpr float iq = 1.0f / 3.0f;

  float s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] = 0.f;
  if (!EXACT) {
    const __half2 iq2 = __float2half2_rn(iq);
    const DeqC dk0 = kdeq(kmm.x, iq2), dk1 = kdeq(kmm.y, iq2);
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t w0 = blk ? kk.y : kk.x, w1 = blk ? kk.w : kk.z;
      const uint32_t w0s = w0 >> 10, w1s = w1 >> 10;
      const uint4 qa = qs.ld2(0, 2 * blk), qb = qs.ld2(0, 2 * blk + 1);
#define KD(W, WS, D, I) wdeq(K2<I>::hi ? WS : W, 0x00030003u << K2<I>::j, mg, D)
      mma_16816(s, KD(w0, w0s, dk0, 0), KD(w1, w1s, dk1, 0), KD(w0, w0s, dk0, 1), KD(w1, w1s, dk1, 1), lo2(qa));
      mma_16816(s2, KD(w0, w0s, dk0, 2), KD(w1, w1s, dk1, 2), KD(w0, w0s, dk0, 3), KD(w1, w1s, dk1, 3), hi2(qa));
      mma_16816(s, KD(w0, w0s, dk0, 4), KD(w1, w1s, dk1, 4), KD(w0, w0s, dk0, 5), KD(w1, w1s, dk1, 5), lo2(qb));
      mma_16816(s2, KD(w0, w0s, dk0, 6), KD(w1, w1s, dk1, 6), KD(w0, w0s, dk0, 7), KD(w1, w1s, dk1, 7), hi2(qb));
#undef KD
    }
    mma_16816(s2, prmt(kmm.x, kmm.x, 0x1010), prmt(kmm.y, kmm.y, 0x1010), 0u, 0u, qs.aug(), 0u);
  } else {
    const __half2 sc0 = __float2half2_rn(meta_scale(kmm.x, iq)), sc1 = __float2half2_rn(meta_scale(kmm.y, iq));
    const __half2 lo0 = u32_as_h2(prmt(kmm.x, kmm.x, 0x1010)), lo1 = u32_as_h2(prmt(kmm.y, kmm.y, 0x1010));
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int blk = ks >> 2, i0 = 2 * (ks & 3), i1 = i0 + 1;
      const uint32_t w0 = blk ? kk.y : kk.x, w1 = blk ? kk.w : kk.z;
      const int j0 = i0 <= 4 ? 2 * i0 : 2 * (i0 - 5), j1 = i1 <= 4 ? 2 * i1 : 2 * (i1 - 5);
      const uint32_t x00 = i0 <= 4 ? w0 : w0 >> 10, x10 = i0 <= 4 ? w1 : w1 >> 10;
      const uint32_t x01 = i1 <= 4 ? w0 : w0 >> 10, x11 = i1 <= 4 ? w1 : w1 >> 10;
      mma_16816(s, edeq(x00, j0, 0x00030003u, sc0, lo0), edeq(x10, j0, 0x00030003u, sc1, lo1),
                edeq(x01, j1, 0x00030003u, sc0, lo0), edeq(x11, j1, 0x00030003u, sc1, lo1), qs.ld(2, ks));
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] += s2[e];
}

template <bool EXACT>
__device__ __forceinline__ void pv_int2(uint32_t sl, const MetaOff& mo, uint32_t mg, WarpState& st, uint32_t bp0, uint32_t bp1) {
  // codes: word g of tokens (2c | 2c+1) lo halves, hi halves, then (2c+8 | 2c+9)
  const uint4 vv = lds128(sl + 512);
  const uint4 vmm = lds128(sl + 1280 + mo.v);  // (lo 2c|2c+1), (hi ...), (lo 2c+8|2c+9), (hi ...)
  constexpr float iq = 1.0f / 3.0f;
  const uint32_t c01lo = vv.x, c01hi = vv.y, c23lo = vv.z, c23hi = vv.w;
  if (!EXACT) {
    const DeqC d01 = vdeq(vmm.x, vmm.y, iq), d23 = vdeq(vmm.z, vmm.w, iq);
    const uint32_t a8 = c01lo >> 8, b8 = c01hi >> 8, e8 = c23lo >> 8, f8 = c23hi >> 8;
    // m-tile mt uses code mt of each 8-code half: j = 2 (mt & 3), from x (mt < 4) or x >> 8
#define PV2(MT)                                                                                     \
  {                                                                                                 \
    constexpr uint32_t m_ = 0x00030003u << (2 * ((MT) & 3));                                       \
    mma_16816(st.acc[MT], wdeq((MT) < 4 ? c01lo : a8, m_, mg, d01), wdeq((MT) < 4 ? c01hi : b8, m_, mg, d01), \
              wdeq((MT) < 4 ? c23lo : e8, m_, mg, d23), wdeq((MT) < 4 ? c23hi : f8, m_, mg, d23), bp0, bp1); \
  }
    PV2(0) PV2(1) PV2(2) PV2(3) PV2(4) PV2(5) PV2(6) PV2(7)
#undef PV2
    lo_mma(st, vmm.x, vmm.z, bp0, bp1);
  } else {
    const __half2 sc01 = exact_sc2(vmm.x, vmm.y, iq), sc23 = exact_sc2(vmm.z, vmm.w, iq);
    const __half2 lo01 = u32_as_h2(vmm.x), lo23 = u32_as_h2(vmm.z);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int j = 2 * (mt & 3);
      const uint32_t x0 = mt < 4 ? c01lo : c01lo >> 8, x1 = mt < 4 ? c01hi : c01hi >> 8;
      const uint32_t x2 = mt < 4 ? c23lo : c23lo >> 8, x3 = mt < 4 ? c23hi : c23hi >> 8;
      mma_16816(st.acc[mt], edeq(x0, j, 0x00030003u, sc01, lo01), edeq(x1, j, 0x00030003u, sc01, lo01),
                edeq(x2, j, 0x00030003u, sc23, lo23), edeq(x3, j, 0x00030003u, sc23, lo23), bp0, bp1);
    }
  }
}

template <bool EXACT>
__device__ __forceinline__ void qk_int4(uint32_t sl, const MetaOff& mo, const QS& qs, uint32_t mg, float (&s)[4]) {
  // group c of tok g / tok g+8, words paired as (lo w0, lo w1), (hi w0, hi w1), (lo w2, lo w3), (hi ...)
  const uint4 kw0 = lds128(sl), kw1 = lds128(sl + 512);
  const uint2 kmm = lds64(sl + 2048 + mo.k);
  constexpr float iq = 1.0f / 15.0f;

  float s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] = 0.f;
  const uint32_t kwa[4] = {kw0.x, kw0.y, kw0.z, kw0.w}, kwb[4] = {kw1.x, kw1.y, kw1.z, kw1.w};
  if (!EXACT) {
    const __half2 iq2 = __float2half2_rn(iq);
    const DeqC dk0 = kdeq(kmm.x, iq2), dk1 = kdeq(kmm.y, iq2);
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      // pairs (d0, d0+8) = (word 2blk code i, word 2blk+1 code i)
      const uint32_t a_lo = kwa[2 * blk], a_hi = kwa[2 * blk + 1];
      const uint32_t b_lo = kwb[2 * blk], b_hi = kwb[2 * blk + 1];
      const uint32_t a_lo8 = a_lo >> 8, a_hi8 = a_hi >> 8, b_lo8 = b_lo >> 8, b_hi8 = b_hi >> 8;
      const uint4 qa = qs.ld2(1, 2 * blk), qb = qs.ld2(1, 2 * blk + 1);
#define KD(X, X8, D, I) wdeq(K4<I>::hi ? X8 : X, 0x000F000Fu << K4<I>::j, mg, D)
      mma_16816(s, KD(a_lo, a_lo8, dk0, 0), KD(b_lo, b_lo8, dk1, 0), KD(a_lo, a_lo8, dk0, 1), KD(b_lo, b_lo8, dk1, 1), lo2(qa));
      mma_16816(s2, KD(a_lo, a_lo8, dk0, 2), KD(b_lo, b_lo8, dk1, 2), KD(a_lo, a_lo8, dk0, 3), KD(b_lo, b_lo8, dk1, 3), hi2(qa));
      mma_16816(s, KD(a_hi, a_hi8, dk0, 0), KD(b_hi, b_hi8, dk1, 0), KD(a_hi, a_hi8, dk0, 1), KD(b_hi, b_hi8, dk1, 1), lo2(qb));
      mma_16816(s2, KD(a_hi, a_hi8, dk0, 2), KD(b_hi, b_hi8, dk1, 2), KD(a_hi, a_hi8, dk0, 3), KD(b_hi, b_hi8, dk1, 3), hi2(qb));
#undef KD
    }
    mma_16816(s2, prmt(kmm.x, kmm.x, 0x1010), prmt(kmm.y, kmm.y, 0x1010), 0u, 0u, qs.aug(), 0u);
  } else {
    const __half2 sc0 = __float2half2_rn(meta_scale(kmm.x, iq)), sc1 = __float2half2_rn(meta_scale(kmm.y, iq));
    const __half2 lo0 = u32_as_h2(prmt(kmm.x, kmm.x, 0x1010)), lo1 = u32_as_h2(prmt(kmm.y, kmm.y, 0x1010));
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t a_lo = kwa[2 * blk], a_hi = kwa[2 * blk + 1];
      const uint32_t b_lo = kwb[2 * blk], b_hi = kwb[2 * blk + 1];
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        const uint32_t ca = q2 < 2 ? a_lo : a_hi, cb = q2 < 2 ? b_lo : b_hi;
        const int i = 2 * (q2 & 1);  // pairs i, i+1 of the 4-pair word
        const uint32_t xa0 = i < 2 ? ca : ca >> 8, xb0 = i < 2 ? cb : cb >> 8;
        const uint32_t xa1 = (i + 1) < 2 ? ca : ca >> 8, xb1 = (i + 1) < 2 ? cb : cb >> 8;
        mma_16816(s, edeq(xa0, 4 * (i & 1), 0x000F000Fu, sc0, lo0), edeq(xb0, 4 * (i & 1), 0x000F000Fu, sc1, lo1),
                  edeq(xa1, 4 * ((i + 1) & 1), 0x000F000Fu, sc0, lo0), edeq(xb1, 4 * ((i + 1) & 1), 0x000F000Fu, sc1, lo1),
                  qs.ld(2, 4 * blk + q2));
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] += s2[e];
}

template <bool EXACT>
__device__ __forceinline__ void pv_int4(uint32_t sl, const MetaOff& mo, uint32_t mg, WarpState& st, uint32_t bp0, uint32_t bp1) {
  // V (tok 2c | 2c+1) and (2c+8 | 2c+9) for d = 16g + mt (word 2g) and 16g + 8 + mt (word 2g+1):
  // (lo w2g), (hi w2g), (lo w2g+1), (hi w2g+1) per token pair
  const uint4 va = lds128(sl + 1024), vb = lds128(sl + 1536);
  const uint4 vmm = lds128(sl + 2304 + mo.v);
  constexpr float iq = 1.0f / 15.0f;
  const uint32_t x01[4] = {va.x, va.y, va.z, va.w};
  const uint32_t x23[4] = {vb.x, vb.y, vb.z, vb.w};
  if (!EXACT) {
    const DeqC d01 = vdeq(vmm.x, vmm.y, iq), d23 = vdeq(vmm.z, vmm.w, iq);
    // m-tile mt: code k = mt & 3 of x[mt >> 2] sits at bits 4k; move it to j = 2k (>> 2k)
#define PV4(MT)                                                                                     \
  {                                                                                                 \
    constexpr int k_ = (MT) & 3, u_ = (MT) >> 2;                                                    \
    constexpr uint32_t m_ = 0x000F000Fu << (2 * k_);                                               \
    mma_16816(st.acc[MT], wdeq(x01[u_] >> (2 * k_), m_, mg, d01), wdeq(x01[2 + u_] >> (2 * k_), m_, mg, d01), \
              wdeq(x23[u_] >> (2 * k_), m_, mg, d23), wdeq(x23[2 + u_] >> (2 * k_), m_, mg, d23), bp0, bp1); \
  }
    PV4(0) PV4(1) PV4(2) PV4(3) PV4(4) PV4(5) PV4(6) PV4(7)
#undef PV4
    lo_mma(st, vmm.x, vmm.z, bp0, bp1);
  } else {
    const __half2 sc01 = exact_sc2(vmm.x, vmm.y, iq), sc23 = exact_sc2(vmm.z, vmm.w, iq);
    const __half2 lo01 = u32_as_h2(vmm.x), lo23 = u32_as_h2(vmm.z);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int k = mt & 3, u = mt >> 2;
      const int j = 4 * (k & 1);
      const uint32_t sh = k < 2 ? 0 : 8;
      mma_16816(st.acc[mt], edeq(x01[u] >> sh, j, 0x000F000Fu, sc01, lo01), edeq(x01[2 + u] >> sh, j, 0x000F000Fu, sc01, lo01),
                edeq(x23[u] >> sh, j, 0x000F000Fu, sc23, lo23), edeq(x23[2 + u] >> sh, j, 0x000F000Fu, sc23, lo23), bp0, bp1);
    }
  }
}

// ---- precise K path (wide-span units) ---------------------------------------------------
// The normal path feeds the tensor cores fp16 values sc*code*2^(j-6), so the score error grows
// with the K group span times |q|.  The precise path feeds the exact magic values
// 16 + code*2^(j-6) instead and applies bias and scale per group in fp32: two MMAs per k-step
// whose B fragments are the tier's q fragments (sets 0 / 1) masked to two groups each
// (column n = (q row n & 3, group 2v + n / 4)), so D holds per-(token, q row, group)
// partial sums  sum_{d in G} q'_d (16 + code_d 2^(j-6)) = 16 Q'_G + (1/f) sum_{d in G} q_d code_d
// (f = the set's fp16(1/qmax) fold), and S = sum_G span_G fp16(1/qmax) (D_G - 16 Q'_G) + lo term.
// A thread holds groups c/2 and 2 + c/2 of q rows (2c)&3, (2c)&3 + 1; lanes c and c^2 hold the
// other two groups.  Needs no shared memory beyond a 128-byte bias table.
// With 5-8 q rows (ROWS8) a second pass over the same raw K operands covers q rows 4-7 (q
// fragments of lane ((g & 3) + 4, c)); lanes c >= 2 keep its sums (their S columns are rows
// 2c, 2c+1), lanes c < 2 the first pass's.
struct PreciseOff {
  int32_t m0, m1;   // byte offsets (from the lane slot `sl`) of the metadata of groups G0, G1
  uint32_t bias;    // shared-memory address of this thread's 16 Q' constants (INT2 tier)
  int32_t qoff;     // q-fragment offset of lane ((g & 3), c) relative to this lane
  int32_t qoff2;    // ... of lane ((g & 3) + 4, c) (q rows 4-7)
  uint32_t msk0, msk1;  // all-ones when this lane's B column takes group c in variant 0 / 1
  bool hi_rows;     // c >= 2: this lane's S columns are q rows 4-7 when m > 4
};
constexpr int kBiasRows = 8;
constexpr int kBiasG = kBiasRows * 4;      // bias table f32 16 Q' [tier][group][q row]
constexpr int kBiasTier = 4 * kBiasG;

__device__ __forceinline__ uint32_t raw_pair(uint32_t x, uint32_t mask, uint32_t magic) {
  return (x & mask) | magic;
}
__device__ __forceinline__ uint2 masked(uint32_t x, uint32_t y, uint32_t m) { return make_uint2(x & m, y & m); }

__device__ __forceinline__ void precise_combine(const float (&P0)[4], const float (&P1)[4], float sc0g,
                                                float sc0g8, float sc1g, float sc1g8,
                                                uint32_t bias_addr, float (&t)[4]) {
  const uint2 b0 = lds64(bias_addr), b1 = lds64(bias_addr + 2 * kBiasG);  // (G0, a..a+1), (G0 + 2, ..)
  const float b0x = __uint_as_float(b0.x), b0y = __uint_as_float(b0.y);
  const float b1x = __uint_as_float(b1.x), b1y = __uint_as_float(b1.y);
  t[0] = fmaf(sc1g, P1[0] - b1x, sc0g * (P0[0] - b0x));
  t[1] = fmaf(sc1g, P1[1] - b1y, sc0g * (P0[1] - b0y));
  t[2] = fmaf(sc1g8, P1[2] - b1x, sc0g8 * (P0[2] - b0x));
  t[3] = fmaf(sc1g8, P1[3] - b1y, sc0g8 * (P0[3] - b0y));
#pragma unroll
  for (int e = 0; e < 4; ++e) t[e] += __shfl_xor_sync(0xffffffffu, t[e], 2);
}

// span * fp16(1/qmax) in fp32 from a (lo, hi) metadata word (matches the fold in the q sets)
__device__ __forceinline__ float precise_scale(uint32_t meta, float inv_q16) {
  const float2 lh = __half22float2(u32_as_h2(meta));
  return (lh.y - lh.x) * inv_q16;
}

template <int BITS, bool ROWS8>
__device__ __forceinline__ void qk_precise(uint32_t sl, const MetaOff& mo, const PreciseOff& po,
                                           const QS& qs, uint32_t mg, float (&s)[4]) {
  constexpr int set = BITS == 2 ? 0 : 1;
  constexpr uint32_t meta_at = BITS == 2 ? 1024 : 2048;
  const float inv_q16 = __half2float(__float2half_rn(BITS == 2 ? 1.0f / 3.0f : 1.0f / 15.0f));
  float P0[4] = {0.f, 0.f, 0.f, 0.f}, P1[4] = {0.f, 0.f, 0.f, 0.f};
  float R0[4] = {0.f, 0.f, 0.f, 0.f}, R1[4] = {0.f, 0.f, 0.f, 0.f};  // q rows 4-7 (ROWS8)
  const uint32_t qsrc = qs.base + po.qoff + set * kQSet;
  const uint32_t qsrc2 = qs.base + po.qoff2 + set * kQSet;
#define PSTEP(X, Y, X2, Y2)                                                        \
  {                                                                                \
    mma_16816(P0, x0, x1, x2, x3, masked(X, Y, po.msk0));                          \
    mma_16816(P1, x0, x1, x2, x3, masked(X, Y, po.msk1));                          \
    if (ROWS8) {                                                                   \
      mma_16816(R0, x0, x1, x2, x3, masked(X2, Y2, po.msk0));                      \
      mma_16816(R1, x0, x1, x2, x3, masked(X2, Y2, po.msk1));                      \
    }                                                                              \
  }
  if (BITS == 2) {
    const uint4 kk = lds128(sl);
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t w0 = blk ? kk.y : kk.x, w1 = blk ? kk.w : kk.z;
      const uint32_t w0s = w0 >> 10, w1s = w1 >> 10;
      const uint4 qa = lds128(qsrc + 512 * (2 * blk)), qb = lds128(qsrc + 512 * (2 * blk + 1));
      uint4 qa2 = qa, qb2 = qb;
      if (ROWS8) {
        qa2 = lds128(qsrc2 + 512 * (2 * blk));
        qb2 = lds128(qsrc2 + 512 * (2 * blk + 1));
      }
#define KR(W, WS, I) raw_pair(K2<I>::hi ? WS : W, 0x00030003u << K2<I>::j, mg)
#define KSTEP(I0, I1, X, Y, X2, Y2)                                                \
      {                                                                          \
        const uint32_t x0 = KR(w0, w0s, I0), x1 = KR(w1, w1s, I0);               \
        const uint32_t x2 = KR(w0, w0s, I1), x3 = KR(w1, w1s, I1);               \
        PSTEP(X, Y, X2, Y2)                                                      \
      }
      KSTEP(0, 1, qa.x, qa.y, qa2.x, qa2.y)
      KSTEP(2, 3, qa.z, qa.w, qa2.z, qa2.w)
      KSTEP(4, 5, qb.x, qb.y, qb2.x, qb2.y)
      KSTEP(6, 7, qb.z, qb.w, qb2.z, qb2.w)
#undef KSTEP
#undef KR
    }
  } else {
    const uint4 kw0 = lds128(sl), kw1 = lds128(sl + 512);
    const uint32_t kwa[4] = {kw0.x, kw0.y, kw0.z, kw0.w}, kwb[4] = {kw1.x, kw1.y, kw1.z, kw1.w};
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t a_lo = kwa[2 * blk], a_hi = kwa[2 * blk + 1];
      const uint32_t b_lo = kwb[2 * blk], b_hi = kwb[2 * blk + 1];
      const uint32_t a_lo8 = a_lo >> 8, a_hi8 = a_hi >> 8, b_lo8 = b_lo >> 8, b_hi8 = b_hi >> 8;
      const uint4 qa = lds128(qsrc + 512 * (2 * blk)), qb = lds128(qsrc + 512 * (2 * blk + 1));
      uint4 qa2 = qa, qb2 = qb;
      if (ROWS8) {
        qa2 = lds128(qsrc2 + 512 * (2 * blk));
        qb2 = lds128(qsrc2 + 512 * (2 * blk + 1));
      }
#define KR(X, X8, I) raw_pair(K4<I>::hi ? X8 : X, 0x000F000Fu << K4<I>::j, mg)
#define KSTEP(XA, XA8, XB, XB8, I0, I1, X, Y, X2, Y2)                              \
      {                                                                          \
        const uint32_t x0 = KR(XA, XA8, I0), x1 = KR(XB, XB8, I0);               \
        const uint32_t x2 = KR(XA, XA8, I1), x3 = KR(XB, XB8, I1);               \
        PSTEP(X, Y, X2, Y2)                                                      \
      }
      KSTEP(a_lo, a_lo8, b_lo, b_lo8, 0, 1, qa.x, qa.y, qa2.x, qa2.y)
      KSTEP(a_lo, a_lo8, b_lo, b_lo8, 2, 3, qa.z, qa.w, qa2.z, qa2.w)
      KSTEP(a_hi, a_hi8, b_hi, b_hi8, 0, 1, qb.x, qb.y, qb2.x, qb2.y)
      KSTEP(a_hi, a_hi8, b_hi, b_hi8, 2, 3, qb.z, qb.w, qb2.z, qb2.w)
#undef KSTEP
#undef KR
    }
  }
#undef PSTEP
  const uint2 m0 = lds64(sl + meta_at + po.m0), m1 = lds64(sl + meta_at + po.m1);
  const float s0g = precise_scale(m0.x, inv_q16), s0g8 = precise_scale(m0.y, inv_q16);
  const float s1g = precise_scale(m1.x, inv_q16), s1g8 = precise_scale(m1.y, inv_q16);
  float t[4];
  precise_combine(P0, P1, s0g, s0g8, s1g, s1g8, po.bias + (BITS == 2 ? 0 : kBiasTier), t);
  if (ROWS8) {
    float t2[4];
    precise_combine(R0, R1, s0g, s0g8, s1g, s1g8, po.bias + (BITS == 2 ? 0 : kBiasTier) + 16, t2);
#pragma unroll
    for (int e = 0; e < 4; ++e) t[e] = po.hi_rows ? t2[e] : t[e];
  }
  const uint2 kmm = lds64(sl + meta_at + mo.k);
  float s2[4] = {0.f, 0.f, 0.f, 0.f};
  mma_16816(s2, prmt(kmm.x, kmm.x, 0x1010), prmt(kmm.y, kmm.y, 0x1010), 0u, 0u, qs.aug(), 0u);
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] = t[e] + s2[e];
}

// ---- FP16 tile straight from global memory (FP16 chunks, tail, decode tokens) ------------
template <bool EXACT>
__device__ __forceinline__ void tile_fp16(const uint16_t* kf, const uint16_t* vf, int valid,
                                          const QS& qs, WarpState& st, int g, int c) {
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int blk = 0; blk < 2; ++blk) {
    // tokens g, g+8; d 32c + 16 blk .. +16 (8 words each)
    const uint4* p0 = reinterpret_cast<const uint4*>(kf + g * kHeadDim + 32 * c + 16 * blk);
    const uint4* p1 = reinterpret_cast<const uint4*>(kf + (g + 8) * kHeadDim + 32 * c + 16 * blk);
    const uint4 x0 = __ldg(p0), x1 = __ldg(p0 + 1), y0 = __ldg(p1), y1 = __ldg(p1 + 1);
    const uint32_t ka[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    const uint32_t kb[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // pair (d0, d0+8), d0 = 16blk + 2kk: words kk and kk+4 of the block
      mma_16816(s, prmt(ka[kk], ka[kk + 4], 0x5410), prmt(kb[kk], kb[kk + 4], 0x5410),
                prmt(ka[kk], ka[kk + 4], 0x7632), prmt(kb[kk], kb[kk + 4], 0x7632), qs.ld(2, 4 * blk + kk));
    }
  }
  if (g >= valid) { s[0] = -INFINITY; s[1] = -INFINITY; }
  if (g + 8 >= valid) { s[2] = -INFINITY; s[3] = -INFINITY; }
  uint32_t bp0, bp1;
  softmax_tile<true>(s, st, bp0, bp1);
  const int toks[4] = {2 * c, 2 * c + 1, 2 * c + 8, 2 * c + 9};
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t w[4][4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint2 a = __ldg(reinterpret_cast<const uint2*>(vf + toks[t] * kHeadDim + 16 * g) + half);
      const uint2 b = __ldg(reinterpret_cast<const uint2*>(vf + toks[t] * kHeadDim + 16 * g + 8) + half);
      w[t][0] = a.x; w[t][1] = a.y; w[t][2] = b.x; w[t][3] = b.y;
    }
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      const int mt = 4 * half + mm;
      const uint32_t sel = (mm & 1) ? 0x7632 : 0x5410;
      const int w0 = mm >> 1, w1 = 2 + (mm >> 1);
      uint32_t a0 = prmt(w[0][w0], w[1][w0], sel), a1 = prmt(w[0][w1], w[1][w1], sel);
      uint32_t a2 = prmt(w[2][w0], w[3][w0], sel), a3 = prmt(w[2][w1], w[3][w1], sel);
      if (!EXACT) {  // match the quantized tiles' m-tile weight 2^(2(mt&3) - 6)
        const __half2 wt = __float2half2_rn((float)(1 << (2 * (mt & 3))) * (1.0f / 64.0f));
        a0 = h2_as_u32(__hmul2(u32_as_h2(a0), wt)); a1 = h2_as_u32(__hmul2(u32_as_h2(a1), wt));
        a2 = h2_as_u32(__hmul2(u32_as_h2(a2), wt)); a3 = h2_as_u32(__hmul2(u32_as_h2(a3), wt));
      }
      mma_16816(st.acc[mt], a0, a1, a2, a3, bp0, bp1);
    }
  }
}

// Per-lane byte offsets (from the interleaved tile buffers' bases, which stay in kernel
// parameters) of tile 0 of this CTA's INT2 / INT4 ranges, + 16 lane.  A tile is one
// contiguous block [K codes | V codes | K meta | V meta] (include/ckv.h), copied verbatim into
// the stage with 16-byte cp.async: 3 per lane (INT2) / 5 (INT4), every one a warp-wide
// contiguous 512-byte run.
struct TileSrc {
  int64_t c2, c4;
};

// Warp-wide: stage tile t (< n) of one kind's range (tile 0 at `base`) into the stage whose lane slot is `sl`.
// Commits a (possibly empty) group.  The INT2 and INT4 ranges run as separate phases, so
// every issue is of a known kind: one address and 3 / 5 copies, nothing predicated off.
template <int BITS>
__device__ __forceinline__ const char* tile_base(const DecArgs& a, const TileSrc& o) {
  return BITS == 2 ? reinterpret_cast<const char*>(a.K.codes2) + o.c2 : reinterpret_cast<const char*>(a.K.codes4) + o.c4;
}
template <int BITS>
__device__ __forceinline__ void issue_at(int t, int n, const char* base, uint32_t sl) {
  if (t < n) {
    const char* p = base + (int64_t)t * (BITS == 2 ? kBlock2 : kBlock4);
    cp_async16(sl, p);
    cp_async16(sl + 512, p + 512);
    cp_async16(sl + 1024, p + 1024);
    if (BITS == 4) {
      cp_async16(sl + 1536, p + 1536);
      cp_async16(sl + 2048, p + 2048);
    }
  }
  cp_commit();
}

// Prologue of a phase: put this warp's first kStages-1 tiles of the range in flight.
template <int BITS>
__device__ __forceinline__ void prologue(int n, const DecArgs& a, const TileSrc& src, uint32_t ring_l, int warp,
                                         int stride = kDecWarps) {
  const char* base = tile_base<BITS>(a, src);
#pragma unroll
  for (int s = 0; s < Ring<BITS>::stages - 1; ++s) issue_at<BITS>(warp + stride * s, n, base, ring_l + s * Ring<BITS>::bytes);
}

// decode modes of a unit: normal; precise K (wide span x |q|; m <= 4, or m <= 8 in two passes);
// exact (scales or q
// too wide for the fp16-weighted forms)
constexpr int kModeNormal = 0, kModePrecise = 1, kModeExact = 2, kModePrecise8 = 3;

template <int MODE>
__device__ __forceinline__ void qk2(uint32_t sl, const MetaOff& mo, const PreciseOff& po, const QS& qs, uint32_t mg, float (&s)[4]) {
  if (MODE == kModePrecise || MODE == kModePrecise8) qk_precise<2, MODE == kModePrecise8>(sl, mo, po, qs, mg, s);
  else qk_int2<MODE == kModeExact>(sl, mo, qs, mg, s);
}
template <int MODE>
__device__ __forceinline__ void qk4(uint32_t sl, const MetaOff& mo, const PreciseOff& po, const QS& qs, uint32_t mg, float (&s)[4]) {
  if (MODE == kModePrecise || MODE == kModePrecise8) qk_precise<4, MODE == kModePrecise8>(sl, mo, po, qs, mg, s);
  else qk_int4<MODE == kModeExact>(sl, mo, qs, mg, s);
}
// The tile loop of one warp over one kind's range [0, n) (tiles warp, warp + 4, ...) through
// the cp.async ring (prologue already issued), software-pipelined so that q.K^T of tile i+1
// and P.V of tile i form one straight-line block (independent MMA chains the scheduler can
// interleave).
template <int MODE, int BITS>
__device__ __forceinline__ void run_tiles(int n, const DecArgs& a, const TileSrc& src, const MetaOff& mo,
                                          const PreciseOff& po, uint32_t ring_l, const QS& qs, uint32_t mg,
                                          WarpState& st, int warp, int stride = kDecWarps) {
  constexpr bool EXACT = MODE == kModeExact;
  constexpr int kStages = Ring<BITS>::stages, kStageBytes = Ring<BITS>::bytes;
  const uint32_t ring_end = ring_l + kStages * kStageBytes;
  auto next = [&](uint32_t x) { return x + kStageBytes == ring_end ? ring_l : x + kStageBytes; };
  int t = warp;
  const int64_t kStep = (int64_t)stride * (BITS == 2 ? kBlock2 : kBlock4);
  // address of the next tile to issue (kStages-1 ahead of the one consumed), advanced by one
  // warp stride per iteration: a loop-carried pointer instead of base + t * block each time
  const char* pn = tile_base<BITS>(a, src) + (int64_t)(warp + stride * (kStages - 1)) * (BITS == 2 ? kBlock2 : kBlock4);
  if (t < n) {
    uint32_t cur = ring_l, put = ring_l + (kStages - 1) * kStageBytes;
    cp_wait<kStages - 2>();
    __syncwarp();
    float s0[4];
    if (BITS == 2) qk2<MODE>(cur, mo, po, qs, mg, s0);
    else qk4<MODE>(cur, mo, po, qs, mg, s0);
    uint32_t bp0, bp1;
    softmax_tile<EXACT>(s0, st, bp0, bp1);
    while (true) {
      const int tn = t + stride;
      issue_at<BITS>(t + stride * (kStages - 1) < n ? 0 : 1, 1, pn, put);
      pn += kStep;
      if (tn >= n) {
        if (BITS == 2) pv_int2<EXACT>(cur, mo, mg, st, bp0, bp1);
        else pv_int4<EXACT>(cur, mo, mg, st, bp0, bp1);
        break;
      }
      cp_wait<kStages - 2>();
      __syncwarp();
      const uint32_t nx = next(cur);
      float sn[4];
      if (BITS == 2) {
        qk2<MODE>(nx, mo, po, qs, mg, sn);
        pv_int2<EXACT>(cur, mo, mg, st, bp0, bp1);
      } else {
        qk4<MODE>(nx, mo, po, qs, mg, sn);
        pv_int4<EXACT>(cur, mo, mg, st, bp0, bp1);
      }
      __syncwarp();  // slot `cur` may be refilled from now on
      softmax_tile<EXACT>(sn, st, bp0, bp1);
      put = cur;  // the refill slot trails the consumed one by a full ring (kStages - 1 ahead)
      cur = nx;
      t = tn;
    }
  }
  cp_wait<0>();
}

// Both phases of a CTA's quantized tiles: INT2 (its prologue issued before the PDL wait), then
// INT4 (prologue here, or before the wait when the CTA has no INT2 tiles).
__device__ __forceinline__ int rotate(int warp, int done, int stride) {  // (warp - done) mod stride
  const int r = (warp - done) % stride;
  return r < 0 ? r + stride : r;
}

template <int MODE>
__device__ __forceinline__ void quantized_tiles(int n2, int n4, const DecArgs& a, const TileSrc& src,
                                                const MetaOff& mo, const PreciseOff& po, uint32_t ring_l,
                                                const QS& qs, uint32_t mg, WarpState& st, int warp,
                                                int stride = kDecWarps) {
  // the INT4 phase starts at the warp after the one that took the last INT2 tile, so every
  // warp's tile count over both phases is within one of the others' (the CTA's warps meet at
  // the merge barrier)
  const int w4 = rotate(warp, n2, stride);
  if (n2 > 0) {
    run_tiles<MODE, 2>(n2, a, src, mo, po, ring_l, qs, mg, st, warp, stride);
    if (n4 > 0) {
      __syncwarp();
      prologue<4>(n4, a, src, ring_l, w4, stride);
    }
  }
  if (n4 > 0) run_tiles<MODE, 4>(n4, a, src, mo, po, ring_l, qs, mg, st, w4, stride);
}

// This CTA's share of its unit's FP16-region tiles (FP16-tier chunks, tail, decode tokens),
// interleaved over the warps; pointers and ranges re-derived here (len_fp may have grown by
// decode appends: read after the programmatic-dependent-launch wait).
template <bool EXACT>
__device__ __forceinline__ void fp16_tiles(const DecArgs& a, const QS& qs, WarpState& st, int nq) {
  // thread coordinates re-read here (volatile): values carried from the kernel's start would be
  // spilled across the tile loop and reloaded in every iteration of this one
  uint32_t tid;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
  const int warp = (int)(tid >> 5), g = (int)((tid & 31) >> 2), c = (int)(tid & 3);
  const CtaIds id = cta_ids(a.Bc, a.b0);
  const int off_fp = reinterpret_cast<const int*>(a.seq)[8 * id.b + 4];
  const int len_fp = reinterpret_cast<const int*>(a.seq)[8 * id.b + 5];
  const int nft = (len_fp + kTile - 1) / kTile;
  const int f_begin = (int)((int64_t)nft * id.split / a.splits);
  const int f_end = (int)((int64_t)nft * (id.split + 1) / a.splits);
  const int64_t unit = (int64_t)id.l * a.H + id.h;
  const uint16_t* kf = a.K.fp + (unit * a.K.rows_fp + off_fp) * kHeadDim;
  const uint16_t* vf = a.V.fp + (unit * a.V.rows_fp + off_fp) * kHeadDim;
  // continue the quantized phases' rotation over the warps (nq quantized tiles before)
  for (int tf = f_begin + ((warp - nq) & (kDecWarps - 1)); tf < f_end; tf += kDecWarps) {
    const int r = tf * kTile;
    tile_fp16<EXACT>(kf + (int64_t)r * kHeadDim, vf + (int64_t)r * kHeadDim, len_fp - r, qs, st, g, c);
  }
}

// ---- q staging (shared by both decode kernels) -----------------------------------------
// q row `row` (zero if >= m) of unit (l, b, h), lane's 32 columns 32c.., scaled to log2 units
// and rounded to the fp16 MMA operand.
__device__ __forceinline__ void load_q_rows(const DecArgs& a, int l, int b, int h, int row, int c, float (&qv)[32]) {
  const uint16_t* qrow = a.q + l * a.q_sl + b * a.q_sb + (int64_t)(h * a.m + row) * kHeadDim + 32 * c;
  if (row < a.m) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint4 x = reinterpret_cast<const uint4*>(qrow)[u];
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(u32_as_h2(w[e]));
        qv[8 * u + 2 * e] = __half2float(__float2half_rn(f.x * a.scale_log2));  // the fp16 MMA operand
        qv[8 * u + 2 * e + 1] = __half2float(__float2half_rn(f.y * a.scale_log2));
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e) qv[e] = 0.f;
  }
}

// decode mode of a unit from its q (the warp's 8 rows) and its span bounds
__device__ __forceinline__ int unit_mode(const DecArgs& a, const float (&qv)[32], bool span_wide, float kspan) {
  float qmaxabs = 0.f;
#pragma unroll
  for (int e = 0; e < 32; ++e) qmaxabs = fmaxf(qmaxabs, fabsf(qv[e]));
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) qmaxabs = fmaxf(qmaxabs, __shfl_xor_sync(0xffffffffu, qmaxabs, o));
  const bool wide = qmaxabs > kWideQ || span_wide;
  return wide ? kModeExact
              : (kspan * qmaxabs > kPreciseSpanQ ? (a.m <= 4 ? kModePrecise : kModePrecise8) : kModeNormal);
}

// Part `part` of a unit's q staging into s_qu (kQBytes) / s_biasu: 0-2 the q-fragment sets
// (0: INT2 slot weights, 1: INT4, 2: unweighted; parts 0/1 also the precise-mode bias), 3 the
// zero-point entry.
__device__ __forceinline__ void stage_q_part(const DecArgs& a, const float (&qv)[32], int part, unsigned char* s_qu,
                                             float* s_biasu, int lane) {
  const int g = lane >> 2, c = lane & 3;
  // slot weights 2^(6-j) of K pair i: INT2 j = 2i (i <= 4) or 2(i-5); INT4 j = 4(i & 1)
  auto slot_w = [&](int set, int i) {
    return set == 0 ? exp2f((float)(6 - (i <= 4 ? 2 * i : 2 * (i - 5))))
                    : (set == 1 ? exp2f((float)(6 - 4 * (i & 1))) : 1.0f);
  };
  if (part < 3) {
    float qsw = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int i0 = 2 * (ks & 3), i1 = i0 + 1;  // K pair index inside the 16-d block
      const int d0 = 16 * (ks >> 2) + i0;        // lane-local index within group c
      // INT2 / INT4 sets also carry the fold of the fp16(1/qmax) rounding (see kdeq)
      const float fold = part == 0 ? kscale_fold(1.0f / 3.0f) : (part == 1 ? kscale_fold(1.0f / 15.0f) : 1.0f);
      const float x0 = slot_w(part, i0) * fold, x1 = slot_w(part, i1) * fold;
      const __half2 lo = __floats2half2_rn(qv[d0] * x0, qv[d0 + 8] * x0);
      const __half2 hi = __floats2half2_rn(qv[d0 + 1] * x1, qv[d0 + 9] * x1);
      reinterpret_cast<uint2*>(s_qu + part * kQSet + 512 * (ks >> 1) + 16 * lane)[ks & 1] =
          make_uint2(h2_as_u32(lo), h2_as_u32(hi));
      const float2 fl = __half22float2(lo), fh = __half22float2(hi);
      qsw += (fl.x + fl.y) + (fh.x + fh.y);
    }
    // precise-mode bias 16 Q'[tier][group c][q row g]: the sum of exactly the fp16 weighted
    // values this lane's B fragments hold
    if (part < 2) s_biasu[part * 4 * kBiasRows + c * kBiasRows + g] = 16.0f * qsw;
  } else {
    float qsum = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e) qsum += qv[e];
    const __half qhi = __float2half_rn(qsum);
    const __half qlo = __float2half_rn(qsum - __half2float(qhi));
    reinterpret_cast<uint32_t*>(s_qu + 3 * kQSet)[lane] = h2_as_u32(__halves2half2(qhi, qlo));
  }
}

__global__ void __launch_bounds__(kDecWarps * 32, kMinCtas) decode_kernel(const DecArgs a) {
  extern __shared__ __align__(128) unsigned char s_dyn[];  // ring: [warp][kWarpRing]
  unsigned char (*s_ring)[kWarpRing] = reinterpret_cast<unsigned char (*)[kWarpRing]>(s_dyn);
  __shared__ float s_ml[kDecWarps][8][2];
  __shared__ __align__(16) unsigned char s_q[kQBytes];
  __shared__ int s_last;
  __shared__ __align__(16) float s_bias[2 * 4 * kBiasRows];  // precise modes: 16 Q' [tier][group][q row]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  __shared__ int64_t s_tr[12], s_tend[kDecWarps];
  if (threadIdx.x == 0 && tracing()) { s_tr[0] = gtime(); s_tr[11] = 0; }
  // Segment lengths of the quantized arenas are immutable after the build; len_fp grows with
  // decode appends and is read only after the programmatic-dependent-launch wait below.
  // Split of the quantized tiles: every CTA takes the same 1/splits share of the INT2 tiles
  // AND of the INT4 tiles (and of the FP16-region tiles, fp16_tiles), so all CTAs carry the
  // same mix and finish together whatever the relative per-tile costs are.
  int cnt2, nloc;
  TileSrc src;  // tile-native arenas: a row range starting at a tile is contiguous bytes
  {
    const CtaIds id = cta_ids(a.Bc, a.b0);
    const int4 s0 = reinterpret_cast<const int4*>(a.seq)[2 * id.b];
    const int n2t = s0.y / kTile, n4t = s0.w / kTile;
    const int a2 = (int)((int64_t)n2t * id.split / a.splits), b2 = (int)((int64_t)n2t * (id.split + 1) / a.splits);
    const int a4 = (int)((int64_t)n4t * id.split / a.splits), b4 = (int)((int64_t)n4t * (id.split + 1) / a.splits);
    cnt2 = b2 - a2;  // INT2 tiles [0, cnt2) of this CTA, then INT4 tiles [0, nloc - cnt2)
    nloc = cnt2 + (b4 - a4);
    const int64_t unit = (int64_t)id.l * a.H + id.h;
    const int64_t r2 = s0.x + (int64_t)a2 * kTile, r4 = s0.z + (int64_t)a4 * kTile;  // first rows
    src.c2 = (unit * a.K.rows2 + r2) / kTileRows * kBlock2 + 16 * lane;
    src.c4 = (unit * a.K.rows4 + r4) / kTileRows * kBlock4 + 16 * lane;
  }
  MetaOff mo;
  mo.k = -8 * lane;
  mo.v = 16 * ((g >> 1) * 4 + c) - 16 * lane;
  const uint32_t ring_l = (uint32_t)__cvta_generic_to_shared(&s_ring[warp][0]) + 16 * lane;
  if (cnt2 > 0) prologue<2>(cnt2, a, src, ring_l, warp);
  else prologue<4>(nloc, a, src, ring_l, warp);

  // Everything above touched only build-time data.  q, the FP16 region and len_fp may come
  // from the preceding kernel on the stream: wait for it (no-op without PDL), and let the next
  // decode launch (next layer) start its own prologue as soon as SMs free up.
  // the unit's span bounds are build-time data too: read them before the wait
  bool span_wide;
  float kspan;
  {
    const CtaIds id = cta_ids(a.Bc, a.b0);
    const int64_t fidx = ((int64_t)id.l * a.H + id.h) * a.B + id.b;  // span flags are [L][H][B]
    span_wide = (a.K.span_flags != nullptr && a.K.span_flags[fidx] != 0u) ||
                (a.V.span_flags != nullptr && a.V.span_flags[fidx] != 0u);
    kspan = a.K.span_max != nullptr ? __uint_as_float(a.K.span_max[fidx]) : 0.f;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0 && tracing()) s_tr[1] = gtime();

  // Q B-fragments (scaled to log2 units), q-row i = g (zero if g >= m).  Every warp loads the
  // same 8 rows and derives the unit's mode from max |q| and the K span bound; then warps 0-2
  // write q-fragment sets 0-2 (precise mode: the group-masked INT2 / INT4 sets and their 16 Q'
  // bias constants instead of sets 0 and 1), warp 3 the zero-point entry.
  int mode;
  {
    const CtaIds id = cta_ids(a.Bc, a.b0);
    float qv[32];
    load_q_rows(a, id.l, id.b, id.h, g, c, qv);
    mode = unit_mode(a, qv, span_wide, kspan);
    stage_q_part(a, qv, warp < 3 ? warp : 3, s_q, s_bias, lane);
  }
  __syncthreads();
  if (threadIdx.x == 0 && tracing()) s_tr[2] = gtime();
  QS qs;
  qs.base = (uint32_t)__cvta_generic_to_shared(s_q) + 16 * lane;
  qs.aug_addr = (uint32_t)__cvta_generic_to_shared(s_q) + 3 * kQSet + 4 * lane;
  PreciseOff po;
  {
    const int G0 = c >> 1, qa = (2 * c) & 3;
    po.m0 = (g * 4 + G0) * 8 - 16 * lane;
    po.m1 = (g * 4 + G0 + 2) * 8 - 16 * lane;
    po.bias = (uint32_t)__cvta_generic_to_shared(s_bias) + (G0 * kBiasRows + qa) * 4;
    po.qoff = 16 * (((g & 3) * 4 + c) - lane);
    po.qoff2 = 16 * ((((g & 3) + 4) * 4 + c) - lane);
    po.hi_rows = c >= 2;
    const bool in = (g >> 2) == (c & 1);  // column g takes group c (variant c / 2)
    po.msk0 = in && (c >> 1) == 0 ? 0xffffffffu : 0u;
    po.msk1 = in && (c >> 1) == 1 ? 0xffffffffu : 0u;
  }
  const uint32_t mg = kMagic16 | a.zero;

  WarpState st;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) st.acc[mt][0] = st.acc[mt][1] = st.acc[mt][2] = st.acc[mt][3] = 0.f;
  st.lacc[0] = st.lacc[1] = 0.f;
  st.lsq[0] = st.lsq[1] = 0.f;
  st.mrun[0] = st.mrun[1] = -INFINITY;
  st.lsum[0] = st.lsum[1] = 0.f;

  if (mode == kModeExact) {
    quantized_tiles<kModeExact>(cnt2, nloc - cnt2, a, src, mo, po, ring_l, qs, mg, st, warp);
    fp16_tiles<true>(a, qs, st, nloc);
  } else {
    if (mode == kModePrecise) quantized_tiles<kModePrecise>(cnt2, nloc - cnt2, a, src, mo, po, ring_l, qs, mg, st, warp);
    else if (mode == kModePrecise8) quantized_tiles<kModePrecise8>(cnt2, nloc - cnt2, a, src, mo, po, ring_l, qs, mg, st, warp);
    else quantized_tiles<kModeNormal>(cnt2, nloc - cnt2, a, src, mo, po, ring_l, qs, mg, st, warp);
    fp16_tiles<false>(a, qs, st, nloc);
    // undo the V m-tile weights 2^(2(mt&3) - 6)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const float f = (float)(64 >> (2 * (mt & 3)));
      st.acc[mt][0] *= f; st.acc[mt][1] *= f; st.acc[mt][2] *= f; st.acc[mt][3] *= f;
    }
  }

  if (lane == 0 && tracing()) s_tend[warp] = gtime();
  // finish the warp: fold the zero-point term, reduce row sums over the 8 row-groups
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
  st.lsum[0] += st.lsq[0];  // already summed over the 16 tokens of every tile
  st.lsum[1] += st.lsq[1];
  __syncthreads();  // ring -> merge buffer reuse
  if (threadIdx.x == 0 && tracing()) s_tr[8] = gtime();
  float (*s_acc)[8][kHeadDim] = reinterpret_cast<float (*)[8][kHeadDim]>(&s_ring[0][0]);
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
  const CtaIds id = cta_ids(a.Bc, a.b0);
  const int split = id.split, h = id.h, l = id.l, b = id.b;
  const int d = threadIdx.x;
  const int hq0 = h * a.m;
  const int Hq = a.H * a.m;
  for (int qi = 0; qi < a.m; ++qi) {
    float ms = -INFINITY;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) ms = fmaxf(ms, s_ml[w][qi][0]);
    float acc = 0.f, lsum = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) {
      const float mw = s_ml[w][qi][0];
      const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
      acc += f * s_acc[w][qi][d];
      lsum += f * s_ml[w][qi][1];
    }
    const int64_t row = ((int64_t)l * a.B + b) * Hq + hq0 + qi;
    if (a.splits == 1) {
      if (a.partial_out) {
        float* dst = a.partial_out + row * kPartStride;
        dst[d] = acc;
        if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
      } else {
        a.out[l * a.o_sl + b * a.o_sb + (int64_t)(hq0 + qi) * kHeadDim + d] =
            __half_as_ushort(__float2half_rn(acc / lsum));
      }
    } else {
      float* dst = a.ws + (row * a.splits + split) * kWsStride;
      dst[d] = acc;
      if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
    }
  }
  auto trace_out = [&]() {
    if (threadIdx.x == 0 && tracing()) {
      s_tr[3] = s_tend[0];
      s_tr[4] = gtime();
      int64_t* dst = g_trace + 16 * atomicAdd(&g_trace_n, 1ull);
      for (int i = 0; i < 5; ++i) dst[i] = s_tr[i];
      for (int i = 8; i < 12; ++i) dst[i] = s_tr[i];
      for (int i = 0; i < kDecWarps; ++i) dst[12 + i] = s_tend[i];
      // launch position | split << 20 | (sequence * H + kv head) << 40
      dst[5] = smid();
      dst[6] = (int64_t)((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) | ((int64_t)split << 20) |
               ((int64_t)(b * a.H + h) << 40);
      dst[7] = (int64_t)a.q;
    }
  };
  if (a.splits == 1) { trace_out(); return; }
  // split-KV: the last CTA of this unit to arrive merges all partials (in-launch, no 2nd
  // kernel).  The CTA barrier orders every thread's partial stores before thread 0's
  // device-scope release RMW; the acquiring side sees them after its own barrier.
  __syncthreads();
  if (threadIdx.x == 0 && tracing()) s_tr[9] = gtime();
  if (threadIdx.x == 0) {
    cuda::atomic_ref<uint32_t, cuda::thread_scope_device> ctr(a.counters[((int64_t)l * a.B + b) * a.H + h]);
    const uint32_t prev = ctr.fetch_add(1u, cuda::memory_order_acq_rel);
    s_last = prev == (uint32_t)(a.splits - 1);
    if (s_last) ctr.store(0u, cuda::memory_order_relaxed);  // ready for the next launch
  }
  __syncthreads();
  if (threadIdx.x == 0 && tracing()) { s_tr[10] = gtime(); s_tr[11] = s_last; }
  if (!s_last) { trace_out(); return; }
  // All m x splits partial rows of this unit are contiguous in the workspace: stage them in
  // shared memory with every 16-B copy in flight at once (one L2 round trip), then merge.
  const int64_t row0 = ((int64_t)l * a.B + b) * Hq + hq0;
  const float* p0 = a.ws + row0 * a.splits * kWsStride;
  const int nrows = a.m * a.splits;
  float* s_part = reinterpret_cast<float*>(&s_ring[0][0]);
  if ((nrows * (kWsStride + 1) + 2 * a.m) * (int)sizeof(float) <= kDynSmem) {
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_part);
    const int nvec = nrows * kWsStride / 4;
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) cp_async16(sbase + 16 * i, p0 + 4 * i);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  } else {
    s_part = nullptr;
  }
  if (s_part != nullptr && nrows <= (int)blockDim.x) {
    // weights first, one thread per partial row: w = 2^(m_row - max over the q row's splits),
    // then each thread (d) sums every q row's splits independently (no serial max pass per d)
    float* s_w = s_part + nrows * kWsStride;  // [nrows] weights, then [m] (max, sum) pairs
    float* s_ml2 = s_w + nrows;
    const int r = threadIdx.x;
    if (r < nrows) {
      const float* pq = s_part + (r / a.splits) * a.splits * kWsStride;
      float ms = -INFINITY;
      for (int s = 0; s < a.splits; ++s) ms = fmaxf(ms, pq[s * kWsStride + kHeadDim]);
      const float mw = s_part[r * kWsStride + kHeadDim];
      const float w = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
      s_w[r] = w;
      if (r % a.splits == 0) s_ml2[2 * (r / a.splits)] = ms;
    }
    __syncthreads();
    if (r < a.m) {
      float lsum = 0.f;
      for (int s = 0; s < a.splits; ++s) lsum += s_w[r * a.splits + s] * s_part[(r * a.splits + s) * kWsStride + kHeadDim + 1];
      s_ml2[2 * r + 1] = lsum;
    }
    __syncthreads();
    for (int qi = 0; qi < a.m; ++qi) {
      const float* pq = s_part + qi * a.splits * kWsStride + d;
      const float* wq = s_w + qi * a.splits;
      float acc = 0.f;
      for (int s = 0; s < a.splits; ++s) acc += wq[s] * pq[s * kWsStride];
      const int64_t row = row0 + qi;
      if (a.partial_out) {
        float* dst = a.partial_out + row * kPartStride;
        dst[d] = acc;
        if (d == 0) { dst[kHeadDim] = s_ml2[2 * qi]; dst[kHeadDim + 1] = s_ml2[2 * qi + 1]; }
      } else {
        a.out[l * a.o_sl + b * a.o_sb + (int64_t)(hq0 + qi) * kHeadDim + d] =
            __half_as_ushort(__float2half_rn(acc / s_ml2[2 * qi + 1]));
      }
    }
    trace_out();
    return;
  }
  for (int qi = 0; qi < a.m; ++qi) {
    const int64_t row = row0 + qi;
    const float* p = s_part ? s_part + qi * a.splits * kWsStride : a.ws + row * a.splits * kWsStride;
    float ms = -INFINITY, acc = 0.f, lsum = 0.f;
    for (int s = 0; s < a.splits; ++s) ms = fmaxf(ms, p[s * kWsStride + kHeadDim]);
    for (int s = 0; s < a.splits; ++s) {
      const float mw = p[s * kWsStride + kHeadDim];
      const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
      acc += f * p[s * kWsStride + d];
      lsum += f * p[s * kWsStride + kHeadDim + 1];
    }
    if (a.partial_out) {
      float* dst = a.partial_out + row * kPartStride;
      dst[d] = acc;
      if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
    } else {
      a.out[l * a.o_sl + b * a.o_sb + (int64_t)(hq0 + qi) * kHeadDim + d] =
          __half_as_ushort(__float2half_rn(acc / lsum));
    }
  }
  trace_out();
}

// ---- warp-plan decode (one 16-warp CTA per SM) -------------------------------------------
// The layer's (sequence, kv head) units are split at WARP granularity: unit u gets n_u warps
// (host plan, proportional to its tile cost, sum = 16 x SMs), the global warp list is
// unit-major and CTA c runs warps [16c, 16c + 16) — one CTA per SM, so there are no co-resident
// CTAs whose scheduling priorities differ (with 4 CTAs per SM the late-launched ones run up to
// ~30% slower and set the layer's tail).  Every warp carries the same mix of tile kinds.  A CTA spans a few units: q is staged per unit, the warps of a unit merge in shared
// memory, and a unit split over several CTAs merges their partials in the last one to arrive.
// Each CTA's part of a unit is a contiguous share of the unit's tiles of each kind, in
// proportion to the part's warps (adjacent tiles stream through one SM).
#ifndef CKV_WP_WARPS
#define CKV_WP_WARPS 16
#endif
constexpr int kWpWarps = CKV_WP_WARPS;  // warps per CTA; 16 / kWpWarps CTAs per SM

struct WpArgs {
  DecArgs d;
  const int32_t* prefix;  // [U + 1] first global warp of each unit (U = B * H per layer),
                          // then [16 * ctas] the unit of every global warp
  int U;
  int max_slots;          // most units any CTA spans (q staging slots)
  int max_ctas;           // most CTAs any unit spans (partial slots per unit)
};

__device__ __forceinline__ int wp_unit_of(const int32_t* prefix, int U, int gw) {  // prefix[u] <= gw < prefix[u+1]
  int lo = 0, hi = U - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(prefix + mid) <= gw) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kWpWarps * 32, 16 / kWpWarps) decode_wp_kernel(const WpArgs w) {
  const DecArgs& a = w.d;
  extern __shared__ __align__(128) unsigned char s_dyn[];  // ring [16][kWarpRing] | q sets [slots][kQBytes]
  unsigned char (*s_ring)[kWarpRing] = reinterpret_cast<unsigned char (*)[kWarpRing]>(s_dyn);
  unsigned char* s_qall = s_dyn + kWpWarps * kWarpRing;
  __shared__ float s_ml[kWpWarps][8][2];
  __shared__ __align__(16) float s_biasall[8][2 * 4 * kBiasRows];
  __shared__ int s_lastu[8];
  __shared__ int4 s_slot[8];             // per unit slot: warps [x, y) of this CTA, first / last CTA of the unit
  __shared__ unsigned short s_rtab[64];  // merge row r -> (slot << 8 | q row)
  __shared__ int64_t s_tr[12], s_tend[kWpWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int cta = blockIdx.x, l = blockIdx.z;
  if (threadIdx.x == 0 && tracing()) { s_tr[0] = gtime(); s_tr[11] = 0; }
  const int gw = cta * kWpWarps + warp;
  const int32_t* wunit = w.prefix + w.U + 1;  // unit of every global warp (one load, no search)
  const int u = __ldg(wunit + gw);
  const int u0 = __ldg(wunit + cta * kWpWarps);
  const int p0 = __ldg(w.prefix + u), p1 = __ldg(w.prefix + u + 1);
  const int nw = p1 - p0;  // the unit's warps
  // this CTA's part of the unit: its warps [w_lo, w_hi) of the unit take a contiguous share of
  // each tile kind (adjacent tiles on one SM, as the 4-warp kernel's CTAs), interleaved inside
  const int w_lo = max(p0, cta * kWpWarps) - p0, w_hi = min(p1, cta * kWpWarps + kWpWarps) - p0;
  const int k = gw - p0 - w_lo, np = w_hi - w_lo;  // this warp's index among the part's np warps
  const int slot = u - u0;
  const int b = u / a.H, h = u % a.H;
  int n2t, n4t;
  TileSrc src;
  {
    const int4 s0 = reinterpret_cast<const int4*>(a.seq)[2 * b];
    const int n2u = s0.y / kTile, n4u = s0.w / kTile;
    const int a2 = (int)((int64_t)n2u * w_lo / nw), a4 = (int)((int64_t)n4u * w_lo / nw);
    n2t = (int)((int64_t)n2u * w_hi / nw) - a2;
    n4t = (int)((int64_t)n4u * w_hi / nw) - a4;
    const int64_t unit = (int64_t)l * a.H + h;
    src.c2 = (unit * a.K.rows2 + s0.x + (int64_t)a2 * kTile) / kTileRows * kBlock2 + 16 * lane;
    src.c4 = (unit * a.K.rows4 + s0.z + (int64_t)a4 * kTile) / kTileRows * kBlock4 + 16 * lane;
  }
  MetaOff mo;
  mo.k = -8 * lane;
  mo.v = 16 * ((g >> 1) * 4 + c) - 16 * lane;
  const uint32_t ring_l = (uint32_t)__cvta_generic_to_shared(&s_ring[warp][0]) + 16 * lane;
  if (n2t > 0) prologue<2>(n2t, a, src, ring_l, k, np);
  else prologue<4>(n4t, a, src, ring_l, k, np);
  bool span_wide;
  float kspan;
  {
    const int64_t fidx = ((int64_t)l * a.H + h) * a.B + b;  // span flags are [L][H][B]
    span_wide = (a.K.span_flags != nullptr && a.K.span_flags[fidx] != 0u) ||
                (a.V.span_flags != nullptr && a.V.span_flags[fidx] != 0u);
    kspan = a.K.span_max != nullptr ? __uint_as_float(a.K.span_max[fidx]) : 0.f;
  }
  // per-slot facts for the merge (build-time plan data: before the wait)
  const int u_last = __ldg(wunit + cta * kWpWarps + kWpWarps - 1);
  const int nslots = u_last - u0 + 1;
  if ((int)threadIdx.x < nslots) {
    const int us = u0 + threadIdx.x;
    const int q0 = __ldg(w.prefix + us), q1 = __ldg(w.prefix + us + 1);
    s_slot[threadIdx.x] = make_int4(max(q0, cta * kWpWarps) - cta * kWpWarps,
                                    min(q1, cta * kWpWarps + kWpWarps) - cta * kWpWarps, q0 / kWpWarps,
                                    (q1 - 1) / kWpWarps);
  }
  if ((int)threadIdx.x < nslots * a.m)
    s_rtab[threadIdx.x] = (unsigned short)(((threadIdx.x / a.m) << 8) | (threadIdx.x % a.m));
  // pull this warp's q rows into L2 while the previous launch drains (L2 is the point of
  // coherence: a producer writing q before the wait below still wins; a prefetch reads nothing
  // into this SM)
  if (g < a.m) {
    const uint16_t* qrow = a.q + l * a.q_sl + b * a.q_sb + (int64_t)(h * a.m + g) * kHeadDim + 32 * c;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow));
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0 && tracing()) s_tr[1] = gtime();

  // q staging: every unit slot of the CTA needs parts 0-3; the warps share the jobs
  int mode;
  {
    float qv[32];
    load_q_rows(a, l, b, h, g, c, qv);  // this warp's unit: its mode (and its staging jobs)
    mode = unit_mode(a, qv, span_wide, kspan);
    for (int j = warp; j < 4 * nslots; j += kWpWarps) {
      const int uj = u0 + (j >> 2);
      if (uj == u) {
        stage_q_part(a, qv, j & 3, s_qall + (j >> 2) * kQBytes, s_biasall[j >> 2], lane);
      } else {
        float qj[32];
        load_q_rows(a, l, uj / a.H, uj % a.H, g, c, qj);
        stage_q_part(a, qj, j & 3, s_qall + (j >> 2) * kQBytes, s_biasall[j >> 2], lane);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && tracing()) s_tr[2] = gtime();
  QS qs;
  qs.base = (uint32_t)__cvta_generic_to_shared(s_qall + slot * kQBytes) + 16 * lane;
  qs.aug_addr = (uint32_t)__cvta_generic_to_shared(s_qall + slot * kQBytes) + 3 * kQSet + 4 * lane;
  PreciseOff po;
  {
    const int G0 = c >> 1, qa = (2 * c) & 3;
    po.m0 = (g * 4 + G0) * 8 - 16 * lane;
    po.m1 = (g * 4 + G0 + 2) * 8 - 16 * lane;
    po.bias = (uint32_t)__cvta_generic_to_shared(s_biasall[slot]) + (G0 * kBiasRows + qa) * 4;
    po.qoff = 16 * (((g & 3) * 4 + c) - lane);
    po.qoff2 = 16 * ((((g & 3) + 4) * 4 + c) - lane);
    po.hi_rows = c >= 2;
    const bool in = (g >> 2) == (c & 1);
    po.msk0 = in && (c >> 1) == 0 ? 0xffffffffu : 0u;
    po.msk1 = in && (c >> 1) == 1 ? 0xffffffffu : 0u;
  }
  const uint32_t mg = kMagic16 | a.zero;

  WarpState st;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) st.acc[mt][0] = st.acc[mt][1] = st.acc[mt][2] = st.acc[mt][3] = 0.f;
  st.lacc[0] = st.lacc[1] = 0.f;
  st.lsq[0] = st.lsq[1] = 0.f;
  st.mrun[0] = st.mrun[1] = -INFINITY;
  st.lsum[0] = st.lsum[1] = 0.f;

  // this warp's FP16-region tiles: the unit's, continuing the rotation after the quantized ones
  auto fp16_part = [&](auto exact_tag) {
    constexpr bool EXACT = decltype(exact_tag)::value;
    const int off_fp = reinterpret_cast<const int*>(a.seq)[8 * b + 4];
    const int len_fp = reinterpret_cast<const int*>(a.seq)[8 * b + 5];
    const int nft = (len_fp + kTile - 1) / kTile;
    const int f_begin = (int)((int64_t)nft * w_lo / nw), f_end = (int)((int64_t)nft * w_hi / nw);
    const int64_t unit = (int64_t)l * a.H + h;
    const uint16_t* kf = a.K.fp + (unit * a.K.rows_fp + off_fp) * kHeadDim;
    const uint16_t* vf = a.V.fp + (unit * a.V.rows_fp + off_fp) * kHeadDim;
    for (int tf = f_begin + rotate(k, n2t + n4t, np); tf < f_end; tf += np) {
      const int r = tf * kTile;
      tile_fp16<EXACT>(kf + (int64_t)r * kHeadDim, vf + (int64_t)r * kHeadDim, len_fp - r, qs, st, g, c);
    }
  };
  if (mode == kModeExact) {
    quantized_tiles<kModeExact>(n2t, n4t, a, src, mo, po, ring_l, qs, mg, st, k, np);
    fp16_part(std::true_type{});
  } else {
    if (mode == kModePrecise) quantized_tiles<kModePrecise>(n2t, n4t, a, src, mo, po, ring_l, qs, mg, st, k, np);
    else if (mode == kModePrecise8) quantized_tiles<kModePrecise8>(n2t, n4t, a, src, mo, po, ring_l, qs, mg, st, k, np);
    else quantized_tiles<kModeNormal>(n2t, n4t, a, src, mo, po, ring_l, qs, mg, st, k, np);
    fp16_part(std::false_type{});
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const float f = (float)(64 >> (2 * (mt & 3)));
      st.acc[mt][0] *= f; st.acc[mt][1] *= f; st.acc[mt][2] *= f; st.acc[mt][3] *= f;
    }
  }
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
  st.lsum[0] += st.lsq[0];
  st.lsum[1] += st.lsq[1];
  if (lane == 0 && tracing()) s_tend[warp] = gtime();
  // Park this warp's partial (rows < m) in its own ring region (its copies are all waited:
  // no barrier needed before the stores).  Column of (q row, d): d's low 4 bits XOR
  // (g >> 1 | row/2 << 2), g = d / 16 — every store instruction of a warp hits 32 distinct
  // banks (unswizzled: 16 lanes per bank).
  auto swz = [](int row, int d) { return (d & ~15) | ((d ^ ((((d >> 4) & 7) >> 1) | ((row >> 1) << 2))) & 15); };
  {
    __syncwarp();
    float (*s_accw)[kHeadDim] = reinterpret_cast<float (*)[kHeadDim]>(&s_ring[warp][0]);
    const bool r0 = 2 * c < a.m, r1 = 2 * c + 1 < a.m;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      if (r0) {
        s_accw[2 * c][swz(2 * c, 16 * g + mt)] = st.acc[mt][0];
        s_accw[2 * c][swz(2 * c, 16 * g + 8 + mt)] = st.acc[mt][2];
      }
      if (r1) {
        s_accw[2 * c + 1][swz(2 * c + 1, 16 * g + mt)] = st.acc[mt][1];
        s_accw[2 * c + 1][swz(2 * c + 1, 16 * g + 8 + mt)] = st.acc[mt][3];
      }
    }
    if (g == 0) {
      s_ml[warp][2 * c][0] = st.mrun[0]; s_ml[warp][2 * c][1] = st.lsum[0];
      s_ml[warp][2 * c + 1][0] = st.mrun[1]; s_ml[warp][2 * c + 1][1] = st.lsum[1];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && tracing()) s_tr[8] = gtime();
  // in-CTA merge, one pass: thread item (slot, q row, d) -> the slot's running max over its
  // warps, then the weighted acc and l sums.  A unit entirely inside this CTA writes its output,
  // otherwise this CTA's partial goes to its slot of the unit's workspace.
  const int Hq = a.H * a.m;
  float* ws_l = a.ws + (int64_t)l * w.U * w.max_ctas * a.m * kWsStride;
  for (int p = threadIdx.x; p < nslots * a.m * kHeadDim; p += blockDim.x) {
    const int d = p & (kHeadDim - 1), rt = s_rtab[p >> 7];
    const int sl = rt >> 8, qi = rt & 255;
    const int4 si = s_slot[sl];
    float ms = -INFINITY;
    for (int ww = si.x; ww < si.y; ++ww) ms = fmaxf(ms, s_ml[ww][qi][0]);
    const int dq = qi * kHeadDim + swz(qi, d);
    float acc0 = 0.f, acc1 = 0.f, lsum = 0.f;
    for (int ww = si.x; ww < si.y; ++ww) {
      const float mw = s_ml[ww][qi][0];
      const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
      const float x = reinterpret_cast<const float*>(&s_ring[ww][0])[dq];
      if (ww & 1) acc1 = fmaf(f, x, acc1);
      else acc0 = fmaf(f, x, acc0);
      lsum = fmaf(f, s_ml[ww][qi][1], lsum);
    }
    const float acc = acc0 + acc1;
    const int us = u0 + sl, bs = us / a.H, hs = us - bs * a.H;
    if (si.z == si.w) {
      const int64_t row = ((int64_t)l * a.B + bs) * Hq + hs * a.m + qi;
      if (a.partial_out) {
        float* dst = a.partial_out + row * kPartStride;
        dst[d] = acc;
        if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
      } else {
        a.out[l * a.o_sl + bs * a.o_sb + (int64_t)(hs * a.m + qi) * kHeadDim + d] =
            __half_as_ushort(__float2half_rn(acc / lsum));
      }
    } else {
      float* dst = ws_l + (((int64_t)us * w.max_ctas + (cta - si.z)) * a.m + qi) * kWsStride;
      dst[d] = acc;
      if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && tracing()) s_tr[9] = gtime();
  // arrival per split unit: the CTA that completes a unit's set of partials merges them.  The
  // barrier above orders every thread's partial stores before the device-scope release RMW.
  if ((int)threadIdx.x < nslots) {
    const int4 si = s_slot[threadIdx.x];
    int last = 0;
    if (si.z != si.w) {
      cuda::atomic_ref<uint32_t, cuda::thread_scope_device> ctr(a.counters[(int64_t)l * w.U + u0 + threadIdx.x]);
      const uint32_t prev = ctr.fetch_add(1u, cuda::memory_order_acq_rel);
      last = prev == (uint32_t)(si.w - si.z);
      if (last) ctr.store(0u, cuda::memory_order_relaxed);
    }
    s_lastu[threadIdx.x] = last;
  }
  __syncthreads();
  if (threadIdx.x == 0 && tracing()) {
    s_tr[10] = gtime();
    int nl = 0;
    for (int i = 0; i < nslots; ++i) nl += s_lastu[i];
    s_tr[11] = nl;
  }
  // units this CTA completes, one at a time: stage the unit's partials (every CTA's rows, one L2
  // round trip) in shared memory (the ring) when they fit, then merge per (q row, d)
  float* s_part = reinterpret_cast<float*>(&s_ring[0][0]);
  for (int sl = 0; sl < nslots; ++sl) {
    if (!s_lastu[sl]) continue;
    const int us = u0 + sl;
    const int4 si = s_slot[sl];
    const int nc = si.w - si.z + 1;
    const int bs = us / a.H, hs = us - bs * a.H;
    const float* src_p = ws_l + (int64_t)us * w.max_ctas * a.m * kWsStride;  // [ctas][m][stride]
    const bool staged = nc * a.m * kWsStride * (int)sizeof(float) <= kWpWarps * kWarpRing;
    if (staged) {
      const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_part);
      const int nvec = nc * a.m * kWsStride / 4;
      for (int i = threadIdx.x; i < nvec; i += blockDim.x) cp_async16(sbase + 16 * i, src_p + 4 * i);
      cp_commit();
      cp_wait<0>();
      __syncthreads();
    }
    const float* pbase = staged ? s_part : src_p;
    for (int p = threadIdx.x; p < a.m * kHeadDim; p += blockDim.x) {
      const int qi = p >> 7, d = p & (kHeadDim - 1);
      const float* pp = pbase + qi * kWsStride;
      float ms = -INFINITY;
      for (int s2 = 0; s2 < nc; ++s2) ms = fmaxf(ms, pp[s2 * a.m * kWsStride + kHeadDim]);
      float acc = 0.f, lsum = 0.f;
      for (int s2 = 0; s2 < nc; ++s2) {
        const float* ps = pp + s2 * a.m * kWsStride;
        const float mw = ps[kHeadDim];
        const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
        acc = fmaf(f, ps[d], acc);
        lsum = fmaf(f, ps[kHeadDim + 1], lsum);
      }
      const int64_t row = ((int64_t)l * a.B + bs) * Hq + hs * a.m + qi;
      if (a.partial_out) {
        float* dst = a.partial_out + row * kPartStride;
        dst[d] = acc;
        if (d == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
      } else {
        a.out[l * a.o_sl + bs * a.o_sb + (int64_t)(hs * a.m + qi) * kHeadDim + d] =
            __half_as_ushort(__float2half_rn(acc / lsum));
      }
    }
    __syncthreads();  // s_part reuse by the next unit
  }
  if (threadIdx.x == 0 && tracing()) {
    int64_t tmax = 0;
    for (int i = 0; i < kWpWarps; ++i) tmax = max(tmax, s_tend[i]);
    s_tr[3] = tmax;
    s_tr[4] = gtime();
    int64_t* dst = g_trace + 16 * atomicAdd(&g_trace_n, 1ull);
    for (int i = 0; i < 5; ++i) dst[i] = s_tr[i];
    for (int i = 8; i < 12; ++i) dst[i] = s_tr[i];
    for (int i = 0; i < 4; ++i) dst[12 + i] = s_tend[i * 5];
    dst[5] = smid();
    dst[6] = (int64_t)cta | ((int64_t)u0 << 40);
    dst[7] = (int64_t)a.q;
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

static bool ensure_decode_attr() {
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem) != cudaSuccess) {
      (void)cudaGetLastError();
      return false;
    }
    attr_set = true;
  }
  return true;
}

extern "C" {

int64_t ckv_decode_workspace_bytes(int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                                   int32_t splits) {
  const int64_t units = (int64_t)layers * batch * kv_heads;
  const int64_t counters = cdiv(units * (int64_t)sizeof(uint32_t), 256) * 256;
  if (splits <= 1) return counters;
  return counters + units * m * splits * kWsStride * (int64_t)sizeof(float);
}

int32_t ckv_decode_attention(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                             ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                             int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                             float scale, int32_t splits, void* workspace, uint16_t* out,
                             int64_t o_s_layer, int64_t o_s_batch, float* partial_out,
                             int32_t flags, void* stream) {
  return ckv_decode_attention_seqs(q, q_s_layer, q_s_batch, k_arena, v_arena, seq, layers, batch, 0,
                                   batch, kv_heads, m, scale, splits, workspace, out, o_s_layer,
                                   o_s_batch, partial_out, flags, stream);
}

int32_t ckv_decode_attention_seqs(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                  ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                  int32_t layers, int32_t batch, int32_t seq_begin, int32_t seq_count,
                                  int32_t kv_heads, int32_t m, float scale, int32_t splits,
                                  void* workspace, uint16_t* out, int64_t o_s_layer, int64_t o_s_batch,
                                  float* partial_out, int32_t flags, void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0 || splits < 1) return CKV_ERR_ARG;
  if (seq_begin < 0 || seq_count < 0 || seq_begin + seq_count > batch) return CKV_ERR_ARG;
  if (m < 1 || m > 8) return CKV_ERR_UNSUPPORTED;
  if (!q || !seq || (!out && !partial_out)) return CKV_ERR_ARG;
  if (splits > 1 && !workspace) return CKV_ERR_ARG;
  if ((q_s_layer % 8) || (q_s_batch % 8)) return CKV_ERR_UNSUPPORTED;
  if (layers * seq_count * kv_heads == 0) return CKV_OK;
  {  // interleaved K/V tile buffers (include/ckv.h)
    const char* k2 = reinterpret_cast<const char*>(k_arena.codes2);
    const char* k4 = reinterpret_cast<const char*>(k_arena.codes4);
    const bool ok2 = k_arena.rows2 == 0 ||
                     (reinterpret_cast<const char*>(v_arena.codes2) == k2 + kTileBytes2 &&
                      reinterpret_cast<const char*>(k_arena.meta2) == k2 + 2 * kTileBytes2 &&
                      reinterpret_cast<const char*>(v_arena.meta2) == k2 + 2 * kTileBytes2 + kTileBytesMeta);
    const bool ok4 = k_arena.rows4 == 0 ||
                     (reinterpret_cast<const char*>(v_arena.codes4) == k4 + kTileBytes4 &&
                      reinterpret_cast<const char*>(k_arena.meta4) == k4 + 2 * kTileBytes4 &&
                      reinterpret_cast<const char*>(v_arena.meta4) == k4 + 2 * kTileBytes4 + kTileBytesMeta);
    if (!ok2 || !ok4 || k_arena.rows2 != v_arena.rows2 || k_arena.rows4 != v_arena.rows4) return CKV_ERR_ARG;
  }
  DecArgs a;
  a.q = q; a.q_sl = q_s_layer; a.q_sb = q_s_batch;
  a.K = k_arena; a.V = v_arena; a.seq = seq;
  a.L = layers; a.B = batch; a.H = kv_heads; a.m = m; a.splits = splits;
  a.b0 = seq_begin; a.Bc = seq_count;
  a.scale_log2 = scale * 1.4426950408889634f;
  const int64_t units = (int64_t)layers * batch * kv_heads;
  a.counters = reinterpret_cast<uint32_t*>(workspace);
  a.ws = workspace ? reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                              cdiv(units * (int64_t)sizeof(uint32_t), 256) * 256)
                   : nullptr;
  a.out = out; a.o_sl = o_s_layer; a.o_sb = o_s_batch;
  a.partial_out = partial_out;
  a.zero = 0u;
  if (!ensure_decode_attr()) return CKV_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)splits, (unsigned)kv_heads, (unsigned)(layers * seq_count));
  cfg.blockDim = dim3(kDecWarps * 32);
  cfg.dynamicSmemBytes = kDynSmem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (flags & CKV_DECODE_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, decode_kernel, a) != cudaSuccess) {
    (void)cudaGetLastError();
    return CKV_ERR_CUDA;
  }
  return CKV_OK;
}

int32_t ckv_decode_ctas_per_sm(void) {
  if (!ensure_decode_attr()) return -1;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_kernel, kDecWarps * 32, kDynSmem) != cudaSuccess) {
    (void)cudaGetLastError();
    return -1;
  }
  return n;
}

// Tuning aid (not part of the ABI): point the decode timeline at buf (null disables) and
// reset its counter.
int32_t ckv_decode_set_trace(int64_t* buf) {
  unsigned long long z = 0;
  if (cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z)) != cudaSuccess) {
    (void)cudaGetLastError();
    return CKV_ERR_CUDA;
  }
  return CKV_OK;
}

static size_t g_wp_smem = 0;

int32_t ckv_decode_wp_cta_warps(void) { return kWpWarps; }

int64_t ckv_decode_wp_workspace_bytes(int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                                      int32_t max_ctas) {
  const int64_t units = (int64_t)layers * batch * kv_heads;
  return cdiv(units * (int64_t)sizeof(uint32_t), 256) * 256 +
         units * (int64_t)(max_ctas > 0 ? max_ctas : 1) * m * kWsStride * (int64_t)sizeof(float);
}

int32_t ckv_decode_attention_wp(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                int32_t layers, int32_t batch, int32_t kv_heads, int32_t m, float scale,
                                const int32_t* warp_prefix, int32_t ctas, int32_t max_slots,
                                int32_t max_ctas, void* workspace, uint16_t* out, int64_t o_s_layer,
                                int64_t o_s_batch, float* partial_out, int32_t flags, void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0 || ctas < 1) return CKV_ERR_ARG;
  if (m < 1 || m > 8) return CKV_ERR_UNSUPPORTED;
  if (max_slots < 1 || max_slots > 8 || max_ctas < 1) return CKV_ERR_UNSUPPORTED;
  if (!q || !seq || !warp_prefix || !workspace || (!out && !partial_out)) return CKV_ERR_ARG;
  if ((q_s_layer % 8) || (q_s_batch % 8)) return CKV_ERR_UNSUPPORTED;
  if (layers * batch * kv_heads == 0) return CKV_OK;
  {
    const char* k2 = reinterpret_cast<const char*>(k_arena.codes2);
    const char* k4 = reinterpret_cast<const char*>(k_arena.codes4);
    const bool ok2 = k_arena.rows2 == 0 ||
                     (reinterpret_cast<const char*>(v_arena.codes2) == k2 + kTileBytes2 &&
                      reinterpret_cast<const char*>(k_arena.meta2) == k2 + 2 * kTileBytes2 &&
                      reinterpret_cast<const char*>(v_arena.meta2) == k2 + 2 * kTileBytes2 + kTileBytesMeta);
    const bool ok4 = k_arena.rows4 == 0 ||
                     (reinterpret_cast<const char*>(v_arena.codes4) == k4 + kTileBytes4 &&
                      reinterpret_cast<const char*>(k_arena.meta4) == k4 + 2 * kTileBytes4 &&
                      reinterpret_cast<const char*>(v_arena.meta4) == k4 + 2 * kTileBytes4 + kTileBytesMeta);
    if (!ok2 || !ok4 || k_arena.rows2 != v_arena.rows2 || k_arena.rows4 != v_arena.rows4) return CKV_ERR_ARG;
  }
  WpArgs w;
  DecArgs& a = w.d;
  a.q = q; a.q_sl = q_s_layer; a.q_sb = q_s_batch;
  a.K = k_arena; a.V = v_arena; a.seq = seq;
  a.L = layers; a.B = batch; a.H = kv_heads; a.m = m; a.splits = 1;
  a.b0 = 0; a.Bc = batch;
  a.scale_log2 = scale * 1.4426950408889634f;
  const int64_t units = (int64_t)layers * batch * kv_heads;
  a.counters = reinterpret_cast<uint32_t*>(workspace);
  a.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + cdiv(units * (int64_t)sizeof(uint32_t), 256) * 256);
  a.out = out; a.o_sl = o_s_layer; a.o_sb = o_s_batch;
  a.partial_out = partial_out;
  a.zero = 0u;
  w.prefix = warp_prefix;
  w.U = batch * kv_heads;
  w.max_slots = max_slots;
  w.max_ctas = max_ctas;
  const size_t smem = (size_t)kWpWarps * kWarpRing + (size_t)max_slots * kQBytes;
  if (smem > g_wp_smem) {
    if (cudaFuncSetAttribute(decode_wp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      (void)cudaGetLastError();
      return CKV_ERR_CUDA;
    }
    g_wp_smem = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas, 1u, (unsigned)layers);
  cfg.blockDim = dim3(kWpWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (flags & CKV_DECODE_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, decode_wp_kernel, w) != cudaSuccess) {
    (void)cudaGetLastError();
    return CKV_ERR_CUDA;
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
