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
//   S^T[16 tok x 8 q] = lo.Q + sum_G sigma_G (K_G . Q'_G^T)   mma.m16n8k16: 1 + 2 per group G
//   P = exp2(S - m) (online, lazy rescale), P^T -> P via movmatrix
//   O^T[128 d x 8 q] += V_G^T[32 x 16] . (P x span_G)^T      mma.m16n8k16: 2 per group (+1 lo term)
// Quantized tiles stream through a per-warp 4-stage cp.async ring in shared memory (tile bytes
// permuted so every fragment read is one conflict-free shared load); FP16 tiles (<4% of bytes)
// are read straight from global memory.  The packed codes enter the tensor cores as fp16
// subnormals (code << j is the fp16 value code * 2^(j-24): one AND per pair of codes, no
// bias), every 32-element group forms its own k-steps (K) / m-tiles (V), and the group scales
// are applied per (token, group) instead of per element: on the K side to the group's fp32
// partial sums, on the V side folded into the P operand.  Per-unit powers of two keep every
// fp16 operand in range (see "operand scaling").
#include <math.h>

#include <cuda/atomic>
#include <algorithm>
#include <vector>
#include <type_traits>

#include "ckv_common.cuh"

namespace ckv {

#ifndef CKV_DEC_WARPS
#define CKV_DEC_WARPS 4
#endif
constexpr int kDecWarps = CKV_DEC_WARPS;  // warps per split-kernel CTA (4; 8 as a build variant)
static_assert(kDecWarps == 4 || kDecWarps == 8, "split kernel: 4 or 8 warps per CTA");
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
constexpr int kDynSmem = kDecWarps * kWarpRing;  // 40 KB per CTA (4 warps x 4 x 2560 B)
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
  int h0;               // and its kv heads [h0, h0 + gridDim.y) (split kernel)
  float scale_log2;
  float* ws;            // [L*B*H*m][splits][130] partials
  uint32_t* counters;   // [L*B*H] arrival counters (self-resetting)
  uint16_t* out;
  int64_t o_sl, o_sb;
  float* partial_out;   // [L][B][H*m][130] or null
  int64_t* trace;       // per-CTA timeline buffer (tuning aid) or null
};

// Optional per-CTA timeline (tuning aid, not part of the ABI): when set, every CTA appends 16
// int64: globaltimer at start, after the PDL wait, after q staging, after warp 0's tiles, at
// exit; smid, linear block index, q pointer (launch id); after all warps' tiles, before the
// arrival atomic, after it, is-last; per-warp tile end times.
__device__ unsigned long long g_trace_n = 0;
__device__ __forceinline__ int64_t gtime() {
  int64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// The trace buffer is a kernel parameter (DecArgs::trace, null unless ckv_decode_set_trace
// armed it): the probe points cost no memory round trip when tracing is off.
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
__device__ __forceinline__ CtaIds cta_ids(int Bc, int b0, int h0) {
  uint32_t x, y, z;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(x));
  asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(y));
  asm volatile("mov.u32 %0, %%ctaid.z;" : "=r"(z));
  return CtaIds{(int)x, h0 + (int)y, (int)z / Bc, b0 + (int)z % Bc};
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


// ---- operand scaling -------------------------------------------------------------------
// Quantized codes enter the tensor cores as fp16 SUBNORMALS: a code c at bits [j, j+b) of a
// 16-bit lane (no exponent bits) is the fp16 value c * 2^(j-24) exactly, so extracting a pair
// of codes is one AND and there is no bias term.  HMMA multiplies subnormal operands exactly
// (tools/subnormal_probe.cu).  The per-slot power of two 2^(j-24) is folded into q (K side) and
// into the output rows (V side); the group scales are applied per (token, group) outside the
// per-element path: K in fp32 on the per-group q.K^T partial sums, V folded into P.
//   q side: q' = q 2^(E - j) in fp16, E per unit so max|q| 2^E is in [2^14, 2^15) (no overflow,
//           no fp16 range limit on q); S = lo-term + sum_G sigma_G X_G, sigma = span 2^(24-E)/qmax.
//   V side: p'_G = fp16(p span_G 2^F), F per unit from the unit's largest V group span so that
//           p' <= 2^15; O accumulates sum_t p'_G code 2^(j-24) and is brought back to value
//           units (x 2^(24-F-j) / qmax per accumulator row) when a phase ends.
__device__ __forceinline__ int q_exponent(float maxabs) {  // E: max|q| 2^E in [2^14, 2^15)
  if (!(maxabs > 0.f) || !(maxabs < INFINITY)) return 0;
  int x;
  (void)frexpf(maxabs, &x);  // maxabs = m 2^x, m in [0.5, 1)
  return 15 - x;
}
__device__ __forceinline__ int v_exponent(float span_max) {  // F: span_max 2^F < 2^7
  if (!(span_max > 0.f) || !(span_max < INFINITY)) return 0;
  int x;
  (void)frexpf(span_max, &x);
  return min(7 - x, 15);  // 2^F stays an fp16 normal
}

// scale (hi - lo) * k of one (lo, hi) half2 metadata word (hi - lo exact: mixed f16/f32 subtract)
__device__ __forceinline__ float meta_scale(uint32_t meta, float k) {
  float d;
  asm("{.reg .f16 lo, hi; .reg .f32 a; mov.b32 {lo, hi}, %1; cvt.f32.f16 a, lo; sub.rn.f32.f16 %0, hi, a;}"
      : "=f"(d) : "r"(meta));
  return d * k;
}
// (hi - lo) 2^F of two groups in one rounding: hi 2^F - lo 2^F (the scaled operands cannot
// overflow where hi - lo itself would, e.g. lo = -60000, hi = 60000)
__device__ __forceinline__ uint32_t span2(uint32_t hi, uint32_t lo, uint32_t f2) {
  const __half2 f = u32_as_h2(f2);
  return h2_as_u32(__hfma2(u32_as_h2(hi), f, __hneg2(__hmul2(u32_as_h2(lo), f))));
}
__device__ __forceinline__ uint32_t hmul2u(uint32_t a, uint32_t b) { return h2_as_u32(__hmul2(u32_as_h2(a), u32_as_h2(b))); }

struct WarpState {
  float acc[8][4];  // O^T C-fragments, m-tile mt (group mt / 2): rows d = 32 (mt >> 1) + 4 g + 2 (mt & 1)
                    // (c0, c1) and d + 1 (c2, c3), columns (q rows) 2c, 2c+1
  float lacc[2];    // sum_t p_t lo_{t,G} for G = g (lanes g < 4; rows g >= 4 duplicate), cols 2c, 2c+1
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

// Q B-fragments live in shared memory as three sets ([set][group G][32 lanes] x 16 B, one
// copy per CTA: the fragments of k-steps 2G, 2G+1 of a lane side by side, one conflict-free
// 128-bit load): 0 = INT2 slot weights, 1 = INT4 slot weights, 2 = unweighted (FP16 tiles).
// K-step 2G + h, lane (g, c): b0 = q'[g][32G + 8c + 2h], q'[g][32G + 8c + 4 + 2h];
// b1 = q'[g][32G + 8c + 2h + 1], q'[g][32G + 8c + 5 + 2h] — the d order of the tile layouts
// (ckv_common.cuh).  After the sets, [32 lanes] x 4 B: the (hi, lo) fp16 split of
// Q[g][G = c] = sum_{d in G} q[g][d] for the zero-point MMA.
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
__device__ __forceinline__ void sts32d(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts64d(uint32_t a, uint32_t v0, uint32_t v1) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v0), "r"(v1) : "memory");
}

// The V zero-point term sum_t p_t lo_{t,G} (A rows g: group g & 3) and, on the A rows g+8 set
// to fp16 ones, the tile's row sums sum_t p_t of the same fp16 P the P.V MMAs use.
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
// `sl` = stage + 16 * lane (this lane's code slots).  Per-lane constants:
struct LaneOff {
  int32_t mk;   // K meta entry (tok g, g+8; group c) relative to sl: -8 lane
  int32_t mv;   // V meta entry (group g & 3, c) relative to sl
  uint32_t sk;  // this warp's scale scratch + 4 lane: K sigma of (tok g, group c); +128: tok g+8
  uint32_t kc;  // scratch + 16 g: the sigmas of tok g, groups 0-3; +128: tok g+8
  uint32_t vp;  // scratch + 256 + 8 (4 c + (g & 3)): span pairs of group g & 3
  uint32_t vc;  // scratch + 256 + 32 c: span pairs of groups 0-3 for this lane's tokens
};
constexpr int kScratch = 384;  // per warp: K sigmas [16 tok][4 G] f32 | V span pairs [4 c][4 G][2] half2

template <int BITS> struct TL {
  static constexpr uint32_t vc = BITS == 2 ? 512 : 1024;
  static constexpr uint32_t km = BITS == 2 ? 1024 : 2048;
  static constexpr uint32_t vm = km + 256;
  static constexpr int set = BITS == 2 ? 0 : 1;
};

// S^T[16 tok x 8 q] of a quantized tile: zero-point MMA (lo x Q), then per group G two MMAs on
// the raw subnormal codes into the group's own accumulator X_G, combined in fp32 with the
// (token, group) sigmas shared through the warp's scratch.  kappa = 2^(24-E) / qmax.
template <int BITS>
__device__ __forceinline__ void qk_tile(uint32_t sl, const LaneOff& lo, const QS& qs, float kappa, float (&s)[4]) {
  const uint2 kmm = lds64(sl + TL<BITS>::km + lo.mk);  // (lo, hi) of (tok g, G = c), (tok g+8, G = c)
  sts32d(lo.sk, __float_as_uint(meta_scale(kmm.x, kappa)));
  sts32d(lo.sk + 128, __float_as_uint(meta_scale(kmm.y, kappa)));
#pragma unroll
  for (int e = 0; e < 4; ++e) s[e] = 0.f;
  mma_16816(s, prmt(kmm.x, kmm.x, 0x1010), prmt(kmm.y, kmm.y, 0x1010), 0u, 0u, qs.aug(), 0u);
  float X[4][4];
  if (BITS == 2) {
    // word G = [tok g: byte 8G+2c | tok g+8: 8G+2c | tok g: 8G+2c+1 | tok g+8: 8G+2c+1]
    const uint4 kk = lds128(sl);
    const uint32_t w[4] = {kk.x, kk.y, kk.z, kk.w};
#pragma unroll
    for (int G = 0; G < 4; ++G) {
      const uint32_t W = w[G], W8 = W >> 8;
      const uint4 q = qs.ld2(0, G);
#pragma unroll
      for (int e = 0; e < 4; ++e) X[G][e] = 0.f;
      mma_16816(X[G], W & 0x00030003u, W8 & 0x00030003u, W & 0x000C000Cu, W8 & 0x000C000Cu, lo2(q));
      mma_16816(X[G], W & 0x00300030u, W8 & 0x00300030u, W & 0x00C000C0u, W8 & 0x00C000C0u, hi2(q));
    }
  } else {
    // tok g: the reference's words 4G + c (G = 0..3); +512: tok g+8
    const uint4 ka = lds128(sl), kb = lds128(sl + 512);
    const uint32_t wa[4] = {ka.x, ka.y, ka.z, ka.w}, wb[4] = {kb.x, kb.y, kb.z, kb.w};
#pragma unroll
    for (int G = 0; G < 4; ++G) {
      const uint32_t A = wa[G], B = wb[G], A8 = A >> 8, B8 = B >> 8;
      const uint4 q = qs.ld2(1, G);
#pragma unroll
      for (int e = 0; e < 4; ++e) X[G][e] = 0.f;
      mma_16816(X[G], A & 0x000F000Fu, B & 0x000F000Fu, A & 0x00F000F0u, B & 0x00F000F0u, lo2(q));
      mma_16816(X[G], A8 & 0x000F000Fu, B8 & 0x000F000Fu, A8 & 0x00F000F0u, B8 & 0x00F000F0u, hi2(q));
    }
  }
  __syncwarp();
  const uint4 ga = lds128(lo.kc), gb = lds128(lo.kc + 128);  // sigma (tok g | tok g+8, G = 0..3)
  const float sa[4] = {__uint_as_float(ga.x), __uint_as_float(ga.y), __uint_as_float(ga.z), __uint_as_float(ga.w)};
  const float sb[4] = {__uint_as_float(gb.x), __uint_as_float(gb.y), __uint_as_float(gb.z), __uint_as_float(gb.w)};
#pragma unroll
  for (int G = 0; G < 4; ++G) {
    s[0] = fmaf(sa[G], X[G][0], s[0]);
    s[1] = fmaf(sa[G], X[G][1], s[1]);
    s[2] = fmaf(sb[G], X[G][2], s[2]);
    s[3] = fmaf(sb[G], X[G][3], s[3]);
  }
}

// O^T += V^T P' of a quantized tile: the group's span pairs x 2^F (from lanes g < 4 through the
// scratch) fold the V scales into P per group; m-tiles 2G, 2G+1 take group G's codes, rows
// (mt, g) / (mt, g+8) = code e = 2 (mt & 1) / 2 (mt & 1) + 1 of the lane's byte (INT2) or
// 16-bit piece (INT4) of that group.  f2 = 2^F in both halves.
template <int BITS>
__device__ __forceinline__ void pv_tile(uint32_t sl, const LaneOff& lo, WarpState& st, uint32_t bp0, uint32_t bp1,
                                        uint32_t f2) {
  // entry (G = g & 3, c): (lo 2c | 2c+1), (hi 2c | 2c+1), (lo 2c+8 | 2c+9), (hi 2c+8 | 2c+9)
  const uint4 vmm = lds128(sl + TL<BITS>::vm + lo.mv);
  sts64d(lo.vp, span2(vmm.y, vmm.x, f2), span2(vmm.w, vmm.z, f2));
  lo_mma(st, vmm.x, vmm.z, bp0, bp1);
  __syncwarp();
  const uint4 ga = lds128(lo.vc), gb = lds128(lo.vc + 16);  // (G0: 2c|2c+1, 2c+8|2c+9), (G1 ..), (G2), (G3)
  const uint32_t pa[4] = {hmul2u(bp0, ga.x), hmul2u(bp0, ga.z), hmul2u(bp0, gb.x), hmul2u(bp0, gb.z)};
  const uint32_t pb[4] = {hmul2u(bp1, ga.y), hmul2u(bp1, ga.w), hmul2u(bp1, gb.y), hmul2u(bp1, gb.w)};
  if (BITS == 2) {
    // words: (tok 2c | 2c+1) x (G0, G1), (tok 2c | 2c+1) x (G2, G3), then tokens 2c+8 | 2c+9
    const uint4 vv = lds128(sl + TL<2>::vc);
#pragma unroll
    for (int G = 0; G < 4; ++G) {
      const uint32_t ua = ((G >> 1) ? vv.y : vv.x) >> (8 * (G & 1));
      const uint32_t ub = ((G >> 1) ? vv.w : vv.z) >> (8 * (G & 1));
      mma_16816(st.acc[2 * G], ua & 0x00030003u, ua & 0x000C000Cu, ub & 0x00030003u, ub & 0x000C000Cu, pa[G], pb[G]);
      mma_16816(st.acc[2 * G + 1], ua & 0x00300030u, ua & 0x00C000C0u, ub & 0x00300030u, ub & 0x00C000C0u, pa[G], pb[G]);
    }
  } else {
    // words G: (tok 2c | 2c+1) 16-bit pieces of group G; +512: tokens 2c+8 | 2c+9
    const uint4 va = lds128(sl + TL<4>::vc), vb = lds128(sl + TL<4>::vc + 512);
    const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
    for (int G = 0; G < 4; ++G) {
      const uint32_t ua = wa[G], ub = wb[G], ua8 = ua >> 8, ub8 = ub >> 8;
      mma_16816(st.acc[2 * G], ua & 0x000F000Fu, ua & 0x00F000F0u, ub & 0x000F000Fu, ub & 0x00F000F0u, pa[G], pb[G]);
      mma_16816(st.acc[2 * G + 1], ua8 & 0x000F000Fu, ua8 & 0x00F000F0u, ub8 & 0x000F000Fu, ub8 & 0x00F000F0u, pa[G], pb[G]);
    }
  }
}

// Accumulator row weights of a phase: O_acc = W(e) O (value units), code e = 2 (mt & 1) + (row
// half), W(e) = qmax 2^(F + j(e) - 24) with the code's bit position j: INT2 j = 2e, INT4
// j = 4 (e & 1).  Scaling by w_next / w_prev per row class moves the accumulator between phases.
__device__ __forceinline__ void phase_weights(int bits, int F, float (&w)[4]) {
  const float qmax = bits == 2 ? 3.0f : 15.0f;
#pragma unroll
  for (int e = 0; e < 4; ++e) w[e] = qmax * exp2f((float)(F + (bits == 2 ? 2 * e : 4 * (e & 1)) - 24));
}
__device__ __forceinline__ void scale_acc(WarpState& st, const float (&f)[4]) {
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const float a = f[2 * (mt & 1)], b = f[2 * (mt & 1) + 1];
    st.acc[mt][0] *= a; st.acc[mt][1] *= a; st.acc[mt][2] *= b; st.acc[mt][3] *= b;
  }
}

// ---- FP16 tile straight from global memory (FP16 chunks, tail, decode tokens) ------------
// Same d order as the quantized tiles (q set 2 = unweighted q); V in value units.
#ifndef CKV_DEC_FP16_VEARLY
#define CKV_DEC_FP16_VEARLY 1
#endif
__device__ __forceinline__ void tile_fp16(const uint16_t* kf, const uint16_t* vf, int valid,
                                          const QS& qs, WarpState& st, int g, int c) {
  const int toks[4] = {2 * c, 2 * c + 1, 2 * c + 8, 2 * c + 9};
  uint2 w[2][4][2];  // [half][token][G - 2 half]: d = 32G + 4g + [0, 4)
  auto load_v = [&](int half) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int i = 0; i < 2; ++i)
        w[half][t][i] = __ldg(reinterpret_cast<const uint2*>(vf + toks[t] * kHeadDim + 32 * (2 * half + i) + 4 * g));
  };
#if CKV_DEC_FP16_VEARLY
  // the V rows are issued with the K rows: one memory round trip per tile instead of two (K,
  // then V after the softmax)
  load_v(0);
  load_v(1);
#endif
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int G = 0; G < 4; ++G) {
    // tokens g, g+8: d = 32G + 8c + [0, 8)
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(kf + g * kHeadDim + 32 * G + 8 * c));
    const uint4 y = __ldg(reinterpret_cast<const uint4*>(kf + (g + 8) * kHeadDim + 32 * G + 8 * c));
    const uint4 q = qs.ld2(2, G);
    mma_16816(s, prmt(x.x, x.z, 0x5410), prmt(y.x, y.z, 0x5410), prmt(x.x, x.z, 0x7632), prmt(y.x, y.z, 0x7632), lo2(q));
    mma_16816(s, prmt(x.y, x.w, 0x5410), prmt(y.y, y.w, 0x5410), prmt(x.y, x.w, 0x7632), prmt(y.y, y.w, 0x7632), hi2(q));
  }
  if (g >= valid) { s[0] = -INFINITY; s[1] = -INFINITY; }
  if (g + 8 >= valid) { s[2] = -INFINITY; s[3] = -INFINITY; }
  uint32_t bp0, bp1;
  softmax_tile<true>(s, st, bp0, bp1);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
#if !CKV_DEC_FP16_VEARLY
    load_v(half);
#endif
    const uint2 (&wh)[4][2] = w[half];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int G = 2 * half + i;
      // m-tile 2G: rows (e 0 | e 1); 2G+1: (e 2 | e 3); tokens (2c | 2c+1) and (2c+8 | 2c+9)
      mma_16816(st.acc[2 * G], prmt(wh[0][i].x, wh[1][i].x, 0x5410), prmt(wh[0][i].x, wh[1][i].x, 0x7632),
                prmt(wh[2][i].x, wh[3][i].x, 0x5410), prmt(wh[2][i].x, wh[3][i].x, 0x7632), bp0, bp1);
      mma_16816(st.acc[2 * G + 1], prmt(wh[0][i].y, wh[1][i].y, 0x5410), prmt(wh[0][i].y, wh[1][i].y, 0x7632),
                prmt(wh[2][i].y, wh[3][i].y, 0x5410), prmt(wh[2][i].y, wh[3][i].y, 0x7632), bp0, bp1);
    }
  }
}

// L2 prefetch of an FP16-region tile (its K and V rows are each one contiguous 4 KB run: one
// 128-byte line per lane and operand), issued one warp step ahead of the tile's loads.  Split
// schedule only (all-FP16 cfg4 maps, 2-layer sweep: 5220 -> 6612 GB/s); the warp plan, whose
// FP16-heavy units are spread over more warps, measured 6313 -> 6070 with it.
__device__ __forceinline__ void prefetch_fp16_tile(const uint16_t* kf, const uint16_t* vf, int lane) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(kf + 64 * lane));
  asm volatile("prefetch.global.L2 [%0];" ::"l"(vf + 64 * lane));
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
// Ring synchronisation.  Default: 16-byte cp.async per lane, one commit group per stage, the
// consumer waits for all but the kStages-2 youngest groups.  CKV_DEC_BULK: one lane issues the
// whole contiguous tile as ONE bulk copy (cp.async.bulk, the 1-D TMA path) completing on the
// stage's mbarrier (expect_tx of the tile bytes); the consumer waits on that mbarrier's phase.
// The warp's kStages mbarriers live in a file-scope shared array (both decode kernels).
#ifndef CKV_DEC_BULK
#define CKV_DEC_BULK 0
#endif
// Programmatic-dependent-launch trigger of the split kernel: right after its own wait (0),
// after its tiles (1, default) or after its in-CTA merge (2).  With concurrent micro-batch
// chains an early trigger lets the next layer's CTAs sit in SM slots for a whole tile phase
// waiting for this one: cfg2 8 chains 4703 (0) / 4754 (1) / 4755 (2) GB/s, e2e 4578 / 4707.
#ifndef CKV_DEC_LATE_TRIGGER
#define CKV_DEC_LATE_TRIGGER 1
#endif
#ifndef CKV_DEC_Q_PREFETCH
#define CKV_DEC_Q_PREFETCH 1
#endif


#if CKV_DEC_BULK
__shared__ __align__(8) uint64_t g_ring_mbar[16][4];
__device__ __forceinline__ uint32_t ring_mbar(int slot) {
  return (uint32_t)__cvta_generic_to_shared(&g_ring_mbar[threadIdx.x >> 5][slot]);
}
__device__ __forceinline__ void ring_init() {  // whole warp, before its first issue
  if ((threadIdx.x & 31) < 4)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ring_mbar(threadIdx.x & 31)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
}
__device__ __forceinline__ void ring_wait(int slot, uint32_t& ph) {
  const uint32_t mb = ring_mbar(slot), par = (ph >> slot) & 1u;
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(mb), "r"(par) : "memory");
  ph ^= 1u << slot;
}
#else
__device__ __forceinline__ void ring_init() {}
#endif

template <int BITS>
__device__ __forceinline__ void issue_at(int t, int n, const char* base, uint32_t sl, int slot) {
  constexpr int kB = BITS == 2 ? kBlock2 : kBlock4;
#if CKV_DEC_BULK
  // lane 0's stage slot and source are the tile's first bytes (both carry + 16 lane)
  if (t < n && (threadIdx.x & 31) == 0) {
    const char* p = base + (int64_t)t * kB;
    const uint32_t mb = ring_mbar(slot);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "n"(kB) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sl), "l"(p), "n"(kB), "r"(mb) : "memory");
  }
#else
  (void)slot;
  if (t < n) {
    const char* p = base + (int64_t)t * kB;
    cp_async16(sl, p);
    cp_async16(sl + 512, p + 512);
    cp_async16(sl + 1024, p + 1024);
    if (BITS == 4) {
      cp_async16(sl + 1536, p + 1536);
      cp_async16(sl + 2048, p + 2048);
    }
  }
  cp_commit();
#endif
}

// Prologue of a phase: put this warp's first kStages-1 tiles of the range in flight.
template <int BITS>
__device__ __forceinline__ void prologue(int n, const DecArgs& a, const TileSrc& src, uint32_t ring_l, int warp,
                                         int stride = kDecWarps) {
  const char* base = tile_base<BITS>(a, src);
#pragma unroll
  for (int s = 0; s < Ring<BITS>::stages - 1; ++s)
    issue_at<BITS>(warp + stride * s, n, base, ring_l + s * Ring<BITS>::bytes, s);
}

// Per-unit operand scaling of a warp (E: q, F: V; see "operand scaling").
struct UnitScale {
  int E, F;
};

// The tile loop of one warp over one kind's range [0, n) (tiles warp, warp + 4, ...) through
// the cp.async ring (prologue already issued), software-pipelined so that q.K^T of tile i+1
// and P.V of tile i form one straight-line block (independent MMA chains the scheduler can
// interleave).
template <int BITS>
__device__ __forceinline__ void run_tiles(int n, const DecArgs& a, const TileSrc& src, const LaneOff& lo,
                                          uint32_t ring_l, const QS& qs, const UnitScale& us,
                                          WarpState& st, int warp, uint32_t& ph, int stride = kDecWarps) {
  constexpr int kStages = Ring<BITS>::stages, kStageBytes = Ring<BITS>::bytes;
  const uint32_t ring_end = ring_l + kStages * kStageBytes;
  auto next = [&](uint32_t x) { return x + kStageBytes == ring_end ? ring_l : x + kStageBytes; };
  auto nslot = [](int x) { return x + 1 == kStages ? 0 : x + 1; };
  auto wait = [&](int slot) {
#if CKV_DEC_BULK
    ring_wait(slot, ph);
#else
    (void)slot;
    cp_wait<kStages - 2>();
    __syncwarp();
#endif
  };
  int t = warp;
  const int64_t kStep = (int64_t)stride * (BITS == 2 ? kBlock2 : kBlock4);
  // address of the next tile to issue (kStages-1 ahead of the one consumed), advanced by one
  // warp stride per iteration: a loop-carried pointer instead of base + t * block each time
  const char* pn = tile_base<BITS>(a, src) + (int64_t)(warp + stride * (kStages - 1)) * (BITS == 2 ? kBlock2 : kBlock4);
  const float kappa = exp2f((float)(24 - us.E)) * (BITS == 2 ? 1.0f / 3.0f : 1.0f / 15.0f);
  const uint32_t f2 = h2_as_u32(__float2half2_rn(exp2f((float)us.F)));
  if (t < n) {
    uint32_t cur = ring_l, put = ring_l + (kStages - 1) * kStageBytes;
    int cs = 0, ps = kStages - 1;
    wait(cs);
    float s0[4];
    qk_tile<BITS>(cur, lo, qs, kappa, s0);
    uint32_t bp0, bp1;
    softmax_tile<false>(s0, st, bp0, bp1);
    while (true) {
      const int tn = t + stride;
      issue_at<BITS>(t + stride * (kStages - 1) < n ? 0 : 1, 1, pn, put, ps);
      pn += kStep;
      if (tn >= n) {
        pv_tile<BITS>(cur, lo, st, bp0, bp1, f2);
        break;
      }
      const uint32_t nx = next(cur);
      const int ns = nslot(cs);
      wait(ns);
      float sn[4];
      qk_tile<BITS>(nx, lo, qs, kappa, sn);
      pv_tile<BITS>(cur, lo, st, bp0, bp1, f2);
      __syncwarp();  // slot `cur` (and the scratch) may be refilled from now on
      softmax_tile<false>(sn, st, bp0, bp1);
      put = cur;  // the refill slot trails the consumed one by a full ring (kStages - 1 ahead)
      ps = cs;
      cur = nx;
      cs = ns;
      t = tn;
    }
  }
#if !CKV_DEC_BULK
  cp_wait<0>();
#endif
}

// Both phases of a CTA's quantized tiles: INT2 (its prologue issued before the PDL wait), then
// INT4 (prologue here, or before the wait when the CTA has no INT2 tiles).  The accumulator
// moves from INT2 to INT4 row weights between the phases and to value units after them.
__device__ __forceinline__ int rotate(int warp, int done, int stride) {  // (warp - done) mod stride
  const int r = (warp - done) % stride;
  return r < 0 ? r + stride : r;
}

__device__ __forceinline__ void quantized_tiles(int n2, int n4, const DecArgs& a, const TileSrc& src,
                                                const LaneOff& lo, uint32_t ring_l, const QS& qs,
                                                const UnitScale& us, WarpState& st, int warp,
                                                int stride = kDecWarps) {
  uint32_t ph = 0u;  // mbarrier phase parity per ring slot (bulk-copy ring)
  // the INT4 phase starts at the warp after the one that took the last INT2 tile, so every
  // warp's tile count over both phases is within one of the others' (the CTA's warps meet at
  // the merge barrier)
  const int w4 = rotate(warp, n2, stride);
  if (n2 > 0) {
    run_tiles<2>(n2, a, src, lo, ring_l, qs, us, st, warp, ph, stride);
    if (n4 > 0) {
      __syncwarp();
      prologue<4>(n4, a, src, ring_l, w4, stride);
    }
  }
  float w2[4], w4w[4], f[4];
  phase_weights(2, us.F, w2);
  phase_weights(4, us.F, w4w);
  if (n4 > 0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) f[e] = w4w[e] / w2[e];
    scale_acc(st, f);
    run_tiles<4>(n4, a, src, lo, ring_l, qs, us, st, w4, ph, stride);
#pragma unroll
    for (int e = 0; e < 4; ++e) f[e] = 1.0f / w4w[e];
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) f[e] = 1.0f / w2[e];
  }
  scale_acc(st, f);
}

// This CTA's share of its unit's FP16-region tiles (FP16-tier chunks, tail, decode tokens),
// interleaved over the warps; pointers and ranges re-derived here (len_fp may have grown by
// decode appends: read after the programmatic-dependent-launch wait).
__device__ __forceinline__ void fp16_tiles(const DecArgs& a, const QS& qs, WarpState& st, int nq) {
  // thread coordinates re-read here (volatile): values carried from the kernel's start would be
  // spilled across the tile loop and reloaded in every iteration of this one
  uint32_t tid;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
  const int warp = (int)(tid >> 5), g = (int)((tid & 31) >> 2), c = (int)(tid & 3);
  const CtaIds id = cta_ids(a.Bc, a.b0, a.h0);
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
    if (tf + kDecWarps < f_end)
      prefetch_fp16_tile(kf + (int64_t)(r + kDecWarps * kTile) * kHeadDim, vf + (int64_t)(r + kDecWarps * kTile) * kHeadDim,
                         (int)(tid & 31));
    tile_fp16(kf + (int64_t)r * kHeadDim, vf + (int64_t)r * kHeadDim, len_fp - r, qs, st, g, c);
  }
}

// Finish a warp: add the V zero-point sums of each m-tile's group (held by lanes (G, c)) and
// reduce the row sums over the 8 row-groups.
__device__ __forceinline__ void finish_warp(WarpState& st, int c) {
#pragma unroll
  for (int G = 0; G < 4; ++G) {
    const float l0 = __shfl_sync(0xffffffffu, st.lacc[0], 4 * G + c);
    const float l1 = __shfl_sync(0xffffffffu, st.lacc[1], 4 * G + c);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      st.acc[2 * G + h][0] += l0; st.acc[2 * G + h][1] += l1;
      st.acc[2 * G + h][2] += l0; st.acc[2 * G + h][3] += l1;
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    st.lsum[0] += __shfl_xor_sync(0xffffffffu, st.lsum[0], o);
    st.lsum[1] += __shfl_xor_sync(0xffffffffu, st.lsum[1], o);
  }
  st.lsum[0] += st.lsq[0];  // already summed over the 16 tokens of every tile
  st.lsum[1] += st.lsq[1];
}
// head-dim index of accumulator element (mt, e2 = element >> 1) of lane row-group g
__device__ __forceinline__ int acc_d(int mt, int e2, int g) { return 32 * (mt >> 1) + 4 * g + 2 * (mt & 1) + e2; }

// ---- q staging (shared by both decode kernels) -----------------------------------------
// the unit's V exponent F (span_max is build-time data: readable before the PDL wait)
__device__ __forceinline__ int unit_v_exponent(const DecArgs& a, int l, int b, int h) {
  const int64_t fidx = ((int64_t)l * a.H + h) * a.B + b;  // [L][H][B]
  return a.V.span_max ? v_exponent(__uint_as_float(a.V.span_max[fidx])) : 0;
}

// Quarter staging: one warp stages group G of every set for one unit (a quarter of the q values:
// one 16-byte load per lane), in two phases around a barrier that combines the quarters' max |q|.
// q row g (zero if >= m), elements 32G + 8c + [0, 8), scaled to log2 units and rounded like the
// fp16 operand.
__device__ __forceinline__ void load_q_quarter(const DecArgs& a, int l, int b, int h, int G, int g, int c,
                                               float (&qv)[8]) {
  const uint16_t* qrow = a.q + l * a.q_sl + b * a.q_sb + (int64_t)(h * a.m + g) * kHeadDim + 32 * G + 8 * c;
  uint4 x = make_uint4(0u, 0u, 0u, 0u);
  if (g < a.m) x = *reinterpret_cast<const uint4*>(qrow);
  const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __half22float2(u32_as_h2(w4[e]));
    qv[2 * e] = __half2float(__float2half_rn(f.x * a.scale_log2));
    qv[2 * e + 1] = __half2float(__float2half_rn(f.y * a.scale_log2));
  }
}
// phase 1: the quarter's max |q| (returned, warp-uniform) and its zero-point entries (lanes c == G)
__device__ __forceinline__ float stage_q_quarter_aug(const float (&qv)[8], int G, int lane, unsigned char* s_qu) {
  float mx = 0.f, P = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) { mx = fmaxf(mx, fabsf(qv[e])); P += qv[e]; }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  P += __shfl_xor_sync(0xffffffffu, P, 1);
  P += __shfl_xor_sync(0xffffffffu, P, 2);
  if ((lane & 3) == G) {  // lane (g, c = G): Q[g][G] as an fp16 (hi, lo) pair
    const __half qhi = __float2half_rn(P);
    const __half qlo = __float2half_rn(P - __half2float(qhi));
    reinterpret_cast<uint32_t*>(s_qu + 3 * kQSet)[lane] = h2_as_u32(__halves2half2(qhi, qlo));
  }
  return mx;
}
// phase 2: group G of the three fragment sets with the unit's exponent E
__device__ __forceinline__ void stage_q_quarter_sets(const float (&qv)[8], int G, int E, unsigned char* s_qu, int lane) {
#pragma unroll
  for (int part = 0; part < 3; ++part) {
    uint32_t v[4];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int j0 = part == 0 ? 4 * hh : 0, j1 = part == 0 ? 4 * hh + 2 : 4;
      const float w0 = part == 2 ? 1.0f : exp2f((float)(E - j0)), w1 = part == 2 ? 1.0f : exp2f((float)(E - j1));
      v[2 * hh] = h2_as_u32(__floats2half2_rn(qv[2 * hh] * w0, qv[4 + 2 * hh] * w0));
      v[2 * hh + 1] = h2_as_u32(__floats2half2_rn(qv[2 * hh + 1] * w1, qv[5 + 2 * hh] * w1));
    }
    reinterpret_cast<uint4*>(s_qu + part * kQSet + 512 * G)[lane] = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

// per-lane constants of the tile functions; `scratch` = this warp's kScratch bytes
__device__ __forceinline__ LaneOff lane_offsets(uint32_t scratch, int lane) {
  const int g = lane >> 2, c = lane & 3;
  LaneOff lo;
  lo.mk = -8 * lane;
  lo.mv = 16 * (4 * (g & 3) + c) - 16 * lane;
  lo.sk = scratch + 4 * lane;
  lo.kc = scratch + 16 * g;
  lo.vp = scratch + 256 + 8 * (4 * c + (g & 3));
  lo.vc = scratch + 256 + 32 * c;
  return lo;
}

__global__ void __launch_bounds__(kDecWarps * 32, kMinCtas) decode_kernel(const DecArgs a) {
  extern __shared__ __align__(128) unsigned char s_dyn[];  // ring: [warp][kWarpRing]
  unsigned char (*s_ring)[kWarpRing] = reinterpret_cast<unsigned char (*)[kWarpRing]>(s_dyn);
  __shared__ float s_ml[kDecWarps][8][2];
  __shared__ __align__(16) unsigned char s_q[kQBytes];
  __shared__ float s_qmax[kDecWarps];
  __shared__ int s_last;
  __shared__ __align__(16) unsigned char s_scr[kDecWarps][kScratch];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  __shared__ int64_t s_tr[12], s_tend[kDecWarps];
  if (threadIdx.x == 0 && (a.trace != nullptr)) { s_tr[0] = gtime(); s_tr[11] = 0; }
  // Segment lengths of the quantized arenas are immutable after the build; len_fp grows with
  // decode appends and is read only after the programmatic-dependent-launch wait below.
  // Split of the quantized tiles: every CTA takes the same 1/splits share of the INT2 tiles
  // AND of the INT4 tiles (and of the FP16-region tiles, fp16_tiles), so all CTAs carry the
  // same mix and finish together whatever the relative per-tile costs are.
  int cnt2, nloc;
  TileSrc src;  // tile-native arenas: a row range starting at a tile is contiguous bytes
  {
    const CtaIds id = cta_ids(a.Bc, a.b0, a.h0);
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
  const uint32_t ring_l = (uint32_t)__cvta_generic_to_shared(&s_ring[warp][0]) + 16 * lane;
  ring_init();
  if (cnt2 > 0) prologue<2>(cnt2, a, src, ring_l, warp);
  else prologue<4>(nloc, a, src, ring_l, warp);

  // Everything above touched only build-time data.  q, the FP16 region and len_fp may come
  // from the preceding kernel on the stream: wait for it (no-op without PDL), and let the next
  // decode launch (next layer) start its own prologue as soon as SMs free up.
  // the unit's V span bound is build-time data too: read it before the wait
  UnitScale us;
  {
    const CtaIds id = cta_ids(a.Bc, a.b0, a.h0);
    us.F = unit_v_exponent(a, id.l, id.b, id.h);
#if CKV_DEC_Q_PREFETCH
    // pull the unit's q rows into L2 while the previous launch drains (L2 is the point of
    // coherence: a producer writing q before the wait below still wins)
    if (warp == 0 && g < a.m)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.q + id.l * a.q_sl + id.b * a.q_sb +
                                                     (int64_t)(id.h * a.m + g) * kHeadDim + 32 * c));
#endif
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if !CKV_DEC_LATE_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[1] = gtime();

  // Q B-fragments (scaled to log2 units), q-row i = g (zero if g >= m):
  // warp w stages group G = w of every set (a quarter of the q values each: one 16-byte load per
  // lane), the unit's max |q| combined through shared memory
  {
    const CtaIds id = cta_ids(a.Bc, a.b0, a.h0);
    float qv[8];
    if (warp < 4) {
      load_q_quarter(a, id.l, id.b, id.h, warp, g, c, qv);
      const float mx = stage_q_quarter_aug(qv, warp, lane, s_q);
      if (lane == 0) s_qmax[warp] = mx;
    }
    __syncthreads();
    us.E = q_exponent(fmaxf(fmaxf(s_qmax[0], s_qmax[1]), fmaxf(s_qmax[2], s_qmax[3])));
    if (warp < 4) stage_q_quarter_sets(qv, warp, us.E, s_q, lane);
  }
  __syncthreads();
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[2] = gtime();
  QS qs;
  qs.base = (uint32_t)__cvta_generic_to_shared(s_q) + 16 * lane;
  qs.aug_addr = (uint32_t)__cvta_generic_to_shared(s_q) + 3 * kQSet + 4 * lane;
  const LaneOff lo = lane_offsets((uint32_t)__cvta_generic_to_shared(&s_scr[warp][0]), lane);

  WarpState st;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) st.acc[mt][0] = st.acc[mt][1] = st.acc[mt][2] = st.acc[mt][3] = 0.f;
  st.lacc[0] = st.lacc[1] = 0.f;
  st.lsq[0] = st.lsq[1] = 0.f;
  st.mrun[0] = st.mrun[1] = -INFINITY;
  st.lsum[0] = st.lsum[1] = 0.f;

  quantized_tiles(cnt2, nloc - cnt2, a, src, lo, ring_l, qs, us, st, warp);
  fp16_tiles(a, qs, st, nloc);
#if CKV_DEC_LATE_TRIGGER == 1
  // the next launch on the stream may start once every CTA of this one is past its tiles: its
  // early CTAs then wait a merge tail for this layer, not a whole tile phase, in SM slots other
  // launches' tiles could use
  asm volatile("griddepcontrol.launch_dependents;");
#endif

  if (lane == 0 && (a.trace != nullptr)) s_tend[warp] = gtime();
  finish_warp(st, c);
  __syncthreads();  // ring -> merge buffer reuse
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[8] = gtime();
  float (*s_acc)[8][kHeadDim] = reinterpret_cast<float (*)[8][kHeadDim]>(&s_ring[0][0]);
  // only the m real q rows; column of (row, d) = d XOR ((row / 2) & 3), so the lanes of one
  // store instruction (rows 2c, 2c+1 x d = 32G + 4g + e) hit 32 distinct banks
  {
    const bool r0 = 2 * c < a.m, r1 = 2 * c + 1 < a.m;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      if (r0) {
        s_acc[warp][2 * c][acc_d(mt, 0, g) ^ c] = st.acc[mt][0];
        s_acc[warp][2 * c][acc_d(mt, 1, g) ^ c] = st.acc[mt][2];
      }
      if (r1) {
        s_acc[warp][2 * c + 1][acc_d(mt, 0, g) ^ c] = st.acc[mt][1];
        s_acc[warp][2 * c + 1][acc_d(mt, 1, g) ^ c] = st.acc[mt][3];
      }
    }
  }
  if (g == 0) {
    s_ml[warp][2 * c][0] = st.mrun[0]; s_ml[warp][2 * c][1] = st.lsum[0];
    s_ml[warp][2 * c + 1][0] = st.mrun[1]; s_ml[warp][2 * c + 1][1] = st.lsum[1];
  }
  __syncthreads();
  // merge the 4 warps: thread -> d
  const CtaIds id = cta_ids(a.Bc, a.b0, a.h0);
  const int split = id.split, h = id.h, l = id.l, b = id.b;
  const int d = threadIdx.x;
  const int hq0 = h * a.m;
  const int Hq = a.H * a.m;
  for (int qi = 0; qi < a.m && d < kHeadDim; ++qi) {
    float ms = -INFINITY;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) ms = fmaxf(ms, s_ml[w][qi][0]);
    float acc = 0.f, lsum = 0.f;
    const int dsw = d ^ ((qi >> 1) & 3);  // the parking swizzle
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) {
      const float mw = s_ml[w][qi][0];
      const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - ms);
      acc += f * s_acc[w][qi][dsw];
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
    if (threadIdx.x == 0 && (a.trace != nullptr)) {
      s_tr[3] = s_tend[0];
      s_tr[4] = gtime();
      int64_t* dst = a.trace + 16 * atomicAdd(&g_trace_n, 1ull);
      for (int i = 0; i < 5; ++i) dst[i] = s_tr[i];
      for (int i = 8; i < 12; ++i) dst[i] = s_tr[i];
      for (int i = 0; i < 4; ++i) dst[12 + i] = s_tend[i];
      // launch position | split << 20 | (sequence * H + kv head) << 40
      dst[5] = smid();
      dst[6] = (int64_t)((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) | ((int64_t)split << 20) |
               ((int64_t)(b * a.H + h) << 40);
      dst[7] = (int64_t)a.q;
    }
  };
#if CKV_DEC_LATE_TRIGGER == 2
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  if (a.splits == 1) { trace_out(); return; }
  // split-KV: the last CTA of this unit to arrive merges all partials (in-launch, no 2nd
  // kernel).  The CTA barrier orders every thread's partial stores before thread 0's
  // device-scope release RMW; the acquiring side sees them after its own barrier.
  __syncthreads();
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[9] = gtime();
  if (threadIdx.x == 0) {
    cuda::atomic_ref<uint32_t, cuda::thread_scope_device> ctr(a.counters[((int64_t)l * a.B + b) * a.H + h]);
    const uint32_t prev = ctr.fetch_add(1u, cuda::memory_order_acq_rel);
    s_last = prev == (uint32_t)(a.splits - 1);
    if (s_last) ctr.store(0u, cuda::memory_order_relaxed);  // ready for the next launch
  }
  __syncthreads();
  if (threadIdx.x == 0 && (a.trace != nullptr)) { s_tr[10] = gtime(); s_tr[11] = s_last; }
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
    for (int qi = 0; qi < a.m && d < kHeadDim; ++qi) {
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
  for (int qi = 0; qi < a.m && d < kHeadDim; ++qi) {
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

// Plan table (ckv_decode_wp_plan, device memory), int32:
//   warp records [16 * ctas][8]: unit u, k | np << 16 (the warp's index in its CTA's part of
//     the unit, the part's warps), INT2 / INT4 tiles of the warp's part, first INT2 / INT4 row
//     of the part in the unit's segment (seq off + tile share), w_lo | w_hi << 16 (the part's
//     warps within the unit's nw), nw;
//   CTA records [ctas][4]: first unit u0, unit slots;
//   slot records [ctas][8][4]: the slot unit's warps [x, y) within the CTA, first / last CTA.
// Every CTA reads its records with independent loads (no dependent chain before its prologue).
constexpr int kPlanWarpInts = 8, kPlanCtaInts = 4, kPlanSlots = 8;
constexpr int64_t kMergeSpin = 20000;  // ns a designated merger waits for its unit's partners
struct WpArgs {
  DecArgs d;
  const int32_t* plan;
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
  __shared__ __align__(16) unsigned char s_scr[kWpWarps][kScratch];
  __shared__ int s_lastu[8], s_do[8];
  __shared__ float s_qmax[4 * kPlanSlots];  // per (slot, group) max |q| of the q staging
  __shared__ int4 s_slot[8];             // per unit slot: warps [x, y) of this CTA, first / last CTA of the unit
  __shared__ unsigned short s_rtab[64];  // merge row r -> (slot << 8 | q row)
  __shared__ int64_t s_tr[12], s_tend[kWpWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int cta = blockIdx.x, l = blockIdx.z;
  if (threadIdx.x == 0 && (a.trace != nullptr)) { s_tr[0] = gtime(); s_tr[11] = 0; }
  const int gw = cta * kWpWarps + warp;
  const int nctas = gridDim.x;
  const int4* wrec = reinterpret_cast<const int4*>(w.plan) + 2 * gw;
  const int4 r0 = __ldg(wrec), r1 = __ldg(wrec + 1);
  const int4 crec = __ldg(reinterpret_cast<const int4*>(w.plan + kPlanWarpInts * kWpWarps * nctas) + cta);
  const int u = r0.x, u0 = crec.x, nslots = crec.y;
  // this CTA's part of the unit: its warps [w_lo, w_hi) of the unit's nw take a contiguous share
  // of each tile kind (adjacent tiles on one SM), interleaved inside
  const int k = r0.y & 0xffff, np = r0.y >> 16;  // this warp's index among the part's np warps
  const int w_lo = r1.z & 0xffff, w_hi = r1.z >> 16, nw = r1.w;
  const int slot = u - u0;
  const int b = a.b0 + u / a.H, h = u % a.H;  // units of this launch: sequences [b0, b0 + Bc)
  const int n2t = r0.z, n4t = r0.w;
  TileSrc src;
  {
    const int64_t unit = (int64_t)l * a.H + h;
    src.c2 = (unit * a.K.rows2 + r1.x) / kTileRows * kBlock2 + 16 * lane;
    src.c4 = (unit * a.K.rows4 + r1.y) / kTileRows * kBlock4 + 16 * lane;
  }
  const uint32_t ring_l = (uint32_t)__cvta_generic_to_shared(&s_ring[warp][0]) + 16 * lane;
  ring_init();
  if (n2t > 0) prologue<2>(n2t, a, src, ring_l, k, np);
  else prologue<4>(n4t, a, src, ring_l, k, np);
  UnitScale us;
  us.F = unit_v_exponent(a, l, b, h);
  // per-slot facts for the merge (build-time plan data: before the wait)
  if ((int)threadIdx.x < nslots) {
    s_slot[threadIdx.x] = __ldg(reinterpret_cast<const int4*>(w.plan + (kPlanWarpInts * kWpWarps + kPlanCtaInts) * nctas) +
                                kPlanSlots * cta + threadIdx.x);
    s_do[threadIdx.x] = 0;
  }
  if ((int)threadIdx.x < nslots * a.m)
    s_rtab[threadIdx.x] = (unsigned short)(((threadIdx.x / a.m) << 8) | (threadIdx.x % a.m));
  // pull this warp's q rows into L2 while the previous launch drains (L2 is the point of
  // coherence: a producer writing q before the wait below still wins; a prefetch reads nothing
  // into this SM)
  if (g < a.m) {
    const uint16_t* qrow = a.q + l * a.q_sl + b * a.q_sb + (int64_t)(h * a.m + g) * kHeadDim + 32 * c;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow));  // the row's 4 lanes cover its 256 B
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");  // (after the tiles instead: no change, 1 CTA/SM)
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[1] = gtime();

  // q staging: every unit slot of the CTA needs groups 0-3 of every set; job j = (slot j / 4,
  // group j % 4) goes to warp j % 16 (a quarter of the slot's q per job), in two phases around
  // the barrier that combines each slot's quarter maxima into its exponent
  {
    float qv[8];  // the warp's first job's quarter (kept for phase 2; further jobs reload)
    const int uj0 = u0 + (warp >> 2);
    if (warp < 4 * nslots) load_q_quarter(a, l, a.b0 + uj0 / a.H, uj0 % a.H, warp & 3, g, c, qv);
    for (int j = warp; j < 4 * nslots; j += kWpWarps) {
      const int uj = u0 + (j >> 2);
      float qj[8];
      if (j == warp) {
#pragma unroll
        for (int e = 0; e < 8; ++e) qj[e] = qv[e];
      } else {
        load_q_quarter(a, l, a.b0 + uj / a.H, uj % a.H, j & 3, g, c, qj);
      }
      const float mx = stage_q_quarter_aug(qj, j & 3, lane, s_qall + (j >> 2) * kQBytes);
      if (lane == 0) s_qmax[j] = mx;
    }
    __syncthreads();
    auto slot_e = [&](int sl) {
      return q_exponent(fmaxf(fmaxf(s_qmax[4 * sl], s_qmax[4 * sl + 1]), fmaxf(s_qmax[4 * sl + 2], s_qmax[4 * sl + 3])));
    };
    us.E = slot_e(slot);
    for (int j = warp; j < 4 * nslots; j += kWpWarps) {
      const int uj = u0 + (j >> 2);
      float qj[8];
      if (j == warp) {
#pragma unroll
        for (int e = 0; e < 8; ++e) qj[e] = qv[e];
      } else {
        load_q_quarter(a, l, a.b0 + uj / a.H, uj % a.H, j & 3, g, c, qj);
      }
      stage_q_quarter_sets(qj, j & 3, slot_e(j >> 2), s_qall + (j >> 2) * kQBytes, lane);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[2] = gtime();
  QS qs;
  qs.base = (uint32_t)__cvta_generic_to_shared(s_qall + slot * kQBytes) + 16 * lane;
  qs.aug_addr = (uint32_t)__cvta_generic_to_shared(s_qall + slot * kQBytes) + 3 * kQSet + 4 * lane;
  const LaneOff lo = lane_offsets((uint32_t)__cvta_generic_to_shared(&s_scr[warp][0]), lane);

  WarpState st;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) st.acc[mt][0] = st.acc[mt][1] = st.acc[mt][2] = st.acc[mt][3] = 0.f;
  st.lacc[0] = st.lacc[1] = 0.f;
  st.lsq[0] = st.lsq[1] = 0.f;
  st.mrun[0] = st.mrun[1] = -INFINITY;
  st.lsum[0] = st.lsum[1] = 0.f;

  // this warp's FP16-region tiles: the unit's, continuing the rotation after the quantized ones
  auto fp16_part = [&]() {
    const int off_fp = reinterpret_cast<const int*>(a.seq)[8 * b + 4];
    const int len_fp = reinterpret_cast<const int*>(a.seq)[8 * b + 5];
    const int nft = (len_fp + kTile - 1) / kTile;
    const int f_begin = (int)((int64_t)nft * w_lo / nw), f_end = (int)((int64_t)nft * w_hi / nw);
    const int64_t unit = (int64_t)l * a.H + h;
    const uint16_t* kf = a.K.fp + (unit * a.K.rows_fp + off_fp) * kHeadDim;
    const uint16_t* vf = a.V.fp + (unit * a.V.rows_fp + off_fp) * kHeadDim;
    for (int tf = f_begin + rotate(k, n2t + n4t, np); tf < f_end; tf += np) {
      const int r = tf * kTile;
      tile_fp16(kf + (int64_t)r * kHeadDim, vf + (int64_t)r * kHeadDim, len_fp - r, qs, st, g, c);
    }
  };
  quantized_tiles(n2t, n4t, a, src, lo, ring_l, qs, us, st, k, np);
  fp16_part();
  finish_warp(st, c);
  if (lane == 0 && (a.trace != nullptr)) s_tend[warp] = gtime();
  // Park this warp's partial (rows < m) in its own ring region (its copies are all waited:
  // no barrier needed before the stores).  Column of (q row, d): d XOR (row / 2) in its low 2
  // bits — a store instruction writes rows 2c (+1) x d = 32G + 4g + e: 32 distinct banks.
  auto swz = [](int row, int d) { return d ^ ((row >> 1) & 3); };
  {
    __syncwarp();
    float (*s_accw)[kHeadDim] = reinterpret_cast<float (*)[kHeadDim]>(&s_ring[warp][0]);
    const bool r0 = 2 * c < a.m, r1 = 2 * c + 1 < a.m;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      if (r0) {
        s_accw[2 * c][swz(2 * c, acc_d(mt, 0, g))] = st.acc[mt][0];
        s_accw[2 * c][swz(2 * c, acc_d(mt, 1, g))] = st.acc[mt][2];
      }
      if (r1) {
        s_accw[2 * c + 1][swz(2 * c + 1, acc_d(mt, 0, g))] = st.acc[mt][1];
        s_accw[2 * c + 1][swz(2 * c + 1, acc_d(mt, 1, g))] = st.acc[mt][3];
      }
    }
    if (g == 0) {
      s_ml[warp][2 * c][0] = st.mrun[0]; s_ml[warp][2 * c][1] = st.lsum[0];
      s_ml[warp][2 * c + 1][0] = st.mrun[1]; s_ml[warp][2 * c + 1][1] = st.lsum[1];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[8] = gtime();
  // Split units: every CTA of the unit draws an arrival ticket now (its tiles are done); the one
  // with the last ticket merges the unit.  It keeps its own partial in shared memory and waits
  // only for CTAs that drew earlier tickets, i.e. that are running or done (no co-residency
  // assumption); the others publish their partial and signal.  Counters per (layer, unit):
  // [0] tickets, [1] published partials; the merger resets both.  The tickets' round trip
  // overlaps the in-CTA merge (stored just before its barrier).
  uint32_t* ctr_l = a.counters + 2 * (int64_t)l * w.U;
  const int tick_t = blockDim.x - 1 - threadIdx.x;  // the last threads draw the tickets
  int ticket = -1;
  if (tick_t < nslots) {
    const int4 si = s_slot[tick_t];
    if (si.z != si.w) ticket = (int)atomicAdd(ctr_l + 2 * (u0 + tick_t), 1u);
  }
  // in-CTA merge, one warp per merged row (slot, q row): lanes 0-15 read the slot's warps'
  // (m, l) and form the weights 2^(m_w - max); every lane then sums 4 columns d = 4 lane + k
  // over the slot's warps (one 128-bit shared load per warp: the parking swizzle only permutes
  // inside aligned groups of 4).  A unit entirely inside this CTA writes its output row, otherwise
  // this CTA's partial goes to shared memory (slot sl: ring region of warp sl, past the parked
  // warp partials; rows of kWsStride floats: acc, m, l).
  const int Hq = a.H * a.m;
  float* ws_l = a.ws + (int64_t)l * w.U * w.max_ctas * a.m * kWsStride;
  auto s_own = [&](int sl) { return reinterpret_cast<float*>(&s_ring[sl][8 * kHeadDim * 4]); };
  for (int r = warp; r < nslots * a.m; r += kWpWarps) {
    const int rt = s_rtab[r], sl = rt >> 8, qi = rt & 255;
    const int4 si = s_slot[sl];
    const bool mine = lane >= si.x && lane < si.y;  // lane v <-> the CTA's warp v
    const float mw = mine ? s_ml[lane & (kWpWarps - 1)][qi][0] : -INFINITY;
    float ms = mw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
    const float f = mine && mw != -INFINITY ? fast_exp2(mw - ms) : 0.f;
    float lsum = mine ? f * s_ml[lane & (kWpWarps - 1)][qi][1] : 0.f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    float ac[4] = {0.f, 0.f, 0.f, 0.f};
    const uint32_t col = (uint32_t)__cvta_generic_to_shared(&s_ring[0][0]) + (qi * kHeadDim + 4 * lane) * 4;
    for (int ww = si.x; ww < si.y; ++ww) {
      const float fw = __shfl_sync(0xffffffffu, f, ww);
      const uint4 x = lds128(col + ww * kWarpRing);
      ac[0] = fmaf(fw, __uint_as_float(x.x), ac[0]);
      ac[1] = fmaf(fw, __uint_as_float(x.y), ac[1]);
      ac[2] = fmaf(fw, __uint_as_float(x.z), ac[2]);
      ac[3] = fmaf(fw, __uint_as_float(x.w), ac[3]);
    }
    // stored column 4 lane + k holds d = 4 lane + (k ^ sw)
    const int sw = (qi >> 1) & 3;
    float o4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o4[k] = ac[k ^ sw];
    if (si.z == si.w) {
      const int us = u0 + sl, bs = a.b0 + us / a.H, hs = us % a.H;
      const int64_t row = ((int64_t)l * a.B + bs) * Hq + hs * a.m + qi;
      if (a.partial_out) {
        float* dst = a.partial_out + row * kPartStride;
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[4 * lane + k] = o4[k];
        if (lane == 0) { dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum; }
      } else {
        const __half2 h0 = __floats2half2_rn(o4[0] / lsum, o4[1] / lsum), h1 = __floats2half2_rn(o4[2] / lsum, o4[3] / lsum);
        *reinterpret_cast<uint2*>(a.out + l * a.o_sl + bs * a.o_sb + (int64_t)(hs * a.m + qi) * kHeadDim + 4 * lane) =
            make_uint2(h2_as_u32(h0), h2_as_u32(h1));
      }
    } else {  // the partial: shared memory (a merging CTA's own) and its workspace slot (published)
      float* dst = s_own(sl) + qi * kWsStride;
      float* gdst = ws_l + (((int64_t)(u0 + sl) * w.max_ctas + (cta - si.z)) * a.m + qi) * kWsStride;
      const float4 v4 = make_float4(o4[0], o4[1], o4[2], o4[3]);
      *reinterpret_cast<float4*>(dst + 4 * lane) = v4;
      __stcg(reinterpret_cast<float4*>(gdst + 4 * lane), v4);
      if (lane == 0) {
        dst[kHeadDim] = ms; dst[kHeadDim + 1] = lsum;
        __stcg(gdst + kHeadDim, ms); __stcg(gdst + kHeadDim + 1, lsum);
      }
    }
  }
  if (tick_t < nslots) s_lastu[tick_t] = ticket;
  __syncthreads();
  if (threadIdx.x == 0 && (a.trace != nullptr)) s_tr[9] = gtime();
  // Roles per split unit: the CTA with ticket 0 (the first to finish its tiles) is the designated
  // merger: it keeps its partial in shared memory and waits for the others' published partials,
  // for at most kMergeSpin ns; the others publish theirs and count them in the unit's done
  // counter.  A merger that times out (e.g. a partner CTA not yet resident because a concurrent
  // launch holds the SMs) publishes its own partial and leaves; then the CTA whose count completes
  // the set (old value nc - 1) merges.  Exactly one CTA merges, no CTA waits unboundedly.
  // (every split partial is already in its workspace slot: the merge above wrote it there too)
  bool any_pub = false, any_mrg = false;
  for (int sl = 0; sl < nslots; ++sl) {
    const int tk = s_lastu[sl];
    any_mrg |= tk == 0;
    any_pub |= tk > 0;
  }
  if (any_pub) {
    // (the barrier above ordered every thread's partial stores before the device-scope release)
    if ((int)threadIdx.x < nslots) {
      const int4 si = s_slot[threadIdx.x];
      const int tk = s_lastu[threadIdx.x];
      if (tk > 0) {
        cuda::atomic_ref<uint32_t, cuda::thread_scope_device> done(ctr_l[2 * (u0 + threadIdx.x) + 1]);
        s_do[threadIdx.x] = done.fetch_add(1u, cuda::memory_order_acq_rel) == (uint32_t)(si.w - si.z);
      }
    }
  }
  if (threadIdx.x == 0 && (a.trace != nullptr)) {
    s_tr[10] = gtime();
    int nl = 0;
    for (int i = 0; i < nslots; ++i) nl += s_lastu[i] == 0;
    s_tr[11] = nl;
  }
  // designated mergers: warp sl waits for slot sl's partners (bounded), or resigns
  if (any_mrg && warp < nslots && s_lastu[warp] == 0) {
    const int4 si = s_slot[warp];
    const uint32_t others = (uint32_t)(si.w - si.z);
    cuda::atomic_ref<uint32_t, cuda::thread_scope_device> done(ctr_l[2 * (u0 + warp) + 1]);
    int got = 0;
    if (lane == 0) {
      const int64_t t0 = gtime();
      while (true) {
        if (done.load(cuda::memory_order_acquire) == others) { got = 1; break; }
        if (gtime() - t0 > kMergeSpin) break;
        __nanosleep(64);
      }
    }
    got = __shfl_sync(0xffffffffu, got, 0);
    if (!got) {  // resign: count the own partial (already in its workspace slot)
      if (lane == 0) got = done.fetch_add(1u, cuda::memory_order_acq_rel) == others;
      got = __shfl_sync(0xffffffffu, got, 0);
    }
    if (lane == 0) s_do[warp] = got;
  }
  if (any_pub || any_mrg) __syncthreads();
  if ((int)threadIdx.x < nslots && s_do[threadIdx.x]) {  // the merging CTA resets the unit's counters
    ctr_l[2 * (u0 + threadIdx.x) + 1] = 0u;
    ctr_l[2 * (u0 + threadIdx.x)] = 0u;
  }
  // every unit this CTA merges: all partials in CTA order (its own from shared memory, the
  // others from L2), all units' rows at once
  for (int p = threadIdx.x; (any_pub || any_mrg) && p < nslots * a.m * kHeadDim; p += blockDim.x) {
    const int d = p & (kHeadDim - 1), rt = s_rtab[p >> 7];
    const int sl = rt >> 8, qi = rt & 255;
    const int4 si = s_slot[sl];
    if (!s_do[sl]) continue;
    const int us = u0 + sl, nc = si.w - si.z + 1;
    const int bs = a.b0 + us / a.H, hs = us % a.H;
    const float* src_p = ws_l + (int64_t)us * w.max_ctas * a.m * kWsStride;  // [ctas][m][stride]
    {
      const float* own = s_own(sl) + qi * kWsStride;
      // every CTA's (m, acc, l) in CTA order (the merger's own from shared memory; the sum order
      // does not depend on which CTA arrived last): one L2 round trip
      constexpr int kMaxParts = 8;
      float mv[kMaxParts], xv[kMaxParts], lv[kMaxParts];
      const int np0 = min(nc, kMaxParts);
#pragma unroll
      for (int s2 = 0; s2 < kMaxParts; ++s2) {
        if (s2 >= np0) break;
        const float* ps = si.z + s2 == cta ? own : src_p + (s2 * a.m + qi) * kWsStride;
        mv[s2] = si.z + s2 == cta ? ps[kHeadDim] : __ldcg(ps + kHeadDim);
        xv[s2] = si.z + s2 == cta ? ps[d] : __ldcg(ps + d);
        lv[s2] = si.z + s2 == cta ? ps[kHeadDim + 1] : __ldcg(ps + kHeadDim + 1);
      }
      float ms = -INFINITY;
#pragma unroll
      for (int s2 = 0; s2 < kMaxParts; ++s2)
        if (s2 < np0) ms = fmaxf(ms, mv[s2]);
      float acc = 0.f, lsum = 0.f;
#pragma unroll
      for (int s2 = 0; s2 < kMaxParts; ++s2) {
        if (s2 >= np0) break;
        const float f = mv[s2] == -INFINITY ? 0.f : fast_exp2(mv[s2] - ms);
        acc = fmaf(f, xv[s2], acc);
        lsum = fmaf(f, lv[s2], lsum);
      }
      for (int s2 = kMaxParts; s2 < nc; ++s2) {  // units over more than 8 CTAs: the rest streamed
        const float* ps = si.z + s2 == cta ? own : src_p + (s2 * a.m + qi) * kWsStride;
        const float mw = si.z + s2 == cta ? ps[kHeadDim] : __ldcg(ps + kHeadDim);
        const float mn = fmaxf(ms, mw);
        const float fo = ms == -INFINITY ? 0.f : fast_exp2(ms - mn);
        const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - mn);
        acc = fmaf(f, si.z + s2 == cta ? ps[d] : __ldcg(ps + d), acc * fo);
        lsum = fmaf(f, si.z + s2 == cta ? ps[kHeadDim + 1] : __ldcg(ps + kHeadDim + 1), lsum * fo);
        ms = mn;
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
  }
  if (threadIdx.x == 0 && (a.trace != nullptr)) {
    int64_t tmax = 0;
    for (int i = 0; i < kWpWarps; ++i) tmax = max(tmax, s_tend[i]);
    s_tr[3] = tmax;
    s_tr[4] = gtime();
    int64_t* dst = a.trace + 16 * atomicAdd(&g_trace_n, 1ull);
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

// The same merge with the P partial arrays given by pointer (each [rows][130]): peer buffers of
// a symmetric-memory allocation, read over NVLink by ordinary loads (split-KV exchange without a
// gathered copy).
__global__ void lse_merge_ptrs_kernel(const float* const* __restrict__ parts, int P, int64_t rows,
                                      uint16_t* __restrict__ out) {
  const int64_t row = blockIdx.x;
  const int d = threadIdx.x;
  constexpr int kMax = 8;
  float mv[kMax], xv[kMax], lv[kMax];
  float ms = -INFINITY;
#pragma unroll
  for (int p = 0; p < kMax; ++p) {  // every peer's (m, acc[d], l) in flight at once
    if (p < P) {
      const float* q = parts[p] + row * kPartStride;
      mv[p] = __ldcv(q + kHeadDim);
      xv[p] = __ldcv(q + d);
      lv[p] = __ldcv(q + kHeadDim + 1);
      ms = fmaxf(ms, mv[p]);
    }
  }
  float acc = 0.f, lsum = 0.f;
#pragma unroll
  for (int p = 0; p < kMax; ++p) {
    if (p < P) {
      const float f = mv[p] == -INFINITY ? 0.f : fast_exp2(mv[p] - ms);
      acc += f * xv[p];
      lsum += f * lv[p];
    }
  }
  for (int p = kMax; p < P; ++p) {  // more than 8 ranks: the rest streamed
    const float* q = parts[p] + row * kPartStride;
    const float mw = __ldcv(q + kHeadDim), mn = fmaxf(ms, mw);
    const float fo = ms == -INFINITY ? 0.f : fast_exp2(ms - mn), f = mw == -INFINITY ? 0.f : fast_exp2(mw - mn);
    acc = fmaf(f, __ldcv(q + d), acc * fo);
    lsum = fmaf(f, __ldcv(q + kHeadDim + 1), lsum * fo);
    ms = mn;
  }
  out[row * kHeadDim + d] = __half_as_ushort(__float2half_rn(acc / lsum));
}

}  // namespace ckv

using namespace ckv;

static int64_t* g_trace_host = nullptr;  // ckv_decode_set_trace: copied into every launch's DecArgs

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
  return ckv_decode_attention_range(q, q_s_layer, q_s_batch, k_arena, v_arena, seq, layers, batch, seq_begin,
                                    seq_count, kv_heads, 0, kv_heads, m, scale, splits, workspace, out,
                                    o_s_layer, o_s_batch, partial_out, flags, stream);
}

int32_t ckv_decode_attention_range(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                   ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                   int32_t layers, int32_t batch, int32_t seq_begin, int32_t seq_count,
                                   int32_t kv_heads, int32_t head_begin, int32_t head_count, int32_t m,
                                   float scale, int32_t splits, void* workspace, uint16_t* out,
                                   int64_t o_s_layer, int64_t o_s_batch, float* partial_out, int32_t flags,
                                   void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0 || splits < 1) return CKV_ERR_ARG;
  if (seq_begin < 0 || seq_count < 0 || seq_begin + seq_count > batch) return CKV_ERR_ARG;
  if (head_begin < 0 || head_count < 0 || head_begin + head_count > kv_heads) return CKV_ERR_ARG;
  if (head_count == 0) return CKV_OK;
  if (m < 1 || m > 8) return CKV_ERR_UNSUPPORTED;
  if (!q || !seq || (!out && !partial_out)) return CKV_ERR_ARG;
  if (splits > 1 && !workspace) return CKV_ERR_ARG;
  if ((q_s_layer % 8) || (q_s_batch % 8) || (o_s_layer % 8) || (o_s_batch % 8)) return CKV_ERR_UNSUPPORTED;
  if (out && (reinterpret_cast<uintptr_t>(out) & 15)) return CKV_ERR_UNSUPPORTED;
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
    if (!v_arena.span_max && (v_arena.rows2 || v_arena.rows4)) return CKV_ERR_ARG;  // sizes the V operand scaling
  }
  DecArgs a;
  a.q = q; a.q_sl = q_s_layer; a.q_sb = q_s_batch;
  a.K = k_arena; a.V = v_arena; a.seq = seq;
  a.L = layers; a.B = batch; a.H = kv_heads; a.m = m; a.splits = splits;
  a.b0 = seq_begin; a.Bc = seq_count; a.h0 = head_begin;
  a.scale_log2 = scale * 1.4426950408889634f;
  const int64_t units = (int64_t)layers * batch * kv_heads;
  a.counters = reinterpret_cast<uint32_t*>(workspace);
  a.ws = workspace ? reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                              cdiv(units * (int64_t)sizeof(uint32_t), 256) * 256)
                   : nullptr;
  a.out = out; a.o_sl = o_s_layer; a.o_sb = o_s_batch;
  a.partial_out = partial_out;
  a.trace = g_trace_host;
  if (!ensure_decode_attr()) return CKV_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)splits, (unsigned)head_count, (unsigned)(layers * seq_count));
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
  g_trace_host = buf;
  if (cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z)) != cudaSuccess) {
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
  return cdiv(2 * units * (int64_t)sizeof(uint32_t), 256) * 256 +
         units * (int64_t)(max_ctas > 0 ? max_ctas : 1) * m * kWsStride * (int64_t)sizeof(float);
}

int64_t ckv_decode_wp_plan_ints(int32_t ctas) {
  return ctas < 1 ? 0 : (int64_t)ctas * (kPlanWarpInts * kWpWarps + kPlanCtaInts + 4 * kPlanSlots);
}

int32_t ckv_decode_wp_plan(const int32_t* seq_host, int32_t batch, int32_t kv_heads,
                           const int32_t* unit_warps, int32_t ctas, int32_t* plan_host,
                           int32_t* max_slots, int32_t* max_ctas) {
  if (!seq_host || !unit_warps || !plan_host || !max_slots || !max_ctas) return CKV_ERR_ARG;
  if (batch < 1 || kv_heads < 1 || ctas < 1) return CKV_ERR_ARG;
  const int U = batch * kv_heads, T = kWpWarps * ctas;
  int64_t total = 0;
  for (int u = 0; u < U; ++u) {
    if (unit_warps[u] < 1) return CKV_ERR_ARG;
    total += unit_warps[u];
  }
  if (total != T || U > T) return CKV_ERR_ARG;
  std::vector<int> prefix(U + 1, 0), wunit(T);
  for (int u = 0; u < U; ++u) prefix[u + 1] = prefix[u] + unit_warps[u];
  for (int u = 0; u < U; ++u)
    for (int x = prefix[u]; x < prefix[u + 1]; ++x) wunit[x] = u;
  int32_t* wr = plan_host;
  int32_t* cr = plan_host + (int64_t)kPlanWarpInts * T;
  int32_t* sr = cr + (int64_t)kPlanCtaInts * ctas;
  std::fill(plan_host, plan_host + ckv_decode_wp_plan_ints(ctas), 0);
  int ms = 0, mc = 0;
  for (int u = 0; u < U; ++u) mc = std::max(mc, (prefix[u + 1] - 1) / kWpWarps - prefix[u] / kWpWarps + 1);
  for (int c = 0; c < ctas; ++c) {
    const int u0 = wunit[c * kWpWarps], u1 = wunit[c * kWpWarps + kWpWarps - 1];
    const int ns = u1 - u0 + 1;
    if (ns > kPlanSlots) return CKV_ERR_UNSUPPORTED;
    ms = std::max(ms, ns);
    cr[kPlanCtaInts * c] = u0;
    cr[kPlanCtaInts * c + 1] = ns;
    for (int sl = 0; sl < ns; ++sl) {
      const int us = u0 + sl, q0 = prefix[us], q1 = prefix[us + 1];
      int32_t* x = sr + 4 * (kPlanSlots * c + sl);
      x[0] = std::max(q0, c * kWpWarps) - c * kWpWarps;
      x[1] = std::min(q1, c * kWpWarps + kWpWarps) - c * kWpWarps;
      x[2] = q0 / kWpWarps;
      x[3] = (q1 - 1) / kWpWarps;
    }
  }
  for (int gw = 0; gw < T; ++gw) {
    const int u = wunit[gw], c = gw / kWpWarps, b = u / kv_heads;
    const int p0 = prefix[u], p1 = prefix[u + 1], nw = p1 - p0;
    const int w_lo = std::max(p0, c * kWpWarps) - p0, w_hi = std::min(p1, c * kWpWarps + kWpWarps) - p0;
    const int32_t* s0 = seq_host + CKV_SEQ_FIELDS * b;
    const int64_t n2u = s0[1] / kTile, n4u = s0[3] / kTile;
    const int a2 = (int)(n2u * w_lo / nw), a4 = (int)(n4u * w_lo / nw);
    int32_t* x = wr + kPlanWarpInts * gw;
    x[0] = u;
    x[1] = (gw - p0 - w_lo) | ((w_hi - w_lo) << 16);
    x[2] = (int)(n2u * w_hi / nw) - a2;
    x[3] = (int)(n4u * w_hi / nw) - a4;
    x[4] = s0[0] + a2 * kTile;
    x[5] = s0[2] + a4 * kTile;
    x[6] = w_lo | (w_hi << 16);
    x[7] = nw;
  }
  *max_slots = ms;
  *max_ctas = mc;
  return CKV_OK;
}

int32_t ckv_decode_attention_wp(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                int32_t layers, int32_t batch, int32_t kv_heads, int32_t m, float scale,
                                const int32_t* plan, int32_t ctas, int32_t max_slots,
                                int32_t max_ctas, void* workspace, uint16_t* out, int64_t o_s_layer,
                                int64_t o_s_batch, float* partial_out, int32_t flags, void* stream) {
  return ckv_decode_attention_wp_seqs(q, q_s_layer, q_s_batch, k_arena, v_arena, seq, layers, batch, 0, batch,
                                      kv_heads, m, scale, plan, ctas, max_slots, max_ctas, workspace, out,
                                      o_s_layer, o_s_batch, partial_out, flags, stream);
}

int32_t ckv_decode_attention_wp_seqs(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                     ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                     int32_t layers, int32_t batch, int32_t b0, int32_t n_seqs,
                                     int32_t kv_heads, int32_t m, float scale, const int32_t* plan,
                                     int32_t ctas, int32_t max_slots, int32_t max_ctas, void* workspace,
                                     uint16_t* out, int64_t o_s_layer, int64_t o_s_batch,
                                     float* partial_out, int32_t flags, void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0 || ctas < 1) return CKV_ERR_ARG;
  if (b0 < 0 || n_seqs < 0 || b0 + n_seqs > batch) return CKV_ERR_ARG;
  if (m < 1 || m > 8) return CKV_ERR_UNSUPPORTED;
  if (max_slots < 1 || max_slots > 8 || max_ctas < 1) return CKV_ERR_UNSUPPORTED;
  if (!q || !seq || !plan || !workspace || (!out && !partial_out)) return CKV_ERR_ARG;
  if ((q_s_layer % 8) || (q_s_batch % 8) || (o_s_layer % 8) || (o_s_batch % 8)) return CKV_ERR_UNSUPPORTED;
  if (out && (reinterpret_cast<uintptr_t>(out) & 15)) return CKV_ERR_UNSUPPORTED;
  if (layers * n_seqs * kv_heads == 0) return CKV_OK;
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
    if (!v_arena.span_max && (v_arena.rows2 || v_arena.rows4)) return CKV_ERR_ARG;  // sizes the V operand scaling
  }
  WpArgs w;
  DecArgs& a = w.d;
  a.q = q; a.q_sl = q_s_layer; a.q_sb = q_s_batch;
  a.K = k_arena; a.V = v_arena; a.seq = seq;
  a.L = layers; a.B = batch; a.H = kv_heads; a.m = m; a.splits = 1;
  a.b0 = b0; a.Bc = n_seqs; a.h0 = 0;
  a.scale_log2 = scale * 1.4426950408889634f;
  const int64_t units = (int64_t)layers * n_seqs * kv_heads;
  a.counters = reinterpret_cast<uint32_t*>(workspace);
  a.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + cdiv(2 * units * (int64_t)sizeof(uint32_t), 256) * 256);
  a.out = out; a.o_sl = o_s_layer; a.o_sb = o_s_batch;
  a.partial_out = partial_out;
  a.trace = g_trace_host;
  w.plan = plan;
  w.U = n_seqs * kv_heads;  // the plan's units: sequences [b0, b0 + n_seqs) x kv heads
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

int32_t ckv_lse_merge_ptrs(const float* const* parts, int32_t n_parts, int64_t rows, uint16_t* out,
                           void* stream) {
  if (n_parts < 1 || rows < 0 || !parts || !out) return CKV_ERR_ARG;
  if (rows == 0) return CKV_OK;
  lse_merge_ptrs_kernel<<<(unsigned)rows, kHeadDim, 0, as_stream(stream)>>>(parts, n_parts, rows, out);
  CKV_LAUNCH_CHECK();
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
