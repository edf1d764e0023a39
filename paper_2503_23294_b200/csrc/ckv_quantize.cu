// Chunk-level KV reorder + quantize + pack (Module II, prefill side), batched over
// [layers, sequences, kv_heads].  One pass over fp16 K/V:
//   kv_store.build_cache           kv_store.py:169-219 (tier-contiguous gather, perm order)
//   quantizer.quantize             quantizer.py:60-83  (non-finite -> error flag)
//   kernels.quantize_groups        _numpy.py:27-67 / _core.pyx:27-79 (min-max, round-half-up)
//   kernels.pack_codes             _numpy.py:70-86 (row-major little-endian u32 words)
// plus the FP16 region (FP16-tier chunks || context tail, kv_store.py:199-202) and the
// decode-token append (kv_store.py:135-148, 222-224).
//
// Codes are bit-exact with the reference's float64 expression
//   code = floor((x - lo) * qmax / (hi - lo) + 0.5)
// For fp16 inputs that f64 result equals the exact rational floor((2(x-lo)qmax + span) / 2span)
// (x - lo and span are exact in f64; the two remaining roundings move the value by < 2^-49
// while a non-tie is >= 2^-42 from the boundary).  The kernel evaluates a fast fp32 candidate
// whose error is < 2^-17 and recomputes in IEEE f64 (same tree) only when the candidate lies
// within 2^-14 of a rounding boundary.
#include "ckv_common.cuh"

namespace ckv {

constexpr int kQWarps = 4;
constexpr float kGuard = 1.0f / 16384.0f;  // 2^-14

struct SeqRow {
  int off2, len2, off4, len4, off_fp, len_fp, tail_src, ctx;
};

__device__ __forceinline__ SeqRow load_seq(const int32_t* seq, int b) {
  const int4 a = reinterpret_cast<const int4*>(seq)[2 * b];
  const int4 c = reinterpret_cast<const int4*>(seq)[2 * b + 1];
  return SeqRow{a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
}

__device__ __forceinline__ uint32_t exact_code(float x, float lo, float hi, float qinv,
                                               float qmax) {
  const float t = fmaf(x - lo, qinv, 0.5f);
  float n = floorf(t);
  const float fr = t - n;
  if (fr < kGuard || fr > 1.0f - kGuard) {
    // IEEE f64 with the reference's tree (_numpy.py:61): ((x - m) * qmax) / span + 0.5
    const double dd = __dadd_rn(__ddiv_rn(__dmul_rn(__dsub_rn((double)x, (double)lo), (double)qmax),
                                          __dsub_rn((double)hi, (double)lo)), 0.5);
    n = (float)floor(dd);
  }
  n = fminf(fmaxf(n, 0.0f), qmax);
  return (uint32_t)n;
}

// Rare path: every element of a slice exactly (IEEE f64, reference tree); out of line so the
// quantize_chunk instantiations stay small.
__device__ __noinline__ uint32_t exact_slice(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                             float lo, float hi, float qinv, float qmax, uint32_t base) {
  const uint32_t w[4] = {w0, w1, w2, w3};
  uint32_t acc = 0u, p = 1u;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t hb = (w[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
    const float x = __half2float(__ushort_as_half((unsigned short)hb));
    acc += exact_code(x, lo, hi, qinv, qmax) * p;
    p *= base;
  }
  return acc;
}

// Codes per element, fast path (codes8 below, two elements per packed instruction):
//   d = x - lo                     [one mixed f16 - f32 subtract]
//   y = RN(d * qmax / span + 1.5*2^23)   [low mantissa bits = round-half-even]
//   |d * qmax / span - (y - 1.5*2^23)| > 0.5 - 2^-14  -> exact IEEE f64 recomputation (near a tie)
//   acc += bits(y) * base^e        [one IMAD; the constant offset is pre-subtracted]
// The fp32 value is within 3.6e-6 of the exact rational, so away from the guard band
// round-half-even == floor(exact + 0.5) == the reference's f64 result.
__device__ __forceinline__ uint32_t hmin2_nan(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.NaN.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmax2_nan(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t prmt_q(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// packed fp32x2 arithmetic (sm_100: FFMA2, two lanes of f32 per instruction)
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// Codes of 8 elements (4 half2 words) for a group with lower bound lo and qinv = qmax / span,
// packed as the reference's little-endian sub-word codes; element pairs in packed f32x2
// arithmetic (FFMA2: half the issue slots):
//   d = x - lo (fp16 - fp32, one rounding);  y = RN(d qinv + 1.5 2^23) (the code lands in y's low mantissa bits);
//   e = d qinv - (y - 1.5 2^23) (one rounding);  dmax = max |e| (the guard test)
template <int BITS>
__device__ __forceinline__ uint32_t codes8(const uint32_t* w, float lo, float qinv, float& dmax) {
  constexpr uint32_t base = BITS == 2 ? 4u : 16u;
  constexpr uint32_t kM = 0x4B400000u;  // bits of 1.5 * 2^23
  constexpr uint32_t kSum = BITS == 2 ? 21845u : 0x11111111u;  // sum_e base^e, e = 0..7
  uint32_t acc = 0u - kM * kSum;
  const uint64_t qi = f2pack(qinv, qinv), mm = f2pack(12582912.0f, 12582912.0f);
  const uint64_t neg1 = f2pack(-1.0f, -1.0f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float dx, dy;  // x - lo straight from the fp16 halves (mixed f16 - f32 subtract, one rounding)
    asm("{.reg .f16 a, b; mov.b32 {a, b}, %2; sub.rn.f32.f16 %0, a, %3; sub.rn.f32.f16 %1, b, %3;}"
        : "=f"(dx), "=f"(dy) : "r"(w[i]), "f"(lo));
    const uint64_t d = f2pack(dx, dy);
    const uint64_t y = ffma2(d, qi, mm);
    const uint64_t e = ffma2(d, qi, ffma2(y, neg1, mm));
    float e0, e1, y0, y1;
    f2unpack(e, e0, e1);
    f2unpack(y, y0, y1);
    dmax = fmaxf(dmax, fmaxf(fabsf(e0), fabsf(e1)));
    uint32_t p0 = 1u;
#pragma unroll
    for (int k = 0; k < 2 * i; ++k) p0 *= base;
    acc += __float_as_uint(y0) * p0 + __float_as_uint(y1) * (p0 * base);
  }
  return acc;
}

// One 16-element lane slice of a row (2 lanes = one 32-element group): group min / max in fp16
// with NaN propagation ((lo, -hi) travel as one half2, so one min reduces both across the lane
// pair), one scale, and the codes of both 8-element halves (c[0]: elements 0-7, c[1]: 8-15),
// each packed like the reference's words.  A half whose candidate lies within 2^-14 of a
// rounding boundary is recomputed in IEEE f64 (exact_slice, rare).
template <int BITS>
__device__ __forceinline__ void quantize_slice16(const uint32_t (&w)[8], uint32_t (&c)[2], uint32_t& meta,
                                                 float& smax) {
  constexpr float qmax = BITS == 2 ? 3.0f : 15.0f;
  constexpr uint32_t base = BITS == 2 ? 4u : 16u;
  const uint32_t mn = hmin2_nan(hmin2_nan(hmin2_nan(w[0], w[1]), hmin2_nan(w[2], w[3])),
                                hmin2_nan(hmin2_nan(w[4], w[5]), hmin2_nan(w[6], w[7])));
  const uint32_t nmx = hmax2_nan(hmax2_nan(hmax2_nan(w[0], w[1]), hmax2_nan(w[2], w[3])),
                                 hmax2_nan(hmax2_nan(w[4], w[5]), hmax2_nan(w[6], w[7]))) ^ 0x80008000u;
  uint32_t lh = hmin2_nan(prmt_q(mn, nmx, 0x5410), prmt_q(mn, nmx, 0x7632));
  lh = hmin2_nan(lh, __shfl_xor_sync(0xffffffffu, lh, 1));
  meta = lh ^ 0x80000000u;  // the group's fp16 (lo, hi)
  const float2 lhf = __half22float2(u32_as_h2(lh));
  const float lo = lhf.x, hi = -lhf.y;
  const float span = hi - lo;
  // NaN-propagating max: an inf / nan anywhere in a group makes its span inf or nan, so the
  // chunk's non-finite and wide-scale tests are on smax after the loop
  asm("max.NaN.f32 %0, %0, %1;" : "+f"(smax) : "f"(span));
  if (!(span > 0.0f)) {  // constant group: codes 0 (also nan groups; flagged from smax)
    c[0] = c[1] = 0u;
    return;
  }
  // qmax / span via the approximate reciprocal (<= 2 ulp): the candidate stays within 2^-17 of
  // the exact rational, well inside the 2^-14 guard band that triggers the exact path
  float rs;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(span));
  const float qinv = qmax * rs;
  float d0 = 0.0f, d1 = 0.0f;
  c[0] = codes8<BITS>(w, lo, qinv, d0);
  c[1] = codes8<BITS>(w + 4, lo, qinv, d1);
  constexpr float kNear = 0.5f - (1.0f / 16384.0f);
  if (d0 > kNear) c[0] = exact_slice(w[0], w[1], w[2], w[3], lo, hi, qinv, qmax, base);  // rare
  if (d1 > kNear) c[1] = exact_slice(w[4], w[5], w[6], w[7], lo, hi, qinv, qmax, base);
}

// Staging offsets of the tile-native layout (ckv_common.cuh tile_byte_* / tile_off_*): each
// pass computes a per-lane base once and adds (tile h) TB + (step it) part per store (the GPU
// parity tests read every arena back through ckv_arena_export, i.e. through the layout
// functions, and compare with the reference bit for bit).
template <int BITS> struct StageTB {
  static constexpr int TB = BITS == 2 ? kBlock2 : kBlock4;  // staging holds whole K/V blocks
};
template <int BITS, bool ISV> struct MetaStageOff {
  static constexpr int TB = BITS == 2 ? kBlock2 : kBlock4;
  static constexpr int X = ISV ? 8 : 4;
  static constexpr int U = ISV ? 16 : 64;
  __device__ __forceinline__ static int lane(int j, int sub) {  // lo; hi at + (ISV ? 4 : 2)
    return ISV ? (j >> 2) * 64 + sub * 2 : sub * 32 + (j >> 2) * 8;
  }
};

// One 32-row chunk of K (ISV = false) or V rows -> codes and (lo, hi) metadata staged in shared
// memory in the tile-native layout (2 tiles).  Lanes: rs = lane / 8 picks the row
// (rows 2 it + 16 h + (rs & 1) + 8 (rs >> 1)), jj = lane % 8 the 16-element slice (2 lanes = one 32-element group); each
// lane covers the reference's 8-element slices j = 2 jj, 2 jj + 1 of StageOff.  Row r of the
// chunk sits at StageOff's (r4, u, sub) = ((r >> 3) << 2, (r >> 1) & 3, r & 1).  Returns
// whether a group's scale needs the decode's wide-scale mode.
// L2 prefetch of the line holding p (no registers held; the demand load a step later hits L2)
__device__ __forceinline__ void l2_prefetch(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// 32-bit shared-memory stores (staging addresses are 32-bit shared-window offsets: no 64-bit
// generic pointer arithmetic in the quantize loops)
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");  // low byte of v
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t v0, uint32_t v1) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v0), "r"(v1) : "memory");
}

// After a chunk half: non-finite input anywhere (its span max is inf or nan) and the decode's
// wide-scale test (some group scale span / qmax above 4000).
__device__ __forceinline__ bool chunk_flags(float smax, float qmax, bool& bad) {
  bad |= !(smax < INFINITY);
  return smax > 4000.0f * qmax;
}

// V rows: lanes over 16 rows x the 2 halves of one group, so that a warp's V code and
// metadata stores fall in distinct banks (lanes over slices, as for K, would put the 64-byte
// slice stride of the V tile layout on 2 banks).  lane = 2 rr + hg: rows rr (+16 h), group it;
// elements 32 it + 8 hg + [0, 8) and 32 it + 16 + 8 hg + [0, 8), i.e. the reference's
// 8-element slices j = 4 it + hg and 4 it + 2 + hg (each load instruction reads a row's 32
// contiguous bytes with the lane pair).
template <int BITS>
__device__ __forceinline__ bool quantize_chunk_v(const uint16_t* src, int sT, int lane,
                                                 uint32_t sc, uint32_t sm, bool& bad, float& smax) {
  using MO = MetaStageOff<BITS, true>;
  constexpr int TB = StageTB<BITS>::TB;
  const int rr = lane >> 1, hg = lane & 1, sub = rr & 1;
  // row rr of tile h: lane (g = 2 hg (+1, +4, +5), c = (rr & 7) / 2); INT2 byte 2 (rr & 1) of
  // word 2 (rr >= 8) + it / 2 (+ it & 1 per step), INT4 half rr & 1 of word it in half rr >= 8
  const uint32_t cb = BITS == 2 ? sc + 128 * hg + 16 * ((rr & 7) >> 1) + 8 * (rr >> 3) + 2 * (rr & 1)
                                : sc + 512 * (rr >> 3) + 128 * hg + 16 * ((rr & 7) >> 1) + 2 * (rr & 1);
  const uint32_t mbase = sm + ((rr >> 3) & 1) * MO::X + ((rr >> 1) & 3) * MO::U + MO::lane(0, sub);
  const uint4* srow = reinterpret_cast<const uint4*>(src + (int64_t)rr * sT) + hg;
#pragma unroll 1
  for (int it = 0; it < 4; ++it) {  // group it, rows rr and rr + 16
    uint4 xs[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // four 16-byte loads in flight per lane
      const uint4* p = srow + (int64_t)(16 * h) * sT / 8 + 4 * it;
      xs[2 * h] = __ldg(p);
      xs[2 * h + 1] = __ldg(p + 2);
      if (it == 0) l2_prefetch(p + 8);  // the row's second 128-byte line (steps 2, 3)
    }
    // slices j0 = 4 it + hg and j0 + 2 (elements 32 it + 8 hg + [0, 8) and + 16)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t w[8] = {xs[2 * h].x, xs[2 * h].y, xs[2 * h].z, xs[2 * h].w,
                             xs[2 * h + 1].x, xs[2 * h + 1].y, xs[2 * h + 1].z, xs[2 * h + 1].w};
      uint32_t c[2], meta;
      quantize_slice16<BITS>(w, c, meta, smax);
      // c[0]: elements 32 it + 8 hg + [0, 8) -> lanes g = 2 hg, 2 hg + 1; c[1]: +16 -> g + 4
      if (BITS == 2) {
        const uint32_t c0 = cb + h * TB + 4 * (it >> 1) + (it & 1);
        sts8(c0, c[0]);
        sts8(c0 + 64, c[0] >> 8);
        sts8(c0 + 256, c[1]);
        sts8(c0 + 320, c[1] >> 8);
      } else {
        const uint32_t c0 = cb + h * TB + 4 * it;
        sts16(c0, c[0]);
        sts16(c0 + 64, c[0] >> 16);
        sts16(c0 + 256, c[1]);
        sts16(c0 + 320, c[1] >> 16);
      }
      // both lanes of the group hold the same (lo, hi): duplicate stores, no branch
      const uint32_t mb = mbase + h * MO::TB + it * 64;
      sts16(mb, meta);
      sts16(mb + 4, meta >> 16);
    }
  }
  return chunk_flags(smax, BITS == 2 ? 3.0f : 15.0f, bad);
}

template <int BITS, bool ISV>
__device__ __forceinline__ bool quantize_chunk(const uint16_t* src, int sT, int lane, uint32_t sc, uint32_t sm,
                                               bool& bad, float& smax) {
  if (ISV) return quantize_chunk_v<BITS>(src, sT, lane, sc, sm, bad, smax);
  using MO = MetaStageOff<BITS, ISV>;
  constexpr int TB = StageTB<BITS>::TB;
  const int rs = lane >> 3, jj = lane & 7;
  const int sub = rs & 1, j0 = 2 * jj, hi8 = rs >> 1;
  // the lane's row rt = 2 it + sub + 8 hi8 of tile h, reference word jj (INT2: bytes 4 jj ..
  // 4 jj + 3; INT4: words 2 jj, 2 jj + 1).  INT2: the rows rt and rt + 8 of a word interleave
  // byte by byte in the tile (lanes l, l ^ 16 hold them): one shuffle, then each lane stores
  // one whole 32-bit word (c = 2 (jj & 1) + hi8, group jj / 2).  INT4: word 2 jj + k -> lane
  // c = 2 (jj & 1) + k, group jj / 2, half hi8.  Every store instruction: distinct banks.
  const uint32_t cb = BITS == 2 ? sc + 64 * sub + 16 * (2 * (jj & 1) + hi8) + 4 * (jj >> 1)
                                : sc + 512 * hi8 + 64 * sub + 32 * (jj & 1) + 4 * (jj >> 1);
  const uint32_t sel = hi8 ? 0x3726u : 0x5140u;  // [lo.b0 hi.b0 lo.b1 hi.b1] / [lo.b2 hi.b2 lo.b3 hi.b3]
  const uint32_t mbase = sm + MO::lane(j0, sub) + (rs >> 1) * MO::X;
  const uint4* srow = reinterpret_cast<const uint4*>(src + (int64_t)(sub + 8 * (rs >> 1)) * sT) + 2 * jj;
#pragma unroll 1
  for (int it = 0; it < 4; ++it) {  // rows 2 it + 16 h + sub + 8 (rs >> 1)
    uint4 xs[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // four 16-byte loads in flight per lane
      const uint4* p = srow + (int64_t)(2 * it + 16 * h) * sT / 8;
      xs[2 * h] = __ldg(p);
      xs[2 * h + 1] = __ldg(p + 1);
      if (it < 3) l2_prefetch(p + 2 * sT / 8);  // this lane's piece of the next step's row
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t w[8] = {xs[2 * h].x, xs[2 * h].y, xs[2 * h].z, xs[2 * h].w,
                             xs[2 * h + 1].x, xs[2 * h + 1].y, xs[2 * h + 1].z, xs[2 * h + 1].w};
      uint32_t c[2], meta;
      quantize_slice16<BITS>(w, c, meta, smax);
      const uint32_t c0 = cb + h * TB + it * 128;
      if (BITS == 2) {
        const uint32_t v = prmt_q(c[0], c[1], 0x5410);  // the reference's word jj of row rt
        const uint32_t o = __shfl_xor_sync(0xffffffffu, v, 16);  // ... of row rt ^ 8
        sts32(c0, prmt_q(v, o, sel));
      } else {
        sts32(c0, c[0]);
        sts32(c0 + 16, c[1]);
      }
      // both lanes of the group hold the same (lo, hi): duplicate stores, no branch
      sts32(mbase + h * MO::TB + it * MO::U, meta);
    }
  }
  return chunk_flags(smax, BITS == 2 ? 3.0f : 15.0f, bad);
}

struct QTask {
  int tier, rows, src_tok0, dst_row0;
};
__device__ __forceinline__ QTask read_task(uint32_t addr) {
  QTask t;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(t.tier), "=r"(t.rows), "=r"(t.src_tok0), "=r"(t.dst_row0) : "r"(addr));
  return t;
}
struct CtaPos {
  int l, b, h;
};
// (layer, sequence, kv-head) of this CTA from the special registers (volatile: re-read where
// used instead of occupying registers across the loops)
__device__ __forceinline__ CtaPos cta_pos(int B) {
  uint32_t y, z;
  asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(y));
  asm volatile("mov.u32 %0, %%ctaid.z;" : "=r"(z));
  return CtaPos{(int)z / B, (int)z % B, (int)y};
}

// One warp per (layer, sequence, kv-head, destination chunk slot).  Slot p < N takes source
// chunk perm[p]; slot p == N is the context tail (if any).
#ifndef CKV_Q_MIN_CTAS
#define CKV_Q_MIN_CTAS 8
#endif
__global__ void __launch_bounds__(kQWarps * 32, CKV_Q_MIN_CTAS)
reorder_quantize_pack_kernel(const uint16_t* __restrict__ k, const uint16_t* __restrict__ v,
                             int H, int B, int64_t sL, int64_t sB, int64_t sT, int64_t sH,
                             const uint32_t* __restrict__ perm, int max_chunks,
                             const int32_t* __restrict__ seq, ckv_arena KA, ckv_arena VA,
                             int32_t* flag) {
  // staging of one packed chunk: its 2 interleaved K/V tile blocks (ckv_common.cuh), written
  // by the K pass and the V pass, then stored as one contiguous 3 KB / 5 KB run
  __shared__ __align__(16) unsigned char s_blk[kQWarps][2 * kBlock4];
  // the warp's task (tier, rows, first source token, first destination row), re-read from
  // shared memory where used: kept in registers across the quantize loops these would be
  // spilled to local memory at 64 registers
  __shared__ __align__(16) int s_task[kQWarps][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const int p = blockIdx.x * kQWarps + warp;
    const int b = blockIdx.z % B;
    const SeqRow sr = load_seq(seq, b);
    const int N = sr.ctx / kChunk;
    const int tail = sr.ctx - N * kChunk;
    if (p > N || (p == N && tail == 0)) return;
    const int n2 = sr.len2 / kChunk, n4 = sr.len4 / kChunk;
    int tier, rows, src_tok0, dst_row0;
    if (p < N) {
      const int src = (int)perm[(int64_t)b * max_chunks + p];
      src_tok0 = src * kChunk;
      rows = kChunk;
      if (p < n2) { tier = 0; dst_row0 = sr.off2 + p * kChunk; }
      else if (p < n2 + n4) { tier = 1; dst_row0 = sr.off4 + (p - n2) * kChunk; }
      else { tier = 2; dst_row0 = sr.off_fp + (p - n2 - n4) * kChunk; }
    } else {
      tier = 2; rows = tail; src_tok0 = sr.tail_src;
      dst_row0 = sr.off_fp + (N - n2 - n4) * kChunk;
    }
    if (lane == 0) *reinterpret_cast<int4*>(s_task[warp]) = make_int4(tier, rows, src_tok0, dst_row0);
    __syncwarp();
  }
  // nothing but tsel lives across the passes: the thread coordinates, the task and the
  // non-finite flags are re-derived / reported inside each pass (held across the quantize
  // loops, they were spilled at 64 registers, and the spill stores reached DRAM)
#pragma unroll 1
  for (int tsel = 0; tsel < 2; ++tsel) {
    uint32_t tid;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
    const int lane_v = (int)(tid & 31);
    const uint32_t task_addr = (uint32_t)__cvta_generic_to_shared(s_task[tid >> 5]);
    const QTask t = read_task(task_addr);
    const CtaPos c = cta_pos(B);
    const int64_t unit = (int64_t)c.l * H + c.h;
    const uint16_t* src = (tsel ? v : k) + c.l * sL + c.b * sB + c.h * sH + (int64_t)t.src_tok0 * sT;
    if (t.tier == 2) {
      const int sub = lane_v >> 4, j = lane_v & 15;  // 2 rows per warp step, 8 fp16 per lane
      bool bad_fp = false;  // non-finite input in an FP16-region row
      // arena fields by explicit selects (a reference to either parameter struct would put
      // both in local memory)
      uint16_t* dst = (tsel ? VA.fp : KA.fp) + (unit * (tsel ? VA.rows_fp : KA.rows_fp) + t.dst_row0) * kHeadDim;
#pragma unroll 4
      for (int rr = 0; rr < 16; ++rr) {
        const int r = 2 * rr + sub;
        if (r < t.rows) {
          const uint4 x = __ldg(reinterpret_cast<const uint4*>(src + r * sT) + j);
          const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            bad_fp |= !fp16_bits_finite(w[e] & 0xFFFF) || !fp16_bits_finite(w[e] >> 16);
          reinterpret_cast<uint4*>(dst + (int64_t)r * kHeadDim)[j] = x;
        }
      }
      // the reference rejects non-finite values only where it quantizes (build_cache ->
      // quantizer.quantize, quantizer.py:71-72); FP16-region rows are copied as they are
      if (__any_sync(0xffffffffu, bad_fp) && lane_v == 0) atomicOr(flag, CKV_FLAG_NONFINITE_FP16);
      continue;
    }
    const int code_bytes = t.tier == 0 ? kTileBytes2 : kTileBytes4;
    const uint32_t sblk = (uint32_t)__cvta_generic_to_shared(s_blk[tid >> 5]);
    const uint32_t sc = sblk + (tsel ? code_bytes : 0);
    const uint32_t sm = sblk + 2 * code_bytes + (tsel ? kTileBytesMeta : 0);
    bool wide, bad = false;  // bad: non-finite input in a quantized row
    float smax = 0.0f;  // largest group span of the chunk (decode precision routing)
    if (t.tier == 0) wide = tsel ? quantize_chunk<2, true>(src, (int)sT, lane_v, sc, sm, bad, smax)
                                 : quantize_chunk<2, false>(src, (int)sT, lane_v, sc, sm, bad, smax);
    else wide = tsel ? quantize_chunk<4, true>(src, (int)sT, lane_v, sc, sm, bad, smax)
                     : quantize_chunk<4, false>(src, (int)sT, lane_v, sc, sm, bad, smax);
    __syncwarp();
    if (__any_sync(0xffffffffu, bad) && lane_v == 0) atomicOr(flag, CKV_FLAG_NONFINITE);
    const int lane = lane_v;
    const QTask t2 = read_task(task_addr);
    const CtaPos c2 = cta_pos(B);
    const int64_t unit2 = (int64_t)c2.l * H + c2.h;
    if (tsel) {  // both halves staged: 128-bit coalesced stores of the 2 contiguous blocks
      const int64_t blk = t2.tier == 0 ? kBlock2 : kBlock4;
      const int64_t tile0 = (unit2 * (t2.tier == 0 ? KA.rows2 : KA.rows4) + t2.dst_row0) / kTileRows;
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<char*>(t2.tier == 0 ? KA.codes2 : KA.codes4) + tile0 * blk);
      const int n16 = (int)(2 * blk / 16);
      for (int i = lane; i < n16; i += 32) dst[i] = reinterpret_cast<const uint4*>(s_blk[tid >> 5])[i];
    }
    uint32_t* span_flags = tsel ? VA.span_flags : KA.span_flags;
    uint32_t* span_max = tsel ? VA.span_max : KA.span_max;
    if (__any_sync(0xffffffffu, wide) && lane == 0 && span_flags)
      atomicOr(span_flags + unit2 * B + c2.b, t2.tier == 0 ? 1u : 2u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    if (lane == 0 && span_max)  // non-negative floats order like their bit patterns
      atomicMax(span_max + unit2 * B + c2.b, __float_as_uint(smax));
    __syncwarp();
  }
}

// Decode append: row (l, b, h) of k_new/v_new -> FP16 region row off_fp + len_fp.
__global__ void append_rows_kernel(const uint16_t* __restrict__ kn, const uint16_t* __restrict__ vn,
                                   int B, int H, const int32_t* __restrict__ seq, ckv_arena KA,
                                   ckv_arena VA) {
  const int unit = blockIdx.x;  // (l, b, h)
  const int h = unit % H, b = (unit / H) % B, l = unit / (H * B);
  const SeqRow sr = load_seq(seq, b);
  const int t = threadIdx.x;  // 32 threads x 16 B for K, V
  const int tsel = t >> 4, j = t & 15;
  const uint16_t* src = (tsel ? vn : kn) + (int64_t)unit * kHeadDim;
  const ckv_arena& A = tsel ? VA : KA;
  uint16_t* dst = A.fp + (((int64_t)l * H + h) * A.rows_fp + sr.off_fp + sr.len_fp) * kHeadDim;
  reinterpret_cast<uint4*>(dst)[j] = reinterpret_cast<const uint4*>(src)[j];
}

__global__ void bump_len_kernel(int32_t* seq, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) seq[b * CKV_SEQ_FIELDS + 5] += 1;
}

// (lo, hi) fp16 metadata -> the reference's f64 scale = (hi - lo) / qmax, zero_point = lo
// (quantize_groups: scales = span / qmax, zero_points = mins, _numpy.py:65-66).
__global__ void expand_meta_kernel(const uint32_t* __restrict__ meta, int64_t n, double qmax,
                                   double* __restrict__ scales, double* __restrict__ zps) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 lh = __half22float2(u32_as_h2(meta[i]));
  const double lo = lh.x, hi = lh.y;
  scales[i] = __ddiv_rn(__dsub_rn(hi, lo), qmax);
  zps[i] = lo;
}

// Tile-native arena rows -> the reference's row-major packed words (_numpy.py:70-86) and
// (lo, hi) metadata [rows][4]: the inverse gather of the tile layout (ckv_common.cuh).
__global__ void arena_export_kernel(const unsigned char* __restrict__ codes,
                                    const unsigned char* __restrict__ meta, int64_t rows, int words,
                                    int is_v, int64_t stride, uint32_t* __restrict__ out_codes,
                                    uint32_t* __restrict__ out_meta) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n_code = rows * words;
  if (i < n_code) {
    const int64_t r = i / words;
    const int w = (int)(i % words), rt = (int)(r & 15);
    const unsigned char* t = codes + (r >> 4) * stride;
    if (words == 8) {  // INT2: bytes 4w .. 4w+3
      uint32_t x = 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        x |= (uint32_t)t[is_v ? tile_byte_v2(rt, 4 * w + k) : tile_byte_k2(rt, 4 * w + k)] << (8 * k);
      out_codes[i] = x;
    } else {
      const int o0 = is_v ? tile_off_v4(rt, w, 0) : tile_off_k4(rt, w, 0);
      const int o1 = is_v ? tile_off_v4(rt, w, 1) : tile_off_k4(rt, w, 1);
      out_codes[i] = (uint32_t)*reinterpret_cast<const uint16_t*>(t + o0) |
                     ((uint32_t)*reinterpret_cast<const uint16_t*>(t + o1) << 16);
    }
  } else if (i < n_code + rows * kGroupsPerRow) {
    const int64_t k = i - n_code, r = k / kGroupsPerRow;
    const int G = (int)(k % kGroupsPerRow), rt = (int)(r & 15);
    const unsigned char* t = meta + (r >> 4) * stride;
    const int o0 = is_v ? tile_off_vm(rt, G, 0) : tile_off_km(rt, G, 0);
    const int o1 = is_v ? tile_off_vm(rt, G, 1) : tile_off_km(rt, G, 1);
    out_meta[k] = (uint32_t)*reinterpret_cast<const uint16_t*>(t + o0) |
                  ((uint32_t)*reinterpret_cast<const uint16_t*>(t + o1) << 16);
  }
}

// kv_store.reconstruct (kv_store.py:236-253) with token_order (:227-233) on the tile-native
// arenas: one warp per (arena row, unit), 4 elements per lane.  Arena row r of sequence b is
// INT2 row r (< len2), INT4 row r - len2 (< len4) or FP16-region row r - len2 - len4; chunk slot
// p = r / 32 holds source chunk perm[b][p]; FP16-region rows past the FP16-tier chunks are the
// tail then the decode tokens, consecutive in original order from 32 n_chunks.  Quantized
// values are the reference's dequantize (_numpy.py:102-112): zp + scale code in IEEE f64 with
// scale = (hi - lo) / qmax and zp = lo from the fp16 metadata (no FMA: two roundings).
__device__ __forceinline__ double dequant_ref(uint32_t lohi, uint32_t code, double qmax) {
  const double lo = (double)__half2float(__ushort_as_half((unsigned short)(lohi & 0xFFFFu)));
  const double hi = (double)__half2float(__ushort_as_half((unsigned short)(lohi >> 16)));
  return __dadd_rn(lo, __dmul_rn(__ddiv_rn(__dsub_rn(hi, lo), qmax), (double)code));
}
__global__ void reconstruct_kernel(ckv_arena K, ckv_arena V, const int32_t* __restrict__ seq,
                                   const uint32_t* __restrict__ perm, int max_chunks, int B, int H,
                                   double* __restrict__ ok, double* __restrict__ ov, int64_t sl, int64_t sb,
                                   int64_t st, int64_t sh, int t_out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int h = blockIdx.y, l = blockIdx.z / B, b = blockIdx.z % B;
  const SeqRow s = load_seq(seq, b);
  if (r >= (int64_t)s.len2 + s.len4 + s.len_fp) return;
  const int n_chunks = s.ctx / kChunk, n2 = s.len2 / kChunk, n4 = s.len4 / kChunk;
  const int64_t unit = (int64_t)l * H + h;
  int64_t orig;
  int tier;  // 0 INT2, 1 INT4, 2 FP16 region
  int64_t row;  // row in its arena (absolute)
  if (r < s.len2) {
    tier = 0; row = s.off2 + r;
    orig = (int64_t)perm[(int64_t)b * max_chunks + r / kChunk] * kChunk + r % kChunk;
  } else if (r < (int64_t)s.len2 + s.len4) {
    const int64_t r4 = r - s.len2;
    tier = 1; row = s.off4 + r4;
    orig = (int64_t)perm[(int64_t)b * max_chunks + n2 + r4 / kChunk] * kChunk + r4 % kChunk;
  } else {
    const int64_t rf = r - s.len2 - s.len4, nfp = n_chunks - n2 - n4;
    tier = 2; row = s.off_fp + rf;
    orig = rf < nfp * kChunk ? (int64_t)perm[(int64_t)b * max_chunks + n2 + n4 + rf / kChunk] * kChunk + rf % kChunk
                             : (int64_t)n_chunks * kChunk + (rf - nfp * kChunk);
  }
  if (orig >= t_out) return;
  for (int which = 0; which < 2; ++which) {
    const ckv_arena& A = which ? V : K;
    double* dst = (which ? ov : ok) + l * sl + b * sb + orig * st + h * sh;
    if (tier == 2) {
      const uint16_t* src = A.fp + (unit * A.rows_fp + row) * kHeadDim;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        dst[4 * lane + k] = (double)__half2float(__ushort_as_half(src[4 * lane + k]));
      continue;
    }
    const int bits = tier == 0 ? 2 : 4;
    const int64_t ar = unit * (bits == 2 ? A.rows2 : A.rows4) + row, t = ar / kTileRows;
    const int rt = (int)(ar % kTileRows);
    const unsigned char* ct = reinterpret_cast<const unsigned char*>(bits == 2 ? A.codes2 : A.codes4) +
                              t * (bits == 2 ? kBlock2 : kBlock4);
    const unsigned char* mt = reinterpret_cast<const unsigned char*>(bits == 2 ? A.meta2 : A.meta4) +
                              t * (bits == 2 ? kBlock2 : kBlock4);
    const int G = lane >> 3;  // elements 4 lane .. 4 lane + 3 lie in group lane / 8
    const int mo0 = which ? tile_off_vm(rt, G, 0) : tile_off_km(rt, G, 0);
    const int mo1 = which ? tile_off_vm(rt, G, 1) : tile_off_km(rt, G, 1);
    const uint32_t lohi = (uint32_t)*reinterpret_cast<const uint16_t*>(mt + mo0) |
                          ((uint32_t)*reinterpret_cast<const uint16_t*>(mt + mo1) << 16);
    uint32_t codes;  // the 4 codes of elements 4 lane .. 4 lane + 3, b bits each
    if (bits == 2) {
      codes = ct[which ? tile_byte_v2(rt, lane) : tile_byte_k2(rt, lane)];
    } else {  // 16-bit piece P = lane of the row (w = P / 2, hf = P % 2)
      codes = *reinterpret_cast<const uint16_t*>(ct + (which ? tile_off_v4(rt, lane >> 1, lane & 1)
                                                              : tile_off_k4(rt, lane >> 1, lane & 1)));
    }
    const double qmax = bits == 2 ? 3.0 : 15.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[4 * lane + k] = dequant_ref(lohi, (codes >> (bits * k)) & ((1u << bits) - 1u), qmax);
  }
}

}  // namespace ckv

using namespace ckv;

extern "C" {

int32_t ckv_reorder_quantize_pack(const uint16_t* k, const uint16_t* v, int32_t layers,
                                  int32_t batch, int32_t kv_heads, int64_t s_layer,
                                  int64_t s_batch, int64_t s_token, int64_t s_head,
                                  const uint32_t* perm, int32_t max_chunks, const int32_t* seq,
                                  int32_t max_ctx, ckv_arena k_arena, ckv_arena v_arena,
                                  int32_t* flag, void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0 || max_chunks < 0 || max_ctx < 0) return CKV_ERR_ARG;
  if (!k || !v || !seq || !flag) return CKV_ERR_ARG;
  if ((s_token % 8) || (s_head % 8) || (s_batch % 8) || (s_layer % 8)) return CKV_ERR_UNSUPPORTED;
  if (s_token <= 0 || s_token > INT32_MAX) return CKV_ERR_UNSUPPORTED;  // the kernel's row stride is 32-bit
  if (layers == 0 || batch == 0 || kv_heads == 0) return CKV_OK;
  const int slots = (int)(cdiv(max_ctx, kChunk)) + 1;
  dim3 grid((unsigned)cdiv(slots, kQWarps), (unsigned)kv_heads, (unsigned)(layers * batch));
  reorder_quantize_pack_kernel<<<grid, kQWarps * 32, 0, as_stream(stream)>>>(
      k, v, kv_heads, batch, s_layer, s_batch, s_token, s_head, perm, max_chunks, seq, k_arena,
      v_arena, flag);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_append_tokens(const uint16_t* k_new, const uint16_t* v_new, int32_t layers,
                          int32_t batch, int32_t kv_heads, int32_t* seq, ckv_arena k_arena,
                          ckv_arena v_arena, void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0) return CKV_ERR_ARG;
  if (layers * batch * kv_heads == 0) return CKV_OK;
  append_rows_kernel<<<layers * batch * kv_heads, 32, 0, as_stream(stream)>>>(
      k_new, v_new, batch, kv_heads, seq, k_arena, v_arena);
  CKV_LAUNCH_CHECK();
  bump_len_kernel<<<(unsigned)cdiv(batch, 128), 128, 0, as_stream(stream)>>>(seq, batch);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_expand_meta(const uint32_t* meta, int64_t n_groups, int32_t bits, double* scales,
                        double* zero_points, void* stream) {
  if (bits != 2 && bits != 4) return CKV_ERR_BITS;
  if (n_groups < 0) return CKV_ERR_ARG;
  if (n_groups == 0) return CKV_OK;
  expand_meta_kernel<<<(unsigned)cdiv(n_groups, 256), 256, 0, as_stream(stream)>>>(
      meta, n_groups, (double)((1 << bits) - 1), scales, zero_points);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_reconstruct(ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq, const uint32_t* perm,
                        int32_t max_chunks, int32_t layers, int32_t batch, int32_t kv_heads, int32_t max_rows,
                        double* out_k, double* out_v, int64_t s_layer, int64_t s_batch, int64_t s_token,
                        int64_t s_head, int32_t t_out, void* stream) {
  if (layers < 0 || batch < 0 || kv_heads < 0 || max_rows < 0 || t_out < 0 || max_chunks < 0) return CKV_ERR_ARG;
  if (layers * batch * kv_heads == 0 || max_rows == 0 || t_out == 0) return CKV_OK;
  if (!seq || !perm || !out_k || !out_v) return CKV_ERR_ARG;
  if ((int64_t)layers * batch > 65535 || kv_heads > 65535) return CKV_ERR_UNSUPPORTED;
  constexpr int kWarps = 8;
  const dim3 grid((unsigned)cdiv(max_rows, kWarps), (unsigned)kv_heads, (unsigned)(layers * batch));
  reconstruct_kernel<<<grid, 32 * kWarps, 0, as_stream(stream)>>>(k_arena, v_arena, seq, perm, max_chunks, batch,
                                                                  kv_heads, out_k, out_v, s_layer, s_batch, s_token,
                                                                  s_head, t_out);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_arena_export(const uint32_t* codes, const uint32_t* meta, int64_t rows, int32_t bits,
                         int32_t is_v, int64_t tile_stride, uint32_t* out_codes,
                         uint32_t* out_meta, void* stream) {
  if (bits != 2 && bits != 4) return CKV_ERR_BITS;
  if (rows < 0 || (rows % kTileRows)) return CKV_ERR_SHAPE;
  if (rows == 0) return CKV_OK;
  if (!codes || !meta || !out_codes || !out_meta || tile_stride <= 0) return CKV_ERR_ARG;
  const int words = bits == 2 ? 8 : 16;
  const int64_t n = rows * (words + kGroupsPerRow);
  arena_export_kernel<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const unsigned char*>(codes), reinterpret_cast<const unsigned char*>(meta),
      rows, words, is_v, tile_stride, out_codes, out_meta);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

}  // extern "C"
