// Generic per-block kernels behind chunkkv.kernels' five callables
// (reference: pkg/src/chunkkv/kernels/_core.pyx, _numpy.py) and the float64
// pieces of attention.py used by the per-head drop-in API.
//
// These serve the per-head (reference-shaped, float64) API: any rows/cols,
// any group_size, bits in {2, 4}.  Arithmetic follows the reference's f64
// expression trees with explicit round-to-nearest intrinsics (no FMA
// contraction, as the reference builds with -ffp-contract=off), so codes,
// packed words and metadata are bit-identical.  The fp16 D=128 hot path lives
// in ckv_quantize.cu / ckv_decode.cu.
#include <float.h>
#include <math.h>

#include "ckv_common.cuh"

namespace ckv {

// ---------------------------------------------------------------------------
// quantize_groups: _core.pyx:27-79 (scan order, strict < / > updates) and
// _numpy.py:59-61 (code = floor((x - lo) * qmax / span + 0.5)).
// One thread per (row, group).
template <typename T>
__device__ __forceinline__ double load_val(const T* p, int64_t i);
template <>
__device__ __forceinline__ double load_val<double>(const double* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ double load_val<uint16_t>(const uint16_t* p, int64_t i) {
  return (double)__half2float(__ushort_as_half(p[i]));
}

template <typename T>
__global__ void quantize_groups_kernel(const T* __restrict__ x, int64_t rows, int64_t cols,
                                       int64_t gs, int64_t gpr, double qmax,
                                       uint8_t* __restrict__ codes, double* __restrict__ scales,
                                       double* __restrict__ zps, int32_t* flag) {
  int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gi >= rows * gpr) return;
  int64_t r = gi / gpr, g = gi % gpr;
  int64_t c0 = g * gs, c1 = min(c0 + gs, cols);
  const int64_t base = r * cols;
  double lo = load_val(x, base + c0), hi = lo;
  bool finite = isfinite(lo);
  for (int64_t c = c0 + 1; c < c1; ++c) {
    double v = load_val(x, base + c);
    finite &= (bool)isfinite(v);
    if (v < lo) lo = v;
    if (v > hi) hi = v;
  }
  if (!finite) atomicOr(flag, CKV_FLAG_NONFINITE);
  double span = __dsub_rn(hi, lo);
  scales[gi] = __ddiv_rn(span, qmax);
  zps[gi] = lo;
  if (span > 0.0) {
    for (int64_t c = c0; c < c1; ++c) {
      double t = floor(__dadd_rn(__ddiv_rn(__dmul_rn(__dsub_rn(load_val(x, base + c), lo), qmax), span), 0.5));
      t = t < 0.0 ? 0.0 : (t > qmax ? qmax : t);
      codes[base + c] = (uint8_t)t;
    }
  } else {
    for (int64_t c = c0; c < c1; ++c) codes[base + c] = 0;
  }
}

// pack_codes: element i at bits [i*b, (i+1)*b) of LE word i*b/32 (_core.pyx:82-97).
__global__ void pack_kernel(const uint8_t* __restrict__ codes, int64_t n, int bits,
                            int64_t n_words, uint32_t* __restrict__ packed) {
  int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= n_words) return;
  const int per = 32 / bits;
  uint32_t word = 0;
  int64_t i0 = w * per;
  for (int k = 0; k < per; ++k) {
    int64_t i = i0 + k;
    if (i < n) word |= (uint32_t)codes[i] << (k * bits);
  }
  packed[w] = word;
}

// unpack_codes (_core.pyx:100-116).
__global__ void unpack_kernel(const uint32_t* __restrict__ packed, int bits, int64_t count,
                              uint8_t* __restrict__ codes) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  int64_t bitpos = i * bits;
  codes[i] = (uint8_t)((packed[bitpos >> 5] >> (bitpos & 31)) & ((1u << bits) - 1u));
}

__device__ __forceinline__ double deq_elem(const uint32_t* packed, const double* s,
                                           const double* z, int64_t r, int64_t c, int64_t cols,
                                           int64_t gs, int64_t gpr, int bits) {
  int64_t bitpos = (r * cols + c) * bits;
  uint32_t code = (packed[bitpos >> 5] >> (bitpos & 31)) & ((1u << bits) - 1u);
  int64_t gi = r * gpr + c / gs;
  return __dadd_rn(z[gi], __dmul_rn(s[gi], (double)code));  // _core.pyx:144
}

// dequantize_codes (_core.pyx:119-145).
__global__ void dequant_kernel(const uint32_t* __restrict__ packed, const double* __restrict__ s,
                               const double* __restrict__ z, int64_t rows, int64_t cols,
                               int64_t gs, int64_t gpr, int bits, double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  out[i] = deq_elem(packed, s, z, i / cols, i % cols, cols, gs, gpr, bits);
}

// B element accessor: packed-quantized or dense.
struct PackedB {
  const uint32_t* packed; const double* s; const double* z;
  int64_t cols, gs, gpr; int bits;
  __device__ __forceinline__ double at(int64_t r, int64_t c) const {
    return deq_elem(packed, s, z, r, c, cols, gs, gpr, bits);
  }
};
struct DenseB {
  const double* b; int64_t ldb;
  __device__ __forceinline__ double at(int64_t r, int64_t c) const { return b[r * ldb + c]; }
};

// out[i, j] (+)= sum_k a[i, k] * B(k, j)      (transpose == 0, B stored [k][j])
// out[i, j] (+)= sum_k a[i, k] * B(j, k)      (transpose == 1, B stored [j][k])
// CTA = 8 warps on a 32-wide output slab of one row i; each warp strides over k,
// partial sums reduced through shared memory in fixed order (deterministic).
template <typename BT>
__global__ void matmul_f64_kernel(const double* __restrict__ a, int64_t lda, int64_t inner,
                                  int64_t n_out, BT B, int transpose, double* __restrict__ out,
                                  int64_t ldo, int accumulate) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  double acc = 0.0;
  if (!transpose) {
    const int64_t j = j0 + lane;
    if (j < n_out)
      for (int64_t k = warp; k < inner; k += 8) acc = fma(a[i * lda + k], B.at(k, j), acc);
  } else {
    // each warp owns output columns j0..j0+31 in turn; lanes stride over k (coalesced on B rows)
    for (int jj = 0; jj < 32; ++jj) {
      const int64_t j = j0 + jj;
      if (j >= n_out) break;
      if ((jj & 7) != warp) continue;
      double s = 0.0;
      for (int64_t k = lane; k < inner; k += 32) s = fma(a[i * lda + k], B.at(j, k), s);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) part[0][jj] = s;  // slot per column (written by exactly one warp)
    }
    __syncthreads();
    if (warp == 0) {
      const int64_t j = j0 + lane;
      if (j < n_out) {
        double v = part[0][lane];
        out[i * ldo + j] = accumulate ? out[i * ldo + j] + v : v;
      }
    }
    return;
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    const int64_t j = j0 + lane;
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += part[w][lane];
    if (j < n_out) out[i * ldo + j] = accumulate ? out[i * ldo + j] + v : v;
  }
}

// stable_softmax with fused scale and additive mask (attention.py:24-31,79-81).
__global__ void softmax_f64_kernel(double* __restrict__ x, int64_t n, double scale,
                                   const double* __restrict__ mask) {
  __shared__ double red[32];
  const int64_t row = blockIdx.x;
  double* xr = x + row * n;
  const double* mr = mask ? mask + row * n : nullptr;
  double mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double v = __dmul_rn(xr[j], scale);
    if (mr) v = __dadd_rn(v, mr[j]);
    xr[j] = v;
    mx = fmax(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  double sum = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double e = exp(xr[j] - mx);
    xr[j] = e;
    sum += e;
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  sum = red[0];
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) xr[j] = xr[j] / sum;
}

__global__ void scatter_rows_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                    const int64_t* __restrict__ order, double* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  int64_t r = i / cols, c = i % cols;
  dst[order[r] * cols + c] = src[i];
}

}  // namespace ckv

using namespace ckv;

static int32_t check_bits_gs(int32_t bits, int64_t gs) {
  if (bits != 2 && bits != 4) return CKV_ERR_BITS;
  if (gs < 1) return CKV_ERR_GROUP;
  return CKV_OK;
}

template <typename T>
static int32_t quantize_groups_impl(const T* x, int64_t rows, int64_t cols, int32_t bits,
                                    int64_t gs, uint8_t* codes, double* scales, double* zps,
                                    int32_t* flag, void* stream) {
  int32_t st = check_bits_gs(bits, gs);
  if (st) return st;
  if (rows < 0 || cols < 0) return CKV_ERR_ARG;
  if (rows == 0 || cols == 0) return CKV_OK;
  const int64_t gpr = cdiv(cols, gs);
  const int64_t n = rows * gpr;
  quantize_groups_kernel<T><<<(unsigned)cdiv(n, 128), 128, 0, as_stream(stream)>>>(
      x, rows, cols, gs, gpr, (double)((1 << bits) - 1), codes, scales, zps, flag);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

extern "C" {

int32_t ckv_abi_version(void) { return 1; }

const char* ckv_status_string(int32_t s) {
  switch (s) {
    case CKV_OK: return "ok";
    case CKV_ERR_BITS: return "bitwidth must be one of (2, 4)";
    case CKV_ERR_GROUP: return "group_size must be >= 1";
    case CKV_ERR_SHAPE: return "inner dimension mismatch";
    case CKV_ERR_CAPACITY: return "count exceeds packed capacity";
    case CKV_ERR_UNSUPPORTED: return "shape outside the specialised kernels (head_dim 128, group 32, chunk 32)";
    case CKV_ERR_ARG: return "invalid argument";
    case CKV_ERR_CUDA: return "CUDA launch failure";
    default: return "unknown status";
  }
}

int32_t ckv_quantize_groups_f64(const double* x, int64_t rows, int64_t cols, int32_t bits,
                                int64_t group_size, uint8_t* codes, double* scales,
                                double* zero_points, int32_t* flag, void* stream) {
  return quantize_groups_impl(x, rows, cols, bits, group_size, codes, scales, zero_points, flag, stream);
}

int32_t ckv_quantize_groups_f16(const uint16_t* x, int64_t rows, int64_t cols, int32_t bits,
                                int64_t group_size, uint8_t* codes, double* scales,
                                double* zero_points, int32_t* flag, void* stream) {
  return quantize_groups_impl(x, rows, cols, bits, group_size, codes, scales, zero_points, flag, stream);
}

int32_t ckv_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint32_t* packed, void* stream) {
  if (bits != 2 && bits != 4) return CKV_ERR_BITS;
  if (n < 0) return CKV_ERR_ARG;
  const int64_t n_words = cdiv(n * bits, 32);
  if (n_words == 0) return CKV_OK;
  pack_kernel<<<(unsigned)cdiv(n_words, 256), 256, 0, as_stream(stream)>>>(codes, n, bits, n_words, packed);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_unpack_codes(const uint32_t* packed, int64_t n_words, int32_t bits, int64_t count,
                         uint8_t* codes, void* stream) {
  if (bits != 2 && bits != 4) return CKV_ERR_BITS;
  if (count < 0 || n_words < 0) return CKV_ERR_ARG;
  if (count > n_words * (32 / bits)) return CKV_ERR_CAPACITY;
  if (count == 0) return CKV_OK;
  unpack_kernel<<<(unsigned)cdiv(count, 256), 256, 0, as_stream(stream)>>>(packed, bits, count, codes);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_dequantize_codes_f64(const uint32_t* packed, int64_t n_words, const double* scales,
                                 const double* zero_points, int64_t rows, int64_t cols,
                                 int32_t bits, int64_t group_size, double* out, void* stream) {
  int32_t st = check_bits_gs(bits, group_size);
  if (st) return st;
  if (rows < 0 || cols < 0) return CKV_ERR_ARG;
  if (rows * cols > n_words * (32 / bits)) return CKV_ERR_CAPACITY;
  if (rows == 0 || cols == 0) return CKV_OK;
  const int64_t gpr = cdiv(cols, group_size);
  dequant_kernel<<<(unsigned)cdiv(rows * cols, 256), 256, 0, as_stream(stream)>>>(
      packed, scales, zero_points, rows, cols, group_size, gpr, bits, out);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_matmul_packed_f64(const double* a, int64_t m, int64_t a_cols, int64_t lda,
                              const uint32_t* packed, int64_t n_words, const double* scales,
                              const double* zero_points, int64_t rows, int64_t cols, int32_t bits,
                              int64_t group_size, int32_t transpose, double* out, int64_t ldo,
                              int32_t accumulate, void* stream) {
  int32_t st = check_bits_gs(bits, group_size);
  if (st) return st;
  const int64_t inner = transpose ? cols : rows;
  if (a_cols != inner) return CKV_ERR_SHAPE;
  if (rows * cols > n_words * (32 / bits)) return CKV_ERR_CAPACITY;
  const int64_t n_out = transpose ? rows : cols;
  if (m == 0 || n_out == 0) return CKV_OK;
  PackedB B{packed, scales, zero_points, cols, group_size, cdiv(cols, group_size), bits};
  if (inner == 0) {  // empty contraction: zeros (or untouched when accumulating)
    if (!accumulate) cudaMemset2DAsync(out, ldo * 8, 0, n_out * 8, m, as_stream(stream));
    return CKV_OK;
  }
  dim3 grid((unsigned)cdiv(n_out, 32), (unsigned)m);
  matmul_f64_kernel<PackedB><<<grid, 256, 0, as_stream(stream)>>>(a, lda, inner, n_out, B, transpose,
                                                                  out, ldo, accumulate);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_matmul_f64(const double* a, int64_t m, int64_t k, int64_t lda, const double* b,
                       int64_t n, int64_t ldb, int32_t transpose, double* out, int64_t ldo,
                       int32_t accumulate, void* stream) {
  if (m < 0 || k < 0 || n < 0) return CKV_ERR_ARG;
  if (m == 0 || n == 0) return CKV_OK;
  if (k == 0) {
    if (!accumulate) cudaMemset2DAsync(out, ldo * 8, 0, n * 8, m, as_stream(stream));
    return CKV_OK;
  }
  DenseB B{b, ldb};
  dim3 grid((unsigned)cdiv(n, 32), (unsigned)m);
  matmul_f64_kernel<DenseB><<<grid, 256, 0, as_stream(stream)>>>(a, lda, k, n, B, transpose, out,
                                                                 ldo, accumulate);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_scale_mask_softmax_f64(double* x, int64_t m, int64_t n, double scale,
                                   const double* mask, void* stream) {
  if (m < 0 || n < 0) return CKV_ERR_ARG;
  if (m == 0 || n == 0) return CKV_OK;
  softmax_f64_kernel<<<(unsigned)m, 256, 0, as_stream(stream)>>>(x, n, scale, mask);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_scatter_rows_f64(const double* src, int64_t rows, int64_t cols, const int64_t* order,
                             double* dst, void* stream) {
  if (rows < 0 || cols < 0) return CKV_ERR_ARG;
  if (rows == 0 || cols == 0) return CKV_OK;
  scatter_rows_kernel<<<(unsigned)cdiv(rows * cols, 256), 256, 0, as_stream(stream)>>>(src, rows, cols, order, dst);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

}  // extern "C"
