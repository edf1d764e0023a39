// Hashed bag-of-words chunk encoder (HashedBowEncoder.encode, retrieval.py:70-100) on the GPU:
// the step upstream of the search.  For every text: split on Python's
// str.split() whitespace (the ASCII set and the multi-byte Unicode spaces, decoded from
// UTF-8 here), hash every word with keyed BLAKE2b-64 (RFC 7693; key = the seed's decimal
// ASCII, digest 8 bytes, read little-endian), add the sign of bit 63 to bucket h % dim, then
// L2-normalise.  Bucket counts are small integers, so the norm sqrt(sum c^2) and c / norm are
// the reference's values bit for bit (exact integer sums, IEEE sqrt and division).
//
// Layout: texts are one UTF-8 byte buffer with int64 offsets [n + 1]; output vectors f64
// [n, dim] and norms f64 [n] (1.0, or 0.0 for a text with no words / all buckets cancelled),
// exactly what ckv_search takes as embeddings.  One warp per text (grid-stride), the text's
// bucket histogram in shared memory, every lane hashing the words that start in its 32-byte
// window.
#include "ckv_common.cuh"

namespace ckv {

constexpr int kEncWarps = 4;
constexpr int kMaxBowDim = 8192;

__constant__ uint64_t kB2Iv[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                                  0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                                  0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};

// message schedule of RFC 7693 (rounds 10 and 11 reuse rows 0 and 1)
template <int R, int I>
struct Sigma {
  static constexpr unsigned char t[10][16] = {
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
      {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
      {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
      {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
      {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
      {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
      {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
      {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
      {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
      {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0}};
  static constexpr int v = t[R % 10][I];
};

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

template <int R, int I, int A, int B, int C, int D>
__device__ __forceinline__ void b2_g(uint64_t (&v)[16], const uint64_t (&m)[16]) {
  v[A] = v[A] + v[B] + m[Sigma<R, 2 * I>::v];
  v[D] = rotr64(v[D] ^ v[A], 32);
  v[C] = v[C] + v[D];
  v[B] = rotr64(v[B] ^ v[C], 24);
  v[A] = v[A] + v[B] + m[Sigma<R, 2 * I + 1>::v];
  v[D] = rotr64(v[D] ^ v[A], 16);
  v[C] = v[C] + v[D];
  v[B] = rotr64(v[B] ^ v[C], 63);
}

template <int R>
__device__ __forceinline__ void b2_round(uint64_t (&v)[16], const uint64_t (&m)[16]) {
  b2_g<R, 0, 0, 4, 8, 12>(v, m);
  b2_g<R, 1, 1, 5, 9, 13>(v, m);
  b2_g<R, 2, 2, 6, 10, 14>(v, m);
  b2_g<R, 3, 3, 7, 11, 15>(v, m);
  b2_g<R, 4, 0, 5, 10, 15>(v, m);
  b2_g<R, 5, 1, 6, 11, 12>(v, m);
  b2_g<R, 6, 2, 7, 8, 13>(v, m);
  b2_g<R, 7, 3, 4, 9, 14>(v, m);
}

// F(h, m, t, f) of RFC 7693 section 3.2 (t < 2^64 here)
__device__ __forceinline__ void b2_compress(uint64_t (&h)[8], const uint64_t (&m)[16], uint64_t t, bool last) {
  uint64_t v[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = h[i];
    v[i + 8] = kB2Iv[i];
  }
  v[12] ^= t;
  if (last) v[14] = ~v[14];
  b2_round<0>(v, m); b2_round<1>(v, m); b2_round<2>(v, m); b2_round<3>(v, m);
  b2_round<4>(v, m); b2_round<5>(v, m); b2_round<6>(v, m); b2_round<7>(v, m);
  b2_round<8>(v, m); b2_round<9>(v, m); b2_round<10>(v, m); b2_round<11>(v, m);
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

struct BowKey {
  unsigned char bytes[64];
  int len;
};

// little-endian 8-byte word k of [p, p + n) (zero past the end)
__device__ __forceinline__ uint64_t load_word(const unsigned char* p, int64_t n, int k) {
  uint64_t w = 0;
  const int64_t o = 8 * (int64_t)k;
  if (o < n) {
    const int c = n - o < 8 ? (int)(n - o) : 8;
    for (int i = 0; i < c; ++i) w |= (uint64_t)p[o + i] << (8 * i);
  }
  return w;
}

// state after the key block (parameter block: digest 8 bytes, key length kk)
__device__ void b2_key_state(const BowKey& key, uint64_t (&h)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = kB2Iv[i];
  h[0] ^= 0x01010000ull ^ ((uint64_t)key.len << 8) ^ 8ull;
  uint64_t m[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) m[k] = load_word(key.bytes, key.len, k);
  b2_compress(h, m, 128, false);
}

// keyed BLAKE2b-64 of a non-empty word, from the post-key state
__device__ uint64_t b2_word(const uint64_t (&hk)[8], const unsigned char* w, int64_t n) {
  uint64_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = hk[i];
  for (int64_t off = 0; off < n; off += 128) {
    const int64_t rem = n - off;
    uint64_t m[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) m[k] = load_word(w + off, rem, k);
    const bool last = rem <= 128;
    b2_compress(h, m, 128 + (uint64_t)(last ? n : off + 128), last);
  }
  return h[0];
}

// length of the str.isspace() character starting at byte j of [b0, b1) (0: not whitespace):
// U+0009-000D, U+001C-0020, U+0085, U+00A0, U+1680, U+2000-200A, U+2028, U+2029, U+202F,
// U+205F, U+3000
__device__ __forceinline__ int ws_len(const unsigned char* s, int64_t j, int64_t b0, int64_t b1) {
  if (j < b0 || j >= b1) return 0;
  const unsigned c0 = s[j];
  if ((c0 >= 0x09 && c0 <= 0x0D) || (c0 >= 0x1C && c0 <= 0x20)) return 1;
  if (c0 != 0xC2 && (c0 < 0xE1 || c0 > 0xE3)) return 0;
  const unsigned c1 = j + 1 < b1 ? s[j + 1] : 0u;
  if (c0 == 0xC2) return (c1 == 0x85 || c1 == 0xA0) ? 2 : 0;
  const unsigned c2 = j + 2 < b1 ? s[j + 2] : 0u;
  if (c0 == 0xE1) return (c1 == 0x9A && c2 == 0x80) ? 3 : 0;
  if (c0 == 0xE3) return (c1 == 0x80 && c2 == 0x80) ? 3 : 0;
  if (c1 == 0x80) return ((c2 >= 0x80 && c2 <= 0x8A) || c2 == 0xA8 || c2 == 0xA9 || c2 == 0xAF) ? 3 : 0;
  return (c1 == 0x81 && c2 == 0x9F) ? 3 : 0;
}

// byte j is whitespace (positions outside [b0, b1) count as whitespace: word boundaries)
__device__ __forceinline__ bool is_ws(const unsigned char* s, int64_t j, int64_t b0, int64_t b1) {
  if (j < b0 || j >= b1) return true;
  return ws_len(s, j, b0, b1) >= 1 || ws_len(s, j - 1, b0, b1) >= 2 || ws_len(s, j - 2, b0, b1) >= 3;
}

__global__ void __launch_bounds__(kEncWarps * 32)
bow_encode_kernel(const unsigned char* __restrict__ text, const int64_t* __restrict__ offsets, int n_texts,
                  int dim, const BowKey key, double* __restrict__ vectors, double* __restrict__ norms) {
  extern __shared__ int s_hist[];  // [warp][dim]
  __shared__ uint64_t s_hk[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    uint64_t hk[8];
    b2_key_state(key, hk);
#pragma unroll
    for (int i = 0; i < 8; ++i) s_hk[i] = hk[i];
  }
  __syncthreads();
  uint64_t hk[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) hk[i] = s_hk[i];
  int* hist = s_hist + warp * dim;
  const bool pow2 = (dim & (dim - 1)) == 0;
  for (int t = blockIdx.x * kEncWarps + warp; t < n_texts; t += gridDim.x * kEncWarps) {
    for (int k = lane; k < dim; k += 32) hist[k] = 0;
    __syncwarp();
    const int64_t b0 = offsets[t], b1 = offsets[t + 1];
    for (int64_t base = b0; base < b1; base += 32) {
      const int64_t i = base + lane;
      if (i < b1 && !is_ws(text, i, b0, b1) && is_ws(text, i - 1, b0, b1)) {
        int64_t e = i + 1;
        while (e < b1 && !is_ws(text, e, b0, b1)) ++e;
        const uint64_t h = b2_word(hk, text + i, e - i);
        const unsigned bucket = pow2 ? (unsigned)(h & (uint64_t)(dim - 1)) : (unsigned)(h % (uint64_t)dim);
        atomicAdd(&hist[bucket], (h >> 63) ? -1 : 1);
      }
    }
    __syncwarp();
    long long sq = 0;
    for (int k = lane; k < dim; k += 32) sq += (long long)hist[k] * hist[k];
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const double norm = __dsqrt_rn((double)sq);  // exact integer sum of squares, IEEE sqrt
    double* out = vectors + (int64_t)t * dim;
    for (int k = lane; k < dim; k += 32) out[k] = norm > 0.0 ? __ddiv_rn((double)hist[k], norm) : 0.0;
    if (lane == 0) norms[t] = norm > 0.0 ? 1.0 : 0.0;
    __syncwarp();
  }
}

// TF-IDF (TfidfEncoder.encode, retrieval.py:122-138) from host-mapped vocabulary ids: one warp
// per text zeroes its row, counts its ids with f64 atomics (exact small integers), weights by
// idf (count x idf: the reference's one rounding), and L2-normalises (the norm's summation
// order is not BLAS's: a few ulp).
__global__ void __launch_bounds__(kEncWarps * 32)
tfidf_encode_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ offsets, int n_texts,
                    const double* __restrict__ idf, int vocab, int ld, double* __restrict__ vectors,
                    double* __restrict__ norms) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = blockIdx.x * kEncWarps + warp; t < n_texts; t += gridDim.x * kEncWarps) {
    double* row = vectors + (int64_t)t * ld;
    for (int k = lane; k < ld; k += 32) row[k] = 0.0;
    __syncwarp();
    for (int64_t j = offsets[t] + lane; j < offsets[t + 1]; j += 32) atomicAdd(row + ids[j], 1.0);
    __syncwarp();
    double sq = 0.0;
    for (int k = lane; k < vocab; k += 32) {
      const double v = __dmul_rn(__ldcg(row + k), idf[k]);
      row[k] = v;
      sq = fma(v, v, sq);
    }
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const double norm = __dsqrt_rn(sq);
    if (norm > 0.0)
      for (int k = lane; k < vocab; k += 32) row[k] = __ddiv_rn(row[k], norm);
    if (lane == 0) norms[t] = norm > 0.0 ? 1.0 : 0.0;
    __syncwarp();
  }
}

}  // namespace ckv

using namespace ckv;

extern "C" {

int32_t ckv_bow_encode(const uint8_t* text, const int64_t* offsets, int32_t n_texts, int32_t dim,
                       const uint8_t* key, int32_t key_len, double* vectors, double* norms,
                       void* stream) {
  if (n_texts < 0 || dim < 1 || key_len < 0 || key_len > 64 || (key_len && !key)) return CKV_ERR_ARG;
  if (dim > kMaxBowDim) return CKV_ERR_UNSUPPORTED;
  if (n_texts == 0) return CKV_OK;
  if (!text || !offsets || !vectors || !norms) return CKV_ERR_ARG;
  BowKey k = {};
  for (int i = 0; i < key_len; ++i) k.bytes[i] = key[i];
  k.len = key_len;
  const size_t smem = (size_t)kEncWarps * dim * sizeof(int);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(bow_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    (void)cudaGetLastError();
    return CKV_ERR_CUDA;
  }
  const int grid = (int)std::min<int64_t>(cdiv((int64_t)n_texts, kEncWarps), 148 * 8);
  bow_encode_kernel<<<grid, kEncWarps * 32, smem, as_stream(stream)>>>(
      reinterpret_cast<const unsigned char*>(text), offsets, n_texts, dim, k, vectors, norms);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

int32_t ckv_tfidf_encode(const int32_t* ids, const int64_t* offsets, int32_t n_texts, const double* idf,
                         int32_t vocab, int32_t ld, double* vectors, double* norms, void* stream) {
  if (n_texts < 0 || vocab < 0 || ld < vocab || ld < 1) return CKV_ERR_ARG;
  if (n_texts == 0) return CKV_OK;
  if (!ids || !offsets || (vocab && !idf) || !vectors || !norms) return CKV_ERR_ARG;
  const int grid = (int)std::min<int64_t>(cdiv((int64_t)n_texts, kEncWarps), 148 * 8);
  tfidf_encode_kernel<<<grid, kEncWarps * 32, 0, as_stream(stream)>>>(ids, offsets, n_texts, idf, vocab, ld,
                                                                      vectors, norms);
  CKV_LAUNCH_CHECK();
  return CKV_OK;
}

}  // extern "C"
