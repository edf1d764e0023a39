// Shared device helpers for the ckv kernels (sm_100a).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ckv.h"

#define CKV_LAUNCH_CHECK()                                   \
  do {                                                       \
    if (cudaPeekAtLastError() != cudaSuccess) {              \
      (void)cudaGetLastError();                              \
      return CKV_ERR_CUDA;                                   \
    }                                                        \
  } while (0)

namespace ckv {

constexpr int kHeadDim = 128;   // D of the specialised batched path
constexpr int kGroup = 32;      // group_size (harness.py:44 default)
constexpr int kChunk = 32;      // chunk_size (harness.py:43 default)
constexpr int kGroupsPerRow = kHeadDim / kGroup;  // gpr = 4

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u32_as_h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

__device__ __forceinline__ bool fp16_bits_finite(uint16_t b) { return (b & 0x7C00u) != 0x7C00u; }

// D[16x8] += A[16x16] . B[16x8], fp16 operands, fp32 accumulate.
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Transpose an 8x8 b16 matrix held in mma-fragment layout across the warp.
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- Tile-native arena layout ----------------------------------------------------------
// The quantized arenas are stored in 16-row tiles whose bytes are laid out in the order the
// decode kernel's MMA fragments consume them (lane-ordered 16-byte slots), so a tile moves
// HBM -> shared memory with fully coalesced 16-byte copies and every fragment read is one
// conflict-free shared load with no shuffling.  Tile t of a segment covers arena rows
// [16t, 16t+16) (segments start at multiples of 32 rows).  Within a tile, rt = row % 16.  The
// reference row packing (_numpy.py:70-86) puts element i at bits [i b, (i+1) b) of LE word
// i b / 32: an INT2 row is 32 bytes (byte B = elements 4B..4B+3), an INT4 row 16 words (16-bit
// piece P = elements 4P..4P+3).  The decode takes every 32-element group G as its own k-steps
// (K) / m-tiles (V), so lane (g, c) of a tile holds, per group:
//   K: elements 32G + 8c + [0, 8) of tokens g and g+8 (INT2: bytes 8G+2c, 8G+2c+1 of both
//      tokens interleaved in one word; INT4: the reference's word 4G + c of each token);
//   V: elements 32G + 4g + [0, 4) of tokens 2c, 2c+1 (and 2c+8, 2c+9), the two tokens in the
//      two halves of a word (INT2: bytes 8G + g, one per half; INT4: pieces 8G + g).
// The functions give the byte offset of that byte (INT2) / 16-bit piece (INT4) inside its
// tile; metadata (lo, hi) of group G has hf 0 = lo, 1 = hi.  The reference row format is
// recovered exactly by the inverse gather (ckv_arena_export).
constexpr int kTileRows = 16;
constexpr int kTileBytes2 = 512;    // INT2 codes tile (16 rows x 32 B)
constexpr int kTileBytes4 = 1024;   // INT4 codes tile (16 rows x 64 B)
constexpr int kTileBytesMeta = 256; // metadata tile (16 rows x 4 groups x (lo, hi))
// K and V share one interleaved buffer per tier: [K codes | V codes | K meta | V meta]
constexpr int kBlock2 = 2 * kTileBytes2 + 2 * kTileBytesMeta;  // 1536 B per INT2 tile
constexpr int kBlock4 = 2 * kTileBytes4 + 2 * kTileBytesMeta;  // 2560 B per INT4 tile

// K INT2 byte B of row rt: lane (rt & 7, c = (B & 7) / 2), word G = B / 8,
// byte [tok rt < 8: 0 | rt >= 8: 1] + 2 (B & 1)
__host__ __device__ __forceinline__ int tile_byte_k2(int rt, int B) {
  return 16 * (4 * (rt & 7) + ((B & 7) >> 1)) + 4 * (B >> 3) + (rt >> 3) + 2 * (B & 1);
}
// V INT2 byte B: lane (g = B & 7, c = (rt & 7) / 2), word 2 (rt >= 8) + G / 2 (G = B / 8),
// byte 2 (rt & 1) + (G & 1)
__host__ __device__ __forceinline__ int tile_byte_v2(int rt, int B) {
  return 16 * (4 * (B & 7) + ((rt & 7) >> 1)) + 4 * (2 * (rt >> 3) + (B >> 4)) + 2 * (rt & 1) + ((B >> 3) & 1);
}
// K INT4 piece hf of word w: rows g / g+8 in two 512-B halves; lane (rt & 7, w & 3), word w / 4
__host__ __device__ __forceinline__ int tile_off_k4(int rt, int w, int hf) {
  return 512 * (rt >> 3) + 16 * (4 * (rt & 7) + (w & 3)) + 4 * (w >> 2) + 2 * hf;
}
// V INT4 piece P = 2w + hf: tokens 2c, 2c+1 / 2c+8, 2c+9 in two 512-B halves; lane
// (P & 7, (rt & 7) / 2), word G = P / 8, half rt & 1
__host__ __device__ __forceinline__ int tile_off_v4(int rt, int w, int hf) {
  const int P = 2 * w + hf;
  return 512 * (rt >> 3) + 16 * (4 * (P & 7) + ((rt & 7) >> 1)) + 4 * (P >> 3) + 2 * (rt & 1);
}
// K metadata: lane (g, c) = [(lo, hi) tok g group c, (lo, hi) tok g+8 group c]
__host__ __device__ __forceinline__ int tile_off_km(int rt, int G, int hf) {
  return ((rt & 7) * 4 + G) * 8 + (rt >> 3) * 4 + hf * 2;
}
// V metadata: entry (G, c) = [(lo tok 2c, 2c+1), (hi tok 2c, 2c+1), (lo 2c+8, 2c+9), (hi ...)]
__host__ __device__ __forceinline__ int tile_off_vm(int rt, int G, int hf) {
  return (G * 4 + ((rt & 7) >> 1)) * 16 + ((rt >> 3) * 2 + hf) * 4 + (rt & 1) * 2;
}

}  // namespace ckv
