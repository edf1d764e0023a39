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
// [16t, 16t+16) (segments start at multiples of 32 rows).  Within a tile, rt = row % 16,
// w = 32-bit word of the reference row packing (_numpy.py:70-86: INT2 w = 0..7, INT4 w =
// 0..15), hf = 16-bit half of that word; metadata (lo, hi) of group G has hf 0 = lo, 1 = hi.
// The functions give the byte offset of that 16-bit piece inside its tile; the reference row
// format is recovered exactly by the inverse gather (ckv_arena_export).
constexpr int kTileRows = 16;
constexpr int kTileBytes2 = 512;    // INT2 codes tile (16 rows x 32 B)
constexpr int kTileBytes4 = 1024;   // INT4 codes tile (16 rows x 64 B)
constexpr int kTileBytesMeta = 256; // metadata tile (16 rows x 4 groups x (lo, hi))
// K and V share one interleaved buffer per tier: [K codes | V codes | K meta | V meta]
constexpr int kBlock2 = 2 * kTileBytes2 + 2 * kTileBytesMeta;  // 1536 B per INT2 tile
constexpr int kBlock4 = 2 * kTileBytes4 + 2 * kTileBytesMeta;  // 2560 B per INT4 tile

// K INT2: lane (g, c) = [tok g: w 2c, 2c+1 | tok g+8: w 2c, 2c+1]
__host__ __device__ __forceinline__ int tile_off_k2(int rt, int w, int hf) {
  return ((rt & 7) * 4 + (w >> 1)) * 16 + (rt >> 3) * 8 + (w & 1) * 4 + hf * 2;
}
// V INT2: lane (g, c) = [(w g: lo half of tok 2c, 2c+1), (hi halves), same for tok 2c+8, 2c+9]
__host__ __device__ __forceinline__ int tile_off_v2(int rt, int w, int hf) {
  return (w * 4 + ((rt & 7) >> 1)) * 16 + ((rt >> 3) * 2 + hf) * 4 + (rt & 1) * 2;
}
// K INT4: rows g / g+8 in two 512-B halves; lane (g, c) = group c as
//   [(lo w4c, lo w4c+1), (hi w4c, hi w4c+1), (lo w4c+2, lo w4c+3), (hi w4c+2, hi w4c+3)]
__host__ __device__ __forceinline__ int tile_off_k4(int rt, int w, int hf) {
  const int wi = w & 3;
  return (rt >> 3) * 512 + ((rt & 7) * 4 + (w >> 2)) * 16 + ((wi >> 1) * 2 + hf) * 4 + (wi & 1) * 2;
}
// V INT4: toks 2c, 2c+1 / 2c+8, 2c+9 in two 512-B halves; lane (g, c) =
//   [(lo w2g of tok 2c, 2c+1), (hi w2g ...), (lo w2g+1 ...), (hi w2g+1 ...)]
__host__ __device__ __forceinline__ int tile_off_v4(int rt, int w, int hf) {
  return (rt >> 3) * 512 + ((w >> 1) * 4 + ((rt & 7) >> 1)) * 16 + ((w & 1) * 2 + hf) * 4 + (rt & 1) * 2;
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
