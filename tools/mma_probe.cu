// Probes (tuning aid): (1) mma.sync m16n8k16 f16->f32 throughput per SM at 4/8/16 warps per SM
// with independent accumulator chains; (2) whether fp16 subnormal A operands are exact in HMMA.
#include <cstdio>
#include <cuda_fp16.h>
#include <cstdint>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CH>
__global__ void tput(float* out, int iters, uint32_t seed) {
  float d[CH][4] = {};
  uint32_t a = 0x3c003c00u ^ (seed & threadIdx.x), b = 0x38003800u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma(d[c], a, a + c, a, a, b, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1234.5f) out[0] = s;
}

// A = subnormal fp16 codes (c << j), B = 1.0: D row sums must equal sum(c) * 2^(j-24) exactly
__global__ void subn(float* out) {
  const int lane = threadIdx.x;
  const uint32_t one = 0x3c003c00u;
  float d[4] = {0, 0, 0, 0};
  // a-regs: codes 1..3 at bit j in each half
  uint32_t x = ((uint32_t)(lane % 4) << 2) | ((uint32_t)((lane + 1) % 4) << 18);  // j = 2
  mma(d, x, x, x, x, one, one);
  for (int e = 0; e < 4; ++e) out[lane * 4 + e] = d[e];
}

int main() {
  float* o;
  cudaMalloc(&o, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      tput<8><<<sms, 32 * warps>>>(o, iters, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double mmas_per_sm = (double)warps * iters * 8;
      double cyc = ms * 1e-3 * clk * 1e3;
      if (rep) printf("warps/SM %2d: %.2f cycles per HMMA.16816 per SM (%.2f per SMSP), %.1f TFLOP/s\n", warps,
                      cyc / mmas_per_sm, 4 * cyc / mmas_per_sm, mmas_per_sm * sms * 4096.0 / (ms * 1e-3) / 1e12);
    }
  }
  subn<<<1, 32>>>(o);
  float h[128];
  cudaMemcpy(h, o, 512, cudaMemcpyDeviceToHost);
  // expected: every D element = sum over k of A[row][k] * 1 = for row r: 8 halves... compute on host
  double want_unit = 1.0 / (1 << 22);  // code at bit 2 of a subnormal = c * 2^-22
  printf("subnormal probe D[0..7]: ");
  for (int i = 0; i < 8; ++i) printf("%.9g ", h[i] / want_unit);
  printf("(in units of 2^-22)\n");
  return 0;
}
