// Probe (tuning aid): is mma.sync m16n8k32 s8 x s8 -> s32 a native tensor-core instruction on
// sm_100a (IMMA in the SASS), and its throughput against m16n8k16 f16 (HMMA) at 16 warps/SM with
// 8 independent accumulator chains.  Context: INT2/INT4 codes in int8 operands would take 4 codes
// per AND (one LOP3 per register) instead of 2 as fp16 subnormals, at the price of an integer q.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int8_probe tools/int8_probe.cu
// cuobjdump -sass int8_probe | grep -c IMMA
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mma_s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <bool S8>
__global__ void tput(int* out, int iters, uint32_t seed) {
  int di[8][4] = {};
  float df[8][4] = {};
  uint32_t a = 0x01020304u ^ (seed & threadIdx.x), b = 0x01010101u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (S8) mma_s8(di[c], a, a + c, a, a, b, b);
      else mma_f16(df[c], a, a + c, a, a, b, b);
    }
    a += 0x01000000u;  // loop-variant operand: no hoisting
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += di[c][0] + di[c][1] + di[c][2] + di[c][3] + (int)(df[c][0] + df[c][3]);
  if (s == 123456789) out[0] = s;
}

int main() {
  int* o;
  cudaMalloc(&o, 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int s8 = 0; s8 < 2; ++s8) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (s8) tput<true><<<sms, 512>>>(o, iters, 0);
      else tput<false><<<sms, 512>>>(o, iters, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double n = (double)sms * 16 * iters * 8;  // warp-level MMAs
      if (rep) printf("%s: %.1f warp-MMAs per SM per us (16 warps/SM), %.2f ns per MMA per SMSP; %.1f dense T(FL)OP/s\n",
                      s8 ? "m16n8k32 s8" : "m16n8k16 f16", n / sms / (ms * 1e3), ms * 1e6 / (n / sms / 4),
                      n * 2.0 * 16 * 8 * (s8 ? 32 : 16) / (ms * 1e-3) / 1e12);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
