// Probe (tuning aid): mma.sync m16n8k32 e4m3 x e4m3 -> f32 on sm_100a.  Finding: NOT a native
// tensor-core instruction there — ptxas lowers each one to 16 F2FP.F16.E4M3.UNPACK_B + 4
// HMMA.16816 + 8 FADD (cuobjdump -sass of this binary); (1) below hoists the conversions of its
// loop-invariant operands, so its "throughput" is not that of real code.
//  (1) throughput against m16n8k16 f16 at 16 warps/SM, 8 independent accumulator chains;
//  (2) precision: D = C + A.B with A = small integer codes as e4m3 bytes (c < 16 is exactly
//      c * 2^-9), B random finite e4m3, C random fp32; compared with the exact sum in double.
//      Reports the largest error in units of 2^-24 of (|C| + sum |a b|), i.e. whether the
//      products are summed at fp32 precision or truncated to fewer bits.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp8_probe tools/fp8_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>

__device__ __forceinline__ void mma8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <bool FP8>
__global__ void tput(float* out, int iters, uint32_t seed) {
  float d[8][4] = {};
  uint32_t a = 0x01020304u ^ (seed & threadIdx.x), b = 0x38383838u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (FP8) mma8(d[c], a, a + c, a, a, b, b);
      else mma16(d[c], a, a + c, a, a, b, b);
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1234.5f) out[0] = s;
}

// one warp: A [16][32] bytes, B [32][8] bytes (B[k][n]), C/D [16][8] f32; `chain` MMAs with
// independent B matrices accumulate into the same D (as a split q would)
__global__ void prec(const uint8_t* A, const uint8_t* B, const float* C, float* D, int chain) {
  const int lane = threadIdx.x, g = lane >> 2, c = lane & 3;
  auto ldA = [&](int row, int k0) {
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= (uint32_t)A[row * 32 + k0 + i] << (8 * i);
    return r;
  };
  float d[4] = {C[g * 8 + 2 * c], C[g * 8 + 2 * c + 1], C[(g + 8) * 8 + 2 * c], C[(g + 8) * 8 + 2 * c + 1]};
  const uint32_t a0 = ldA(g, 4 * c), a1 = ldA(g + 8, 4 * c), a2 = ldA(g, 16 + 4 * c), a3 = ldA(g + 8, 16 + 4 * c);
  for (int s = 0; s < chain; ++s) {
    const uint8_t* Bs = B + s * 256;
    uint32_t b0 = 0, b1 = 0;
    for (int i = 0; i < 4; ++i) {
      b0 |= (uint32_t)Bs[(4 * c + i) * 8 + g] << (8 * i);
      b1 |= (uint32_t)Bs[(16 + 4 * c + i) * 8 + g] << (8 * i);
    }
    mma8(d, a0, a1, a2, a3, b0, b1);
  }
  D[g * 8 + 2 * c] = d[0]; D[g * 8 + 2 * c + 1] = d[1];
  D[(g + 8) * 8 + 2 * c] = d[2]; D[(g + 8) * 8 + 2 * c + 1] = d[3];
}

static double e4m3(uint8_t x) {
  const int s = x >> 7, e = (x >> 3) & 15, m = x & 7;
  double v = e == 0 ? std::ldexp((double)m, -9) : std::ldexp(1.0 + m / 8.0, e - 7);
  return s ? -v : v;
}

int main() {
  float* o;
  cudaMalloc(&o, 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int fp8 = 0; fp8 < 2; ++fp8) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (fp8) tput<true><<<sms, 512>>>(o, iters, 0);
      else tput<false><<<sms, 512>>>(o, iters, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double n = (double)sms * 16 * iters * 8;  // warp-level MMAs
      if (rep) printf("%s: %.1f warp-MMAs per SM per us (16 warps/SM), %.2f ns per MMA per SMSP\n",
                      fp8 ? "m16n8k32 e4m3" : "m16n8k16 f16", n / sms / (ms * 1e3), ms * 1e6 / (n / sms / 4));
    }
  }
  std::mt19937 rng(7);
  uint8_t *dA, *dB;
  float *dC, *dD;
  cudaMalloc(&dA, 512);
  cudaMalloc(&dB, 256 * 4);
  cudaMalloc(&dC, 512);
  cudaMalloc(&dD, 512);
  for (int chain : {1, 2, 3}) {
    for (int cmode = 0; cmode < 3; ++cmode) {
      double worst = 0;
      for (int trial = 0; trial < 200; ++trial) {
        uint8_t hA[512], hB[1024];
        float hC[128], hD[128];
        for (int i = 0; i < 512; ++i) hA[i] = (uint8_t)(rng() % 16);
        for (int i = 0; i < 256 * chain; ++i) {
          uint8_t x;
          do { x = (uint8_t)(rng() & 0xff); } while ((x & 0x7f) == 0x7f);
          // the s-th split: magnitudes ~ 2^-4s of the first (as q hi / mid / lo terms)
          if (i >= 256) { const int e = (x >> 3) & 15; x = (uint8_t)((x & 0x87) | ((e > 4 * (i / 256) ? e - 4 * (i / 256) : 0) << 3)); }
          hB[i] = x;
        }
        std::uniform_real_distribution<float> U(-1.f, 1.f);
        for (int i = 0; i < 128; ++i) hC[i] = cmode == 0 ? 0.f : (cmode == 1 ? U(rng) : 1000.f * U(rng));
        cudaMemcpy(dA, hA, 512, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, 256 * chain, cudaMemcpyHostToDevice);
        cudaMemcpy(dC, hC, 512, cudaMemcpyHostToDevice);
        prec<<<1, 32>>>(dA, dB, dC, dD, chain);
        cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
        for (int r = 0; r < 16; ++r)
          for (int n = 0; n < 8; ++n) {
            double ex = hC[r * 8 + n], mag = std::fabs(hC[r * 8 + n]);
            for (int s = 0; s < chain; ++s)
              for (int k = 0; k < 32; ++k) {
                const double p = e4m3(hA[r * 32 + k]) * e4m3(hB[s * 256 + k * 8 + n]);
                ex += p;
                mag += std::fabs(p);
              }
            if (mag > 0) worst = std::fmax(worst, std::fabs(hD[r * 8 + n] - ex) / mag * 16777216.0);
          }
      }
      printf("chain %d, C %s: max |D - exact| = %.2f x 2^-24 (|C| + sum|ab|)\n", chain,
             cmode == 0 ? "0" : (cmode == 1 ? "U(-1,1)" : "1000 U(-1,1)"), worst);
    }
  }
  return 0;
}
