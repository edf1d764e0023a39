// Probe (tuning aid): HMMA m16n8k16 with fp16 SUBNORMAL A operands (raw codes c << j, no
// exponent bits: value c * 2^(j-24)) against normal fp16 B operands of wide range.  The decode
// kernel's quantized tiles feed the codes this way (no bias term, no per-element dequant): the
// products must be exact (no flush to zero) and the fp32 accumulation within its usual rounding.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A [16][16] halves (row-major), B [16][8] (k-major), D [16][8]
__global__ void k(const uint16_t* A, const uint16_t* B, float* D) {
  const int lane = threadIdx.x, g = lane >> 2, c = lane & 3;
  auto a2 = [&](int r, int k0) { return (uint32_t)A[r * 16 + k0] | ((uint32_t)A[r * 16 + k0 + 1] << 16); };
  auto b2 = [&](int k0, int n) { return (uint32_t)B[k0 * 8 + n] | ((uint32_t)B[(k0 + 1) * 8 + n] << 16); };
  float d[4] = {0, 0, 0, 0};
  mma(d, a2(g, 2 * c), a2(g + 8, 2 * c), a2(g, 2 * c + 8), a2(g + 8, 2 * c + 8), b2(2 * c, g), b2(2 * c + 8, g));
  D[g * 8 + 2 * c] = d[0]; D[g * 8 + 2 * c + 1] = d[1]; D[(g + 8) * 8 + 2 * c] = d[2]; D[(g + 8) * 8 + 2 * c + 1] = d[3];
}

static float h2f(uint16_t h) { __half x; memcpy(&x, &h, 2); return __half2float(x); }

int main() {
  uint16_t *A, *B; float* D;
  cudaMallocManaged(&A, 512); cudaMallocManaged(&B, 256); cudaMallocManaged(&D, 512);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s >> 8; };
  double worst = 0; int zero_flush = 0;
  for (int trial = 0; trial < 2000; ++trial) {
    const int j = (trial % 6) * 2;  // INT2 slots j = 0..10; INT4 uses j = 0, 4
    const int bits = trial & 1 ? 4 : 2;
    for (int i = 0; i < 256; ++i) A[i] = (uint16_t)((rnd() & ((1u << bits) - 1)) << (bits == 4 ? (j & 4) : j));
    const float range = (trial % 7 == 0) ? 60000.f : (trial % 3 == 0 ? 1000.f : 8.f);
    for (int i = 0; i < 128; ++i) { __half hb = __float2half_rn(((rnd() & 0xffff) / 65536.f * 2 - 1) * range); memcpy(&B[i], &hb, 2); }
    k<<<1, 32>>>(A, B, D);
    cudaDeviceSynchronize();
    for (int r = 0; r < 16; ++r)
      for (int n = 0; n < 8; ++n) {
        double ex = 0, mag = 0;
        for (int kk = 0; kk < 16; ++kk) { const double t = (double)A[r * 16 + kk] * ldexp(1.0, -24) * h2f(B[kk * 8 + n]); ex += t; mag += fabs(t); }
        const double err = fabs(D[r * 8 + n] - ex) / (mag > 0 ? mag : 1);
        if (mag > 0 && D[r * 8 + n] == 0.0f && ex != 0) ++zero_flush;
        if (err > worst) worst = err;
      }
  }
  printf("subnormal-A HMMA: worst |D - exact| / sum|terms| = %.3g (fp32 eps 1.19e-7), flushed results %d\n", worst, zero_flush);
  return 0;
}
