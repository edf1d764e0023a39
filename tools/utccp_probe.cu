// Probe (next-round design check): ptxas accepts tcgen05.cp with the 4-bit -> 8-bit expansion
// (.b8x16.b4x16_p64 -> SASS UTCCP...U4x16P64) for sm_100a.  Compile-only:
// nvcc -gencode arch=compute_100a,code=sm_100a -c tools/utccp_probe.cu -o /tmp/u.o && cuobjdump -sass /tmp/u.o | grep UTCCP
#include <cstdint>
__global__ void k(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b.b8x16.b4x16_p64 [%0], %1;" :: "r"(taddr), "l"(desc));
  asm volatile("tcgen05.cp.cta_group::1.128x128b.b8x16.b4x16_p64 [%0], %1;" :: "r"(taddr), "l"(desc));
}
