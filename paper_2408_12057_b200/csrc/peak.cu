// Generator peak microbenchmark (compiled like the fp32 pass: FMA contraction on).
#include "engine_kernels.h"

namespace asmcdev {
// Peak-rate microbenchmark of the exact generator + transform the fp32 shared-memory
// pass runs (PhiloxKeyC: round keys in the kernel's parameter bank, normals4<float> ->
// SFU Box-Muller, the quad loop unrolled 4x like the pass's MH loop), with no memory
// traffic: the denominator of the pass kernel's issue roofline.
__global__ void __launch_bounds__(256) peak_normals_kernel(const __grid_constant__ PhiloxRoundKeys rk,
                                                           uint64_t quads_per_thread, float* sink) {
  PhiloxKeyC k;
  k.init(rk, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, 1);
  float acc = 0.f;
#pragma unroll 4
  for (uint64_t q = 0; q < quads_per_thread; ++q) {
    float z[4];
    k.normals4<float>((uint32_t)q, z);
    acc += (z[0] + z[1]) + (z[2] + z[3]);
  }
  if (acc == 1234.5f) sink[0] = acc;  // keep the work observable
}
cudaError_t launch_peak_normals(int blocks, uint64_t quads_per_thread, float* sink, cudaStream_t s) {
  PhiloxRoundKeys rk;
  philox_round_keys(1, 1, 1, rk);
  peak_normals_kernel<<<blocks, 256, 0, s>>>(rk, quads_per_thread, sink);
  return cudaGetLastError();
}
}  // namespace asmcdev
