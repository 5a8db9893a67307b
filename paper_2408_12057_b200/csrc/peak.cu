// Generator peak microbenchmark (compiled like the fp32 pass: FMA contraction on).
#include "engine_kernels.h"

namespace asmcdev {
// Peak-rate microbenchmark of the exact generator + transform the fp32 pass
// uses (PhiloxKey::normals4<float>, bm_pair_f32), with no memory traffic: the
// denominator of the pass kernel's issue roofline.
__global__ void __launch_bounds__(256) peak_normals_kernel(uint64_t quads_per_thread, float* sink) {
  PhiloxKey k;
  k.init(1, 1, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, 1, 1);
  float acc = 0.f;
  for (uint64_t q = 0; q < quads_per_thread; ++q) {
    float z[4];
    k.normals4<float>((uint32_t)q, z);
    acc += (z[0] + z[1]) + (z[2] + z[3]);
  }
  if (acc == 1234.5f) sink[0] = acc;  // keep the work observable
}
cudaError_t launch_peak_normals(int blocks, uint64_t quads_per_thread, float* sink, cudaStream_t s) {
  peak_normals_kernel<<<blocks, 256, 0, s>>>(quads_per_thread, sink);
  return cudaGetLastError();
}
}  // namespace asmcdev
