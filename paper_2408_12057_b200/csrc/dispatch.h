// Host-side dispatch of the particle-pass instantiations.
#pragma once
#include <cuda_runtime.h>

#include "pass_kernel.cuh"
#include "pass_smem.cuh"

namespace asmcdev {

struct Layout {
  int lanes;  // G
  int kmax;   // coordinates per lane held in registers / local memory
};

// fp64 reference-order path (pass_fp64.cu, -fmad=false): lanes == 1, kmax 16 or 1024
cudaError_t launch_pass_fp64(int kind, int rng, Layout L, const PassArgs& A, uint64_t blocks,
                             cudaStream_t s);
// fp32 fast path (pass_fp32.cu)
cudaError_t launch_pass_fp32(int kind, int rng, Layout L, const PassArgs& A, uint64_t blocks,
                             cudaStream_t s);

}  // namespace asmcdev
