// Dispatch of launch_pass_fp64 / launch_pass_fp32 onto the per-target slices.
#include "dispatch.h"

namespace asmcdev {

#define DECL(P, T)                                                                        \
  cudaError_t launch_pass_fp##P##_##T(int rng, Layout L, const PassArgs& A, uint64_t blocks, \
                                      cudaStream_t s);
DECL(64, 0) DECL(64, 1) DECL(64, 2) DECL(32, 0) DECL(32, 1) DECL(32, 2)

cudaError_t launch_pass_fp64(int kind, int rng, Layout L, const PassArgs& A, uint64_t blocks,
                             cudaStream_t s) {
  switch (kind) {
    case 0: return launch_pass_fp64_0(rng, L, A, blocks, s);
    case 1: return launch_pass_fp64_1(rng, L, A, blocks, s);
    case 2: return launch_pass_fp64_2(rng, L, A, blocks, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pass_fp32(int kind, int rng, Layout L, const PassArgs& A, uint64_t blocks,
                             cudaStream_t s) {
  switch (kind) {
    case 0: return launch_pass_fp32_0(rng, L, A, blocks, s);
    case 1: return launch_pass_fp32_1(rng, L, A, blocks, s);
    case 2: return launch_pass_fp32_2(rng, L, A, blocks, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace asmcdev
