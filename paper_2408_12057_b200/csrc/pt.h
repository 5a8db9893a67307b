// Non-reversible parallel tempering (src/pt.cpp) on the device: argument block.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pass_kernel.cuh"

namespace asmcdev {

constexpr int kPtMaxLevels = 255;  // one CTA (<= 256 threads) per run

struct PtArgs {
  TgtParams tg;
  KernelCfg kc;
  const double* betas;  // levels + 1
  int levels;
  int iterations;
  uint64_t seed0;       // replica r runs seed0 + r (experiment.cpp:96-101)
  uint64_t round;
  int replicas;
  int pad;
  void* scratch;        // replicas x (levels + 1) x dim Real: swap exchange rows
  double* trace;        // replicas x iterations x (levels + 1): V post-exploration, pre-swap
  uint8_t* accepted;    // replicas x iterations x (levels + 1): pair (n, n+1) swapped
};

cudaError_t launch_pt(const PtArgs& A, bool fp64, int rng, cudaStream_t s);

}  // namespace asmcdev
