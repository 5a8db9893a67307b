// Config-5 (relaxed Ising on an L x L torus) device path: argument block and launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pass_kernel.cuh"

namespace asmcdev {

// Particle state rows (shared layout with the logistic engine, so the weight kernel,
// resampling gather and SMC loop are reused): [y_0 .. y_{n-1}, V (double at float
// offset n), pad] -> row = n + 4 floats.
struct IsArgs {
  float* const* state;  // device array of the two state buffers
  const int* xcur;      // live buffer index
  uint64_t n_local, p_begin, seed, round;
  int L;
  int row;
  float K;       // coupling (beta_phys J)
  float c;       // delta + 4 K: diagonal of A
  float inv_s2;  // 1 / sigma^2 of the reference
  float sigma;
  double vconst;  // n (log sigma + log sqrt(2 pi)): constant part of V
  KernelCfg kc;
  int* err;
};

bool ising_side_supported(int L);
size_t ising_smem_bytes(int L);
// mode 0: y ~ eta (init stream) and V(y); mode 1: the kernel's move at beta_t (RWMH
// cycle or HMC cycle), V(y) refreshed
cudaError_t launch_is_move(const IsArgs& A, int mode, const double* betas, int t, cudaStream_t s);

}  // namespace asmcdev
