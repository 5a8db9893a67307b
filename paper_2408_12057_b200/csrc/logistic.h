// Config-4 (logistic regression) device path: argument block and launchers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_common.cuh"

namespace asmcdev {

// Particle state rows: [theta_0 .. theta_{d-1}, V (double at float offset d), pad]
// -> row = d + 4 floats, 16-byte aligned for d % 4 == 0.
struct LgArgs {
  float* const* state;  // device array of the two state buffers (double buffer)
  const int* xcur;      // live buffer index
  double* lw;
  const float* y;
  const double* w;   // X^T y (d): the linear part sum_j y_j l_j = theta . w
  uint64_t n;        // data rows
  uint64_t n_local;  // particles of this launch
  uint64_t p_begin;
  int d;
  int row;  // floats per state row
  uint64_t seed, round;
  int t;    // annealing step (RNG key)
  int pad;
  double sigma_p;
  int* err;
};

size_t logistic_smem_bytes(int d);
cudaError_t make_x_maps(const void* hi, const void* lo, uint64_t n_pad, int d, CUtensorMap* mhi,
                        CUtensorMap* mlo);
cudaError_t launch_lg_split(const float* X, uint64_t n, int d, uint64_t n_pad, void* hi, void* lo,
                            cudaStream_t s);
cudaError_t launch_lg_init(const LgArgs& A, cudaStream_t s);
// w = X^T y in fp64, fixed summation order (one CTA per column)
cudaError_t launch_lg_xty(const float* X, const float* y, uint64_t n, int d, double* w, cudaStream_t s);
cudaError_t launch_lg_weight(const LgArgs& A, const double* betas, int t, LogAcc* part, uint64_t stride,
                             cudaStream_t s);
cudaError_t launch_lg_eval(const CUtensorMap& mhi, const CUtensorMap& mlo, const LgArgs& A, int mode,
                           const double* betas, float step, int q, cudaStream_t s);

}  // namespace asmcdev
