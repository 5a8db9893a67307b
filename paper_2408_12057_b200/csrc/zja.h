// Online schedule adaptation (ZJA; src/schedule.cpp:201-264, src/drivers.cpp:234-341):
// device argument block and launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_common.cuh"
#include "targets.cuh"

namespace asmcdev {

struct ZjaArgs {
  const double* lw;  // current log-weights [n]
  const double* lr;  // log eta(x_p) [n]            (reference order, from zja_eval)
  const double* V;   // V(x_p) [n]
  uint64_t n;
  double* betas;     // betas[t-1] = current beta; betas[t] <- next beta
  int t;
  int exact;         // 1: sequential reference-order accumulators (one thread)
  double delta;      // delta_star
  double tol;        // bisection tolerance (schedule.hpp:61-64 default 1e-10)
  int* warn;         // set when the non-monotone fallback was taken
  int* err;          // ASMC_ERR_DEGENERATE when all log-weights are -inf
  LogAcc* part;      // cooperative mode: 2 buffers x 2 accumulators x gridDim
};

// lr / V of every particle of the live state buffer (fp64 target terms, summed in
// coordinate order, as AnnealedTarget::log_gamma does)
cudaError_t launch_zja_eval(const TgtParams& T, bool fp64_state, const void* const* xbuf, const int* xcur,
                            uint64_t n, double* lr, double* V, const int* err, cudaStream_t s);
// zja_next_beta for step t; `grid_blocks` (cooperative mode) from zja_grid_blocks
cudaError_t launch_zja_next_beta(const ZjaArgs& A, int grid_blocks, cudaStream_t s);
int zja_grid_blocks(int device);
// multi-GPU probes: block partials (m1, m2) of dhat(b2) (b2 < 0: lse of lw in m1)
cudaError_t launch_zja_probe_blocks(const double* lw, const double* V, uint64_t n, double beta, double b2,
                                    LogAcc* part, uint64_t stride, cudaStream_t s);

// multi-GPU device-resident search (zja_search as a state machine; see zja.cu)
constexpr int kZjaSearchDone = 5;  // ZjaSearch::phase once beta_t is chosen
struct ZjaSearch {
  double beta, delta, tol, log_m0;
  double b2;            // the next probe point (phase 0: the log-weights' lse)
  double lo, hi, root;  // bisection interval / first root
  double chosen;        // beta_t once phase == done
  int phase, scan_i, warn, probes;
};
cudaError_t launch_zja_search_init(ZjaSearch* S, const double* betas, int t, double delta, double tol,
                                   cudaStream_t s);
cudaError_t launch_zja_probe_dev(const double* lw, const double* V, uint64_t n, const ZjaSearch* S, LogAcc* part,
                                 uint64_t stride, cudaStream_t s);
cudaError_t launch_zja_interleave(const LogAcc* zchunk, uint64_t nch, const ZjaSearch* S, LogAcc* out,
                                  cudaStream_t s);
cudaError_t launch_zja_search_step(ZjaSearch* S, const LogAcc* all, uint64_t nch, double* betas, int t, int* warn,
                                   int* err, cudaStream_t s);

}  // namespace asmcdev
