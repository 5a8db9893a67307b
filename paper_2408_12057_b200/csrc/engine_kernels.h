// Device-side estimator state and the launchers of engine_kernels.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_common.cuh"
#include "rng.cuh"

namespace asmcdev {

// run_smc's running estimator state (engine.cpp:120-127), device-resident so
// the step loop never waits on the host.
struct SmcState {
  double log_z, elbo, acc_dhat, den_log;
  double u;       // resampling uniform of the current step
  double max_lw;  // max post-update log-weight (CDF shift)
  double total;   // CDF total
  double err_val;
  int resample_now;
  int n_resample;
  int err;
  int err_step;
};

// Per-round outputs in device memory (arrays of T+1 unless noted).
struct RoundDev {
  double* log_g0;
  double* log_g1;
  double* log_g2;
  double* ess;
  double* cum_log_z;
  uint8_t* resampled;
  int32_t* resample_times;  // capacity T
  double* lambda;
  double* scalars;  // [0] log_z_hat, [1] elbo_hat
  SmcState* state;
};

cudaError_t launch_fold(bool exact, const LogAcc* part, uint64_t stride, uint64_t nblk, int row0,
                        int nrows, int nacc, LogAcc* chunk_scratch, LogAcc* out, cudaStream_t s);
cudaError_t launch_fold_chunks(const LogAcc* part, uint64_t stride, uint64_t nblk, int row0,
                               int nrows, int nacc, uint64_t nchunks, LogAcc* chunk_out,
                               cudaStream_t s);
cudaError_t launch_fold_chunks_final(const LogAcc* chunk, uint64_t nchunks, int row0, int nrows,
                                     int nacc, LogAcc* out, cudaStream_t s);
cudaError_t launch_sais_report(const LogAcc* tot, int T, uint64_t n, RoundDev* rd, cudaStream_t s);
cudaError_t launch_smc_decide(const LogAcc* tot_row, int t, int T, uint64_t n, int policy,
                              double rho, uint64_t seed, uint64_t round, int rng, RoundDev* rd,
                              cudaStream_t s, const double* zja_betas = nullptr);
cudaError_t launch_resample(const double* lw_in, uint64_t n, SmcState* st, double* cum,
                            double* btot, uint32_t* anc, cudaStream_t s);
cudaError_t launch_gather(const uint32_t* anc, uint64_t n, uint64_t row_bytes, void* const* xbuf,
                          int* xcur, double* lw, SmcState* st, int sms, cudaStream_t s);
cudaError_t launch_max(const double* lw, uint64_t n, SmcState* st, cudaStream_t s);
cudaError_t launch_generate_schedule(const double* lambda, const double* beta, int knots, int t_new,
                                     double* out, double* scratch, int* err, cudaStream_t s);
cudaError_t launch_local_barrier(const double* lambda, const double* beta, int knots, double* out,
                                 double* scratch, int* err, cudaStream_t s);
cudaError_t launch_barrier(const double* g0, const double* g1, const double* g2, int T,
                           double* lambda, int* err, cudaStream_t s);
cudaError_t launch_rng(int rng, int what, int precision, const uint64_t key[5], uint64_t count,
                       void* out, cudaStream_t s);
cudaError_t launch_peak_normals(int blocks, uint64_t quads_per_thread, float* sink, cudaStream_t s);
cudaError_t launch_ess(const double* lw, uint64_t n, double* out, int* err, cudaStream_t s);

// ---- sharded SSMC (one particle shard per GPU) ----
// per-shard chunk partials [a][c] -> exchange layout [c][a]
cudaError_t launch_chunk_major(const LogAcc* in, uint64_t nch, LogAcc* out, cudaStream_t s);
// sequential fold of [C][a] chunk partials into tot[a] (== fold_chunks_final order)
cudaError_t launch_fold_chunk_major(const LogAcc* in, uint64_t nch, LogAcc* tot, cudaStream_t s);
// local block CDF (no-op unless st->resample_now)
cudaError_t launch_cdf_blocks(const double* lw, uint64_t n, const SmcState* st, double* cum,
                              double* btot, cudaStream_t s);
// scan the all-gathered block totals (in place -> exclusive offsets, st->total),
// shift the local CDF by this shard's offsets, and find every shard's output-slot
// range: slot_begin[r] = #{m : pos_m <= boff[rank_blk[r]]}
cudaError_t launch_shard_plan(double* btot_all, uint64_t nblk_all, double* cum, uint64_t n_local,
                              uint64_t blk_begin, const uint64_t* rank_blk, int world, uint64_t n,
                              SmcState* st, uint64_t* slot_begin, cudaStream_t s);
// ancestors of output slots [slot_lo, slot_lo + count) within the local CDF,
// rows gathered into dst in slot order
cudaError_t launch_shard_pack(const double* cum, uint64_t n_local, const SmcState* st,
                              uint64_t slot_lo, uint64_t count, uint64_t n, uint32_t* anc,
                              uint64_t row_bytes, const void* x, void* dst, int sms, cudaStream_t s);

}  // namespace asmcdev
