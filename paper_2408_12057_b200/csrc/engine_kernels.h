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
  double max_lw;  // max post-update log-weight
  double total;   // CDF total cum[n-1]
  double err_val;
  int resample_now;
  int gather_pending;  // SSMC: the last event's gather is deferred into the next step pass
  int n_resample;
  int err;
  int err_step;
};
static_assert(sizeof(SmcState) == 88, "distributed.py SIZEOF_SMCSTATE mirrors this (e2e byte counts)");

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

// Scratch of the reference-CDF resampler (refcdf.cu), per 256-particle block.
struct RefCdfWork {
  double* bmax;    // block max -> exclusive prefix max (l1 pass)
  double* ba;      // approximate block composite s -> ba s + bb
  double* bb;
  double* sstart;  // approximate running value at each block start (nblk + 1)
  unsigned long long* tot;     // exact integer total of a stable block at its binade
  unsigned long long* bstart;  // exact start of each stable block, in units of its binade
  int* kb;         // binade of a stable block, or unstable
  unsigned long long* ovf;  // slot runs of heavy ancestors (lo, hi, j), at most n / 1024
  unsigned int* novf;
  double* gmax;    // max log-weight
  double* l1;      // logsumexp of the log-weights (the reference's bits)
  double* opv;     // per particle: the element operation's exp value of the current chain
                   // (written once by the block-affine phase, read by classification,
                   // replays and materialisation); sign bit set = LogAccumulator rescale
  unsigned long long* prof;  // optional: %globaltimer at each phase end (16 entries)
};
size_t refcdf_work_bytes(uint64_t n);
void refcdf_work_carve(void* base, uint64_t n, RefCdfWork* w);
// Systematic resampling (engine.cpp:61-80) with the reference's sequential CDF, bit for
// bit: st->u is the uniform, ancestors to anc (want_anc), the CDF to cum (n doubles),
// st->total = cum[n-1].  gated: return at once unless st->resample_now.  One cooperative
// launch.
cudaError_t launch_refcdf(const double* lw, uint64_t n, SmcState* st, int gated, const RefCdfWork* w,
                          double* cum, uint32_t* anc, int want_anc, int sms, cudaStream_t s);

// parity hook: which = 0 -> gexp (glibc's exp), 1 -> crlog (correctly rounded log)
cudaError_t launch_exact_math(int which, const double* x, uint64_t n, double* out, cudaStream_t s);

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
cudaError_t launch_gather(const uint32_t* anc, uint64_t n, uint64_t row_bytes, void* const* xbuf,
                          int* xcur, double* lw, SmcState* st, int sms, cudaStream_t s);
// deferred gather (the pass kernels' SSMC step): mark the event's rows pending instead of
// copying them; settle flips the buffers after the pass that consumed them
cudaError_t launch_defer_gather(SmcState* st, cudaStream_t s);
cudaError_t launch_settle(int* xcur, SmcState* st, cudaStream_t s);
cudaError_t launch_generate_schedule(const double* lambda, const double* beta, int knots, int t_new,
                                     double* out, double* scratch, int* err, cudaStream_t s);
// batched seeds (SAIS round loop over many seeds in one launch per kernel)
cudaError_t launch_sais_report_batch(const LogAcc* tot, int T, uint64_t n, RoundDev* rd, int nseeds,
                                     cudaStream_t s);
cudaError_t launch_generate_schedule_batch(const double* lambda, uint64_t lam_stride, const double* beta, int knots,
                                           int t_new, double* out, double* scratch, int* err, int nseeds,
                                           cudaStream_t s);
cudaError_t launch_local_barrier(const double* lambda, const double* beta, int knots, double* out,
                                 double* scratch, int* err, cudaStream_t s);
cudaError_t launch_barrier(const double* g0, const double* g1, const double* g2, int T,
                           double* lambda, int* err, cudaStream_t s);
cudaError_t launch_rng(int rng, int what, int precision, const uint64_t key[5], uint64_t count,
                       void* out, cudaStream_t s);
cudaError_t launch_peak_normals(int blocks, uint64_t quads_per_thread, float* sink, cudaStream_t s);
cudaError_t launch_ess(const double* lw, uint64_t n, double* out, int* err, cudaStream_t s);

// ---- multi-GPU SAIS: chunk partials <-> exchange layout, on the device ----
cudaError_t launch_chunks_to_exchange(const LogAcc* chunk, uint64_t nch, int T, LogAcc* x, cudaStream_t s);
cudaError_t launch_exchange_to_chunks(const LogAcc* x, uint64_t nch, int T, LogAcc* chunk, cudaStream_t s);

// ---- sharded SSMC (one particle shard per GPU) ----
// per-shard chunk partials [a][c] -> exchange layout [c][a]
cudaError_t launch_chunk_major(const LogAcc* in, uint64_t nch, LogAcc* out, cudaStream_t s);
// sequential fold of [C][a] chunk partials into tot[a] (== fold_chunks_final order)
cudaError_t launch_fold_chunk_major(const LogAcc* in, uint64_t nch, LogAcc* tot, cudaStream_t s);
// resampling exchange: every rank runs launch_refcdf on the all-gathered log-weights
// (the global CDF and ancestors a_m, identical on every rank); shard r's output slots are
// [slot_begin[r], slot_begin[r+1]) = the slots whose ancestor it owns (a_m non-decreasing)
cudaError_t launch_slot_bounds(const uint32_t* anc, uint64_t n, const uint64_t* shard_p, int world,
                               const SmcState* st, uint64_t* slot_begin, cudaStream_t s);
// rows x[anc[i] - p0] for i < count into dst, in slot order
cudaError_t launch_pack_rows(const uint32_t* anc, uint64_t count, uint64_t p0, uint64_t row_bytes, const void* x,
                             void* dst, int sms, cudaStream_t s);

}  // namespace asmcdev
