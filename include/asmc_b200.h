/*
 * asmc_b200.h -- C-ABI of the B200-native SAIS / SSMC sampler hot path.
 *
 * This is the drop-in boundary between the host side (the C++ mirror of the
 * reference `asmc` API in paper_2408_12057_b200/csrc/host/, its pybind11
 * module, bench.py) and the sm_100a CUDA kernels in libasmc_b200.so.  Plain C
 * types only: pointers, sizes, PODs; host buffers in, host buffers out.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/).  The reference has no FFI of its
 * own besides pybind11 (python/bindings.cpp), so the entry points are what
 * those bindings call into:
 *
 *   asmc_run_smc          <- asmc::run_smc            include/asmc/engine.hpp:77-78, src/engine.cpp:97-188
 *   asmc_run_sais_single  <- asmc::run_sais_single    include/asmc/drivers.hpp:84-86, src/drivers.cpp:72-182
 *   asmc_run_rounds       <- asmc::run_ssmc/run_sais  include/asmc/drivers.hpp:48-55, src/drivers.cpp:186-232
 *   asmc_sais_partials    <- the per-wave block fold of run_sais_single, src/drivers.cpp:113-146
 *                            (one particle range per GPU; see asmc_fold_partials)
 *   asmc_fold_partials    <- the ordered fold + report tail, src/drivers.cpp:137-176
 *   asmc_smc_shard_*      <- asmc::run_smc split per GPU: step_pass (src/engine_detail.hpp:113-156),
 *                            ess/decide (src/engine.cpp:46-59,82-95,140-160), systematic
 *                            resample + gather (src/engine.cpp:61-80,161-173)
 *   asmc_run_zja          <- asmc::run_zja            include/asmc/drivers.hpp:88-111, src/drivers.cpp:234-341
 *   asmc_zja_next_beta    <- asmc::zja_next_beta      include/asmc/schedule.hpp:51-64, src/schedule.cpp:199-264
 *   asmc_run_pt           <- asmc::run_pt (NRPT)      include/asmc/pt.hpp:14-77, src/pt.cpp:21-152
 *   asmc_systematic_resample <- asmc::systematic_resample  src/engine.cpp:61-80
 *   asmc_ess              <- asmc::ess                src/engine.cpp:46-59
 *   asmc_barrier_estimate <- asmc::barrier_estimate   src/schedule.cpp:41-56
 *   asmc_generate_schedule<- asmc::generate_schedule  src/schedule.cpp:144-187
 *   asmc_local_barrier    <- asmc::local_barrier      src/schedule.cpp:189-197
 *   asmc_budget           <- asmc::budget             src/drivers.cpp:33-49
 *   asmc_rng_*            <- asmc::rng::Stream        include/asmc/rng.hpp:41-105 (parity hooks)
 *   asmc_trajectories     <- detail::weight_and_move  src/engine_detail.hpp:27-41 (parity hook:
 *                            per-particle states after every step of a SAIS pass)
 *
 * Error convention: every function returns ASMC_OK (0) or one of the codes
 * below; asmc_last_error() returns the thread-local message.  The host C++
 * mirror rethrows the reference exception class with that message
 * (include/asmc/errors.hpp:9-37, std::invalid_argument, std::domain_error).
 * There is no CPU fallback: a target or kernel the device does not implement
 * returns ASMC_ERR_CAPABILITY, a missing GPU returns ASMC_ERR_CUDA.
 */
#ifndef ASMC_B200_H
#define ASMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ---- */
#define ASMC_OK 0
#define ASMC_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument            */
#define ASMC_ERR_DOMAIN 2           /* std::domain_error                */
#define ASMC_ERR_CAPABILITY 3       /* asmc::capability_error           */
#define ASMC_ERR_DEGENERATE 4       /* asmc::degenerate_weights_error   */
#define ASMC_ERR_EVALUATION 5       /* asmc::evaluation_error           */
#define ASMC_ERR_CUDA 6             /* device missing / CUDA failure    */
#define ASMC_ERR_INTERNAL 7

/* ---- target plugins (include/asmc/target.hpp:54-96 + new plugins) ---- */
#define ASMC_TARGET_GAUSSIAN_SHIFT 0 /* p = {mu0, mu1, sigma}                       target.cpp:57-113  */
#define ASMC_TARGET_MIXTURE 1        /* p = {ref_sigma, weight, mu1, s1, mu2, s2}   target.cpp:115-157 */
#define ASMC_TARGET_SCALE_GAUSSIAN 2 /* p = {sigma0, sigma1}: N(0,s0^2 I) -> N(0,s1^2 I), config 2 (new) */
/* Bayesian logistic regression, config 4 (new): eta = N(0, sigma_p^2 I), V(theta) =
 * sum_i y_i x_i.theta - softplus(x_i.theta); p = {sigma_p, n}; data = X (n x dim), y (n).
 * Device path: rng = philox, precision = fp32, likelihood on tcgen05 (split-bf16). */
#define ASMC_TARGET_LOGISTIC 3
/* Relaxed Ising model on an L x L torus, config 5 (new): spins marginalised by the
 * Hubbard-Stratonovich transform, coordinates y in R^{L*L} (i = a L + b), A = delta I +
 * K (Adj + 4 I), u = A y, log p(y) = sum_i -y_i u_i / 2 + log 2cosh(u_i);
 * eta = N(0, sigma^2 I), V = log p - log eta; p = {L, K, delta, sigma}, dim = L * L.
 * Z(1) = (2 pi)^{n/2} |A|^{-1/2} e^{(delta + 4K) n / 2} Z_Ising(K) (Kaufman, exact).
 * Device path: rng = philox, precision = fp32, L in {8, 16, 32, 64}; rwmh_cycle, hmc, identity. */
#define ASMC_TARGET_ISING 4

/* ---- forward kernels (include/asmc/kernel.hpp:11-27) ---- */
#define ASMC_KERNEL_IDEALIZED 0
#define ASMC_KERNEL_RWMH 1
#define ASMC_KERNEL_IDENTITY 2
/* new: Hamiltonian Monte Carlo cycling through step_sizes as the leapfrog
 * epsilon (one trajectory of `leapfrog` steps per step size per sweep; unit
 * mass; momentum = the trajectory's d normals, accept uniform after them) */
#define ASMC_KERNEL_HMC 3
/* new: elliptical slice sampling w.r.t. the Gaussian reference eta (Murray, Adams &
 * MacKay 2010), `sweeps` updates per step.  Draw order per update: d normals for
 * nu ~ eta, uniform u (log y = beta V(x) + log u), uniform for theta in [0, 2 pi),
 * one uniform per bracket shrink (at most ASMC_SLICE_MAX_SHRINK, then x is kept).
 * Accept x' = mu + (x - mu) cos theta + (nu - mu) sin theta iff beta V(x') > log y. */
#define ASMC_KERNEL_SLICE 4
#define ASMC_SLICE_MAX_SHRINK 100
#define ASMC_MAX_STEP_SIZES 16

/* ---- resampling policies (include/asmc/engine.hpp:22) ---- */
#define ASMC_POLICY_NEVER 0
#define ASMC_POLICY_ALWAYS 1
#define ASMC_POLICY_ADAPTIVE_ESS 2
#define ASMC_POLICY_STABILIZED 3

/* ---- driver modes (include/asmc/drivers.hpp:12) ---- */
#define ASMC_MODE_SSMC 0
#define ASMC_MODE_SAIS 1

/* ---- execution options (new; the reference has one CPU path) ---- */
#define ASMC_RNG_XOSHIRO 0 /* the reference's keyed xoshiro256++ streams, bit-identical words */
#define ASMC_RNG_PHILOX 1  /* counter-based Philox4x32-10 (oracle/shadow/asmc/rng.hpp)       */
#define ASMC_PREC_FP64 0   /* reference arithmetic: fp64 state, reference operation order   */
#define ASMC_PREC_FP32 1   /* fp32 positions/densities, fp64 log-weights and accumulators   */

typedef struct asmc_target_desc {
  int32_t kind;
  int32_t reserved;
  uint64_t dim;
  double p[8];
  /* host data of data-backed plugins (LOGISTIC: X row-major n x dim float32,
   * then y[n] float32 in {0,1}); copied to the device per call */
  const void* data;
  uint64_t data_bytes;
} asmc_target_desc;

typedef struct asmc_kernel_desc {
  int32_t kind;
  int32_t n_step_sizes;
  int32_t sweeps;
  int32_t leapfrog; /* HMC leapfrog steps per trajectory */
  double step_sizes[ASMC_MAX_STEP_SIZES];
} asmc_kernel_desc;

typedef struct asmc_exec {
  int32_t rng;       /* ASMC_RNG_*  */
  int32_t precision; /* ASMC_PREC_* */
  int32_t device;    /* CUDA ordinal */
  int32_t lanes;     /* lanes per particle: 0 = auto, else 1/4/32 (fp32 + philox only) */
  uint64_t stream;   /* cudaStream_t to enqueue on; 0 = the library's own stream */
} asmc_exec;

/* LogAccumulator state (include/asmc/logsum.hpp:47-48 / :82-83). */
typedef struct asmc_logacc {
  double max;
  double sum;
} asmc_logacc;

/* RunReport fields (include/asmc/engine.hpp:33-45).  Arrays are caller-owned,
 * length T+1 (resample_times: capacity T); any of them may be NULL. */
typedef struct asmc_report {
  double* log_g0;
  double* log_g1;
  double* log_g2;
  double* ess_trace; /* run_smc only; left untouched by SAIS (empty in the reference) */
  double* cum_log_z;
  uint8_t* resampled;
  int32_t* resample_times;
  int32_t n_resample_times;
  int32_t reserved;
  double log_z_hat;
  double elbo_hat;
  double wall_seconds;
  uint64_t kernel_applications;
} asmc_report;

/* ---- library ---- */
const char* asmc_last_error(void);
int asmc_version(void);
/* number of CUDA devices; 0 on a host without a GPU (never a CPU fallback) */
int asmc_device_count(void);
/* kernels launched on the calling thread since the last reset (bench accounting) */
uint64_t asmc_launch_count(int reset);

/* ---- samplers ---- */
int asmc_run_smc(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                 const double* betas, int32_t steps, uint64_t n_particles, int32_t policy,
                 double rho, uint64_t seed, uint64_t round, const asmc_exec* exec,
                 asmc_report* out);

int asmc_run_sais_single(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                         const double* betas, int32_t steps, uint64_t n_particles,
                         uint64_t seed, uint64_t round, const asmc_exec* exec,
                         asmc_report* out);

/* Per-round outputs of asmc_run_rounds; arrays sized rounds (scalars) or
 * rounds * (max_steps + 1) (per-step rows, row k = round k+1). */
typedef struct asmc_rounds_out {
  int32_t max_steps; /* row stride - 1; must be >= every round's T */
  int32_t reserved;
  uint64_t* n_particles;
  int32_t* steps;
  double* betas;
  double* log_g0;
  double* log_g1;
  double* log_g2;
  double* ess_trace; /* ssmc only */
  double* cum_log_z;
  uint8_t* resampled;
  double* lambda; /* barrier knots Lambda_hat_t, schedule.cpp:41-56 */
  double* log_z_hat;
  double* elbo_hat;
  double* wall_seconds;
  uint64_t* kernel_applications;
} asmc_rounds_out;

int asmc_run_rounds(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                    int32_t mode, uint64_t n_particles, int32_t rounds, int32_t policy,
                    double rho, uint64_t seed, uint64_t memory_cap_bytes,
                    const asmc_exec* exec, asmc_rounds_out* out);

/* Batched seeds (replaces the replicate loop of experiment.cpp:96-140 for
 * run_sais): the round loop of asmc_run_rounds(ASMC_MODE_SAIS) for nseeds seeds at once,
 * the seed an extra launch dimension of the one-lane pass (lanes 1, dim <= 1024).  Each
 * seed's results equal its own asmc_run_rounds call bit for bit.  Host outputs:
 * per (seed s, round k) at [s * rounds + k]: log_z_hat, elbo_hat, lambda_total (Lambda-hat);
 * per round k: n_particles, steps, wall_seconds (CUDA events around the round, all seeds). */
typedef struct asmc_seeds_out {
  uint64_t* n_particles;
  int32_t* steps;
  double* wall_seconds;
  double* log_z_hat;
  double* elbo_hat;
  double* lambda_total;
} asmc_seeds_out;
int asmc_run_sais_seeds(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                        uint64_t n_particles, int32_t rounds, const uint64_t* seeds, int32_t nseeds,
                        const asmc_exec* exec, asmc_seeds_out* out);

/* Multi-GPU SAIS: partials of particles [p_begin, p_end) of an n_particles round.
 * p_begin must be a multiple of ASMC_FOLD_CHUNK.  Writes per fold chunk
 * (ASMC_FOLD_CHUNK particles) and per step t = 1..T the four accumulators
 * g0, g1, g2, elbo as asmc_logacc:
 *   partials[((c * (T + 1) + t) * 4 + a]   for c in [0, chunks(p_begin, p_end)).
 * The chunk partial is a fixed tree over 256-particle blocks, so the fold of
 * all chunks (in chunk order) is independent of how chunks map to GPUs. */
#define ASMC_FOLD_CHUNK 262144
uint64_t asmc_fold_chunks(uint64_t p_begin, uint64_t p_end);
int asmc_sais_partials(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                       const double* betas, int32_t steps, uint64_t n_particles,
                       uint64_t p_begin, uint64_t p_end, uint64_t seed, uint64_t round,
                       const asmc_exec* exec, asmc_logacc* partials);
/* Ordered fold of all chunk partials of a round (chunk order) and the report
 * tail of run_sais_single (drivers.cpp:148-176). Host-side scalar code. */
int asmc_fold_partials(const asmc_logacc* partials, uint64_t chunks, int32_t steps,
                       uint64_t n_particles, asmc_report* out);
/* Device-buffer variants (multi-GPU SAIS, distributed.run_sais): the partials are
 * written to / read from DEVICE memory in the same exchange layout, on exec->stream,
 * so the all-gather runs device to device and the fold runs on the GPU. */
int asmc_sais_partials_dev(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                           const double* betas, int32_t steps, uint64_t n_particles,
                           uint64_t p_begin, uint64_t p_end, uint64_t seed, uint64_t round,
                           const asmc_exec* exec, asmc_logacc* partials_dev);
int asmc_fold_partials_dev(const asmc_logacc* partials_dev, uint64_t chunks, int32_t steps,
                           uint64_t n_particles, const asmc_exec* exec, asmc_report* out);

/* Multi-GPU SSMC: run_smc (src/engine.cpp:97-188) with the particles of one round
 * split into contiguous shards, one per GPU, each shard starting at a multiple of
 * ASMC_FOLD_CHUNK.  The caller owns the communication (NCCL/gloo through
 * torch.distributed, or anything else) and passes DEVICE buffers; the library
 * never syncs except where a host decision is needed (decide, plan).  Every rank
 * computes the same totals, decisions and ancestors as a single-GPU asmc_run_smc
 * with rng = philox, precision = fp32 (bit-identical report).  Per step t:
 *   1. asmc_smc_shard_step    pass + local fold -> this shard's chunk partials,
 *                             chunk-major: partials[c * ASMC_SHARD_NACC + a]
 *   2. caller all-gathers the partials of all shards in rank order
 *   3. asmc_smc_shard_decide  fold + ESS + policy (engine.cpp:82-95,140-160);
 *                             if *resample, copies this shard's log-weights
 *                             (asmc_smc_shard_exchange_len entries) to lw_out
 *   4. (resample) caller all-gathers the log-weights in rank order (8 B/particle)
 *   5. asmc_smc_shard_plan    every rank builds the reference's sequential CDF over
 *                             all n log-weights (engine.cpp:61-80, bit for bit) and the
 *                             global ancestors; slot_begin[r] (host, world+1) = first
 *                             output slot whose ancestor lies in shard r
 *   6. asmc_smc_shard_pack    rows of the ancestors of slots [slot_begin[me],
 *                             slot_begin[me+1]) in slot order (row_bytes each)
 *   7. caller all-to-all: shard r's packed rows for slots in shard q go to q
 *   8. asmc_smc_shard_accept  the received rows (this shard's slots, in order)
 *                             become the particles; log-weights reset to 0
 * asmc_smc_shard_report after step T fills the (replicated) run_smc report. */
#define ASMC_SHARD_NACC 6 /* accumulators per chunk partial: g0 g1 g2 elbo sq top2 */
typedef struct asmc_smc_shard asmc_smc_shard;
int asmc_smc_shard_create(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                          const double* betas, int32_t steps, uint64_t n_particles,
                          uint64_t p_begin, uint64_t p_end, int32_t policy, double rho,
                          uint64_t seed, uint64_t round, const asmc_exec* exec,
                          asmc_smc_shard** out);
void asmc_smc_shard_destroy(asmc_smc_shard* shard);
uint64_t asmc_smc_shard_chunks(const asmc_smc_shard* shard);
uint64_t asmc_smc_shard_exchange_len(const asmc_smc_shard* shard);
uint64_t asmc_smc_shard_row_bytes(const asmc_smc_shard* shard);
int asmc_smc_shard_step(asmc_smc_shard* shard, int32_t t, asmc_logacc* partials_dev);
int asmc_smc_shard_decide(asmc_smc_shard* shard, int32_t t, const asmc_logacc* all_partials_dev,
                          uint64_t all_chunks, double* lw_out_dev, int32_t* resample);
int asmc_smc_shard_plan(asmc_smc_shard* shard, const double* all_log_weights_dev, uint64_t n_all,
                        int32_t world, const uint64_t* shard_p_begin, uint64_t* slot_begin);
int asmc_smc_shard_pack(asmc_smc_shard* shard, void* rows_dev);
int asmc_smc_shard_accept(asmc_smc_shard* shard, const void* rows_dev);
int asmc_smc_shard_report(asmc_smc_shard* shard, asmc_report* out);
/* Multi-GPU ZJA (drivers.cpp:234-341 across GPUs): a shard in ZJA mode has an open-ended
 * schedule (run_smc(never) whose step t is the last iff beta_t = 1).  Per step: eval
 * (cache log eta, V), probes -- each returns this shard's per-chunk (m1, m2) partials of
 * the one-step discrepancy at b2 (b2 < 0: the log-weights' lse) for the caller to
 * all-gather and fold in chunk order (schedule.cpp:201-264's bisection runs on every rank,
 * identically) --, set_beta(t, chosen), then asmc_smc_shard_step / decide as in SSMC. */
int asmc_zja_shard_create(const asmc_target_desc* target, const asmc_kernel_desc* kernel, uint64_t n_particles,
                          uint64_t p_begin, uint64_t p_end, uint64_t seed, uint64_t round, int32_t max_steps,
                          const asmc_exec* exec, asmc_smc_shard** out);
int asmc_zja_shard_eval(asmc_smc_shard* shard);
int asmc_zja_shard_probe(asmc_smc_shard* shard, double beta, double b2, asmc_logacc* chunk_partials);
int asmc_zja_shard_set_beta(asmc_smc_shard* shard, int32_t t, double beta);
/* The same search kept on the device (no host round trip per probe): search_begin arms
 * it for step t; probe_dev writes this shard's (chunks, 2) partials at the search's
 * current point to DEVICE memory (stream-ordered, no sync); the caller all-gathers them
 * (e.g. ncclAllGather, chunk order over ranks) and search_step folds them in chunk order
 * and advances the bisection identically on every rank, writing betas[t] when done;
 * probes after that are no-ops.  search_poll (the one synchronising call) reports
 * done / the chosen beta / the non-monotone warning / probes taken. */
int asmc_zja_shard_search_begin(asmc_smc_shard* shard, int32_t t, double delta_star);
int asmc_zja_shard_probe_dev(asmc_smc_shard* shard, asmc_logacc* chunk_partials_dev);
int asmc_zja_shard_search_step(asmc_smc_shard* shard, const asmc_logacc* all_partials_dev, uint64_t all_chunks);
int asmc_zja_shard_search_poll(asmc_smc_shard* shard, int32_t* done, double* beta, int32_t* warn,
                               int32_t* probes);
/* parity hook: copy this shard's particles (row-major, row_bytes each) and log-weights */
int asmc_smc_shard_state(asmc_smc_shard* shard, void* rows_host, double* log_w_host);

/* ---- online schedule adaptation (ZJA) ---- */
/* ZjaOptions (drivers.hpp:88-97) */
typedef struct asmc_zja_opts {
  uint64_t n_particles;
  int32_t target_steps; /* K: pilot resolution when delta_star == 0 */
  int32_t max_steps;
  double delta_star;    /* 0 -> pilot round sets (Lambda_hat / K)^2 */
  uint64_t seed;
} asmc_zja_opts;

/* ZjaOutcome (drivers.hpp:99-104).  Main-round arrays have `capacity` entries
 * (>= steps + 1); pilot arrays target_steps + 1.  Any array may be NULL. */
typedef struct asmc_zja_out {
  int32_t capacity;  /* in */
  int32_t steps;     /* out: adaptive run's T */
  int32_t pilot_ran; /* out: 1 when delta_star == 0 (pilot = round 1, main = round 2) */
  int32_t warning;   /* out: the non-monotone bisection fallback was taken */
  double delta_star; /* out: threshold used */
  double* betas;     /* main schedule */
  double* lambda;    /* main barrier estimate */
  asmc_report main;
  double* pilot_lambda;
  asmc_report pilot;
} asmc_zja_out;

/* Device path: one probe = a log-sum-exp over the particles with log eta and V
 * cached per particle.  precision fp64: the reference's sequential accumulation
 * (one device thread); fp32: the whole bisection in one cooperative launch. */
int asmc_run_zja(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                 const asmc_zja_opts* options, const asmc_exec* exec, asmc_zja_out* out);
/* positions: n x dim row-major (host) */
int asmc_zja_next_beta(const asmc_target_desc* target, double beta, const double* positions,
                       uint64_t n_particles, const double* log_weights, double delta_star,
                       double tol, const asmc_exec* exec, double* beta_next, int32_t* warning);

/* ---- non-reversible parallel tempering (NRPT) ---- */
/* PtOptions (pt.hpp:18-24) + `replicas`: independent runs with seeds seed .. seed +
 * replicas - 1, all in one launch (one CTA per run, one thread per level). */
typedef struct asmc_pt_opts {
  int32_t iterations;
  int32_t burn_in; /* -1 -> iterations / 10 */
  uint64_t seed;
  uint64_t round;
  int32_t replicas;
  int32_t reserved;
} asmc_pt_opts;

/* PtReport (pt.hpp:45-58) per replica r; caller-owned arrays, any may be NULL:
 *   log_z_hat[r], trace[(r * iterations + it) * (levels + 1) + n],
 *   swap_accepted[(r * iterations + it) * (levels + 1) + lo],
 *   swap_attempts / swap_accepts[r * (levels + 1) + lo] */
typedef struct asmc_pt_out {
  double* log_z_hat;
  double* trace;
  uint8_t* swap_accepted;
  uint64_t* swap_attempts;
  uint64_t* swap_accepts;
  uint64_t kernel_applications; /* per replica: levels * iterations */
  double wall_seconds;
  int32_t burn_in;              /* resolved */
  int32_t reserved;
} asmc_pt_out;

/* levels <= 255; targets with a device pass (shift, mixture, scale), d <= 1024 */
int asmc_run_pt(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const double* betas,
                int32_t levels, const asmc_pt_opts* options, const asmc_exec* exec, asmc_pt_out* out);

/* ---- parity hooks ---- */
/* key = {seed, round, particle, step, substep} (rng.hpp:11-17) */
int asmc_rng_u64(int32_t rng, const uint64_t key[5], uint64_t count, uint64_t* out);
int asmc_rng_uniform(int32_t rng, const uint64_t key[5], uint64_t count, double* out);
/* normals computed in `precision` (fp64: double Box-Muller; fp32: device fp32 path) */
int asmc_rng_normal(int32_t rng, int32_t precision, const uint64_t key[5], uint64_t count,
                    double* out);

/* States after every step of a SAIS pass for the listed particles:
 * x_out[(i * (T + 1) + t) * dim + k], log_w_out[i * (T + 1) + t], t = 0 is the init draw. */
int asmc_trajectories(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                      const double* betas, int32_t steps, uint64_t seed, uint64_t round,
                      const uint64_t* particles, uint64_t count, const asmc_exec* exec,
                      double* x_out, double* log_w_out);

/* Systematic resampling on the device (engine.cpp:61-80): the reference's SEQUENTIAL
 * fp64 CDF reproduced bit for bit by a parallel exact scan:
 * l1 = logsumexp (logsum.hpp:97-101), cum_j = fl(cum_{j-1} + exp(lw_j - l1)),
 * a_m = first j with !(cum_j < (m + u)/n), clamped.  u is the uniform the reference
 * draws from key (seed, round, 0, t, resample). */
int asmc_systematic_resample(const double* log_weights, uint64_t n, double u, int32_t device,
                             uint32_t* ancestors);
/* parity hooks: the CDF the search runs on (n doubles) and l1; logsumexp alone
 * (asmc::logsumexp, logsum.hpp:97-101; -inf for an empty or all -inf input) */
int asmc_resample_cdf(const double* log_weights, uint64_t n, int32_t device, double* cum_out,
                      double* l1_out);
int asmc_logsumexp(const double* log_weights, uint64_t n, int32_t device, double* out);
/* parity hook: which = 0 -> the device's glibc-exact exp, 1 -> its correctly rounded log */
int asmc_exact_math(int32_t which, const double* x, uint64_t n, int32_t device, double* out);
int asmc_ess(const double* log_weights, uint64_t n, int32_t device, double* out);

/* ---- schedule adaptation (device kernels, bit-exact with the host oracle) ---- */
int asmc_barrier_estimate(const double* log_g0, const double* log_g1, const double* log_g2,
                          const double* betas, int32_t steps, int32_t device, double* lambda);
int asmc_generate_schedule(const double* lambda, const double* beta, int32_t knots,
                           int32_t t_new, int32_t device, double* betas_out);
int asmc_local_barrier(const double* lambda, const double* beta, int32_t knots, int32_t device,
                       double* out);
int asmc_budget(uint64_t n_particles, int32_t steps, uint64_t dim, uint64_t memory_cap_bytes,
                int32_t mode, uint64_t* n_out, int32_t* steps_out);

/* ---- measurement hooks (bench.py; not part of the reference interface) ---- */
/* When enabled, every particle-pass launch on the calling thread is bracketed
 * by CUDA events on its own stream; collect returns per-launch milliseconds
 * and the algorithmic normal draws each launch had to make. */
int asmc_profile_enable(int on);
int asmc_profile_collect(double* ms, double* normals, int max_launches, int* n_launches);
/* same, plus the normals each launch actually generated (the shared-memory RWMH pass
 * draws fewer than the algorithmic count when proposals are rejected early); equals
 * the algorithmic count for launches without a counter */
int asmc_profile_collect_drawn(double* ms, double* units, double* drawn, int max_launches, int* n_launches);
/* Generator peak: `blocks` CTAs x 256 threads each drawing quads_per_thread
 * Philox quads (4 fp32 normals) in registers; returns kernel seconds. */
int asmc_peak_normals(int32_t device, int32_t blocks, uint64_t quads_per_thread, double* seconds);

#ifdef __cplusplus
}
#endif
#endif /* ASMC_B200_H */
