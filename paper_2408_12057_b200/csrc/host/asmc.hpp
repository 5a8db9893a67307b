// Host C++ mirror of the reference `asmc` sampler API (/root/reference/proj/include/asmc/*.hpp):
// same namespace, type and function names, argument meaning and exception
// classes, so code written against the reference recompiles against this
// header.  Every sampler entry point forwards through the C-ABI of
// include/asmc_b200.h to the B200 kernels; nothing here samples on the CPU.
//
// The reference's include layout is kept: asmc/{rng,logsum,errors}.hpp hold their
// definitions, asmc/{target,kernel,engine,schedule,drivers,pt,theory}.hpp forward here,
// so `#include "asmc/target.hpp"` code (the reference's own test fixtures) compiles
// unchanged against -I csrc/host.
//
// Differences from the reference interface (documented in INTEGRATION.md):
//  * A target is a device plugin: AnnealedTarget subclasses provide a
//    descriptor (device_descriptor); the per-point virtuals (log_reference,
//    potential, sample_reference, exact_sample, log_gamma, analytic_*) keep the
//    reference's signatures for callers and plugins, but a target the device does
//    not implement raises capability_error when sampled (no CPU fallback).
//  * RunOptions / DriverOptions gain execution fields (rng, precision, device,
//    lanes).  Defaults reproduce the reference: keyed xoshiro streams, fp64
//    reference arithmetic.  `workers` and `chunk` are accepted and ignored
//    (results never depended on them).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "asmc/errors.hpp"
#include "asmc/logsum.hpp"
#include "asmc/rng.hpp"
#include "asmc_b200.h"

namespace asmc {

// ---- target.hpp -----------------------------------------------------------
struct Capabilities {
  bool analytic_log_z = false;
  bool exact_sampler = false;
  bool analytic_delta = false;
};

class AnnealedTarget {
 public:
  virtual ~AnnealedTarget() = default;
  virtual std::size_t dim() const = 0;
  virtual double log_reference(std::span<const double> x) const = 0;
  virtual double potential(std::span<const double> x) const = 0;
  virtual void sample_reference(rng::Stream& stream, std::span<double> out) const = 0;
  virtual Capabilities capabilities() const { return {}; }
  double log_gamma(double beta, std::span<const double> x) const;
  virtual double analytic_log_z(double beta) const;
  virtual double analytic_delta(double beta) const;
  virtual double analytic_discrepancy(double beta, double beta2) const;
  // exact draw from pi_beta (requires exact_sampler); host code for callers: the device
  // path draws with its own kernels
  virtual void exact_sample(double beta, rng::Stream& stream, std::span<double> out) const;
  // B200 plugin boundary: fill the device descriptor, or return false.
  virtual bool device_descriptor(asmc_target_desc* out) const { return false; }

 protected:
  void check_point(std::span<const double> x) const;
  static void check_beta(double beta);
};

class GaussianShiftTarget final : public AnnealedTarget {
 public:
  GaussianShiftTarget(double mu0, double mu1, double sigma, std::size_t dim);
  std::size_t dim() const override { return dim_; }
  double log_reference(std::span<const double> x) const override;
  double potential(std::span<const double> x) const override;
  void sample_reference(rng::Stream& stream, std::span<double> out) const override;
  Capabilities capabilities() const override { return {true, true, true}; }
  double analytic_log_z(double beta) const override;
  double analytic_delta(double beta) const override;
  double analytic_discrepancy(double beta, double beta2) const override;
  void exact_sample(double beta, rng::Stream& stream, std::span<double> out) const override;
  bool device_descriptor(asmc_target_desc* out) const override;
  double z() const { return z_; }

 private:
  double mu0_, mu1_, sigma_, z_;
  std::size_t dim_;
};

class MixtureTarget final : public AnnealedTarget {
 public:
  MixtureTarget(double ref_sigma, double weight, double mu1, double sigma1, double mu2,
                double sigma2, std::size_t dim);
  std::size_t dim() const override { return dim_; }
  double log_reference(std::span<const double> x) const override;
  double potential(std::span<const double> x) const override;
  void sample_reference(rng::Stream& stream, std::span<double> out) const override;
  bool device_descriptor(asmc_target_desc* out) const override;

 private:
  double ref_sigma_, weight_, mu1_, sigma1_, mu2_, sigma2_;
  std::size_t dim_;
};

// Config-2 plugin (new): N(0, s0^2 I) -> N(0, s1^2 I), both normalized.
class ScaleGaussianTarget final : public AnnealedTarget {
 public:
  ScaleGaussianTarget(double sigma0, double sigma1, std::size_t dim);
  std::size_t dim() const override { return dim_; }
  double log_reference(std::span<const double> x) const override;
  double potential(std::span<const double> x) const override;
  void sample_reference(rng::Stream& stream, std::span<double> out) const override;
  Capabilities capabilities() const override { return {true, true, true}; }
  double analytic_log_z(double beta) const override;
  double analytic_delta(double beta) const override;
  double analytic_discrepancy(double beta, double beta2) const override;
  void exact_sample(double beta, rng::Stream& stream, std::span<double> out) const override;
  bool device_descriptor(asmc_target_desc* out) const override;

 private:
  double tau(double beta) const;
  double s0_, s1_;
  std::size_t dim_;
};

// Config-4 plugin (new): Bayesian logistic regression posterior; X is n x dim
// row-major, y in {0, 1}; prior N(0, sigma_p^2 I).  Sampled on the tcgen05 path.
class LogisticTarget final : public AnnealedTarget {
 public:
  LogisticTarget(std::vector<float> X, std::vector<float> y, std::size_t dim, double sigma_p);
  std::size_t dim() const override { return dim_; }
  double log_reference(std::span<const double> x) const override;
  double potential(std::span<const double> x) const override;
  void sample_reference(rng::Stream& stream, std::span<double> out) const override;
  bool device_descriptor(asmc_target_desc* out) const override;
  std::size_t n_data() const { return y_.size(); }

 private:
  std::vector<float> data_;  // X then y, the C-ABI's packed layout
  std::vector<float> y_;
  std::size_t dim_;
  double sp_;
};

// Config-5 plugin (new): relaxed Ising model on an L x L torus (include/asmc_b200.h,
// ASMC_TARGET_ISING); coordinates y in R^{L*L}, coupling K, relaxation delta, eta = N(0, sigma^2 I).
class IsingTarget final : public AnnealedTarget {
 public:
  IsingTarget(int side, double coupling, double delta = 1.0, double sigma = 1.0);
  std::size_t dim() const override { return static_cast<std::size_t>(L_) * L_; }
  double log_reference(std::span<const double> x) const override;
  double potential(std::span<const double> x) const override;
  void sample_reference(rng::Stream& stream, std::span<double> out) const override;
  bool device_descriptor(asmc_target_desc* out) const override;
  int side() const { return L_; }

 private:
  int L_;
  double K_, delta_, sigma_;
};

double log_normal_pdf(double x, double mu, double sigma);

// ---- kernel.hpp -----------------------------------------------------------
// hmc (new): Hamiltonian Monte Carlo cycling through step_sizes as epsilon
// slice (new): elliptical slice sampling w.r.t. the Gaussian reference, `sweeps` updates
enum class KernelKind { idealized_exact, rwmh_cycle, identity, hmc, slice };

struct Kernel {
  KernelKind kind = KernelKind::idealized_exact;
  std::vector<double> step_sizes = {0.1, 1.0, 10.0};
  int sweeps = 1;
  int leapfrog = 10;  // new: HMC leapfrog steps per trajectory
};

void validate_kernel(const Kernel& kernel);

// ---- engine.hpp -----------------------------------------------------------
struct Schedule {
  std::vector<double> betas;
  static Schedule uniform(int steps);
  int steps() const { return static_cast<int>(betas.size()) - 1; }
  void validate() const;
};

enum class ResamplePolicy { never, always, adaptive_ess, stabilized };

// execution choices of the device path (new)
enum class Rng { xoshiro = ASMC_RNG_XOSHIRO, philox = ASMC_RNG_PHILOX };
enum class Precision { fp64 = ASMC_PREC_FP64, fp32 = ASMC_PREC_FP32 };

struct IncrementStats {
  std::vector<double> log_g0, log_g1, log_g2;
  int steps() const { return static_cast<int>(log_g0.size()) - 1; }
};

struct RunReport {
  Schedule schedule;
  std::size_t n_particles = 0;
  double log_z_hat = 0.0;
  double elbo_hat = 0.0;
  IncrementStats stats;
  std::vector<int> resample_times;
  std::vector<double> ess_trace;
  std::vector<double> cum_log_z;
  std::vector<std::uint8_t> resampled;
  std::uint64_t kernel_applications = 0;
  double wall_seconds = 0.0;
};

struct RunOptions {
  std::size_t n_particles = 1024;
  ResamplePolicy policy = ResamplePolicy::adaptive_ess;
  double rho = 0.5;
  std::uint64_t seed = 0;
  std::uint64_t round = 0;
  int workers = 1;
  // device execution (new)
  Rng rng = Rng::xoshiro;
  Precision precision = Precision::fp64;
  int device = 0;
  int lanes = 0;

  void validate() const;
};

double ess(std::span<const double> log_weights);
// engine.cpp:61-80 on the device, bit for bit (the reference's sequential CDF):
// the reference's signature (u = stream.uniform(), as the reference draws it) and a
// given-u overload
std::vector<std::uint32_t> systematic_resample(std::span<const double> log_weights, rng::Stream& stream);
std::vector<std::uint32_t> systematic_resample(std::span<const double> log_weights, double u,
                                               int device = 0);
bool decide_resample(ResamplePolicy policy, int t, int total_steps, double ess_value,
                     std::size_t n_particles, double accumulated_dhat, double rho);
RunReport run_smc(const AnnealedTarget& target, const Kernel& kernel, const Schedule& schedule,
                  const RunOptions& options);

// ---- schedule.hpp ---------------------------------------------------------
double discrepancy_hat(const IncrementStats& stats, int t);
double cess(const IncrementStats& stats, int t, std::size_t n_particles);

struct BarrierEstimate {
  std::vector<double> lambda;
  std::vector<double> beta;
  double total() const { return lambda.empty() ? 0.0 : lambda.back(); }
};

BarrierEstimate barrier_estimate(const IncrementStats& stats, const Schedule& schedule);
Schedule generate_schedule(const BarrierEstimate& estimate, int t_new);
std::vector<double> local_barrier(const BarrierEstimate& estimate);

// schedule.hpp:51-64
struct ZjaResult {
  double beta_next = 1.0;
  bool warning = false;
};
ZjaResult zja_next_beta(const AnnealedTarget& target, double beta, std::span<const double> positions,
                        std::size_t n_particles, std::span<const double> log_weights, double delta_star,
                        double tol = 1e-10);

// ---- drivers.hpp ----------------------------------------------------------
enum class DriverMode { ssmc, sais };

struct BudgetPlan {
  std::size_t n_particles = 1;
  int steps = 1;
};

BudgetPlan budget(std::size_t n_particles, int steps, std::size_t dim,
                  std::uint64_t memory_cap_bytes, DriverMode mode);

struct DriverOptions {
  std::size_t n_particles = 1024;
  int rounds = 1;
  ResamplePolicy policy = ResamplePolicy::adaptive_ess;
  double rho = 0.5;
  std::uint64_t seed = 0;
  int workers = 1;
  std::uint64_t memory_cap_bytes = std::uint64_t{4096} << 20;
  std::size_t chunk = 0;
  // device execution (new)
  Rng rng = Rng::xoshiro;
  Precision precision = Precision::fp64;
  int device = 0;
  int lanes = 0;

  void validate() const;
};

struct RoundResult {
  int round = 1;
  RunReport report;
  BarrierEstimate barrier;
};

std::vector<RoundResult> run_ssmc(const AnnealedTarget& target, const Kernel& kernel,
                                  const DriverOptions& options);
std::vector<RoundResult> run_sais(const AnnealedTarget& target, const Kernel& kernel,
                                  const DriverOptions& options);
RunReport run_sais_single(const AnnealedTarget& target, const Kernel& kernel,
                          const Schedule& schedule, const RunOptions& options,
                          std::size_t chunk = 0);

// drivers.hpp:88-111
struct ZjaOptions {
  std::size_t n_particles = 1024;
  int target_steps = 32;
  double delta_star = 0.0;
  std::uint64_t seed = 0;
  int workers = 1;
  int max_steps = 100000;
  // device execution (new)
  Rng rng = Rng::xoshiro;
  Precision precision = Precision::fp64;
  int device = 0;
  int lanes = 0;

  void validate() const;
};

struct ZjaOutcome {
  std::vector<RoundResult> rounds;  // pilot round first (when one ran), then the adaptive run
  double delta_star = 0.0;
  bool warning = false;
};

ZjaOutcome run_zja(const AnnealedTarget& target, const Kernel& kernel, const ZjaOptions& options);

// ---- pt.hpp (non-reversible parallel tempering) -------------------------------
struct PtOptions {
  int iterations = 1024;
  int burn_in = -1;  // -1 -> iterations / 10
  std::uint64_t seed = 0;
  std::uint64_t round = 1;
  // device execution (new)
  Rng rng = Rng::xoshiro;
  Precision precision = Precision::fp64;
  int device = 0;
  void validate() const;
};

struct PotentialTrace {
  int iterations = 0;
  int levels = 0;
  std::vector<double> values;
  double at(int iteration, int level) const {
    return values[static_cast<std::size_t>(iteration) * (levels + 1) + level];
  }
};

struct PtReport {
  Schedule schedule;
  int iterations = 0;
  int burn_in = 0;
  double log_z_hat = 0.0;
  PotentialTrace trace;
  std::vector<std::uint8_t> swap_accepted;
  std::vector<std::uint64_t> swap_attempts;
  std::vector<std::uint64_t> swap_accepts;
  std::uint64_t kernel_applications = 0;
  double wall_seconds = 0.0;
};

PtReport run_pt(const AnnealedTarget& target, const Kernel& kernel, const Schedule& schedule,
                const PtOptions& options);
// new: `replicas` independent runs (seeds seed + r) in one device launch
std::vector<PtReport> run_pt_replicas(const AnnealedTarget& target, const Kernel& kernel,
                                      const Schedule& schedule, const PtOptions& options, int replicas);
double stepping_stone(const PotentialTrace& trace, const Schedule& schedule, int burn_in);

struct SaisMemoryProfile {
  std::size_t moment_accumulators = 0;
  std::size_t signed_accumulators = 0;
  std::size_t wave_block_slots = 0;
};
SaisMemoryProfile sais_memory_profile(int total_steps, int workers, std::size_t chunk);

int device_count();

// ---- theory.hpp (closed-form variance model, host scalar math) ------------
namespace theory {
double rel_variance(double d_total, double r_eff, double n_particles);
double log1p_rel_variance(double d_total, double r_eff, double n_particles);
double solve_r_eff(double d_total, double n_particles, double observed_rel_var);
struct ParticleBounds {
  double n_min = 0.0;
  double n_max = 0.0;
};
ParticleBounds particle_bounds(double lambda, double kappa, double r_eff, double t_steps,
                               double eps);
enum class Regime { coarse, stable, dense };
Regime classify_regime(double alpha_r, double alpha_t);
std::string regime_name(Regime regime);
struct REffBounds {
  double lower = 1.0;
  double upper = 1.0;
};
REffBounds stabilized_r_eff_bounds(double lambda, double kappa, double t_steps, double rho);
}  // namespace theory

}  // namespace asmc
