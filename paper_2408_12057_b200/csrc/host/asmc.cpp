// Host C++ mirror of the reference API over the C-ABI (see asmc.hpp).
// Per-point target evaluations and scalar helpers (discrepancy_hat, cess,
// decide_resample, theory) are host arithmetic, as in the reference; every
// sampler, reduction, resampling and schedule inversion call goes to the GPU.
#include "asmc.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

namespace asmc {

namespace {

constexpr double kLogSqrt2Pi = 0.91893853320467274178;

// Rethrow a C-ABI error as the reference's exception class.
void check(int rc) {
  if (rc == ASMC_OK) return;
  const std::string msg = asmc_last_error();
  switch (rc) {
    case ASMC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ASMC_ERR_DOMAIN: throw std::domain_error(msg);
    case ASMC_ERR_CAPABILITY: throw capability_error(msg);
    case ASMC_ERR_DEGENERATE: throw degenerate_weights_error(msg);
    case ASMC_ERR_EVALUATION: throw evaluation_error(msg);
    default: throw device_error(msg);
  }
}

asmc_target_desc descriptor(const AnnealedTarget& t) {
  asmc_target_desc d;
  std::memset(&d, 0, sizeof d);
  if (!t.device_descriptor(&d))
    throw capability_error("target has no B200 device implementation (no CPU fallback)");
  return d;
}

asmc_kernel_desc kernel_desc(const Kernel& k) {
  asmc_kernel_desc d;
  std::memset(&d, 0, sizeof d);
  d.kind = static_cast<int32_t>(k.kind);
  if (k.step_sizes.size() > ASMC_MAX_STEP_SIZES)
    throw capability_error("at most 16 rwmh step sizes are supported on the device");
  d.n_step_sizes = static_cast<int32_t>(k.step_sizes.size());
  d.sweeps = k.sweeps;
  d.leapfrog = k.leapfrog;
  for (std::size_t i = 0; i < k.step_sizes.size(); ++i) d.step_sizes[i] = k.step_sizes[i];
  return d;
}

asmc_exec exec_of(Rng rng, Precision p, int device, int lanes) {
  asmc_exec e;
  std::memset(&e, 0, sizeof e);
  e.rng = static_cast<int32_t>(rng);
  e.precision = static_cast<int32_t>(p);
  e.device = device;
  e.lanes = lanes;
  return e;
}

struct ReportBufs {
  std::vector<double> g0, g1, g2, ess, cz;
  std::vector<std::uint8_t> rs;
  std::vector<int32_t> rt;
  asmc_report rep;
  explicit ReportBufs(int T)
      : g0(T + 1, kNegInf), g1(T + 1, kNegInf), g2(T + 1, kNegInf), ess(T + 1), cz(T + 1),
        rs(T + 1), rt(T + 1) {
    std::memset(&rep, 0, sizeof rep);
    rep.log_g0 = g0.data();
    rep.log_g1 = g1.data();
    rep.log_g2 = g2.data();
    rep.ess_trace = ess.data();
    rep.cum_log_z = cz.data();
    rep.resampled = rs.data();
    rep.resample_times = rt.data();
  }
  RunReport to_report(const Schedule& s, std::size_t n, bool smc) const {
    RunReport r;
    r.schedule = s;
    r.n_particles = n;
    r.log_z_hat = rep.log_z_hat;
    r.elbo_hat = rep.elbo_hat;
    r.stats.log_g0 = g0;
    r.stats.log_g1 = g1;
    r.stats.log_g2 = g2;
    r.resample_times.assign(rt.begin(), rt.begin() + rep.n_resample_times);
    if (smc) r.ess_trace = ess;
    r.cum_log_z = cz;
    r.resampled = rs;
    r.kernel_applications = rep.kernel_applications;
    r.wall_seconds = rep.wall_seconds;
    return r;
  }
};

}  // namespace

// ---- targets (target.cpp) -------------------------------------------------
double log_normal_pdf(double x, double mu, double sigma) {
  const double s = (x - mu) / sigma;
  return -0.5 * s * s - std::log(sigma) - kLogSqrt2Pi;
}

void AnnealedTarget::check_point(std::span<const double> x) const {
  if (x.size() != dim())
    throw std::invalid_argument("point has dimension " + std::to_string(x.size()) +
                                ", target has dimension " + std::to_string(dim()));
}

void AnnealedTarget::check_beta(double beta) {
  if (!(beta >= 0.0 && beta <= 1.0))
    throw std::domain_error("beta must lie in [0, 1], got " + std::to_string(beta));
}

double AnnealedTarget::log_gamma(double beta, std::span<const double> x) const {
  check_beta(beta);
  check_point(x);
  const double lr = log_reference(x);
  return beta == 0.0 ? lr : lr + beta * potential(x);
}

void AnnealedTarget::exact_sample(double, rng::Stream&, std::span<double>) const {
  throw capability_error("target does not provide an exact sampler");
}

double AnnealedTarget::analytic_log_z(double) const {
  throw capability_error("target does not provide analytic_log_z");
}
double AnnealedTarget::analytic_delta(double) const {
  throw capability_error("target does not provide analytic_delta");
}
double AnnealedTarget::analytic_discrepancy(double, double) const {
  throw capability_error("target does not provide analytic_discrepancy");
}

GaussianShiftTarget::GaussianShiftTarget(double mu0, double mu1, double sigma, std::size_t dim)
    : mu0_(mu0), mu1_(mu1), sigma_(sigma), dim_(dim) {
  if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
  if (dim == 0) throw std::invalid_argument("dim must be at least 1");
  z_ = std::abs(mu1 - mu0) / sigma;
}
double GaussianShiftTarget::log_reference(std::span<const double> x) const {
  double s = 0.0;
  for (double v : x) s += log_normal_pdf(v, mu0_, sigma_);
  return s;
}
double GaussianShiftTarget::potential(std::span<const double> x) const {
  const double a = (mu1_ - mu0_) / (sigma_ * sigma_), mid = 0.5 * (mu0_ + mu1_);
  double s = 0.0;
  for (double v : x) s += a * (v - mid);
  return s;
}
double GaussianShiftTarget::analytic_log_z(double beta) const {
  check_beta(beta);
  return static_cast<double>(dim_) * (-0.5 * beta * (1.0 - beta) * z_ * z_);
}
double GaussianShiftTarget::analytic_delta(double beta) const {
  check_beta(beta);
  return static_cast<double>(dim_) * z_ * z_;
}
double GaussianShiftTarget::analytic_discrepancy(double beta, double beta2) const {
  check_beta(beta);
  check_beta(beta2);
  if (beta2 < beta) throw std::domain_error("analytic_discrepancy requires beta2 >= beta");
  if (2.0 * beta2 - beta > 1.0 + 1e-15)
    throw std::domain_error("analytic_discrepancy undefined for 2*beta2 - beta > 1");
  const double db = beta2 - beta;
  return static_cast<double>(dim_) * z_ * z_ * db * db;
}
void GaussianShiftTarget::sample_reference(rng::Stream& stream, std::span<double> out) const {
  check_point(out);
  for (double& v : out) v = mu0_ + sigma_ * stream.normal();
}
void GaussianShiftTarget::exact_sample(double beta, rng::Stream& stream, std::span<double> out) const {
  check_beta(beta);
  check_point(out);
  const double mu = (1.0 - beta) * mu0_ + beta * mu1_;
  for (double& v : out) v = mu + sigma_ * stream.normal();
}
bool GaussianShiftTarget::device_descriptor(asmc_target_desc* o) const {
  o->kind = ASMC_TARGET_GAUSSIAN_SHIFT;
  o->dim = dim_;
  o->p[0] = mu0_;
  o->p[1] = mu1_;
  o->p[2] = sigma_;
  return true;
}

MixtureTarget::MixtureTarget(double ref_sigma, double weight, double mu1, double sigma1,
                             double mu2, double sigma2, std::size_t dim)
    : ref_sigma_(ref_sigma), weight_(weight), mu1_(mu1), sigma1_(sigma1), mu2_(mu2),
      sigma2_(sigma2), dim_(dim) {
  if (!(ref_sigma > 0.0 && sigma1 > 0.0 && sigma2 > 0.0))
    throw std::invalid_argument("mixture sigmas must be positive");
  if (!(weight > 0.0 && weight < 1.0))
    throw std::invalid_argument("mixture weight must lie strictly in (0, 1)");
  if (dim == 0) throw std::invalid_argument("dim must be at least 1");
}
double MixtureTarget::log_reference(std::span<const double> x) const {
  double s = 0.0;
  for (double v : x) s += log_normal_pdf(v, 0.0, ref_sigma_);
  return s;
}
double MixtureTarget::potential(std::span<const double> x) const {
  const double l1 = std::log(weight_), l2 = std::log1p(-weight_);
  double s = 0.0;
  for (double v : x) {
    const double a = l1 + log_normal_pdf(v, mu1_, sigma1_);
    const double b = l2 + log_normal_pdf(v, mu2_, sigma2_);
    const double hi = std::max(a, b), lo = std::min(a, b);
    s += hi + std::log1p(std::exp(lo - hi)) - log_normal_pdf(v, 0.0, ref_sigma_);
  }
  return s;
}
void MixtureTarget::sample_reference(rng::Stream& stream, std::span<double> out) const {
  check_point(out);
  for (double& v : out) v = ref_sigma_ * stream.normal();
}
bool MixtureTarget::device_descriptor(asmc_target_desc* o) const {
  o->kind = ASMC_TARGET_MIXTURE;
  o->dim = dim_;
  const double p[6] = {ref_sigma_, weight_, mu1_, sigma1_, mu2_, sigma2_};
  for (int i = 0; i < 6; ++i) o->p[i] = p[i];
  return true;
}

ScaleGaussianTarget::ScaleGaussianTarget(double s0, double s1, std::size_t dim)
    : s0_(s0), s1_(s1), dim_(dim) {
  if (!(s0 > 0.0 && s1 > 0.0)) throw std::invalid_argument("scale sigmas must be positive");
  if (dim == 0) throw std::invalid_argument("dim must be at least 1");
}
double ScaleGaussianTarget::tau(double beta) const {
  return (1.0 - beta) / (s0_ * s0_) + beta / (s1_ * s1_);
}
double ScaleGaussianTarget::log_reference(std::span<const double> x) const {
  double s = 0.0;
  for (double v : x) s += log_normal_pdf(v, 0.0, s0_);
  return s;
}
double ScaleGaussianTarget::potential(std::span<const double> x) const {
  double s = 0.0;
  for (double v : x) s += log_normal_pdf(v, 0.0, s1_) - log_normal_pdf(v, 0.0, s0_);
  return s;
}
double ScaleGaussianTarget::analytic_log_z(double beta) const {
  check_beta(beta);
  return static_cast<double>(dim_) *
         (-(1.0 - beta) * std::log(s0_) - beta * std::log(s1_) - 0.5 * std::log(tau(beta)));
}
double ScaleGaussianTarget::analytic_delta(double beta) const {
  check_beta(beta);
  const double c = 0.5 / (s0_ * s0_) - 0.5 / (s1_ * s1_), t = tau(beta);
  return static_cast<double>(dim_) * 2.0 * c * c / (t * t);
}
double ScaleGaussianTarget::analytic_discrepancy(double beta, double beta2) const {
  check_beta(beta);
  check_beta(beta2);
  if (beta2 < beta) throw std::domain_error("analytic_discrepancy requires beta2 >= beta");
  const double b3 = 2.0 * beta2 - beta;
  if (b3 > 1.0 + 1e-15)
    throw std::domain_error("analytic_discrepancy undefined for 2*beta2 - beta > 1");
  return analytic_log_z(std::min(1.0, b3)) + analytic_log_z(beta) - 2.0 * analytic_log_z(beta2);
}
void ScaleGaussianTarget::sample_reference(rng::Stream& stream, std::span<double> out) const {
  check_point(out);
  for (double& v : out) v = s0_ * stream.normal();
}
void ScaleGaussianTarget::exact_sample(double beta, rng::Stream& stream, std::span<double> out) const {
  check_beta(beta);
  check_point(out);
  const double sd = 1.0 / std::sqrt(tau(beta));  // pi_beta = N(0, I / tau_beta)
  for (double& v : out) v = sd * stream.normal();
}
bool ScaleGaussianTarget::device_descriptor(asmc_target_desc* o) const {
  o->kind = ASMC_TARGET_SCALE_GAUSSIAN;
  o->dim = dim_;
  o->p[0] = s0_;
  o->p[1] = s1_;
  return true;
}

LogisticTarget::LogisticTarget(std::vector<float> X, std::vector<float> y, std::size_t dim, double sp)
    : y_(std::move(y)), dim_(dim), sp_(sp) {
  if (!(sp > 0.0)) throw std::invalid_argument("prior sigma must be positive");
  if (dim == 0 || y_.empty() || X.size() != y_.size() * dim)
    throw std::invalid_argument("logistic target needs X (n x dim) and y (n)");
  data_ = std::move(X);
  data_.insert(data_.end(), y_.begin(), y_.end());
}
double LogisticTarget::log_reference(std::span<const double> x) const {
  double s = 0.0;
  for (double v : x) s += log_normal_pdf(v, 0.0, sp_);
  return s;
}
double LogisticTarget::potential(std::span<const double> th) const {
  double acc = 0.0;
  for (std::size_t j = 0; j < y_.size(); ++j) {
    double l = 0.0;
    for (std::size_t i = 0; i < dim_; ++i) l += static_cast<double>(data_[j * dim_ + i]) * th[i];
    acc += y_[j] * l - (l > 0.0 ? l + std::log1p(std::exp(-l)) : std::log1p(std::exp(l)));
  }
  return acc;
}
void LogisticTarget::sample_reference(rng::Stream& stream, std::span<double> out) const {
  check_point(out);
  for (double& v : out) v = sp_ * stream.normal();
}
bool LogisticTarget::device_descriptor(asmc_target_desc* o) const {
  o->kind = ASMC_TARGET_LOGISTIC;
  o->dim = dim_;
  o->p[0] = sp_;
  o->p[1] = static_cast<double>(y_.size());
  o->data = data_.data();
  o->data_bytes = data_.size() * sizeof(float);
  return true;
}

IsingTarget::IsingTarget(int side, double coupling, double delta, double sigma)
    : L_(side), K_(coupling), delta_(delta), sigma_(sigma) {
  if (side < 3) throw std::invalid_argument("ising target needs an integer side L >= 3");
  if (!(coupling >= 0.0)) throw std::invalid_argument("ising coupling must be non-negative");
  if (!(delta > 0.0)) throw std::invalid_argument("ising relaxation delta must be positive");
  if (!(sigma > 0.0)) throw std::invalid_argument("reference sigma must be positive");
}
double IsingTarget::log_reference(std::span<const double> x) const {
  check_point(x);
  double s = 0.0;
  for (double v : x) s += log_normal_pdf(v, 0.0, sigma_);
  return s;
}
double IsingTarget::potential(std::span<const double> y) const {
  check_point(y);
  const double c = delta_ + 4.0 * K_;
  double acc = 0.0;
  for (int a = 0; a < L_; ++a)
    for (int b = 0; b < L_; ++b) {
      const double nb = (y[((a + L_ - 1) % L_) * L_ + b] + y[((a + 1) % L_) * L_ + b]) +
                        (y[a * L_ + (b + L_ - 1) % L_] + y[a * L_ + (b + 1) % L_]);
      const double yi = y[a * L_ + b], u = c * yi + K_ * nb, au = std::fabs(u);
      acc += -0.5 * yi * u + (au + std::log1p(std::exp(-2.0 * au))) - log_normal_pdf(yi, 0.0, sigma_);
    }
  return acc;
}
void IsingTarget::sample_reference(rng::Stream& stream, std::span<double> out) const {
  check_point(out);
  for (double& v : out) v = sigma_ * stream.normal();
}
bool IsingTarget::device_descriptor(asmc_target_desc* o) const {
  o->kind = ASMC_TARGET_ISING;
  o->dim = dim();
  o->p[0] = L_;
  o->p[1] = K_;
  o->p[2] = delta_;
  o->p[3] = sigma_;
  return true;
}

// ---- kernel / engine ------------------------------------------------------
void validate_kernel(const Kernel& k) {  // kernel.cpp:12-22
  if (k.kind == KernelKind::slice && k.sweeps < 1) throw std::invalid_argument("slice sweeps must be at least 1");
  if (k.kind == KernelKind::hmc) {
    if (k.step_sizes.empty()) throw std::invalid_argument("hmc requires at least one step size");
    for (double s : k.step_sizes)
      if (!(s > 0.0)) throw std::invalid_argument("hmc step sizes must be positive");
    if (k.sweeps < 1) throw std::invalid_argument("hmc sweeps must be at least 1");
    if (k.leapfrog < 1) throw std::invalid_argument("hmc leapfrog steps must be at least 1");
  }
  if (k.kind == KernelKind::rwmh_cycle) {
    if (k.step_sizes.empty()) throw std::invalid_argument("rwmh_cycle requires at least one step size");
    for (double s : k.step_sizes)
      if (!(s > 0.0)) throw std::invalid_argument("rwmh step sizes must be positive");
    if (k.sweeps < 1) throw std::invalid_argument("rwmh sweeps must be at least 1");
  }
}

Schedule Schedule::uniform(int steps) {  // engine.cpp:16-27
  if (steps < 1) throw std::invalid_argument("schedule needs at least one step");
  Schedule s;
  s.betas.resize(steps + 1);
  for (int t = 0; t <= steps; ++t) s.betas[t] = static_cast<double>(t) / static_cast<double>(steps);
  s.betas[0] = 0.0;
  s.betas[steps] = 1.0;
  return s;
}

void Schedule::validate() const {  // engine.cpp:29-39
  if (betas.size() < 2) throw std::invalid_argument("schedule needs at least one step");
  if (betas.front() != 0.0) throw std::invalid_argument("schedule must start at beta = 0");
  if (betas.back() != 1.0) throw std::invalid_argument("schedule must end at beta = 1");
  for (std::size_t t = 1; t < betas.size(); ++t)
    if (!(betas[t] > betas[t - 1]))
      throw std::invalid_argument("schedule must be strictly increasing at index " + std::to_string(t));
}

void RunOptions::validate() const {
  if (n_particles < 1) throw std::invalid_argument("n_particles must be at least 1");
  if (workers < 1) throw std::invalid_argument("workers must be at least 1");
  if (!(rho >= 0.0 && rho <= 1.0)) throw std::invalid_argument("rho must lie in [0, 1]");
}

double ess(std::span<const double> lw) {
  if (lw.empty()) throw std::invalid_argument("ess of empty weight vector");
  double out = 0.0;
  check(asmc_ess(lw.data(), lw.size(), 0, &out));
  return out;
}

std::vector<std::uint32_t> systematic_resample(std::span<const double> lw, rng::Stream& stream) {
  if (lw.empty()) throw std::invalid_argument("cannot resample an empty system");
  return systematic_resample(lw, stream.uniform(), 0);  // engine.cpp:67: one uniform per call
}

std::vector<std::uint32_t> systematic_resample(std::span<const double> lw, double u, int device) {
  std::vector<std::uint32_t> a(lw.size());
  check(asmc_systematic_resample(lw.data(), lw.size(), u, device, a.data()));
  return a;
}

bool decide_resample(ResamplePolicy policy, int t, int total_steps, double ess_value,
                     std::size_t n, double acc_dhat, double rho) {  // engine.cpp:82-95
  switch (policy) {
    case ResamplePolicy::never: return t == total_steps;
    case ResamplePolicy::always: return true;
    case ResamplePolicy::adaptive_ess: return ess_value < rho * static_cast<double>(n);
    case ResamplePolicy::stabilized: return acc_dhat > -std::log(rho);
  }
  throw std::invalid_argument("unknown resampling policy");
}

RunReport run_smc(const AnnealedTarget& target, const Kernel& kernel, const Schedule& schedule,
                  const RunOptions& o) {
  schedule.validate();
  o.validate();
  validate_kernel(kernel);
  const asmc_target_desc td = descriptor(target);
  const asmc_kernel_desc kd = kernel_desc(kernel);
  const asmc_exec ex = exec_of(o.rng, o.precision, o.device, o.lanes);
  ReportBufs b(schedule.steps());
  check(asmc_run_smc(&td, &kd, schedule.betas.data(), schedule.steps(), o.n_particles,
                     static_cast<int32_t>(o.policy), o.rho, o.seed, o.round, &ex, &b.rep));
  return b.to_report(schedule, o.n_particles, true);
}

RunReport run_sais_single(const AnnealedTarget& target, const Kernel& kernel,
                          const Schedule& schedule, const RunOptions& o, std::size_t) {
  schedule.validate();
  o.validate();
  validate_kernel(kernel);
  const asmc_target_desc td = descriptor(target);
  const asmc_kernel_desc kd = kernel_desc(kernel);
  const asmc_exec ex = exec_of(o.rng, o.precision, o.device, o.lanes);
  ReportBufs b(schedule.steps());
  check(asmc_run_sais_single(&td, &kd, schedule.betas.data(), schedule.steps(), o.n_particles,
                             o.seed, o.round, &ex, &b.rep));
  return b.to_report(schedule, o.n_particles, false);
}

// ---- schedule -------------------------------------------------------------
namespace {
void check_step_index(const IncrementStats& s, int t) {  // schedule.cpp:14-24
  if (t < 1 || t > s.steps())
    throw std::invalid_argument("step index " + std::to_string(t) + " out of range");
  if (s.log_g0[t] == kNegInf)
    throw std::invalid_argument("no increment statistics recorded for step " + std::to_string(t));
}
}  // namespace

double discrepancy_hat(const IncrementStats& s, int t) {
  check_step_index(s, t);
  const double raw = s.log_g2[t] - 2.0 * s.log_g1[t] + s.log_g0[t];
  return raw > 0.0 ? raw : 0.0;
}

double cess(const IncrementStats& s, int t, std::size_t n_particles) {
  check_step_index(s, t);
  const double raw = s.log_g2[t] - 2.0 * s.log_g1[t] + s.log_g0[t];
  const double n = static_cast<double>(n_particles);
  return std::min(n, std::max(1.0, n * std::exp(-raw)));
}

BarrierEstimate barrier_estimate(const IncrementStats& stats, const Schedule& schedule) {
  schedule.validate();
  const int T = schedule.steps();
  if (stats.steps() != T)
    throw std::invalid_argument("statistics cover " + std::to_string(stats.steps()) +
                                " steps, schedule has " + std::to_string(T));
  BarrierEstimate e;
  e.lambda.assign(T + 1, 0.0);
  e.beta = schedule.betas;
  check(asmc_barrier_estimate(stats.log_g0.data(), stats.log_g1.data(), stats.log_g2.data(),
                              schedule.betas.data(), T, 0, e.lambda.data()));
  return e;
}

Schedule generate_schedule(const BarrierEstimate& est, int t_new) {
  if (est.lambda.size() != est.beta.size())
    throw std::invalid_argument("barrier estimate needs at least two matched knots");
  Schedule s;
  s.betas.assign(std::max(t_new, 0) + 1, 0.0);
  check(asmc_generate_schedule(est.lambda.data(), est.beta.data(),
                               static_cast<int32_t>(est.lambda.size()), t_new, 0, s.betas.data()));
  return s;
}

std::vector<double> local_barrier(const BarrierEstimate& est) {
  if (est.lambda.size() != est.beta.size())
    throw std::invalid_argument("barrier estimate needs at least two matched knots");
  std::vector<double> out(est.beta.size());
  check(asmc_local_barrier(est.lambda.data(), est.beta.data(),
                           static_cast<int32_t>(est.lambda.size()), 0, out.data()));
  return out;
}

// ---- drivers --------------------------------------------------------------
BudgetPlan budget(std::size_t n, int steps, std::size_t dim, std::uint64_t cap, DriverMode mode) {
  uint64_t nn = 0;
  int32_t tt = 0;
  check(asmc_budget(n, steps, dim, cap, mode == DriverMode::sais ? ASMC_MODE_SAIS : ASMC_MODE_SSMC,
                    &nn, &tt));
  return BudgetPlan{static_cast<std::size_t>(nn), tt};
}

void DriverOptions::validate() const {  // drivers.cpp:16-21
  if (n_particles < 1) throw std::invalid_argument("n_particles must be at least 1");
  if (rounds < 1) throw std::invalid_argument("rounds must be at least 1");
  if (workers < 1) throw std::invalid_argument("workers must be at least 1");
  if (!(rho >= 0.0 && rho <= 1.0)) throw std::invalid_argument("rho must lie in [0, 1]");
}

namespace {
std::vector<RoundResult> round_loop(const AnnealedTarget& target, const Kernel& kernel,
                                    const DriverOptions& o, DriverMode mode) {
  o.validate();
  validate_kernel(kernel);
  const asmc_target_desc td = descriptor(target);
  const asmc_kernel_desc kd = kernel_desc(kernel);
  const asmc_exec ex = exec_of(o.rng, o.precision, o.device, o.lanes);
  const int32_t m = mode == DriverMode::sais ? ASMC_MODE_SAIS : ASMC_MODE_SSMC;
  // the (N_k, T_k) plan is the budget rule alone
  int tmax = 1, t = 1;
  std::size_t n = o.n_particles;
  for (int k = 1; k < o.rounds; ++k) {
    const BudgetPlan p = budget(n, t, target.dim(), o.memory_cap_bytes, mode);
    n = p.n_particles;
    t = p.steps;
    tmax = std::max(tmax, t);
  }
  const int R = o.rounds, S = tmax + 1;
  std::vector<uint64_t> ns(R), ka(R);
  std::vector<int32_t> ts(R);
  std::vector<double> betas(R * S), g0(R * S), g1(R * S), g2(R * S), es(R * S), cz(R * S), lam(R * S),
      lz(R), el(R), wall(R);
  std::vector<uint8_t> rs(R * S);
  asmc_rounds_out out;
  std::memset(&out, 0, sizeof out);
  out.max_steps = tmax;
  out.n_particles = ns.data();
  out.steps = ts.data();
  out.betas = betas.data();
  out.log_g0 = g0.data();
  out.log_g1 = g1.data();
  out.log_g2 = g2.data();
  out.ess_trace = es.data();
  out.cum_log_z = cz.data();
  out.resampled = rs.data();
  out.lambda = lam.data();
  out.log_z_hat = lz.data();
  out.elbo_hat = el.data();
  out.wall_seconds = wall.data();
  out.kernel_applications = ka.data();
  check(asmc_run_rounds(&td, &kd, m, o.n_particles, R, static_cast<int32_t>(o.policy), o.rho, o.seed,
                        o.memory_cap_bytes, &ex, &out));
  std::vector<RoundResult> res;
  res.reserve(R);
  for (int k = 0; k < R; ++k) {
    const int T = ts[k];
    const std::size_t r0 = static_cast<std::size_t>(k) * S;
    RoundResult rr;
    rr.round = k + 1;
    RunReport& rep = rr.report;
    rep.schedule.betas.assign(betas.begin() + r0, betas.begin() + r0 + T + 1);
    rep.n_particles = ns[k];
    rep.log_z_hat = lz[k];
    rep.elbo_hat = el[k];
    rep.stats.log_g0.assign(g0.begin() + r0, g0.begin() + r0 + T + 1);
    rep.stats.log_g1.assign(g1.begin() + r0, g1.begin() + r0 + T + 1);
    rep.stats.log_g2.assign(g2.begin() + r0, g2.begin() + r0 + T + 1);
    if (mode == DriverMode::ssmc) rep.ess_trace.assign(es.begin() + r0, es.begin() + r0 + T + 1);
    rep.cum_log_z.assign(cz.begin() + r0, cz.begin() + r0 + T + 1);
    rep.resampled.assign(rs.begin() + r0, rs.begin() + r0 + T + 1);
    for (int i = 1; i <= T; ++i)
      if (i == T || (mode == DriverMode::ssmc && rep.resampled[i]))
        rep.resample_times.push_back(i);
    rep.kernel_applications = ka[k];
    rep.wall_seconds = wall[k];
    rr.barrier.lambda.assign(lam.begin() + r0, lam.begin() + r0 + T + 1);
    rr.barrier.beta = rep.schedule.betas;
    res.push_back(std::move(rr));
  }
  return res;
}
}  // namespace

std::vector<RoundResult> run_ssmc(const AnnealedTarget& t, const Kernel& k, const DriverOptions& o) {
  return round_loop(t, k, o, DriverMode::ssmc);
}
std::vector<RoundResult> run_sais(const AnnealedTarget& t, const Kernel& k, const DriverOptions& o) {
  return round_loop(t, k, o, DriverMode::sais);
}

void ZjaOptions::validate() const {  // drivers.cpp:23-31
  if (n_particles < 1) throw std::invalid_argument("n_particles must be at least 1");
  if (target_steps < 1) throw std::invalid_argument("target_steps must be at least 1");
  if (workers < 1) throw std::invalid_argument("workers must be at least 1");
  if (max_steps < 1) throw std::invalid_argument("max_steps must be at least 1");
  if (!(delta_star >= 0.0) || !std::isfinite(delta_star))
    throw std::invalid_argument("delta_star must be finite and >= 0");
}

ZjaResult zja_next_beta(const AnnealedTarget& target, double beta, std::span<const double> positions,
                        std::size_t n, std::span<const double> log_weights, double delta_star, double tol) {
  if (n == 0 || log_weights.size() != n || positions.size() != n * target.dim())
    throw std::invalid_argument("particle arrays inconsistent with n_particles");
  const asmc_target_desc td = descriptor(target);
  const asmc_exec ex = exec_of(Rng::xoshiro, Precision::fp64, 0, 0);
  ZjaResult r;
  int32_t w = 0;
  check(asmc_zja_next_beta(&td, beta, positions.data(), n, log_weights.data(), delta_star, tol, &ex,
                           &r.beta_next, &w));
  r.warning = w != 0;
  return r;
}

ZjaOutcome run_zja(const AnnealedTarget& target, const Kernel& kernel, const ZjaOptions& o) {
  o.validate();
  validate_kernel(kernel);
  const asmc_target_desc td = descriptor(target);
  const asmc_kernel_desc kd = kernel_desc(kernel);
  const asmc_exec ex = exec_of(o.rng, o.precision, o.device, o.lanes);
  asmc_zja_opts zo{o.n_particles, o.target_steps, o.max_steps, o.delta_star, o.seed};
  ReportBufs main(o.max_steps), pilot(o.target_steps);
  std::vector<double> betas(o.max_steps + 1), lam(o.max_steps + 1), plam(o.target_steps + 1);
  asmc_zja_out out;
  std::memset(&out, 0, sizeof out);
  out.capacity = o.max_steps + 1;
  out.betas = betas.data();
  out.lambda = lam.data();
  out.main = main.rep;
  out.pilot_lambda = plam.data();
  out.pilot = pilot.rep;
  check(asmc_run_zja(&td, &kd, &zo, &ex, &out));
  ZjaOutcome res;
  res.delta_star = out.delta_star;
  res.warning = out.warning != 0;
  if (out.pilot_ran) {
    pilot.rep = out.pilot;
    RoundResult rr;
    rr.round = 1;
    rr.report = pilot.to_report(Schedule::uniform(o.target_steps), o.n_particles, false);
    rr.barrier.lambda = plam;
    rr.barrier.beta = rr.report.schedule.betas;
    res.rounds.push_back(std::move(rr));
  }
  const int T = out.steps;
  main.rep = out.main;
  Schedule s;
  s.betas.assign(betas.begin(), betas.begin() + T + 1);
  RoundResult rr;
  rr.round = out.pilot_ran ? 2 : 1;
  rr.report = main.to_report(s, o.n_particles, true);
  auto cut = [T](auto& v) { v.resize(T + 1); };
  cut(rr.report.stats.log_g0);
  cut(rr.report.stats.log_g1);
  cut(rr.report.stats.log_g2);
  cut(rr.report.ess_trace);
  cut(rr.report.cum_log_z);
  cut(rr.report.resampled);
  rr.barrier.lambda.assign(lam.begin(), lam.begin() + T + 1);
  rr.barrier.beta = s.betas;
  res.rounds.push_back(std::move(rr));
  return res;
}

void PtOptions::validate() const {  // pt.cpp:14-19
  if (iterations < 1) throw std::invalid_argument("iterations must be at least 1");
  if (burn_in >= iterations) throw std::invalid_argument("burn_in must leave at least one recorded iteration");
}

std::vector<PtReport> run_pt_replicas(const AnnealedTarget& target, const Kernel& kernel, const Schedule& schedule,
                                      const PtOptions& o, int replicas) {
  schedule.validate();
  o.validate();
  validate_kernel(kernel);
  if (replicas < 1) throw std::invalid_argument("replicas must be at least 1");
  const asmc_target_desc td = descriptor(target);
  const asmc_kernel_desc kd = kernel_desc(kernel);
  const asmc_exec ex = exec_of(o.rng, o.precision, o.device, 0);
  const int L = schedule.steps(), I = o.iterations;
  const std::size_t rows = static_cast<std::size_t>(replicas) * I * (L + 1);
  std::vector<double> lz(replicas), tr(rows);
  std::vector<std::uint8_t> ac(rows);
  std::vector<std::uint64_t> att(static_cast<std::size_t>(replicas) * (L + 1)), acc(att.size());
  asmc_pt_opts po{I, o.burn_in, o.seed, o.round, replicas, 0};
  asmc_pt_out out{lz.data(), tr.data(), ac.data(), att.data(), acc.data(), 0, 0.0, 0, 0};
  check(asmc_run_pt(&td, &kd, schedule.betas.data(), L, &po, &ex, &out));
  std::vector<PtReport> res(replicas);
  const std::size_t per = static_cast<std::size_t>(I) * (L + 1);
  for (int r = 0; r < replicas; ++r) {
    PtReport& p = res[r];
    p.schedule = schedule;
    p.iterations = I;
    p.burn_in = out.burn_in;
    p.log_z_hat = lz[r];
    p.trace.iterations = I;
    p.trace.levels = L;
    p.trace.values.assign(tr.begin() + r * per, tr.begin() + (r + 1) * per);
    p.swap_accepted.assign(ac.begin() + r * per, ac.begin() + (r + 1) * per);
    p.swap_attempts.assign(att.begin() + r * (L + 1), att.begin() + (r + 1) * (L + 1));
    p.swap_accepts.assign(acc.begin() + r * (L + 1), acc.begin() + (r + 1) * (L + 1));
    p.kernel_applications = out.kernel_applications;
    p.wall_seconds = out.wall_seconds;
  }
  return res;
}

PtReport run_pt(const AnnealedTarget& target, const Kernel& kernel, const Schedule& schedule, const PtOptions& o) {
  return run_pt_replicas(target, kernel, schedule, o, 1)[0];
}

double stepping_stone(const PotentialTrace& trace, const Schedule& schedule, int burn_in) {  // pt.cpp:130-152
  schedule.validate();
  const int levels = schedule.steps();
  if (trace.levels != levels) throw std::invalid_argument("trace level count does not match schedule");
  if (burn_in < 0 || burn_in >= trace.iterations)
    throw std::invalid_argument("burn_in must leave at least one recorded iteration");
  const double log_used = std::log(static_cast<double>(trace.iterations - burn_in));
  double log_z = 0.0;
  for (int n = 1; n <= levels; ++n) {
    const double delta_beta = schedule.betas[n] - schedule.betas[n - 1];
    double mx = kNegInf, sum = 0.0;  // LogAccumulator (logsum.hpp:18-49)
    for (int it = burn_in; it < trace.iterations; ++it) {
      const double l = delta_beta * trace.at(it, n - 1);
      if (l == kNegInf) continue;
      if (l <= mx) {
        sum += std::exp(l - mx);
      } else {
        sum = sum * std::exp(mx - l) + 1.0;
        mx = l;
      }
    }
    log_z += (mx == kNegInf ? kNegInf : mx + std::log(sum)) - log_used;
  }
  return log_z;
}

SaisMemoryProfile sais_memory_profile(int total_steps, int workers, std::size_t chunk) {
  // drivers.cpp:59-70 semantics: adaptation storage 3(T+1) + (T+1), never N
  if (total_steps < 1) throw std::invalid_argument("profile needs at least one step");
  if (workers < 1) throw std::invalid_argument("workers must be at least 1");
  const std::size_t cp = chunk > 0 ? chunk : static_cast<std::size_t>(workers) * 8;
  SaisMemoryProfile p;
  p.moment_accumulators = 3 * (static_cast<std::size_t>(total_steps) + 1);
  p.signed_accumulators = static_cast<std::size_t>(total_steps) + 1;
  p.wave_block_slots = std::max((cp - 1) / 256 + 1, static_cast<std::size_t>(workers));
  return p;
}

int device_count() { return asmc_device_count(); }

// ---- theory: restatement of the closed-form model (theory.cpp) -----------
namespace theory {
namespace {
void require(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(std::string("theory: ") + what);
}
}  // namespace

double log1p_rel_variance(double d, double r, double n) {
  require(d >= 0.0 && std::isfinite(d), "d_total must be finite and >= 0");
  require(n >= 1.0 && std::isfinite(n), "n_particles must be finite and >= 1");
  require(r >= 1.0 && std::isfinite(r), "r_eff must be finite and >= 1");
  return r * std::log1p(std::expm1(d / r) / n);
}

double rel_variance(double d, double r, double n) { return std::expm1(log1p_rel_variance(d, r, n)); }

double solve_r_eff(double d, double n, double observed) {
  require(d >= 0.0 && std::isfinite(d), "d_total must be finite and >= 0");
  require(n >= 1.0 && std::isfinite(n), "n_particles must be finite and >= 1");
  require(observed > 0.0 && std::isfinite(observed), "observed_rel_var must be finite and > 0");
  require(d != 0.0, "r_eff is unidentified at d_total = 0");
  const double goal = std::log1p(observed);
  const double at_one = std::log1p(std::expm1(d) / n), at_inf = d / n;
  const double slack = 1e-12 * std::max(1.0, std::abs(goal));
  if (goal > at_one + slack || goal < at_inf - slack)
    throw std::domain_error("theory: observed_rel_var outside the attainable range");
  if (goal >= at_one) return 1.0;
  // log1p_rel_variance decreases in r: bracket by doubling, then bisect
  double lo = 1.0, hi = 2.0;
  while (log1p_rel_variance(d, hi, n) > goal) {
    lo = hi;
    hi *= 2.0;
    if (hi > 1e18) return hi;
  }
  for (int i = 0; i < 200 && hi - lo > 1e-12 * hi; ++i) {
    const double mid = 0.5 * (lo + hi);
    (log1p_rel_variance(d, mid, n) > goal ? lo : hi) = mid;
  }
  return 0.5 * (lo + hi);
}

ParticleBounds particle_bounds(double lambda, double kappa, double r, double t, double eps) {
  require(lambda >= 0.0 && std::isfinite(lambda), "lambda must be finite and >= 0");
  require(kappa >= 1.0 && std::isfinite(kappa), "kappa must be finite and >= 1");
  require(r >= 1.0 && t >= 1.0, "r_eff and t_steps must be >= 1");
  require(eps > 0.0 && std::isfinite(eps), "eps must be finite and > 0");
  const double l2 = lambda * lambda;
  return ParticleBounds{(r / eps) * std::expm1(l2 / (kappa * r * t)),
                        (r / std::log1p(eps)) * std::expm1(kappa * l2 / (r * t))};
}

Regime classify_regime(double ar, double at) {
  require(std::isfinite(ar) && std::isfinite(at), "regime exponents must be finite");
  if (at > 2.0) return Regime::dense;
  return ar + at >= 2.0 ? Regime::stable : Regime::coarse;
}

std::string regime_name(Regime r) {
  return r == Regime::coarse ? "coarse" : (r == Regime::stable ? "stable" : "dense");
}

REffBounds stabilized_r_eff_bounds(double lambda, double kappa, double t, double rho) {
  require(lambda >= 0.0 && std::isfinite(lambda), "lambda must be finite and >= 0");
  require(kappa >= 1.0 && std::isfinite(kappa), "kappa must be finite and >= 1");
  require(t >= 1.0 && std::isfinite(t), "t_steps must be finite and >= 1");
  require(rho >= 0.0 && rho <= 1.0, "rho must lie in [0, 1]");
  if (rho == 0.0) return REffBounds{1.0, 1.0};
  const double l2 = lambda * lambda, x = -std::log(rho);
  if (l2 == 0.0) return REffBounds{1.0, x == 0.0 ? t : 1.0};
  REffBounds b;
  b.lower = std::max(1.0, l2 * t / (kappa * kappa * l2 + kappa * x * t * t));
  b.upper = x == 0.0 ? t : std::min(t, 1.0 + kappa * l2 / (x * t));
  return b;
}
}  // namespace theory

}  // namespace asmc
