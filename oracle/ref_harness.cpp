// ORACLE TEST INFRASTRUCTURE -- not product code.  Only tests/, bench.py's
// cpu_baseline / --impl reference legs and __graft_entry__.smoke() may load it.
//
// C-ABI harness over the UNMODIFIED reference library (/root/reference/proj),
// compiled from the reference's own sources by oracle/Makefile into
// oracle/_ref/libasmc_ref.so (keyed xoshiro streams, rng.hpp) and
// oracle/_ref/libasmc_ref_philox.so (same sources, oracle/shadow/asmc/rng.hpp
// first on the include path).  Functions mirror include/asmc_b200.h so tests can
// feed identical descriptors to the device and to the reference.
//
// The only non-reference code here is (a) descriptor -> object plumbing, and
// (b) ScaleGaussianTarget, the config-2 plugin the reference does not ship,
// written against the reference's AnnealedTarget plugin API (target.hpp:23-52)
// exactly like its own test fixtures (tests/test_kernel.cpp:20-30).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "asmc/config.hpp"
#include "asmc/drivers.hpp"
#include "asmc/experiment.hpp"
#include "asmc/engine.hpp"
#include "asmc/errors.hpp"
#include "asmc/kernel.hpp"
#include "asmc/pt.hpp"
#include "asmc/logsum.hpp"
#include "asmc/rng.hpp"
#include "asmc/schedule.hpp"
#include "asmc/target.hpp"
#include "asmc_b200.h"
#include "engine_detail.hpp"

namespace {

thread_local std::string g_err;

// N(0, s0^2 I) reference -> N(0, s1^2 I) target (both normalized; Z(1) = 1).
// pi_beta = N(0, 1/tau_beta I), tau_beta = (1-beta)/s0^2 + beta/s1^2.
class ScaleGaussianTarget final : public asmc::AnnealedTarget {
 public:
  ScaleGaussianTarget(double s0, double s1, std::size_t dim) : s0_(s0), s1_(s1), dim_(dim) {
    if (!(s0 > 0.0 && s1 > 0.0)) throw std::invalid_argument("scale sigmas must be positive");
    if (dim == 0) throw std::invalid_argument("dim must be at least 1");
  }
  std::size_t dim() const override { return dim_; }
  double log_reference(std::span<const double> x) const override {
    double acc = 0.0;
    for (double xi : x) acc += asmc::log_normal_pdf(xi, 0.0, s0_);
    return acc;
  }
  double potential(std::span<const double> x) const override {
    double acc = 0.0;
    for (double xi : x) {
      acc += asmc::log_normal_pdf(xi, 0.0, s1_) - asmc::log_normal_pdf(xi, 0.0, s0_);
    }
    return acc;
  }
  void sample_reference(asmc::rng::Stream& stream, std::span<double> out) const override {
    check_point(out);
    for (double& xi : out) xi = s0_ * stream.normal();
  }
  asmc::Capabilities capabilities() const override { return {true, true, true}; }
  double tau(double beta) const { return (1.0 - beta) / (s0_ * s0_) + beta / (s1_ * s1_); }
  double analytic_log_z(double beta) const override {
    check_beta(beta);
    return static_cast<double>(dim_) *
           (-(1.0 - beta) * std::log(s0_) - beta * std::log(s1_) - 0.5 * std::log(tau(beta)));
  }
  double analytic_delta(double beta) const override {
    check_beta(beta);
    const double c = 0.5 / (s0_ * s0_) - 0.5 / (s1_ * s1_);
    const double t = tau(beta);
    return static_cast<double>(dim_) * c * c * 2.0 / (t * t);
  }
  double analytic_discrepancy(double beta, double beta2) const override {
    check_beta(beta);
    check_beta(beta2);
    if (beta2 < beta) throw std::domain_error("analytic_discrepancy requires beta2 >= beta");
    const double b3 = 2.0 * beta2 - beta;
    if (b3 > 1.0 + 1e-15) {
      throw std::domain_error("analytic_discrepancy undefined for 2*beta2 - beta > 1");
    }
    return analytic_log_z(std::min(1.0, b3)) + analytic_log_z(beta) - 2.0 * analytic_log_z(beta2);
  }
  void exact_sample(double beta, asmc::rng::Stream& stream, std::span<double> out) const override {
    check_beta(beta);
    check_point(out);
    const double sd = 1.0 / std::sqrt(tau(beta));
    for (double& xi : out) xi = sd * stream.normal();
  }

 private:
  double s0_, s1_;
  std::size_t dim_;
};

// Config-4 plugin: Bayesian logistic regression posterior, eta = N(0, sp^2 I),
// gamma = eta * prod_j sigmoid(x_j.theta)^y_j (1 - sigmoid)^(1 - y_j).
class LogisticTarget final : public asmc::AnnealedTarget {
 public:
  LogisticTarget(double sp, std::size_t n, std::size_t dim, const float* data)
      : sp_(sp), n_(n), dim_(dim), X_(data), y_(data + n * dim) {
    if (!(sp > 0.0)) throw std::invalid_argument("prior sigma must be positive");
    if (dim == 0 || n == 0 || !data) throw std::invalid_argument("logistic target needs data");
  }
  std::size_t dim() const override { return dim_; }
  double log_reference(std::span<const double> x) const override {
    double acc = 0.0;
    for (double xi : x) acc += asmc::log_normal_pdf(xi, 0.0, sp_);
    return acc;
  }
  double potential(std::span<const double> th) const override {
    double acc = 0.0;
    for (std::size_t j = 0; j < n_; ++j) {
      double l = 0.0;
      for (std::size_t i = 0; i < dim_; ++i) l += static_cast<double>(X_[j * dim_ + i]) * th[i];
      const double sp = l > 0.0 ? l + std::log1p(std::exp(-l)) : std::log1p(std::exp(l));
      acc += static_cast<double>(y_[j]) * l - sp;
    }
    return acc;
  }
  void sample_reference(asmc::rng::Stream& stream, std::span<double> out) const override {
    check_point(out);
    for (double& xi : out) xi = sp_ * stream.normal();
  }

 private:
  double sp_;
  std::size_t n_, dim_;
  const float* X_;
  const float* y_;
};

// Config-5 plugin: relaxed Ising model on an L x L torus (include/asmc_b200.h,
// ASMC_TARGET_ISING): y in R^{L^2}, u = A y, A = delta I + K (Adj + 4 I),
// V = sum_i -y_i u_i / 2 + log 2cosh(u_i) - log N(y_i; 0, sigma).
class IsingTarget final : public asmc::AnnealedTarget {
 public:
  IsingTarget(int L, double K, double delta, double sigma)
      : L_(L), K_(K), c_(delta + 4.0 * K), sigma_(sigma) {
    if (L < 3 || !(K >= 0.0) || !(delta > 0.0) || !(sigma > 0.0))
      throw std::invalid_argument("ising needs L >= 3, K >= 0, delta > 0, sigma > 0");
  }
  std::size_t dim() const override { return static_cast<std::size_t>(L_) * L_; }
  double log_reference(std::span<const double> x) const override {
    double acc = 0.0;
    for (double xi : x) acc += asmc::log_normal_pdf(xi, 0.0, sigma_);
    return acc;
  }
  double potential(std::span<const double> y) const override {
    double acc = 0.0;
    for (int a = 0; a < L_; ++a)
      for (int b = 0; b < L_; ++b) {
        const double nb = (y[((a + L_ - 1) % L_) * L_ + b] + y[((a + 1) % L_) * L_ + b]) +
                          (y[a * L_ + (b + L_ - 1) % L_] + y[a * L_ + (b + 1) % L_]);
        const double yi = y[a * L_ + b];
        const double u = c_ * yi + K_ * nb;
        const double au = std::fabs(u);
        acc += -0.5 * yi * u + (au + std::log1p(std::exp(-2.0 * au))) - asmc::log_normal_pdf(yi, 0.0, sigma_);
      }
    return acc;
  }
  void sample_reference(asmc::rng::Stream& stream, std::span<double> out) const override {
    check_point(out);
    for (double& xi : out) xi = sigma_ * stream.normal();
  }

 private:
  int L_;
  double K_, c_, sigma_;
};

std::unique_ptr<asmc::AnnealedTarget> make_target(const asmc_target_desc* t) {
  if (!t) throw std::invalid_argument("null target descriptor");
  const double* p = t->p;
  switch (t->kind) {
    case ASMC_TARGET_GAUSSIAN_SHIFT:
      return std::make_unique<asmc::GaussianShiftTarget>(p[0], p[1], p[2], t->dim);
    case ASMC_TARGET_MIXTURE:
      return std::make_unique<asmc::MixtureTarget>(p[0], p[1], p[2], p[3], p[4], p[5], t->dim);
    case ASMC_TARGET_SCALE_GAUSSIAN:
      return std::make_unique<ScaleGaussianTarget>(p[0], p[1], t->dim);
    case ASMC_TARGET_LOGISTIC:
      return std::make_unique<LogisticTarget>(p[0], static_cast<std::size_t>(p[1]), t->dim,
                                              static_cast<const float*>(t->data));
    case ASMC_TARGET_ISING:
      return std::make_unique<IsingTarget>(static_cast<int>(p[0]), p[1], p[2], p[3]);
  }
  throw asmc::capability_error("unknown target kind " + std::to_string(t->kind));
}

asmc::Kernel make_kernel(const asmc_kernel_desc* k) {
  if (!k) throw std::invalid_argument("null kernel descriptor");
  asmc::Kernel out;
  out.kind = static_cast<asmc::KernelKind>(k->kind);
  out.step_sizes.assign(k->step_sizes, k->step_sizes + k->n_step_sizes);
  out.sweeps = k->sweeps;
  return out;
}

asmc::Schedule make_schedule(const double* betas, int steps) {
  asmc::Schedule s;
  s.betas.assign(betas, betas + steps + 1);
  return s;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return ASMC_OK;
  } catch (const asmc::capability_error& e) {
    g_err = e.what();
    return ASMC_ERR_CAPABILITY;
  } catch (const asmc::degenerate_weights_error& e) {
    g_err = e.what();
    return ASMC_ERR_DEGENERATE;
  } catch (const asmc::evaluation_error& e) {
    g_err = e.what();
    return ASMC_ERR_EVALUATION;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return ASMC_ERR_DOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ASMC_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ASMC_ERR_INTERNAL;
  }
}

void fill_report(const asmc::RunReport& rep, asmc_report* out) {
  const std::size_t m = rep.stats.log_g0.size();
  auto copy = [m](const std::vector<double>& v, double* dst) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(double) * std::min(m, v.size()));
  };
  copy(rep.stats.log_g0, out->log_g0);
  copy(rep.stats.log_g1, out->log_g1);
  copy(rep.stats.log_g2, out->log_g2);
  copy(rep.ess_trace, out->ess_trace);
  copy(rep.cum_log_z, out->cum_log_z);
  if (out->resampled) std::memcpy(out->resampled, rep.resampled.data(), rep.resampled.size());
  out->n_resample_times = static_cast<int32_t>(rep.resample_times.size());
  if (out->resample_times) {
    for (std::size_t i = 0; i < rep.resample_times.size(); ++i) {
      out->resample_times[i] = rep.resample_times[i];
    }
  }
  out->log_z_hat = rep.log_z_hat;
  out->elbo_hat = rep.elbo_hat;
  out->wall_seconds = rep.wall_seconds;
  out->kernel_applications = rep.kernel_applications;
}

}  // namespace

extern "C" {

const char* ora_last_error(void) { return g_err.c_str(); }
int ora_is_reference(void) { return 1; }

int ora_run_smc(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                const double* betas, int32_t steps, uint64_t n, int32_t policy, double rho,
                uint64_t seed, uint64_t round, int32_t workers, asmc_report* out) {
  return guard([&] {
    const auto tg = make_target(target);
    asmc::RunOptions o;
    o.n_particles = n;
    o.policy = static_cast<asmc::ResamplePolicy>(policy);
    o.rho = rho;
    o.seed = seed;
    o.round = round;
    o.workers = workers;
    fill_report(asmc::run_smc(*tg, make_kernel(kernel), make_schedule(betas, steps), o), out);
  });
}

int ora_run_sais_single(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                        const double* betas, int32_t steps, uint64_t n, uint64_t seed,
                        uint64_t round, int32_t workers, uint64_t chunk, asmc_report* out) {
  return guard([&] {
    const auto tg = make_target(target);
    asmc::RunOptions o;
    o.n_particles = n;
    o.policy = asmc::ResamplePolicy::never;
    o.seed = seed;
    o.round = round;
    o.workers = workers;
    fill_report(
        asmc::run_sais_single(*tg, make_kernel(kernel), make_schedule(betas, steps), o, chunk),
        out);
  });
}

int ora_run_rounds(const asmc_target_desc* target, const asmc_kernel_desc* kernel, int32_t mode,
                   uint64_t n, int32_t rounds, int32_t policy, double rho, uint64_t seed,
                   uint64_t memory_cap, int32_t workers, asmc_rounds_out* out) {
  return guard([&] {
    const auto tg = make_target(target);
    asmc::DriverOptions o;
    o.n_particles = n;
    o.rounds = rounds;
    o.policy = static_cast<asmc::ResamplePolicy>(policy);
    o.rho = rho;
    o.seed = seed;
    o.workers = workers;
    o.memory_cap_bytes = memory_cap;
    const auto res = mode == ASMC_MODE_SAIS ? asmc::run_sais(*tg, make_kernel(kernel), o)
                                            : asmc::run_ssmc(*tg, make_kernel(kernel), o);
    const int stride = out->max_steps + 1;
    for (std::size_t k = 0; k < res.size(); ++k) {
      const auto& rep = res[k].report;
      const int T = rep.schedule.steps();
      if (T > out->max_steps) throw std::invalid_argument("max_steps too small");
      if (out->n_particles) out->n_particles[k] = rep.n_particles;
      if (out->steps) out->steps[k] = T;
      for (int t = 0; t <= T; ++t) {
        const std::size_t r = k * stride + t;
        if (out->betas) out->betas[r] = rep.schedule.betas[t];
        if (out->log_g0) out->log_g0[r] = rep.stats.log_g0[t];
        if (out->log_g1) out->log_g1[r] = rep.stats.log_g1[t];
        if (out->log_g2) out->log_g2[r] = rep.stats.log_g2[t];
        if (out->ess_trace && !rep.ess_trace.empty()) out->ess_trace[r] = rep.ess_trace[t];
        if (out->cum_log_z) out->cum_log_z[r] = rep.cum_log_z[t];
        if (out->resampled) out->resampled[r] = rep.resampled[t];
        if (out->lambda) out->lambda[r] = res[k].barrier.lambda[t];
      }
      if (out->log_z_hat) out->log_z_hat[k] = rep.log_z_hat;
      if (out->elbo_hat) out->elbo_hat[k] = rep.elbo_hat;
      if (out->wall_seconds) out->wall_seconds[k] = rep.wall_seconds;
      if (out->kernel_applications) out->kernel_applications[k] = rep.kernel_applications;
    }
  });
}

// Per-particle SAIS pass through the reference's own per-particle body
// (drivers.cpp:95-111 -> engine_detail.hpp:27-41), recording the state after
// every step.  lg_out[t] is the incremental log-weight of step t (slot 0 = 0).
int ora_trajectory(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                   const double* betas, int32_t steps, uint64_t seed, uint64_t round,
                   uint64_t particle, double* x_out, double* lw_out, double* lg_out) {
  return guard([&] {
    const auto tg = make_target(target);
    const asmc::Kernel kern = make_kernel(kernel);
    const std::size_t d = tg->dim();
    std::vector<double> x(d);
    asmc::rng::Stream si(asmc::rng::Key{seed, round, particle, 0, asmc::rng::kSubstepInit});
    tg->sample_reference(si, {x.data(), d});
    double log_w = 0.0;
    std::memcpy(x_out, x.data(), d * sizeof(double));
    lw_out[0] = 0.0;
    if (lg_out) lg_out[0] = 0.0;
    asmc::LogAccumulator g0, g1, g2;
    asmc::SignedLogAccumulator el;
    for (int t = 1; t <= steps; ++t) {
      asmc::rng::Stream se(asmc::rng::Key{seed, round, particle, static_cast<std::uint64_t>(t),
                                          asmc::rng::kSubstepExplore});
      const double before = log_w;
      asmc::detail::weight_and_move(*tg, kern, betas[t - 1], betas[t], {x.data(), d}, log_w, g0,
                                    g1, g2, el, se);
      std::memcpy(x_out + static_cast<std::size_t>(t) * d, x.data(), d * sizeof(double));
      lw_out[t] = log_w;
      if (lg_out) lg_out[t] = log_w - before;
    }
  });
}

int ora_rng_u64(const uint64_t key[5], uint64_t count, uint64_t* out) {
  return guard([&] {
    asmc::rng::Stream s(asmc::rng::Key{key[0], key[1], key[2], key[3], key[4]});
    for (uint64_t i = 0; i < count; ++i) out[i] = s.next_u64();
  });
}
int ora_rng_uniform(const uint64_t key[5], uint64_t count, double* out) {
  return guard([&] {
    asmc::rng::Stream s(asmc::rng::Key{key[0], key[1], key[2], key[3], key[4]});
    for (uint64_t i = 0; i < count; ++i) out[i] = s.uniform();
  });
}
int ora_rng_normal(const uint64_t key[5], uint64_t count, double* out) {
  return guard([&] {
    asmc::rng::Stream s(asmc::rng::Key{key[0], key[1], key[2], key[3], key[4]});
    for (uint64_t i = 0; i < count; ++i) out[i] = s.normal();
  });
}

int ora_systematic_resample(const double* lw, uint64_t n, const uint64_t key[5], uint32_t* out) {
  return guard([&] {
    asmc::rng::Stream s(asmc::rng::Key{key[0], key[1], key[2], key[3], key[4]});
    const auto a = asmc::systematic_resample({lw, n}, s);
    std::memcpy(out, a.data(), n * sizeof(uint32_t));
  });
}

int ora_ess(const double* lw, uint64_t n, double* out) {
  return guard([&] { *out = asmc::ess({lw, n}); });
}

static asmc::IncrementStats make_stats(const double* g0, const double* g1, const double* g2,
                                       int steps) {
  asmc::IncrementStats st;
  st.log_g0.assign(g0, g0 + steps + 1);
  st.log_g1.assign(g1, g1 + steps + 1);
  st.log_g2.assign(g2, g2 + steps + 1);
  return st;
}

int ora_barrier_estimate(const double* g0, const double* g1, const double* g2,
                         const double* betas, int32_t steps, double* lambda) {
  return guard([&] {
    const auto est = asmc::barrier_estimate(make_stats(g0, g1, g2, steps),
                                            make_schedule(betas, steps));
    std::memcpy(lambda, est.lambda.data(), est.lambda.size() * sizeof(double));
  });
}

int ora_discrepancy_hat(const double* g0, const double* g1, const double* g2, int32_t steps,
                        int32_t t, double* out) {
  return guard([&] { *out = asmc::discrepancy_hat(make_stats(g0, g1, g2, steps), t); });
}

int ora_cess(const double* g0, const double* g1, const double* g2, int32_t steps, int32_t t,
             uint64_t n, double* out) {
  return guard([&] { *out = asmc::cess(make_stats(g0, g1, g2, steps), t, n); });
}

int ora_generate_schedule(const double* lambda, const double* beta, int32_t knots, int32_t t_new,
                          double* out) {
  return guard([&] {
    asmc::BarrierEstimate est;
    est.lambda.assign(lambda, lambda + knots);
    est.beta.assign(beta, beta + knots);
    const auto s = asmc::generate_schedule(est, t_new);
    std::memcpy(out, s.betas.data(), s.betas.size() * sizeof(double));
  });
}

int ora_local_barrier(const double* lambda, const double* beta, int32_t knots, double* out) {
  return guard([&] {
    asmc::BarrierEstimate est;
    est.lambda.assign(lambda, lambda + knots);
    est.beta.assign(beta, beta + knots);
    const auto v = asmc::local_barrier(est);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

int ora_budget(uint64_t n, int32_t steps, uint64_t dim, uint64_t cap, int32_t mode,
               uint64_t* n_out, int32_t* t_out) {
  return guard([&] {
    const auto p = asmc::budget(n, steps, dim, cap, static_cast<asmc::DriverMode>(mode));
    *n_out = p.n_particles;
    *t_out = p.steps;
  });
}

int ora_analytic_log_z(const asmc_target_desc* target, double beta, double* out) {
  return guard([&] { *out = make_target(target)->analytic_log_z(beta); });
}

// asmc::run_zja (drivers.cpp:234-341) and asmc::zja_next_beta (schedule.cpp:219-264)
int ora_run_zja(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const asmc_zja_opts* o,
                int32_t workers, asmc_zja_out* out) {
  return guard([&] {
    const auto tg = make_target(target);
    asmc::ZjaOptions zo;
    zo.n_particles = o->n_particles;
    zo.target_steps = o->target_steps;
    zo.delta_star = o->delta_star;
    zo.seed = o->seed;
    zo.workers = workers;
    zo.max_steps = o->max_steps;
    const asmc::ZjaOutcome r = asmc::run_zja(*tg, make_kernel(kernel), zo);
    out->delta_star = r.delta_star;
    out->warning = r.warning ? 1 : 0;
    out->pilot_ran = r.rounds.size() == 2 ? 1 : 0;
    const asmc::RoundResult& m = r.rounds.back();
    const int T = m.report.schedule.steps();
    if (T + 1 > out->capacity) throw std::invalid_argument("output capacity too small");
    out->steps = T;
    if (out->betas) std::memcpy(out->betas, m.report.schedule.betas.data(), sizeof(double) * (T + 1));
    if (out->lambda) std::memcpy(out->lambda, m.barrier.lambda.data(), sizeof(double) * (T + 1));
    fill_report(m.report, &out->main);
    if (out->pilot_ran) {
      fill_report(r.rounds[0].report, &out->pilot);
      if (out->pilot_lambda)
        std::memcpy(out->pilot_lambda, r.rounds[0].barrier.lambda.data(),
                    sizeof(double) * r.rounds[0].barrier.lambda.size());
    }
  });
}

int ora_zja_next_beta(const asmc_target_desc* target, double beta, const double* xs, uint64_t n,
                      const double* lw, double delta, double tol, double* beta_next, int32_t* warning) {
  return guard([&] {
    const auto tg = make_target(target);
    const auto r = asmc::zja_next_beta(*tg, beta, std::span<const double>(xs, n * tg->dim()), n,
                                       std::span<const double>(lw, n), delta, tol);
    *beta_next = r.beta_next;
    if (warning) *warning = r.warning ? 1 : 0;
  });
}

// asmc::run_experiment (experiment.cpp:200-233) on a key=value config text: the
// reference's own CSV writer, used to pin the report/CSV format of the B200 path.
int ora_run_experiment(const char* config_text, const char* out_dir) {
  return guard([&] {
    asmc::RunConfig c = asmc::parse_config_text(config_text);
    c.out_dir = out_dir;
    if (asmc::run_experiment(c) != 0) throw std::runtime_error("run_experiment failed");
  });
}

// asmc::run_pt (pt.cpp:84-128) for replicas r = 0..R-1 with seeds seed + r
int ora_run_pt(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const double* betas,
               int32_t levels, const asmc_pt_opts* o, asmc_pt_out* out) {
  return guard([&] {
    const auto tg = make_target(target);
    const asmc::Kernel k = make_kernel(kernel);
    const asmc::Schedule sched = make_schedule(betas, levels);
    const std::size_t L1 = static_cast<std::size_t>(levels) + 1, I = o->iterations;
    for (int r = 0; r < o->replicas; ++r) {
      asmc::PtOptions po;
      po.iterations = o->iterations;
      po.burn_in = o->burn_in;
      po.seed = o->seed + static_cast<std::uint64_t>(r);
      po.round = o->round;
      const asmc::PtReport rep = asmc::run_pt(*tg, k, sched, po);
      if (out->log_z_hat) out->log_z_hat[r] = rep.log_z_hat;
      if (out->trace) std::memcpy(out->trace + r * I * L1, rep.trace.values.data(), sizeof(double) * I * L1);
      if (out->swap_accepted) std::memcpy(out->swap_accepted + r * I * L1, rep.swap_accepted.data(), I * L1);
      if (out->swap_attempts)
        std::memcpy(out->swap_attempts + r * L1, rep.swap_attempts.data(), sizeof(std::uint64_t) * L1);
      if (out->swap_accepts)
        std::memcpy(out->swap_accepts + r * L1, rep.swap_accepts.data(), sizeof(std::uint64_t) * L1);
      out->kernel_applications = rep.kernel_applications;
      out->burn_in = rep.burn_in;
    }
  });
}

int ora_hardware_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
