/*
 * ORACLE TEST INFRASTRUCTURE -- not product code.  Only tests/, bench.py's
 * cpu_baseline / --impl reference legs and __graft_entry__.smoke() may load it
 * (as oracle/_ref/liborarestate.so).
 *
 * Plain-C restatement of the reference `asmc` sampler hot path, in the
 * reference's operation order so that, linked against the same libm and
 * compiled without FMA contraction, it reproduces the reference bit for bit
 * (tests/test_oracle.py pins it against oracle/_ref/libasmc_ref*.so, which is
 * the unmodified reference).  Each function cites the reference lines it
 * restates (paths relative to /root/reference/proj/).  Two stream families:
 *   rng 0 = keyed xoshiro256++     include/asmc/rng.hpp:27-86
 *   rng 1 = keyed Philox4x32-10    oracle/shadow/asmc/rng.hpp (shadow header)
 * Systematic resampling is the reference's own sequential-CDF rule
 * (engine.cpp:61-80); the device reproduces its CDF bit for bit (csrc/refcdf.cu),
 * and ora_resample_cdf exposes the CDF so the tests compare it value by value.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "asmc_b200.h"

static _Thread_local char g_err[512];
static int g_rng = ASMC_RNG_XOSHIRO;

#define FAIL(code, ...)                                   \
  do {                                                    \
    snprintf(g_err, sizeof g_err, __VA_ARGS__);           \
    return (code);                                        \
  } while (0)
#define TRY(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_) return rc_;     \
  } while (0)

const char* ora_last_error(void) { return g_err; }
int ora_is_reference(void) { return 0; }
void ora_set_rng(int rng) { g_rng = rng; }

/* ------------------------------------------------------------------ RNG -- */
/* rng.hpp:27-31 */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

typedef struct {
  int kind;
  /* xoshiro */
  uint64_t s[4];
  double cached;
  int have_cached;
  /* philox */
  uint32_t k0, k1, c1, c2, c3;
  uint64_t n_u64, n_normal, block;
  uint32_t words[4];
} stream_t;

static void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

/* rng.hpp:43-55 (xoshiro) / shadow rng.hpp Stream ctor (philox) */
static void stream_init(stream_t* st, uint64_t seed, uint64_t round, uint64_t particle,
                        uint64_t step, uint64_t substep) {
  memset(st, 0, sizeof *st);
  st->kind = g_rng;
  if (g_rng == ASMC_RNG_XOSHIRO) {
    uint64_t acc = mix64(seed + 0x9E3779B97F4A7C15ULL);
    acc = mix64(acc ^ (round + 0xD1B54A32D192ED03ULL));
    acc = mix64(acc ^ (particle + 0x8CB92BA72F3D8DD7ULL));
    acc = mix64(acc ^ (step + 0xA24BAED4963EE407ULL));
    acc = mix64(acc ^ (substep + 0x9FB21C651E98DF25ULL));
    for (int i = 0; i < 4; ++i) {
      acc += 0x9E3779B97F4A7C15ULL;
      st->s[i] = mix64(acc);
    }
    if ((st->s[0] | st->s[1] | st->s[2] | st->s[3]) == 0) st->s[0] = 1;
  } else {
    uint64_t acc = mix64(seed + 0x9E3779B97F4A7C15ULL);
    acc = mix64(acc ^ (round + 0xD1B54A32D192ED03ULL));
    acc = mix64(acc ^ (substep + 0x9FB21C651E98DF25ULL));
    st->k0 = (uint32_t)acc;
    st->k1 = (uint32_t)(acc >> 32);
    st->c1 = (uint32_t)step;
    st->c2 = (uint32_t)particle;
    st->c3 = (uint32_t)(particle >> 32) ^ ((uint32_t)(step >> 32) * 0x9E3779B9u);
    st->block = ~(uint64_t)0;
  }
}

/* rng.hpp:57-68 */
static uint64_t next_u64(stream_t* st) {
  if (st->kind == ASMC_RNG_XOSHIRO) {
    uint64_t* s = st->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
  }
  uint32_t c[4] = {0x80000000u | (uint32_t)(st->n_u64++), st->c1, st->c2, st->c3};
  philox10(c, st->k0, st->k1);
  return ((uint64_t)c[0] << 32) | c[1];
}

/* rng.hpp:71 */
static double uniform(stream_t* st) { return (double)(next_u64(st) >> 11) * 0x1.0p-53; }

/* rng.hpp:73-86 (xoshiro, cached sine) / shadow normal() (philox) */
static double normal(stream_t* st) {
  if (st->kind == ASMC_RNG_XOSHIRO) {
    if (st->have_cached) {
      st->have_cached = 0;
      return st->cached;
    }
    double u1 = uniform(st);
    while (u1 == 0.0) u1 = uniform(st);
    const double u2 = uniform(st);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586477 * u2;
    st->cached = r * sin(a);
    st->have_cached = 1;
    return r * cos(a);
  }
  const uint64_t j = st->n_normal++;
  const uint64_t b = j >> 2;
  if (b != st->block) {
    uint32_t c[4] = {(uint32_t)b, st->c1, st->c2, st->c3};
    philox10(c, st->k0, st->k1);
    memcpy(st->words, c, sizeof c);
    st->block = b;
  }
  const unsigned w = (unsigned)(j & 3);
  const double u1 = ((double)st->words[w & 2u] + 1.0) * 0x1.0p-32;
  const double u2 = (double)st->words[(w & 2u) + 1u] * 0x1.0p-32;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586477 * u2;
  return (w & 1u) ? r * sin(a) : r * cos(a);
}

/* ------------------------------------------------------- accumulators -- */
/* logsum.hpp:18-49 */
typedef struct { double max, sum; } lacc_t;
static const lacc_t LACC0 = {-INFINITY, 0.0};
static void lacc_add(lacc_t* a, double l) {
  if (l == -INFINITY) return;
  if (l <= a->max) {
    a->sum += exp(l - a->max);
  } else {
    a->sum = a->sum * exp(a->max - l) + 1.0;
    a->max = l;
  }
}
static void lacc_combine(lacc_t* a, const lacc_t* o) {
  if (o->max == -INFINITY) return;
  if (o->max <= a->max) {
    a->sum += o->sum * exp(o->max - a->max);
  } else {
    a->sum = a->sum * exp(a->max - o->max) + o->sum;
    a->max = o->max;
  }
}
static double lacc_total(const lacc_t* a) {
  return a->max == -INFINITY ? -INFINITY : a->max + log(a->sum);
}
/* logsum.hpp:53-84 */
static void sacc_add(lacc_t* a, double log_abs, double sign) {
  if (log_abs == -INFINITY || sign == 0.0) return;
  if (log_abs <= a->max) {
    a->sum += sign * exp(log_abs - a->max);
  } else {
    a->sum = a->sum * exp(a->max - log_abs) + sign;
    a->max = log_abs;
  }
}
static double sacc_value_scaled(const lacc_t* a, double log_scale) {
  if (a->max == -INFINITY) return 0.0;
  return a->sum * exp(a->max - log_scale);
}

/* ------------------------------------------------------------ targets -- */
static const double kLogSqrt2Pi = 0.91893853320467274178; /* target.cpp:13 */

/* target.cpp:16-19 */
static double log_normal_pdf(double x, double mu, double sigma) {
  const double s = (x - mu) / sigma;
  return -0.5 * s * s - log(sigma) - kLogSqrt2Pi;
}

static int check_target(const asmc_target_desc* t) {
  if (!t) FAIL(ASMC_ERR_INVALID_ARGUMENT, "null target");
  const double* p = t->p;
  switch (t->kind) {
    case ASMC_TARGET_GAUSSIAN_SHIFT: /* target.cpp:57-63 */
      if (!(p[2] > 0.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "sigma must be positive");
      break;
    case ASMC_TARGET_MIXTURE: /* target.cpp:115-131 */
      if (!(p[0] > 0.0 && p[3] > 0.0 && p[5] > 0.0))
        FAIL(ASMC_ERR_INVALID_ARGUMENT, "mixture sigmas must be positive");
      if (!(p[1] > 0.0 && p[1] < 1.0))
        FAIL(ASMC_ERR_INVALID_ARGUMENT, "mixture weight must lie strictly in (0, 1)");
      break;
    case ASMC_TARGET_SCALE_GAUSSIAN:
      if (!(p[0] > 0.0 && p[1] > 0.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "scale sigmas must be positive");
      break;
    case ASMC_TARGET_LOGISTIC:
      if (!(p[0] > 0.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "prior sigma must be positive");
      if (!t->data || t->data_bytes < (uint64_t)p[1] * (t->dim + 1) * sizeof(float))
        FAIL(ASMC_ERR_INVALID_ARGUMENT, "logistic target needs X (n x dim) and y (n) data");
      break;
    case ASMC_TARGET_ISING:
      if (!(p[0] >= 3.0 && p[0] == floor(p[0]) && t->dim == (uint64_t)p[0] * (uint64_t)p[0]))
        FAIL(ASMC_ERR_INVALID_ARGUMENT, "ising target needs an integer side L >= 3 and dim = L * L");
      if (!(p[1] >= 0.0 && p[2] > 0.0 && p[3] > 0.0))
        FAIL(ASMC_ERR_INVALID_ARGUMENT, "ising needs K >= 0, delta > 0, sigma > 0");
      break;
    default:
      FAIL(ASMC_ERR_CAPABILITY, "unknown target kind %d", t->kind);
  }
  if (t->dim == 0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "dim must be at least 1");
  return 0;
}

/* NEW plugin (config 4): Bayesian logistic regression, V = sum_j y_j l_j - softplus(l_j),
 * l_j = x_j . theta, accumulated in double in row then column order. */
static double logistic_potential(const asmc_target_desc* t, const double* th) {
  const uint64_t d = t->dim, n = (uint64_t)t->p[1];
  const float* X = (const float*)t->data;
  const float* y = X + n * d;
  double acc = 0.0;
  for (uint64_t j = 0; j < n; ++j) {
    double l = 0.0;
    for (uint64_t i = 0; i < d; ++i) l += (double)X[j * d + i] * th[i];
    const double sp = l > 0.0 ? l + log1p(exp(-l)) : log1p(exp(l));
    acc += (double)y[j] * l - sp;
  }
  return acc;
}

/* NEW plugin (config 5): relaxed Ising on an L x L torus (include/asmc_b200.h).
 * u = A y with A = delta I + K (Adj + 4 I), neighbour sum grouped (a-1 + a+1) + (b-1 + b+1). */
static void ising_stencil(const asmc_target_desc* t, const double* y, double* u) {
  const int L = (int)t->p[0];
  const double K = t->p[1], c = t->p[2] + 4.0 * t->p[1];
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) {
      const double nb = (y[((a + L - 1) % L) * L + b] + y[((a + 1) % L) * L + b]) +
                        (y[a * L + (b + L - 1) % L] + y[a * L + (b + 1) % L]);
      u[a * L + b] = c * y[a * L + b] + K * nb;
    }
}

static double log2cosh(double u) {
  const double a = fabs(u);
  return a + log1p(exp(-2.0 * a));
}

/* V = sum_i -y_i u_i / 2 + log 2cosh(u_i) - log N(y_i; 0, sigma) */
static double ising_potential(const asmc_target_desc* t, const double* y) {
  const uint64_t n = t->dim;
  double* u = malloc(n * sizeof(double));
  ising_stencil(t, y, u);
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc += -0.5 * y[i] * u[i] + log2cosh(u[i]) - log_normal_pdf(y[i], 0.0, t->p[3]);
  free(u);
  return acc;
}

/* grad log gamma_beta = beta A (tanh(u) - y) - (1 - beta) y / sigma^2;  work: 2 n doubles */
static void ising_grad(const asmc_target_desc* t, double beta, const double* y, double* g, double* work) {
  const uint64_t n = t->dim;
  double* u = work;
  double* v = work + n;
  ising_stencil(t, y, u);
  for (uint64_t i = 0; i < n; ++i) v[i] = tanh(u[i]) - y[i];
  ising_stencil(t, v, g);
  const double is2 = 1.0 / (t->p[3] * t->p[3]);
  for (uint64_t i = 0; i < n; ++i) g[i] = beta * g[i] - (1.0 - beta) * is2 * y[i];
}

/* target.cpp:65-69, 133-137 and the scale / logistic / ising plugins (oracle/ref_harness.cpp) */
static double log_reference(const asmc_target_desc* t, const double* x) {
  double acc = 0.0;
  const double* p = t->p;
  const double mu = t->kind == ASMC_TARGET_GAUSSIAN_SHIFT ? p[0] : 0.0;
  const double sg = t->kind == ASMC_TARGET_GAUSSIAN_SHIFT ? p[2] : t->kind == ASMC_TARGET_ISING ? p[3] : p[0];
  for (uint64_t i = 0; i < t->dim; ++i) acc += log_normal_pdf(x[i], mu, sg);
  return acc;
}

/* target.cpp:71-78, 139-152 */
static double potential(const asmc_target_desc* t, const double* x) {
  const double* p = t->p;
  double acc = 0.0;
  if (t->kind == ASMC_TARGET_LOGISTIC) return logistic_potential(t, x);
  if (t->kind == ASMC_TARGET_ISING) return ising_potential(t, x);
  if (t->kind == ASMC_TARGET_GAUSSIAN_SHIFT) {
    const double a = (p[1] - p[0]) / (p[2] * p[2]);
    const double mid = 0.5 * (p[0] + p[1]);
    for (uint64_t i = 0; i < t->dim; ++i) acc += a * (x[i] - mid);
  } else if (t->kind == ASMC_TARGET_MIXTURE) {
    const double lw1 = log(p[1]);
    const double lw2 = log1p(-p[1]);
    for (uint64_t i = 0; i < t->dim; ++i) {
      const double xi = x[i];
      const double a = lw1 + log_normal_pdf(xi, p[2], p[3]);
      const double b = lw2 + log_normal_pdf(xi, p[4], p[5]);
      const double hi = a > b ? a : b;
      const double lo = a > b ? b : a;
      const double log_mix = hi + log1p(exp(lo - hi));
      acc += log_mix - log_normal_pdf(xi, 0.0, p[0]);
    }
  } else {
    for (uint64_t i = 0; i < t->dim; ++i)
      acc += log_normal_pdf(x[i], 0.0, p[1]) - log_normal_pdf(x[i], 0.0, p[0]);
  }
  return acc;
}

/* target.cpp:34-39 */
static double log_gamma(const asmc_target_desc* t, double beta, const double* x) {
  if (beta == 0.0) return log_reference(t, x);
  return log_reference(t, x) + beta * potential(t, x);
}

/* target.cpp:80-83, 154-157 */
static void sample_reference(const asmc_target_desc* t, stream_t* st, double* out) {
  const double* p = t->p;
  for (uint64_t i = 0; i < t->dim; ++i) {
    if (t->kind == ASMC_TARGET_GAUSSIAN_SHIFT) out[i] = p[0] + p[2] * normal(st);
    else if (t->kind == ASMC_TARGET_ISING) out[i] = p[3] * normal(st);
    else out[i] = p[0] * normal(st);
  }
}

/* target.cpp:107-113 and the scale plugin */
static int exact_sample(const asmc_target_desc* t, double beta, stream_t* st, double* out) {
  const double* p = t->p;
  if (t->kind == ASMC_TARGET_GAUSSIAN_SHIFT) {
    const double mu = (1.0 - beta) * p[0] + beta * p[1];
    for (uint64_t i = 0; i < t->dim; ++i) out[i] = mu + p[2] * normal(st);
    return 0;
  }
  if (t->kind == ASMC_TARGET_SCALE_GAUSSIAN) {
    const double tau = (1.0 - beta) / (p[0] * p[0]) + beta / (p[1] * p[1]);
    const double sd = 1.0 / sqrt(tau);
    for (uint64_t i = 0; i < t->dim; ++i) out[i] = sd * normal(st);
    return 0;
  }
  FAIL(ASMC_ERR_CAPABILITY, "idealized_exact kernel requires an exact sampler");
}

/* ------------------------------------------------------------ kernels -- */
/* kernel.cpp:12-22 */
static int validate_kernel(const asmc_kernel_desc* k) {
  if (!k) FAIL(ASMC_ERR_INVALID_ARGUMENT, "null kernel");
  if (k->kind == ASMC_KERNEL_RWMH) {
    if (k->n_step_sizes < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "rwmh_cycle requires at least one step size");
    for (int i = 0; i < k->n_step_sizes; ++i)
      if (!(k->step_sizes[i] > 0.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "rwmh step sizes must be positive");
    if (k->sweeps < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "rwmh sweeps must be at least 1");
  } else if (k->kind == ASMC_KERNEL_HMC) {
    if (k->n_step_sizes < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "hmc requires at least one step size");
    for (int i = 0; i < k->n_step_sizes; ++i)
      if (!(k->step_sizes[i] > 0.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "hmc step sizes must be positive");
    if (k->sweeps < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "hmc sweeps must be at least 1");
    if (k->leapfrog < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "hmc leapfrog steps must be at least 1");
  } else if (k->kind == ASMC_KERNEL_SLICE) {
    if (k->sweeps < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "slice sweeps must be at least 1");
  } else if (k->kind != ASMC_KERNEL_IDEALIZED && k->kind != ASMC_KERNEL_IDENTITY) {
    FAIL(ASMC_ERR_INVALID_ARGUMENT, "unknown kernel kind");
  }
  return 0;
}

/* kernel.cpp:26-42 (scratch passed in instead of allocated per call) */
static void rwmh_cycle_move(const asmc_target_desc* t, const asmc_kernel_desc* k, double beta,
                            double* x, double* proposal, stream_t* st) {
  const uint64_t d = t->dim;
  double log_gamma_x = log_gamma(t, beta, x);
  for (int sweep = 0; sweep < k->sweeps; ++sweep) {
    for (int si = 0; si < k->n_step_sizes; ++si) {
      const double s = k->step_sizes[si];
      for (uint64_t i = 0; i < d; ++i) proposal[i] = x[i] + s * normal(st);
      const double log_gamma_p = log_gamma(t, beta, proposal);
      const double log_u = log(uniform(st));
      if (log_u < log_gamma_p - log_gamma_x) {
        for (uint64_t i = 0; i < d; ++i) x[i] = proposal[i];
        log_gamma_x = log_gamma_p;
      }
    }
  }
}

/* d/dx_i log gamma_beta(x), per coordinate (product-form targets).  NEW -- the
 * reference has no gradient-based kernel; the device's HMC uses these exact
 * expressions (csrc/targets.cuh grad64). */
static double grad_log_gamma(const asmc_target_desc* t, double beta, double xi) {
  const double* p = t->p;
  if (t->kind == ASMC_TARGET_GAUSSIAN_SHIFT) {
    const double a = (p[1] - p[0]) / (p[2] * p[2]);
    return -(xi - p[0]) / (p[2] * p[2]) + beta * a;
  }
  if (t->kind == ASMC_TARGET_SCALE_GAUSSIAN) {
    const double tau = (1.0 - beta) / (p[0] * p[0]) + beta / (p[1] * p[1]);
    return -tau * xi;
  }
  /* mixture: grad log eta + beta * grad V, V = log_mix - log eta */
  const double a = log(p[1]) + log_normal_pdf(xi, p[2], p[3]);
  const double b = log1p(-p[1]) + log_normal_pdf(xi, p[4], p[5]);
  const double r1 = 1.0 / (1.0 + exp(b - a));
  const double glm = -(r1 * (xi - p[2]) / (p[3] * p[3]) + (1.0 - r1) * (xi - p[4]) / (p[5] * p[5]));
  const double gref = -xi / (p[0] * p[0]);
  return gref + beta * (glm - gref);
}

/* whole-vector gradient (work: 2 d doubles); separable targets per coordinate */
static void grad_vec(const asmc_target_desc* t, double beta, const double* x, double* g, double* work) {
  if (t->kind == ASMC_TARGET_ISING) {
    ising_grad(t, beta, x, g, work);
    return;
  }
  for (uint64_t i = 0; i < t->dim; ++i) g[i] = grad_log_gamma(t, beta, x[i]);
}

/* NEW kernel (no reference code): HMC cycling through the step sizes as the
 * leapfrog epsilon, unit mass, `leapfrog` steps per trajectory.  Draw order per
 * trajectory: d momentum normals, then one uniform (as RWMH: kernel.cpp:31-36).
 * Accept iff log u < (log g(x') - log g(x)) + (|p0|^2 - |p1|^2) / 2. */
static void hmc_cycle_move(const asmc_target_desc* t, const asmc_kernel_desc* k, double beta,
                           double* x, double* scratch, stream_t* st) {
  const uint64_t d = t->dim;
  double* xp = scratch;
  double* pm = scratch + d;
  double* g = scratch + 2 * d;
  double* work = scratch + 3 * d;  /* 2 d */
  double log_gamma_x = log_gamma(t, beta, x);
  for (int sweep = 0; sweep < k->sweeps; ++sweep) {
    for (int si = 0; si < k->n_step_sizes; ++si) {
      const double eps = k->step_sizes[si];
      double k0 = 0.0;
      for (uint64_t i = 0; i < d; ++i) {
        pm[i] = normal(st);
        k0 += pm[i] * pm[i];
      }
      for (uint64_t i = 0; i < d; ++i) xp[i] = x[i];
      for (int l = 0; l < k->leapfrog; ++l) {
        grad_vec(t, beta, xp, g, work);
        for (uint64_t i = 0; i < d; ++i) pm[i] += 0.5 * eps * g[i];
        for (uint64_t i = 0; i < d; ++i) xp[i] += eps * pm[i];
        grad_vec(t, beta, xp, g, work);
        for (uint64_t i = 0; i < d; ++i) pm[i] += 0.5 * eps * g[i];
      }
      double k1 = 0.0;
      for (uint64_t i = 0; i < d; ++i) k1 += pm[i] * pm[i];
      const double log_gamma_p = log_gamma(t, beta, xp);
      const double log_u = log(uniform(st));
      if (log_u < (log_gamma_p - log_gamma_x) + 0.5 * (k0 - k1)) {
        for (uint64_t i = 0; i < d; ++i) x[i] = xp[i];
        log_gamma_x = log_gamma_p;
      }
    }
  }
}

/* NEW kernel (no reference code): elliptical slice sampling w.r.t. the Gaussian
 * reference eta = N(mu, sigma^2 I) (Murray, Adams & MacKay 2010), include/asmc_b200.h
 * ASMC_KERNEL_SLICE.  Per update: nu ~ eta (d normals), log y = beta V(x) + log u,
 * theta ~ U[0, 2 pi), bracket [theta - 2 pi, theta]; x' = mu + (x - mu) cos + (nu - mu) sin,
 * accept iff beta V(x') > log y, else shrink toward 0 with a fresh uniform. */
static void slice_move(const asmc_target_desc* t, const asmc_kernel_desc* k, double beta, double* x,
                       double* scratch, stream_t* st) {
  const uint64_t d = t->dim;
  double* nu = scratch;
  double* xp = scratch + d;
  const double two_pi = 6.283185307179586476925286766559;
  const double mu = t->kind == ASMC_TARGET_GAUSSIAN_SHIFT ? t->p[0] : 0.0;
  for (int sweep = 0; sweep < k->sweeps; ++sweep) {
    sample_reference(t, st, nu);
    const double ll = beta == 0.0 ? 0.0 : beta * potential(t, x);
    const double log_y = ll + log(uniform(st));
    double theta = uniform(st) * two_pi;
    double lo = theta - two_pi, hi = theta;
    for (int it = 0; it < ASMC_SLICE_MAX_SHRINK; ++it) {
      const double c = cos(theta), sn = sin(theta);
      for (uint64_t i = 0; i < d; ++i) xp[i] = mu + (x[i] - mu) * c + (nu[i] - mu) * sn;
      const double llp = beta == 0.0 ? 0.0 : beta * potential(t, xp);
      if (llp > log_y) {
        for (uint64_t i = 0; i < d; ++i) x[i] = xp[i];
        break;
      }
      if (theta < 0.0) lo = theta;
      else hi = theta;
      theta = lo + (hi - lo) * uniform(st);
    }
  }
}

/* kernel.cpp:46-63 (+ the new HMC and slice branches) */
static int propagate(const asmc_target_desc* t, const asmc_kernel_desc* k, double beta, double* x,
                     double* scratch, stream_t* st) {
  switch (k->kind) {
    case ASMC_KERNEL_IDEALIZED: return exact_sample(t, beta, st, x);
    case ASMC_KERNEL_RWMH: rwmh_cycle_move(t, k, beta, x, scratch, st); return 0;
    case ASMC_KERNEL_HMC: hmc_cycle_move(t, k, beta, x, scratch, st); return 0;
    case ASMC_KERNEL_SLICE: slice_move(t, k, beta, x, scratch, st); return 0;
    default: return 0;
  }
}

/* kernel.cpp:65-73 */
static int log_incremental_weight(const asmc_target_desc* t, double b0, double b1, const double* x,
                                  double* out) {
  const double from = log_gamma(t, b0, x);
  if (from == -INFINITY)
    FAIL(ASMC_ERR_EVALUATION, "incremental weight undefined: gamma_beta(x) = 0 at beta = %f", b0);
  *out = log_gamma(t, b1, x) - from;
  return 0;
}

typedef struct { lacc_t g0, g1, g2, el; } step_acc_t;
static void step_acc_init(step_acc_t* a) { a->g0 = a->g1 = a->g2 = a->el = LACC0; }
static void step_acc_combine(step_acc_t* a, const step_acc_t* o) {
  lacc_combine(&a->g0, &o->g0);
  lacc_combine(&a->g1, &o->g1);
  lacc_combine(&a->g2, &o->g2);
  lacc_combine(&a->el, &o->el);
}

/* engine_detail.hpp:27-41 */
static int weight_and_move(const asmc_target_desc* t, const asmc_kernel_desc* k, double b0,
                           double b1, double* x, double* log_w, step_acc_t* acc, double* scratch,
                           stream_t* st) {
  double lg;
  TRY(log_incremental_weight(t, b0, b1, x, &lg));
  lacc_add(&acc->g0, *log_w);
  lacc_add(&acc->g1, *log_w + lg);
  lacc_add(&acc->g2, *log_w + 2.0 * lg);
  if (lg != 0.0) sacc_add(&acc->el, *log_w + log(fabs(lg)), lg > 0.0 ? 1.0 : -1.0);
  TRY(propagate(t, k, b1, x, scratch, st));
  *log_w += lg;
  return 0;
}

/* ------------------------------------------------------------- engine -- */
static int validate_schedule(const double* b, int T) { /* engine.cpp:29-39 */
  if (T < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "schedule needs at least one step");
  if (b[0] != 0.0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "schedule must start at beta = 0");
  if (b[T] != 1.0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "schedule must end at beta = 1");
  for (int t = 1; t <= T; ++t)
    if (!(b[t] > b[t - 1])) FAIL(ASMC_ERR_INVALID_ARGUMENT, "schedule must be strictly increasing at index %d", t);
  return 0;
}

#define KBLOCK 256 /* logsum.hpp:15 */
static uint64_t block_count(uint64_t n) { return n == 0 ? 0 : (n - 1) / KBLOCK + 1; }

/* engine.cpp:61-80 (sequential CDF) */
static int systematic_resample_seq(const double* lw, uint64_t n, double u, uint32_t* anc) {
  lacc_t a = LACC0;
  for (uint64_t i = 0; i < n; ++i) lacc_add(&a, lw[i]);
  const double l1 = lacc_total(&a);
  if (l1 == -INFINITY) FAIL(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  double cum = exp(lw[0] - l1);
  uint64_t j = 0;
  for (uint64_t m = 0; m < n; ++m) {
    const double pos = ((double)m + u) / (double)n;
    while (cum < pos && j + 1 < n) {
      ++j;
      cum += exp(lw[j] - l1);
    }
    anc[m] = (uint32_t)j;
  }
  return 0;
}

/* engine.cpp:61-80 with a given uniform (the reference draws u from key
 * (seed, round, 0, t, resample) inside systematic_resample) */
int ora_systematic_resample_u(const double* lw, uint64_t n, double u, uint32_t* anc) {
  if (n == 0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "cannot resample an empty system");
  return systematic_resample_seq(lw, n, u, anc);
}

/* The CDF systematic_resample walks (engine.cpp:64-75), every value: l1 =
 * logsumexp(lw) (logsum.hpp:97-101), cum_0 = exp(lw_0 - l1), cum_j = cum_{j-1} +
 * exp(lw_j - l1) in particle order. */
int ora_resample_cdf(const double* lw, uint64_t n, double* cum, double* l1_out) {
  if (n == 0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "cannot resample an empty system");
  lacc_t a = LACC0;
  for (uint64_t i = 0; i < n; ++i) lacc_add(&a, lw[i]);
  const double l1 = lacc_total(&a);
  if (l1_out) *l1_out = l1;
  if (l1 == -INFINITY) FAIL(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  double c = exp(lw[0] - l1);
  cum[0] = c;
  for (uint64_t j = 1; j < n; ++j) {
    c += exp(lw[j] - l1);
    cum[j] = c;
  }
  return 0;
}

/* the CDF for a given l1 (isolates the chain of adds from the one log) */
int ora_cdf_given_l1(const double* lw, uint64_t n, double l1, double* cum) {
  double c = exp(lw[0] - l1);
  cum[0] = c;
  for (uint64_t j = 1; j < n; ++j) {
    c += exp(lw[j] - l1);
    cum[j] = c;
  }
  return 0;
}

/* the host libm the reference links (glibc): which 0 = exp, 1 = log */
int ora_libm(int which, const double* x, uint64_t n, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = which == 0 ? exp(x[i]) : log(x[i]);
  return 0;
}

/* engine.cpp:82-95 */
static int decide_resample(int policy, int t, int T, double ess_v, uint64_t n, double dhat, double rho) {
  switch (policy) {
    case ASMC_POLICY_NEVER: return t == T;
    case ASMC_POLICY_ALWAYS: return 1;
    case ASMC_POLICY_ADAPTIVE_ESS: return ess_v < rho * (double)n;
    case ASMC_POLICY_STABILIZED: return dhat > -log(rho);
  }
  return 0;
}

/* schedule.cpp:27-31 */
static double discrepancy_hat_raw(double g0, double g1, double g2) {
  const double raw = g2 - 2.0 * g1 + g0;
  return raw > 0.0 ? raw : 0.0;
}

/* engine_detail.hpp:159-168 */
static int check_degenerate(uint64_t n, double ess_t, double m1, double m2, int t) {
  if (n > 1 && ess_t < 1.0 + 1e-9) {
    const double gap = m2 == -INFINITY ? INFINITY : m1 - m2;
    if (gap > 700.0)
      FAIL(ASMC_ERR_DEGENERATE, "weights degenerate at step %d (max log-weight %f)", t, m1);
  }
  return 0;
}

static int run_smc_impl(const asmc_target_desc* tg, const asmc_kernel_desc* k, const double* betas,
                        int T, uint64_t n, int policy, double rho, uint64_t seed, uint64_t round,
                        asmc_report* out) {
  TRY(validate_schedule(betas, T));
  if (n < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (!(rho >= 0.0 && rho <= 1.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "rho must lie in [0, 1]");
  TRY(validate_kernel(k));
  TRY(check_target(tg));
  const uint64_t d = tg->dim;
  const double log_n = log((double)n);
  double* xs = calloc(n * d, sizeof(double));
  double* xb = calloc(n * d, sizeof(double));
  double* lw = calloc(n, sizeof(double));
  double* scratch = calloc(5 * d, sizeof(double));  /* proposal / HMC (x', p, g, work) */
  uint32_t* anc = calloc(n, sizeof(uint32_t));
  int rc = 0;
  /* engine_detail.hpp:91-100 */
  for (uint64_t p = 0; p < n; ++p) {
    stream_t st;
    stream_init(&st, seed, round, p, 0, 0);
    sample_reference(tg, &st, xs + p * d);
  }
  for (int t = 0; t <= T; ++t) {
    if (out->log_g0) out->log_g0[t] = -INFINITY;
    if (out->log_g1) out->log_g1[t] = -INFINITY;
    if (out->log_g2) out->log_g2[t] = -INFINITY;
    if (out->ess_trace) out->ess_trace[t] = (double)n;
    if (out->cum_log_z) out->cum_log_z[t] = 0.0;
    if (out->resampled) out->resampled[t] = 0;
  }
  out->kernel_applications = 0;
  out->n_resample_times = 0;
  double log_z = 0.0, elbo = 0.0, acc_dhat = 0.0, den_log = log_n;
  const uint64_t nb = block_count(n);
  for (int t = 1; t <= T && !rc; ++t) {
    /* step_pass, engine_detail.hpp:113-156 */
    step_acc_t tot;
    step_acc_init(&tot);
    lacc_t sq_tot = LACC0;
    double max1 = -INFINITY, max2 = -INFINITY;
    for (uint64_t b = 0; b < nb && !rc; ++b) {
      step_acc_t a;
      step_acc_init(&a);
      lacc_t s2 = LACC0;
      double m1 = -INFINITY, m2 = -INFINITY;
      const uint64_t lo = b * KBLOCK, hi = lo + KBLOCK < n ? lo + KBLOCK : n;
      for (uint64_t p = lo; p < hi; ++p) {
        stream_t st;
        stream_init(&st, seed, round, p, (uint64_t)t, 1);
        rc = weight_and_move(tg, k, betas[t - 1], betas[t], xs + p * d, lw + p, &a, scratch, &st);
        if (rc) break;
        lacc_add(&s2, 2.0 * lw[p]);
        if (lw[p] > m1) { m2 = m1; m1 = lw[p]; }
        else if (lw[p] > m2) m2 = lw[p];
      }
      step_acc_combine(&tot, &a);
      lacc_combine(&sq_tot, &s2);
      if (m1 > max1) { max2 = max1 > m2 ? max1 : m2; max1 = m1; }
      else max2 = max2 > m1 ? max2 : m1;
    }
    if (rc) break;
    out->kernel_applications += n;
    const double g0 = lacc_total(&tot.g0), g1 = lacc_total(&tot.g1), g2 = lacc_total(&tot.g2);
    if (out->log_g0) out->log_g0[t] = g0;
    if (out->log_g1) out->log_g1[t] = g1;
    if (out->log_g2) out->log_g2[t] = g2;
    /* engine.cpp:140-188 */
    if (g1 == -INFINITY) { snprintf(g_err, sizeof g_err, "all log-weights are -inf at step %d", t); rc = ASMC_ERR_DEGENERATE; break; }
    double ess_t = exp(2.0 * g1 - lacc_total(&sq_tot));
    ess_t = fmin((double)n, fmax(1.0, ess_t));
    if (out->ess_trace) out->ess_trace[t] = ess_t;
    rc = check_degenerate(n, ess_t, max1, max2, t);
    if (rc) break;
    elbo += sacc_value_scaled(&tot.el, den_log);
    acc_dhat += discrepancy_hat_raw(g0, g1, g2);
    const int fire = decide_resample(policy, t, T, ess_t, n, acc_dhat, rho);
    const int select = fire && policy != ASMC_POLICY_NEVER;
    if (t == T || fire) {
      log_z += g1 - log_n;
      if (select) {
        stream_t rs;
        stream_init(&rs, seed, round, 0, (uint64_t)t, 2);
        const double u = uniform(&rs);
        rc = systematic_resample_seq(lw, n, u, anc);
        if (rc) break;
        for (uint64_t p = 0; p < n; ++p) memcpy(xb + p * d, xs + (uint64_t)anc[p] * d, d * sizeof(double));
        double* tmp = xs; xs = xb; xb = tmp;
        for (uint64_t p = 0; p < n; ++p) lw[p] = 0.0;
        if (out->resampled) out->resampled[t] = 1;
      }
      den_log = log_n;
      acc_dhat = 0.0;
      if (out->resample_times) out->resample_times[out->n_resample_times] = t;
      out->n_resample_times++;
    } else {
      den_log = g1;
    }
    if (out->cum_log_z) out->cum_log_z[t] = log_z;
  }
  out->log_z_hat = log_z;
  out->elbo_hat = elbo;
  out->wall_seconds = 0.0;
  free(xs); free(xb); free(lw); free(scratch); free(anc);
  return rc;
}

int ora_run_smc(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const double* betas,
                int32_t steps, uint64_t n, int32_t policy, double rho, uint64_t seed, uint64_t round,
                int32_t workers, asmc_report* out) {
  (void)workers;
  return run_smc_impl(target, kernel, betas, steps, n, policy, rho, seed, round, out);
}

/* drivers.cpp:72-182: per particle, init then t = 1..T into per-(block, t)
 * accumulators; ordered fold over blocks.  Bit-identical to run_smc(never). */
int ora_run_sais_single(const asmc_target_desc* tg, const asmc_kernel_desc* k, const double* betas,
                        int32_t T, uint64_t n, uint64_t seed, uint64_t round, int32_t workers,
                        uint64_t chunk, asmc_report* out) {
  (void)workers; (void)chunk;
  TRY(validate_schedule(betas, T));
  if (n < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  TRY(validate_kernel(k));
  TRY(check_target(tg));
  const uint64_t d = tg->dim;
  const double log_n = log((double)n);
  step_acc_t* glob = malloc((size_t)(T + 1) * sizeof(step_acc_t));
  step_acc_t* blk = malloc((size_t)(T + 1) * sizeof(step_acc_t));
  double* x = calloc(d, sizeof(double));
  double* scratch = calloc(5 * d, sizeof(double));  /* proposal / HMC (x', p, g, work) */
  for (int t = 0; t <= T; ++t) step_acc_init(&glob[t]);
  int rc = 0;
  const uint64_t nb = block_count(n);
  for (uint64_t b = 0; b < nb && !rc; ++b) {
    for (int t = 0; t <= T; ++t) step_acc_init(&blk[t]);
    const uint64_t lo = b * KBLOCK, hi = lo + KBLOCK < n ? lo + KBLOCK : n;
    for (uint64_t p = lo; p < hi && !rc; ++p) {
      stream_t si;
      stream_init(&si, seed, round, p, 0, 0);
      sample_reference(tg, &si, x);
      double log_w = 0.0;
      for (int t = 1; t <= T && !rc; ++t) {
        stream_t se;
        stream_init(&se, seed, round, p, (uint64_t)t, 1);
        rc = weight_and_move(tg, k, betas[t - 1], betas[t], x, &log_w, &blk[t], scratch, &se);
      }
    }
    for (int t = 1; t <= T; ++t) step_acc_combine(&glob[t], &blk[t]);
  }
  if (!rc) {
    for (int t = 0; t <= T; ++t) {
      if (out->log_g0) out->log_g0[t] = t ? lacc_total(&glob[t].g0) : -INFINITY;
      if (out->log_g1) out->log_g1[t] = t ? lacc_total(&glob[t].g1) : -INFINITY;
      if (out->log_g2) out->log_g2[t] = t ? lacc_total(&glob[t].g2) : -INFINITY;
      if (out->cum_log_z) out->cum_log_z[t] = 0.0;
      if (out->resampled) out->resampled[t] = 0;
    }
    for (int t = 1; t <= T; ++t)
      if (lacc_total(&glob[t].g1) == -INFINITY) {
        snprintf(g_err, sizeof g_err, "all log-weights are -inf at step %d", t);
        rc = ASMC_ERR_DEGENERATE;
        break;
      }
  }
  if (!rc) {
    double elbo = 0.0, den_log = log_n;
    for (int t = 1; t <= T; ++t) {
      elbo += sacc_value_scaled(&glob[t].el, den_log);
      den_log = lacc_total(&glob[t].g1);
    }
    const double log_z = lacc_total(&glob[T].g1) - log_n;
    if (out->cum_log_z) out->cum_log_z[T] = log_z;
    if (out->resample_times) out->resample_times[0] = T;
    out->n_resample_times = 1;
    out->log_z_hat = log_z;
    out->elbo_hat = elbo;
    out->wall_seconds = 0.0;
    out->kernel_applications = n * (uint64_t)T;
  }
  free(glob); free(blk); free(x); free(scratch);
  return rc;
}

/* engine_detail.hpp:27-41 driven per particle as in drivers.cpp:95-111 */
int ora_trajectory(const asmc_target_desc* tg, const asmc_kernel_desc* k, const double* betas,
                   int32_t T, uint64_t seed, uint64_t round, uint64_t particle, double* x_out,
                   double* lw_out, double* lg_out) {
  TRY(validate_kernel(k));
  TRY(check_target(tg));
  const uint64_t d = tg->dim;
  double* scratch = calloc(5 * d, sizeof(double));  /* proposal / HMC (x', p, g, work) */
  stream_t si;
  stream_init(&si, seed, round, particle, 0, 0);
  sample_reference(tg, &si, x_out);
  double log_w = 0.0;
  lw_out[0] = 0.0;
  if (lg_out) lg_out[0] = 0.0;
  int rc = 0;
  step_acc_t acc;
  step_acc_init(&acc);
  for (int t = 1; t <= T && !rc; ++t) {
    memcpy(x_out + (uint64_t)t * d, x_out + (uint64_t)(t - 1) * d, d * sizeof(double));
    stream_t se;
    stream_init(&se, seed, round, particle, (uint64_t)t, 1);
    const double before = log_w;
    rc = weight_and_move(tg, k, betas[t - 1], betas[t], x_out + (uint64_t)t * d, &log_w, &acc, scratch, &se);
    lw_out[t] = log_w;
    if (lg_out) lg_out[t] = log_w - before;
  }
  free(scratch);
  return rc;
}

int ora_rng_u64(const uint64_t key[5], uint64_t count, uint64_t* out) {
  stream_t s;
  stream_init(&s, key[0], key[1], key[2], key[3], key[4]);
  for (uint64_t i = 0; i < count; ++i) out[i] = next_u64(&s);
  return 0;
}
int ora_rng_uniform(const uint64_t key[5], uint64_t count, double* out) {
  stream_t s;
  stream_init(&s, key[0], key[1], key[2], key[3], key[4]);
  for (uint64_t i = 0; i < count; ++i) out[i] = uniform(&s);
  return 0;
}
int ora_rng_normal(const uint64_t key[5], uint64_t count, double* out) {
  stream_t s;
  stream_init(&s, key[0], key[1], key[2], key[3], key[4]);
  for (uint64_t i = 0; i < count; ++i) out[i] = normal(&s);
  return 0;
}

int ora_systematic_resample(const double* lw, uint64_t n, const uint64_t key[5], uint32_t* out) {
  if (n == 0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "cannot resample an empty system");
  stream_t s;
  stream_init(&s, key[0], key[1], key[2], key[3], key[4]);
  /* engine.cpp:65-68: l1 is checked before the uniform is drawn */
  lacc_t a = LACC0;
  for (uint64_t i = 0; i < n; ++i) lacc_add(&a, lw[i]);
  if (lacc_total(&a) == -INFINITY) FAIL(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  return systematic_resample_seq(lw, n, uniform(&s), out);
}

/* engine.cpp:46-59 */
int ora_ess(const double* lw, uint64_t n, double* out) {
  if (n == 0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "ess of empty weight vector");
  lacc_t l1 = LACC0, l2 = LACC0;
  for (uint64_t i = 0; i < n; ++i) {
    lacc_add(&l1, lw[i]);
    lacc_add(&l2, 2.0 * lw[i]);
  }
  if (lacc_total(&l1) == -INFINITY) FAIL(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  const double e = exp(2.0 * lacc_total(&l1) - lacc_total(&l2));
  *out = fmin((double)n, fmax(1.0, e));
  return 0;
}

/* ----------------------------------------------------------- schedule -- */
/* schedule.cpp:41-56 */
int ora_barrier_estimate(const double* g0, const double* g1, const double* g2, const double* betas,
                         int32_t T, double* lambda) {
  TRY(validate_schedule(betas, T));
  lambda[0] = 0.0;
  for (int t = 1; t <= T; ++t) {
    if (g0[t] == -INFINITY) FAIL(ASMC_ERR_INVALID_ARGUMENT, "no increment statistics recorded for step %d", t);
    lambda[t] = lambda[t - 1] + sqrt(discrepancy_hat_raw(g0[t], g1[t], g2[t]));
  }
  return 0;
}

/* schedule.cpp:58-90 (Fritsch-Carlson slopes) */
static int mono_init(const double* x, const double* y, int n, double* m) {
  if (n < 2) FAIL(ASMC_ERR_INVALID_ARGUMENT, "interpolant needs at least two matched knots");
  for (int i = 1; i < n; ++i)
    if (!(x[i] > x[i - 1])) FAIL(ASMC_ERR_INVALID_ARGUMENT, "interpolant abscissae must be strictly increasing");
  double* h = malloc(sizeof(double) * (size_t)(n - 1));
  double* d = malloc(sizeof(double) * (size_t)(n - 1));
  for (int i = 0; i + 1 < n; ++i) {
    h[i] = x[i + 1] - x[i];
    d[i] = (y[i + 1] - y[i]) / h[i];
  }
  m[0] = d[0];
  m[n - 1] = d[n - 2];
  for (int i = 1; i + 1 < n; ++i) {
    if (d[i - 1] == 0.0 || d[i] == 0.0 || (d[i - 1] > 0.0) != (d[i] > 0.0)) {
      m[i] = 0.0;
    } else {
      const double w1 = 2.0 * h[i] + h[i - 1];
      const double w2 = h[i] + 2.0 * h[i - 1];
      m[i] = (w1 + w2) / (w1 / d[i - 1] + w2 / d[i]);
    }
  }
  free(h); free(d);
  return 0;
}
static int upper_idx(const double* x, int n, double q) { /* std::upper_bound - 1 */
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = lo + (hi - lo) / 2;
    if (q < x[mid]) hi = mid; else lo = mid + 1;
  }
  return lo - 1;
}
/* schedule.cpp:92-106 */
static double mono_eval(const double* x, const double* y, const double* m, int n, double q) {
  if (q <= x[0]) return y[0] + m[0] * (q - x[0]);
  if (q >= x[n - 1]) return y[n - 1] + m[n - 1] * (q - x[n - 1]);
  const int i = upper_idx(x, n, q);
  const double h = x[i + 1] - x[i];
  const double s = (q - x[i]) / h;
  const double s2 = s * s;
  const double s3 = s2 * s;
  const double h00 = 2.0 * s3 - 3.0 * s2 + 1.0;
  const double h10 = s3 - 2.0 * s2 + s;
  const double h01 = -2.0 * s3 + 3.0 * s2;
  const double h11 = s3 - s2;
  return h00 * y[i] + h10 * h * m[i] + h01 * y[i + 1] + h11 * h * m[i + 1];
}
/* schedule.cpp:108-117 */
static double mono_deriv(const double* x, const double* y, const double* m, int n, double q) {
  if (q <= x[0]) return m[0];
  if (q >= x[n - 1]) return m[n - 1];
  const int i = upper_idx(x, n, q);
  const double h = x[i + 1] - x[i];
  const double s = (q - x[i]) / h;
  const double s2 = s * s;
  const double g00 = (6.0 * s2 - 6.0 * s) / h;
  const double g10 = 3.0 * s2 - 4.0 * s + 1.0;
  const double g01 = (-6.0 * s2 + 6.0 * s) / h;
  const double g11 = 3.0 * s2 - 2.0 * s;
  return g00 * y[i] + g10 * m[i] + g01 * y[i + 1] + g11 * m[i + 1];
}

/* schedule.cpp:121-141 */
static int validate_barrier(const double* lambda, const double* beta, int n) {
  if (n < 2) FAIL(ASMC_ERR_INVALID_ARGUMENT, "barrier estimate needs at least two matched knots");
  if (lambda[0] != 0.0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "barrier estimate must start at Lambda = 0");
  if (beta[0] != 0.0 || beta[n - 1] != 1.0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "barrier estimate must span beta in [0, 1]");
  for (int i = 1; i < n; ++i) {
    if (lambda[i] < lambda[i - 1]) FAIL(ASMC_ERR_INVALID_ARGUMENT, "barrier knots must be nondecreasing");
    if (!(beta[i] > beta[i - 1])) FAIL(ASMC_ERR_INVALID_ARGUMENT, "barrier beta knots must be strictly increasing");
  }
  return 0;
}

/* schedule.cpp:144-187 */
int ora_generate_schedule(const double* lambda, const double* beta, int32_t knots, int32_t t_new,
                          double* out) {
  TRY(validate_barrier(lambda, beta, knots));
  if (t_new < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "schedule needs at least one step");
  const double total = lambda[knots - 1];
  int uniform_fallback = total == 0.0;
  double* xs = malloc(sizeof(double) * (size_t)knots);
  double* ys = malloc(sizeof(double) * (size_t)knots);
  double* m = malloc(sizeof(double) * (size_t)knots);
  int cnt = 0;
  if (!uniform_fallback) {
    for (int i = 0; i < knots; ++i) {
      if (cnt > 0 && lambda[i] == xs[cnt - 1]) {
        ys[cnt - 1] = beta[i];
      } else {
        xs[cnt] = lambda[i];
        ys[cnt] = beta[i];
        ++cnt;
      }
    }
    if (cnt < 2) uniform_fallback = 1;
  }
  int rc = 0;
  if (uniform_fallback) { /* engine.cpp:16-27 */
    for (int t = 0; t <= t_new; ++t) out[t] = (double)t / (double)t_new;
    out[0] = 0.0;
    out[t_new] = 1.0;
  } else {
    rc = mono_init(xs, ys, cnt, m);
    if (!rc) {
      out[0] = 0.0;
      out[t_new] = 1.0;
      for (int t = 1; t < t_new; ++t) {
        const double q = total * (double)t / (double)t_new;
        double b = mono_eval(xs, ys, m, cnt, q);
        b = fmin(1.0, fmax(0.0, b));
        out[t] = b;
      }
      for (int t = 1; t < t_new; ++t)
        if (out[t] <= out[t - 1]) out[t] = nextafter(out[t - 1], 1.0);
      for (int t = t_new - 1; t >= 1; --t)
        if (out[t] >= out[t + 1]) out[t] = nextafter(out[t + 1], 0.0);
      rc = validate_schedule(out, t_new);
    }
  }
  free(xs); free(ys); free(m);
  return rc;
}

/* schedule.cpp:189-197 */
int ora_local_barrier(const double* lambda, const double* beta, int32_t knots, double* out) {
  TRY(validate_barrier(lambda, beta, knots));
  double* m = malloc(sizeof(double) * (size_t)knots);
  int rc = mono_init(beta, lambda, knots, m);
  if (!rc)
    for (int i = 0; i < knots; ++i) out[i] = mono_deriv(beta, lambda, m, knots, beta[i]);
  free(m);
  return rc;
}

/* drivers.cpp:33-49 */
int ora_budget(uint64_t n, int32_t steps, uint64_t dim, uint64_t cap, int32_t mode, uint64_t* n_out,
               int32_t* t_out) {
  if (n < 1 || steps < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "budget needs n_particles and steps >= 1");
  const double root2 = sqrt(2.0);
  const uint64_t gn = (uint64_t)ceil(root2 * (double)n);
  const int gt = (int)ceil(root2 * (double)steps);
  if (mode == ASMC_MODE_SSMC) {
    const double bytes = (double)gn * (double)dim * 8.0;
    if (bytes > (double)cap) {
      *n_out = n;
      *t_out = 2 * steps;
      return 0;
    }
  }
  *n_out = gn;
  *t_out = gt;
  return 0;
}

/* drivers.cpp:186-220 */
int ora_run_rounds(const asmc_target_desc* tg, const asmc_kernel_desc* k, int32_t mode, uint64_t n,
                   int32_t rounds, int32_t policy, double rho, uint64_t seed, uint64_t cap,
                   int32_t workers, asmc_rounds_out* out) {
  (void)workers;
  if (n < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (rounds < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "rounds must be at least 1");
  if (!(rho >= 0.0 && rho <= 1.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "rho must lie in [0, 1]");
  const int stride = out->max_steps + 1;
  double* sched = malloc(sizeof(double) * (size_t)stride);
  double* g0 = malloc(sizeof(double) * (size_t)stride);
  double* g1 = malloc(sizeof(double) * (size_t)stride);
  double* g2 = malloc(sizeof(double) * (size_t)stride);
  double* ess = malloc(sizeof(double) * (size_t)stride);
  double* cz = malloc(sizeof(double) * (size_t)stride);
  uint8_t* rs = malloc((size_t)stride);
  int32_t* rt = malloc(sizeof(int32_t) * (size_t)stride);
  double* lam = malloc(sizeof(double) * (size_t)stride);
  int steps = 1, rc = 0;
  sched[0] = 0.0;
  sched[1] = 1.0;
  for (int kk = 1; kk <= rounds && !rc; ++kk) {
    if (steps > out->max_steps) { snprintf(g_err, sizeof g_err, "max_steps too small"); rc = ASMC_ERR_INVALID_ARGUMENT; break; }
    asmc_report rep = {g0, g1, g2, ess, cz, rs, rt, 0, 0, 0, 0, 0, 0};
    rc = mode == ASMC_MODE_SAIS
             ? ora_run_sais_single(tg, k, sched, steps, n, seed, (uint64_t)kk, 1, 0, &rep)
             : ora_run_smc(tg, k, sched, steps, n, policy, rho, seed, (uint64_t)kk, 1, &rep);
    if (rc) break;
    rc = ora_barrier_estimate(g0, g1, g2, sched, steps, lam);
    if (rc) break;
    const size_t r0 = (size_t)(kk - 1) * (size_t)stride;
    if (out->n_particles) out->n_particles[kk - 1] = n;
    if (out->steps) out->steps[kk - 1] = steps;
    for (int t = 0; t <= steps; ++t) {
      if (out->betas) out->betas[r0 + t] = sched[t];
      if (out->log_g0) out->log_g0[r0 + t] = g0[t];
      if (out->log_g1) out->log_g1[r0 + t] = g1[t];
      if (out->log_g2) out->log_g2[r0 + t] = g2[t];
      if (out->ess_trace && mode == ASMC_MODE_SSMC) out->ess_trace[r0 + t] = ess[t];
      if (out->cum_log_z) out->cum_log_z[r0 + t] = cz[t];
      if (out->resampled) out->resampled[r0 + t] = rs[t];
      if (out->lambda) out->lambda[r0 + t] = lam[t];
    }
    if (out->log_z_hat) out->log_z_hat[kk - 1] = rep.log_z_hat;
    if (out->elbo_hat) out->elbo_hat[kk - 1] = rep.elbo_hat;
    if (out->wall_seconds) out->wall_seconds[kk - 1] = 0.0;
    if (out->kernel_applications) out->kernel_applications[kk - 1] = rep.kernel_applications;
    if (kk < rounds) {
      uint64_t nn;
      int tt;
      ora_budget(n, steps, tg->dim, cap, mode, &nn, &tt);
      if (tt > out->max_steps) { snprintf(g_err, sizeof g_err, "max_steps too small"); rc = ASMC_ERR_INVALID_ARGUMENT; break; }
      double* ns = malloc(sizeof(double) * (size_t)(tt + 1));
      rc = ora_generate_schedule(lam, sched, steps + 1, tt, ns);
      if (!rc) memcpy(sched, ns, sizeof(double) * (size_t)(tt + 1));
      free(ns);
      n = nn;
      steps = tt;
    }
  }
  free(sched); free(g0); free(g1); free(g2); free(ess); free(cz); free(rs); free(rt); free(lam);
  return rc;
}

int ora_hardware_threads(void) { return 1; }

/* ---------------------------------------------------------------- ZJA -- */
/* schedule.cpp:201-215 */
static int zja_dhat(const asmc_target_desc* tg, double beta, double b2, const double* xs, uint64_t n,
                    const double* lw, double log_m0, double* out) {
  lacc_t m1 = LACC0, m2 = LACC0;
  for (uint64_t p = 0; p < n; ++p) {
    double lg;
    TRY(log_incremental_weight(tg, beta, b2, xs + p * tg->dim, &lg));
    lacc_add(&m1, lw[p] + lg);
    lacc_add(&m2, lw[p] + 2.0 * lg);
  }
  const double raw = lacc_total(&m2) - 2.0 * lacc_total(&m1) + log_m0;
  *out = raw > 0.0 ? raw : 0.0;
  return 0;
}

static int zja_bisect(const asmc_target_desc* tg, double beta, const double* xs, uint64_t n, const double* lw,
                      double log_m0, double delta, double tol, double lo, double hi, double* out) {
  while (hi - lo > tol) {
    const double mid = 0.5 * (lo + hi);
    double dh;
    TRY(zja_dhat(tg, beta, mid, xs, n, lw, log_m0, &dh));
    if (dh <= delta) lo = mid;
    else hi = mid;
  }
  *out = lo;
  return 0;
}

/* schedule.cpp:219-264 */
int ora_zja_next_beta(const asmc_target_desc* tg, double beta, const double* xs, uint64_t n, const double* lw,
                      double delta, double tol, double* beta_next, int32_t* warning) {
  if (!(beta >= 0.0 && beta < 1.0)) FAIL(ASMC_ERR_DOMAIN, "zja_next_beta requires beta in [0, 1)");
  if (!(delta > 0.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "delta_star must be positive");
  if (!(tol > 0.0)) FAIL(ASMC_ERR_INVALID_ARGUMENT, "tol must be positive");
  if (n == 0) FAIL(ASMC_ERR_INVALID_ARGUMENT, "particle arrays inconsistent with n_particles");
  TRY(check_target(tg));
  lacc_t m0 = LACC0;
  for (uint64_t p = 0; p < n; ++p) lacc_add(&m0, lw[p]);
  const double log_m0 = lacc_total(&m0);
  if (log_m0 == -INFINITY) FAIL(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  if (warning) *warning = 0;
  double dh;
  TRY(zja_dhat(tg, beta, 1.0, xs, n, lw, log_m0, &dh));
  if (dh <= delta) {
    *beta_next = 1.0;
    return 0;
  }
  double root;
  TRY(zja_bisect(tg, beta, xs, n, lw, log_m0, delta, tol, beta, 1.0, &root));
  for (int i = 1; i < 16; ++i) {
    const double probe = beta + (root - beta) * (double)i / 16;
    TRY(zja_dhat(tg, beta, probe, xs, n, lw, log_m0, &dh));
    if (dh > delta * (1.0 + 1e-12)) {
      if (warning) *warning = 1;
      return zja_bisect(tg, beta, xs, n, lw, log_m0, delta, tol, beta, probe, beta_next);
    }
  }
  *beta_next = root;
  return 0;
}

/* drivers.cpp:234-341 */
int ora_run_zja(const asmc_target_desc* tg, const asmc_kernel_desc* k, const asmc_zja_opts* o, int32_t workers,
                asmc_zja_out* out) {
  (void)workers;
  if (o->n_particles < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (o->target_steps < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "target_steps must be at least 1");
  if (o->max_steps < 1) FAIL(ASMC_ERR_INVALID_ARGUMENT, "max_steps must be at least 1");
  if (!(o->delta_star >= 0.0) || !isfinite(o->delta_star))
    FAIL(ASMC_ERR_INVALID_ARGUMENT, "delta_star must be finite and >= 0");
  TRY(validate_kernel(k));
  TRY(check_target(tg));
  const uint64_t n = o->n_particles, d = tg->dim;
  double delta = o->delta_star;
  uint64_t main_round = 1;
  out->pilot_ran = 0;
  out->warning = 0;
  if (delta <= 0.0) {
    const int K = o->target_steps;
    double* pb = malloc((size_t)(K + 1) * sizeof(double));
    double* lam = malloc((size_t)(K + 1) * sizeof(double));
    for (int t = 0; t <= K; ++t) pb[t] = (double)t / (double)K;
    pb[0] = 0.0;
    pb[K] = 1.0;
    int rc = run_smc_impl(tg, k, pb, K, n, ASMC_POLICY_NEVER, 0.5, o->seed, 1, &out->pilot);
    if (!rc) rc = ora_barrier_estimate(out->pilot.log_g0, out->pilot.log_g1, out->pilot.log_g2, pb, K, lam);
    if (!rc) {
      if (out->pilot_lambda) memcpy(out->pilot_lambda, lam, (size_t)(K + 1) * sizeof(double));
      const double step_lam = lam[K] / (double)K;
      delta = step_lam * step_lam > 1e-12 ? step_lam * step_lam : 1e-12;
    }
    free(pb);
    free(lam);
    TRY(rc);
    out->pilot_ran = 1;
    main_round = 2;
  }
  out->delta_star = delta;
  const int cap = o->max_steps;
  double* xs = calloc(n * d, sizeof(double));
  double* lw = calloc(n, sizeof(double));
  double* scratch = calloc(5 * d, sizeof(double));
  double* betas = calloc((size_t)cap + 1, sizeof(double));
  double* g0 = malloc(((size_t)cap + 1) * sizeof(double));
  double* g1 = malloc(((size_t)cap + 1) * sizeof(double));
  double* g2 = malloc(((size_t)cap + 1) * sizeof(double));
  asmc_report* r = &out->main;
  for (uint64_t p = 0; p < n; ++p) {
    stream_t st;
    stream_init(&st, o->seed, main_round, p, 0, 0);
    sample_reference(tg, &st, xs + p * d);
  }
  g0[0] = g1[0] = g2[0] = -INFINITY;
  const double log_n = log((double)n);
  double log_z = 0.0, elbo = 0.0, den_log = log_n;
  int rc = 0, t = 0;
  const uint64_t nb = block_count(n);
  r->n_resample_times = 0;
  if (r->ess_trace) r->ess_trace[0] = (double)n;
  if (r->cum_log_z) r->cum_log_z[0] = 0.0;
  if (r->resampled) r->resampled[0] = 0;
  while (betas[t] < 1.0 && !rc) {
    ++t;
    if (t > cap) {
      snprintf(g_err, sizeof g_err, "online adaptation failed to reach beta = 1 within %d steps", cap);
      rc = ASMC_ERR_EVALUATION;
      break;
    }
    int32_t w = 0;
    rc = ora_zja_next_beta(tg, betas[t - 1], xs, n, lw, delta, 1e-10, &betas[t], &w);
    if (rc) break;
    out->warning |= w;
    /* step_pass (engine_detail.hpp:113-156) from betas[t-1] to betas[t] */
    step_acc_t tot;
    step_acc_init(&tot);
    lacc_t sq_tot = LACC0;
    double max1 = -INFINITY, max2 = -INFINITY;
    for (uint64_t b = 0; b < nb && !rc; ++b) {
      step_acc_t a;
      step_acc_init(&a);
      lacc_t s2 = LACC0;
      double m1 = -INFINITY, m2 = -INFINITY;
      const uint64_t lo = b * KBLOCK, hi = lo + KBLOCK < n ? lo + KBLOCK : n;
      for (uint64_t p = lo; p < hi; ++p) {
        stream_t st;
        stream_init(&st, o->seed, main_round, p, (uint64_t)t, 1);
        rc = weight_and_move(tg, k, betas[t - 1], betas[t], xs + p * d, lw + p, &a, scratch, &st);
        if (rc) break;
        lacc_add(&s2, 2.0 * lw[p]);
        if (lw[p] > m1) { m2 = m1; m1 = lw[p]; }
        else if (lw[p] > m2) m2 = lw[p];
      }
      step_acc_combine(&tot, &a);
      lacc_combine(&sq_tot, &s2);
      if (m1 > max1) { max2 = max1 > m2 ? max1 : m2; max1 = m1; }
      else max2 = max2 > m1 ? max2 : m1;
    }
    if (rc) break;
    g0[t] = lacc_total(&tot.g0);
    g1[t] = lacc_total(&tot.g1);
    g2[t] = lacc_total(&tot.g2);
    if (g1[t] == -INFINITY) { snprintf(g_err, sizeof g_err, "all log-weights are -inf at step %d", t); rc = ASMC_ERR_DEGENERATE; break; }
    double ess_t = exp(2.0 * g1[t] - lacc_total(&sq_tot));
    ess_t = fmin((double)n, fmax(1.0, ess_t));
    if (r->ess_trace) r->ess_trace[t] = ess_t;
    rc = check_degenerate(n, ess_t, max1, max2, t);
    if (rc) break;
    elbo += sacc_value_scaled(&tot.el, den_log);
    if (betas[t] == 1.0) {
      log_z += g1[t] - log_n;
      den_log = log_n;
      if (r->resample_times) r->resample_times[r->n_resample_times] = t;
      r->n_resample_times++;
    } else {
      den_log = g1[t];
    }
    if (r->cum_log_z) r->cum_log_z[t] = log_z;
    if (r->resampled) r->resampled[t] = 0;
  }
  if (!rc && t + 1 > out->capacity) {
    snprintf(g_err, sizeof g_err, "output capacity too small (%d needed)", t + 1);
    rc = ASMC_ERR_INVALID_ARGUMENT;
  }
  if (!rc) {
    out->steps = t;
    for (int i = 0; i <= t; ++i) {
      if (r->log_g0) r->log_g0[i] = g0[i];
      if (r->log_g1) r->log_g1[i] = g1[i];
      if (r->log_g2) r->log_g2[i] = g2[i];
      if (out->betas) out->betas[i] = betas[i];
    }
    r->log_z_hat = log_z;
    r->elbo_hat = elbo;
    r->kernel_applications = n * (uint64_t)t;
    r->wall_seconds = 0.0;
    if (out->lambda) {
      out->lambda[0] = 0.0;
      for (int i = 1; i <= t; ++i) out->lambda[i] = out->lambda[i - 1] + sqrt(discrepancy_hat_raw(g0[i], g1[i], g2[i]));
    }
  }
  free(xs); free(lw); free(scratch); free(betas); free(g0); free(g1); free(g2);
  return rc;
}
