// Device target plugins: per-coordinate terms of the product-form annealing
// families  log gamma_beta(x) = log eta(x) + beta V(x).
//
// Two arithmetic contracts per target:
//  * fp64 "reference" terms (lr64, v64, draws) reproduce the reference's
//    expressions operation for operation (src/target.cpp:16-19, 57-157 and the
//    config-2 plugin in oracle/ref_harness.cpp).  Logs of parameters are
//    precomputed on the host with glibc so they are the reference's bits.
//  * fp32 "fast" terms: the MH log-ratio in difference form
//    f_beta(x + h) - f_beta(x) (no cancellation of two large absolute log
//    densities), and the potential's x-dependent part for the weight.
#pragma once

#include <math.h>
#include <stdint.h>

namespace asmcdev {

constexpr double kLogSqrt2Pi = 0.91893853320467274178;  // src/target.cpp:13

// log2 on the SFU (lg2.approx: ~2^-22 absolute on [0.5, 2), relative elsewhere)
__device__ __forceinline__ float sfu_lg2(float v) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

struct TgtParams {
  int kind;
  int pad;
  uint64_t dim;
  double p[8];
  double c[8];  // host-precomputed constants (see host make_params)
  float f[16];  // host-precomputed beta-independent fp32 constants (TgtMixture::F32)
};

// target.cpp:16-19 with log(sigma) supplied.  A power-of-two sigma (every configured target)
// divides exactly by scaling: the multiply by 2^-k rounds the same exact value as the
// division, so the bits are the reference's (an fp64 division is ~20 instructions)
__device__ __forceinline__ double lnpdf64(double x, double mu, double sigma, double log_sigma) {
  const long long b = __double_as_longlong(sigma);
  const int ex = (int)((b >> 52) & 0x7ff);
  const bool pow2 = (b & 0x000FFFFFFFFFFFFFll) == 0 && ex > 1 && ex < 0x7fe && b > 0;
  const double dx = x - mu;
  const double s = pow2 ? dx * __drcp_rn(sigma) : dx / sigma;
  return -0.5 * s * s - log_sigma - kLogSqrt2Pi;
}

// ------------------------------------------------- GaussianShiftTarget --
// p = {mu0, mu1, sigma}; c = {log sigma, a, mid, 1/sigma^2}
struct TgtGaussShift {
  static constexpr bool kExact = true;
  static constexpr bool kCacheV = false;
  __device__ static double lr64(const TgtParams& T, double x) {
    return lnpdf64(x, T.p[0], T.p[2], T.c[0]);
  }
  __device__ static double v64(const TgtParams& T, double x) { return T.c[1] * (x - T.c[2]); }
  __device__ static double ref_draw(const TgtParams& T, double n) { return T.p[0] + T.p[2] * n; }
  // fp32 paths: the same draw without the float -> double -> float round trip
  __device__ static float ref_draw32(const TgtParams& T, float n) { return fmaf((float)T.p[2], n, (float)T.p[0]); }
  // target.cpp:107-113: mu computed once, then mu + sigma * normal
  __device__ static double exact_mu(const TgtParams& T, double beta) {
    return (1.0 - beta) * T.p[0] + beta * T.p[1];
  }
  __device__ static double exact_draw(const TgtParams& T, double mu, double n) {
    return mu + T.p[2] * n;
  }
  // fp32 fast path ----------------------------------------------------
  struct F32 {
    float mu0, inv_s2, ba;  // ba = beta * a
  };
  __device__ static F32 f32(const TgtParams& T, double beta) {
    return F32{(float)T.p[0], (float)T.c[3], (float)(beta * T.c[1])};
  }
  // f(x+h) - f(x) = h * (beta a - (x - mu0 + h/2) / sigma^2)
  __device__ static float dlg(const F32& k, float x, float h) {
    return h * (k.ba - (x - k.mu0 + 0.5f * h) * k.inv_s2);
  }
  // d/dx log gamma_beta (oracle/restate.c:grad_log_gamma)
  __device__ static double grad64(const TgtParams& T, double beta, double x) {
    return -(x - T.p[0]) / (T.p[2] * T.p[2]) + beta * T.c[1];
  }
  __device__ static float grad32(const F32& k, float x) { return fmaf(-(x - k.mu0), k.inv_s2, k.ba); }
  __device__ static float vpart(const F32&, float x) { return x; }
  // early rejection: max over h of dlg(x, h) (a concave quadratic in h)
  static constexpr bool kEarly = true;
  static constexpr unsigned kCheckMask = 0x7Fu;  // early-rejection checks after quad-iterations 0..6
  static constexpr bool kPerProposalCheck = false;
  static constexpr bool kBoundFromV = false;
  static constexpr bool kQuadMH = false;
  __device__ static float bound_of_v(const F32&, float) { return 0.f; }
  __device__ static float dmax(const F32& k, float x, float) {
    const float g = k.ba - (x - k.mu0) * k.inv_s2;
    return __fdividef(0.5f * g * g, k.inv_s2);
  }
  // V = a * (sum x - d * mid)
  __device__ static double v_from(const TgtParams& T, double s) {
    return T.c[1] * (s - (double)T.dim * T.c[2]);
  }
};

// ------------------------------------------------------ MixtureTarget --
// p = {ref_sigma, w, mu1, s1, mu2, s2}; c = {log ref_sigma, log w, log1p(-w), log s1, log s2}
struct TgtMixture {
  static constexpr bool kExact = false;
  static constexpr bool kCacheV = true;  // smem pass keeps vterm(x_i) beside x_i
  __device__ static double lr64(const TgtParams& T, double x) {
    return lnpdf64(x, 0.0, T.p[0], T.c[0]);
  }
  // target.cpp:139-152
  __device__ static double v64(const TgtParams& T, double x) {
    const double a = T.c[1] + lnpdf64(x, T.p[2], T.p[3], T.c[3]);
    const double b = T.c[2] + lnpdf64(x, T.p[4], T.p[5], T.c[4]);
    const double hi = a > b ? a : b;
    const double lo = a > b ? b : a;
    const double log_mix = hi + log1p(exp(lo - hi));
    return log_mix - lnpdf64(x, 0.0, T.p[0], T.c[0]);
  }
  __device__ static double ref_draw(const TgtParams& T, double n) { return T.p[0] * n; }
  __device__ static float ref_draw32(const TgtParams& T, float n) { return (float)T.p[0] * n; }
  __device__ static double exact_mu(const TgtParams&, double) { return 0.0; }
  __device__ static double exact_draw(const TgtParams&, double, double n) { return n; }
  // fp32 ----------------------------------------------------------------
  struct F32 {
    float beta, inv_r, lw1, mu1, inv_s1, lw2, mu2, inv_s2;
    float lmix;  // log(e^lw1 + e^lw2) >= hi + log1p(e^(lo-hi)) for every x (early rejection)
    // vterm in base-2 units: u_k = x c_k + d_k = sqrt(log2(e)/2) (x - mu_k)/s_k,
    // a_k = L_k - u_k^2 = log2(e) (lw_k - ((x - mu_k)/s_k)^2 / 2), kr = log2(e) / (2 r^2)
    float c1, d1, c2, d2, L1, L2, kr;
    float hr;  // 1 / (2 r^2)
  };
  // every field but beta is beta-independent: the host folds them once per call
  // (capi.cu make_params -> TgtParams::f, in this order); per (particle, step) only beta
  // is set -- no fp64 log1p / exp / sqrt / divisions on the device
  __device__ static F32 f32(const TgtParams& T, double beta) {
    return F32{(float)beta, T.f[0], T.f[1], T.f[2], T.f[3], T.f[4], T.f[5], T.f[6], T.f[7],
               T.f[8], T.f[9], T.f[10], T.f[11], T.f[12], T.f[13], T.f[14], T.f[15]};
  }
  // early rejection: f_beta(y) = beta (hi + log1p) - (1 - beta) sr^2 / 2 <= beta lmix, so
  // max_h dlg(x, h) <= beta (lmix - vterm(x)) + sr(x)^2 / 2  (v = the cached vterm(x))
  // one check, after the first quad-iteration (c0 = 4G coordinates), and only for the
  // proposals it can plausibly reject (early_worth; warp-uniform, a cost heuristic --
  // the check is exact whenever it runs): the large steps of a {0.1, 1, 10} cycle, whose
  // per-coordinate drop s^2 ((1 - beta) / 2r^2 + beta / 2 sigma_min^2) summed over the
  // first c0 coordinates already exceeds ~1 per remaining coordinate of the bound.
  // A/B on config 3 (tools/c3_drawn.py, ab_libs.py): checking every proposal at every
  // quad-iteration draws 31 % fewer normals but issues 2.5 % more instructions (+1.2 %
  // p-steps/s: per-coordinate bound terms, re-bounding after every accept, the vote
  // between the interleaved Philox chains); this form +8 %; one predicted check per
  // proposal at a runtime iteration (also catching the unit step near beta = 1) 0 %.
  static constexpr bool kEarly = true;
  static constexpr unsigned kCheckMask = 0x01u;
  static constexpr bool kPerProposalCheck = true;
  // sum of dmax over n coordinates from their sums: beta (n lmix - sum v) + sum x^2 / 2r^2
  __device__ static float bound_of_sums(const F32& k, int n, float vsum, float x2sum) {
    return fmaf(k.beta, fmaf((float)n, k.lmix, -vsum), k.hr * x2sum);
  }
  __device__ static bool early_worth(const F32& k, float s, int d, int c0) {
    const float is = fminf(k.inv_s1, k.inv_s2);
    const float drop = s * s * fmaf(k.beta, 0.5f * is * is - k.hr, k.hr);
    return (float)c0 * drop > (float)(d - c0);
  }
  static constexpr bool kBoundFromV = false;
  static constexpr bool kQuadMH = false;
  __device__ static float bound_of_v(const F32&, float) { return 0.f; }
  __device__ static float dmax(const F32& k, float x, float v) {
    const float sr = x * k.inv_r;
    return fmaf(k.beta, k.lmix - v, 0.5f * sr * sr);
  }
  // log_mix(x) - log eta(x) with the common -log(sqrt(2 pi)) - log(ref_sigma) folded out.
  // log1p(e^{lo-hi}) with lo <= hi: the MUFU ex2/lg2 pair is accurate to ~2e-7
  // absolute on (0, ln 2] (no cancellation: the argument of lg2 is in [1, 2]).
  // Evaluated in base 2 with the constants folded (F32): 13 ALU + 2 MUFU per coordinate.
  __device__ static float vterm(const F32& k, float x) {
    const float u1 = fmaf(x, k.c1, k.d1), u2 = fmaf(x, k.c2, k.d2);
    const float a = fmaf(-u1, u1, k.L1), b = fmaf(-u2, u2, k.L2);
    const float hi = fmaxf(a, b), lo = fminf(a, b);
    const float l = lg2f_approx(1.0f + exp2f_approx(lo - hi));
    return (hi + fmaf(k.kr * x, x, l)) * 0.69314718055994531f;
  }
  __device__ static float exp2f_approx(float v) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
  }
  __device__ static float lg2f_approx(float v) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
  }
  // f_beta(x) up to a beta-dependent constant: log eta + beta V
  __device__ static float f(const F32& k, float x) {
    const float sr = x * k.inv_r;
    return -0.5f * sr * sr + k.beta * vterm(k, x);
  }
  __device__ static float dlg(const F32& k, float x, float h) { return f(k, x + h) - f(k, x); }
  // gradient: grad log eta + beta (grad log_mix - grad log eta), responsibilities r1, 1 - r1
  __device__ static double grad64(const TgtParams& T, double beta, double x) {
    const double a = T.c[1] + lnpdf64(x, T.p[2], T.p[3], T.c[3]);
    const double b = T.c[2] + lnpdf64(x, T.p[4], T.p[5], T.c[4]);
    const double r1 = 1.0 / (1.0 + exp(b - a));
    const double glm = -(r1 * (x - T.p[2]) / (T.p[3] * T.p[3]) +
                         (1.0 - r1) * (x - T.p[4]) / (T.p[5] * T.p[5]));
    const double gref = -x / (T.p[0] * T.p[0]);
    return gref + beta * (glm - gref);
  }
  __device__ static float grad32(const F32& k, float x) {
    const float s1 = (x - k.mu1) * k.inv_s1;
    const float s2 = (x - k.mu2) * k.inv_s2;
    const float a = k.lw1 - 0.5f * s1 * s1;
    const float b = k.lw2 - 0.5f * s2 * s2;
    const float r1 = __frcp_rn(1.0f + exp2f_approx((b - a) * 1.4426950408889634f));
    const float glm = -(r1 * s1 * k.inv_s1 + (1.0f - r1) * s2 * k.inv_s2);
    const float gref = -x * k.inv_r * k.inv_r;
    return fmaf(k.beta, glm - gref, gref);
  }
  // difference form with the cached potential term v = vterm(x): one evaluation
  __device__ static float dlg_cached(const F32& k, float x, float v, float p) {
    return dlg_vv(k, x, v, p, vterm(k, p));
  }
  // the same with vterm(p) already evaluated: beta (vp - v) + (x^2 - p^2) / (2 r^2)
  __device__ static float dlg_vv(const F32& k, float x, float v, float p, float vp) {
    return fmaf(k.beta, vp - v, ((x - p) * k.hr) * (x + p));
  }
  __device__ static float vpart(const F32& k, float x) { return vterm(k, x); }
  __device__ static double v_from(const TgtParams&, double s) { return s; }
};

// ------------------------------------------------ ScaleGaussianTarget --
// N(0, s0^2 I) -> N(0, s1^2 I).  p = {s0, s1};
// c = {log s0, log s1, 1/s0^2, 1/s1^2, 0.5(1/s0^2 - 1/s1^2), log s1 - log s0}
struct TgtScale {
  static constexpr bool kExact = true;
  static constexpr bool kCacheV = false;
  __device__ static double lr64(const TgtParams& T, double x) {
    return lnpdf64(x, 0.0, T.p[0], T.c[0]);
  }
  __device__ static double v64(const TgtParams& T, double x) {
    return lnpdf64(x, 0.0, T.p[1], T.c[1]) - lnpdf64(x, 0.0, T.p[0], T.c[0]);
  }
  __device__ static double ref_draw(const TgtParams& T, double n) { return T.p[0] * n; }
  __device__ static float ref_draw32(const TgtParams& T, float n) { return (float)T.p[0] * n; }
  // ref_harness.cpp ScaleGaussianTarget::exact_sample: sd = 1/sqrt(tau), x = sd * normal
  __device__ static double exact_mu(const TgtParams& T, double beta) {
    const double tau = (1.0 - beta) / (T.p[0] * T.p[0]) + beta / (T.p[1] * T.p[1]);
    return 1.0 / sqrt(tau);
  }
  __device__ static double exact_draw(const TgtParams&, double sd, double n) { return sd * n; }
  // fp32 ----------------------------------------------------------------
  struct F32 {
    float tau;
  };
  __device__ static F32 f32(const TgtParams& T, double beta) {
    return F32{(float)((1.0 - beta) * T.c[2] + beta * T.c[3])};
  }
  // f(x+h) - f(x) = -tau h (x + h/2)
  __device__ static float dlg(const F32& k, float x, float h) {
    return -k.tau * h * (x + 0.5f * h);
  }
  __device__ static double grad64(const TgtParams& T, double beta, double x) {
    const double tau = (1.0 - beta) / (T.p[0] * T.p[0]) + beta / (T.p[1] * T.p[1]);
    return -tau * x;
  }
  __device__ static float grad32(const F32& k, float x) { return -k.tau * x; }
  __device__ static float vpart(const F32&, float x) { return x * x; }
  // early rejection: max over h of -tau h (x + h/2) = tau x^2 / 2
  static constexpr bool kEarly = true;
  static constexpr unsigned kCheckMask = 0x7Fu;  // early-rejection checks after quad-iterations 0..6
  static constexpr bool kPerProposalCheck = false;
  __device__ static float dmax(const F32& k, float x, float) { return 0.5f * k.tau * x * x; }
  // dmax summed over coordinates = (tau / 2) * sum vpart(x): the pass derives the bound of
  // the unprocessed coordinates from the carried vpart sum, no separate bound pass
  static constexpr bool kBoundFromV = true;
  __device__ static float bound_of_v(const F32& k, float v) { return 0.5f * k.tau * v; }
  // the MH log-ratio of a proposal x + s z as two running sums (2 FFMA per coordinate
  // instead of the 4 of sum dlg):  sum_i dlg(x_i, s z_i) = -tau (s A + s^2 B / 2),
  // A = sum z_i x_i, B = sum z_i^2 -- no cancellation between the terms
  static constexpr bool kQuadMH = true;
  __device__ static float dl_from(const F32& k, float s, float A, float B) {
    return -k.tau * s * fmaf(0.5f * s, B, A);
  }
  __device__ static double v_from(const TgtParams& T, double s) {
    return T.c[4] * s - (double)T.dim * T.c[5];
  }
};

}  // namespace asmcdev
