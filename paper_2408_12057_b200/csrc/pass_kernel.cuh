// The fused particle pass: for each particle, init from eta (or load the SSMC
// state), then for each annealing step t the incremental weight
// (beta_t - beta_{t-1}) V(x), the per-step log-moment accumulators and the
// MCMC move -- detail::weight_and_move (src/engine_detail.hpp:27-41) driven
// particle-outer as in run_sais_single (src/drivers.cpp:95-111) or one step
// at a time as in step_pass (src/engine_detail.hpp:113-156).
//
// Layout: one CTA = one 256-particle reduction block (kReductionBlock).  G
// lanes cooperate on one particle (G = 1, 4 or 32); the 256/G groups of the
// CTA walk G particles each, in lockstep, so every (particle-iteration, step)
// ends in one CTA reduction of the per-particle (log w, lg) pairs.  Particle
// coordinates live in registers (KMAX per lane) for the whole pass; the SAIS
// pass therefore moves no particle bytes through HBM at all.
//
// Arithmetic contracts:
//   Real = double: the reference's operation order (log_gamma = sum log-ref
//     terms + beta * sum potential terms; MH on absolute log densities), G = 1,
//     block accumulators added sequentially in particle order  -> agrees with
//     the unmodified reference to libm ulps.  Built with -fmad=false.
//   Real = float: fp32 positions, difference-form MH ratio, fp64 weights and
//     accumulators, fixed-tree block reductions.
#pragma once

#include "dev_common.cuh"
#include "rng.cuh"
#include "targets.cuh"

#include <type_traits>

namespace asmcdev {

constexpr double kTwoPi = 6.283185307179586476925286766559;

// kModeSaisFirst / kModeSaisNext: long-T SAIS in t-tiles (drivers.cpp:86-146 has no T
// cap): the first tile draws the particle and runs steps t_begin..t_end, later tiles
// reload it from the state rows; every tile stores it back.  Same per-(block, step)
// partials as one kModeSais launch over all T steps.
enum PassMode : int {
  kModeSais = 0, kModeSmcInit = 1, kModeSmcStep = 2, kModeTraj = 3, kModeSaisFirst = 4, kModeSaisNext = 5
};
__host__ __device__ __forceinline__ bool mode_loads(int m) { return m == kModeSmcStep || m == kModeSaisNext; }
__host__ __device__ __forceinline__ bool mode_stores(int m) {
  return m == kModeSmcStep || m == kModeSaisFirst || m == kModeSaisNext;
}
__host__ __device__ __forceinline__ int mode_nacc(int m) { return m == kModeSmcStep ? 6 : 4; }

struct KernelCfg {
  int kind;  // ASMC_KERNEL_*
  int n_steps;
  int sweeps;
  int leapfrog;  // HMC
  int no_early;  // test hook (env ASMC_NO_EARLY_REJECT=1): run every MH pass to the end
  int pad;
  double steps[ASMC_MAX_STEP_SIZES];
};

struct PassArgs {
  TgtParams tg;
  KernelCfg kc;
  const double* betas;  // device, T + 1
  int T;
  int t_begin, t_end;  // steps run by this launch (inclusive)
  int mode;
  int row_base;        // partial row = t - row_base
  int pad;
  uint64_t n;          // particles in the round
  uint64_t p_begin;    // global index of this launch's first particle
  uint64_t n_local;    // particles handled by this launch
  uint64_t seed, round;
  void* const* xbuf;   // SSMC state double buffer, particle-major [n_local * dim] Real
  const int* xcur;     // device index of the live buffer (flipped by resampling)
  double* lw;          // SSMC log-weights [n_local]
  LogAcc* part;        // block partials: part[(row * kNAcc + a) * part_stride + block]
  uint64_t part_stride;
  const uint64_t* pids;  // kModeTraj: particle ids
  double* rec_x;         // kModeTraj: [(i * (T+1) + t) * dim + k]
  double* rec_lw;        // kModeTraj: [i * (T+1) + t]
  int* err;
  // batched seeds (one-lane pass, SAIS): launch = nseeds x blocks_per_seed CTAs; seed
  // s uses seeds[s], betas + s * betas_stride and part + s * part_seed_stride
  const uint64_t* seeds;
  uint64_t blocks_per_seed, betas_stride, part_seed_stride;
  unsigned long long* drawn;  // profiling: normals actually generated (null = off)
  PhiloxRoundKeys rk[2];      // Philox round keys of (seed, round, substep 0 | 1): set at launch
  // SSMC step after a resampling event whose gather was deferred (*pend != 0): slot m
  // reads row anc[m] of the live buffer with log w = 0 and writes its row to the other
  // buffer (flipped after the pass) -- the gather's row copy fused into the step's loads
  const uint32_t* anc;
  const int* pend;
};

__device__ __forceinline__ bool pass_pending(const PassArgs& A) {
  return A.mode == kModeSmcStep && A.pend && *(volatile const int*)A.pend;
}

// coordinate owned by (lane, slot k): quads of 4 consecutive coordinates dealt
// round-robin over the G lanes (G = 1 gives k itself).
template <int G>
__device__ __forceinline__ int coord_of(int lane, int k) {
  return 4 * (lane + G * (k >> 2)) + (k & 3);
}

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int m = 1; m < G; m <<= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
template <int G>
__device__ __forceinline__ float group_sumf(float v) {
#pragma unroll
  for (int m = 1; m < G; m <<= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// ====================================================== fp64 reference path
template <class Tgt, class Seq, int KMAX>
struct Exact {
  // target.cpp:34-39: log_reference(x) + beta * potential(x), two ordered sums
  __device__ static double log_gamma(const TgtParams& T, int d, double beta, const double* x) {
    double L = 0.0;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
    for (int k = 0; k < KMAX; ++k)
      if (k < d) L += Tgt::lr64(T, x[k]);
    if (beta == 0.0) return L;
    double V = 0.0;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
    for (int k = 0; k < KMAX; ++k)
      if (k < d) V += Tgt::v64(T, x[k]);
    return L + beta * V;
  }

  __device__ static double potential(const TgtParams& T, int d, const double* x) {
    double V = 0.0;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
    for (int k = 0; k < KMAX; ++k)
      if (k < d) V += Tgt::v64(T, x[k]);
    return V;
  }

  __device__ static void init(const TgtParams& T, int d, double* x, Seq& st) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
    for (int k = 0; k < KMAX; ++k)
      if (k < d) x[k] = Tgt::ref_draw(T, (double)st.normal());
  }

  // kernel.cpp:65-73
  __device__ static double weight(const TgtParams& T, int d, double b0, double b1,
                                  const double* x, int* err) {
    const double from = log_gamma(T, d, b0, x);
    if (from == -__builtin_huge_val()) raise_error(err, ASMC_ERR_EVALUATION);
    return log_gamma(T, d, b1, x) - from;
  }

  // kernel.cpp:26-63
  __device__ static void move(const TgtParams& T, const KernelCfg& kc, int d, double beta,
                              double* x, double* prop, Seq& st) {
    if (kc.kind == ASMC_KERNEL_IDEALIZED) {
      const double mu = Tgt::exact_mu(T, beta);
#pragma unroll(KMAX <= 64 ? KMAX : 1)
      for (int k = 0; k < KMAX; ++k)
        if (k < d) x[k] = Tgt::exact_draw(T, mu, (double)st.normal());
      return;
    }
    if (kc.kind == ASMC_KERNEL_HMC) {
      // oracle/restate.c:hmc_cycle_move; product targets are separable, so each
      // coordinate's trajectory runs to completion before the next is drawn
      // (same draws, same per-coordinate arithmetic, same summation order).
      double lgx = log_gamma(T, d, beta, x);
      for (int sw = 0; sw < kc.sweeps; ++sw) {
        for (int si = 0; si < kc.n_steps; ++si) {
          const double eps = kc.steps[si];
          double k0 = 0.0, k1 = 0.0;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
          for (int k = 0; k < KMAX; ++k) {
            if (k < d) {
              double p = (double)st.normal();
              k0 += p * p;
              double xx = x[k];
              double g = Tgt::grad64(T, beta, xx);
              for (int l = 0; l < kc.leapfrog; ++l) {
                p += 0.5 * eps * g;
                xx += eps * p;
                g = Tgt::grad64(T, beta, xx);
                p += 0.5 * eps * g;
              }
              k1 += p * p;
              prop[k] = xx;
            }
          }
          const double lgp = log_gamma(T, d, beta, prop);
          const double log_u = log(st.uniform());
          if (log_u < (lgp - lgx) + 0.5 * (k0 - k1)) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
            for (int k = 0; k < KMAX; ++k)
              if (k < d) x[k] = prop[k];
            lgx = lgp;
          }
        }
      }
      return;
    }
    if (kc.kind == ASMC_KERNEL_SLICE) {
      // oracle/restate.c:slice_move: elliptical slice w.r.t. eta = N(mu, sigma^2 I)
      const double mu = Tgt::ref_draw(T, 0.0);
      double nu[KMAX];
      for (int sw = 0; sw < kc.sweeps; ++sw) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
        for (int k = 0; k < KMAX; ++k)
          if (k < d) nu[k] = Tgt::ref_draw(T, (double)st.normal());
        const double ll = beta == 0.0 ? 0.0 : beta * potential(T, d, x);
        const double log_y = ll + log(st.uniform());
        double theta = st.uniform() * kTwoPi;
        double lo = theta - kTwoPi, hi = theta;
        for (int it = 0; it < ASMC_SLICE_MAX_SHRINK; ++it) {
          const double c = cos(theta), sn = sin(theta);
#pragma unroll(KMAX <= 64 ? KMAX : 1)
          for (int k = 0; k < KMAX; ++k)
            if (k < d) prop[k] = mu + (x[k] - mu) * c + (nu[k] - mu) * sn;
          const double llp = beta == 0.0 ? 0.0 : beta * potential(T, d, prop);
          if (llp > log_y) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
            for (int k = 0; k < KMAX; ++k)
              if (k < d) x[k] = prop[k];
            break;
          }
          if (theta < 0.0) lo = theta;
          else hi = theta;
          theta = lo + (hi - lo) * st.uniform();
        }
      }
      return;
    }
    if (kc.kind != ASMC_KERNEL_RWMH) return;
    double lgx = log_gamma(T, d, beta, x);
    for (int sw = 0; sw < kc.sweeps; ++sw) {
      for (int si = 0; si < kc.n_steps; ++si) {
        const double s = kc.steps[si];
#pragma unroll(KMAX <= 64 ? KMAX : 1)
        for (int k = 0; k < KMAX; ++k)
          if (k < d) prop[k] = x[k] + s * (double)st.normal();
        const double lgp = log_gamma(T, d, beta, prop);
        const double log_u = log(st.uniform());
        if (log_u < lgp - lgx) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
          for (int k = 0; k < KMAX; ++k)
            if (k < d) x[k] = prop[k];
          lgx = lgp;
        }
      }
    }
  }
};

// ======================================================= fp32 fast path
// Normal source: G == 1 -> sequential stream object (xoshiro or Philox);
// G > 1 -> Philox random access (normal #j of the (p, t) stream).
template <class Tgt, int RNG, int G, int KMAX>
struct Fast {
  using Seq = typename std::conditional<RNG == ASMC_RNG_XOSHIRO, XoSeq<float>, PhSeq<float>>::type;
  static constexpr bool kSeq = (G == 1);

  struct Src {
    Seq seq;      // G == 1
    PhiloxKey ph; // G > 1
    __device__ void init(uint64_t seed, uint64_t round, uint64_t pid, uint64_t step, uint64_t sub) {
      if constexpr (kSeq) seq.init(seed, round, pid, step, sub);
      else ph.init(seed, round, pid, step, sub);
    }
  };

  __device__ static bool valid(int lane, int k, int d) { return coord_of<G>(lane, k) < d; }

  __device__ static void init(const TgtParams& T, int lane, int d, float* x, Src& src) {
    if constexpr (kSeq) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
      for (int k = 0; k < KMAX; ++k)
        x[k] = k < d ? (float)Tgt::ref_draw(T, (double)src.seq.normal()) : 0.0f;
    } else {
#pragma unroll
      for (int m = 0; m < KMAX / 4; ++m) {
        float q[4] = {0.f, 0.f, 0.f, 0.f};
        if (4 * (lane + G * m) < d) quad(src, lane, m, 0, q);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          x[4 * m + e] = valid(lane, 4 * m + e, d) ? (float)Tgt::ref_draw(T, (double)q[e]) : 0.0f;
      }
    }
  }

  // (b1 - b0) V(x); V from per-lane fp32 partial sums combined in fp64
  __device__ static double weight(const TgtParams& T, int lane, int d, double b0, double b1,
                                  const float* x) {
    const typename Tgt::F32 k0 = Tgt::f32(T, b1);
    float s = 0.0f;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
    for (int k = 0; k < KMAX; ++k)
      if (valid(lane, k, d)) s += Tgt::vpart(k0, x[k]);
    const double V = Tgt::v_from(T, group_sum<G>((double)s));
    return (b1 - b0) * V;
  }

  // one quad of normals (coordinates 4*(lane+G*m) .. +3) of the draw set at `base`
  __device__ static void quad(const Src& src, int lane, int m, uint64_t base, float q[4]) {
    const uint64_t j0 = base + 4 * (uint64_t)(lane + G * m);
    if ((base & 3) == 0) src.ph.template normals4<float>((uint32_t)(j0 >> 2), q);
    else src.ph.template normals4_at<float>(j0, q);
  }

  // kernel.cpp:26-42 in fp32 difference form.  G == 1 keeps the proposal in
  // registers; G > 1 (counter-based normals) regenerates the accepted
  // proposal's normals instead, so a lane holds only its x slice.
  __device__ static void move(const TgtParams& T, const KernelCfg& kc, int lane, int d,
                              double beta, float* x, Src& src) {
    if (kc.kind == ASMC_KERNEL_IDEALIZED) {
      const double mu = Tgt::exact_mu(T, beta);
      if constexpr (kSeq) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
        for (int k = 0; k < KMAX; ++k)
          if (k < d) x[k] = (float)Tgt::exact_draw(T, mu, (double)src.seq.normal());
      } else {
#pragma unroll
        for (int m = 0; m < KMAX / 4; ++m) {
          if (4 * (lane + G * m) >= d) continue;
          float q[4];
          quad(src, lane, m, 0, q);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (valid(lane, 4 * m + e, d)) x[4 * m + e] = (float)Tgt::exact_draw(T, mu, (double)q[e]);
        }
      }
      return;
    }
    if (kc.kind == ASMC_KERNEL_HMC) {  // one lane per particle (G > 1 runs pass_smem)
      if constexpr (kSeq) {
        const typename Tgt::F32 kf = Tgt::f32(T, beta);
        for (int sw = 0; sw < kc.sweeps; ++sw) {
          for (int si = 0; si < kc.n_steps; ++si) {
            const float eps = (float)kc.steps[si], he = 0.5f * eps;
            float prop[KMAX];
            float dl = 0.0f;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
            for (int k = 0; k < KMAX; ++k) {
              if (k < d) {
                const float p0 = src.seq.normal();
                float p = p0, xx = x[k], g = Tgt::grad32(kf, xx);
                for (int l = 0; l < kc.leapfrog; ++l) {
                  p = fmaf(he, g, p);
                  xx = fmaf(eps, p, xx);
                  g = Tgt::grad32(kf, xx);
                  p = fmaf(he, g, p);
                }
                dl += Tgt::dlg(kf, x[k], xx - x[k]) + 0.5f * (p0 - p) * (p0 + p);
                prop[k] = xx;
              }
            }
            if (log(src.seq.uniform()) < (double)dl) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
              for (int k = 0; k < KMAX; ++k)
                if (k < d) x[k] = prop[k];
            }
          }
        }
      }
      return;
    }
    if (kc.kind == ASMC_KERNEL_SLICE) {  // elliptical slice, one lane per particle
      if constexpr (kSeq) {
        const typename Tgt::F32 kb = Tgt::f32(T, beta), k0 = Tgt::f32(T, 0.0);
        const float mu = (float)Tgt::ref_draw(T, 0.0);
        for (int sw = 0; sw < kc.sweeps; ++sw) {
          float nu[KMAX], prop[KMAX];
#pragma unroll(KMAX <= 64 ? KMAX : 1)
          for (int k = 0; k < KMAX; ++k)
            if (k < d) nu[k] = (float)Tgt::ref_draw(T, (double)src.seq.normal());
          const double log_u = log(src.seq.uniform());
          double theta = src.seq.uniform() * kTwoPi;
          double lo = theta - kTwoPi, hi = theta;
          for (int it = 0; it < ASMC_SLICE_MAX_SHRINK; ++it) {
            const float c = (float)cos(theta), sn = (float)sin(theta);
            float dl = 0.0f;  // beta (V(x') - V(x)) as a difference of log-density differences
#pragma unroll(KMAX <= 64 ? KMAX : 1)
            for (int k = 0; k < KMAX; ++k) {
              if (k < d) {
                const float xp = mu + (x[k] - mu) * c + (nu[k] - mu) * sn;
                const float h = xp - x[k];
                dl += Tgt::dlg(kb, x[k], h) - Tgt::dlg(k0, x[k], h);
                prop[k] = xp;
              }
            }
            if ((double)dl > log_u) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
              for (int k = 0; k < KMAX; ++k)
                if (k < d) x[k] = prop[k];
              break;
            }
            if (theta < 0.0) lo = theta;
            else hi = theta;
            theta = lo + (hi - lo) * src.seq.uniform();
          }
        }
      }
      return;
    }
    if (kc.kind != ASMC_KERNEL_RWMH) return;
    const typename Tgt::F32 kf = Tgt::f32(T, beta);
    const int nq = kc.sweeps * kc.n_steps;
    double lu_pre = 0.0;  // G > 1: lane l holds log u of proposal (q0 + l)
    for (int q = 0; q < nq; ++q) {
      const float s = (float)kc.steps[q % kc.n_steps];
      const uint64_t base = (uint64_t)q * (uint64_t)d;
      if constexpr (kSeq) {
        float prop[KMAX];
        float dl = 0.0f;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
        for (int k = 0; k < KMAX; ++k) {
          if (k < d) {
            const float h = s * src.seq.normal();
            prop[k] = x[k] + h;
            dl += Tgt::dlg(kf, x[k], h);
          }
        }
        const double log_u = log(src.seq.uniform());
        if (log_u < (double)dl) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
          for (int k = 0; k < KMAX; ++k)
            if (k < d) x[k] = prop[k];
        }
      } else {
        if ((q % G) == 0) {
          const int qq = q + lane;
          lu_pre = qq < nq ? log(src.ph.uniform((uint32_t)qq)) : 0.0;
        }
        float dl = 0.0f;
#pragma unroll
        for (int m = 0; m < KMAX / 4; ++m) {
          if (4 * (lane + G * m) >= d) continue;
          float z[4];
          quad(src, lane, m, base, z);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (valid(lane, 4 * m + e, d)) dl += Tgt::dlg(kf, x[4 * m + e], s * z[e]);
        }
        const double delta = group_sum<G>((double)dl);
        const double log_u =
            __shfl_sync(0xffffffffu, lu_pre, (int)(threadIdx.x & 31 & ~(G - 1)) + (q % G));
        if (log_u < delta) {
#pragma unroll
          for (int m = 0; m < KMAX / 4; ++m) {
            if (4 * (lane + G * m) >= d) continue;
            float z[4];
            quad(src, lane, m, base, z);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (valid(lane, 4 * m + e, d)) x[4 * m + e] += s * z[e];
          }
        }
      }
    }
  }
};

// ============================================================ reductions
// Per-step CTA reduction of the groups' (pre-update log w, lg, post log w)
// into accumulator a, combined into the block partial across iterations r.
template <bool kExactOrder, int NG, bool kChain = false>
__device__ void block_reduce(const double* s_lw, const double* s_lg, const double* s_post,
                             const int* s_act, int nacc, LogAcc* dst, bool first) {
  const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  if constexpr (kExactOrder) {
    // engine_detail.hpp:122-140 / drivers.cpp:95-111: sequential in particle order.
    // lacc_add / sacc_add need, per element, only the running max BEFORE it: that is an
    // exclusive prefix max, so the block scans it in parallel and every thread computes
    // its element's exp (the same argument, the same exp -> the same bits); one thread
    // per accumulator then replays the particle-order chain of adds, which is now only
    // FADD/FMA (no exp on the sequential path).  Called by all NG == blockDim threads.
    static_assert(NG == kBlock, "exact-order fold: one thread per particle of the block");
    constexpr int kL = kAccTop2;  // log-sum accumulators g0, g1, g2, elbo, sq
    // kChain (register-resident instantiations): element q's add as sum <- sum * m + a in
    // two roundings -- below the running max (m, a) = (1, sign e), the reference's
    // sum += e; a new max (e, sign), its sum = sum e + 1; skipped (1, -0), an identity --
    // a branch-free chain.  Otherwise the chain branches on the flag and reads e (half
    // the shared memory for the local-memory instantiations).
    struct ChainS {
      double m[kL][NG], a[kL][NG];
    };
    struct FlagS {
      double e[kL][NG];
    };
    __shared__ typename std::conditional<kChain, ChainS, FlagS>::type S;
    __shared__ unsigned char s_f[kL][NG];  // 0 = skipped, 1 = below the running max, 2 = new max
    __shared__ double s_wmax[NG / 32][kL];
    const int g = threadIdx.x;
    const double lw = s_lw[g], lg = s_lg[g], post = s_post[g];
    const bool act = s_act[g] != 0;
    double l[kL], sg[kL];
#pragma unroll
    for (int k = 0; k < kL; ++k) sg[k] = 1.0;
    l[kAccG0] = lw;
    l[kAccG1] = lw + lg;
    l[kAccG2] = lw + 2.0 * lg;
    l[kAccElbo] = lg != 0.0 ? lw + log(fabs(lg)) : -__builtin_huge_val();
    sg[kAccElbo] = lg > 0.0 ? 1.0 : -1.0;
    l[kAccSq] = 2.0 * post;
    const int nl = nacc < kL ? nacc : kL;
    double inc[kL];
#pragma unroll
    for (int k = 0; k < kL; ++k) {
      if (!act) l[k] = -__builtin_huge_val();
      inc[k] = l[k];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, inc[k], off);
        if (ln >= off) inc[k] = fmax(inc[k], o);
      }
      if (ln == 31) s_wmax[warp][k] = inc[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kL; ++k) {
      double pre = -__builtin_huge_val();  // max over the earlier warps
      for (int w = 0; w < warp; ++w) pre = fmax(pre, s_wmax[w][k]);
      const double up = __shfl_up_sync(0xffffffffu, inc[k], 1);
      const double ex = ln == 0 ? pre : fmax(pre, up);  // running max before element g
      if (k >= nl || l[k] == -__builtin_huge_val()) {
        s_f[k][g] = 0;
        if constexpr (kChain) {
          S.m[k][g] = 1.0;
          S.a[k][g] = -0.0;
        } else {
          S.e[k][g] = 0.0;
        }
      } else {
        const bool below = l[k] <= ex;
        const double e = exp(below ? l[k] - ex : ex - l[k]);
        s_f[k][g] = below ? 1 : 2;
        if constexpr (kChain) {
          S.m[k][g] = below ? 1.0 : e;
          S.a[k][g] = below ? sg[k] * e : sg[k];
        } else {
          S.e[k][g] = e;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < nacc) {
      const int a = threadIdx.x;
      LogAcc acc = (a == kAccTop2) ? LogAcc{-__builtin_huge_val(), -__builtin_huge_val()} : lacc_empty();
      if (a == kAccTop2) {
        for (int q = 0; q < NG; ++q)
          if (s_act[q]) top2_add(acc, s_post[q]);
      } else {
        // the particle-order chain
        double sum = 0.0;
        int qlast = -1;  // the last new max: the accumulator's max after the block
        if constexpr (kChain) {
#pragma unroll 8
          for (int q = 0; q < NG; ++q) {
            sum = __dadd_rn(__dmul_rn(sum, S.m[a][q]), S.a[a][q]);
            qlast = s_f[a][q] == 2 ? q : qlast;
          }
        } else {
          for (int q = 0; q < NG; ++q) {
            const unsigned char f = s_f[a][q];
            if (f == 0) continue;
            const double sq = a == kAccElbo ? (s_lg[q] > 0.0 ? 1.0 : -1.0) : 1.0;
            if (f == 1) {
              sum = __dadd_rn(sum, __dmul_rn(sq, S.e[a][q]));
            } else {
              sum = __dadd_rn(__dmul_rn(sum, S.e[a][q]), sq);
              qlast = q;
            }
          }
        }
        double mx = -__builtin_huge_val();
        if (qlast >= 0) {
          const int q = qlast;
          mx = a == kAccG0 ? s_lw[q]
               : a == kAccG1 ? s_lw[q] + s_lg[q]
               : a == kAccG2 ? s_lw[q] + 2.0 * s_lg[q]
               : a == kAccElbo ? s_lw[q] + log(fabs(s_lg[q]))
                               : 2.0 * s_post[q];
        }
        acc = LogAcc{mx, sum};
      }
      if (first) dst[a] = acc;
      else acc_merge(a, dst[a], acc);
    }
    return;
  }
  if (warp < nacc) {
    const int a = warp;
    LogAcc acc = (a == kAccTop2) ? LogAcc{-__builtin_huge_val(), -__builtin_huge_val()} : lacc_empty();
    constexpr int per = NG >= 32 ? NG / 32 : 1;
    const int g0 = NG >= 32 ? ln * per : ln;
    if (NG >= 32 || ln < NG) {
#pragma unroll
      for (int e = 0; e < per; ++e) {
        const int g = g0 + e;
        if (!s_act[g]) continue;
        const double lw = s_lw[g], lg = s_lg[g];
        switch (a) {
          case kAccG0: lacc_add(acc, lw); break;
          case kAccG1: lacc_add(acc, lw + lg); break;
          case kAccG2: lacc_add(acc, lw + 2.0 * lg); break;
          case kAccElbo:
            if (lg != 0.0) sacc_add(acc, lw + log(fabs(lg)), lg > 0.0 ? 1.0 : -1.0);
            break;
          case kAccSq: lacc_add(acc, 2.0 * s_post[g]); break;
          default: top2_add(acc, s_post[g]); break;
        }
      }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const LogAcc o = shfl_xor_acc(acc, m);
      if (a == kAccTop2) top2_merge(acc, o);
      else lacc_combine(acc, o);
    }
    if (ln == 0) {
      if (first) dst[a] = acc;
      else acc_merge(a, dst[a], acc);
    }
  }
}

// =============================================================== kernel
// small-dimension (register-resident, KMAX = 16) instantiations: 2 CTAs per SM, so a
// round of up to 296 blocks (~76k particles) is resident at once (config 1's rounds are
// 64-182 blocks: with one 236-register CTA per SM its last round ran in two waves); the
// local-memory (KMAX = 1024) ones 3 per SM (they otherwise drift to 120 registers, 2 per
// SM: 1.0e7 -> 7.7e6 p-steps/s on config 2's shape in reference arithmetic)
template <class Tgt, int RNG, typename Real, int G, int KMAX>
__global__ void __launch_bounds__(kBlock, KMAX <= 16 ? 2 : 3) pass_kernel(const __grid_constant__ PassArgs A) {
  constexpr int NG = kBlock / G;
  constexpr bool kExact = std::is_same<Real, double>::value;
  static_assert(!kExact || G == 1, "reference-order path is one lane per particle");
  const int tid = threadIdx.x, g = tid / G, lane = tid % G;
  const int d = (int)A.tg.dim;
  const uint64_t bps = A.blocks_per_seed ? A.blocks_per_seed : gridDim.x;
  const uint64_t si = blockIdx.x / bps;  // batched seeds: this CTA's seed (0 otherwise)
  const uint64_t blk = blockIdx.x % bps;
  const uint64_t seed = A.seeds ? A.seeds[si] : A.seed;
  const double* betas = A.betas + si * A.betas_stride;
  LogAcc* part = A.part + si * A.part_seed_stride;
  const int nacc = mode_nacc(A.mode);
  if (block_err_set(A.err)) return;  // an earlier step failed: skip the work

  __shared__ double s_lw[NG], s_lg[NG], s_post[NG];
  __shared__ int s_act[NG];
  __shared__ LogAcc s_dst[kNAcc];

  using SeqT = typename std::conditional<RNG == ASMC_RNG_XOSHIRO, XoSeq<Real>, PhSeq<Real>>::type;
  using FastT = Fast<Tgt, RNG, G, KMAX>;
  using ExactT = Exact<Tgt, SeqT, KMAX>;

  const bool pend = pass_pending(A);
  for (int r = 0; r < G; ++r) {
    const uint64_t local = blk * kBlock + (uint64_t)r * NG + g;
    const bool active = local < A.n_local;
    const uint64_t pid = A.mode == kModeTraj ? (active ? A.pids[local] : 0) : A.p_begin + local;
    Real x[KMAX];
    double lw = 0.0;

    // ---- init / load -----------------------------------------------------
    if (mode_loads(A.mode)) {
      const uint64_t row = (pend && active) ? (uint64_t)A.anc[local] : local;
      const Real* xs = reinterpret_cast<const Real*>(A.xbuf[*A.xcur]) + row * (uint64_t)d;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
      for (int k = 0; k < KMAX; ++k) {
        const int i = coord_of<G>(lane, k);
        x[k] = (active && i < d) ? xs[i] : (Real)0;
      }
      lw = (active && !pend) ? A.lw[local] : 0.0;
    } else {
      if constexpr (kExact) {
        SeqT st;
        st.init(seed, A.round, pid, 0, 0);
        ExactT::init(A.tg, d, x, st);
      } else {
        typename FastT::Src src;
        src.init(seed, A.round, pid, 0, 0);
        FastT::init(A.tg, lane, d, x, src);
      }
    }
    if (A.mode == kModeSmcInit) {
      if (active) {
        Real* xs = reinterpret_cast<Real*>(A.xbuf[*A.xcur]) + local * (uint64_t)d;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
        for (int k = 0; k < KMAX; ++k) {
          const int i = coord_of<G>(lane, k);
          if (i < d) xs[i] = x[k];
        }
        if (lane == 0) A.lw[local] = 0.0;
      }
      continue;
    }
    if (A.mode == kModeTraj && active) {
      double* rx = A.rec_x + (local * (uint64_t)(A.T + 1)) * d;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
      for (int k = 0; k < KMAX; ++k) {
        const int i = coord_of<G>(lane, k);
        if (i < d) rx[i] = (double)x[k];
      }
      if (lane == 0) A.rec_lw[local * (uint64_t)(A.T + 1)] = 0.0;
    }

    // ---- annealing steps -----------------------------------------------------
    for (int t = A.t_begin; t <= A.t_end; ++t) {
      const double b0 = betas[t - 1], b1 = betas[t];
      double lg;
      if constexpr (kExact) {
        Real prop[KMAX];
        lg = ExactT::weight(A.tg, d, b0, b1, x, A.err);
        SeqT st;
        st.init(seed, A.round, pid, (uint64_t)t, 1);
        ExactT::move(A.tg, A.kc, d, b1, x, prop, st);
      } else {
        lg = FastT::weight(A.tg, lane, d, b0, b1, x);
        typename FastT::Src src;
        src.init(seed, A.round, pid, (uint64_t)t, 1);
        FastT::move(A.tg, A.kc, lane, d, b1, x, src);
      }
      const double pre = lw;
      lw += lg;

      if (A.mode == kModeTraj) {
        if (active) {
          double* rx = A.rec_x + (local * (uint64_t)(A.T + 1) + t) * d;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
          for (int k = 0; k < KMAX; ++k) {
            const int i = coord_of<G>(lane, k);
            if (i < d) rx[i] = (double)x[k];
          }
          if (lane == 0) A.rec_lw[local * (uint64_t)(A.T + 1) + t] = lw;
        }
        continue;
      }
      if (lane == 0) {
        s_lw[g] = pre;
        s_lg[g] = lg;
        s_post[g] = lw;
        s_act[g] = active ? 1 : 0;
      }
      __syncthreads();
      const bool first = (r == 0);
      if (!first && tid < nacc) {
        s_dst[tid] = part[((size_t)(t - A.row_base) * kNAcc + tid) * A.part_stride + blk];
      }
      __syncthreads();
      block_reduce<kExact, NG, (KMAX <= 16)>(s_lw, s_lg, s_post, s_act, nacc, s_dst, first);
      __syncthreads();
      if (tid < nacc) part[((size_t)(t - A.row_base) * kNAcc + tid) * A.part_stride + blk] = s_dst[tid];
    }

    if (mode_stores(A.mode) && active) {
      Real* xs = reinterpret_cast<Real*>(A.xbuf[*A.xcur ^ (pend ? 1 : 0)]) + local * (uint64_t)d;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
      for (int k = 0; k < KMAX; ++k) {
        const int i = coord_of<G>(lane, k);
        if (i < d) xs[i] = x[k];
      }
      if (lane == 0) A.lw[local] = lw;
    }
  }
}

}  // namespace asmcdev
